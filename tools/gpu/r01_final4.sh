OUT=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $OUT/final4_tests.log 2>&1; tail -2 $OUT/final4_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > $OUT/bench_v21.json 2> $OUT/bench_v21.err; tail -2 $OUT/bench_v21.err
