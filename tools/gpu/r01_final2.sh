OUT=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 > $OUT/final2_tests.log 2>&1; tail -2 $OUT/final2_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > $OUT/bench_v18.json 2> $OUT/bench_v18.err; tail -3 $OUT/bench_v18.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file $OUT/r01_launches_bench_v5.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-cublas --no-trmm --no-fp32 > /dev/null 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2>/dev/null; cat $OUT/bench_ref.json | cut -c1-300
