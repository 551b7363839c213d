OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; tail -2 $OUT/smoke.log
python tools/c4_sweep.py > $OUT/c4_v2.jsonl 2> $OUT/c4_v2.err; tail -3 $OUT/c4_v2.err; wc -l $OUT/c4_v2.jsonl
timeout 900 python bench.py > $OUT/bench_v17.json 2> $OUT/bench_v17.err; tail -4 $OUT/bench_v17.err
