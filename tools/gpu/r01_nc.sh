OUT=gpurun_out
timeout 900 python bench.py --no-e2e --no-cpu-baseline > $OUT/bench_nc.json 2> $OUT/bench_nc.err; tail -4 $OUT/bench_nc.err
python -c "import json;d=json.load(open('$OUT/bench_nc.json'));print(d['value'],d['ms_per_step'],d['trmm']['ms_per_step'],d['fp32']['ms_per_step'])"
python tools/small_probe.py trmm f64 4096,8192
