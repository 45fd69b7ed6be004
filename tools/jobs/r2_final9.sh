set -x
for c in c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --build-breakdown --gt-queries 1000 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
done
timeout 600 python bench.py --mode lut --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_lut.json 2>/dev/null; echo "lut rc=$?"
for f in bench_c1 bench_c2 bench_c4 bench_c5 bench_c3_lut; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); r=d['roofline']; print('$f', round(d['value']), d['ms_per_step'], round(d['e2e']['value']), d['quality']['recall_at_10'], d['build']['seconds'], r['kernel'], r['kernel_ms_per_launch'], r['frac'])"; done
