set -x
timeout 600 python bench.py --mode lut --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_lut.json 2>/dev/null; echo "lut rc=$?"
for c in c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --build-breakdown --gt-queries 1000 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
done
for f in bench_c3_lut bench_c4 bench_c5; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d['ms_per_step'], d['e2e']['value'], d['quality']['recall_at_10'], d['roofline']['kernel'], d['roofline']['frac'], d['stage_ms_per_step'])"; done
