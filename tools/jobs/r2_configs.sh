# every BASELINE config through bench.py (C3 twice for noise), LUT at C3
for c in c3 c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --build-breakdown --gt-queries 1000 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"; python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', d['value'], d['ms_per_step'], d['e2e']['value'], d['quality']['recall_at_10'], d['build']['seconds'], d['stage_ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'])"
done
