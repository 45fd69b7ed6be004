set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
for c in c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --build-breakdown --gt-queries 1000 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3q.json 2> gpurun_out/bench_c3q.err; echo "c3 rc=$?"
for f in bench_c4 bench_c5 bench_c3q; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d['ms_per_step'], d['e2e']['value'], d['quality']['recall_at_10'], d['roofline']['kernel'], d['roofline']['frac'], d['stage_ms_per_step'])"; done
