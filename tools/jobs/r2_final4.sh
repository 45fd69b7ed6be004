# probe changes: suite, then the records they move (C3 default, C1, C2, C4, C5, launch list)
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -2 gpurun_out/gpu_tests.log
[ $rc -eq 0 ] || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
for c in c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --build-breakdown --gt-queries 1000 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
done
timeout 600 python bench.py --mode lut --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_lut.json 2>/dev/null; echo "lut rc=$?"
BENCH_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
for f in bench_default bench_c3_lut bench_c1 bench_c2 bench_c4 bench_c5; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d['ms_per_step'], d['e2e']['value'], d['quality']['recall_at_10'], d['roofline']['kernel'], d['roofline']['frac'], d['stage_ms_per_step'])"; done
