# round-end records on the final code (re-entry session): suite, smoke, every configuration,
# reference arm, LUT mode, e2e pipeline A/B, bench launch list, scan traffic, full capture
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --mode lut --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_lut.json 2>/dev/null; echo "lut rc=$?"
for c in c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --build-breakdown --gt-queries 1000 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
done
timeout 300 python tools/e2e_ab.py --threads 8 --pieces 1,2,4,8 > gpurun_out/e2e_ab.log 2>&1; grep -E "threads|timeline" gpurun_out/e2e_ab.log
BENCH_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_c3.csv python tools/prof_search.py --config c3 --nprobe 8 --reps 1 > /dev/null 2>&1; echo "traffic rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"tc_refine|scan_rda" -c 2 -o gpurun_out/prof_c3_final python tools/prof_search.py --config c3 --nprobe 8 --reps 1 > /dev/null 2>&1; echo "ncu full rc=$?"
for f in bench_default bench_c3_lut bench_c1 bench_c2 bench_c4 bench_c5; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d['ms_per_step'], d['e2e']['value'], d['quality']['recall_at_10'], d['roofline']['kernel'], d['roofline']['bound'], d['roofline']['frac'])"; done
