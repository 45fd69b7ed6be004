set -x
bash tools/jobs/final.sh
for c in c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --build-breakdown --gt-queries 1000 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"
done
BENCH_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
