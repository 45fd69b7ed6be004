# every BASELINE config through bench.py (no CPU baseline), C3 with it
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
for c in c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --build-breakdown --gt-queries 1000 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"
done
