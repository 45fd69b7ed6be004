# GPU tests, then C4/C5 search stage timings and the C3 bench line
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
for c in "c4 64" "c5 32"; do
  set -- $c
  timeout 600 python tools/prof_search.py --config $1 --nprobe $2 --reps 3 > gpurun_out/ps_$1.log 2>&1; grep -E "step|Error" gpurun_out/ps_$1.log | tail -3
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 600 gpurun_out/bench_c3.json
