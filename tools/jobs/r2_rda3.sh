set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
IVRQ_KERNEL_TIMING=1 timeout 300 python tools/prof_search.py --config c3 --nprobe 8 --reps 4 2>&1 | grep -E "step|_kernel|Error" | tail -6
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print(d['value'], d['ms_per_step'], d['e2e'], d['stage_ms_per_step'], d['quality']['recall_at_10'])"
