# front pipelining iteration: GPU suite, C3 bench, e2e A/B
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print(d['value'], d['ms_per_step'], d['e2e'], d['stage_ms_per_step'])"
IVRQ_KERNEL_TIMING=1 timeout 300 python tools/prof_search.py --config c3 --nprobe 8 --reps 3 2>&1 | grep -E "step|Error" | tail -3
for pc in 1 2 4 8; do IVRQ_STAGE_PIECES=$pc timeout 300 python tools/prof_search.py --config c3 --nprobe 8 --reps 3 2>&1 | grep -E "step|Error" | tail -1; done
timeout 300 python tools/e2e_ab.py --threads 8 --pieces 2,4 > gpurun_out/e2e_ab.log 2>&1; grep -E "threads|timeline" gpurun_out/e2e_ab.log
