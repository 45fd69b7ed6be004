# iteration: GPU tests (fail fast), C3 search timing with kernel events, short bench
set -x
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -30 gpurun_out/gpu_tests.log | grep -vE "^\s*$" | tail -25
IVRQ_KERNEL_TIMING=1 timeout 600 python tools/prof_search.py --config ${CFG:-c3} --nprobe ${NPROBE:-8} --reps 3 2>&1 | grep -E "step ms|tc_|scan_|Error|error" | tail -6
