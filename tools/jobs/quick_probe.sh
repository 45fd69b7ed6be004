set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "probe or select" > gpurun_out/gpu_tests_probe.log 2>&1; tail -15 gpurun_out/gpu_tests_probe.log
timeout 600 python tools/prof_search.py --config c3 --nprobe 8 --reps 3 2>&1 | grep step
timeout 600 python tools/prof_search.py --config c4 --nprobe 64 --reps 2 2>&1 | grep step
