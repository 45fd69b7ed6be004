set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "probe or select or golden or search" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
for c in "c3 8" "c4 64" "c5 32"; do set -- $c; timeout 300 python tools/prof_search.py --config $1 --nprobe $2 --reps 4 2>&1 | grep -E "step|Error" | tail -1; done
