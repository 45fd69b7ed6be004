set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 300 python tools/prof_search.py --config c3 --nprobe 8 --reps 5 2>&1 | grep -E "step|Error" | tail -2
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cs.csv -k regex:"cs_" python tools/prof_search.py --config c3 --nprobe 8 --reps 2 > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/launches_cs.csv | head -8
