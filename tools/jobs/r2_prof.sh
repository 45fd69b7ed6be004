# CLI GPU tests, tc_refine wait-cycle counters, full ncu capture of tc_refine at C3
set -x
timeout 600 python -m pytest tests/test_cli.py -m gpu -x -q > gpurun_out/cli_tests.log 2>&1; echo "cli rc=$?"; tail -15 gpurun_out/cli_tests.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"^(tc_refine_kernel)" -c 1 \
   -o gpurun_out/prof_refine_c3_r2 python tools/prof_search.py --config c3 --nprobe 8 --reps 1 > /dev/null 2>&1; echo "ncu rc=$?"
bash tools/jobs/tc_prof.sh
