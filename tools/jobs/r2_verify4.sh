# copy-out on native threads, sanitizers on the final kernels, probe / final-pass captures
set -x
timeout 600 python -m pytest tests -m gpu -x -q -k "search_batch or smoke or end_to_end or acceptance" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 300 python tools/e2e_ab.py --threads 8 --pieces 4 > gpurun_out/e2e_ab2.log 2>&1; grep -E "setup|threads|timeline" gpurun_out/e2e_ab2.log
bash tools/jobs/r2_sanitize.sh
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"probe_rescore|rda_final" -c 2 -o gpurun_out/prof_c3_probe python tools/prof_search.py --config c3 --nprobe 8 --reps 1 > /dev/null 2>&1; echo "ncu rc=$?"
