set -x
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/e2e_probe.py --config c3 --nprobe 8 > gpurun_out/e2e_probe.log 2>&1; echo "e2e rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^(scan_kernel|first_list_kernel)" -s 4 -c 2 -o gpurun_out/prof_scan_c3_r1c python tools/prof_search.py --config c3 --nprobe 8 > gpurun_out/prof.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_search.csv python tools/prof_search.py --config c3 --nprobe 8 --reps 2 > gpurun_out/prof2.log 2>&1; echo "launches rc=$?"
