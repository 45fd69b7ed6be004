timeout 900 python -m pytest tests -m gpu -x -q -k "tensor_core or scan or search or edge" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_search.csv -k regex:"scan_|first_list|ip_|pair_|qhat|gemm_kernel|probe|prepare|select|merge" python tools/prof_search.py --config c3 --nprobe 8 --reps 2 > gpurun_out/prof2.log 2>&1; echo "launches rc=$?"
python tools/launch_summary.py gpurun_out/launches_c3_search.csv | head -12
