IVRQ_KERNEL_TIMING=1 python tools/prof_search.py --config c3 --nprobe 8 --reps 3 2>&1 | grep -E "step ms|tc_|scan_" | tail -6
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"scan_rda" -c 1 -o gpurun_out/prof_rda python tools/prof_search.py --config c3 --nprobe 8 --reps 1 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/prof_rda.ncu-rep
