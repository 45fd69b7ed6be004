# per-kernel launch list of the C3 search (serialised, cold cache) with DRAM bytes
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3_r2.csv python tools/prof_search.py --config ${CFG:-c3} --nprobe ${NPROBE:-8} --reps 1 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/launches_c3_r2.csv | head -40
