# profile artefacts for profiles/<round>: per-search launch list, scan DRAM traffic, full captures
set -x
for spec in "c3 8" "c1 16" "c2 16"; do
  set -- $spec
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file gpurun_out/traffic_$1.csv python tools/prof_search.py --config $1 --nprobe $2 --reps 1 > /dev/null 2>&1
  python tools/ncu_traffic.py gpurun_out/traffic_$1.csv $1 $2 > gpurun_out/traffic_$1.json
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^(tc_refine_kernel|tc_ip_kernel|scan_rd_kernel)" -c 3 \
   -o gpurun_out/prof_scan_c3_r1e python tools/prof_search.py --config c3 --nprobe 8 --reps 1 > /dev/null 2>&1
echo done
