# profile artefacts for profiles/<round>: per-search launch lists with DRAM traffic (searches only),
# a full capture of the C3 dominant kernel
set -x
for spec in "c3 8" "c1 16" "c2 16" "c4 64" "c5 32"; do
  set -- $spec
  timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
     --clock-control none --csv --log-file gpurun_out/traffic_$1.csv python tools/prof_search.py --config $1 --nprobe $2 --reps 1 \
     > gpurun_out/prof_$1.log 2>&1
  python tools/ncu_traffic.py gpurun_out/traffic_$1.csv $1 $2 > gpurun_out/traffic_$1.json
done
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"^(tc_refine_kernel)" -c 1 \
   -o gpurun_out/prof_refine_c3 python tools/prof_search.py --config c3 --nprobe 8 --reps 1 > /dev/null 2>&1
echo done
