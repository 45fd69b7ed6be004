# C4/C5 per-kernel launch list with DRAM traffic (searches only: --profile-from-start off)
set -x
for spec in "c4 64" "c5 32"; do
  set -- $spec
  timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
     --clock-control none --csv --log-file gpurun_out/traffic_$1.csv python tools/prof_search.py --config $1 --nprobe $2 --reps 1 \
     > gpurun_out/prof_$1.log 2>&1
  python tools/ncu_traffic.py gpurun_out/traffic_$1.csv $1 $2 > gpurun_out/traffic_$1.json
done
echo done
