# A/B of env toggles on the C3 search (launch list per variant)
for v in ${AB_VARIANTS}; do
  env $v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_$v.csv -k regex:"scan_|first_|ip_|tc_" python tools/prof_search.py --config c3 --nprobe 8 --reps 2 > /dev/null 2>&1
  echo "== $v"; python tools/launch_summary.py gpurun_out/ab_$v.csv 2>/dev/null | head -6
done
