# tc_refine diagnostics at C3 (IVRQ_TC_DBG: 1 no epilogue, 2 no MMAs, 3 neither; results invalid), ncu durations
for v in IVRQ_TC_DBG=0 IVRQ_TC_DBG=3 "IVRQ_TC_DBG=3 IVRQ_TC_G=8" "IVRQ_TC_DBG=0 IVRQ_TC_G=8"; do
  echo "== $v"
  env $v timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum -k regex:"^(tc_refine)" --csv python tools/prof_search.py --config c3 --nprobe 8 --reps 1 2>/dev/null | grep -E "tc_refine" | awk -F'","' '{print $(NF-2), $NF}' | tail -3
done
