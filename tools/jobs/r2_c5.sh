for v in "" "IVRQ_TC_REFINE=1"; do
  echo "== c5 ${v:-default}"
  env $v IVRQ_KERNEL_TIMING=1 timeout 600 python tools/prof_search.py --config c5 --nprobe 32 --reps 3 2>&1 | grep -E "step ms" | tail -2
done
