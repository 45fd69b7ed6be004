# C4 / C5 with the dense approximate refine forced on, against the default (in-warp survivor refine)
for c in "c4 64" "c5 32" "c2 16"; do
  set -- $c
  for v in "" "IVRQ_TC_REFINE=1"; do
    echo "== $1 ${v:-default}"
    env $v IVRQ_KERNEL_TIMING=1 timeout 600 python tools/prof_search.py --config $1 --nprobe $2 --reps 3 2>&1 | grep -E "step ms|tc_|scan_" | tail -4
  done
done
