# occupancy A/B of rda_final / scan_rda (prebuilt variants tools/lib_*.so)
export IVRQ_NO_AUTOBUILD=1
cp paper_2602_23999_b200/libivrq_b200.so /tmp/lib_keep.so
for v in base fin10 fin12 rda5 base; do
  cp tools/lib_$v.so paper_2602_23999_b200/libivrq_b200.so
  echo "== $v"; IVRQ_KERNEL_TIMING=1 timeout 300 python tools/prof_search.py --config c3 --nprobe 8 --reps 5 2>&1 | grep -E "step|_kernel|Error" | tail -3
done
for v in base rda5; do
  cp tools/lib_$v.so paper_2602_23999_b200/libivrq_b200.so
  echo "== c2 $v"; IVRQ_KERNEL_TIMING=1 timeout 300 python tools/prof_search.py --config c2 --nprobe 16 --reps 4 2>&1 | grep -E "step|_kernel|Error" | tail -2
done
cp /tmp/lib_keep.so paper_2602_23999_b200/libivrq_b200.so
