# RSUB A/B of scan_rda (prebuilt variants tools/lib_*.so)
export IVRQ_NO_AUTOBUILD=1
cp paper_2602_23999_b200/libivrq_b200.so /tmp/lib_keep.so
for v in base rs2 rs6 rs8 base; do
  cp tools/lib_$v.so paper_2602_23999_b200/libivrq_b200.so
  echo "== $v"; IVRQ_KERNEL_TIMING=1 timeout 300 python tools/prof_search.py --config c3 --nprobe 8 --reps 5 2>&1 | grep -E "step|scan_rd|Error" | tail -2
done
cp /tmp/lib_keep.so paper_2602_23999_b200/libivrq_b200.so
