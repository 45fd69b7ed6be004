# mbarrier suspend-time hint A/B (prebuilt variants tools/lib_*.so)
export IVRQ_NO_AUTOBUILD=1
cp paper_2602_23999_b200/libivrq_b200.so /tmp/lib_keep.so
for v in base hint base hint; do
  cp tools/lib_$v.so paper_2602_23999_b200/libivrq_b200.so
  echo "== $v"; IVRQ_KERNEL_TIMING=1 timeout 300 python tools/prof_search.py --config c3 --nprobe 8 --reps 5 2>&1 | grep -E "step|_kernel|Error" | tail -3
done
for v in base hint; do
  cp tools/lib_$v.so paper_2602_23999_b200/libivrq_b200.so
  echo "== c5 $v"; IVRQ_KERNEL_TIMING=1 timeout 300 python tools/prof_search.py --config c5 --nprobe 32 --reps 3 2>&1 | grep -E "step|Error" | tail -1
done
cp tools/lib_hint.so paper_2602_23999_b200/libivrq_b200.so
timeout 600 python -m pytest tests -m gpu -x -q -k "tensor_core or golden or refine or probe" > gpurun_out/gpu_tests_hint.log 2>&1; echo "hint tests rc=$?"; tail -1 gpurun_out/gpu_tests_hint.log
cp /tmp/lib_keep.so paper_2602_23999_b200/libivrq_b200.so
