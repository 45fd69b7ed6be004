# tc_refine timelines of CTA 0 under experiment switches (dev builds)
for v in ${VARIANTS}; do
  v=$(echo "$v" | tr ',' ' ')
  python -c "from paper_2602_23999_b200 import _build; _build.build(force=True, extra_flags=['-DIVRQ_TCR_TRACE'] + '$v'.split())" > gpurun_out/b.log 2>&1 || tail gpurun_out/b.log
  tag=$(echo "x$v" | tr -d ' -' )
  echo "== $v"
  IVRQ_KERNEL_TIMING=1 IVRQ_TCR_TRACE_OUT=gpurun_out/tcr_trace_$tag.bin python tools/prof_search.py --config c3 --nprobe 8 --reps 2 2>&1 | grep -E "tc_refine" | tail -1
done
