# Development builds with tc_refine wait-cycle counters (-DIVRQ_TC_PROFILE), then a C3 search.
# Rebuilds the box's scratch copy of the library only.  EXTRA="-DIVRQ_TC_NO_EPI" etc. for A/B.
for extra in "" ${EXTRA}; do
  python -c "from paper_2602_23999_b200 import _build; _build.build(force=True, extra_flags=['-DIVRQ_TC_PROFILE'] + '${extra}'.split())" > gpurun_out/tc_prof_build.log 2>&1
  echo "== variant: ${extra:-default}"
  python tools/prof_search.py --config ${CFG:-c3} --nprobe ${NPROBE:-8} --reps 3 2>&1 | grep -E "tc_refine prof|step ms" | tail -2
done
