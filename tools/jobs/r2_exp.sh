# dev builds with experiment switches (comma-separated flags per variant), C3 search step + kernel event times
for extra in "" ${EXTRA}; do
  extra=$(echo "$extra" | tr ',' ' ')
  python -c "from paper_2602_23999_b200 import _build; _build.build(force=True, extra_flags='${extra}'.split())" > gpurun_out/exp_build.log 2>&1 || { echo build failed; tail gpurun_out/exp_build.log; }
  echo "== variant: ${extra:-default}"
  IVRQ_KERNEL_TIMING=1 python tools/prof_search.py --config ${CFG:-c3} --nprobe ${NPROBE:-8} --reps 3 2>&1 | grep -E "step ms|tc_refine|tc_ip|scan_rd" | tail -3
done
