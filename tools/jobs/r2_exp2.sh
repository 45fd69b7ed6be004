for v in "-DIVRQ_EXP_NOTMA -DIVRQ_EXP_NOEPI" "-DIVRQ_EXP_NOTMA -DIVRQ_EXP_NOEPI -DIVRQ_EXP_NOMMA" "-DIVRQ_EXP_NOTMA -DIVRQ_EXP_NOEPI -DIVRQ_EXP_NOB" "-DIVRQ_EXP_NOTMA -DIVRQ_EXP_NOEPI -DIVRQ_EXP_NOB -DIVRQ_EXP_NOMMA" "-DIVRQ_EXP_NOB"; do
  python -c "from paper_2602_23999_b200 import _build; _build.build(force=True, extra_flags='$v'.split())" > gpurun_out/b.log 2>&1 || tail gpurun_out/b.log
  echo "== $v"
  IVRQ_KERNEL_TIMING=1 python tools/prof_search.py --config c3 --nprobe 8 --reps 2 2>&1 | grep -E "tc_refine" | tail -1
done
