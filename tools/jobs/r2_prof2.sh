# tc_refine timeline (dev build) + scan_rda ncu (release build)
python -c "from paper_2602_23999_b200 import _build; _build.build(force=True, extra_flags=['-DIVRQ_TCR_TRACE'])" > gpurun_out/b.log 2>&1 || tail gpurun_out/b.log
IVRQ_TCR_TRACE_OUT=gpurun_out/tcr_trace.bin python tools/prof_search.py --config c3 --nprobe 8 --reps 2 2>&1 | grep -E "step ms" | tail -2
python -c "from paper_2602_23999_b200 import _build; _build.build(force=True)" > gpurun_out/b.log 2>&1 || tail gpurun_out/b.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"scan_rda" -c 1 -o gpurun_out/prof_rda2 python tools/prof_search.py --config c3 --nprobe 8 --reps 1 > /dev/null 2>&1; echo "ncu rc=$?"
