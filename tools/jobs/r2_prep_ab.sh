set -x
timeout 600 python -m pytest tests -m gpu -x -q -k "probe or select or search_batch" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
for mode in bitwise lut; do for v in "IVRQ_PREP_SEQ=0" "IVRQ_PREP_SEQ=1" "IVRQ_PREP_PRIO=1"; do
  echo "== $mode $v"; env $v timeout 300 python tools/prof_search.py --config c3 --nprobe 8 --reps 4 --mode $mode 2>&1 | grep -E "step|Error" | tail -2
done; done
for c in "c4 64" "c5 32"; do set -- $c; timeout 300 python tools/prof_search.py --config $1 --nprobe $2 --reps 3 2>&1 | grep -E "step|Error" | tail -1; done
