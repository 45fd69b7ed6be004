# probe candidate statistics (IVRQ_PROBE_STATS) for C4/C5 at 2 and 4 digits, plus the counting-sort tests
set -x
timeout 600 python -m pytest tests -m gpu -x -q -k "sort or csr or parity" > gpurun_out/gpu_tests_cs.log 2>&1; tail -2 gpurun_out/gpu_tests_cs.log
for c in "c4 64" "c5 32"; do
  set -- $c
  for nd in 2 4; do
    IVRQ_PROBE_STATS=1 IVRQ_PROBE_DIGITS=$nd timeout 600 python tools/prof_search.py --config $1 --nprobe $2 --reps 2 > gpurun_out/ps_$1_$nd.log 2>&1; grep -E "probe|step|Error" gpurun_out/ps_$1_$nd.log | tail -4
  done
done
