# A/B of env toggles on a config's search step (events, no profiler): CFG NPROBE VARIANTS...
CFG=$1; NP=$2; shift 2
for v in "$@"; do
  echo "== $v"; env $v timeout 600 python tools/prof_search.py --config $CFG --nprobe $NP --reps 4 2>&1 | grep step | tail -2
done
