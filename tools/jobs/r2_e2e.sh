# e2e pipeline iteration: pipeline tests, A/B of the host pipeline, default bench
set -x
timeout 400 python -m pytest tests -m gpu -x -q -k "search_batch or smoke or end_to_end" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/gpu_tests.log
timeout 300 python tools/e2e_ab.py --threads ${TH:-8} --pieces ${PC:-1,4,8} > gpurun_out/e2e_ab.log 2>&1; tail -12 gpurun_out/e2e_ab.log
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print(d['value'], d['ms_per_step'], d['e2e'])"
