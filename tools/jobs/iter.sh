# quick iteration: parity subset, C3 bench, e2e probe, search launch list
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"
timeout 600 python tools/e2e_probe.py --config c3 --nprobe 8 > gpurun_out/e2e_probe.log 2>&1; echo "e2e rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_search.csv -k regex:"scan|first_list|ip_tile|pair_|cs_|gemm|probe|prepare|select|merge" python tools/prof_search.py --config c3 --nprobe 8 --reps 2 > gpurun_out/prof2.log 2>&1; echo "launches rc=$?"
