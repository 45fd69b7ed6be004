# tests on the tensor-core paths, C3 bench (bitwise, LUT), ncu evidence: traffic launch list,
# full capture of tc_refine, full captures of the GEMMs (query rotation; k-means labels in the build)
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "lut or near_dup or tensor_core or b8_d768 or sharded" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
for m in bitwise lut; do
  timeout 600 python bench.py --mode $m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_$m.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bench_c3_$m.json')); print('$m', d['value'], d['ms_per_step'], d['stage_ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'])"
done
timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_c3.csv python tools/prof_search.py --config c3 --nprobe 8 --reps 1 > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/traffic_c3.csv c3 8 > gpurun_out/traffic_c3.json
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"tc_refine|gemm_kernel" -c 2 -o gpurun_out/prof_c3_r2 python tools/prof_search.py --config c3 --nprobe 8 --reps 1 > /dev/null 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:"gemm_argmin" -s 30 -c 1 -o gpurun_out/prof_kmeans_c3 python tools/prof_search.py --config c3 --nprobe 8 --reps 1 > /dev/null 2>&1; echo "ncu km rc=$?"
