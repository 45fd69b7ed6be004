set -x
for c in c2 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --build-breakdown --gt-queries 1000 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 2 -c 1 -o gpurun_out/prof_scan_c3_r1b python tools/prof_search.py --config c3 --nprobe 8 > gpurun_out/prof.log 2>&1
echo "ncu rc=$?"
