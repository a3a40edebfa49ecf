# one full ncu capture of the cfg2 scan kernel (source counters) in the bench workload
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"k_scan_packed16" -s 140 -c 1 \
   -o gpurun_out/prof_scan python bench.py --steps 20 --warmup 3 ${NCU_BENCH_ARGS} > gpurun_out/ncu_scan.log 2>&1
echo "ncu rc=$?"
ls -la gpurun_out
