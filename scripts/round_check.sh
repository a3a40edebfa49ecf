# full round evidence: smoke, GPU suite, bench (all configs + reference arm), launch list, ncu captures
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for C in cfg1 cfg4; do python bench.py --config $C --steps 30 --warmup 3 > gpurun_out/bench_$C.json 2>/dev/null; done
python bench.py --incremental off --steps 30 --warmup 3 > gpurun_out/bench_full_recompute.json 2>/dev/null
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
VATE_PROFILE_REGION=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
   python bench.py --steps 10 --warmup 3 > gpurun_out/launches.csv 2> gpurun_out/ncu_launch_run.log
for K in k_scan_packed16 k_bitmap k_inc_apply k_final_all k_active k_sweep; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 140 -c 1 \
     -o gpurun_out/prof_$K python bench.py --steps 20 --warmup 3 > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_g0" -s 130 -c 1 \
   -o gpurun_out/prof_k_g0_full python bench.py --steps 20 --warmup 3 --incremental off > /dev/null 2>&1
tail -2 gpurun_out/smoke.log; tail -3 gpurun_out/pytest_gpu.log; ls gpurun_out
