# ncu evidence for the bench workload (1 GPU): launch list + full captures of the top kernels
mkdir -p gpurun_out
# every launch of a few timed steps with its device time (cold, serialised: compare SHARES)
VATE_PROFILE_REGION=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
   python bench.py --steps 10 --warmup 3 > gpurun_out/launches.csv 2> gpurun_out/ncu_launch_run.log
echo "launches rc=$?"
# incremental path kernels (default bench), one capture each, after the prefill
for K in k_scan_packed16 k_bitmap k_inc_apply k_inc_lookup k_final_write k_active k_g0; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 140 -c 1 \
     -o gpurun_out/prof_$K python bench.py --steps 20 --warmup 3 > gpurun_out/ncu_$K.log 2>&1
  echo "$K rc=$?"
done
# the full-recompute gather (reference-equivalent per-slice g0), for the L1TEX-bound evidence
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_g0" -s 130 -c 1 \
   -o gpurun_out/prof_k_g0_full python bench.py --steps 20 --warmup 3 --incremental off > gpurun_out/ncu_k_g0_full.log 2>&1
echo "g0 full rc=$?"
ls -la gpurun_out/
