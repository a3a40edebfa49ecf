# ncu evidence for the bench workload (1 GPU): launch list + full capture of the top kernels
mkdir -p gpurun_out
# every launch with its device time (cold, serialised): the prefill is 120 slices x ~12 launches
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 150 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 > gpurun_out/ncu_launch_run.log 2>&1
echo "launches rc=$?"
for K in k_g0 k_scan_packed16 k_active k_bitmap; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 125 -c 1 \
     -o gpurun_out/prof_$K python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_$K.log 2>&1
  echo "$K rc=$?"
done
ls -la gpurun_out/
