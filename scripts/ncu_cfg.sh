# ncu evidence for one bench config (1 GPU), from the bench's timed region
# (VATE_PROFILE_REGION=1 brackets it with cudaProfilerStart/Stop):
#  1. the launch list (gpu__time_duration per launch; cold and serialised:
#     compare SHARES, not absolutes) -> gpurun_out/<tag>_launches.csv
#  2. one --set full capture of each kernel in KERNELS -> gpurun_out/<tag>_<kernel>.ncu-rep
# usage: CFG=cfg4 TAG=r02a KERNELS="k_bitmap k_scan_packed16" bash scripts/ncu_cfg.sh
mkdir -p gpurun_out
CFG=${CFG:-cfg4}; TAG=${TAG:-prof}
VATE_PROFILE_REGION=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  --profile-from-start off --csv python bench.py --config $CFG --steps 4 --warmup 3 ${BENCH_ARGS} \
  > gpurun_out/${TAG}_${CFG}_launches.csv 2> gpurun_out/${TAG}_${CFG}_launches.err
for k in ${KERNELS:-k_bitmap k_scan_packed16}; do
  VATE_PROFILE_REGION=1 timeout 900 ncu --set full --clock-control none --import-source on \
    --profile-from-start off -k regex:"$k" -s 1 -c 1 -o gpurun_out/${TAG}_${CFG}_$k \
    python bench.py --config $CFG --steps 4 --warmup 3 ${BENCH_ARGS} > gpurun_out/${TAG}_${CFG}_$k.log 2>&1
done
