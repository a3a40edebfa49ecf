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
  # summaries on the box (gpurun_out comes back only under 64 MiB): metrics,
  # opcode mix; the report itself only with KEEP_REP=1
  python scripts/ncu_summary.py gpurun_out/${TAG}_${CFG}_$k.ncu-rep >> gpurun_out/${TAG}_ncu_kernels.txt 2>&1
  python scripts/ncu_ops.py gpurun_out/${TAG}_${CFG}_$k.ncu-rep 16 > gpurun_out/${TAG}_${CFG}_${k}_ops.txt 2>&1
  [ "${KEEP_REP:-0}" = "1" ] || rm -f gpurun_out/${TAG}_${CFG}_$k.ncu-rep
done
python scripts/launch_summary.py gpurun_out/${TAG}_${CFG}_launches.csv > gpurun_out/${TAG}_${CFG}_launches_summary.txt 2>&1
