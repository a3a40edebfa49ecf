# DRAM traffic of the slice's kernels with the L2 as the pipeline leaves it
# (ncu --cache-control none: no flush before each launch, unlike the --set full
# captures, whose dram__bytes count a cold L2).  Launches are still serialised
# by ncu, so aux-stream kernels no longer overlap; the bytes are what matters.
# usage: CFG=cfg4 TAG=r02f bash scripts/ncu_incontext.sh
mkdir -p gpurun_out
CFG=${CFG:-cfg4}; TAG=${TAG:-prof}
VATE_PROFILE_REGION=1 timeout 900 ncu --cache-control none --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors.sum \
  --profile-from-start off --csv python bench.py --config $CFG --steps 4 --warmup 3 ${BENCH_ARGS} \
  > gpurun_out/${TAG}_${CFG}_incontext.csv 2> gpurun_out/${TAG}_${CFG}_incontext.err
python scripts/incontext_summary.py gpurun_out/${TAG}_${CFG}_incontext.csv \
  > gpurun_out/${TAG}_${CFG}_incontext_summary.txt 2>&1
