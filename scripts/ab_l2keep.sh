# A/B of the scan's L2 evict_last hints (VATE_OPT_L2_KEEP): one bench line per
# setting and config, twice.
mkdir -p gpurun_out
for r in 1 2; do
for v in 0 1; do
  for cfg in ${CFGS:-cfg4 cfg3 cfg2}; do
    timeout 300 python bench.py --config $cfg --opt l2_keep=$v > gpurun_out/ab_${cfg}.json 2>/dev/null
    python -c "import json,sys;d=json.load(open('gpurun_out/ab_${cfg}.json'));k=d['kernels'];print('$cfg l2_keep=$v', round(d['ms_per_step'],4), 'scan', round(k['scan']['ms_per_launch']*1e3,1), 'pass', round(k['bitmap']['ms_per_launch']*1e3,1), 'reg', round(k['registry']['ms_per_launch']*1e3,1))" >> gpurun_out/ab_l2keep.txt
  done
done
done
