# A/B of one pool option: OPT=name VALS="0 1" CFGS="cfg4 cfg3" bash scripts/ab_opt.sh
# -> gpurun_out/ab_<name>.txt (ms per slice, CUDA-event us per launch)
mkdir -p gpurun_out
for r in 1 2; do
for v in ${VALS:-0 1}; do
  for cfg in ${CFGS:-cfg4 cfg3 cfg2}; do
    timeout 300 python bench.py --config $cfg --opt $OPT=$v $EXTRA > gpurun_out/ab_${cfg}.json 2>/dev/null
    python -c "import json,sys;d=json.load(open('gpurun_out/ab_${cfg}.json'));k=d['kernels'];print('$cfg $OPT=$v', round(d['ms_per_step'],4), 'scan', round(k['scan']['ms_per_launch']*1e3,1), 'pass', round(k['bitmap']['ms_per_launch']*1e3,1), 'reg', round(k['registry']['ms_per_launch']*1e3,1), 'sweep', round(k['sweep']['ms_per_launch']*1e3,1))" >> gpurun_out/ab_$OPT.txt
  done
done
done
