mkdir -p gpurun_out
MICRO_CK=24,60 timeout 300 python scripts/micro_scan.py > gpurun_out/micro_cfg2.log 2>&1
MICRO_CK=28,300 timeout 300 python scripts/micro_scan.py > gpurun_out/micro_cfg4.log 2>&1
cat gpurun_out/micro_cfg2.log gpurun_out/micro_cfg4.log
VARIANTS="--config cfg3 --steps 20 --warmup 3;--config cfg3 --steps 20 --warmup 3 --scan-check 1;--config cfg3 --steps 20 --warmup 3 --scan-check 1 --l2-persist 1;--steps 20 --warmup 3 --l2-persist 1;--config cfg4 --steps 20 --warmup 3 --l2-persist 1" bash scripts/bench_variants.sh
