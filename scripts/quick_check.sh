mkdir -p gpurun_out
MICRO_CK=24,60 timeout 300 python scripts/micro_scan.py 2>&1 | grep "l2=0" | head -3
MICRO_CK=28,300 timeout 300 python scripts/micro_scan.py 2>&1 | grep "l2=0" | head -3
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 400 -p no:cacheprovider ${PYTEST_ARGS} 2>&1 | tail -3
VARIANTS="--steps 30 --warmup 3;--config cfg3 --steps 20 --warmup 3 --scan-check 1;--config cfg4 --steps 20 --warmup 3" bash scripts/bench_variants.sh
