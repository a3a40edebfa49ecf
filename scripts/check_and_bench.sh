# GPU suite + the scan micro + bench cfg2/3/4 (one gpurun session)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 400 -p no:cacheprovider ${PYTEST_ARGS} 2>&1 | tail -3
MICRO_CK=24,60 timeout 300 python scripts/micro_scan.py 2>&1 | grep "check=0 V=1\|only"
MICRO_CK=26,60 MICRO_ZIPF=1 timeout 300 python scripts/micro_scan.py 2>&1 | grep "V=1\|only"
VARIANTS="--steps 30 --warmup 3;--config cfg3 --steps 20 --warmup 3;--config cfg4 --steps 20 --warmup 3" bash scripts/bench_variants.sh
