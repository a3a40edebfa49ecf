# one gpurun session: smoke, the GPU parity suite, bench variants
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for V in ${BENCH_VARIANTS:-"--incremental on" "--incremental off"}; do :; done
timeout 400 python bench.py --steps 30 --warmup 3 --incremental on > gpurun_out/bench_inc.log 2>&1
echo "bench inc rc=$?" >> gpurun_out/bench_inc.log
timeout 400 python bench.py --steps 30 --warmup 3 --incremental off > gpurun_out/bench_full.log 2>&1
echo "bench full rc=$?" >> gpurun_out/bench_full.log
tail -3 gpurun_out/smoke.log; tail -25 gpurun_out/pytest_gpu.log
for f in gpurun_out/bench_inc.log gpurun_out/bench_full.log; do python - "$f" <<'PY'
import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line); print(sys.argv[1], 'value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1), 'est_ms', round(d['estimate_ms_per_slice'],3), d.get('incremental'))
        print({k:(round(v['ms_per_launch'],4), v['launches']) for k,v in d['kernels'].items()})
    elif 'rc=' in line or 'Error' in line: print(line.strip())
PY
done
