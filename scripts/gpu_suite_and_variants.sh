# one gpurun session: GPU suite + bench variants (counters, configs)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for V in "cfg2 at" "cfg2 dr" "cfg2 ts" "cfg3 at" "cfg4 at" "cfg4 dr"; do
  set -- $V
  timeout 600 python bench.py --config $1 --counter $2 --steps 30 --warmup 3 > gpurun_out/bench_$1_$2.json 2> gpurun_out/bench_$1_$2.err
  echo "bench $1 $2 rc=$?"
done
tail -3 gpurun_out/pytest_gpu.log
for f in gpurun_out/bench_cfg*.json; do python - "$f" <<'PY'
import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line)
        print(sys.argv[1], 'value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1), 'est_ms', round(d['estimate_ms_per_slice'],3), 'maint_ms', round(d['maintain_ms_per_slice'],4), 'frac', round(d['roofline']['frac'],3), d['roofline']['kernel'])
PY
done
