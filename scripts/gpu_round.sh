# One gpurun session: smoke, the GPU suite (minus the long BASELINE-shape
# parity unless LONG=1), then bench lines.  Outputs under gpurun_out/.
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
SEL="tests -m gpu"
[ "${LONG:-0}" = "1" ] || SEL="$SEL --deselect tests/test_gpu_long_parity.py"
timeout ${SUITE_TIMEOUT:-1500} python -m pytest $SEL -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for cfg in ${BENCH_CFGS:-cfg4 cfg2}; do
  timeout 600 python bench.py --config $cfg ${BENCH_ARGS} > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
done
