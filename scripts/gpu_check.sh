# one gpurun session: smoke, the GPU parity suite, bench variants
mkdir -p gpurun_out
python -c "import torch;p=torch.cuda.get_device_properties(0);print(p, p.L2_cache_size)" > gpurun_out/props.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for K in gather smem; do
  timeout 400 python bench.py --steps 30 --warmup 3 --g0-kernel $K > gpurun_out/bench_$K.log 2>&1
  echo "bench $K rc=$?" >> gpurun_out/bench_$K.log
done
tail -3 gpurun_out/smoke.log; tail -15 gpurun_out/pytest_gpu.log; tail -c 1500 gpurun_out/bench_*.log
