# Round evidence in one gpurun session (outputs under gpurun_out/, kept under
# 64 MiB): smoke, the whole GPU suite (BASELINE-shape parity included), bench
# lines for every config and the reference arm, the launch list and ncu
# summaries of the headline's kernels, sanitizers, ingest throughput.
mkdir -p gpurun_out
TAG=${TAG:-r02i}
LONG=1 SUITE_TIMEOUT=2400 BENCH_CFGS="cfg4 cfg2 cfg3 cfg1 cfg5" bash scripts/gpu_round.sh
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
CFG=cfg4 TAG=$TAG KERNELS="k_scan_packed16 k_bp_window k_bp_groups k_bp_resolve" bash scripts/ncu_cfg.sh
CFG=cfg2 TAG=$TAG KERNELS="k_scan_packed16 k_bp_window" bash scripts/ncu_cfg.sh
CFG=cfg4 TAG=$TAG bash scripts/ncu_incontext.sh
timeout 900 python scripts/ingest_bench.py > gpurun_out/ingest.json 2> gpurun_out/ingest.err
du -sh gpurun_out
