"""A small workload that touches every kernel family, for compute-sanitizer:
the one-call and the pipelined slice step (scan forms, registry growth, parked
inserts, merges, prune), the comparators, snapshots, trace bucketing."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1812_00282_b200 as vb

rng = np.random.default_rng(5)
for kind in ("at", "dr", "ts"):
    cfg = vb.EstimatorConfig(128, 14, 6, seed=3, counter_kind=kind)
    pool = cfg.build_pool()
    pipe = vb.Pipeline(pool, cfg, 5, floor=0.0)
    outs = [tuple(np.empty(20_000, dt) for dt in (np.uint64, np.float64, np.float64, np.uint8))
            for _ in range(2)]
    for t in range(14):
        n = int(rng.integers(1, 6000))
        span = 12_000 if t < 3 else 800
        a = (0x0A000000 + rng.integers(0, span, n)).astype(np.uint32)
        b = rng.integers(1, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        pairs = np.ascontiguousarray(np.stack([a, b], axis=1))
        if t % 2:
            pipe.step_lagged(t, pairs.ctypes.data, n, "host", outs[t % 2])
        else:
            if t:
                pipe.flush_lagged(outs[0])
            pipe.process_slice_soa(t, a.astype(np.uint64), b.astype(np.uint64))
        pipe.wait_reports()
        if kind == "at" and t in (4, 9):   # deferred marks + bit-plane history for slices 4-8
            pool.set_option("deferred", 1 if t == 4 else 0)
            pool.set_option("bitplane", 1 if t == 4 else 0)
        if kind == "at" and t == 9:
            for form in (0, 1):
                pool.set_option("scan_filter", form)
    pipe.flush_lagged(outs[0])
    pipe.wait_reports()
    if kind == "at":
        blob = pool.snapshot_bytes()
        vb.AtPool.from_bytes(blob).close()
    pipe.close()
    pool.close()
print("sanitize workload done")
