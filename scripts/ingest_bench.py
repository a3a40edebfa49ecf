"""Trace-ingest throughput (SURVEY §8f rank 1; traceio.py:77-106, :188-230).

Writes a binary trace of 16-byte records (default 2.1 GB: 134M records, 5M
records per 1-second slice, 1M hosts) to a scratch file, then times
traceio.DeviceSlices over it -- pinned double-buffered reads, async H2D,
packing and slice runs on the device -- (a) alone and (b) feeding the slice
step (Pipeline.step_fast on a cfg-2 shape pool), with the page cache warm and,
when the box allows it, dropped first.  One JSON line per measurement.

    python scripts/ingest_bench.py [--records N] [--path /tmp/vate_trace.bin]
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def write_trace(path, n, per_slice, hosts):
    from paper_1812_00282_b200 import traceio
    rng = np.random.default_rng(0)
    step = 1 << 22
    with open(path, "wb") as fh:
        for lo in range(0, n, step):
            m = min(step, n - lo)
            i = np.arange(lo, lo + m, dtype=np.uint64)
            ts = (i * np.uint64(1_000_000)) // np.uint64(per_slice)      # per_slice per second
            rec = traceio.make_records(ts, (0x0A000000 + rng.integers(0, hosts, m)).astype(np.uint32),
                                       rng.integers(1, 1 << 32, m, dtype=np.uint64).astype(np.uint32))
            fh.write(rec.tobytes())


def drop_caches():
    try:
        subprocess.run(["sync"], check=True)
        with open("/proc/sys/vm/drop_caches", "w") as fh:
            fh.write("3\n")
        return True
    except OSError:
        return False


def _steady(stamps, start, records, skip=3):
    """One-time setup (pinned staging buffers, the pool's log table, incremental
    index and bit-plane ring) lands on the first slices: report the time to the
    end of slice `skip` apart and the rate over the slices after it (uniform
    slices: records per slice = records / slices)."""
    if len(stamps) <= skip + 1:
        return {}
    per = records / len(stamps)
    span = stamps[-1] - stamps[skip]
    return {"first_slices_s": stamps[skip] - start, "first_slices": skip + 1,
            "after_last_slice_s": time.perf_counter() - stamps[-1],
            "steady_GB_per_s": 16 * per * (len(stamps) - skip - 1) / span / 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--records", type=int, default=134_217_728)
    ap.add_argument("--path", default="/tmp/vate_ingest_trace.bin")
    ap.add_argument("--per-slice", type=int, default=5_000_000)
    args = ap.parse_args()
    import torch
    import paper_1812_00282_b200 as vb
    from paper_1812_00282_b200 import traceio

    t0 = time.perf_counter()
    write_trace(args.path, args.records, args.per_slice, 1_000_000)
    subprocess.run(["sync"], check=False)   # no dirty-page write-back under the warm runs
    size = os.path.getsize(args.path)
    print(json.dumps({"trace_bytes": size, "records": args.records,
                      "write_s": time.perf_counter() - t0}), flush=True)
    cfg = vb.EstimatorConfig(1024, 24, 60)
    for cache in ("warm", "dropped"):
        if cache == "dropped" and not drop_caches():
            print(json.dumps({"cache": "dropped", "skipped": "no permission to drop caches"}))
            continue
        # (a) ingest alone: records -> device pairs + slice runs
        pool = cfg.build_pool()
        torch.cuda.synchronize()
        a = time.perf_counter()
        slices = pairs = 0
        stamps = []
        for t, dptr, n in traceio.DeviceSlices(pool, args.path, traceio.BINARY, 1_000_000):
            slices += 1
            pairs += n
            stamps.append(time.perf_counter())
        pool.synchronize()
        dt = time.perf_counter() - a
        print(json.dumps({"cache": cache, "mode": "ingest only", "slices": slices, "records": pairs,
                          "s": dt, "GB_per_s": size / dt / 1e9, "Mrecords_per_s": pairs / dt / 1e6,
                          **_steady(stamps, a, pairs)}), flush=True)
        if cache == "dropped":
            drop_caches()
        # (b) ingest feeding the slice step (scan, estimate of ~1M hosts, advance)
        pipe = vb.Pipeline(pool, cfg, 60)
        outs = [tuple(np.empty(1 << 21, dt) for dt in (np.uint64, np.float64, np.float64, np.uint8))
                for _ in range(2)]
        a = time.perf_counter()
        slices = pairs = 0
        stamps = []
        marks = []          # (t_wait: next slice handed over, t_step: step call returned)
        it = iter(traceio.DeviceSlices(pool, args.path, traceio.BINARY, 1_000_000))
        while True:
            w0 = time.perf_counter()
            try:
                t, dptr, n = next(it)
            except StopIteration:
                break
            w1 = time.perf_counter()
            pipe.step_fast(t, dptr, n, "device", outs[t % 2])
            marks.append((w1 - w0, time.perf_counter() - w1))
            stamps.append(time.perf_counter())
            slices += 1
            pairs += n
        pipe.wait_reports()
        pool.synchronize()
        dt = time.perf_counter() - a
        print(json.dumps({"cache": cache, "mode": "ingest + slice step (cfg 2 pool, 1M hosts)",
                          "slices": slices, "records": pairs, "s": dt,
                          "GB_per_s": size / dt / 1e9, "Mrecords_per_s": pairs / dt / 1e6,
                          **_steady(stamps, a, pairs),
                          "per_slice_ms": [[round(1e3 * x, 2), round(1e3 * y, 2)] for x, y in marks]}),
              flush=True)
        pipe.close()
        pool.close()
    os.remove(args.path)


if __name__ == "__main__":
    main()
