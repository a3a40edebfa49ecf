#!/usr/bin/env python
"""Benchmark of the VATE hot path on B200 (contract: one JSON line on rank 0).

A step is one whole slice of the reference's pipeline (pipeline.py:142-160).
The default workload is BASELINE.json configs[3] (cfg 4), the largest
single-GPU shape and the north star's k = 300 window: 5,000,000 packets per
slice from 1,000,000 hosts, pool 2^28 (512 MiB of u16 cells, beyond L2),
k = k' = 300, g = 1024, tail partition, seed 0, floor 0 (every active host's
report is produced):

    scan (hash 5M packets, mark their cells, register hosts)
    -> estimate (sorted active hosts, Z_p + inactive bitmap, g0 of every
       active host, float path; SoA reports land in host memory)
    -> maintain (advance clocks, sweep the two due blocks), prune every k.

`value`  = packets / device time of K steps with packets resident in HBM and
           the SoA report rows left in HBM (every slice distinct, 40 MB each).
`e2e`    = the same K steps through the public API from pinned HOST packet
           buffers: H2D of every slice's packets + D2H of every report row.
--config cfg1/cfg2/cfg3/cfg5 select the other BASELINE shapes (cfg 5: 100M
packets per slice).

--impl reference: the reference algorithm on the box's host cores, through
the oracle port (oracle/: the reference is pure Python and cannot travel to
the GPU box): per step one full slice -- the whole scan, host-set update,
Z_p, advance -- with g0 + float path timed on a sample of the active hosts
and scaled to all of them (the factor is in the line).  Multi-GPU (torchrun,
N > 1): each rank scans its own shard into a replica pool; replicas merge
every slice (fused peer-memory merge, or NCCL all-gathers); the active-host
union is range-split for the estimate.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # BASELINE.json configs[1]: the 40 Gb/s-equivalent trace, L2-resident pool
    "cfg2": dict(name="cfg2-40Gbps-equivalent", c=24, k=60, k_prime=60, g=1024,
                 hosts=1_000_000, packets=5_000_000, seed=0, partition="tail", floor=0.0,
                 base_aip=0x0A000000),
    # configs[0]: the reference's CPU-runnable shape (1M packets as 10 x 100k slices)
    "cfg1": dict(name="cfg1-cpu-reference-shape", c=20, k=10, k_prime=10, g=1024,
                 hosts=10_000, packets=100_000, seed=0, partition="tail", floor=0.0,
                 base_aip=0x0A000000),
    # configs[2]: Zipf(1.1) host popularity + 64 super-spreaders (10% of packets,
    # random peers), pool 2^26
    "cfg3": dict(name="cfg3-zipf-superspreaders", c=26, k=60, k_prime=60, g=1024,
                 hosts=1_000_000, packets=5_000_000, seed=0, partition="tail", floor=0.0,
                 base_aip=0x0A000000, zipf=True),
    # configs[3]: long window, 512 MiB of u16 cells beyond L2 -- the headline
    # (default): the largest single-GPU config and the north star's k = 300
    "cfg4": dict(name="cfg4-long-window-k300", c=28, k=300, k_prime=300, g=1024,
                 hosts=1_000_000, packets=5_000_000, seed=0, partition="tail", floor=0.0,
                 base_aip=0x0A000000),
    # configs[4]: 100M packets per slice in total (k=300, 2^28), split across the
    # ranks (strong scaling); on one GPU the whole 100M-packet slice
    "cfg5": dict(name="cfg5-100M-packets-per-slice-k300", c=28, k=300, k_prime=300, g=1024,
                 hosts=1_000_000, packets=100_000_000, seed=0, partition="tail", floor=0.0,
                 base_aip=0x0A000000, strong=True),
}
WORKLOAD = WORKLOADS["cfg4"]
METRIC = "Mpackets/s AT scan+update (full slice: scan+estimate+maintain)"
UNIT = "Mpackets/s"
PEAKS_FALLBACK = dict(hbm_gbs=6650.0)


KERNEL_SYMBOL = {"scan": ("k_scan_packed16",), "bitmap": ("k_bp_window", "k_bitmap"),
                 "g0": ("k_g0",), "final": ("k_final_all",), "registry": ("k_active",),
                 "sweep": ("k_bp_groups", "k_sweep")}


def _ncu_traffic(kind, cfg, bitplane=False):
    """dram read+write bytes per launch of the kernel behind `kind` for this workload,
    from the committed ncu --set full summaries (profiles/*ncu_kernels.txt, sections
    "## <tag>_<cfg>_<kernel>..."; newest file first); None if not captured."""
    import glob
    syms = KERNEL_SYMBOL.get(kind)
    if syms is None:
        return None
    sym = syms[0] if bitplane else syms[-1]
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu_kernels.txt")), reverse=True):
        cur, vals = None, {}
        for line in open(path):
            if line.startswith("## "):
                cur = line
            elif cur and f"_{cfg}_{sym}" in cur and "dram__bytes" in line:
                parts = line.split()
                v, unit = float(parts[1]), parts[2] if len(parts) > 2 else "byte"
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                vals[parts[0]] = v * scale
        if vals:
            return sum(vals.values())
    return None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock and throttle reasons sampled by NVML while the timed region runs."""

    BAD = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
           "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device: int):
        self.samples, self.reasons, self._stop = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                mask = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.BAD.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv is not None:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------------
# CPU arm: the oracle port on the box's host cores
# ----------------------------------------------------------------------------------

def cpu_sample(w, steps=1, host_sample=250_000, kind="at", warmup=0):
    """The reference algorithm on the host cores, per slice of the workload.

    AT pools: the oracle's C half (oracle/native.py, OpenMP over every host
    thread) plus its numpy parts, one FULL slice per step: hashing and setting
    all of the slice's packets with the reference's per-block value histogram
    (pools.py:163-178), the host-set update and active set (pipeline.py:43-64),
    Z_p from the histogram (pools.py:195-204), g0 + float path for
    `host_sample` of the active hosts (estimator.py:107-181; the one phase that
    is sampled: its time is scaled by active / sampled hosts), and the
    two-block advance (pools.py:221-249).  DR / TS comparators: the numpy
    oracle pipeline on a 1M-packet sample.  Returns (mean seconds per full
    slice by phase, threads, sample description).
    """
    from oracle import vate_oracle as vo
    threads = len(os.sched_getaffinity(0))
    cfg = vo.OracleConfig(w["g"], w["c"], w["k"], seed=w["seed"], partition=w["partition"])
    tables = (vo.zipf_cdf(w["hosts"]), vo.spreader_cdf()) if w.get("zipf") else None
    n = w["packets"]
    per_step = []
    if kind != "at":
        pipe = vo.OraclePipeline(cfg, w["k_prime"], floor=w["floor"], workers=threads, kind=kind)
        m = min(n, 1_000_000)
        for t in range(warmup + steps):
            a, b = vo.synthetic_slice(t, m, w["hosts"], w["base_aip"])
            t0 = time.perf_counter()
            pipe.scan(a, b)
            t1 = time.perf_counter()
            hosts = np.unique(a)[:1000]
            p = pipe.pool.count_inactive(w["k_prime"])
            g0 = pipe.g0(hosts)
            vo.reports_soa(cfg, hosts, g0, p, t, w["k_prime"])
            t2 = time.perf_counter()
            pipe.pool.advance()
            t3 = time.perf_counter()
            if t >= warmup:
                per_step.append(dict(scan_s=(t1 - t0) * n / m, estimate_s=(t2 - t1) * w["hosts"] / 1000,
                                     maintain_s=t3 - t2))
        pipe.close()
        sample = (f"numpy oracle ({kind} pool), {m:,} of {n:,} packets and g0 of 1,000 hosts "
                  f"per step, both scaled to the full slice")
    else:
        from oracle import native
        pool = vo.OraclePool(w["c"], w["k"], w["partition"]).track_histogram()
        hosts = vo.OracleHostsVec(w["k"])
        scale = []
        for t in range(warmup + steps):
            if tables is not None:
                a, b = vo.synthetic_zipf_slice(t, n, w["hosts"], *tables, base_aip=w["base_aip"])
            else:
                a, b = native.synthetic_slice(t, n, w["hosts"], w["base_aip"])
            t0 = time.perf_counter()
            native.set_cells(pool, native.pair_cells(cfg, a, b))     # scan (estimator.py:96-104)
            hosts.update(a.astype(np.uint32), t)                       # SlidingHostSet.update
            t1 = time.perf_counter()
            act = hosts.active(t, w["k_prime"])
            p = pool.count_inactive(w["k_prime"])
            sub = act[:host_sample] if len(act) > host_sample else act
            t2 = time.perf_counter()
            g0 = native.host_g0(pool, cfg, sub, w["k_prime"])
            rep = vo.reports_soa(cfg, sub, g0, p, t, w["k_prime"])
            if w["floor"] > 0:
                rep = rep.select(rep.estimate >= w["floor"])
            t3 = time.perf_counter()
            pool.advance()
            if t % w["k"] == 0:
                hosts.prune(t)
            t4 = time.perf_counter()
            f = len(act) / max(1, len(sub))
            if t >= warmup:
                scale.append(f)
                per_step.append(dict(scan_s=t1 - t0, estimate_s=(t2 - t1) + (t3 - t2) * f,
                                     maintain_s=t4 - t3))
        sample = (f"oracle port (C half, {threads} threads + numpy): per step one full slice -- "
                  f"all {n:,} packets scanned, host set, Z_p, advance -- with g0 + float path "
                  f"for {min(host_sample, w['hosts']):,} of the ~{w['hosts']:,} active hosts, "
                  f"scaled by x{float(np.mean(scale)):.1f}")
    mean = {k: float(np.mean([s_[k] for s_ in per_step])) for k in per_step[0]}
    mean["slice_s"] = mean["scan_s"] + mean["estimate_s"] + mean["maintain_s"]
    return mean, threads, sample


def run_reference(args, rank, world):
    if rank != 0:
        return
    w = WORKLOAD
    mean, cores, sample = cpu_sample(w, steps=args.steps, kind=args.counter, warmup=args.warmup)
    value = w["packets"] / mean["slice_s"] / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean["slice_s"] * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": _dtype(w),
        "data": "synthetic (oracle.synthetic_slice == csrc k_synth)",
        "config": _config(w, world),
        "path": {"counter": args.counter},
        "phases_ms_per_slice": {k[:-2]: v * 1e3 for k, v in mean.items() if k != "slice_s"},
        "scan_mpps": w["packets"] / mean["scan_s"] / 1e6,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _dtype(w):
    """Cell storage type of the pool (the arithmetic type of the path)."""
    return "u8" if 2 * w["k"] <= 254 else ("u16" if 2 * w["k"] <= 65534 else "u32")


def _config(w, world):
    per_gpu = w["packets"] // world if w.get("strong") else w["packets"]
    return {"workload": w["name"], "c": w["c"], "k": w["k"], "k_prime": w["k_prime"],
            "g": w["g"], "hosts": w["hosts"], "packets_per_slice_per_gpu": per_gpu,
            "packets_per_slice_total": per_gpu * world,
            "floor": w["floor"], "partition": w["partition"], "seed": w["seed"],
            "parallelism": f"dp{world}" if world > 1 else "single",
            "l2": _l2_note(w)}


def _l2_note(w):
    """How the timed region relates to the 126 MB L2 (timing rule: say which)."""
    cb = 1 if 2 * w["k"] <= 254 else 2
    pool_mib = (1 << w["c"]) * cb / 2**20
    total = w["packets"] * 8 / 1e6
    inputs = (f"every slice distinct ({total:.1f} MB of packets each, pre-generated; the timed "
              f"region streams > L2 of never-reused input)" if total <= 256 else
              f"slices of {total:.0f} MB cycle through a ring of 24 distinct ones (19 GB, "
              f">> L2: no input is L2-hot)")
    return (inputs + f"; the {pool_mib:.0f} MiB pool "
            + ("stays L2-resident by design" if pool_mib <= 64 else "exceeds L2 (HBM-bound)"))


# ----------------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------------

def run_gpu(args, rank, world, local_rank):
    import torch
    import paper_1812_00282_b200 as vb
    from paper_1812_00282_b200 import _lib
    from paper_1812_00282_b200._lib import lib, check
    from paper_1812_00282_b200.parallel import PeerStep, ReplicaStep

    dist = None
    # --share-device (functional check only): every rank on cuda:0, gloo plumbing
    dev = 0 if args.share_device else local_rank
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(dev)
        if args.share_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    w = WORKLOAD
    cfg = vb.EstimatorConfig(w["g"], w["c"], w["k"], seed=w["seed"], partition=w["partition"],
                             counter_kind=args.counter)
    pool = cfg.build_pool(device=dev)
    pipe = vb.Pipeline(pool, cfg, w["k_prime"], floor=w["floor"])
    h = pool.handle
    check(lib.vate_pool_set_option(h, 0, ("auto", "gather", "smem").index(args.g0_kernel)))
    pool.set_option("incremental", 1 if args.incremental == "on" else 0)
    # scan form: auto (the library picks the registry-stamp filter for skewed
    # traffic) unless forced
    scan_filter = args.scan_filter
    if scan_filter != -1:
        pool.set_option("scan_filter", scan_filter)
    if args.deferred != -1:
        pool.set_option("deferred", args.deferred)
    if args.bitplane != -1:
        pool.set_option("bitplane", args.bitplane)
    pool.set_option("concurrent", args.concurrent)
    for kv in args.opt:                       # experiments: --opt spin_wait=0 ...
        name, val = kv.split("=")
        pool.set_option(name, int(val))
    # strong-scaling workloads fix the packets per slice of the whole job
    n = w["packets"] // world if w.get("strong") else w["packets"]
    slice_bytes = n * 8
    torch.cuda.set_device(dev)
    # Every slice of the run is distinct (no ring reuse): a repeated slice would
    # re-set only cells that are already active and hide the real per-slice churn
    # of the inactive bitmap.  Slices are generated on the device before the timed
    # regions (k_synth == oracle.synthetic_slice), 40 MB each, >> L2 in total.
    t_base = 1000 * rank
    prefill = 2 * w["k"]
    zt = None
    if w.get("zipf"):
        from paper_1812_00282_b200.synth import ZipfTables
        zt = ZipfTables(dev, w["hosts"])

    def synth(t_, out_ptr):
        if zt is not None:
            zt.packets(pool, t_, n, w["base_aip"], w["seed"], out_ptr)
        else:
            check(lib.vate_synth_packets(h, t_, n, w["hosts"], w["base_aip"], w["seed"], out_ptr))
    # distinct device slices; 800 MB slices (cfg 5) cycle through a ring of 24 (19 GB,
    # >> L2, so the timed region still never finds its input in L2)
    n_dev = args.warmup + 2 * args.steps
    if slice_bytes > (256 << 20):
        n_dev = min(n_dev, 24)
    scratch = torch.empty((n, 2), dtype=torch.int32, device=f"cuda:{dev}")
    dslices = torch.empty((n_dev, n, 2), dtype=torch.int32, device=f"cuda:{dev}")
    for i in range(n_dev):
        synth(t_base + prefill + i, dslices[i].data_ptr())
    # e2e host slices (pinned): every one distinct; 800 MB slices (cfg 5) capped at 4
    n_host = args.warmup + (args.steps if slice_bytes <= (256 << 20) else min(args.steps, 4))
    hslices = torch.empty((n_host, n, 2), dtype=torch.int32, pin_memory=True)
    for i in range(n_host):
        synth(t_base + prefill + n_dev + i, scratch.data_ptr())
        pool.synchronize()
        hslices[i].copy_(scratch)
    pool.synchronize()
    nh_cap = w["hosts"] + 1024   # (+ cfg 3's 64 super-spreaders)

    def pinned_outs():
        return (torch.empty(nh_cap, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64),
                torch.empty(nh_cap, dtype=torch.float64, pin_memory=True).numpy(),
                torch.empty(nh_cap, dtype=torch.float64, pin_memory=True).numpy(),
                torch.empty(nh_cap, dtype=torch.uint8, pin_memory=True).numpy())
    out_sets = (pinned_outs(), pinned_outs())   # reports double-buffered across slices
    outs = out_sets[0]

    # N > 1: replica merge + host exchange + this rank's share of the estimate
    replica = None
    if world > 1 and args.exchange == "p2p":     # fused merge over peer memory (NVLink)
        replica = PeerStep(pipe, dist, key_cap=n, mode=("auto", "one", "two").index(args.p2p_mode))
    elif world > 1:                               # NCCL all-gathers + merge kernel
        replica = ReplicaStep(pipe, dist, torch)
    run_slice = replica if replica is not None else pipe.step_fast
    # the pipelined step: one GPU, or N GPUs with the peer-memory exchange run
    # inside it (PeerStep.bind_lagged); the NCCL form stays one call per slice
    lagged = bool(args.lagged) and (replica is None or args.exchange == "p2p")
    if lagged and replica is not None:
        replica.bind_lagged()

    def _lagged_rows(res):
        return None if res is None else res[1]

    if lagged:   # software-pipelined step: slice t-1 completes beside slice t's scan
        def run_slice(t_, src_, n_, where_, out_):
            return _lagged_rows(pipe.step_lagged(t_, src_, n_, where_, out_))

    def flush(out=None):
        """Complete the pending slice of a lagged run (no-op otherwise)."""
        if lagged:
            rep = _lagged_rows(pipe.flush_lagged(out))
            return 0 if rep is None else (rep if out is None else len(rep))
        return 0

    def step(t, src, on_device):
        """One slice; report rows stay in HBM (e2e moves them); returns the row count."""
        rep = run_slice(t, src, n, "device" if on_device else "host", None)
        return 0 if rep is None else rep

    def step_host(t, i):
        """e2e slice from pinned host packets; slice i+1's H2D overlaps slice i."""
        rep = run_slice(t, staged[i % 2], n, "staged", out_sets[t % 2])
        return 0 if rep is None else len(rep)

    t = 0
    for _ in range(prefill):             # fill the window: every block swept twice
        synth(t_base + t, scratch.data_ptr())
        step(t, scratch.data_ptr(), True)
        t += 1
    di = 0
    for _ in range(args.warmup):
        step(t, dslices[di % n_dev].data_ptr(), True)
        t += 1
        di += 1

    flush()

    def barrier():
        pipe.wait_reports()
        torch.cuda.synchronize(dev)
        pool.synchronize()
        if dist is not None:
            dist.barrier()

    # --- device-resident inputs (value) ---------------------------------------------
    pool.set_timing(False)
    barrier()
    launches0 = pool.launches()
    inc0 = pool.inc_stats()
    profile_region = os.environ.get("VATE_PROFILE_REGION") == "1"
    with ClockSampler(dev) as clocks:
        if profile_region:
            check(lib.vate_profiler(1))
        check(lib.vate_mark(h, 0))
        rows = 0
        for _ in range(args.steps):
            rows += step(t, dslices[di % n_dev].data_ptr(), True)
            t += 1
            di += 1
        rows += flush()                  # the last slice's reports are part of the work
        check(lib.vate_mark(h, 1))
        barrier()
        if profile_region:
            check(lib.vate_profiler(0))
        ms = C.c_double()
        check(lib.vate_mark_elapsed(h, 0, 1, C.byref(ms)))
        dev_ms = ms.value
        launches = pool.launches() - launches0
        inc1 = pool.inc_stats()

        # --- per-kernel breakdown (separate pass, CUDA events around each launch) -----
        pool.set_timing(True)
        for _ in range(args.steps):
            step(t, dslices[di % n_dev].data_ptr(), True)
            t += 1
            di += 1
        flush()
        barrier()
        kt = {kind: pool.kernel_time(kind) for kind in _lib.KERNEL_KINDS}
        pool.set_timing(False)

        # --- end to end from pinned host buffers (e2e) --------------------------------
        # e2e warm-up: W host-fed slices (PCIe link and staging buffers warm)
        staged = [None, None]
        staged[0] = pipe.stage_packed(hslices[0].data_ptr(), n)
        for i in range(args.warmup):
            if i + 1 < args.warmup:
                staged[(i + 1) % 2] = pipe.stage_packed(hslices[i + 1].data_ptr(), n)
            step_host(t, i)
            t += 1
        flush(out_sets[t % 2])
        barrier()
        e0 = time.perf_counter()
        e2e_rows = 0
        host_ms = {"stage": 0.0, "step": 0.0}
        # every timed slice's H2D is inside the timed region, the first one too
        staged[args.warmup % 2] = pipe.stage_packed(hslices[args.warmup].data_ptr(), n)
        for i in range(args.warmup, n_host):
            a = time.perf_counter()
            if i + 1 < n_host:
                staged[(i + 1) % 2] = pipe.stage_packed(hslices[i + 1].data_ptr(), n)
            b = time.perf_counter()
            e2e_rows += step_host(t, i)
            host_ms["stage"] += (b - a) * 1e3
            host_ms["step"] += (time.perf_counter() - b) * 1e3
            t += 1
        e2e_rows += flush(out_sets[t % 2])
        barrier()
        e2e_s = time.perf_counter() - e0

    max_ms = dev_ms
    max_e2e = e2e_s
    if dist is not None:
        v = torch.tensor([dev_ms, e2e_s], dtype=torch.float64,
                         device="cpu" if args.share_device else f"cuda:{dev}")
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        max_ms, max_e2e = float(v[0]), float(v[1])
    total_packets = n * world * args.steps
    e2e_steps = n_host - args.warmup
    value = total_packets / (max_ms / 1e3) / 1e6
    e2e_value = n * world * e2e_steps / max_e2e / 1e6
    if rank != 0:
        _teardown(dist)
        return

    # --- after the timed regions (rank 0): latency, the list API, ceilings -----------
    extra = {}
    if world == 1 and args.counter == "at":
        extra = after_timing(args, w, vb, pipe, pool, n, t, dslices, n_dev, di, out_sets, lagged)
        t = extra.pop("_t")
    pcie = pcie_ceiling(torch, dev, hslices[0], int(e2e_rows / e2e_steps * 25), n)

    # speed of light of the scan's memory pattern on this pool shape: one random
    # 32-B registry-sized load + one random cell store per packet, no hashing,
    # no input stream (scratch pool; csrc vate_bench_sol_scatter)
    scratch_pool = vb.AtPool(w["c"], w["k"], w["partition"], device=dev)
    table_bytes = 16 * (1 << max(12, (2 * w["hosts"] - 1).bit_length()))
    sol_ms = C.c_double()
    check(lib.vate_bench_sol_scatter(scratch_pool.handle, n, table_bytes, 10, C.byref(sol_ms)))
    l2 = scratch_pool.l2_ceilings()
    # the deferred scan's own skeleton: the packet stream, one red.or into the
    # 2^c-bit mark bitmap and one registry home-sector read per packet, on the
    # scan's grid (vate_bench_scan_skeleton)
    skel_ms = scratch_pool.scan_skeleton_ms(w["c"], table_bytes, n - n % 2)
    scratch_pool.close()
    sol = {"ms_per_slice_of_packets": sol_ms.value, "registry_table_bytes": table_bytes,
           "pool_bytes": (1 << w["c"]) * pool.cell_bytes,
           "deferred_skeleton_ms": skel_ms}

    peaks, peak_src = _peaks()
    hbm = float(peaks["hbm_gbs"])
    per_kind = {k: {"ms_total": v[0], "launches": v[1],
                    "ms_per_launch": (v[0] / v[1] if v[1] else 0.0)} for k, v in kt.items()}
    nh = pipe.last_active
    S = 1 << w["c"]
    cb = pool.cell_bytes
    mode = pool.mode()
    deferred, bitplane = mode["deferred"], mode["bitplane"]
    inc_on = args.incremental == "on"
    nblocks = 2 * w["k"]
    block_words = (S // nblocks + 31) // 32
    # algorithmic bytes per launch: the scan 40 B per
    # packet (8 B streamed pair + one 32-B sector for its scattered cell write);
    # the pool pass reads every cell and writes the bitmap, plus the previous
    # bitmap (incremental delta) and the pending marks (deferred pools)
    # bit-plane mode: the pass reads S, P, M_e (+ the previous bitmap) and writes
    # the bitmap and P, 2^c/8 bytes each; the due-block work reads the two blocks'
    # k pending epochs of marks and reads + writes their cells
    alg_bytes = {
        "scan": n * 40,
        "bitmap": ((S // 8) * (5 + (1 if inc_on else 0)) if bitplane else
                   S * cb + S // 8 + (S // 8 if inc_on else 0) + (S // 8 if deferred else 0)),
        "g0": (nh * (32 * w["g"] + 12) if not inc_on else None),
        "sweep": ((w["k"] * block_words * 4 + 2 * cb * pool.max_block_size) if bitplane else
                  2 * cb * 2 * pool.max_block_size if args.counter == "at" else
                  2 * cb * S if args.counter == "dr" else 0),
        "final": nh * (4 + 8 + 8 + 8 + 8 + 1),
        "registry": nh * 32,
        "sort": nh * 8 * 4 * 2,
        "other": 0,
    }
    for kind, v in per_kind.items():   # the same accounting for every kernel, for context
        if v["ms_per_launch"] and alg_bytes.get(kind):
            v["alg_gbs"] = alg_bytes[kind] / (v["ms_per_launch"] / 1e3) / 1e9
            v["frac_of_hbm"] = v["alg_gbs"] / hbm
    # the dominant kernel: largest event time among the main-stream kernels (the
    # aux-stream ones run beside them; profiles/*launches* has the serialised view)
    main_stream = ("scan", "bitmap", "g0") if not inc_on else ("scan", "bitmap")
    checked = pool.scan_form() == 1
    rooflines = {k: _roofline(k, per_kind[k], alg_bytes[k], hbm, peak_src, l2, n, S, cb, w,
                              deferred, args.config, bitplane, checked)
                 for k in main_stream if alg_bytes.get(k) and per_kind[k]["ms_per_launch"]}
    dom = max(rooflines, key=lambda k: per_kind[k]["ms_total"])
    step_ms = max_ms / args.steps
    cpu = cpu_sample(w, steps=1, kind=args.counter) if world == 1 else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong" if w.get("strong") else "weak", "vs_baseline": None,
        "dtype": _dtype(w),
        "data": "synthetic (csrc k_synth == oracle.synthetic_slice)",
        "config": _config(w, world),
        "path": {"counter": args.counter,
                 "scan_filter": {-1: "auto (registry-stamp filter at >= 8 packets per host)",
                                 0: "off", 1: "on"}[args.scan_filter],
                 "deferred_scatter": deferred, "bitplane": bitplane,
                 "bitplane_window": mode["window"] if bitplane else None,
                 "incremental_g0": inc_on,
                 "slice_step": "lagged (Pipeline.step_lagged)" if lagged else "Pipeline.step_fast"},
        "roofline": rooflines[dom],
        "rooflines": rooflines,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": slice_bytes,
                "d2h_bytes_per_step": int(e2e_rows / e2e_steps * 25),
                "steps": e2e_steps,
                "host_ms_per_step": {k: v / e2e_steps for k, v in host_ms.items()},
                "pcie": dict(pcie, frac=e2e_value / pcie["ceiling_value"])},
        "gpu_launches": int(launches),
        **extra,
        "scan_update_mpps": n / ((per_kind["scan"]["ms_total"] + per_kind["sweep"]["ms_total"])
                                 / args.steps / 1e3) / 1e6,
        "reports_per_slice": nh,
        "maintain_note": (("AT: the two due blocks (pools.py:221-249)" +
                           ("" if per_kind["sweep"]["launches"] else
                            ", swept inside the pool pass (no separate launch)"))
                          if args.counter == "at" else
                          "DR: every cell slides (pools.py:339-349)" if args.counter == "dr" else
                          "TS: no maintenance (pools.py:399-401)"),
        "kernels": per_kind,
        "kernels_note": "CUDA-event time per launch on each kernel's own stream; aux-stream "
                        "kernels (registry compaction, delta apply, float path) overlap the "
                        "scan or the pool pass and their times include that overlap; "
                        "profiles/*launches* has the serialised ncu times",
        "l2_ceilings": l2,
        "scan_speed_of_light": dict(sol, scan_ms_per_launch=per_kind["scan"]["ms_per_launch"],
                                    scan_over_sol=per_kind["scan"]["ms_per_launch"]
                                    / (skel_ms if deferred else sol["ms_per_slice_of_packets"]),
                                    note="direct pools: random 32-B load (registry-sized "
                                         "table) + random cell store per packet, no hashing "
                                         "or packet stream; deferred pools "
                                         "(deferred_skeleton_ms): the packet stream + one "
                                         "random red.or into the 2^c-bit mark bitmap + one "
                                         "random registry sector read per packet on the "
                                         "scan's grid, i.e. the scan's memory operations "
                                         "without its hashing and compare chain"),
        "active_set_ordering": pool.sort_stats(),
        "incremental": {"enabled": inc_on,
                        **{k: inc1[k] - inc0[k] for k in ("rebuilds", "delta_slices",
                                                          "refresh_slices", "full_slices",
                                                          "extends")},
                        "last_delta_cells": inc1["last_delta_cells"],
                        "last_delta_work": inc1["last_delta_work"],
                        "identity_slices": inc1["identity_slices"] - inc0["identity_slices"],
                        "hosts_indexed": inc1["hosts_indexed"],
                        "rebuild_ms_total_run": inc1["rebuild_us_total"] / 1e3,
                        "misses_since_rebuild": inc1["miss_accum"]},
        "clocks": clocks.summary(),
    }
    if world > 1:
        line["exchange"] = {"kind": args.exchange,
                            **(replica.info() if args.exchange == "p2p" else {})}
        if args.share_device:
            line["config"]["parallelism"] += " (ranks share cuda:0: functional check, not scaling)"
    if cpu is not None:
        cpu_mean, cores, sample = cpu
        line["cpu_baseline"] = {"value": w["packets"] / cpu_mean["slice_s"] / 1e6, "unit": UNIT,
                                "cores": cores, "kind": "port", "sample": sample}
    print(json.dumps(line), flush=True)
    _teardown(dist)


def _roofline(kind, k, alg, hbm, peak_src, l2, n, S, cb, w, deferred, cfg, bitplane=False,
              checked=False):
    """One kernel's roofline: HBM (algorithmic bytes / launch time against the
    measured copy bandwidth; `bound` stays "hbm", the contract's memory bound)
    and, for work L2 serves, `l2`: the time the L2 probes need for the
    kernel's random accesses (or its stream) over the launch time, with
    `binding` set when L2, not HBM, is what limits the kernel."""
    t = k["ms_per_launch"] / 1e3
    achieved = alg / t / 1e9
    r = {"bound": "hbm", "kernel": kind, "achieved": achieved, "peak": hbm,
         "peak_source": peak_src, "unit": "GB/s", "frac": achieved / hbm,
         "traffic": _ncu_traffic(kind, cfg, bitplane),
         "traffic_source": "profiles/*ncu_kernels.txt (ncu --set full, one launch)",
         "algorithmic_bytes_per_launch": alg}
    pool_in_l2 = S * cb <= (64 << 20)
    if kind == "scan":
        # per packet: one random sector read of the host registry and its cell
        # write -- a red.or into the L2-resident mark bitmap when deferred (for
        # skewed traffic the stamp-filter form reads the mark word first and
        # issues the red only for a new mark: counted as a read, a lower bound),
        # a random store into an L2-resident pool otherwise; beyond L2 a direct
        # store is the HBM sector above
        reads = l2["random_sector_reads_G_per_s"] * 1e9
        if deferred:
            write_rate = reads if checked else l2["random_red_or_G_per_s"] * 1e9
        else:
            write_rate = l2["random_u16_stores_G_per_s"] * 1e9
        t_l2 = n / reads
        if deferred or pool_in_l2:
            t_l2 += n / write_rate
        r["l2"] = {"ceiling_ms": t_l2 * 1e3, "frac": t_l2 / t,
                   "model": "n random 32-B registry reads + n random cell writes "
                            "(red.or marks when deferred; mark-word reads in the "
                            "stamp-filter form) at the probed L2 rates",
                   "binding": bool(deferred or pool_in_l2)}
    elif kind == "bitmap" and pool_in_l2:
        t_l2 = (S * cb + 3 * S // 8) / (l2["stream_read_GB_per_s"] * 1e9)
        r["l2"] = {"ceiling_ms": t_l2 * 1e3, "frac": t_l2 / t,
                   "model": "the pool and bitmaps streamed at the probed L2 read rate",
                   "binding": True}
    elif kind == "g0":
        t_l2 = w["g"] * (alg / (32 * w["g"] + 12)) / (l2["random_sector_reads_G_per_s"] * 1e9)
        r["l2"] = {"ceiling_ms": t_l2 * 1e3, "frac": t_l2 / t,
                   "model": "g random 32-B bitmap reads per host at the probed L2 rate",
                   "binding": True}
        # the gathers hit the L2-resident bitmap: their ceiling is the L2's
        # random-sector rate, not HBM (the HBM figures stay alongside)
        l2_gbs = l2["random_sector_reads_G_per_s"] * 32
        r.update({"hbm_peak": hbm, "hbm_frac": achieved / hbm, "peak": l2_gbs,
                  "peak_source": "measured L2 probe: random 32-B sector reads (l2_ceilings)",
                  "frac": achieved / l2_gbs})
    return r


def after_timing(args, w, vb, pipe, pool, n, t, dslices, n_dev, di, out_sets, lagged):
    """Measurements after the timed regions (rank 0, N = 1): the per-slice
    estimate latency (CUDA events from the end of a slice's scan to its SoA
    report rows in pinned host memory) for the one-call step
    with the incremental g0 and with the full recompute, and for the lagged
    step; then the reference's own list API (Pipeline.process_slice from u64
    host arrays -> list[EstimateReport], pipeline.py:142-166), with the
    EstimateReport materialisation timed apart."""
    import torch
    res = {}

    def lat_run(fn, m):
        nonlocal t
        for i in range(2):   # unmeasured: index rebuilds after a switch land here
            fn(t, dslices[(di + i) % n_dev].data_ptr(), n, "device", out_sets[t % 2])
            t += 1
        pipe.wait_reports()
        pool.set_latency(True)
        for i in range(m):
            fn(t, dslices[(di + i) % n_dev].data_ptr(), n, "device", out_sets[t % 2])
            t += 1
        pipe.wait_reports()
        r = pool.latency()
        pool.set_latency(False)
        return r

    def fast(t_, ptr_, n_, where, out):
        rep = pipe.step_fast(t_, ptr_, n_, where, out)
        pipe.wait_reports()
        return rep

    m = 6
    res_lat = {"definition": "CUDA events: end of the slice's scan (compute stream) -> its "
                             "SoA report rows (host, estimate, z_v, saturated) landed in "
                             "pinned host memory (copy stream)",
               "hosts": None}
    res_lat["step_fast_incremental"] = lat_run(fast, m)
    res_lat["hosts"] = pipe.last_active
    inc_was = args.incremental == "on"
    pool.set_option("incremental", 0)
    res_lat["step_fast_full_recompute"] = lat_run(fast, m)
    pool.set_option("incremental", 1 if inc_was else 0)
    if lagged:
        lat = lat_run(lambda *a: pipe.step_lagged(*a), m)
        pipe.flush_lagged(out_sets[t % 2])
        pipe.wait_reports()
        lat["note"] = ("the lagged step completes slice t during the call for slice t+1, "
                       "so this includes the next slice's scan")
        res_lat["step_lagged"] = lat
    res["estimate_latency_ms"] = res_lat

    # the reference's list API from u64 host arrays (two slices)
    rows = []
    for i in range(2):
        pr = dslices[(di + i) % n_dev].cpu().numpy().view(np.uint32)
        a, b = pr[:, 0].astype(np.uint64), pr[:, 1].astype(np.uint64)
        t0 = time.perf_counter()
        soa, stats = pipe.process_slice_soa(t, a, b)
        t1 = time.perf_counter()
        lst = [] if soa is None else soa.to_list()
        t2 = time.perf_counter()
        rows.append({"slice_ms": (t1 - t0) * 1e3, "to_list_ms": (t2 - t1) * 1e3,
                     "reports": len(lst), "slice_stats_us": {"scan": stats.scan_us,
                                                              "estimate": stats.estimate_us,
                                                              "maintain": stats.maintain_us}})
        t += 1
        del lst
    res["list_api"] = {
        "call": "Pipeline.process_slice(t, u64 aips, u64 bips) -> list[EstimateReport]",
        "slices": rows,
        "mpps_without_objects": n / (np.mean([r["slice_ms"] for r in rows]) / 1e3) / 1e6,
        "mpps_with_objects": n / (np.mean([r["slice_ms"] + r["to_list_ms"] for r in rows]) / 1e3)
                             / 1e6,
        "note": "the u64 arrays (16 B per packet) cross PCIe each slice; the 1M Python "
                "EstimateReport objects are the reference's own output type"}
    res["_t"] = t
    return res


def pcie_ceiling(torch, dev, src_pinned, d2h_bytes, n, reps=10):
    """What PCIe alone allows the e2e line: the step's H2D (this slice's packets
    from pinned memory) and D2H (its report rows into pinned memory) bytes as
    bare copies, alone and on two streams at once (CUDA events, no kernels).
    The concurrent pair bounds an e2e slice from below."""
    nbytes = src_pinned.numel() * src_pinned.element_size()
    h_src = src_pinned.reshape(-1).view(torch.uint8)
    d_dst = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{dev}")
    d_src = torch.empty(max(d2h_bytes, 1), dtype=torch.uint8, device=f"cuda:{dev}")
    h_dst = torch.empty(max(d2h_bytes, 1), dtype=torch.uint8, pin_memory=True)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(h2d, d2h):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize(dev)
        cur = torch.cuda.current_stream(dev)
        ev[0].record(cur)
        s_in.wait_stream(cur)
        s_out.wait_stream(cur)
        for _ in range(reps):
            if h2d:
                with torch.cuda.stream(s_in):
                    d_dst.copy_(h_src, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s_out):
                    h_dst.copy_(d_src, non_blocking=True)
        cur.wait_stream(s_in)
        cur.wait_stream(s_out)
        ev[1].record(cur)
        torch.cuda.synchronize(dev)
        return ev[0].elapsed_time(ev[1]) / reps

    timed(True, True)  # warm
    # a ceiling: the best of three trials each (shared PCIe / host-memory noise)
    h2d_ms = min(timed(True, False) for _ in range(3))
    d2h_ms = min(timed(False, True) for _ in range(3))
    both_ms = min(timed(True, True) for _ in range(3))
    return {"h2d_gbs": nbytes / h2d_ms / 1e6, "d2h_gbs": d2h_bytes / d2h_ms / 1e6,
            "h2d_plus_d2h_ms_per_slice": both_ms,
            "ceiling_value": n / (both_ms / 1e3) / 1e6,
            "note": "bare pinned copies of one step's H2D and D2H bytes on two streams (CUDA "
                    "events): the PCIe bound on the e2e value"}


def _teardown(dist):
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("vate", "reference"), default="vate")
    ap.add_argument("--g0-kernel", choices=("auto", "gather", "smem"), default="auto",
                    help="g0 gather variant (VATE_OPT_G0)")
    ap.add_argument("--scan-filter", type=int, choices=(-1, 0, 1), default=-1,
                    help="per-CTA registry-stamp filter in the scan (VATE_OPT_SCAN_FILTER)")
    ap.add_argument("--deferred", type=int, choices=(-1, 0, 1), default=-1,
                    help="deferred scatter: scans mark an L2-resident pending-set bitmap and "
                         "the pool pass stores the clocks (VATE_OPT_DEFERRED; auto: cells > 64 MiB)")
    ap.add_argument("--hosts", type=int, default=0,
                    help="override the workload's host count (experiments; not a BASELINE shape)")
    ap.add_argument("--bitplane", type=int, choices=(-1, 0, 1), default=-1,
                    help="bit-plane mode for deferred pools (VATE_OPT_BITPLANE; auto: on)")
    ap.add_argument("--opt", action="append", default=[],
                    help="extra pool option name=value (AtPool.set_option), for A/B runs")
    ap.add_argument("--lagged", type=int, choices=(0, 1), default=1,
                    help="software-pipelined slice step (Pipeline.step_lagged): slice t's "
                         "reports complete beside slice t+1's scan")
    ap.add_argument("--concurrent", type=int, choices=(0, 1), default=1,
                    help="registry compaction beside the bitmap pass, advance beside g0 + float "
                         "path, on a second stream (VATE_OPT_CONCURRENT)")
    ap.add_argument("--config", choices=sorted(WORKLOADS), default="cfg4",
                    help="workload shape (BASELINE.json configs); cfg4 is the headline")
    ap.add_argument("--incremental", choices=("on", "off"), default="on",
                    help="exact incremental g0 through the inverse index (VATE_OPT_INCREMENTAL)")
    ap.add_argument("--counter", choices=("at", "dr", "ts"), default="at",
                    help="counter pool: AT (the product) or the DR / TS comparators "
                         "(pools.py:301-410) for the paper's maintenance contrast")
    ap.add_argument("--exchange", choices=("p2p", "nccl"), default="p2p",
                    help="N > 1 slice exchange: fused peer-memory merge (default) or NCCL "
                         "all-gathers + merge kernel")
    ap.add_argument("--p2p-mode", choices=("auto", "one", "two"), default="auto",
                    help="peer merge form: one-shot, two-shot, or auto (two-shot above 2 ranks)")
    ap.add_argument("--share-device", action="store_true",
                    help="run every rank on cuda:0 over gloo (exercises the N > 1 path on "
                         "one GPU; not a scaling measurement)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be at least 3")
    global WORKLOAD
    WORKLOAD = dict(WORKLOADS[args.config])
    if args.hosts:   # experiments only: the line then names a non-BASELINE workload
        WORKLOAD["hosts"] = args.hosts
        WORKLOAD["name"] += f"-hosts{args.hosts}"
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_gpu(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
