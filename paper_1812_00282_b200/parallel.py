"""Multi-GPU slice processing: one process per GPU.

The packet stream shards across ranks; every rank scans its shard into a
private replica pool.  Replicas share bact0 and hold identical cells at slice
start, so the only per-slice exchange is "which cells were set this slice":
each rank builds a 1-bit-per-cell dirty bitmap on the device
(vate_dirty_bitmap), the bitmaps are all-gathered (NCCL over NVLink), and
every rank ORs them and writes its block clock into the dirty cells
(vate_merge_dirty).  That is the reference's single-pool state exactly (the
window-aware newest-timestamp max of SURVEY.md §8e).

Host estimation then splits by aip range: the union of the ranks' active host
sets is sorted, rank r estimates the r-th contiguous range, and concatenating
the ranks' reports in rank order gives the reference's ascending host order
(pipeline.py:57).

The pure functions here (``split_range``, ``union_sorted``) are shared with
the CPU tests, which run the same protocol over gloo with the oracle as the
per-rank pool (tests/test_multirank_cpu.py).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import VATE_HOST, check, lib, ptr
from .estimator import HostReports, log_zp


def union_sorted(parts) -> np.ndarray:
    """Sorted union of per-rank sorted host arrays."""
    parts = [np.asarray(p, dtype=np.uint64) for p in parts if len(p)]
    if not parts:
        return np.zeros(0, dtype=np.uint64)
    return np.unique(np.concatenate(parts))


def split_range(n: int, rank: int, world: int):
    """[lo, hi) of the rank's contiguous share of n sorted hosts."""
    return (n * rank) // world, (n * (rank + 1)) // world


def all_gather_hosts(local: np.ndarray, dist, device) -> list:
    """Variable-length all-gather of uint64 host arrays (sizes first, then padded)."""
    import torch
    world = dist.get_world_size()
    n = torch.tensor([len(local)], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(s.item()) for s in sizes]
    cap = max(sizes + [1])
    buf = torch.zeros(cap, dtype=torch.int64, device=device)
    if len(local):
        buf[: len(local)] = torch.from_numpy(local.view(np.int64)).to(device)
    bufs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf)
    return [b[:s].cpu().numpy().view(np.uint64) for b, s in zip(bufs, sizes)]


def range_split_estimate(pipe, t: int, outs, dist, torch) -> HostReports | None:
    """Estimate this rank's aip range of the global active set (device pool merged)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    device = f"cuda:{pipe.pool.device}"
    local = pipe.hosts.active(t, pipe.k_prime)
    hosts = union_sorted(all_gather_hosts(local, dist, device))
    lo, hi = split_range(len(hosts), rank, world)
    mine = np.ascontiguousarray(hosts[lo:hi])
    p = C.c_uint64()
    check(lib.vate_estimate_begin_hosts(pipe.pool.handle, ptr(mine), mine.size, VATE_HOST,
                                        pipe.cfg.g, pipe.cfg.cell_stream, pipe.k_prime,
                                        C.byref(p)))
    if mine.size == 0:
        return None
    lzp, z_p = log_zp(p.value, pipe.pool.size)
    host, est, zv, sat = outs
    kept = C.c_uint64()
    check(lib.vate_estimate_finish(pipe.pool.handle, pipe.cfg.g, p.value, lzp, float(pipe.floor),
                                   ptr(host), ptr(est), ptr(zv), ptr(sat), len(host),
                                   C.byref(kept)))
    m = kept.value
    pipe.last_pool_inactive = p.value
    pipe.last_active = len(hosts)
    return HostReports(host[:m], est[:m], zv[:m], sat[:m].view(bool), z_p,
                       t - pipe.k_prime + 1, pipe.k_prime)
