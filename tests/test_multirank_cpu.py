"""The N>1 protocol on CPU: world_size 2 over gloo, oracle pools per rank.

Each rank scans its round-robin shard of every slice into a private replica
pool, replicas merge through an all-gather of dirty bitmaps (cells that hold
their block clock), the hosts each rank saw this slice are all-gathered and
registered everywhere, every rank range-splits the (now identical) sorted
active set, and rank-ordered concatenation of the per-rank reports must equal
a single pool fed every packet -- snapshots, host sets, host order and floats,
slice by slice.  The device path (paper_1812_00282_b200.parallel.ReplicaStep,
bench.py --gpus N) runs the same protocol with vate_dirty_bitmap /
vate_merge_dirty / vate_hosts_touched / vate_estimate_begin_part over NCCL.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dirty_bits(pool):
    """1 bit per cell: the cell holds its own block clock (set this slice)."""
    dirty = (pool.cells.astype(np.int64) == pool.cell_clocks()).astype(np.uint8)
    return np.packbits(dirty, bitorder="little")


def _merge(pool, gathered):
    bits = np.bitwise_or.reduce(np.stack(gathered), axis=0)
    dirty = np.unpackbits(bits, bitorder="little")[: pool.size].astype(bool)
    pool.cells[dirty] = pool.cell_clocks()[dirty].astype(np.uint32)


def _gather_varlen(keys):
    """Sizes first, then a padded all-gather (the shape ReplicaStep uses on NCCL)."""
    world = dist.get_world_size()
    n = torch.tensor([len(keys)], dtype=torch.int64)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(x) for x in sizes]
    cap = max(sizes + [1])
    buf = torch.zeros(cap, dtype=torch.int64)
    buf[: len(keys)] = torch.from_numpy(np.asarray(keys, dtype=np.uint64).view(np.int64))
    bufs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf)
    return [b[:m].numpy().view(np.uint64) for b, m in zip(bufs, sizes)]


def _worker(rank, world, port, result_q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle import vate_oracle as vo
    from paper_1812_00282_b200.parallel import split_range, union_sorted

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = vo.OracleConfig(256, 14, 6, seed=2)
    kp = 5
    pool = vo.OraclePool(14, 6)
    hosts = vo.OracleHosts(6)
    ref = vo.OraclePipeline(cfg, kp) if rank == 0 else None
    rng = np.random.default_rng(0)
    ok = True
    for t in range(20):
        n = int(rng.integers(0, 3000)) if t != 4 else 0
        a = (0x0A000000 + rng.integers(0, 400, n)).astype(np.uint64)
        b = rng.integers(1, 1 << 32, n).astype(np.uint64)
        mine = slice(rank, None, world)
        pool.set_cells(cfg.pair_cells(a[mine], b[mine]))
        if len(a[mine]):
            hosts.update(a[mine], t)
        touched = np.unique(a[mine])     # what vate_hosts_touched returns here
        # replica merge
        bits = _dirty_bits(pool)
        gathered = [torch.zeros(len(bits), dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(bits))
        _merge(pool, [g.numpy() for g in gathered])
        # every registry absorbs the others' touched hosts -> identical host sets
        for r, keys in enumerate(_gather_varlen(touched)):
            if r != rank and len(keys):
                hosts.update(keys, t)
        union = hosts.active(t, kp)
        everyone = _gather_varlen(union)
        ok &= all(np.array_equal(x, union) for x in everyone)
        ok &= np.array_equal(union, union_sorted(everyone))
        # aip-range-split estimate
        lo, hi = split_range(len(union), rank, world)
        part = union[lo:hi]
        rep = None
        if len(union):
            p = pool.count_inactive(kp)
            rep = vo.reports_soa(cfg, part, vo.host_g0(pool, cfg, part, kp), p, t, kp)
        parts = [None] * world
        dist.all_gather_object(parts, None if rep is None else
                               (rep.host, rep.estimate, rep.z_v, rep.saturated))
        pool.advance()
        if t % 6 == 0:
            hosts.prune(t)
        if rank == 0:
            want = ref.process_slice(t, a, b)
            if want.reports is None:
                ok &= all(x is None for x in parts) or len(union) == 0
            else:
                host = np.concatenate([x[0] for x in parts if x is not None])
                est = np.concatenate([x[1] for x in parts if x is not None])
                ok &= np.array_equal(host, want.reports.host)
                ok &= np.array_equal(est, want.reports.estimate)
            ok &= pool.snapshot_bytes() == ref.pool.snapshot_bytes()
    if rank == 0:
        result_q.put(bool(ok))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shard_merge_and_range_split_equal_one_pool():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True


def test_split_range_covers_everything():
    from paper_1812_00282_b200.parallel import split_range
    for n in (0, 1, 7, 1000):
        for world in (1, 2, 3, 8):
            spans = [split_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
