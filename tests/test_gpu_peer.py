"""The peer-memory exchange (csrc/vate_peer.cu, parallel.PeerStep) on one GPU.

Only one B200 is available to this build, so the multi-GPU protocol runs as
world_size 2 or 3 *processes on the same device*: each process owns a replica
pool and registry, the exchange windows are CUDA-IPC mapped between the
processes exactly as between GPUs, and the fused OR-and-apply merge and host
absorb read the peers' windows directly (gloo carries only the one-time handle
exchange).  Every slice, every rank's ATP1 snapshot must equal the oracle pool
fed every packet, and the ranks' report shares concatenated in rank order must
equal the oracle's reports (hosts, estimates, z_v, saturation) -- for the
one-shot and the two-shot merge, ragged segment splits included (world 3).
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, c, k, result_q, kind="peer", deferred=-1, uneven=False):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    import paper_1812_00282_b200 as vb
    from oracle import native
    from oracle import vate_oracle as vo
    from paper_1812_00282_b200.parallel import PeerStep, ReplicaStep, split_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    msgs = []
    try:
        kp, g = 5, 256
        cfg = vb.EstimatorConfig(g, c, k, seed=9)
        ocfg = vo.OracleConfig(g, c, k, seed=9)
        pool = cfg.build_pool(device=0)
        if deferred != -1:
            pool.set_option("deferred", deferred)
        pipe = vb.Pipeline(pool, cfg, kp)
        ref = vo.OraclePipeline(ocfg, kp)
        torch.cuda.set_device(0)
        step = (PeerStep(pipe, dist, key_cap=40_000, mode=mode) if kind.startswith("peer")
                else ReplicaStep(pipe, dist, torch))
        lagged = kind == "peer_lagged"
        if lagged:
            step.bind_lagged()
        pending = {}
        rng = np.random.default_rng(11)
        for t in range(18):
            n = int(rng.integers(0, 30_000)) if t != 5 else 0
            lo_host = 0 if t < 9 else 600        # host churn: half the hosts expire
            a = (0x0A000000 + rng.integers(lo_host, lo_host + 1200, n)).astype(np.uint32)
            b = rng.integers(1, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
            allp = np.stack([a, b], axis=1)
            if uneven:   # rank 0 gets 95 % of the packets, the rest a sliver
                cut = [0, (n * 95) // 100] + [(n * (95 + 5 * r)) // 100 for r in range(1, world)]
                cut[-1] = n
                mine = np.ascontiguousarray(allp[cut[rank]:cut[rank + 1]])
            else:
                mine = np.ascontiguousarray(allp[rank::world])
            cap = 4096
            out = (np.empty(cap, np.uint64), np.empty(cap, np.float64), np.empty(cap, np.float64),
                   np.empty(cap, np.uint8))
            outs_l = [tuple(np.empty(cap, dt) for dt in (np.uint64, np.float64, np.float64,
                                                           np.uint8)) for _ in range(2)]
            if lagged:
                res = pipe.step_lagged(t, mine.ctypes.data if len(mine) else 0, len(mine),
                                       "host", outs_l[t % 2])
            else:
                rep = step(t, mine.ctypes.data if len(mine) else 0, len(mine), "host", out)
            pipe.wait_reports()
            want = ref.process_slice(t, a.astype(np.uint64), b.astype(np.uint64))
            big = c >= 24
            if not big or t % 6 == 5:
                want_snap = native.snapshot_bytes(ref.pool) if big else ref.pool.snapshot_bytes()
                if pipe.pool.snapshot_bytes() != want_snap:
                    msgs.append(f"rank {rank} t {t}: snapshot differs")
            if lagged:   # the rows of slice t-1 came with this call
                pending[t] = want
                if res is None:
                    continue
                tp, rep = res
                want = pending.pop(tp)
            if want.reports is None:
                if rep is not None and len(rep.host):
                    msgs.append(f"rank {rank} t {t}: reports where the oracle has none")
                continue
            lo, hi = split_range(len(want.reports.host), rank, world)
            got_host = np.zeros(0, np.uint64) if rep is None else rep.host
            got_est = np.zeros(0, np.float64) if rep is None else rep.estimate
            got_zv = np.zeros(0, np.float64) if rep is None else rep.z_v
            if not np.array_equal(got_host, want.reports.host[lo:hi]):
                msgs.append(f"rank {rank} t {t}: host share differs")
            elif not (np.array_equal(got_est, want.reports.estimate[lo:hi])
                      and np.array_equal(got_zv, want.reports.z_v[lo:hi])):
                msgs.append(f"rank {rank} t {t}: estimates differ")
            if pipe.last_pool_inactive != want.pool_inactive:
                msgs.append(f"rank {rank} t {t}: pool_inactive differs")
        if lagged:
            res = pipe.flush_lagged(outs_l[0])
            pipe.wait_reports()
            if res is not None:
                pending.pop(res[0], None)
            if pending:
                msgs.append(f"rank {rank}: slices never completed {sorted(pending)}")
        if kind.startswith("peer"):
            info = step.info()
            if info["two_shot"] != (mode == 2 or (mode == 0 and world > 2)):
                msgs.append(f"rank {rank}: unexpected merge form {info}")
            step.close()
        pipe.close()
        pipe.pool.close()
    except Exception as e:  # report, do not hang the peers' barrier
        msgs.append(f"rank {rank}: {type(e).__name__}: {e}")
    result_q.put((rank, msgs))
    dist.destroy_process_group()


def _run(world, mode, c=15, k=6, kind="peer", deferred=-1, uneven=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, c, k, q, kind, deferred,
                                                uneven)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(world):
        r, msgs = q.get(timeout=400)
        results[r] = msgs
    for p in procs:
        p.join(timeout=60)
    problems = [m for r in sorted(results) for m in results[r]]
    assert not problems, problems[:10]
    assert all(p.exitcode == 0 for p in procs)


@pytest.mark.timeout(500)
def test_peer_exchange_two_ranks_one_shot():
    _run(2, 1)


@pytest.mark.timeout(500)
def test_peer_exchange_two_ranks_two_shot():
    _run(2, 2)


@pytest.mark.timeout(500)
def test_peer_exchange_three_ranks_auto_two_shot_u16():
    """world 3 (auto picks two-shot): 2^13 cells = 256 words split into 128-B
    segments of 96, 96 and 64 words; k = 130 makes the cells u16."""
    _run(3, 0, c=13, k=130)


@pytest.mark.timeout(500)
def test_peer_exchange_deferred_pools_uneven_shards():
    """Deferred pools (the pending marks are the dirty bitmap; the merge writes
    the union back as marks) with 95 % / 5 % shards."""
    _run(2, 0, kind="peer", deferred=1, uneven=True)


@pytest.mark.timeout(500)
@pytest.mark.parametrize("deferred", [0, 1])
def test_replica_step_two_ranks_uneven_shards(deferred):
    """The NCCL-form exchange (all-gathers of bitmaps and touched keys, here
    over gloo on one device) with a rank whose shard is smaller than the
    other rank's touched-host set (the key buffer grows to the
    gathered maximum before the key all-gather)."""
    _run(2, 0, kind="replica", deferred=deferred, uneven=True)


@pytest.mark.timeout(500)
@pytest.mark.parametrize("world,deferred", [(2, 0), (3, 1)])
def test_peer_exchange_in_the_lagged_step(world, deferred):
    """The multi-GPU step in the software-pipelined form (vate_pool_set_peer):
    the exchange between each slice's scan and its pool pass, slice t-1's tail
    beside slice t's scan; snapshots every slice and every rank's share of the
    previous slice's reports equal the oracle's."""
    _run(world, 0, kind="peer_lagged", deferred=deferred)


@pytest.mark.timeout(900)
def test_peer_exchange_cfg4_shape_two_ranks():
    """The cfg 4 pool shape (c = 28, k = 300: u16 cells, deferred marks and the
    bit-plane history by default) with two ranks in the lagged step."""
    _run(2, 0, c=28, k=300, kind="peer_lagged")
