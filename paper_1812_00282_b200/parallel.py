"""Multi-GPU slice processing: one process per GPU.

The packet stream shards across ranks; every rank scans its shard into a
private replica pool.  Replicas share bact0 and hold identical cells at slice
start, so the only per-slice exchange is "which cells were set this slice":
each rank has a 1-bit-per-cell dirty bitmap on the device (vate_dirty_bitmap:
a deferred pool's pending-set marks as they are, a direct-store pool's cells
holding their block clock), the bitmaps are all-gathered (NCCL over NVLink),
and every rank ORs them and writes its block clock into the dirty cells, or,
deferred, takes the union as its pending marks (vate_merge_dirty).  That is the reference's single-pool state exactly (the
window-aware newest-timestamp max of SURVEY.md §8e).

Host estimation then splits by aip range without leaving the device: each
rank compacts the hosts its scans registered this slice (vate_hosts_touched),
those lists are all-gathered (the SURVEY's "ncclAllGather of newly seen aips")
and inserted into every registry, so every rank holds the same sliding host
set; rank r then estimates the r-th contiguous share of the sorted active set
(vate_estimate_begin_part), and concatenating the ranks' reports in rank
order gives the reference's ascending host order (pipeline.py:57).

The pure functions here (``split_range``, ``union_sorted``) are shared with
the CPU tests, which run the same protocol over gloo with the oracle as the
per-rank pool (tests/test_multirank_cpu.py); the device phases
(``dirty_bitmap`` … ``absorb_hosts``) are what ``ReplicaStep`` calls between
collectives, and what the single-GPU replica test drives by hand.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import VATE_DEVICE, check, lib


def union_sorted(parts) -> np.ndarray:
    """Sorted union of per-rank sorted host arrays."""
    parts = [np.asarray(p, dtype=np.uint64) for p in parts if len(p)]
    if not parts:
        return np.zeros(0, dtype=np.uint64)
    return np.unique(np.concatenate(parts))


def split_range(n: int, rank: int, world: int):
    """[lo, hi) of the rank's contiguous share of n sorted hosts."""
    return (n * rank) // world, (n * (rank + 1)) // world


# --- device phases (one rank) ------------------------------------------------------------

def dirty_bitmap(pipe, out_ptr: int) -> None:
    """1 bit per cell: cells this replica set in the current slice."""
    check(lib.vate_dirty_bitmap(pipe.pool.handle, int(out_ptr)))


def merge_dirty(pipe, all_ptr: int, world: int) -> None:
    """OR the world's bitmaps and write each dirty cell's block clock."""
    check(lib.vate_merge_dirty(pipe.pool.handle, int(all_ptr), world))


def touched_hosts(pipe, t: int, out_ptr: int, cap: int) -> int:
    """Hosts this replica's scans registered in slice t -> device u64[cap]; count."""
    n = C.c_uint64()
    check(lib.vate_hosts_touched(pipe.hosts.handle, t, int(out_ptr), int(cap), C.byref(n)))
    return n.value


def absorb_hosts(pipe, keys_ptr: int, n: int, t: int) -> None:
    """Register another rank's touched hosts (device pointer) as seen in slice t."""
    if n:
        check(lib.vate_hosts_update(pipe.hosts.handle, int(keys_ptr), int(n), t, VATE_DEVICE))


class _SliceStepBase:
    """scan own shard -> exchange -> estimate own share (advance enqueued)."""

    def exchange(self, t: int, n_packets: int) -> None:  # pragma: no cover - abstract
        raise NotImplementedError

    def check_shard(self, n_packets: int) -> None:
        """Reject a shard the exchange cannot carry BEFORE it is scanned (a
        failure after the scan would leave this replica ahead of its peers)."""

    def __call__(self, t: int, pairs: int, n: int, where: str = "device", out=None):
        """Rows of this rank's share (HostReports, or a count with out=None), streamed.

        ``pairs``/``where`` as Pipeline.step_fast (device or host pointer, or a
        staging slot from stage_packed)."""
        pipe = self.pipe
        self.check_shard(n)
        if where == "staged":
            check(lib.vate_scan_staged(pipe.pool.handle, pipe.cfg.g, pipe.cfg.cell_stream,
                                       pipe.cfg.group_stream, int(pairs), int(n),
                                       pipe.hosts.handle, t))
        else:
            pipe.scan_packed(t, pairs, n, where == "device")
        self.exchange(t, n)
        rep = pipe.estimate_soa(t, out, advance=True, wait=False, keep_on_device=out is None,
                                part=self.rank, nparts=self.world)
        pipe._deferred_t = t
        return rep


class ReplicaStep(_SliceStepBase):
    """One slice on one rank of a torch.distributed (NCCL) job.

    scan own shard -> [dirty bitmap, touched hosts] -> all-gather both ->
    merge cells, absorb hosts -> estimate own share -> advance (overlapped).
    Collectives run on torch's stream; the pool's stream is synchronised
    around them (the touched-host count is read on the host anyway).
    """

    def __init__(self, pipe, dist, torch):
        self.pipe, self.dist, self.torch = pipe, dist, torch
        self.world, self.rank = dist.get_world_size(), dist.get_rank()
        self.dev = f"cuda:{pipe.pool.device}"
        nwords = (pipe.pool.size + 31) // 32
        self.mine = torch.empty(nwords, dtype=torch.int32, device=self.dev)
        self.all = torch.empty(self.world * nwords, dtype=torch.int32, device=self.dev)
        self.keys = torch.empty(1, dtype=torch.int64, device=self.dev)
        self.keys_all = torch.empty(self.world, dtype=torch.int64, device=self.dev)
        self.count = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.counts = torch.zeros(self.world, dtype=torch.int64, device=self.dev)

    def exchange(self, t: int, n_packets: int) -> None:
        torch, dist, pipe = self.torch, self.dist, self.pipe
        if self.keys.numel() < max(n_packets, 1):      # touched <= packets scanned
            self.keys = torch.empty(max(n_packets, 1), dtype=torch.int64, device=self.dev)
        dirty_bitmap(pipe, self.mine.data_ptr())
        nt = touched_hosts(pipe, t, self.keys.data_ptr(), self.keys.numel())  # syncs the pool
        self.count.fill_(nt)
        dist.all_gather_into_tensor(self.counts, self.count)
        dist.all_gather_into_tensor(self.all, self.mine)
        counts = self.counts.tolist()
        cap = max(counts + [1])
        if self.keys.numel() < cap:   # a smaller shard than a peer's touched set
            grown = torch.empty(cap, dtype=torch.int64, device=self.dev)
            grown[:nt] = self.keys[:nt]
            self.keys = grown
        if self.keys_all.numel() < self.world * cap:
            self.keys_all = torch.empty(self.world * cap, dtype=torch.int64, device=self.dev)
        dist.all_gather_into_tensor(self.keys_all[: self.world * cap], self.keys[:cap])
        torch.cuda.current_stream(self.dev).synchronize()  # gathers visible to the pool stream
        merge_dirty(pipe, self.all.data_ptr(), self.world)
        base = self.keys_all.data_ptr()
        for r, c in enumerate(counts):
            if r != self.rank:
                absorb_hosts(pipe, base + 8 * r * cap, c, t)



class PeerStep(_SliceStepBase):
    """One slice on one rank, exchanging over peer memory instead of NCCL.

    Every rank's exchange window lives in its own HBM and is mapped by every
    peer (CUDA IPC over NVLink/NVSwitch); ``vate_peer_exchange`` publishes the
    rank's dirty bitmap and touched hosts, raises its arrival flags and runs
    the fused OR-and-apply merge and the host absorb as kernels that read the
    peers' windows directly (csrc/vate_peer.cu).  ``dist`` carries only the
    one-time 64-byte IPC handle exchange and a barrier (any backend: gloo on
    one device for the tests, NCCL under torchrun).  ``key_cap`` bounds the
    hosts one rank registers per slice (its packets per slice suffice) and must
    be the same on every rank.  mode: 0 auto, 1 one-shot, 2 two-shot.
    """

    _is_peer = True

    def __init__(self, pipe, dist, key_cap: int, mode: int = 0):
        from ._lib import track
        self.pipe, self.dist = pipe, dist
        self.world, self.rank = dist.get_world_size(), dist.get_rank()
        self.key_cap = int(key_cap)
        h = C.c_void_p()
        handle = (C.c_uint8 * 64)()
        check(lib.vate_peer_create(C.byref(h), pipe.pool.handle, pipe.hosts.handle, self.rank,
                                   self.world, self.key_cap, handle))
        self.handle = h.value
        track(self)
        check(lib.vate_peer_set_mode(self.handle, int(mode)))
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(handle))
        buf = (C.c_uint8 * (64 * self.world)).from_buffer_copy(b"".join(handles))
        check(lib.vate_peer_open(self.handle, buf))
        dist.barrier()                   # every window mapped before anyone arrives
        self.touched_total = 0

    def check_shard(self, n_packets: int) -> None:
        if n_packets > self.key_cap:
            raise ValueError(f"{n_packets} packets exceed the peer key_cap {self.key_cap}")

    def bind_lagged(self, on: bool = True) -> None:
        """Run the exchange inside the pipeline's lagged step (vate_pool_set_peer):
        ``pipe.step_lagged`` then merges the replicas between each slice's scan
        and its pool pass, and its rows are this rank's share -- slice t-1's
        tail runs beside slice t's scan on every rank, as on one GPU."""
        check(lib.vate_pool_set_peer(self.pipe.pool.handle, self.handle if on else None,
                                     self.rank if on else 0, self.world if on else 1))

    def exchange(self, t: int, n_packets: int, count_touched: bool = False) -> None:
        """One slice's exchange; count_touched also sums the ranks' touched-host
        counts (one small read per peer window, so off on the hot path)."""
        self.check_shard(n_packets)
        tot = C.c_uint64()
        check(lib.vate_peer_exchange(self.handle, t, C.byref(tot) if count_touched else None))
        if count_touched:
            self.touched_total = tot.value

    def info(self) -> dict:
        wb, nb, ts = C.c_uint64(), C.c_uint64(), C.c_int()
        check(lib.vate_peer_info(self.handle, C.byref(wb), C.byref(nb), C.byref(ts)))
        return {"window_bytes": wb.value, "peer_read_bytes_per_slice": nb.value,
                "two_shot": bool(ts.value)}

    def close(self) -> None:
        if getattr(self, "handle", None):
            pool = self.pipe.pool
            if pool.handle is not None and pool.handle.value:
                lib.vate_pool_set_peer(pool.handle, None, 0, 1)
            lib.vate_peer_destroy(self.handle)
            self.handle = None

    def __del__(self):
        from ._lib import shutting_down
        if not shutting_down():
            self.close()
