"""Slice driver over the device pool (reference: pipeline.py).

Each slice runs the reference's three ordered phases (pipeline.py:142-160):
scan (hash + scatter the slice's pairs, register their hosts), estimate (the
sorted active hosts, Z_p, g0 per host, the float path, the floor filter) and
maintain (advance the clocks, sweep the two due blocks), then prunes the host
registry every k slices.  All three phases are CUDA kernels on the pool's
stream; stream order gives the hard barriers between them (SURVEY.md §7 hard
part 4).  ``workers`` is accepted for signature compatibility; the device path
has no host thread fan-out and its output never depended on it.
"""

from __future__ import annotations

import ctypes as C
import dataclasses
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import VATE_DEVICE, VATE_HOST, check, lib, ptr
from .estimator import (EstimatorConfig, HostReports, _check_pool_cfg, _ensure_log_table,
                        _u64, context_pool, log_zp, log_zp_table)
from .pools import AtPool, MaintenanceReport, maintenance_blocks

SCAN_CHUNK = 1 << 15  # pipeline.py:26 (the device scan takes a whole slice at once)


@dataclass(frozen=True)
class SliceStats:
    """Timing and maintenance accounting for one processed slice (pipeline.py:30-40)."""

    slice_index: int
    pairs: int
    scan_us: int
    estimate_us: int
    maintain_us: int
    cells_maintained: int
    cells_cleared: int


class SlidingHostSet:
    """Hosts seen recently, with the slice each was last seen in (pipeline.py:43-64).

    Lives on the device next to ``pool`` (or a private context pool).
    """

    def __init__(self, k: int, pool: AtPool | None = None, device: int = 0):
        self.k = k
        self._pool = pool if pool is not None else context_pool(device)
        h = C.c_void_p()
        check(lib.vate_hosts_create(C.byref(h), self._pool.handle, k))
        self._h = h
        self._is_registry = True
        _lib.track(self)

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value and not _lib.shutting_down():
            lib.vate_hosts_destroy(h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def update(self, aips, t: int) -> None:
        a = _u64(aips)
        if a.size:
            check(lib.vate_hosts_update(self._h, ptr(a), a.size, t, VATE_HOST))

    def __len__(self) -> int:
        n = C.c_uint64()
        check(lib.vate_hosts_size(self._h, C.byref(n)))
        return n.value

    def active(self, t: int, k_prime: int) -> np.ndarray:
        """Sorted hosts seen within the last k' slices."""
        out = np.empty(len(self), dtype=np.uint64)
        n = C.c_uint64()
        check(lib.vate_hosts_active(self._h, t, k_prime, ptr(out), out.size, C.byref(n)))
        return out[: n.value]

    def prune(self, t: int) -> None:
        check(lib.vate_hosts_prune(self._h, t))


class Pipeline:
    """Runs one device pool and estimator layout over a sliced pair stream."""

    def __init__(self, pool: AtPool, cfg: EstimatorConfig, k_prime: int, floor: float = 0.0,
                 workers: int = 1):
        if not 1 <= k_prime <= pool.k:
            raise ValueError(f"k'={k_prime} outside [1, {pool.k}]")
        if workers < 1:
            raise ValueError(f"workers must be at least 1, got {workers}")
        _check_pool_cfg(pool, cfg)
        self.pool = pool
        self.cfg = cfg
        self.k_prime = k_prime
        self.floor = floor
        self.workers = workers
        self.hosts = SlidingHostSet(pool.k, pool=pool)
        self.total_maintained = 0
        self.total_cleared = 0
        self._deferred_t = None   # slice whose advance result is still to be collected
        _ensure_log_table(pool, cfg.g)

    def close(self) -> None:
        if self.hosts is not None:
            self.hosts.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    # --- phases --------------------------------------------------------------------
    def _scan(self, aips, bips) -> int:
        a, b = _u64(aips), _u64(bips)
        if a.shape != b.shape:
            raise ValueError("aips and bips must have the same length")
        if a.size:
            check(lib.vate_scan_pairs(self.pool.handle, self.cfg.g, self.cfg.cell_stream,
                                      self.cfg.group_stream, ptr(a), ptr(b), a.size, VATE_HOST,
                                      self.hosts.handle, self._t))
        return a.size

    def scan_packed(self, t: int, pairs, n: int, on_device: bool) -> None:
        """Scan packed {u32 aip, u32 bip} records and register their hosts in slice t."""
        check(lib.vate_scan_packed(self.pool.handle, self.cfg.g, self.cfg.cell_stream,
                                   self.cfg.group_stream, int(pairs), int(n),
                                   VATE_DEVICE if on_device else VATE_HOST,
                                   self.hosts.handle, t))

    def estimate_soa(self, t: int, out=None, advance: bool = False,
                     wait: bool = True, keep_on_device: bool = False,
                     part: int = 0, nparts: int = 1):
        """The estimate phase (pipeline.py:120-138) as arrays; None without hosts.

        ``out`` may supply preallocated (pinned) host arrays
        (host u64, estimate f64, z_v f64, saturated u8) of equal capacity.
        With ``advance=True`` the slice advance is enqueued right after the g0
        gather (it touches cells, the float path does not), so the float path
        and the sweep share one host round trip; collect it with _collect().
        With ``wait=False`` the report rows are copied on the pool's D2H stream
        while the caller moves on (double-buffered): the arrays are complete
        after ``wait_reports()``; alternate two ``out`` sets between slices.
        ``part``/``nparts`` estimate only that contiguous share of the sorted
        active set (the multi-GPU split, parallel.ReplicaStep).
        """
        _ensure_log_table(self.pool, self.cfg.g)   # an ad-hoc estimate may have swapped it
        nh, p = C.c_uint64(), C.c_uint64()
        if nparts > 1:
            check(lib.vate_estimate_begin_part(self.pool.handle, self.hosts.handle, self.cfg.g,
                                               self.cfg.cell_stream, t, self.k_prime, part,
                                               nparts, C.byref(nh), C.byref(p)))
        else:
            check(lib.vate_estimate_begin(self.pool.handle, self.hosts.handle, self.cfg.g,
                                          self.cfg.cell_stream, t, self.k_prime, C.byref(nh),
                                          C.byref(p)))
        if self._deferred_t is not None:   # last slice's sweep finished before this sync
            self._collect(self._deferred_t)
            self._deferred_t = None
        if advance:
            check(lib.vate_advance_async(self.pool.handle))
        n = nh.value
        self.last_active = n
        if n == 0:
            return None
        lzp, z_p = log_zp(p.value, self.pool.size)
        if keep_on_device:   # rows stay in HBM (reports_device()); return the row count
            kept = C.c_uint64()
            check(lib.vate_estimate_finish_async(self.pool.handle, self.cfg.g, p.value, lzp,
                                                 float(self.floor), None, None, None, None, 0,
                                                 C.byref(kept)))
            self.last_pool_inactive = p.value
            return kept.value
        if out is None or len(out[0]) < n:
            out = (np.empty(n, np.uint64), np.empty(n, np.float64), np.empty(n, np.float64),
                   np.empty(n, np.uint8))
        host, est, zv, sat = out
        kept = C.c_uint64()
        finish = lib.vate_estimate_finish if wait else lib.vate_estimate_finish_async
        check(finish(self.pool.handle, self.cfg.g, p.value, lzp, float(self.floor), ptr(host),
                     ptr(est), ptr(zv), ptr(sat), len(host), C.byref(kept)))
        m = kept.value
        self.last_pool_inactive = p.value
        host, est, zv, sat = self._full_rows(out, m, wait)
        return HostReports(host[:m], est[:m], zv[:m], sat[:m].view(bool), z_p,
                           t - self.k_prime + 1, self.k_prime)

    def _full_rows(self, out, m: int, wait: bool = False):
        """``out`` if it holds all m rows; otherwise fresh arrays with every row
        (the async copy filled only len(out[0]) of them; the rest come from the
        device synchronously -- no row is ever dropped)."""
        host = out[0]
        if len(host) >= m:
            return out
        full = (np.empty(m, np.uint64), np.empty(m, np.float64), np.empty(m, np.float64),
                np.empty(m, np.uint8))
        check(lib.vate_reports_copy(self.pool.handle, 0, m, *(ptr(a) for a in full)))
        return full

    def _collect(self, t: int) -> MaintenanceReport:
        """Finish an advance enqueued by estimate_soa(advance=True); prune every k."""
        blocks = (C.c_int32 * 2)()
        maint, cleared = C.c_uint64(), C.c_uint64()
        check(lib.vate_advance_result(self.pool.handle, blocks, C.byref(maint), C.byref(cleared)))
        rep = MaintenanceReport(maintenance_blocks(blocks[0], blocks[1]), maint.value, cleared.value)
        return self._account(t, rep)

    def _account(self, t: int, rep: MaintenanceReport, prune: bool = True) -> MaintenanceReport:
        self.total_maintained += rep.cells_maintained
        self.total_cleared += rep.cells_cleared
        if prune and t % max(1, self.pool.k) == 0:   # (the lagged step prunes in the library)
            self.hosts.prune(t)
        self.last_maintenance = rep
        return rep

    def _maintain(self, t: int) -> MaintenanceReport:
        return self._account(t, self.pool.advance_slice())

    def wait_reports(self) -> None:
        """Block until every report row enqueued with wait=False is in host memory
        and every deferred slice advance is accounted."""
        check(lib.vate_estimate_wait(self.pool.handle))
        if self._deferred_t is not None:
            self._collect(self._deferred_t)
            self._deferred_t = None

    def stage_packed(self, pairs_host_ptr: int, n: int) -> int:
        """Start the H2D copy of a slice's packed records (pinned host memory) on the
        pool's copy stream; returns the staging slot for step_staged."""
        slot = C.c_int()
        check(lib.vate_stage_packed(self.pool.handle, int(pairs_host_ptr), int(n), C.byref(slot)))
        return slot.value

    def step_packed(self, t: int, pairs, n: int, on_device: bool, out=None, wait: bool = True):
        """One slice from packed records: scan, estimate (+ advance overlapped), prune.

        wait=False streams: report rows land asynchronously (see estimate_soa) and
        the advance report of slice t is collected during slice t+1's estimate
        (its one host round trip), so a slice costs a single host sync."""
        self.scan_packed(t, pairs, n, on_device)
        return self._estimate_advance(t, out, wait)

    def _estimate_advance(self, t: int, out, wait: bool):
        rep = self.estimate_soa(t, out, advance=True, wait=wait)
        if wait:
            self._collect(t)
        else:
            self._deferred_t = t
        return rep

    def step_fast(self, t: int, pairs: int, n: int, where: str, out):
        """One whole slice in a single library call (vate_slice_step), streaming.

        ``pairs`` is a device pointer (where='device'), a host pointer
        ('host') or a staging slot from stage_packed ('staged').  Report rows
        land asynchronously in ``out`` (alternate two sets); with out=None they
        stay in device memory (reports_device()) and the call returns the row
        count.  The advance of slice t is accounted during the next call or
        wait_reports()."""
        _ensure_log_table(self.pool, self.cfg.g)
        tab = getattr(self, "_lzp_tab", None)
        if tab is None:
            tab = self._lzp_tab = log_zp_table(self.pool.c)
        if tab is None:   # pool too large for the table: same slice, log_zp per slice
            if where == "staged":
                check(lib.vate_scan_staged(self.pool.handle, self.cfg.g, self.cfg.cell_stream,
                                           self.cfg.group_stream, int(pairs), int(n),
                                           self.hosts.handle, t))
            else:
                self.scan_packed(t, pairs, n, where == "device")
            check(lib.vate_pool_lat_mark(self.pool.handle, t, 0))
            rep = self.estimate_soa(t, out, advance=True, wait=False,
                                    keep_on_device=out is None)
            check(lib.vate_pool_lat_mark(self.pool.handle, t, 1))
            self._deferred_t = t
            return rep
        host, est, zv, sat = out if out is not None else (None, None, None, None)
        res = _lib.StepResult()
        where_code = {"host": VATE_HOST, "device": VATE_DEVICE, "staged": _lib.VATE_STAGED}[where]
        check(lib.vate_slice_step(self.pool.handle, self.hosts.handle, self.cfg.g,
                                  self.cfg.cell_stream, self.cfg.group_stream, int(pairs), int(n),
                                  where_code, t, self.k_prime, float(self.floor), ptr(tab),
                                  *(ptr(a) if a is not None else None for a in (host, est, zv, sat)),
                                  len(host) if host is not None else 0, C.byref(res)))
        if res.prev_collected:
            self._account(self._deferred_t, MaintenanceReport(
                maintenance_blocks(res.prev_blocks[0], res.prev_blocks[1]), res.prev_maintained,
                res.prev_cleared))
        self._deferred_t = t
        self.last_active = res.nhosts
        if res.nhosts == 0:
            return None
        self.last_pool_inactive = res.pool_inactive
        m = res.nkept
        if out is None:
            return m
        host, est, zv, sat = self._full_rows(out, m)
        return HostReports(host[:m], est[:m], zv[:m], sat[:m].view(bool),
                           res.pool_inactive / float(self.pool.size), t - self.k_prime + 1,
                           self.k_prime)

    def step_lagged(self, t: int, pairs: int, n: int, where: str, out):
        # (pools too large for the log table take two library calls per slice)
        """Software-pipelined step_fast (vate_slice_step_lagged): enqueue slice t
        and complete the previous slice, whose rows this returns as
        ``(t_prev, rows)`` -- ``rows`` as step_fast returns them -- or None on the
        first call.  The previous slice's g0 lookups and float path run beside
        slice t's scan, so the GPU never waits on the host round trip.  ``out``
        receives the previous slice's rows; call ``flush_lagged`` after the last
        slice.  Results are identical to step_fast's, one call later."""
        return self._lagged(None, out, t, pairs, n, where)

    def flush_lagged(self, out):
        """Complete the last slice of a step_lagged run: ``(t, rows)`` or None."""
        return self._lagged(None, out)

    def _lagged(self, fn, out, t=None, pairs=0, n=0, where="device"):
        _ensure_log_table(self.pool, self.cfg.g)
        tab = getattr(self, "_lzp_tab", None)
        if tab is None:
            tab = self._lzp_tab = log_zp_table(self.pool.c)
        host, est, zv, sat = out if out is not None else (None, None, None, None)
        res = _lib.StepResult()
        outs = (*(ptr(a) if a is not None else None for a in (host, est, zv, sat)),
                len(host) if host is not None else 0, C.byref(res))
        h, hs, cfg = self.pool.handle, self.hosts.handle, self.cfg
        where_code = {"host": VATE_HOST, "device": VATE_DEVICE, "staged": _lib.VATE_STAGED}[where]
        if tab is not None:      # one call; np.log of P from the table
            if t is None:
                check(lib.vate_slice_flush(h, hs, cfg.g, cfg.cell_stream, float(self.floor),
                                           ptr(tab), *outs))
            else:
                check(lib.vate_slice_step_lagged(h, hs, cfg.g, cfg.cell_stream, cfg.group_stream,
                                                 int(pairs), int(n), where_code, t, self.k_prime,
                                                 float(self.floor), ptr(tab), *outs))
        else:                    # two halves around np.log of the previous slice's P
            if t is None:
                check(lib.vate_slice_lagged_flush_begin(h, hs, cfg.g, cfg.cell_stream,
                                                        C.byref(res)))
            else:
                check(lib.vate_slice_lagged_begin(h, hs, cfg.g, cfg.cell_stream, cfg.group_stream,
                                                  int(pairs), int(n), where_code, t,
                                                  self.k_prime, C.byref(res)))
            lzp = log_zp(res.pool_inactive, self.pool.size)[0] if res.nhosts else 0.0
            check(lib.vate_slice_lagged_end(h, hs, cfg.g, cfg.cell_stream, cfg.group_stream,
                                            float(self.floor), lzp, *outs))
        if not res.prev_valid:
            return None
        tp = res.prev_t
        if res.prev_collected:
            self._account(tp, MaintenanceReport(
                maintenance_blocks(res.prev_blocks[0], res.prev_blocks[1]), res.prev_maintained,
                res.prev_cleared), prune=False)
        self.last_active = res.nhosts
        if res.nhosts == 0:
            return tp, None
        self.last_pool_inactive = res.pool_inactive
        m = res.nkept
        if out is None:
            return tp, m
        host, est, zv, sat = self._full_rows(out, m)
        return tp, HostReports(host[:m], est[:m], zv[:m], sat[:m].view(bool),
                               res.pool_inactive / float(self.pool.size), tp - self.k_prime + 1,
                               self.k_prime)

    def reports_device(self):
        """(host, estimate, z_v, saturated) device addresses of the last report rows."""
        ptrs = [C.c_void_p() for _ in range(4)]
        check(lib.vate_reports_device(self.pool.handle, *(C.byref(q) for q in ptrs)))
        return tuple(q.value for q in ptrs)

    def step_staged(self, t: int, slot: int, n: int, out=None, wait: bool = True):
        """One slice from a staged buffer (see stage_packed)."""
        check(lib.vate_scan_staged(self.pool.handle, self.cfg.g, self.cfg.cell_stream,
                                   self.cfg.group_stream, slot, int(n), self.hosts.handle, t))
        return self._estimate_advance(t, out, wait)

    # --- driving ---------------------------------------------------------------------
    # SliceStats phase times (pipeline.py:144-159 measures each phase's wall
    # time on the CPU): here each phase is timed by CUDA events on the pool's
    # stream around it -- the scan (with its H2D and host registration), the
    # estimate up to its report rows in host memory, the advance -- read after
    # the phase's own synchronisation, so timing adds no sync.
    _M0, _M1, _M2, _M3 = 12, 13, 14, 15

    def _phase_us(self, a: int, b: int) -> int:
        ms = C.c_double()
        check(lib.vate_mark_elapsed(self.pool.handle, a, b, C.byref(ms)))
        return int(ms.value * 1000)

    def _phases(self, t: int, n: int, scan, out=None):
        h = self.pool.handle
        check(lib.vate_mark(h, self._M0))
        scan()
        check(lib.vate_mark(h, self._M1))
        reports = self.estimate_soa(t, out)     # returns once the rows are in host memory
        check(lib.vate_mark(h, self._M2))
        rep = self._maintain(t)                  # returns once the advance is collected
        check(lib.vate_mark(h, self._M3))
        stats = SliceStats(t, n, self._phase_us(self._M0, self._M1),
                           self._phase_us(self._M1, self._M2),
                           self._phase_us(self._M2, self._M3),
                           rep.cells_maintained, rep.cells_cleared)
        return reports, stats

    def process_slice_soa(self, t: int, aips, bips, out=None):
        """All three phases for slice t; returns (HostReports | None, SliceStats)."""
        self._t = t
        n = len(aips)
        return self._phases(t, n, lambda: self._scan(aips, bips), out)

    def process_packed(self, t: int, pairs_dev: int, n: int):
        """All three phases for a slice of packed {u32 aip, u32 bip} records already
        on the device (e.g. from traceio.DeviceSlices); (HostReports | None, SliceStats)."""
        return self._phases(t, n, lambda: n and self.scan_packed(t, pairs_dev, n, True))

    def process_slice(self, t: int, aips, bips):
        """Run all three phases for slice t; returns (reports, stats) (pipeline.py:142-160).
        estimate_us includes building the EstimateReport list, as the reference's
        _estimate does (pipeline.py:120-138)."""
        soa, stats = self.process_slice_soa(t, aips, bips)
        t0 = time.perf_counter_ns()
        reports = [] if soa is None else soa.to_list()
        stats = dataclasses.replace(stats, estimate_us=stats.estimate_us
                                    + (time.perf_counter_ns() - t0) // 1000)
        return reports, stats

    def run(self, sliced):
        """Process a (slice, aips, bips) stream; yields (t, reports, stats)."""
        for t, aips, bips in sliced:
            reports, stats = self.process_slice(t, aips, bips)
            yield t, reports, stats
