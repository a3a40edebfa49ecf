"""The benchmarked slice step at BASELINE shapes, slice by slice, against the oracle.

``Pipeline.step_lagged`` (vate_slice_step_lagged: the sweep fused into the
bitmap pass, the exact incremental g0 index, the early delta apply, the
aux-stream tail, default grid caps) is the path bench.py times.  These tests
drive it at BASELINE cfg 4 (c = 28, k = 300, 512 MiB of u16 cells beyond L2,
1M hosts, g = 1024) for 2k + 5 slices -- the clock wraps and every block is
swept at least twice -- and at cfg 2 (c = 24, k = 60) with the full 5M packets
per slice for 125 slices, and compare with the oracle (the reference's
per-slice phase order, pipeline.py:142-160, and two-block advance,
pools.py:221-249):

* every slice: the full sorted active host list (floor 0, so every active
  host has a row), P (Z_p's numerator) and the MaintenanceReport;
* on selected slices: every report row (estimate, z_v, saturated), with the
  oracle's g0 of all ~1M active hosts from its C half (oracle/native.py);
* the SHA-256 of the ATP1 snapshot at t = 2k, 2k + 4 and at the end.

cfg 3 (Zipf hosts + super-spreaders, c = 26) runs the same checks on its traffic.

The oracle keeps the reference's per-block value histogram (pools.py:195-204)
so that its P costs O(2k k') per slice instead of a pass over 2^28 cells.
"""

import hashlib

import numpy as np
import pytest

from oracle import native
from oracle import vate_oracle as vo

pytestmark = pytest.mark.gpu

vb = pytest.importorskip("paper_1812_00282_b200")


def _run_long(c, k, hosts, pkts, slices, rows_at, snaps_at, seed=0, zipf=False):
    import torch
    g = 1024
    cfg = vb.EstimatorConfig(g, c, k, seed=seed)
    ocfg = vo.OracleConfig(g, c, k, seed=seed)
    pool = cfg.build_pool()
    pool.set_option("incremental", 1)
    pipe = vb.Pipeline(pool, cfg, k, floor=0.0)
    opool = vo.OraclePool(c, k).track_histogram()
    ohosts = vo.OracleHostsVec(k)
    cap = hosts + 16   # cfg 3 (1M ranks + 64 spreaders) overflows it: rows come back in full anyway
    outs = [(torch.empty(cap, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64),
             torch.empty(cap, dtype=torch.float64, pin_memory=True).numpy(),
             torch.empty(cap, dtype=torch.float64, pin_memory=True).numpy(),
             torch.empty(cap, dtype=torch.uint8, pin_memory=True).numpy()) for _ in range(2)]
    want = {}
    checked = {"rows": 0, "full": 0, "snap": 0}

    def check(res):
        if res is None:
            return
        tp, rows = res
        w = want.pop(tp)
        assert rows is not None, tp
        assert np.array_equal(rows.host, w["hosts"]), tp          # full sorted host list
        assert pipe.last_pool_inactive == w["p"], tp
        m = pipe.last_maintenance
        assert (m.blocks, m.cells_maintained, m.cells_cleared) == w["maint"], tp
        assert rows.window_start == tp - k + 1
        checked["rows"] += 1
        if "rep" in w:
            r = w["rep"]
            assert rows.z_p == r.z_p, tp
            assert np.array_equal(rows.estimate, r.estimate), tp
            assert np.array_equal(rows.z_v, r.z_v), tp
            assert np.array_equal(rows.saturated, r.saturated), tp
            checked["full"] += 1

    dev = torch.empty((pkts, 2), dtype=torch.int32, device="cuda")
    tables = (vo.zipf_cdf(hosts), vo.spreader_cdf()) if zipf else None
    for t in range(slices):
        if zipf:
            a, b = vo.synthetic_zipf_slice(t, pkts, hosts, *tables)
        else:
            a, b = native.synthetic_slice(t, pkts, hosts)
        pairs = np.ascontiguousarray(np.stack([a.astype(np.uint32), b.astype(np.uint32)], axis=1))
        pool.synchronize()                        # slice t-1's scan has read the buffer
        dev.copy_(torch.from_numpy(pairs.view(np.int32)))
        torch.cuda.synchronize()
        res = pipe.step_lagged(t, dev.data_ptr(), pkts, "device", outs[t % 2])
        # oracle slice t: scan, host update, estimate, advance, prune (pipeline.py:142-160)
        native.set_cells(opool, native.pair_cells(ocfg, a, b))
        ohosts.update(a.astype(np.uint32), t)
        act = ohosts.active(t, k)
        p = opool.count_inactive(k)
        w = {"hosts": act, "p": p}
        if t in rows_at:
            g0 = native.host_g0(opool, ocfg, act, k)
            w["rep"] = vo.reports_soa(ocfg, act, g0, p, t, k)
        due, visited, cleared = opool.advance()
        w["maint"] = (due, visited, cleared)
        want[t] = w
        if t % k == 0:
            ohosts.prune(t)
        pipe.wait_reports()
        check(res)
        if t in snaps_at:
            got = hashlib.sha256(pool.snapshot_bytes()).hexdigest()
            exp = hashlib.sha256(native.snapshot_bytes(opool)).hexdigest()
            assert got == exp, t
            checked["snap"] += 1
    res = pipe.flush_lagged(outs[slices % 2])
    pipe.wait_reports()
    check(res)
    assert not want
    assert hashlib.sha256(pool.snapshot_bytes()).digest() == \
        hashlib.sha256(native.snapshot_bytes(opool)).digest()
    assert checked["rows"] == slices and checked["full"] == len(rows_at)
    assert checked["snap"] == len(snaps_at)
    inc = pool.inc_stats()
    pipe.close()
    pool.close()
    return inc


def test_lagged_step_cfg4_long_window_k300():
    """BASELINE cfg 4: c = 28, k = 300, tail, g = 1024, 1M hosts, 500k packets per
    slice for 2k + 5 = 605 slices (the per-slice packet count is reduced from 5M
    to bound the oracle's cost; pool, window, hosts and step are the bench's)."""
    k = 300
    slices = 2 * k + 5
    inc = _run_long(28, k, 1_000_000, 500_000, slices,
                    rows_at={1, 17, k - 1, k, 2 * k - 1, 2 * k + 3},
                    snaps_at={2 * k, 2 * k + 5 - 1})
    assert inc["delta_slices"] > 0            # the incremental index carried the estimate


def test_lagged_step_cfg2_full_slices():
    """BASELINE cfg 2 with the full 5M packets per slice: c = 24, k = 60, 1M hosts,
    125 slices (every block swept at least twice)."""
    k = 60
    inc = _run_long(24, k, 1_000_000, 5_000_000, 125, rows_at={3, 2 * k - 1, 124},
                    snaps_at={2 * k, 2 * k + 4})
    assert inc["delta_slices"] > 0


def test_lagged_step_cfg3_zipf_full_slices():
    """BASELINE cfg 3: Zipf(1.1) hosts plus 64 super-spreaders, c = 26, k = 60, the
    full 5M packets per slice for 2k + 5 slices (the auto scan form takes the
    registry-stamp filter on this traffic)."""
    k = 60
    _run_long(26, k, 1_000_000, 5_000_000, 2 * k + 5, rows_at={2, 2 * k + 1},
              snaps_at={2 * k}, zipf=True)
