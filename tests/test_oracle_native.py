"""The oracle's fast forms (CPU, no GPU): the C half (oracle/native.py: g0 over
many hosts, ATP1 packing), the histogram count (pools.py:195-204) and the
array host set agree with the numpy oracle, which the golden vectors pin
(tests/test_oracle_golden.py).  These forms carry the full-size parity tests."""

import numpy as np
import pytest

from oracle import native
from oracle import vate_oracle as vo


@pytest.mark.parametrize("c,k,g,part,kp", [(12, 4, 64, "tail", 4), (14, 9, 1000, "low-dev", 5),
                                           (16, 300, 1024, "tail", 300), (10, 2, 3, "tail", 1)])
def test_native_g0_and_pack_equal_numpy(c, k, g, part, kp):
    cfg = vo.OracleConfig(g, c, k, seed=c * 7 + 1, partition=part)
    pool = vo.OraclePool(c, k, part)
    rng = np.random.default_rng(c)
    for t in range(2 * k + 3):
        a = rng.integers(0, 1 << 33, 500, dtype=np.uint64)   # aips >= 2^32 included
        b = rng.integers(0, 1 << 64, 500, dtype=np.uint64)
        pool.set_cells(cfg.pair_cells(a, b))
        if t % max(1, k // 2) == 0 or t == 2 * k + 2:
            hosts = np.unique(a)[:200]
            assert np.array_equal(native.host_g0(pool, cfg, hosts, kp),
                                  vo.host_g0(pool, cfg, hosts, kp)), t
            assert native.snapshot_bytes(pool) == pool.snapshot_bytes(), t
        pool.advance()


@pytest.mark.parametrize("c,k,part", [(12, 5, "tail"), (13, 60, "low-dev"), (14, 300, "tail")])
def test_histogram_count_equals_full_pass(c, k, part):
    cfg = vo.OracleConfig(64, c, k)
    full = vo.OraclePool(c, k, part)
    fast = vo.OraclePool(c, k, part).track_histogram()
    rng = np.random.default_rng(k)
    for t in range(2 * k + 5):
        cells = cfg.pair_cells(rng.integers(0, 5000, 700, dtype=np.uint64),
                               rng.integers(0, 1 << 32, 700, dtype=np.uint64))
        full.set_cells(cells)
        fast.set_cells(cells)
        for kp in {1, k // 2 or 1, k}:
            assert fast.count_inactive(kp) == full.count_inactive(kp), (t, kp)
        assert full.advance() == fast.advance()
        assert np.array_equal(full.cells, fast.cells)


def test_array_host_set_equals_dict_host_set():
    k = 7
    a, b = vo.OracleHosts(k), vo.OracleHostsVec(k)
    rng = np.random.default_rng(3)
    for t in range(40):
        aips = (0x0A000000 + rng.integers(0, 300 if t < 20 else 120, rng.integers(0, 400))).astype(np.uint64)
        if len(aips):
            a.update(aips, t)
            b.update(aips, t)
        for kp in (1, 3, k):
            assert np.array_equal(a.active(t, kp), b.active(t, kp)), (t, kp)
        if t % k == 0:
            a.prune(t)
            b.prune(t)
        assert len(a.last) == len(b)


def test_native_scan_and_synth_equal_numpy():
    for c, k, g, part in ((14, 5, 1000, "tail"), (20, 300, 1024, "low-dev")):
        cfg = vo.OracleConfig(g, c, k, seed=5, partition=part)
        a_np, b_np = vo.synthetic_slice(3, 50_000, 7_000)
        a_c, b_c = native.synthetic_slice(3, 50_000, 7_000)
        assert np.array_equal(a_np, a_c) and np.array_equal(b_np, b_c)
        assert np.array_equal(native.pair_cells(cfg, a_np, b_np), cfg.pair_cells(a_np, b_np))
        p1 = vo.OraclePool(c, k, part).track_histogram()
        p2 = vo.OraclePool(c, k, part).track_histogram()
        for t in range(2 * k + 2):
            a, b = native.synthetic_slice(t, 3000, 700)
            cells = cfg.pair_cells(a, b)
            p1.set_cells(cells)
            native.set_cells(p2, cells)
            assert np.array_equal(p1.cells, p2.cells) and np.array_equal(p1.hist, p2.hist), t
            assert p1.advance() == p2.advance()
        assert np.array_equal(p1.hist, p2.hist)
