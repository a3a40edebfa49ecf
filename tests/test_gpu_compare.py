"""Comparator pools on the device (csrc/vate_compare.cu): DrPool and TsPool
(pools.py:301-410) against the reference's recorded runs and the oracle.

The goldens (tests/golden/cmp_*.npz, made by running the reference) hold, per
slice and per kind, the SHA-256 of every cell value, P, g0 of every live host,
the estimates and the MaintenanceReport; the device pools must reproduce them
exactly, and -- as the reference asserts (test_estimator.py:233-255) -- the AT,
DR and TS estimates of the same traffic are identical.
"""

import numpy as np
import pytest

import paper_1812_00282_b200 as vb
from _golden import CMP_KINDS, CMP_NAMES, check_replay, load, replay_kind
from oracle import vate_oracle as vo
from specs import COMPARATORS, gen_slices

pytestmark = pytest.mark.gpu


def _device_replay(name, kind):
    spec = COMPARATORS[name]
    cfg = vb.EstimatorConfig(spec["g"], spec["c"], spec["k"], seed=spec["seed"],
                             counter_kind=kind, partition=spec["part"])
    pool = cfg.build_pool()
    assert pool.kind == kind
    kp = spec["kp"]
    hosts = vb.SlidingHostSet(spec["k"], pool=pool)

    def scan(t, a, b):
        vb.record_pairs(pool, cfg, a, b)
        if len(a):
            hosts.update(a, t)

    def advance(t):
        r = pool.advance_slice()
        if t % max(1, cfg.k) == 0:
            hosts.prune(t)
        return r.blocks, r.cells_maintained, r.cells_cleared

    got = replay_kind(
        spec, kind, pool, scan, lambda t: hosts.active(t, kp),
        lambda live: vb.inactive_virtual_counts(pool, cfg, live, kp),
        lambda: pool.count_inactive(kp),
        lambda t, live, g0, p: [r.estimate for r in vb.reports_from_counts(cfg, live, g0, p, t, kp)],
        advance, lambda: pool.cells.get_range(0, pool.size))
    return pool, got


@pytest.mark.parametrize("name", CMP_NAMES)
@pytest.mark.parametrize("kind", CMP_KINDS)
def test_device_pools_replay_the_reference(name, kind):
    pool, got = _device_replay(name, kind)
    check_replay(name, kind, got)
    rec = load(f"{name}.npz")
    assert np.array_equal(pool.cells.get_range(0, pool.size), rec[f"{kind}_final_cells"])
    assert pool.bits_per_counter == int(rec[f"{kind}_bits"][0])


@pytest.mark.parametrize("kind", ("dr", "ts"))
def test_comparator_pipeline_equals_at_pipeline(kind):
    """The fused device Pipeline (one host round trip per slice, the incremental
    g0 index on the comparator's bitmap too) gives the AT pipeline's reports,
    and the maintenance the oracle's comparator pool reports (DR: every cell
    visited)."""
    spec = dict(COMPARATORS["cmp_k6"], slices=20, pairs=20_000, hosts=1500)
    at_cfg = vb.EstimatorConfig(spec["g"], spec["c"], spec["k"], seed=spec["seed"])
    cfg = vb.EstimatorConfig(spec["g"], spec["c"], spec["k"], seed=spec["seed"], counter_kind=kind)
    ocfg = vo.OracleConfig(spec["g"], spec["c"], spec["k"], seed=spec["seed"])
    at = vb.Pipeline(at_cfg.build_pool(), at_cfg, spec["kp"])
    cmp_ = vb.Pipeline(cfg.build_pool(), cfg, spec["kp"])
    opipe = vo.OraclePipeline(ocfg, spec["kp"], kind=kind)
    for t, a, b in gen_slices(spec):
        want, _ = at.process_slice_soa(t, a, b)
        got = cmp_.step_fast(t, *_pairs(a, b)) if t % 2 else cmp_.process_slice_soa(t, a, b)[0]
        cmp_.wait_reports()
        ref = opipe.process_slice(t, a, b)
        if want is None:
            assert got is None
            continue
        assert np.array_equal(got.host, want.host), t
        assert np.array_equal(got.estimate, want.estimate), t
        assert np.array_equal(got.z_v, want.z_v), t
        m = cmp_.last_maintenance
        assert (m.blocks, m.cells_maintained, m.cells_cleared) == (ref.due, ref.visited,
                                                                  ref.cleared), t
    assert np.array_equal(cmp_.pool.cells.get_range(0, cmp_.pool.size),
                          np.asarray(opipe.pool.cells, dtype=np.uint64))
    assert cmp_.pool.inc_stats()["delta_slices"] > 0   # the index served the comparator


def _pairs(a, b):
    """(device pointer, n, 'device', out) for step_fast on a slice."""
    import torch
    pairs = torch.from_numpy(np.ascontiguousarray(
        np.stack([a.astype(np.uint32), b.astype(np.uint32)], axis=1)).view(np.int32)).cuda()
    _pairs.keep = pairs
    n = len(a)
    out = tuple(np.empty(4096, dt) for dt in (np.uint64, np.float64, np.float64, np.uint8))
    return pairs.data_ptr(), n, "device", out


def test_comparators_refuse_at_only_operations():
    dr = vb.make_pool("dr", 12, 6)
    ts = vb.make_pool("ts", 12, 6)
    assert isinstance(dr, vb.DrPool) and isinstance(ts, vb.TsPool)
    assert dr.bits_per_counter == 3 and ts.bits_per_counter == 64
    assert dr.cell_bytes == 1 and ts.cell_bytes == 8
    for pool in (dr, ts):
        with pytest.raises(vb.ConfigError):
            pool.snapshot_bytes() if hasattr(pool, "snapshot_bytes") else vb._lib.check(
                vb._lib.lib.vate_snapshot_size(pool.handle, None))
        with pytest.raises(ValueError):
            pool.inactive_mask([1], 7)          # k' > k
        with pytest.raises(ValueError):
            pool.set_many([1 << 12])            # cell outside the pool
    # TS: never-set cells are inactive; set in slice t, active for k' slices
    ts.set_many([5])
    assert ts.check_one(5, 1) and ts.check_one(6, 6) is False
    for _ in range(5):
        ts.advance_slice()
    assert ts.t == 5 and ts.inactive_mask([5], 5)[0] and not ts.inactive_mask([5], 6)[0]
    # DR: set -> 0, slides to k
    dr.set_many([3])
    rep = dr.advance_slice()
    assert rep.blocks == () and rep.cells_maintained == 1 << 12
    assert dr.cells.get_one(3) == 1
