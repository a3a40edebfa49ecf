"""Differential tests: the CPU oracle against the reference package itself, on
randomly drawn shapes and traffic (CPU only; skipped where the read-only
reference is not mounted, e.g. on the GPU box, whose parity tests use the
committed goldens instead).

The goldens pin the oracle on fixed cases; these draw pool shapes (tail and
low-dev partitions, AT / DR / TS kinds), window widths, virtual-layout sizes,
seeds, keys and slice sequences with hypothesis and require the oracle to
reproduce the reference slice by slice: every cell value, P, g0, the floats
of the reports and the MaintenanceReport.
"""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
if not os.path.isdir(REF):
    pytest.skip("reference package not mounted", allow_module_level=True)
sys.path.insert(0, REF)

hyp = pytest.importorskip("hypothesis")
from hypothesis import given, settings, strategies as st  # noqa: E402

from slidecard import estimator as rest  # noqa: E402
from slidecard.pipeline import SlidingHostSet  # noqa: E402

from oracle import vate_oracle as vo  # noqa: E402


@st.composite
def cases(draw):
    k = draw(st.sampled_from([1, 2, 3, 6, 10, 40, 130]))
    c_min = max(3, (2 * k - 1).bit_length())
    c = draw(st.integers(c_min, c_min + 4))
    part = draw(st.sampled_from(["tail", "low-dev"]))
    if part == "tail" and (1 << c) % (2 * k - 1) == 0:
        part = "low-dev"                       # the tail partition rejects b == 0
    kind = draw(st.sampled_from(["at", "at", "dr", "ts"]))
    g = draw(st.sampled_from([1, 2, 7, 64, 256]))
    g = min(g, 1 << c)
    kp = draw(st.integers(1, k))
    seed = draw(st.sampled_from([0, 1, 12345, (1 << 64) - 1]))
    hosts = draw(st.integers(1, 60))
    big = draw(st.booleans())
    slices = draw(st.integers(1, 2 * k + 3))
    data_seed = draw(st.integers(0, 2**32 - 1))
    return dict(k=k, c=c, part=part, kind=kind, g=g, kp=kp, seed=seed, hosts=hosts, big=big,
                slices=slices, data_seed=data_seed)


@settings(max_examples=400, deadline=None, derandomize=True)
@given(cases())
def test_oracle_replays_the_reference(case):
    k, c, g, kp = case["k"], case["c"], case["g"], case["kp"]
    rcfg = rest.EstimatorConfig(g, c, k, case["seed"], case["kind"], case["part"])
    rpool = rcfg.build_pool()
    rhosts = SlidingHostSet(k)
    ocfg = vo.OracleConfig(g, c, k, seed=case["seed"], partition=case["part"])
    opool = vo.make_oracle_pool(case["kind"], c, k, case["part"])
    ohosts = vo.OracleHosts(k)
    rng = np.random.default_rng(case["data_seed"])
    base = (1 << 40) + 3 if case["big"] else 0x0A000000
    for t in range(case["slices"]):
        n = int(rng.integers(0, 200))
        a = (base + rng.integers(0, case["hosts"], n)).astype(np.uint64)
        b = rng.integers(1, 1 << 62 if case["big"] else 1 << 32, n, dtype=np.uint64)
        rest.record_pairs(rpool, rcfg, a, b)
        opool.set_cells(ocfg.pair_cells(a, b))
        if n:
            rhosts.update(a, t)
            ohosts.update(a, t)
        live = rhosts.active(t, kp)
        assert np.array_equal(np.asarray(live, dtype=np.uint64), ohosts.active(t, kp)), t
        p = rpool.count_inactive(kp)
        assert p == opool.count_inactive(kp), t
        if len(live):
            g0 = rest.inactive_virtual_counts(rpool, rcfg, live, kp)
            og0 = vo.host_g0(opool, ocfg, np.asarray(live, dtype=np.uint64), kp)
            assert np.array_equal(np.asarray(g0), og0), t
            reps = rest.reports_from_counts(rcfg, live, g0, p, t, kp)
            orep = vo.reports_soa(ocfg, np.asarray(live, dtype=np.uint64), og0, p, t, kp)
            assert np.array_equal(np.array([r.estimate for r in reps]), orep.estimate), t
            assert np.array_equal(np.array([r.z_v for r in reps]), orep.z_v), t
            assert np.array_equal(np.array([r.saturated for r in reps]), orep.saturated), t
        rm = rpool.advance_slice()
        due, visited, cleared = opool.advance()
        assert (tuple(rm.blocks), rm.cells_maintained, rm.cells_cleared) == \
            (tuple(due), visited, cleared), t
        if t % k == 0:
            rhosts.prune(t)
            ohosts.prune(t)
    cells = rpool.cells.get_range(0, rpool.size) if case["kind"] != "ts" else rpool.cells
    assert np.array_equal(np.asarray(cells, dtype=np.uint64),
                          np.asarray(opool.cells, dtype=np.uint64))
    if case["kind"] == "at":
        assert rpool.snapshot_bytes() == opool.snapshot_bytes()
