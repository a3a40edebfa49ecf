"""Randomised differential tests of the CUDA path against the oracle (GPU).

hypothesis draws pool shapes (AT / DR / TS kinds, tail and low-dev partitions,
k from 1 to 300, g from 1 to 512), seeds, 32- or 64-bit keys, floors, window
widths and slice sequences (empty slices, churn, duplicates); the device
pipeline -- one-call-per-slice or the pipelined step -- must reproduce the
oracle (itself pinned to the reference, tests/test_oracle_*) slice by slice:
host sets, estimates, z_v, saturation, P, maintenance reports and the ATP1
snapshot.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

hyp = pytest.importorskip("hypothesis")
from hypothesis import given, settings, strategies as st  # noqa: E402

import paper_1812_00282_b200 as vb  # noqa: E402
from oracle import vate_oracle as vo  # noqa: E402


@st.composite
def cases(draw):
    k = draw(st.sampled_from([1, 2, 5, 12, 60, 130, 300]))
    c_min = max(4, (2 * k - 1).bit_length())
    c = draw(st.integers(c_min, c_min + 5))
    part = draw(st.sampled_from(["tail", "low-dev"]))
    if part == "tail" and (1 << c) % (2 * k - 1) == 0:
        part = "low-dev"
    kind = draw(st.sampled_from(["at", "at", "at", "dr", "ts"]))
    g = min(draw(st.sampled_from([1, 3, 64, 256, 512])), 1 << c)
    return dict(k=k, c=c, part=part, kind=kind, g=g, kp=draw(st.integers(1, k)),
                seed=draw(st.sampled_from([0, 7, (1 << 64) - 1])),
                hosts=draw(st.integers(1, 400)), big=draw(st.booleans()),
                floor=draw(st.sampled_from([0.0, 0.0, 5.0])),
                slices=draw(st.integers(1, 30)), lagged=draw(st.booleans()),
                data_seed=draw(st.integers(0, 2**32 - 1)))


@settings(max_examples=150, deadline=None, derandomize=True)
@given(cases())
def test_device_pipeline_replays_the_oracle(case):
    k, c, g, kp = case["k"], case["c"], case["g"], case["kp"]
    cfg = vb.EstimatorConfig(g, c, k, case["seed"], case["kind"], case["part"])
    ocfg = vo.OracleConfig(g, c, k, seed=case["seed"], partition=case["part"])
    pool = cfg.build_pool()
    pipe = vb.Pipeline(pool, cfg, kp, floor=case["floor"])
    opipe = vo.OraclePipeline(ocfg, kp, floor=case["floor"], kind=case["kind"])
    rng = np.random.default_rng(case["data_seed"])
    base = (1 << 40) + 9 if case["big"] else 0x0A000000
    lagged = case["lagged"] and not case["big"]       # the packed path carries u32 keys
    want = {}
    out = [tuple(np.empty(512, dt) for dt in (np.uint64, np.float64, np.float64, np.uint8))
           for _ in range(2)]

    def check(tp, rows):
        w = want.pop(tp)
        if w.reports is None or len(w.reports.host) == 0:
            assert rows is None or len(rows.host) == 0, tp
            return
        assert np.array_equal(rows.host, w.reports.host), tp
        assert np.array_equal(rows.estimate, w.reports.estimate), tp
        assert np.array_equal(rows.z_v, w.reports.z_v), tp
        assert np.array_equal(rows.saturated, w.reports.saturated), tp

    for t in range(case["slices"]):
        n = 0 if rng.random() < 0.1 else int(rng.integers(1, 3000))
        a = (base + rng.integers(0, case["hosts"], n)).astype(np.uint64)
        b = rng.integers(1, 1 << 62 if case["big"] else 1 << 32, n, dtype=np.uint64)
        want[t] = opipe.process_slice(t, a, b)
        if lagged:
            pairs = np.ascontiguousarray(np.stack([a, b], axis=1).astype(np.uint32))
            res = pipe.step_lagged(t, pairs.ctypes.data if n else 0, n, "host", out[t % 2])
            pipe.wait_reports()
            if res is not None:
                check(*res)
        else:
            rows, _ = pipe.process_slice_soa(t, a, b)
            check(t, rows)
        if case["kind"] == "at":
            assert pool.snapshot_bytes() == opipe.pool.snapshot_bytes(), t
        else:
            assert np.array_equal(pool.cells.get_range(0, pool.size),
                                  np.asarray(opipe.pool.cells, dtype=np.uint64)), t
    if lagged:
        res = pipe.flush_lagged(out[0])
        pipe.wait_reports()
        if res is not None:
            check(*res)
    assert not want
    pipe.close()
    pool.close()
