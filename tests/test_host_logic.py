"""Host-side logic of the drop-in that needs no GPU (CPU only).

* configuration validation mirrors the reference's messages and exception types
* the block geometry equals the reference's (golden layouts)
* the float-path decomposition the device uses -- g*(log_zp - log_zv[g0]) with
  numpy-made logs -- equals the reference's reports_from_counts bit for bit
"""

import numpy as np
import pytest

from _golden import load
from paper_1812_00282_b200 import ConfigError, EstimatorConfig, hashing
from paper_1812_00282_b200.estimator import log_zp, log_zv_table
from paper_1812_00282_b200.pools import BlockLayout


def test_estimator_config_validation():
    EstimatorConfig(1024, 14, 8)
    for bad in (dict(g=0, c=14, k=8), dict(g=1024, c=0, k=8), dict(g=1024, c=33, k=8),
                dict(g=2048, c=10, k=8), dict(g=1024, c=14, k=8, seed=-1),
                dict(g=1024, c=14, k=8, seed=1 << 64),
                dict(g=1024, c=14, k=8, counter_kind="hll")):
        with pytest.raises(ConfigError):
            EstimatorConfig(**bad)


def test_hash_streams_match_reference():
    kat = load("hash_kats.npz")
    for s, cs, gs in zip(kat["seeds"], kat["cell_stream"], kat["group_stream"]):
        cfg = EstimatorConfig(64, 10, 4, seed=int(s))
        assert cfg.cell_stream == int(cs) and cfg.group_stream == int(gs)
    for z, want in zip(kat["z"][:64], kat["mix"][:64]):
        assert hashing.mix64(int(z)) == int(want)


def test_scalar_slot_and_cell_match_reference():
    kat = load("hash_kats.npz")
    gs0 = int(kat["group_stream"][0])
    for b, want in zip(kat["bips"][:50], kat["group"][4][:50]):   # seed 0, g = 1024
        assert hashing.group_index(int(b), 1024, gs0) == int(want)
    cs0 = int(kat["cell_stream"][0])
    for a, v, want in zip(kat["aips"][:50], kat["vids"][:50], kat["cell"][2][:50]):  # c = 20
        assert hashing.cell_index(int(a), int(v), 20, cs0) == int(want)


def test_pool_shape_validation():
    with pytest.raises(ConfigError):
        BlockLayout(2, 4)
    with pytest.raises(ConfigError):
        BlockLayout(33, 4)
    with pytest.raises(ConfigError):
        BlockLayout(10, 0)
    with pytest.raises(ConfigError):
        BlockLayout(10, 4, "diagonal")
    with pytest.raises(ConfigError, match="low-dev"):
        BlockLayout(4, 1)
    BlockLayout(4, 1, "low-dev")


def test_block_geometry_matches_reference():
    lay = load("layouts.npz")
    keys = sorted({k.rsplit("_", 1)[0] for k in lay.files})
    for key in keys:
        c, k, part = key.split("_", 2)
        L = BlockLayout(int(c), int(k), part)
        for bi, (lo, hi) in zip(lay[key + "_bi"], lay[key + "_ranges"]):
            assert L.block_range(int(bi)) == (int(lo), int(hi)), key
        idx = lay[key + "_idx"]
        assert np.array_equal(L.block_of_vec(idx), lay[key + "_block"]), key
        assert L.block_of(int(idx[0])) == int(lay[key + "_block"][0])


def test_reference_layout_literals():
    assert BlockLayout(10, 4).block_sizes() == [146] * 7 + [2]
    low = BlockLayout(10, 3, "low-dev")
    assert low.block_sizes() == [170, 170, 171, 171, 171, 171]
    assert (low.block_of(339), low.block_of(340), low.block_of(509), low.block_of(900)) == (1, 2, 2, 5)
    assert low.block_range(5) == (853, 1024)


def _device_float_path(g, g0, p, c):
    """What k_final_write computes, restated in numpy (IEEE subtract, multiply, divide)."""
    lzv = log_zv_table(g)
    lzp, zp = log_zp(p, 1 << c)
    raw = np.float64(g) * (np.float64(lzp) - lzv[g0])
    est = np.where(raw < 0, 0.0, raw)
    zv = g0.astype(np.float64) / np.float64(g)
    sat = (g0 == 0) | (raw < 0) | (p == 0)
    return est, zv, sat, zp


def test_float_path_decomposition_is_bit_exact():
    kat = load("estimator_kats.npz")
    for i in range(int(kat["n"][0])):
        g, c, p = (int(x) for x in kat[f"c{i}_meta"])
        g0 = kat[f"c{i}_g0"]
        est, zv, sat, zp = _device_float_path(g, g0, p, c)
        assert np.array_equal(est, kat[f"c{i}_est"]), (g, c, p)
        assert np.array_equal(zv, kat[f"c{i}_zv"])
        assert np.array_equal(sat, kat[f"c{i}_sat"])
        assert zp == float(kat[f"c{i}_zp"][0])


def test_float_path_decomposition_on_pipeline_goldens():
    from _golden import PIPE_NAMES, PipeCase
    for name in PIPE_NAMES:
        case = PipeCase(name)
        g, c = case.spec["g"], case.spec["c"]
        for s in range(case.n):
            if len(case.g0[s]) == 0:
                continue
            est, zv, sat, zp = _device_float_path(g, case.g0[s], int(case.p[s]), c)
            assert np.array_equal(est, case.est[s]), (name, s)
            assert np.array_equal(zv, case.zv[s]) and np.array_equal(sat, case.sat[s])
            assert zp == case.zp[s]


def test_log_zp_table_equals_scalar_path():
    """The per-pool table the one-call slice step indexes by P equals log_zp(P)."""
    from paper_1812_00282_b200.estimator import log_zp_table
    tab = log_zp_table(18)
    size = 1 << 18
    rng = np.random.default_rng(0)
    for p in np.concatenate([[0, 1, 2, size - 1, size], rng.integers(0, size + 1, 20_000)]):
        assert tab[p] == log_zp(int(p), size)[0], p
    assert log_zp_table(27) is None


def _swar_active(vals, act, B, kp, lane_bits):
    """Python restatement of active_bits_simd's guard-bit SWAR (csrc/vate_pool.cu)."""
    n = 32 // lane_bits
    mask32 = 0xFFFFFFFF
    rep = sum(1 << (lane_bits * i) for i in range(n))
    H = (1 << (lane_bits - 1)) * rep
    lo = act - kp + 1
    L = (lo if lo >= 0 else lo + B) * rep
    AH = (act * rep) | H
    Bx, Bp1 = B * rep, (B + 1) * rep
    out, bad = [], 0
    for w in range(0, len(vals), n):
        x = sum(int(v) << (lane_bits * i) for i, v in enumerate(vals[w:w + n]))
        xh = x | H
        bad |= (x & H) | (((xh - Bp1) & mask32) & H)
        ge_lo = ((xh - L) & mask32) & H
        le_act = ((AH - x) & mask32) & H
        m = (ge_lo & le_act) if lo >= 0 else (le_act | (ge_lo & ~(((xh - Bx) & mask32) & H)))
        out += [bool((m >> (lane_bits * i + lane_bits - 1)) & 1) for i in range(n)]
    return out, bad == 0


@pytest.mark.parametrize("lane_bits,bmax", [(8, 127), (16, 700)])
def test_swar_predicate_matches_scalar(lane_bits, bmax):
    rng = np.random.default_rng(lane_bits)
    for _ in range(300):
        k = int(rng.integers(1, bmax // 2 + 1))
        B = 2 * k
        if B >= (1 << (lane_bits - 1)):
            continue
        act = int(rng.integers(0, B))
        kp = int(rng.integers(1, k + 1))
        vals = rng.integers(0, B + 1, 64)        # valid stored values incl. the sentinel
        got, ok = _swar_active(vals.tolist(), act, B, kp, lane_bits)
        assert ok
        want = [(v != B) and ((act - v) % B) < kp for v in vals.tolist()]
        assert got == want, (B, act, kp)
        bad_vals = vals.copy()
        bad_vals[3] = B + 1 + int(rng.integers(0, (1 << lane_bits) - B - 1))
        assert not _swar_active(bad_vals.tolist(), act, B, kp, lane_bits)[1]
