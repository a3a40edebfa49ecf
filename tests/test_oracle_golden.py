"""Pin the CPU oracle to the reference's own outputs (CPU only, no GPU).

The goldens under tests/golden/ were produced by running the reference package
(tests/golden/make_golden.py).  If the oracle reproduces all of them, it is a
trustworthy checker for the CUDA path (the gpu-marked tests).
"""

import hashlib

import numpy as np
import pytest

from _golden import PIPE_NAMES, PipeCase, load
from oracle import vate_oracle as vo


def test_mix64_and_streams_match_reference():
    kat = load("hash_kats.npz")
    assert np.array_equal(vo.mix64(kat["z"]), kat["mix"])
    for z, want in zip(kat["z"][:32], kat["mix"][:32]):
        assert vo.mix64_scalar(int(z)) == int(want)
    for s, cs, gs in zip(kat["seeds"], kat["cell_stream"], kat["group_stream"]):
        assert vo.stream_of(int(s), vo.SALT_CELL) == int(cs)
        assert vo.stream_of(int(s), vo.SALT_GROUP) == int(gs)


def test_survey_appendix_b_scalars():
    # SURVEY.md Appendix B literals, themselves produced by the reference
    assert vo.stream_of(0, vo.SALT_CELL) == 0x968282D39078F867
    assert vo.stream_of(0, vo.SALT_GROUP) == 0x809CDEE1130112A9
    assert vo.mix64_scalar(1) == 0x5692161D100B05E5
    assert vo.mix64_scalar((1 << 64) - 1) == 0xB4D055FCF2CBBD7B
    gs = vo.stream_of(0, vo.SALT_GROUP)
    cs = vo.stream_of(0, vo.SALT_CELL)
    assert int(vo.slot_of(np.array([0xCB007107]), 1024, gs)[0]) == 145
    assert int(vo.slot_of(np.array([0xCB007107]), 1000, gs)[0]) == 89
    assert int(vo.cell_of(np.array([0x0A010203]), np.array([5]), 20, cs)[0]) == 618202
    assert int(vo.cell_of(np.array([0x0A010203]), np.array([5]), 28, cs)[0]) == 264859354


def test_slot_and_cell_hashes_match_reference():
    kat = load("hash_kats.npz")
    row = 0
    for si in range(len(kat["seeds"])):
        for g in kat["gvals"]:
            got = vo.slot_of(kat["bips"], int(g), int(kat["group_stream"][si]))
            assert np.array_equal(got, kat["group"][row]), (si, g)
            row += 1
    row = 0
    for si in range(len(kat["seeds"])):
        for c in kat["cvals"]:
            got = vo.cell_of(kat["aips"], kat["vids"], int(c), int(kat["cell_stream"][si]))
            assert np.array_equal(got, kat["cell"][row]), (si, c)
            row += 1


def test_block_layouts_match_reference():
    lay = load("layouts.npz")
    keys = sorted({k.rsplit("_", 1)[0] for k in lay.files})
    assert len(keys) >= 10
    for key in keys:
        c, k, part = key.split("_", 2)
        starts = vo.block_starts(int(c), int(k), part)
        bi = lay[key + "_bi"]
        want = lay[key + "_ranges"].astype(np.int64)
        assert np.array_equal(starts[bi], want[:, 0]), key
        assert np.array_equal(starts[bi + 1], want[:, 1]), key
        idx = lay[key + "_idx"].astype(np.int64)
        got = np.searchsorted(starts, idx, side="right") - 1
        assert np.array_equal(got, lay[key + "_block"].astype(np.int64)), key


def test_reference_tests_layout_literals():
    # test_pools.py:59-81 hand-worked literals
    assert list(np.diff(vo.block_starts(10, 4, "tail"))) == [146] * 7 + [2]
    assert list(np.diff(vo.block_starts(10, 3, "low-dev"))) == [170, 170, 171, 171, 171, 171]
    with pytest.raises(vo.OracleConfigError):
        vo.block_starts(4, 1, "tail")


def test_estimator_float_path_matches_reference():
    kat = load("estimator_kats.npz")
    for i in range(int(kat["n"][0])):
        g, c, p = (int(x) for x in kat[f"c{i}_meta"])
        cfg = vo.OracleConfig(g, c, 8)
        g0 = kat[f"c{i}_g0"]
        rep = vo.reports_soa(cfg, np.arange(len(g0)), g0, p, 10, 8)
        assert np.array_equal(rep.estimate, kat[f"c{i}_est"]), (g, c, p)
        assert np.array_equal(rep.z_v, kat[f"c{i}_zv"])
        assert np.array_equal(rep.saturated, kat[f"c{i}_sat"])
        assert rep.z_p == float(kat[f"c{i}_zp"][0])


def test_snapshot_format_matches_reference():
    snap = load("snapshot_c8k9.npz")
    blob = snap["blob"].tobytes()
    pool = vo.OraclePool.from_snapshot(blob)
    assert pool.snapshot_bytes() == blob
    assert pool.count_inactive(9) == int(snap["count9"])
    with pytest.raises(vo.OracleConfigError):
        vo.OraclePool.from_snapshot(b"XXXX" + blob[4:])
    with pytest.raises(vo.OracleConfigError):
        vo.OraclePool.from_snapshot(blob[:8])
    with pytest.raises(vo.OracleConfigError):
        vo.OraclePool.from_snapshot(blob[:-8])


@pytest.mark.parametrize("name", PIPE_NAMES)
def test_oracle_pipeline_matches_reference(name):
    case = PipeCase(name)
    spec = case.spec
    cfg = vo.OracleConfig(spec["g"], spec["c"], spec["k"], seed=spec["seed"],
                          partition=spec["part"])
    pipe = vo.OraclePipeline(cfg, spec["kp"], floor=spec["floor"])
    for s, (t, aips, bips) in enumerate(case.slices()):
        out = pipe.process_slice(t, aips, bips)
        assert out.t == case.t[s]
        if len(case.live[s]) == 0:
            assert out.reports is None and case.p[s] == -1
        else:
            assert out.pool_inactive == case.p[s], (name, t)
            assert np.array_equal(out.g0, case.g0[s]), (name, t)
            assert np.array_equal(out.reports.host, case.kept[s]), (name, t)
            unfiltered = vo.reports_soa(cfg, case.live[s], out.g0, out.pool_inactive,
                                        t, spec["kp"])
            assert np.array_equal(unfiltered.estimate, case.est[s])
            assert np.array_equal(unfiltered.z_v, case.zv[s])
            assert np.array_equal(unfiltered.saturated, case.sat[s])
            assert unfiltered.z_p == case.zp[s]
        assert list(out.due) == list(case.blocks[s])
        assert out.visited == case.maintained[s] and out.cleared == case.cleared[s]
        assert pipe.pool.bact0 == case.bact0[s]
        snap = pipe.pool.snapshot_bytes()
        assert hashlib.sha256(snap).hexdigest() == case.snap_sha[s], (name, t)
    if case.final_snapshot:
        assert pipe.pool.snapshot_bytes() == case.final_snapshot
    pipe.close()


def test_oracle_workers_do_not_change_results():
    case = PipeCase("cfg1_small")
    spec = case.spec
    cfg = vo.OracleConfig(spec["g"], spec["c"], spec["k"], seed=spec["seed"])
    pipe = vo.OraclePipeline(cfg, spec["kp"], workers=4)
    for s, (t, aips, bips) in enumerate(case.slices()[:6]):
        out = pipe.process_slice(t, aips, bips)
        assert hashlib.sha256(pipe.pool.snapshot_bytes()).hexdigest() == case.snap_sha[s]
        if out.g0 is not None:
            assert np.array_equal(out.g0, case.g0[s])
    pipe.close()


def test_appendix_b_digest():
    ab = load("appendix_b.npz")
    cfg = vo.OracleConfig(1024, 20, 10)
    pool = vo.OraclePool(20, 10)
    rng = np.random.default_rng(0)
    for t in range(25):
        a = (0x0A000000 + rng.integers(0, 10_000, 100_000)).astype(np.uint64)
        b = rng.integers(1, 2 ** 32, 100_000).astype(np.uint64)
        pool.set_cells(cfg.pair_cells(a, b))
        if t == 24:
            assert pool.count_inactive(10) == int(ab["p24"]) == 422445
            rep = vo.estimate_soa(pool, cfg, ab["hosts24"], 24, 10)
            assert np.array_equal(rep.estimate, ab["est24"])
            assert rep.estimate[0] == 204.07996283727118
        due, visited, cleared = pool.advance()
    assert pool.bact0 == int(ab["bact0_end"]) == 5
    assert (due, visited, cleared) == ((15, 5), 110376, 27266)
    snap = pool.snapshot_bytes()
    assert len(snap) == 655_376
    assert hashlib.sha256(snap).hexdigest() == str(ab["snap_sha"]) == \
        "75f3db138a48c85aee504bafe7d088f4c34cf81ae10c423c21d2d4049a621a24"


def test_synthetic_generator_is_deterministic_and_bounded():
    a1, b1 = vo.synthetic_slice(3, 10_000, 1000)
    a2, b2 = vo.synthetic_slice(3, 10_000, 1000)
    assert np.array_equal(a1, a2) and np.array_equal(b1, b2)
    assert a1.min() >= 0x0A000000 and a1.max() < 0x0A000000 + 1000
    assert b1.max() < (1 << 32)
    # distinct peers per host stay bounded across slices (fixed peer sets)
    pairs = set()
    for t in range(20):
        a, b = vo.synthetic_slice(t, 10_000, 1000)
        pairs.update(zip(a.tolist(), b.tolist()))
    assert len(pairs) < 1000 * 40


# --- comparator pools (DR / TS, pools.py:301-410) ------------------------------------

from _golden import CMP_KINDS, CMP_NAMES, check_replay, replay_kind  # noqa: E402
from specs import COMPARATORS  # noqa: E402


@pytest.mark.parametrize("name", CMP_NAMES)
@pytest.mark.parametrize("kind", CMP_KINDS)
def test_oracle_comparator_pools_match_reference(name, kind):
    """The oracle's AT / DR / TS pools replay the reference slice by slice: cells,
    P, g0, estimates and maintenance reports."""
    spec = COMPARATORS[name]
    cfg = vo.OracleConfig(spec["g"], spec["c"], spec["k"], seed=spec["seed"],
                          partition=spec["part"])
    pipe = vo.OraclePipeline(cfg, spec["kp"], kind=kind)
    kp = spec["kp"]

    def scan(t, a, b):
        pipe.scan(a, b)
        if len(a):
            pipe.hosts.update(a, t)

    def advance(t):
        r = pipe.pool.advance()
        if t % max(1, cfg.k) == 0:
            pipe.hosts.prune(t)
        return r

    got = replay_kind(
        spec, kind, pipe.pool, scan, lambda t: pipe.hosts.active(t, kp),
        lambda live: vo.host_g0(pipe.pool, cfg, live, kp), lambda: pipe.pool.count_inactive(kp),
        lambda t, live, g0, p: vo.reports_soa(cfg, live, g0, p, t, kp).estimate, advance,
        lambda: pipe.pool.cells)
    check_replay(name, kind, got)
    rec = load(f"{name}.npz")
    assert np.array_equal(np.asarray(pipe.pool.cells, dtype=np.uint64),
                          rec[f"{kind}_final_cells"])
