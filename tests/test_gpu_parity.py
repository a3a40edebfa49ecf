"""CUDA path vs the oracle and the reference goldens (B200 only).

Bar: bit-exact for every integer / byte / index result (cells, snapshots,
P, g0, host sets, maintenance reports); the floats of the estimate are
compared bit-for-bit against the oracle run on the same machine (same numpy)
and within rel 1e-12 against the goldens recorded in the build container
(the north star allows 1e-6).
"""

import hashlib

import numpy as np
import pytest

from _golden import PIPE_NAMES, PipeCase, load
from oracle import vate_oracle as vo

pytestmark = pytest.mark.gpu

vb = pytest.importorskip("paper_1812_00282_b200")

REL = 1e-12   # float tolerance against goldens made on another machine's numpy


def _cfgs(spec):
    cfg = vb.EstimatorConfig(spec["g"], spec["c"], spec["k"], seed=spec["seed"],
                             partition=spec["part"])
    ocfg = vo.OracleConfig(spec["g"], spec["c"], spec["k"], seed=spec["seed"],
                           partition=spec["part"])
    return cfg, ocfg


# --- hashing ------------------------------------------------------------------------

def test_pair_cells_matches_reference_hashes():
    kat = load("hash_kats.npz")
    # pair_cells = cell_index(aip, group_index(bip)); check both halves via goldens
    for si, seed in enumerate(kat["seeds"]):
        for c in (5, 20, 28, 32):
            g = 1024 if c >= 10 else 32
            cfg = vb.EstimatorConfig(g, c, 2, seed=int(seed))
            got = vb.pair_cells(cfg, kat["aips"], kat["bips"])
            want = vo.OracleConfig(g, c, 2, seed=int(seed)).pair_cells(kat["aips"], kat["bips"])
            assert np.array_equal(got, want), (seed, c)


def test_host_cells_matches_reference_hashes():
    kat = load("hash_kats.npz")
    cfg = vb.EstimatorConfig(1000, 24, 2, seed=7)
    aips = kat["aips"][:64]
    got = vb.host_cells(cfg, aips)
    want = vo.OracleConfig(1000, 24, 2, seed=7).host_cells(aips)
    assert np.array_equal(got, want)


def test_non_power_of_two_group_counts():
    kat = load("hash_kats.npz")
    for g in (1, 3, 1000, (1 << 20) + 7):
        cfg = vb.EstimatorConfig(g, 24, 2, seed=1)
        got = vb.pair_cells(cfg, kat["aips"], kat["bips"])
        want = vo.OracleConfig(g, 24, 2, seed=1).pair_cells(kat["aips"], kat["bips"])
        assert np.array_equal(got, want), g


# --- whole pipelines against the reference goldens ---------------------------------

@pytest.mark.parametrize("name", PIPE_NAMES)
def test_pipeline_matches_reference_goldens(name):
    case = PipeCase(name)
    spec = case.spec
    cfg, ocfg = _cfgs(spec)
    pool = cfg.build_pool()
    pipe = vb.Pipeline(pool, cfg, spec["kp"], floor=spec["floor"])
    opipe = vo.OraclePipeline(ocfg, spec["kp"], floor=spec["floor"])
    for s, (t, aips, bips) in enumerate(case.slices()):
        got, stats = pipe.process_slice_soa(t, aips, bips)
        want = opipe.process_slice(t, aips, bips)
        assert stats.pairs == len(aips)
        if len(case.live[s]) == 0:
            assert got is None and want.reports is None
        else:
            assert pipe.last_active == len(case.live[s])
            assert pipe.last_pool_inactive == case.p[s], (name, t)
            # host set after the floor: identical to the reference
            assert np.array_equal(got.host, case.kept[s]), (name, t)
            # floats: bit-identical to the oracle on this machine ...
            assert np.array_equal(got.estimate, want.reports.estimate), (name, t)
            assert np.array_equal(got.z_v, want.reports.z_v), (name, t)
            assert np.array_equal(got.saturated, want.reports.saturated), (name, t)
            assert got.z_p == want.reports.z_p == case.zp[s]
            # ... and within REL of the reference's recorded floats
            keep = np.isin(case.live[s], case.kept[s])
            np.testing.assert_allclose(got.estimate, case.est[s][keep], rtol=REL, atol=0)
            assert np.array_equal(got.z_v, case.zv[s][keep])
        m = pipe.last_maintenance
        assert (m.blocks, m.cells_maintained, m.cells_cleared) == \
            (tuple(case.blocks[s]), case.maintained[s], case.cleared[s]), (name, t)
        assert pool.bact0 == case.bact0[s]
        snap = pool.snapshot_bytes()
        assert hashlib.sha256(snap).hexdigest() == case.snap_sha[s], (name, t)
    if case.final_snapshot:
        assert pool.snapshot_bytes() == case.final_snapshot
    pipe.close()


@pytest.mark.parametrize("name", ["cfg1_small", "kprime_floor", "g1000_big_keys"])
def test_list_api_matches_oracle(name):
    case = PipeCase(name)
    spec = case.spec
    cfg, ocfg = _cfgs(spec)
    pipe = vb.Pipeline(cfg.build_pool(), cfg, spec["kp"], floor=spec["floor"])
    opipe = vo.OraclePipeline(ocfg, spec["kp"], floor=spec["floor"])
    for t, aips, bips in case.slices()[:8]:
        reports, _ = pipe.process_slice(t, aips, bips)
        want = opipe.process_slice(t, aips, bips).reports
        if want is None:
            assert reports == []
            continue
        assert [r.host for r in reports] == want.host.tolist()
        assert [r.estimate for r in reports] == want.estimate.tolist()
        assert all(r.window_start == t - spec["kp"] + 1 and r.k_prime == spec["kp"]
                   for r in reports)
        assert all(r.slice_end == t for r in reports)
    pipe.close()


def test_appendix_b_digest():
    ab = load("appendix_b.npz")
    cfg = vb.EstimatorConfig(g=1024, c=20, k=10, seed=0)
    pool = cfg.build_pool()
    rng = np.random.default_rng(0)
    for t in range(25):
        a = (0x0A000000 + rng.integers(0, 10_000, 100_000)).astype(np.uint64)
        b = rng.integers(1, 2 ** 32, 100_000).astype(np.uint64)
        vb.record_pairs(pool, cfg, a, b)
        if t == 24:
            assert pool.count_inactive(10) == 422445
            reps = vb.estimate_hosts(pool, cfg, ab["hosts24"], 24, 10)
            np.testing.assert_allclose([r.estimate for r in reps], ab["est24"], rtol=REL)
            assert [r.z_v for r in reps] == ab["zv24"].tolist()
        rep = pool.advance_slice()
    assert pool.bact0 == 5
    assert rep == vb.MaintenanceReport((15, 5), 110376, 27266)
    snap = pool.snapshot_bytes()
    assert len(snap) == 655_376
    assert hashlib.sha256(snap).hexdigest() == \
        "75f3db138a48c85aee504bafe7d088f4c34cf81ae10c423c21d2d4049a621a24"


# --- the pool protocol against a brute-force model (test_pools.py:120-149) ---------

@pytest.mark.parametrize("partition", ["tail", "low-dev"])
@pytest.mark.parametrize("k", [1, 4, 9, 70, 130])
def test_pool_matches_brute_force(partition, k):
    if partition == "tail" and k == 1:
        partition = "low-dev"
    c = 9 if k < 70 else 12
    pool = vb.AtPool(c, k, partition)
    size = pool.size
    rng = np.random.default_rng(100 * k + 7)
    last_set = {}
    everything = np.arange(size, dtype=np.uint64)
    widths = sorted({1, max(1, k // 2), k})
    for t in range(min(20 * k + 15, 300)):
        idx = rng.integers(0, size, size=25).astype(np.uint64)   # duplicates allowed
        pool.set_many(idx)
        for i in idx.tolist():
            last_set[i] = t
        one = int(rng.integers(0, size))
        pool.set_one(one)
        last_set[one] = t
        for w in widths:
            mask = pool.inactive_mask(everything, w)
            want = np.array([i not in last_set or t - last_set[i] >= w for i in range(size)])
            assert np.array_equal(mask, want), f"slice {t} width {w}"
            assert pool.count_inactive(w) == int(want.sum())
        for i in (0, one, size - 1):
            assert pool.check_one(i, k) == (i in last_set and t - last_set[i] < k)
        pool.advance_slice()


def test_pool_errors():
    pool = vb.AtPool(7, 4)
    with pytest.raises(ValueError):
        pool.count_inactive(0)
    with pytest.raises(ValueError):
        pool.count_inactive(5)
    with pytest.raises(ValueError):
        pool.check_one(200, 2)
    with pytest.raises(ValueError):
        pool.set_many(np.array([128], dtype=np.uint64))
    with pytest.raises(ValueError):
        pool.inactive_mask(np.array([5000], dtype=np.uint64), 2)
    assert isinstance(vb.make_pool("dr", 7, 4), vb.DrPool)   # comparators exist
    with pytest.raises(vb.ConfigError):
        vb.make_pool("hll", 7, 4)
    # the pool keeps working after a rejected call
    pool.set_many(np.array([3], dtype=np.uint64))
    assert pool.check_one(3, 1)


def test_two_blocks_maintained_per_slice():
    pool = vb.AtPool(10, 6)
    k, cycle = pool.k, pool.nblocks
    per_cell = np.zeros(pool.size, dtype=np.int64)
    for step in range(2 * cycle):
        rep = pool.advance_slice()
        assert len(rep.blocks) == 2 and rep.blocks[0] != rep.blocks[1]
        assert pool.block_act(rep.blocks[0]) == 0
        assert pool.block_act(rep.blocks[1]) == k
        span = 0
        for bi in rep.blocks:
            lo, hi = pool.block_range(bi)
            per_cell[lo:hi] += 1
            span += hi - lo
        assert rep.cells_maintained == span <= 2 * pool.max_block_size
        if (step + 1) % cycle == 0:
            assert np.all(per_cell == 2)
            per_cell[:] = 0


def test_cell_widths_and_memory():
    assert vb.AtPool(10, 300).bits_per_counter == 10
    assert vb.AtPool(10, 300).cell_bytes == 2
    assert vb.AtPool(10, 127).cell_bytes == 1
    assert vb.AtPool(17, 1 << 15, "low-dev").cell_bytes == 4
    p = vb.AtPool(20, 300)
    assert p.packed_bytes == (-(-(1 << 20) * 10 // 64) + 1) * 8 + 16   # test_pools.py:249-254


def test_reference_memory_and_width_gates():
    """The reference's own gates on the drop-in: ACCEPTANCE 4
    (test_acceptance.py:130-143), test_pools.py:245-254, test_bitpack.py:49-52."""
    at_bits = vb.AtPool(20, 300).bits_per_counter
    dr_bits = vb.DrPool(20, 300).bits_per_counter
    mem = vb.AtPool(20, 300).memory_bytes
    bound = (1 << 20) * 10 // 8 + 16
    assert at_bits == 10 and dr_bits == 9
    assert abs(mem - bound) / bound <= 0.01
    assert vb.AtPool(10, 300).bits_per_counter == 10
    assert vb.DrPool(10, 300).bits_per_counter == 9
    assert vb.TsPool(10, 300).bits_per_counter == 64
    pool = vb.AtPool(20, 300)
    words = -(-(1 << 20) * 10 // 64) + 1
    assert pool.memory_bytes == words * 8 + 16
    assert pool.cells.nbytes == (163_840 + 1) * 8
    assert pool.device_bytes >= (1 << 20) * pool.cell_bytes   # the HBM footprint, separately
    assert vb.DrPool(12, 300).memory_bytes == (-(-(1 << 12) * 9 // 64) + 1) * 8
    assert vb.TsPool(12, 300).memory_bytes == (1 << 12) * 8


@pytest.mark.parametrize("deferred", [0, 1, 2])
def test_device_cells_write_api(deferred):
    """AtPool.cells set / set_one / set_range / fill on the device, against the
    reference's PackedArray semantics (bitpack.py:57-140): values masked to the
    width, fill rejects values beyond it, reads and snapshots agree, and a
    pending deferred mark never overwrites a later explicit value."""
    k, c = 300, 12
    pool = vb.AtPool(c, k)
    pool.set_option("deferred", min(deferred, 1))
    pool.set_option("bitplane", 1 if deferred == 2 else 0)
    pool.count_inactive(k)              # (bit-plane mode starts at the first estimate)
    assert pool.mode()["bitplane"] == (deferred == 2)
    opool = vo.OraclePool(c, k)
    cells = pool.cells
    cells.fill(3)
    opool.cells[:] = 3
    assert np.all(cells.get_range(0, 1 << c) == 3)
    with pytest.raises(ValueError):
        cells.fill(1 << 10)
    rng = np.random.default_rng(5)
    idx = rng.integers(0, 1 << c, 500).astype(np.uint64)
    vals = rng.integers(0, 1 << 12, 500).astype(np.uint64)     # wider than 10 bits: masked
    idx, first = np.unique(idx, return_index=True)
    vals = vals[first]
    cells.set(idx, vals)
    opool.cells[idx.astype(np.int64)] = (vals & 0x3FF).astype(opool.cells.dtype)
    cells.set_one(7, 1000)
    opool.cells[7] = 1000
    cells.set_range(100, np.arange(20, dtype=np.uint64))
    opool.cells[100:120] = np.arange(20)
    # a set_many mark followed by an explicit value: the value wins
    pool.set_many(np.array([9, 11], dtype=np.uint64))
    opool.set_cells(np.array([9, 11], dtype=np.uint64))
    cells.set_one(9, 5)
    opool.cells[9] = 5
    assert np.array_equal(cells.get_range(0, 1 << c), opool.cells.astype(np.uint64))
    assert cells.get_one(7) == 1000
    assert pool.snapshot_bytes() == opool.snapshot_bytes()
    with pytest.raises(ValueError):
        cells.set_one(1 << c, 1)


# --- snapshots ------------------------------------------------------------------------

def test_snapshot_load_of_reference_bytes(tmp_path):
    snap = load("snapshot_c8k9.npz")
    blob = snap["blob"].tobytes()
    path = tmp_path / "pool.snap"
    path.write_bytes(blob)
    pool = vb.AtPool.load(path)
    assert pool.snapshot_bytes() == blob
    assert pool.count_inactive(9) == int(snap["count9"])
    opool = vo.OraclePool.from_snapshot(blob)
    pool.advance_slice()
    opool.advance()
    assert pool.snapshot_bytes() == opool.snapshot_bytes()
    for bad in (b"XXXX" + blob[4:], blob[:8], blob[:-8]):
        path.write_bytes(bad)
        with pytest.raises(vb.ConfigError):
            vb.AtPool.load(path)


@pytest.mark.parametrize("c,k,part", [(10, 4, "tail"), (12, 300, "tail"), (9, 33, "low-dev"),
                                      (17, 1 << 15, "low-dev"), (3, 2, "tail")])
def test_snapshot_roundtrip_all_cell_widths(c, k, part):
    pool = vb.AtPool(c, k, part)
    opool = vo.OraclePool(c, k, part)
    rng = np.random.default_rng(c * k)
    for _ in range(min(3 * k, 40)):
        idx = rng.integers(0, pool.size, size=max(1, pool.size // 7)).astype(np.uint64)
        pool.set_many(idx)
        opool.set_cells(idx)
        pool.advance_slice()
        opool.advance()
    blob = pool.snapshot_bytes()
    assert blob == opool.snapshot_bytes()
    back = vb.AtPool.from_bytes(blob)
    assert back.snapshot_bytes() == blob
    assert back.count_inactive(k) == pool.count_inactive(k) == opool.count_inactive(k)


# --- estimator entry points ---------------------------------------------------------

def test_estimate_hosts_arbitrary_order_and_duplicates():
    cfg = vb.EstimatorConfig(512, 16, 8, seed=4)
    ocfg = vo.OracleConfig(512, 16, 8, seed=4)
    pool = cfg.build_pool()
    opool = vo.OraclePool(16, 8)
    rng = np.random.default_rng(9)
    a = rng.integers(0, 500, 20000).astype(np.uint64)
    b = rng.integers(0, 1 << 40, 20000).astype(np.uint64)
    vb.record_pairs(pool, cfg, a, b)
    opool.set_cells(ocfg.pair_cells(a, b))
    hosts = np.array([7, 3, 7, 499, 0, 1 << 45, 3], dtype=np.uint64)
    got = vb.estimate_hosts_soa(pool, cfg, hosts, 5, 8)
    want = vo.estimate_soa(opool, ocfg, hosts, 5, 8)
    assert np.array_equal(got.host, hosts)
    assert np.array_equal(got.estimate, want.estimate)
    assert np.array_equal(vb.inactive_virtual_counts(pool, cfg, hosts, 3),
                          vo.host_g0(opool, ocfg, hosts, 3))
    r = vb.estimate_host(pool, cfg, 7, 5, 8)
    assert r.estimate == got.estimate[0] and r.host == 7


def test_reports_from_counts_edge_cases():
    kat = load("estimator_kats.npz")
    for i in range(int(kat["n"][0])):
        g, c, p = (int(x) for x in kat[f"c{i}_meta"])
        cfg = vb.EstimatorConfig(g, c, 8)
        g0 = kat[f"c{i}_g0"]
        rep = vb.reports_from_counts_soa(cfg, np.arange(len(g0)), g0, p, 10, 8)
        ocfg = vo.OracleConfig(g, c, 8)
        want = vo.reports_soa(ocfg, np.arange(len(g0)), g0, p, 10, 8)
        assert np.array_equal(rep.estimate, want.estimate), (g, c, p)
        assert np.array_equal(rep.z_v, want.z_v) and np.array_equal(rep.saturated, want.saturated)
        np.testing.assert_allclose(rep.estimate, kat[f"c{i}_est"], rtol=REL, atol=0)
    with pytest.raises(ValueError):
        vb.reports_from_counts(vb.EstimatorConfig(64, 10, 4), [1], [65], 10, 0, 1)


def test_duplicate_pairs_and_order_do_not_matter():
    cfg = vb.EstimatorConfig(128, 12, 4, seed=3)
    rng = np.random.default_rng(4)
    aips = rng.integers(0, 30, size=2000).astype(np.uint64)
    bips = rng.integers(0, 5000, size=2000).astype(np.uint64)
    perm = rng.permutation(2000)
    a_pool, b_pool = cfg.build_pool(), cfg.build_pool()
    vb.record_pairs(a_pool, cfg, aips, bips)
    vb.record_pairs(b_pool, cfg, np.concatenate([aips[perm], aips]),
                    np.concatenate([bips[perm], bips]))
    assert a_pool.snapshot_bytes() == b_pool.snapshot_bytes()


def test_packed_scan_equals_u64_scan():
    cfg = vb.EstimatorConfig(1024, 20, 10, seed=0)
    p1, p2 = cfg.build_pool(), cfg.build_pool()
    rng = np.random.default_rng(2)
    for n in (1, 2, 3, 1001, 65536):
        a = rng.integers(0, 1 << 32, n, dtype=np.uint64)
        b = rng.integers(0, 1 << 32, n, dtype=np.uint64)
        vb.record_pairs(p1, cfg, a, b)
        vb.record_packed(p2, cfg, np.stack([a, b], axis=1).astype(np.uint32))
        assert p1.snapshot_bytes() == p2.snapshot_bytes(), n
        p1.advance_slice()
        p2.advance_slice()


# --- host registry (test_pipeline.py:100-125) ----------------------------------------

def test_host_registry_window():
    reg = vb.SlidingHostSet(4)
    reg.update(np.array([1, 2], dtype=np.uint64), 0)
    reg.update(np.array([3], dtype=np.uint64), 2)
    assert list(reg.active(2, 3)) == [1, 2, 3]
    assert list(reg.active(2, 1)) == [3]
    assert list(reg.active(4, 4)) == [3]
    reg.prune(6)
    assert list(reg.active(6, 4)) == []
    assert len(reg) == 0


def test_host_registry_growth_matches_dict():
    reg = vb.SlidingHostSet(50)
    ref = vo.OracleHosts(50)
    rng = np.random.default_rng(5)
    for t in range(60):
        n = int(rng.integers(0, 200_000))
        keys = rng.integers(0, 1 << 20, n).astype(np.uint64)
        if t % 7 == 3:
            keys = np.concatenate([keys, [np.uint64((1 << 64) - 1), np.uint64(0)]])
        if t % 5 == 1:
            keys = rng.integers(0, 1 << 64, n, dtype=np.uint64)
        reg.update(keys, t)
        ref.update(keys, t)
        kp = 1 + t % 50
        assert np.array_equal(reg.active(t, kp), ref.active(t, kp)), t
        if t % 50 == 0:
            reg.prune(t)
            ref.prune(t)
        assert len(reg) == len(ref.last)


def test_hosts_age_out_of_reports():
    cfg = vb.EstimatorConfig(64, 12, 6, seed=6)
    quiet = np.empty(0, dtype=np.uint64)
    peers = np.arange(100, 130, dtype=np.uint64)
    sliced = [(0, np.full(30, 9, dtype=np.uint64), peers)]
    sliced += [(t, quiet, quiet) for t in range(1, 5)]
    with vb.Pipeline(cfg.build_pool(), cfg, 2, floor=0.0) as pipe:
        seen = {t: [r.host for r in reports] for t, reports, _ in pipe.run(iter(sliced))}
    assert seen == {0: [9], 1: [9], 2: [], 3: [], 4: []}


def test_pipeline_rejects_bad_args():
    cfg = vb.EstimatorConfig(64, 10, 4)
    pool = cfg.build_pool()
    for kp, workers in ((0, 1), (5, 1), (4, 0)):
        with pytest.raises(ValueError):
            vb.Pipeline(pool, cfg, kp, workers=workers)


# --- full BASELINE sizes: size-independent properties ---------------------------------

def _sample_hosts(pipe_hosts, n, seed):
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(pipe_hosts, size=min(n, len(pipe_hosts)), replace=False))


@pytest.mark.parametrize("c,k,hosts,pkts,slices", [(24, 60, 1_000_000, 5_000_000, 8),
                                                   (26, 60, 1_000_000, 5_000_000, 4)])
def test_full_size_u8_pipeline_against_oracle(c, k, hosts, pkts, slices):
    """BASELINE cfg 2/3 shapes: snapshot, P, the active host count and g0 of sampled
    hosts equal the oracle replaying the same synthetic packets."""
    cfg = vb.EstimatorConfig(1024, c, k)
    ocfg = vo.OracleConfig(1024, c, k)
    pool = cfg.build_pool()
    pipe = vb.Pipeline(pool, cfg, k)
    opool = vo.OraclePool(c, k)
    seen = set()
    for t in range(slices):
        a, b = vo.synthetic_slice(t, pkts, hosts)
        got, _ = pipe.process_slice_soa(t, a, b)
        opool.set_cells(ocfg.pair_cells(a, b))
        seen.update(np.unique(a).tolist())
        assert pipe.last_active == len(seen)
        assert pipe.last_pool_inactive == opool.count_inactive(k)
        assert np.all(np.diff(got.host.astype(np.int64)) > 0)
        sample = _sample_hosts(got.host, 3000, t)
        idx = np.searchsorted(got.host, sample)
        want = vo.reports_soa(ocfg, sample, vo.host_g0(opool, ocfg, sample, k),
                              pipe.last_pool_inactive, t, k)
        assert np.array_equal(got.estimate[idx], want.estimate)
        due, visited, cleared = opool.advance()
        m = pipe.last_maintenance
        assert (m.blocks, m.cells_maintained, m.cells_cleared) == (due, visited, cleared)
    assert hashlib.sha256(pool.snapshot_bytes()).digest() == \
        hashlib.sha256(opool.snapshot_bytes()).digest()


def test_full_size_u16_pool_c28_k300():
    """BASELINE cfg 4 shape (512 MiB of u16 cells, beyond L2): P, sampled cells and
    sampled g0 equal the oracle replaying the same packets."""
    c, k = 28, 300
    cfg = vb.EstimatorConfig(1024, c, k)
    ocfg = vo.OracleConfig(1024, c, k)
    pool = cfg.build_pool()
    assert pool.cell_bytes == 2
    pipe = vb.Pipeline(pool, cfg, k)
    opool = vo.OraclePool(c, k)
    for t in range(3):
        a, b = vo.synthetic_slice(t, 2_000_000, 1_000_000)
        got, _ = pipe.process_slice_soa(t, a, b)
        opool.set_cells(ocfg.pair_cells(a, b))
        assert pipe.last_pool_inactive == opool.count_inactive(k)
        sample = _sample_hosts(got.host, 1000, t)
        idx = np.searchsorted(got.host, sample)
        want = vo.reports_soa(ocfg, sample, vo.host_g0(opool, ocfg, sample, k),
                              pipe.last_pool_inactive, t, k)
        assert np.array_equal(got.estimate[idx], want.estimate)
        due, visited, cleared = opool.advance()
        assert pipe.last_maintenance.cells_cleared == cleared
        cells = np.random.default_rng(t).integers(0, 1 << c, 100_000, dtype=np.uint64)
        assert np.array_equal(pool.cells.get(cells), opool.cells[cells.astype(np.int64)])


# --- both g0 gather kernels (global-memory L2 gather, shared/DSMEM gather) ------------

@pytest.mark.parametrize("c,g", [(5, 32), (12, 64), (20, 1024), (21, 1000), (23, 7), (24, 1024)])
def test_g0_kernels_agree_with_oracle(c, g):
    from paper_1812_00282_b200._lib import check, lib
    k = 8
    cfg = vb.EstimatorConfig(g, c, k, seed=c)
    ocfg = vo.OracleConfig(g, c, k, seed=c)
    pool = cfg.build_pool()
    opool = vo.OraclePool(c, k)
    rng = np.random.default_rng(c)
    for t in range(6):
        a = rng.integers(0, 3000, 200_000).astype(np.uint64)
        b = rng.integers(0, 1 << 32, 200_000).astype(np.uint64)
        vb.record_pairs(pool, cfg, a, b)
        opool.set_cells(ocfg.pair_cells(a, b))
        pool.advance_slice()
        opool.advance()
    hosts = np.arange(0, 3000, 3, dtype=np.uint64)
    want = vo.host_g0(opool, ocfg, hosts, 5)
    for opt in (1, 2, 0):
        check(lib.vate_pool_set_option(pool.handle, 0, opt))
        got = vb.inactive_virtual_counts(pool, cfg, hosts, 5)
        assert np.array_equal(got, want), (c, g, opt)


# --- incremental g0 (inverse index) vs full recompute vs oracle ---------------------

def test_incremental_estimate_paths_match_oracle():
    """Host churn (misses -> rebuild), a burst that flips most cells (refresh
    path) and quiet slices (pure delta) -- every slice equals the oracle, and the
    run exercises each path of the incremental estimate."""
    cfg = vb.EstimatorConfig(256, 16, 8, seed=12)
    ocfg = vo.OracleConfig(256, 16, 8, seed=12)
    pool = cfg.build_pool()
    pipe = vb.Pipeline(pool, cfg, 6)
    opipe = vo.OraclePipeline(ocfg, 6)
    rng = np.random.default_rng(3)
    for t in range(40):
        base = 1000 * (t // 12)                      # new host population every 12 slices
        n = 3000
        a = (base + rng.integers(0, 400, n)).astype(np.uint64)
        b = rng.integers(0, 40, n).astype(np.uint64)  # few peers: a steady, low-churn pool
        if t == 20:                                   # one burst that sets most of the pool
            a = np.concatenate([a, rng.integers(0, 400, 400_000).astype(np.uint64)])
            b = np.concatenate([b, rng.integers(0, 1 << 32, 400_000).astype(np.uint64)])
        got, _ = pipe.process_slice_soa(t, a, b)
        want = opipe.process_slice(t, a, b)
        assert np.array_equal(got.host, want.reports.host), t
        assert np.array_equal(got.estimate, want.reports.estimate), t
        assert pipe.last_pool_inactive == want.pool_inactive, t
    st = pool.inc_stats()
    assert st["rebuilds"] >= 2 and st["delta_slices"] >= 20 and st["refresh_slices"] >= 1, st
    pipe.close()


def test_incremental_survives_outside_pool_changes():
    """set_many / load between estimates are just more flipped cells."""
    cfg = vb.EstimatorConfig(128, 14, 6, seed=5)
    ocfg = vo.OracleConfig(128, 14, 6, seed=5)
    pool = cfg.build_pool()
    pipe = vb.Pipeline(pool, cfg, 6)
    opipe = vo.OraclePipeline(ocfg, 6)
    rng = np.random.default_rng(8)
    for t in range(15):
        a = rng.integers(0, 200, 2000).astype(np.uint64)
        b = rng.integers(0, 30, 2000).astype(np.uint64)
        if t == 7:
            extra = rng.integers(0, 1 << 14, 500).astype(np.uint64)
            pool.set_many(extra)
            opipe.pool.set_cells(extra)
        if t == 11:
            blob = pool.snapshot_bytes()
            pool.set_many(rng.integers(0, 1 << 14, 3000).astype(np.uint64))
            check_blob = vb.AtPool.from_bytes(blob)   # reload the saved state in place
            from paper_1812_00282_b200._lib import lib, ptr
            arr = np.frombuffer(blob, dtype=np.uint8)
            assert lib.vate_load(pool.handle, ptr(arr), arr.size) == 0
            assert check_blob.snapshot_bytes() == pool.snapshot_bytes()
        got, _ = pipe.process_slice_soa(t, a, b)
        want = opipe.process_slice(t, a, b)
        assert np.array_equal(got.estimate, want.reports.estimate), t
    assert pool.inc_stats()["delta_slices"] >= 10
    pipe.close()


def test_incremental_off_equals_on():
    cfg = vb.EstimatorConfig(1024, 20, 10, seed=0)
    p_on, p_off = cfg.build_pool(), cfg.build_pool()
    p_off.set_option("incremental", 0)
    a_on, a_off = vb.Pipeline(p_on, cfg, 10), vb.Pipeline(p_off, cfg, 10)
    from oracle import vate_oracle as vo2
    for t in range(30):
        a, b = vo2.synthetic_slice(t, 200_000, 20_000)
        r1, _ = a_on.process_slice_soa(t, a, b)
        r2, _ = a_off.process_slice_soa(t, a, b)
        assert np.array_equal(r1.host, r2.host) and np.array_equal(r1.estimate, r2.estimate)
    assert p_on.inc_stats()["delta_slices"] >= 25
    assert p_off.inc_stats()["delta_slices"] == 0


def test_active_set_reuse_is_exact():
    """The registry reuses last slice's sorted active list only when no host
    entered or left; interleave quiet slices with joins, departures, k' changes
    and a second registry on the same pool."""
    pool = vb.AtPool(12, 6)
    reg = vb.SlidingHostSet(6, pool=pool)
    other = vb.SlidingHostSet(6, pool=pool)
    ref = vo.OracleHosts(6)
    rng = np.random.default_rng(21)
    keys = rng.integers(0, 1 << 40, 500).astype(np.uint64)
    for t in range(40):
        if t % 9 == 4:
            batch = rng.integers(0, 1 << 40, 50).astype(np.uint64)      # joins
        elif t % 9 == 7:
            batch = np.empty(0, dtype=np.uint64)                       # departures age out
        else:
            batch = keys                                               # quiet
        reg.update(batch, t)
        ref.update(batch, t)
        other.update(keys[:10], t)
        for kp in (6, 6, 3, 6):
            assert np.array_equal(reg.active(t, kp), ref.active(t, kp)), (t, kp)
        assert len(other.active(t, 6)) == 10


@pytest.mark.parametrize("mode", ["streamed", "staged", "fast-device", "fast-staged"])
def test_streaming_steps_match_oracle(mode):
    """The bench's paths: packed records, async report D2H (double-buffered),
    the advance collected one slice late, and (staged) H2D prefetch."""
    cfg = vb.EstimatorConfig(1024, 20, 10, seed=0)
    ocfg = vo.OracleConfig(1024, 20, 10, seed=0)
    pool = cfg.build_pool()
    pipe = vb.Pipeline(pool, cfg, 10)
    opipe = vo.OraclePipeline(ocfg, 10)
    n, hosts = 150_000, 20_000
    cap = hosts + 16
    outs = [(np.empty(cap, np.uint64), np.empty(cap, np.float64), np.empty(cap, np.float64),
             np.empty(cap, np.uint8)) for _ in range(2)]
    pending = None
    cleared = 0
    slices = [vo.synthetic_slice(t, n, hosts) for t in range(30)]
    packed = [np.ascontiguousarray(np.stack([a, b], axis=1).astype(np.uint32)) for a, b in slices]
    staged = pipe.stage_packed(packed[0].ctypes.data, n) if "staged" in mode else None
    import torch
    dev = [torch.from_numpy(x.view(np.int32)).cuda() for x in packed] if mode == "fast-device" else None
    torch.cuda.synchronize()
    for t in range(30):
        if mode == "staged":
            nxt = pipe.stage_packed(packed[t + 1].ctypes.data, n) if t + 1 < 30 else None
            rep = pipe.step_staged(t, staged, n, outs[t % 2], wait=False)
            staged = nxt
        elif mode == "fast-staged":
            nxt = pipe.stage_packed(packed[t + 1].ctypes.data, n) if t + 1 < 30 else None
            rep = pipe.step_fast(t, staged, n, "staged", outs[t % 2])
            staged = nxt
        elif mode == "fast-device":
            rep = pipe.step_fast(t, dev[t].data_ptr(), n, "device", outs[t % 2])
        else:
            rep = pipe.step_packed(t, packed[t].ctypes.data, n, False, outs[t % 2], wait=False)
        want = opipe.process_slice(t, *slices[t])
        cleared += want.cleared
        if pending is not None:          # slice t-1's rows are complete after slice t began
            pipe.wait_reports()
            prev_rep, prev_want = pending
            assert np.array_equal(prev_rep.host, prev_want.reports.host)
            assert np.array_equal(prev_rep.estimate, prev_want.reports.estimate)
            assert np.array_equal(prev_rep.z_v, prev_want.reports.z_v)
        pending = (rep, want)
    pipe.wait_reports()
    assert np.array_equal(pending[0].estimate, pending[1].reports.estimate)
    assert pool.snapshot_bytes() == opipe.pool.snapshot_bytes()
    assert pipe.total_cleared == cleared          # every deferred advance was collected
    st = pool.inc_stats()
    assert st["delta_slices"] > 20, st


def test_identity_path_when_population_is_stable():
    """Every host appears every slice: the sorted active list is reused and the
    index's g0 array is the estimate input (no lookup) -- still oracle-exact."""
    cfg = vb.EstimatorConfig(512, 18, 8, seed=2)
    ocfg = vo.OracleConfig(512, 18, 8, seed=2)
    pool = cfg.build_pool()
    pipe = vb.Pipeline(pool, cfg, 8)
    opipe = vo.OraclePipeline(ocfg, 8)
    rng = np.random.default_rng(4)
    hosts = np.repeat(np.arange(5000, dtype=np.uint64), 4)
    for t in range(20):
        b = rng.integers(0, 12, hosts.size).astype(np.uint64) + (hosts << np.uint64(4))
        got, _ = pipe.process_slice_soa(t, hosts, b)
        want = opipe.process_slice(t, hosts, b)
        assert np.array_equal(got.estimate, want.reports.estimate), t
    st = pool.inc_stats()
    assert st["identity_slices"] >= 15, st


def test_step_fast_device_resident_reports():
    """out=None keeps the rows in HBM; reading them back equals the oracle."""
    import ctypes
    import os

    import nvidia.cuda_runtime
    import torch
    cudart = ctypes.CDLL(os.path.join(os.path.dirname(nvidia.cuda_runtime.__file__), "lib",
                                      "libcudart.so.12"))
    cfg = vb.EstimatorConfig(256, 16, 6, seed=9)
    ocfg = vo.OracleConfig(256, 16, 6, seed=9)
    pipe = vb.Pipeline(cfg.build_pool(), cfg, 6)
    opipe = vo.OraclePipeline(ocfg, 6)
    for t in range(10):
        a, b = vo.synthetic_slice(t, 50_000, 3_000)
        dev = torch.from_numpy(np.stack([a, b], axis=1).astype(np.uint32).view(np.int32)).cuda()
        torch.cuda.synchronize()
        m = pipe.step_fast(t, dev.data_ptr(), len(a), "device", None)
        want = opipe.process_slice(t, a, b).reports
        pipe.wait_reports()
        pipe.pool.synchronize()
        hp, ep, zp, sp = pipe.reports_device()
        assert m == len(want.host) and hp and ep
        est = np.empty(m, np.float64)
        host = np.empty(m, np.uint64)
        assert cudart.cudaMemcpy(ctypes.c_void_p(est.ctypes.data), ctypes.c_void_p(ep),
                                 ctypes.c_size_t(m * 8), 2) == 0   # device -> host
        assert cudart.cudaMemcpy(ctypes.c_void_p(host.ctypes.data), ctypes.c_void_p(hp),
                                 ctypes.c_size_t(m * 8), 2) == 0
        assert np.array_equal(est, want.estimate), t
        assert np.array_equal(host, want.host), t


def test_incremental_extend_merges_new_hosts():
    """A steady population plus a trickle of new hosts: the misses are merged
    into the index (streaming CSR merge) without a rebuild -- every slice
    oracle-exact."""
    cfg = vb.EstimatorConfig(256, 16, 20, seed=13)
    ocfg = vo.OracleConfig(256, 16, 20, seed=13)
    pool = cfg.build_pool()
    pipe = vb.Pipeline(pool, cfg, 20)
    opipe = vo.OraclePipeline(ocfg, 20)
    rng = np.random.default_rng(6)
    base = np.repeat(np.arange(1000, dtype=np.uint64), 3)
    for t in range(60):
        new = (np.arange(1000 + 10 * t, 1010 + 10 * t, dtype=np.uint64) if t < 40
               else np.empty(0, dtype=np.uint64))
        a = np.concatenate([base, new])
        b = (rng.integers(0, 8, a.size).astype(np.uint64) + (a << np.uint64(3)))
        got, _ = pipe.process_slice_soa(t, a, b)
        want = opipe.process_slice(t, a, b)
        assert np.array_equal(got.host, want.reports.host), t
        assert np.array_equal(got.estimate, want.reports.estimate), t
    st = pool.inc_stats()
    assert st["extends"] >= 2 and st["rebuilds"] == 1, st


# --- the multi-GPU merge kernels, exercised with two replicas on one device --------

def test_replica_merge_and_range_split_equal_one_pool():
    """Two replica pools (the N=2 protocol of paper_1812_00282_b200.parallel, with
    the NCCL all-gather replaced by a device concatenation): dirty bitmaps OR'ed
    into both replicas reproduce the single pool's ATP1 bytes every slice, and the
    aip-range-split estimate (vate_estimate_begin_hosts) concatenates to the
    single pipeline's reports."""
    import ctypes as C

    import torch
    from paper_1812_00282_b200._lib import check, lib, ptr
    from paper_1812_00282_b200.estimator import log_zp
    from paper_1812_00282_b200.parallel import split_range, union_sorted

    cfg = vb.EstimatorConfig(256, 16, 8, seed=21)
    single = vb.Pipeline(cfg.build_pool(), cfg, 8)
    reps = [vb.Pipeline(cfg.build_pool(), cfg, 8) for _ in range(2)]
    nwords = (1 << 16) // 32
    bm = torch.zeros(2 * nwords, dtype=torch.int32, device="cuda")
    rng = np.random.default_rng(0)
    for t in range(24):
        a = (0x0A000000 + rng.integers(0, 2000, 30_000)).astype(np.uint64)
        b = rng.integers(1, 1 << 32, 30_000).astype(np.uint64)
        want, _ = single.process_slice_soa(t, a, b)
        for r, pipe in enumerate(reps):            # each replica scans its round-robin shard
            pipe._t = t
            pipe._scan(a[r::2], b[r::2])
        torch.cuda.synchronize()
        for r, pipe in enumerate(reps):
            pipe.pool.synchronize()
            check(lib.vate_dirty_bitmap(pipe.pool.handle, bm[r * nwords:].data_ptr()))
            pipe.pool.synchronize()
        for pipe in reps:
            check(lib.vate_merge_dirty(pipe.pool.handle, bm.data_ptr(), 2))
            pipe.pool.synchronize()
        hosts = union_sorted([p.hosts.active(t, 8) for p in reps])
        got_host, got_est = [], []
        for r, pipe in enumerate(reps):
            lo, hi = split_range(len(hosts), r, 2)
            mine = np.ascontiguousarray(hosts[lo:hi])
            p_in = C.c_uint64()
            check(lib.vate_estimate_begin_hosts(pipe.pool.handle, ptr(mine), mine.size, 0, cfg.g,
                                                cfg.cell_stream, 8, C.byref(p_in)))
            assert p_in.value == single.last_pool_inactive, t
            if mine.size:
                out = (np.empty(mine.size, np.uint64), np.empty(mine.size, np.float64),
                       np.empty(mine.size, np.float64), np.empty(mine.size, np.uint8))
                kept = C.c_uint64()
                check(lib.vate_estimate_finish(pipe.pool.handle, cfg.g, p_in.value,
                                               log_zp(p_in.value, 1 << 16)[0], 0.0,
                                               *(ptr(x) for x in out), mine.size, C.byref(kept)))
                got_host.append(out[0][:kept.value])
                got_est.append(out[1][:kept.value])
        assert np.array_equal(np.concatenate(got_host), want.host), t
        assert np.array_equal(np.concatenate(got_est), want.estimate), t
        for pipe in reps:
            pipe._maintain(t)
            assert pipe.pool.snapshot_bytes() == single.pool.snapshot_bytes(), t


def test_replica_step_protocol_device_resident():
    """ReplicaStep's device phases with two replicas on one device (the NCCL
    all-gathers replaced by device concatenation): dirty bitmaps merge the cells,
    vate_hosts_touched + absorb make both registries hold the single pipeline's
    host set, and vate_estimate_begin_part shares (incremental g0 on) concatenate
    to the single pipeline's reports, slice after slice, with host churn."""
    import torch
    from paper_1812_00282_b200 import parallel as par

    cfg = vb.EstimatorConfig(512, 16, 10, seed=5)
    kp = 7
    single = vb.Pipeline(cfg.build_pool(), cfg, kp)
    reps = [vb.Pipeline(cfg.build_pool(), cfg, kp) for _ in range(2)]
    nwords = (1 << 16) // 32
    bm = torch.zeros(2 * nwords, dtype=torch.int32, device="cuda")
    rng = np.random.default_rng(3)
    for t in range(40):
        n = int(rng.integers(0, 40_000)) if t % 9 != 4 else 0
        lo_host = 200 * (t // 10)                 # the host population drifts
        a = (0x0A000000 + lo_host + rng.integers(0, 3000, n)).astype(np.uint32)
        b = rng.integers(1, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        want, _ = single.process_slice_soa(t, a.astype(np.uint64), b.astype(np.uint64))
        touched = []
        for r, pipe in enumerate(reps):
            pairs = np.ascontiguousarray(np.stack([a[r::2], b[r::2]], axis=1))
            dev = torch.from_numpy(pairs.view(np.int32)).cuda()
            pipe.scan_packed(t, dev.data_ptr(), len(pairs), True)
            par.dirty_bitmap(pipe, bm[r * nwords:].data_ptr())
            keys = torch.empty(max(len(pairs), 1), dtype=torch.int64, device="cuda")
            m = par.touched_hosts(pipe, t, keys.data_ptr(), keys.numel())
            assert m == len(np.unique(a[r::2])), t
            touched.append((keys, m))
        for r, pipe in enumerate(reps):
            par.merge_dirty(pipe, bm.data_ptr(), 2)
            keys, m = touched[1 - r]
            par.absorb_hosts(pipe, keys.data_ptr(), m, t)
        want_hosts = single.hosts.active(t, kp)
        got_host, got_est, got_zv = [], [], []
        for r, pipe in enumerate(reps):
            assert np.array_equal(pipe.hosts.active(t, kp), want_hosts), t
            rep = pipe.estimate_soa(t, advance=True, wait=True, part=r, nparts=2)
            pipe._collect(t)
            if rep is not None:
                assert rep.z_p == want.z_p, t
                got_host.append(rep.host.copy())
                got_est.append(rep.estimate.copy())
                got_zv.append(rep.z_v.copy())
        if want is None:
            assert not got_host, t
        else:
            assert np.array_equal(np.concatenate(got_host), want.host), t
            assert np.array_equal(np.concatenate(got_est), want.estimate), t
            assert np.array_equal(np.concatenate(got_zv), want.z_v), t
        for pipe in reps:
            assert pipe.pool.snapshot_bytes() == single.pool.snapshot_bytes(), t
            assert len(pipe.hosts) == len(single.hosts), t


def test_replica_step_over_nccl_world1():
    """ReplicaStep itself (NCCL plumbing, stream hand-off, staged/host/device
    inputs) on a world-size-1 NCCL group equals the single pipeline."""
    import socket

    import torch
    import torch.distributed as dist
    from paper_1812_00282_b200.parallel import ReplicaStep

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    try:
        cfg = vb.EstimatorConfig(256, 15, 6, seed=8)
        single = vb.Pipeline(cfg.build_pool(), cfg, 5)
        pipe = vb.Pipeline(cfg.build_pool(), cfg, 5)
        step = ReplicaStep(pipe, dist, torch)
        rng = np.random.default_rng(4)
        for t in range(16):
            n = int(rng.integers(1, 20_000))
            a = (0x0A000000 + rng.integers(0, 1500, n)).astype(np.uint32)
            b = rng.integers(1, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
            pairs = np.ascontiguousarray(np.stack([a, b], axis=1))
            want, _ = single.process_slice_soa(t, a.astype(np.uint64), b.astype(np.uint64))
            out = (np.empty(n, np.uint64), np.empty(n, np.float64), np.empty(n, np.float64),
                   np.empty(n, np.uint8))
            mode = ("device", "host", "staged")[t % 3]
            if mode == "device":
                src = torch.from_numpy(pairs.view(np.int32)).cuda()
                rep = step(t, src.data_ptr(), n, "device", out)
            elif mode == "host":
                rep = step(t, pairs.ctypes.data, n, "host", out)
            else:
                rep = step(t, pipe.stage_packed(pairs.ctypes.data, n), n, "staged", out)
            pipe.wait_reports()
            assert np.array_equal(rep.host, want.host), t
            assert np.array_equal(rep.estimate, want.estimate), t
            assert pipe.pool.snapshot_bytes() == single.pool.snapshot_bytes(), t
    finally:
        dist.destroy_process_group()


# --- the synthetic generators: device == oracle ----------------------------------------

def test_device_generators_equal_oracle():
    import torch
    from paper_1812_00282_b200._lib import check, lib
    from paper_1812_00282_b200.synth import ZipfTables
    pool = vb.AtPool(8, 2)
    n = 1_000_000
    out = torch.empty((n, 2), dtype=torch.int32, device="cuda")
    for t in (0, 7, 123456):
        check(lib.vate_synth_packets(pool.handle, t, n, 1_000_000, 0x0A000000, 0, out.data_ptr()))
        pool.synchronize()
        got = out.cpu().numpy().view(np.uint32)
        a, b = vo.synthetic_slice(t, n, 1_000_000)
        assert np.array_equal(got[:, 0], a) and np.array_equal(got[:, 1], b), t
    zt = ZipfTables(0, 1_000_000)
    assert np.array_equal(zt.z.cpu().numpy().view(np.uint64), vo.zipf_cdf(1_000_000))
    assert np.array_equal(zt.s.cpu().numpy().view(np.uint64), vo.spreader_cdf())
    for t in (0, 3):
        zt.packets(pool, t, n, 0x0A000000, 0, out.data_ptr())
        pool.synchronize()
        got = out.cpu().numpy().view(np.uint32)
        a, b = vo.synthetic_zipf_slice(t, n, 1_000_000, vo.zipf_cdf(1_000_000), vo.spreader_cdf())
        assert np.array_equal(got[:, 0], a) and np.array_equal(got[:, 1], b), t


def test_full_size_cfg3_zipf_superspreaders():
    """BASELINE cfg 3: Zipf hosts + 64 super-spreaders with random peers (10 % of
    5M packets), pool 2^26: P, maintenance, sampled g0 (spreaders included) and the
    final ATP1 snapshot equal the oracle replaying the same packets."""
    c, k = 26, 60
    cfg = vb.EstimatorConfig(1024, c, k)
    ocfg = vo.OracleConfig(1024, c, k)
    pool = cfg.build_pool()
    pipe = vb.Pipeline(pool, cfg, k)
    opool = vo.OraclePool(c, k)
    zc, sc = vo.zipf_cdf(1_000_000), vo.spreader_cdf()
    for t in range(4):
        a, b = vo.synthetic_zipf_slice(t, 5_000_000, 1_000_000, zc, sc)
        got, _ = pipe.process_slice_soa(t, a, b)
        opool.set_cells(ocfg.pair_cells(a, b))
        assert pipe.last_pool_inactive == opool.count_inactive(k)
        sample = np.unique(np.concatenate([
            np.random.default_rng(t).choice(got.host, 2000, replace=False),
            np.arange(vo.SPREAD_BASE, vo.SPREAD_BASE + 64, dtype=np.uint64)]))
        idx = np.searchsorted(got.host, sample)
        assert np.array_equal(got.host[idx], sample)
        want = vo.reports_soa(ocfg, sample, vo.host_g0(opool, ocfg, sample, k),
                              pipe.last_pool_inactive, t, k)
        assert np.array_equal(got.estimate[idx], want.estimate), t
        due, visited, cleared = opool.advance()
        m = pipe.last_maintenance
        assert (m.blocks, m.cells_maintained, m.cells_cleared) == (due, visited, cleared)
    assert pool.snapshot_bytes() == opool.snapshot_bytes()


@pytest.mark.parametrize("inc_sort", [1, 0])
def test_active_set_merge_under_small_churn(inc_sort):
    """SlidingHostSet.active (pipeline.py:54-58) when a few hosts join and leave
    each slice: the sorted active set is updated by merging the sorted arrivals
    and dropping the departures (VATE_OPT_INC_SORT) -- equal to the oracle's set,
    reports and all, slice by slice, with the special key 2^64-1 among them."""
    cfg = vb.EstimatorConfig(128, 14, 8, seed=6)
    ocfg = vo.OracleConfig(128, 14, 8, seed=6)
    pool = cfg.build_pool()
    pool.set_option("inc_sort", inc_sort)
    pipe = vb.Pipeline(pool, cfg, 5)
    opipe = vo.OraclePipeline(ocfg, 5)
    rng = np.random.default_rng(12)
    base = rng.choice(1 << 40, 3000, replace=False).astype(np.uint64)
    for t in range(30):
        churn = rng.choice(1 << 40, 20, replace=False).astype(np.uint64) + np.uint64(1 << 41)
        a = np.concatenate([base[rng.integers(0, len(base), 6000)], churn])
        if t % 7 == 3:
            a = np.concatenate([a, np.array([2**64 - 1], dtype=np.uint64)])
        b = rng.integers(1, 1 << 40, len(a)).astype(np.uint64)
        got, _ = pipe.process_slice_soa(t, a, b)
        want = opipe.process_slice(t, a, b)
        assert np.array_equal(got.host, want.reports.host), t
        assert np.array_equal(got.estimate, want.reports.estimate), t
    st = pool.sort_stats()
    if inc_sort:
        assert st["incremental"] > 10, st
    else:
        assert st["incremental"] == 0, st


@pytest.mark.parametrize("form", [(f, d, m) for f in (0, 1) for d in (0, 1, 2) for m in (0, 1)])
def test_scan_forms_are_equivalent(form):
    """Every packed-scan form -- the per-CTA registry-stamp filter on / off
    (VATE_OPT_SCAN_FILTER), direct cell stores or the deferred pending-set
    marks (VATE_OPT_DEFERRED) or the bit-plane history (d = 2,
    VATE_OPT_BITPLANE), 16-byte aligned input (two packets per thread,
    plus the odd last packet) or misaligned input (one packet per thread),
    with the L2 evict_last hints (VATE_OPT_L2_KEEP) paired with the filter --
    leaves the reference's cells and host set: ATP1 bytes, reports and the
    registry after skewed traffic (a heavy host, odd packet counts) equal the
    oracle's, slice by slice."""
    import torch
    filt, deferred, misaligned = form
    cfg = vb.EstimatorConfig(256, 16, 6, seed=5)
    ocfg = vo.OracleConfig(256, 16, 6, seed=5)
    pool = cfg.build_pool()
    pool.set_option("scan_filter", filt)
    pool.set_option("l2_keep", filt)
    pool.set_option("deferred", min(deferred, 1))
    pool.set_option("bitplane", 1 if deferred == 2 else 0)
    pipe = vb.Pipeline(pool, cfg, 5)
    opipe = vo.OraclePipeline(ocfg, 5)
    rng = np.random.default_rng(31)
    for t in range(10):
        n = int(rng.integers(1, 9000)) | 1 if t % 3 else 4096 + 3
        a = (0x0A000000 + rng.integers(0, 900, n)).astype(np.uint32)
        a[rng.random(n) < 0.3] = 0x0A0000FF                      # a heavy hitter
        b = rng.integers(1, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        flat = np.ascontiguousarray(np.stack([a, b], axis=1)).view(np.int32).reshape(-1)
        buf = torch.zeros(flat.size + 2, dtype=torch.int32, device="cuda")
        buf[misaligned * 2: misaligned * 2 + flat.size] = torch.from_numpy(flat).cuda()
        got = pipe.step_fast(t, buf.data_ptr() + 8 * misaligned, n, "device",
                             (np.empty(2048, np.uint64), np.empty(2048), np.empty(2048),
                              np.empty(2048, np.uint8)))
        pipe.wait_reports()
        want = opipe.process_slice(t, a.astype(np.uint64), b.astype(np.uint64))
        assert np.array_equal(got.host, want.reports.host), (form, t)
        assert np.array_equal(got.estimate, want.reports.estimate), (form, t)
        assert pool.snapshot_bytes() == opipe.pool.snapshot_bytes(), (form, t)


@pytest.mark.parametrize("floor,hosts0,two_calls", [(0.0, 900, False), (30.0, 900, False),
                                                   (0.0, 30_000, False), (30.0, 30_000, True)])
def test_lagged_step_equals_oracle(floor, hosts0, two_calls):
    """Pipeline.step_lagged (vate_slice_step_lagged): slice t's reports arrive
    with the call for slice t+1 and equal the oracle's, the ATP1 snapshot after
    each call equals the oracle's after the same slice (scan + advance), with
    host churn, an empty slice, prunes (t % k == 0), a floor, and -- with 30k new
    hosts in the first slices -- registry growth and parked inserts completed
    while the next scan runs."""
    import torch
    cfg = vb.EstimatorConfig(256, 16, 6, seed=12)
    ocfg = vo.OracleConfig(256, 16, 6, seed=12)
    pool = cfg.build_pool()
    pipe = vb.Pipeline(pool, cfg, 5, floor=floor)
    if two_calls:   # as for pools beyond the log table: np.log of P per slice, two calls
        pipe._lzp_tab = None
        import paper_1812_00282_b200.pipeline as pl
        orig = pl.log_zp_table
        pl.log_zp_table = lambda c: None
    opipe = vo.OraclePipeline(ocfg, 5, floor=floor)
    rng = np.random.default_rng(8)
    want = {}
    outs = [tuple(np.empty(40_000, dt) for dt in (np.uint64, np.float64, np.float64, np.uint8))
            for _ in range(2)]

    def check_rows(res):
        if res is None:
            return
        tp, rows = res
        w = want.pop(tp)
        if w.reports is None or len(w.reports.host) == 0:
            assert rows is None or len(rows.host) == 0, tp
            return
        assert np.array_equal(rows.host, w.reports.host), tp
        assert np.array_equal(rows.estimate, w.reports.estimate), tp
        assert np.array_equal(rows.z_v, w.reports.z_v), tp
        assert np.array_equal(rows.saturated, w.reports.saturated), tp

    for t in range(20):
        n = 0 if t == 7 else int(rng.integers(5_000, 20_000))
        span = hosts0 if t < 4 else 900
        lo = 0 if t < 10 else 400
        a = (0x0A000000 + rng.integers(lo, lo + span, n)).astype(np.uint32)
        b = rng.integers(1, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        pairs = torch.from_numpy(np.ascontiguousarray(np.stack([a, b], axis=1)).view(np.int32)).cuda()
        res = pipe.step_lagged(t, pairs.data_ptr() if n else 0, n, "device", outs[t % 2])
        pipe.wait_reports()
        check_rows(res)
        want[t] = opipe.process_slice(t, a.astype(np.uint64), b.astype(np.uint64))
        assert pool.snapshot_bytes() == opipe.pool.snapshot_bytes(), t
    res = pipe.flush_lagged(outs[0])
    pipe.wait_reports()
    check_rows(res)
    assert not want
    if two_calls:
        pl.log_zp_table = orig


@pytest.mark.parametrize("deferred", [0, 1, 2])
def test_u16_pass_forms_over_two_windows(deferred):
    """u16 cells (k = 300, the cfg 4 width) on a small pool for 2k + 5 slices:
    direct or deferred stores or the bit-plane history (2; window k' = 293, so
    two suffix builds), through the lagged slice step; the ATP1 bytes, P, maintenance and every report equal
    the oracle's, with the clock wrapping and every block swept twice."""
    k, c = 300, 16
    cfg = vb.EstimatorConfig(64, c, k, seed=9)
    ocfg = vo.OracleConfig(64, c, k, seed=9)
    pool = cfg.build_pool()
    pool.set_option("deferred", min(deferred, 1))
    pool.set_option("bitplane", 1 if deferred == 2 else 0)
    pipe = vb.Pipeline(pool, cfg, k - 7)
    opipe = vo.OraclePipeline(ocfg, k - 7)
    rng = np.random.default_rng(77)
    outs = [tuple(np.empty(4096, dt) for dt in (np.uint64, np.float64, np.float64, np.uint8))
            for _ in range(2)]
    want = {}

    def check(res):
        if res is None:
            return
        tp, rows = res
        ww = want.pop(tp)
        assert pipe.last_pool_inactive == ww.pool_inactive or ww.reports is None, tp
        m = pipe.last_maintenance
        assert (m.blocks, m.cells_maintained, m.cells_cleared) == (ww.due, ww.visited, ww.cleared)
        if ww.reports is None or len(ww.reports.host) == 0:
            assert rows is None or len(rows.host) == 0, tp
        else:
            assert np.array_equal(rows.host, ww.reports.host), tp
            assert np.array_equal(rows.estimate, ww.reports.estimate), tp
            assert np.array_equal(rows.z_v, ww.reports.z_v), tp

    for t in range(2 * k + 5):
        n = int(rng.integers(0, 300))
        a = (0x0A000000 + rng.integers(0, 500, n)).astype(np.uint32)
        b = rng.integers(1, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        pairs = np.ascontiguousarray(np.stack([a, b], axis=1))
        res = pipe.step_lagged(t, pairs.ctypes.data, n, "host", outs[t % 2])
        want[t] = opipe.process_slice(t, a.astype(np.uint64), b.astype(np.uint64))
        pipe.wait_reports()
        check(res)
        if t % 50 == 0:     # slice t's scan, pass and sweep are enqueued: the pool after t
            assert pool.snapshot_bytes() == opipe.pool.snapshot_bytes(), t
    check(pipe.flush_lagged(outs[(2 * k + 5) % 2]))
    pipe.wait_reports()
    assert not want
    assert pool.snapshot_bytes() == opipe.pool.snapshot_bytes()
    assert pool.mode()["bitplane"] == (deferred == 2)
    pipe.close()
    pool.close()


@pytest.mark.parametrize("c,k,kp", [(12, 6, 6), (12, 6, 4), (14, 40, 33), (10, 2, 2)])
def test_bitplane_mixed_api(c, k, kp):
    """Bit-plane mode under the whole pool protocol, not just the slice step:
    set_many batches, the estimate's width and other widths (count_inactive,
    inactive_mask), advances with and without an estimate in the epoch,
    snapshots mid-epoch, loading a snapshot and writing cells (the history is
    rebuilt), for many windows (block boundaries every k' epochs) -- the cells,
    P and the maintenance reports equal the oracle pool's throughout."""
    pool = vb.AtPool(c, k)
    pool.set_option("bitplane", 1)
    opool = vo.OraclePool(c, k)
    rng = np.random.default_rng(c * 100 + k)
    S = 1 << c
    assert pool.count_inactive(kp) == opool.count_inactive(kp)
    assert pool.mode()["bitplane"] and pool.mode()["window"] == kp
    for t in range(6 * k + 9):
        for _ in range(int(rng.integers(0, 3))):
            idx = rng.integers(0, S, int(rng.integers(0, S // 8 + 1))).astype(np.uint64)
            pool.set_many(idx)
            opool.set_cells(idx)
        if t % 3 != 2:
            assert pool.count_inactive(kp) == opool.count_inactive(kp), t
        if t % 7 == 3:
            k2 = int(rng.integers(1, k + 1))
            assert pool.count_inactive(k2) == opool.count_inactive(k2), (t, k2)
            q = rng.integers(0, S, 64).astype(np.uint64)
            assert np.array_equal(pool.inactive_mask(q, kp), opool.inactive_mask(q, kp)), t
        if t % 11 == 5:
            assert pool.snapshot_bytes() == opool.snapshot_bytes(), t
        if t % 17 == 9:        # reload from bytes: the history is rebuilt from the cells
            blob = pool.snapshot_bytes()
            pool.close()
            pool = vb.AtPool.from_bytes(blob)
            pool.set_option("bitplane", 1)
        if t % 19 == 12:       # explicit cell values: the history is rebuilt
            i = int(rng.integers(0, S))
            pool.cells.set_one(i, 2 * k)
            opool.cells[i] = 2 * k
        rep = pool.advance_slice()
        want = opool.advance()
        assert (rep.blocks, rep.cells_maintained, rep.cells_cleared) == want, t
    assert pool.snapshot_bytes() == opool.snapshot_bytes()
    pool.close()
