"""Generate golden vectors by running the REFERENCE package (slidecard).

Run in the build container, where the read-only reference is mounted:

    python tests/golden/make_golden.py

It imports ``slidecard`` from ``/root/reference/pkg/src`` and records what the
reference computes for hashing, block layout, the estimator float path, and
whole multi-slice pipelines.  The outputs (``*.npz``) are committed so the
tests can use them on the GPU box, where ``/root/reference`` does not exist.

Recorded per pipeline slice (pipeline.py:142-160 order): the sorted active host
set, the reference's pool-wide inactive count P, the integer g0 per host, the
float reports (estimate, z_v, saturated), the floor-filtered host list, the
MaintenanceReport of the advance, and the SHA-256 of the ATP1 snapshot taken
after the advance (pools.py:261-265).
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from slidecard import estimator as est          # noqa: E402
from slidecard import hashing                   # noqa: E402
from slidecard.pipeline import Pipeline          # noqa: E402
from slidecard.pools import AtPool               # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from specs import COMPARATORS, PIPELINES, gen_slices as _slices  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
M64 = (1 << 64) - 1


def hash_kats():
    rng = np.random.default_rng(20240607)
    z = rng.integers(0, 1 << 64, size=256, dtype=np.uint64)
    z[:4] = [0, 1, 2, M64]
    mix = hashing.mix64_vec(z)
    seeds = np.array([0, 1, 7, 123456789012345, M64], dtype=np.uint64)
    cs = np.array([hashing.derive_stream(int(s), hashing.CELL_SALT) for s in seeds], dtype=np.uint64)
    gs = np.array([hashing.derive_stream(int(s), hashing.GROUP_SALT) for s in seeds], dtype=np.uint64)
    bips = rng.integers(0, 1 << 64, size=512, dtype=np.uint64)
    bips[:256] &= np.uint64(0xFFFFFFFF)
    gvals = np.array([1, 2, 3, 1000, 1024, 4096, (1 << 20) + 7, 1 << 32], dtype=np.uint64)
    group = np.stack([hashing.group_index_vec(bips, int(g), int(gs[si]))
                      for si in range(len(seeds)) for g in gvals])
    aips = rng.integers(0, 1 << 64, size=512, dtype=np.uint64)
    aips[:256] &= np.uint64(0xFFFFFFFF)
    vids = rng.integers(0, 1 << 32, size=512, dtype=np.uint64)
    cvals = np.array([1, 5, 20, 24, 28, 32], dtype=np.uint64)
    cell = np.stack([hashing.cell_index_vec(aips, vids, int(c), int(cs[si]))
                     for si in range(len(seeds)) for c in cvals])
    np.savez_compressed(os.path.join(OUT, "hash_kats.npz"), z=z, mix=mix, seeds=seeds,
                        cell_stream=cs, group_stream=gs, bips=bips, gvals=gvals,
                        group=group, aips=aips, vids=vids, cvals=cvals, cell=cell)


LAYOUTS = [(10, 4, "tail"), (10, 3, "low-dev"), (20, 10, "tail"), (24, 60, "tail"),
           (26, 60, "tail"), (28, 300, "tail"), (12, 1, "low-dev"), (14, 600, "low-dev"),
           (3, 2, "tail"), (16, 300, "tail"), (18, 30, "low-dev"), (32, 300, "tail"),
           (32, 1 << 15, "low-dev"), (5, 16, "low-dev")]


def layouts():
    rows = {}
    rng = np.random.default_rng(5)
    for c, k, part in LAYOUTS:
        pool_cls = AtPool.__new__(AtPool)
        # build the layout without allocating 2^c cells: replicate __init__'s
        # shape fields, then use the reference's own block_of / block_range
        pool_cls.c, pool_cls.k, pool_cls.partition = c, k, part
        pool_cls.size, pool_cls.nblocks, pool_cls.sentinel = 1 << c, 2 * k, 2 * k
        if part == "tail":
            pool_cls._a = pool_cls.size // (pool_cls.nblocks - 1)
            pool_cls._b = pool_cls.size % (pool_cls.nblocks - 1)
        else:
            pool_cls._a2 = pool_cls.size // pool_cls.nblocks
            pool_cls._b2 = pool_cls.size % pool_cls.nblocks
            pool_cls._split = pool_cls._a2 * (pool_cls.nblocks - pool_cls._b2 + 1)
        ranges = np.array([pool_cls.block_range(b) for b in range(pool_cls.nblocks)],
                          dtype=np.uint64)
        idx = rng.integers(0, 1 << c, size=4096, dtype=np.uint64)
        edges = np.concatenate([ranges[:, 0], ranges[:, 1] - 1])
        if len(edges) > 2400:
            edges = edges[::37]
        idx = np.concatenate([idx, edges, [0, (1 << c) - 1]]).astype(np.uint64)
        pick = np.arange(len(ranges)) if len(ranges) <= 1200 else \
            np.unique(np.concatenate([np.arange(0, len(ranges), 97), [len(ranges) - 1]]))
        rows[f"{c}_{k}_{part}_bi"] = pick
        rows[f"{c}_{k}_{part}_ranges"] = ranges[pick]
        rows[f"{c}_{k}_{part}_idx"] = idx
        rows[f"{c}_{k}_{part}_block"] = pool_cls.block_of_vec(idx)
    np.savez_compressed(os.path.join(OUT, "layouts.npz"), **rows)


def estimator_kats():
    """reports_from_counts over edge cases and a dense (g0, P) grid (estimator.py:138-162)."""
    cases = []
    for g, c in ((1024, 12), (1024, 20), (1000, 18), (1, 4), (64, 10), (4096, 22)):
        cfg = est.EstimatorConfig(g, c, 8)
        size = 1 << c
        g0 = np.unique(np.concatenate([np.arange(0, g + 1, max(1, g // 97)), [0, 1, g - 1, g]]))
        g0 = g0[(g0 >= 0) & (g0 <= g)].astype(np.int64)
        for p in sorted({0, 1, size // 7, size // 2, (size * 9) // 10, size - 1, size}):
            reps = est.reports_from_counts(cfg, np.arange(len(g0), dtype=np.uint64), g0, p, 10, 8)
            cases.append((g, c, p, g0, np.array([r.estimate for r in reps]),
                          np.array([r.z_v for r in reps]), np.array([r.saturated for r in reps]),
                          reps[0].z_p))
    out = {}
    for i, (g, c, p, g0, e, zv, s, zp) in enumerate(cases):
        out[f"c{i}_meta"] = np.array([g, c, p], dtype=np.int64)
        out[f"c{i}_g0"] = g0
        out[f"c{i}_est"] = e
        out[f"c{i}_zv"] = zv
        out[f"c{i}_sat"] = s
        out[f"c{i}_zp"] = np.array([zp])
    out["n"] = np.array([len(cases)])
    np.savez_compressed(os.path.join(OUT, "estimator_kats.npz"), **out)


# --- whole pipelines ------------------------------------------------------------

def pipelines():
    for name, spec in PIPELINES.items():
        cfg = est.EstimatorConfig(spec["g"], spec["c"], spec["k"], seed=spec["seed"],
                                  partition=spec["part"])
        pool = cfg.build_pool()
        rec = {k: np.array(v) for k, v in spec.items() if k not in ("empty",)}
        rec["empty"] = np.array(sorted(spec.get("empty", ())), dtype=np.int64)
        pipe = Pipeline(pool, cfg, spec["kp"], floor=0.0)
        per_slice = []
        for t, aips, bips in _slices(spec):
            # the unfiltered reports plus P and g0 come from the same pool state
            # the pipeline's estimate phase sees: replay its phases explicitly
            pipe._scan(aips, bips)
            if len(aips):
                pipe.hosts.update(aips, t)
            live = pipe.hosts.active(t, spec["kp"])
            if len(live):
                p = pool.count_inactive(spec["kp"])
                g0 = est.inactive_virtual_counts(pool, cfg, live, spec["kp"])
                reps = est.reports_from_counts(cfg, live, g0, p, t, spec["kp"])
            else:
                p, g0, reps = -1, np.zeros(0, dtype=np.int64), []
            mrep = pool.advance_slice()
            if t % max(1, pool.k) == 0:
                pipe.hosts.prune(t)
            snap = pool.snapshot_bytes()
            per_slice.append(dict(
                t=t, live=live, p=p, g0=g0,
                est=np.array([r.estimate for r in reps], dtype=np.float64),
                zv=np.array([r.z_v for r in reps], dtype=np.float64),
                sat=np.array([r.saturated for r in reps], dtype=bool),
                zp=reps[0].z_p if reps else -1.0,
                kept=np.array([r.host for r in reps if r.estimate >= spec["floor"]]
                              if spec["floor"] > 0 else [r.host for r in reps], dtype=np.uint64),
                blocks=np.array(mrep.blocks, dtype=np.int64),
                maintained=mrep.cells_maintained, cleared=mrep.cells_cleared,
                bact0=pool.bact0, snap_sha=hashlib.sha256(snap).hexdigest()))
        pipe.close()
        # cross-check: the reference Pipeline itself, floor applied, gives the kept lists
        pool2 = cfg.build_pool()
        with Pipeline(pool2, cfg, spec["kp"], floor=spec["floor"]) as p2:
            for (t, reps, _), s in zip(p2.run(iter(_slices(spec))), per_slice):
                assert [r.host for r in reps] == [int(h) for h in s["kept"]], name
        assert pool2.snapshot_bytes() == pool.snapshot_bytes(), name
        n = len(per_slice)
        rec["n_slices"] = np.array([n])
        for key in ("t", "p", "maintained", "cleared", "bact0", "zp"):
            rec[key] = np.array([s[key] for s in per_slice])
        rec["blocks"] = np.stack([s["blocks"] for s in per_slice])
        rec["snap_sha"] = np.array([s["snap_sha"] for s in per_slice])
        for key in ("live", "g0", "est", "zv", "sat", "kept"):
            lens = np.array([len(s[key]) for s in per_slice], dtype=np.int64)
            rec[key + "_len"] = lens
            rec[key + "_cat"] = (np.concatenate([s[key] for s in per_slice])
                                 if lens.sum() else np.zeros(0))
        rec["final_snapshot"] = np.frombuffer(pool.snapshot_bytes(), dtype=np.uint8) \
            if pool.size <= (1 << 16) else np.zeros(0, dtype=np.uint8)
        np.savez_compressed(os.path.join(OUT, f"pipe_{name}.npz"), **rec)
        print(name, n, "slices", os.path.getsize(os.path.join(OUT, f"pipe_{name}.npz")), "bytes")


def comparators():
    """DR and TS pools (pools.py:301-410) next to AT on the same slices."""
    for name, spec in COMPARATORS.items():
        rec = {}
        reports = {}
        for kind in ("at", "dr", "ts"):
            cfg = est.EstimatorConfig(spec["g"], spec["c"], spec["k"], seed=spec["seed"],
                                      counter_kind=kind, partition=spec["part"])
            pool = cfg.build_pool()
            pipe = Pipeline(pool, cfg, spec["kp"], floor=0.0)
            rows = []
            for t, aips, bips in _slices(spec):
                pipe._scan(aips, bips)
                if len(aips):
                    pipe.hosts.update(aips, t)
                live = pipe.hosts.active(t, spec["kp"])
                if len(live):
                    p = pool.count_inactive(spec["kp"])
                    g0 = est.inactive_virtual_counts(pool, cfg, live, spec["kp"])
                    reps = est.reports_from_counts(cfg, live, g0, p, t, spec["kp"])
                else:
                    p, g0, reps = -1, np.zeros(0, dtype=np.int64), []
                cells = pool.cells.get_range(0, pool.size) if kind != "ts" else pool.cells
                cells_sha = hashlib.sha256(np.asarray(cells, dtype=np.uint64).tobytes()).hexdigest()
                mrep = pool.advance_slice()
                if t % max(1, pool.k) == 0:
                    pipe.hosts.prune(t)
                rows.append(dict(p=p, g0=np.asarray(g0, dtype=np.int64),
                                 est=np.array([r.estimate for r in reps], dtype=np.float64),
                                 maintained=mrep.cells_maintained, cleared=mrep.cells_cleared,
                                 nblocks=len(mrep.blocks), cells_sha=cells_sha))
            pipe.close()
            reports[kind] = [r["est"] for r in rows]
            rec[f"{kind}_p"] = np.array([r["p"] for r in rows])
            rec[f"{kind}_maintained"] = np.array([r["maintained"] for r in rows])
            rec[f"{kind}_cleared"] = np.array([r["cleared"] for r in rows])
            rec[f"{kind}_nblocks"] = np.array([r["nblocks"] for r in rows])
            rec[f"{kind}_cells_sha"] = np.array([r["cells_sha"] for r in rows])
            rec[f"{kind}_g0_cat"] = np.concatenate([r["g0"] for r in rows])
            rec[f"{kind}_est_cat"] = np.concatenate([r["est"] for r in rows])
            final = pool.cells.get_range(0, pool.size) if kind != "ts" else pool.cells
            rec[f"{kind}_final_cells"] = np.asarray(final, dtype=np.uint64)
            rec[f"{kind}_bits"] = np.array([pool.bits_per_counter])
        for a, b in zip(reports["at"], reports["dr"]):
            assert np.array_equal(a, b), name
        for a, b in zip(reports["at"], reports["ts"]):
            assert np.array_equal(a, b), name
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **rec)
        print(name, os.path.getsize(os.path.join(OUT, f"{name}.npz")), "bytes")


def appendix_b():
    """SURVEY.md Appendix B digest: c=20, k=10, g=1024, 25 slices x 100k pairs."""
    cfg = est.EstimatorConfig(g=1024, c=20, k=10, seed=0)
    pool = cfg.build_pool()
    rng = np.random.default_rng(0)
    out = {}
    for t in range(25):
        a = (0x0A000000 + rng.integers(0, 10_000, 100_000)).astype(np.uint64)
        b = rng.integers(1, 2 ** 32, 100_000).astype(np.uint64)
        est.record_pairs(pool, cfg, a, b)
        if t == 24:
            out["p24"] = pool.count_inactive(10)
            out["bact0_24"] = pool.bact0
            hosts = np.unique(a)[:1000]
            reps = est.estimate_hosts(pool, cfg, hosts, 24, 10)
            out["hosts24"] = hosts
            out["est24"] = np.array([r.estimate for r in reps])
            out["zv24"] = np.array([r.z_v for r in reps])
            out["zp24"] = reps[0].z_p
        rep = pool.advance_slice()
    out["bact0_end"] = pool.bact0
    out["last_blocks"] = np.array(rep.blocks)
    out["last_maintained"] = rep.cells_maintained
    out["last_cleared"] = rep.cells_cleared
    snap = pool.snapshot_bytes()
    out["snap_sha"] = hashlib.sha256(snap).hexdigest()
    out["snap_len"] = len(snap)
    np.savez_compressed(os.path.join(OUT, "appendix_b.npz"), **out)


def snapshot_blob():
    """The reference tests' scrambled c=8,k=9 pool (test_pools.py:268-275)."""
    pool = AtPool(8, 9)
    rng = np.random.default_rng(9)
    for _ in range(25):
        pool.set_many(rng.integers(0, 256, size=30).astype(np.uint64))
        pool.advance_slice()
    np.savez_compressed(os.path.join(OUT, "snapshot_c8k9.npz"),
                        blob=np.frombuffer(pool.snapshot_bytes(), dtype=np.uint8),
                        count9=pool.count_inactive(9))


def cli_goldens():
    """The reference CLI on a small generated trace: the trace files and the
    byte-exact CSV that `slidecard estimate` writes (cli.py:102-126)."""
    import contextlib
    import io
    import tempfile

    from slidecard import cli
    d = tempfile.mkdtemp()
    trace_txt, truth = os.path.join(d, "t.csv"), os.path.join(d, "truth.csv")
    assert cli.main(["gen", "--out", trace_txt, "--truth", truth, "--hosts", "40",
                     "--n-min", "20", "--n-max", "400", "--k-prime", "6", "--seed", "1"]) == 0
    trace_bin = os.path.join(d, "t.bin")
    assert cli.main(["gen", "--out", trace_bin, "--truth", truth, "--hosts", "40",
                     "--n-min", "20", "--n-max", "400", "--k-prime", "6", "--seed", "1",
                     "--format", "binary"]) == 0
    out = {}
    runs = {
        "est_floor0": ["estimate", "--trace", trace_bin, "--format", "binary", "--c", "14",
                       "--g", "256", "--k", "6", "--floor", "0", "--workers", "1"],
        "est_default": ["estimate", "--trace", trace_txt, "--c", "16", "--g", "256", "--k", "8",
                        "--k-prime", "5", "--workers", "1"],
        "est_lowdev": ["estimate", "--trace", trace_bin, "--format", "binary", "--c", "12",
                       "--g", "128", "--k", "6", "--partition", "low-dev", "--floor", "10",
                       "--seed", "9", "--slice-us", "500000", "--workers", "1"],
    }
    for name, argv in runs.items():
        path = os.path.join(d, name + ".csv")
        assert cli.main(argv + ["--out", path]) == 0
        out[name] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
    ckpt = os.path.join(d, "pool.atp1")
    assert cli.main(runs["est_floor0"] + ["--out", os.path.join(d, "x.csv"),
                                          "--checkpoint", ckpt]) == 0
    out["checkpoint"] = np.frombuffer(open(ckpt, "rb").read(), dtype=np.uint8)
    bench = os.path.join(d, "bench.csv")
    with contextlib.redirect_stderr(io.StringIO()):
        assert cli.main(["bench", "--trace", trace_bin, "--format", "binary", "--c", "14",
                         "--g", "256", "--k", "6", "--floor", "0", "--workers", "1",
                         "--out", bench]) == 0
    out["bench_cols"] = np.array([[int(x) for x in (line.split(",")[0], line.split(",")[4],
                                                     line.split(",")[5])]
                                  for line in open(bench).read().splitlines()[1:]])
    out["trace_bin"] = np.frombuffer(open(trace_bin, "rb").read(), dtype=np.uint8)
    out["trace_txt"] = np.frombuffer(open(trace_txt, "rb").read(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "cli.npz"), **out)


def cli_compare_goldens():
    """`slidecard compare` (cli.py:167-204) and `estimate --counter dr|ts` on the
    committed golden binary trace (cli.npz:trace_bin)."""
    import tempfile

    from slidecard import cli
    d = tempfile.mkdtemp()
    trace_bin = os.path.join(d, "t.bin")
    with open(trace_bin, "wb") as fh:
        fh.write(np.load(os.path.join(OUT, "cli.npz"))["trace_bin"].tobytes())
    common = ["--trace", trace_bin, "--format", "binary", "--c", "14", "--g", "256", "--k", "6",
              "--workers", "1"]
    runs = {
        "compare_floor0": ["compare"] + common + ["--floor", "0"],
        "compare_default": ["compare"] + common + ["--k-prime", "4"],
        "est_dr": ["estimate"] + common + ["--floor", "0", "--counter", "dr"],
        "est_ts": ["estimate"] + common + ["--floor", "20", "--counter", "ts"],
    }
    out = {}
    for name, argv in runs.items():
        path = os.path.join(d, name + ".csv")
        assert cli.main(argv + ["--out", path]) == 0
        out[name] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "cli_compare.npz"), **out)


ALL = (hash_kats, layouts, estimator_kats, snapshot_blob, appendix_b, pipelines, cli_goldens,
       comparators, cli_compare_goldens)

if __name__ == "__main__":
    # no arguments: everything; else only the named generators (e.g. comparators)
    wanted = sys.argv[1:]
    for fn in ALL:
        if not wanted or fn.__name__ in wanted:
            fn()
    print("numpy", np.__version__)
