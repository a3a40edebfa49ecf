"""Loaders for the committed golden vectors (made by tests/golden/make_golden.py)."""

import os

import numpy as np

from specs import PIPELINES, gen_slices

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def _split(rec, key):
    lens = rec[key + "_len"]
    cat = rec[key + "_cat"]
    out, pos = [], 0
    for n in lens:
        out.append(cat[pos:pos + n])
        pos += n
    return out


class PipeCase:
    """One recorded reference pipeline run, slice by slice."""

    def __init__(self, name):
        self.name = name
        self.spec = PIPELINES[name]
        rec = load(f"pipe_{name}.npz")
        self.n = int(rec["n_slices"][0])
        for key in ("t", "p", "maintained", "cleared", "bact0", "zp", "blocks", "snap_sha"):
            setattr(self, key, rec[key])
        self.live = [a.astype(np.uint64) for a in _split(rec, "live")]
        self.g0 = [a.astype(np.int64) for a in _split(rec, "g0")]
        self.est = [a.astype(np.float64) for a in _split(rec, "est")]
        self.zv = [a.astype(np.float64) for a in _split(rec, "zv")]
        self.sat = [a.astype(bool) for a in _split(rec, "sat")]
        self.kept = [a.astype(np.uint64) for a in _split(rec, "kept")]
        self.final_snapshot = rec["final_snapshot"].tobytes()

    def slices(self):
        return gen_slices(self.spec)


PIPE_NAMES = sorted(PIPELINES)


from specs import COMPARATORS  # noqa: E402

CMP_NAMES = sorted(COMPARATORS)
CMP_KINDS = ("at", "dr", "ts")


def replay_kind(spec, kind, pool, scan, live_at, g0_of, p_of, reports_of, advance, cells_of):
    """Replay a comparator golden case through any pool implementation.

    Returns the recorded fields in make_golden.comparators() order so the
    caller compares them with the reference's npz.
    """
    import hashlib
    out = {"p": [], "maintained": [], "cleared": [], "nblocks": [], "cells_sha": [],
           "g0": [], "est": []}
    for t, aips, bips in gen_slices(spec):
        scan(t, aips, bips)
        live = live_at(t)
        if len(live):
            p = p_of()
            g0 = np.asarray(g0_of(live), dtype=np.int64)
            est = np.asarray(reports_of(t, live, g0, p), dtype=np.float64)
        else:
            p, g0, est = -1, np.zeros(0, np.int64), np.zeros(0)
        out["cells_sha"].append(hashlib.sha256(
            np.asarray(cells_of(), dtype=np.uint64).tobytes()).hexdigest())
        blocks, maintained, cleared = advance(t)
        out["p"].append(p)
        out["g0"].append(g0)
        out["est"].append(est)
        out["maintained"].append(maintained)
        out["cleared"].append(cleared)
        out["nblocks"].append(len(blocks))
    return out


def check_replay(name, kind, got):
    rec = load(f"{name}.npz")
    for key in ("p", "maintained", "cleared", "nblocks"):
        assert np.array_equal(np.array(got[key]), rec[f"{kind}_{key}"]), (name, kind, key)
    assert list(got["cells_sha"]) == [str(x) for x in rec[f"{kind}_cells_sha"]], (name, kind)
    assert np.array_equal(np.concatenate(got["g0"]), rec[f"{kind}_g0_cat"]), (name, kind)
    assert np.array_equal(np.concatenate(got["est"]), rec[f"{kind}_est_cat"]), (name, kind)
