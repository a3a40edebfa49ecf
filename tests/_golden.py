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
