"""Pipeline golden-case specs and their seeded slice generator.

Shared by ``make_golden.py`` (which runs the reference on them) and the tests
(which regenerate the same slices to feed the oracle and the CUDA path).
"""

import numpy as np


def gen_slices(spec):
    rng = np.random.default_rng(spec["data_seed"])
    out = []
    for t in range(spec["slices"]):
        n = spec["pairs"]
        if t in spec.get("empty", ()):
            n = 0
        aips = rng.integers(0, spec["hosts"], size=n).astype(np.uint64) + np.uint64(spec["aip_base"])
        bips = rng.integers(spec.get("bip_lo", 1), spec.get("bip_hi", 1 << 32), size=n,
                            dtype=np.uint64)
        if spec.get("dup"):
            aips = np.concatenate([aips, aips[: n // 2]])
            bips = np.concatenate([bips, bips[: n // 2]])
        out.append((t + spec.get("t0", 0), aips, bips))
    return out


PIPELINES = {
    # SURVEY cfg 1 shape at reduced host/pair counts, >2k slices so clocks wrap
    "cfg1_small": dict(g=1024, c=20, k=10, seed=0, part="tail", kp=10, floor=0.0,
                       slices=25, pairs=20_000, hosts=2_000, aip_base=0x0A000000,
                       data_seed=0, empty=(7,)),
    "kprime_floor": dict(g=1024, c=18, k=30, seed=7, part="tail", kp=12, floor=40.0,
                         slices=70, pairs=6_000, hosts=600, aip_base=0x0A000000,
                         data_seed=1, dup=True),
    "lowdev_k1": dict(g=64, c=12, k=1, seed=3, part="low-dev", kp=1, floor=0.0,
                      slices=8, pairs=500, hosts=40, aip_base=0, data_seed=2, empty=(3,)),
    "k300_u16": dict(g=256, c=16, k=300, seed=11, part="tail", kp=150, floor=0.0,
                     slices=620, pairs=300, hosts=60, aip_base=0xC0A80000, data_seed=3),
    "wide_k600": dict(g=128, c=14, k=600, seed=5, part="low-dev", kp=600, floor=0.0,
                      slices=60, pairs=200, hosts=30, aip_base=17, data_seed=4, t0=3),
    "g1000_big_keys": dict(g=1000, c=18, k=30, seed=123456789012345, part="low-dev", kp=30,
                           floor=50.0, slices=40, pairs=3_000, hosts=300,
                           aip_base=(1 << 40) + 5, bip_lo=1 << 33, bip_hi=1 << 62,
                           data_seed=5),
    "tiny_pool": dict(g=2, c=3, k=2, seed=1, part="tail", kp=2, floor=0.0,
                      slices=12, pairs=5, hosts=6, aip_base=100, data_seed=6),
    "g_full_pool": dict(g=512, c=9, k=4, seed=9, part="tail", kp=3, floor=0.0,
                        slices=20, pairs=50, hosts=20, aip_base=1, data_seed=7),
}


# Comparator pools (DR / TS, pools.py:301-410) replayed next to AT on the same
# slices: per-kind cells, P, g0, reports and maintenance; estimates must agree
# across kinds (test_estimator.py:233-255).
COMPARATORS = {
    "cmp_k6": dict(g=256, c=14, k=6, seed=4, part="tail", kp=5, floor=0.0, slices=16,
                   pairs=4_000, hosts=300, aip_base=0x0A000000, data_seed=8, empty=(5,)),
    # k = 300: dr_bits = 9 -> 16-bit DR cells on the device
    "cmp_k300_u16": dict(g=128, c=12, k=300, seed=2, part="low-dev", kp=200, floor=0.0,
                         slices=40, pairs=300, hosts=40, aip_base=0x0A000000, data_seed=9),
}
