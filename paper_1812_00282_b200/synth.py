"""Synthetic traffic for benchmarks and tests, generated on the device.

Two shapes from SURVEY.md §8(d): cfg 2 (uniform hosts, fixed heavy-tailed peer
sets -> ``vate_synth_packets``) and cfg 3 (Zipf(1.1) host popularity plus 64
super-spreaders with random peers -> ``vate_synth_zipf``).  The CDF tables are
fixed point (40 fractional bits) and built here with numpy; the kernels only
do integer searches, so the CPU restatement in oracle/ draws identical packets.
"""

from __future__ import annotations

import numpy as np

from ._lib import check, lib

ZIPF_Q = 40


def _mix64(z: np.ndarray) -> np.ndarray:
    x = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(30)
        x *= np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(27)
        x *= np.uint64(0x94D049BB133111EB)
        x ^= x >> np.uint64(31)
    return x


def _cdf(w: np.ndarray) -> np.ndarray:
    c = np.floor(np.cumsum(w) / w.sum() * float(1 << ZIPF_Q)).astype(np.uint64)
    c[-1] = np.uint64(1 << ZIPF_Q)
    return c


def zipf_cdf(hosts: int, s: float = 1.1) -> np.ndarray:
    return _cdf(1.0 / np.arange(1, hosts + 1, dtype=np.float64) ** s)


def spreader_cdf(n: int = 64, seed: int = 0) -> np.ndarray:
    u = (_mix64(np.arange(n, dtype=np.uint64) ^ np.uint64(seed ^ 0x9E37)) >> np.uint64(11)
         ).astype(np.float64) / 2.0 ** 53
    return _cdf(10.0 ** (4.0 + 2.0 * u))


class ZipfTables:
    """cfg-3 tables resident on the pool's device (torch tensors)."""

    def __init__(self, device: int, hosts: int, nspread: int = 64, seed: int = 0):
        import torch
        self.hosts, self.nspread = hosts, nspread
        self.z = torch.from_numpy(zipf_cdf(hosts).view(np.int64)).to(f"cuda:{device}")
        self.s = torch.from_numpy(spreader_cdf(nspread, seed).view(np.int64)).to(f"cuda:{device}")

    def packets(self, pool, t: int, n: int, base_aip: int, seed: int, out_ptr: int,
                spread_q16: int = 6554) -> None:
        check(lib.vate_synth_zipf(pool.handle, t, n, self.hosts, base_aip, seed,
                                  self.z.data_ptr(), self.s.data_ptr(), self.nspread,
                                  spread_q16, out_ptr))
