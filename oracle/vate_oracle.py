"""CPU oracle for the VATE hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference ``slidecard`` package's
ingest / slice-advance / per-host-estimate path.  It exists so that

* ``tests/`` can check the CUDA path against an independent CPU model,
* ``__graft_entry__.smoke()`` can check one small device run, and
* ``bench.py`` can time a CPU baseline (``cpu_baseline`` / ``--impl reference``).

Nothing in ``paper_1812_00282_b200/`` may import it: the product path is the
CUDA library and fails loudly when that library is missing.

It is deliberately *not* a transcription of the reference classes: cells are
held unpacked (one integer per cell) and packed into the reference's ATP1 byte
format only when a snapshot is taken; block lookup uses ``np.searchsorted`` on
the block start offsets instead of the reference's division formulas.  The
oracle is pinned against golden vectors produced by the reference itself
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``), checked by
``tests/test_oracle_golden.py``.

Every function cites the reference file:line it restates (paths relative to
the reference package root ``pkg/src/slidecard/``).
"""

from __future__ import annotations

import hashlib
import struct
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

U64 = np.uint64
MASK64 = (1 << 64) - 1
PHI = 0x9E3779B97F4A7C15                   # hashing.py:18
SALT_CELL = 0x9D9E26B1D9C4F201             # hashing.py:21
SALT_GROUP = 0x5C5D14FA8A33E96D            # hashing.py:22
MUL1 = 0xBF58476D1CE4E5B9                  # hashing.py:28
MUL2 = 0x94D049BB133111EB                  # hashing.py:29
K_LIMIT = 1 << 15                          # counters.py:27
PARTITION_CODES = {"tail": 0, "low-dev": 1}  # pools.py:27-29, :263
ATP1_MAGIC = b"ATP1"                       # pools.py:31
ATP1_HEADER = struct.Struct("<4sBBHH6x")   # pools.py:32


class OracleConfigError(ValueError):
    """Mirrors ``ConfigError`` (errors.py:9-10) for the oracle's own checks."""


def _unique(x) -> np.ndarray:
    """Sorted distinct values (np.unique's result; sort-based, which is many times
    faster than numpy 2.3's np.unique on large integer arrays)."""
    s = np.sort(np.asarray(x))
    if len(s) < 2:
        return s
    keep = np.empty(len(s), dtype=bool)
    keep[0] = True
    np.not_equal(s[1:], s[:-1], out=keep[1:])
    return s[keep]


# --------------------------------------------------------------------------
# hashing (hashing.py:25-67)
# --------------------------------------------------------------------------

def mix64_scalar(z: int) -> int:
    """splitmix64 finalizer on a Python int (hashing.py:25-30)."""
    z &= MASK64
    z ^= z >> 30
    z = (z * MUL1) & MASK64
    z ^= z >> 27
    z = (z * MUL2) & MASK64
    return z ^ (z >> 31)


def mix64(z: np.ndarray) -> np.ndarray:
    """Vector splitmix64 finalizer with uint64 wraparound (hashing.py:33-40)."""
    x = np.array(z, dtype=U64, copy=True)
    with np.errstate(over="ignore"):
        np.bitwise_xor(x, x >> U64(30), out=x)
        np.multiply(x, U64(MUL1), out=x)
        np.bitwise_xor(x, x >> U64(27), out=x)
        np.multiply(x, U64(MUL2), out=x)
        np.bitwise_xor(x, x >> U64(31), out=x)
    return x


def stream_of(seed: int, salt: int) -> int:
    """Per-family hash stream (hashing.py:43-45)."""
    return mix64_scalar((seed ^ salt) & MASK64)


def slot_of(bips: np.ndarray, g: int, group_stream: int) -> np.ndarray:
    """Virtual slot BH(bip) = mix64(bip*phi + stream) mod g (hashing.py:60-67)."""
    b = np.asarray(bips).astype(U64)
    with np.errstate(over="ignore"):
        h = mix64(b * U64(PHI) + U64(group_stream))
    return h % U64(g)


def cell_of(aips: np.ndarray, slots: np.ndarray, c: int, cell_stream: int) -> np.ndarray:
    """Pool cell H(aip, slot) (hashing.py:48-57).

    The key is ``(aip << 32) | slot`` truncated to 64 bits, so aip bits at or
    above 2**32 do not reach the hash (hashing.py:50).
    """
    a = np.asarray(aips).astype(U64)
    s = np.asarray(slots).astype(U64)
    with np.errstate(over="ignore"):
        key = (a << U64(32)) | s
        h = mix64(key * U64(PHI) + U64(cell_stream))
    return h & U64((1 << c) - 1)


# --------------------------------------------------------------------------
# configuration (estimator.py:32-64, pools.py:57-64)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class OracleConfig:
    """Virtual layout and pool shape (estimator.py:32-64)."""

    g: int
    c: int
    k: int
    seed: int = 0
    partition: str = "tail"

    def __post_init__(self):
        if self.g < 1 or not 1 <= self.c <= 32 or self.g > (1 << self.c):
            raise OracleConfigError("bad g/c")               # estimator.py:43-50
        if not 0 <= self.seed < (1 << 64):
            raise OracleConfigError("seed must fit in 64 bits")  # estimator.py:51-52

    @property
    def cell_stream(self) -> int:
        return stream_of(self.seed, SALT_CELL)               # estimator.py:56-58

    @property
    def group_stream(self) -> int:
        return stream_of(self.seed, SALT_GROUP)              # estimator.py:59-61

    def pair_cells(self, aips, bips) -> np.ndarray:
        """estimator.py:96-99."""
        return cell_of(aips, slot_of(bips, self.g, self.group_stream),
                       self.c, self.cell_stream)

    def host_cells(self, aips) -> np.ndarray:
        """All g cells per host, host-major (estimator.py:107-111)."""
        a = np.asarray(aips).astype(U64)
        hosts = np.repeat(a, self.g)
        slots = np.tile(np.arange(self.g, dtype=U64), len(a))
        return cell_of(hosts, slots, self.c, self.cell_stream)


# --------------------------------------------------------------------------
# the asynchronous-timestamp pool (pools.py:67-298, counters.py:52-127)
# --------------------------------------------------------------------------

def at_width(k: int) -> int:
    """Bits per AT: ceil(log2(2k+1)) (counters.py:52-54)."""
    return (2 * k).bit_length()


def block_starts(c: int, k: int, partition: str) -> np.ndarray:
    """Start offsets of the 2k blocks plus the pool end (pools.py:80-95, :121-136).

    tail:    2k-1 blocks of floor(S/(2k-1)) cells, the remainder in the last.
    low-dev: the first 2k-b' blocks hold floor(S/2k) cells, the rest one more.
    """
    size, nb = 1 << c, 2 * k
    if partition == "tail":
        a = size // (nb - 1)
        if size % (nb - 1) == 0:
            raise OracleConfigError("tail partition leaves the last block empty")
        sizes = [a] * (nb - 1) + [size - a * (nb - 1)]
    elif partition == "low-dev":
        a2, b2 = divmod(size, nb)
        sizes = [a2] * (nb - b2) + [a2 + 1] * b2
    else:
        raise OracleConfigError(f"unknown partition {partition!r}")
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


class OraclePool:
    """2**c ATs in 2k staggered-clock blocks, held unpacked (pools.py:67-100)."""

    def __init__(self, c: int, k: int, partition: str = "tail"):
        if not 1 <= k <= K_LIMIT or c > 32 or c < 1 or (1 << c) < 2 * k:
            raise OracleConfigError("bad pool shape")          # pools.py:57-64
        self.c, self.k, self.partition = c, k, partition
        self.size = 1 << c
        self.nblocks = 2 * k
        self.sentinel = 2 * k
        self.starts = block_starts(c, k, partition)
        self.cells = np.full(self.size, self.sentinel, dtype=np.uint32)
        self.bact0 = 0
        self.hist = None

    def track_histogram(self) -> "OraclePool":
        """Keep the per-block value histogram hist[block, value] (pools.py:98-100)
        so that count_inactive costs O(2k * k') per call instead of a pass over
        the pool (pools.py:195-204).  Updated by set_cells (pools.py:167-174, with
        bincount instead of ufunc.at) and by advance (pools.py:246-248)."""
        nb = self.nblocks
        self.hist = np.zeros((nb, nb + 1), dtype=np.int64)
        for b in range(nb):
            lo, hi = self.block_range(b)
            self.hist[b] = np.bincount(self.cells[lo:hi], minlength=nb + 1)
        return self

    # layout --------------------------------------------------------------
    def block_of(self, idx) -> np.ndarray:
        """Block owning each cell (pools.py:104-119), via searchsorted."""
        i = np.asarray(idx).astype(np.int64)
        return np.searchsorted(self.starts, i, side="right") - 1

    def block_range(self, bi: int):
        return int(self.starts[bi]), int(self.starts[bi + 1])

    def block_sizes(self):
        return list(np.diff(self.starts).astype(int))

    def clock(self, blocks) -> np.ndarray:
        """Block clock (bact0 + block) mod 2k (pools.py:146-149)."""
        return (np.asarray(blocks, dtype=np.int64) + self.bact0) % self.nblocks

    def cell_clocks(self) -> np.ndarray:
        return np.repeat(self.clock(np.arange(self.nblocks)), np.diff(self.starts))

    # ingest -----------------------------------------------------------------
    def set_cells(self, idx) -> None:
        """Each cell takes its block's clock; duplicates are fine (pools.py:153-178)."""
        i = np.asarray(idx).astype(np.int64)
        if i.size and (i.min() < 0 or i.max() >= self.size):
            raise ValueError("cell index out of range")         # pools.py:106-107
        if self.hist is not None:                              # pools.py:167-174
            i = _unique(i)
            blocks = self.block_of(i)
            new = self.clock(blocks)
            rows = blocks * (self.nblocks + 1)
            nbins = self.nblocks * (self.nblocks + 1)
            flat = self.hist.reshape(-1)
            flat -= np.bincount(rows + self.cells[i], minlength=nbins)
            flat += np.bincount(rows + new, minlength=nbins)
            self.cells[i] = new.astype(np.uint32)
            return
        self.cells[i] = self.clock(self.block_of(i)).astype(np.uint32)

    # queries ----------------------------------------------------------------
    def _check_width(self, k_prime: int) -> None:
        if not 1 <= k_prime <= self.k:
            raise ValueError(f"k'={k_prime} outside [1, {self.k}]")  # pools.py:215-217

    @staticmethod
    def _inactive(values, clocks, nb, sentinel, k_prime):
        """Sentinel, or distance (clock - value) mod 2k at least k' (pools.py:187-193)."""
        v = values.astype(np.int64)
        dist = (clocks - v) % nb
        return (v == sentinel) | (dist >= k_prime)

    def inactive_mask(self, idx, k_prime: int) -> np.ndarray:
        self._check_width(k_prime)
        i = np.asarray(idx).astype(np.int64)
        return self._inactive(self.cells[i], self.clock(self.block_of(i)),
                              self.nblocks, self.sentinel, k_prime)

    def inactive_bits(self, k_prime: int) -> np.ndarray:
        """Whole-pool inactive predicate, one bool per cell (block by block)."""
        self._check_width(k_prime)
        out = np.empty(self.size, dtype=bool)
        for b, act in enumerate(self.clock(np.arange(self.nblocks)).tolist()):
            lo, hi = self.block_range(b)
            out[lo:hi] = self._inactive(self.cells[lo:hi], act, self.nblocks,
                                        self.sentinel, k_prime)
        return out

    def count_inactive(self, k_prime: int) -> int:
        """Pool-wide inactive count P (pools.py:195-210): from the histogram when
        tracked (pools.py:198-204), else by a full pass."""
        self._check_width(k_prime)
        if self.hist is not None:
            acts = self.clock(np.arange(self.nblocks))
            recent = (acts[:, None] - np.arange(k_prime)[None, :]) % self.nblocks
            rows = np.arange(self.nblocks)[:, None]
            return self.size - int(self.hist[rows, recent].sum())
        total = 0
        for b, act in enumerate(self.clock(np.arange(self.nblocks)).tolist()):
            lo, hi = self.block_range(b)
            total += int(self._inactive(self.cells[lo:hi], act, self.nblocks,
                                        self.sentinel, k_prime).sum())
        return total

    # maintenance ------------------------------------------------------------
    def advance(self):
        """Advance clocks one slice, refresh the two due blocks (pools.py:221-249).

        Returns ((block at clock 0, block at clock k), visited, cleared).
        """
        self.bact0 = (self.bact0 + 1) % self.nblocks
        k, nb = self.k, self.nblocks
        due = ((-self.bact0) % nb, (k - self.bact0) % nb)
        visited = cleared = 0
        for which, bi in enumerate(due):
            lo, hi = self.block_range(bi)
            v = self.cells[lo:hi]
            if which == 0:     # clock 0: values 0..k are stale (counters.py:120-122)
                stale = v <= k
            else:              # clock k: values k..2k-1 and 0 are stale (counters.py:123-125)
                stale = ((v >= k) & (v < 2 * k)) | (v == 0)
            cleared += int(stale.sum())
            visited += hi - lo
            v[stale] = self.sentinel
            if self.hist is not None:                          # pools.py:246-248
                self.hist[bi] = np.bincount(v, minlength=nb + 1)
        return due, visited, cleared

    # snapshots --------------------------------------------------------------
    def payload_words(self) -> int:
        return -(-self.size * at_width(self.k) // 64)

    def snapshot_bytes(self) -> bytes:
        """ATP1 bytes: header + LSB-first packed cells (pools.py:261-265, bitpack.py:26-56)."""
        header = ATP1_HEADER.pack(ATP1_MAGIC, self.c, PARTITION_CODES[self.partition],
                                  self.k, self.bact0)
        return header + pack_cells(self.cells, at_width(self.k))

    @classmethod
    def from_snapshot(cls, blob: bytes) -> "OraclePool":
        """pools.py:271-298 (validation and payload restore)."""
        if len(blob) < ATP1_HEADER.size:
            raise OracleConfigError("truncated snapshot")
        magic, c, part, k, bact0 = ATP1_HEADER.unpack_from(blob)
        if magic != ATP1_MAGIC:
            raise OracleConfigError("not a pool snapshot")
        names = {v: n for n, v in PARTITION_CODES.items()}
        if part not in names:
            raise OracleConfigError("unknown partition code")
        pool = cls(c, k, names[part])
        if bact0 >= pool.nblocks:
            raise OracleConfigError("snapshot clock out of range")
        payload = blob[ATP1_HEADER.size:]
        if len(payload) != 8 * pool.payload_words():
            raise OracleConfigError("bad payload length")
        pool.cells[:] = unpack_cells(payload, at_width(k), pool.size)
        pool.bact0 = bact0
        return pool


class OracleDrPool:
    """2**c distance recorders (pools.py:301-353): fill k, set -> 0, every
    recorder slides by one per slice saturating at k; inactive iff v >= k'."""

    kind = "dr"

    def __init__(self, c: int, k: int):
        if not 1 <= k <= K_LIMIT or c > 32 or c < 1 or (1 << c) < 2 * k:
            raise OracleConfigError("bad pool shape")          # pools.py:57-64
        self.c, self.k, self.size = c, k, 1 << c
        self.cells = np.full(self.size, k, dtype=np.int64)      # pools.py:311

    def set_cells(self, idx) -> None:
        i = np.asarray(idx).astype(np.int64)
        if i.size and (i.min() < 0 or i.max() >= self.size):
            raise ValueError("cell index out of range")
        self.cells[i] = 0                                       # pools.py:314-315

    def _check_width(self, k_prime: int) -> None:
        if not 1 <= k_prime <= self.k:
            raise ValueError(f"k'={k_prime} outside [1, {self.k}]")

    def inactive_mask(self, idx, k_prime: int) -> np.ndarray:
        self._check_width(k_prime)
        return self.cells[np.asarray(idx).astype(np.int64)] >= k_prime   # pools.py:326-329

    def inactive_bits(self, k_prime: int) -> np.ndarray:
        self._check_width(k_prime)
        return self.cells >= k_prime

    def count_inactive(self, k_prime: int) -> int:
        return int(self.inactive_bits(k_prime).sum())           # pools.py:331-337

    def advance(self):
        """pools.py:339-349: ((), every cell visited, cells reaching k)."""
        slid = np.minimum(self.cells + 1, self.k)
        cleared = int(((self.cells < self.k) & (slid == self.k)).sum())
        self.cells = slid
        return (), self.size, cleared


class OracleTsPool:
    """2**c last-seen slice indices (pools.py:356-410): u64, TS_UNSET when never
    set, set -> the pool's slice index t, advance -> t += 1 with no maintenance;
    inactive iff unset or t - last >= k' (u64 arithmetic)."""

    kind = "ts"
    UNSET = MASK64                                              # counters.py:159

    def __init__(self, c: int, k: int):
        if not 1 <= k <= K_LIMIT or c > 32 or c < 1 or (1 << c) < 2 * k:
            raise OracleConfigError("bad pool shape")
        self.c, self.k, self.size = c, k, 1 << c
        self.cells = np.full(self.size, self.UNSET, dtype=U64)
        self.t = 0

    def set_cells(self, idx) -> None:
        i = np.asarray(idx).astype(np.int64)
        if i.size and (i.min() < 0 or i.max() >= self.size):
            raise ValueError("cell index out of range")
        self.cells[i] = U64(self.t)                             # pools.py:363-364

    def _check_width(self, k_prime: int) -> None:
        if not 1 <= k_prime <= self.k:
            raise ValueError(f"k'={k_prime} outside [1, {self.k}]")

    def _inactive(self, last, k_prime):
        with np.errstate(over="ignore"):
            age = U64(self.t) - last                            # wraps for UNSET
        return (last == U64(self.UNSET)) | (age >= U64(k_prime))   # pools.py:375-380

    def inactive_mask(self, idx, k_prime: int) -> np.ndarray:
        self._check_width(k_prime)
        return self._inactive(self.cells[np.asarray(idx).astype(np.int64)], k_prime)

    def inactive_bits(self, k_prime: int) -> np.ndarray:
        self._check_width(k_prime)
        return self._inactive(self.cells, k_prime)

    def count_inactive(self, k_prime: int) -> int:
        return int(self.inactive_bits(k_prime).sum())

    def advance(self):
        self.t += 1                                             # pools.py:399-401
        return (), 0, 0


def make_oracle_pool(kind: str, c: int, k: int, partition: str = "tail"):
    """make_pool (pools.py:413-421) for the oracle's pool kinds."""
    if kind == "at":
        return OraclePool(c, k, partition)
    if kind == "dr":
        return OracleDrPool(c, k)
    if kind == "ts":
        return OracleTsPool(c, k)
    raise OracleConfigError(f"unknown counter kind {kind!r}")


def pack_cells(cells: np.ndarray, width: int) -> bytes:
    """w-bit cells, LSB-first, into little-endian u64 words, zero pad (bitpack.py:26-78).

    Works in chunks of 2^20 cells (a whole number of u64 words) to bound memory.
    """
    n = len(cells)
    nwords = -(-n * width // 64)
    out = np.zeros(nwords * 8, dtype=np.uint8)
    chunk = 1 << 20
    shifts = np.arange(width, dtype=np.uint32)
    for lo in range(0, n, chunk):
        part = cells[lo:lo + chunk].astype(np.uint32)
        bits = ((part[:, None] >> shifts) & np.uint32(1)).astype(np.uint8).reshape(-1)
        packed = np.packbits(bits, bitorder="little")
        start = lo * width // 8
        out[start:start + len(packed)] = packed
    return out.tobytes()


def unpack_cells(payload: bytes, width: int, n: int) -> np.ndarray:
    bits = np.unpackbits(np.frombuffer(payload, dtype=np.uint8), bitorder="little")
    bits = bits[: n * width].reshape(n, width).astype(np.uint32)
    return (bits << np.arange(width, dtype=np.uint32)).sum(axis=1).astype(np.uint32)


# --------------------------------------------------------------------------
# estimator (estimator.py:114-181)
# --------------------------------------------------------------------------

CELL_BUDGET = 1 << 20   # hosts x g cells per work chunk (estimator.py:29, pipeline.py:27)


def host_g0(pool: OraclePool, cfg: OracleConfig, aips, k_prime: int) -> np.ndarray:
    """Per-host inactive virtual-slot count g0 (estimator.py:114-123)."""
    a = np.asarray(aips).astype(U64)
    out = np.empty(len(a), dtype=np.int64)
    step = max(1, CELL_BUDGET // cfg.g)
    for lo in range(0, len(a), step):
        chunk = a[lo:lo + step]
        mask = pool.inactive_mask(cfg.host_cells(chunk), k_prime)
        out[lo:lo + step] = mask.reshape(len(chunk), cfg.g).sum(axis=1)
    return out


@dataclass
class SoaReports:
    """Structure-of-arrays form of a list of EstimateReport (estimator.py:67-81)."""

    host: np.ndarray          # uint64
    estimate: np.ndarray      # float64
    z_v: np.ndarray           # float64
    saturated: np.ndarray     # bool
    z_p: float
    window_start: int
    k_prime: int

    def __len__(self):
        return len(self.host)

    def select(self, keep) -> "SoaReports":
        return SoaReports(self.host[keep], self.estimate[keep], self.z_v[keep],
                          self.saturated[keep], self.z_p, self.window_start,
                          self.k_prime)

    def digest(self) -> str:
        h = hashlib.sha256()
        for arr in (self.host.astype("<u8"), self.estimate.astype("<f8"),
                    self.z_v.astype("<f8"), self.saturated.astype(np.uint8)):
            h.update(arr.tobytes())
        h.update(struct.pack("<dqq", self.z_p, self.window_start, self.k_prime))
        return h.hexdigest()


def reports_soa(cfg: OracleConfig, aips, g0, pool_inactive: int,
                slice_end: int, k_prime: int) -> SoaReports:
    """Integer counts -> estimates; the reference's float expression (estimator.py:138-162)."""
    g = cfg.g
    size = 1 << cfg.c
    g0 = np.asarray(g0, dtype=np.int64)
    zv = g0 / np.float64(g)
    zp = pool_inactive / np.float64(size)
    zv_c = np.where(g0 == 0, 1.0 / (2 * g), zv)
    zp_c = 1.0 / (2 * size) if pool_inactive == 0 else zp
    raw = g * (np.log(zp_c) - np.log(zv_c))
    sat = (g0 == 0) | (raw < 0) | (pool_inactive == 0)
    return SoaReports(np.asarray(aips).astype(U64), np.maximum(raw, 0.0), zv,
                      sat, float(zp), slice_end - k_prime + 1, k_prime)


def estimate_soa(pool: OraclePool, cfg: OracleConfig, aips, slice_end: int,
                 k_prime: int, pool_inactive=None) -> SoaReports:
    """estimator.py:165-174."""
    if pool_inactive is None:
        pool_inactive = pool.count_inactive(k_prime)
    g0 = host_g0(pool, cfg, aips, k_prime)
    return reports_soa(cfg, aips, g0, pool_inactive, slice_end, k_prime)


# --------------------------------------------------------------------------
# slice driver (pipeline.py:43-166)
# --------------------------------------------------------------------------

class OracleHosts:
    """Last-seen slice per host (pipeline.py:43-64)."""

    def __init__(self, k: int):
        self.k = k
        self.last: dict = {}

    def update(self, aips, t: int) -> None:
        for a in _unique(np.asarray(aips).astype(U64)).tolist():
            self.last[a] = t

    def active(self, t: int, k_prime: int) -> np.ndarray:
        cut = t - k_prime
        return np.array(sorted(a for a, s in self.last.items() if s > cut), dtype=U64)

    def prune(self, t: int) -> None:
        cut = t - self.k
        for a in [a for a, s in self.last.items() if s <= cut]:
            del self.last[a]


class OracleHostsVec:
    """OracleHosts (pipeline.py:43-64) as two sorted arrays (keys, last seen):
    the same semantics at a million hosts without a per-slice Python sort."""

    def __init__(self, k: int):
        self.k = k
        self.keys = np.empty(0, dtype=U64)
        self.last = np.empty(0, dtype=np.int64)

    def update(self, aips, t: int) -> None:
        u = _unique(np.asarray(aips).astype(U64))
        pos = np.searchsorted(self.keys, u)
        hit = pos < len(self.keys)
        hit[hit] = self.keys[pos[hit]] == u[hit]
        self.last[pos[hit]] = t
        new = u[~hit]
        if len(new):
            at = np.searchsorted(self.keys, new)
            self.keys = np.insert(self.keys, at, new)
            self.last = np.insert(self.last, at, t)

    def __len__(self):
        return len(self.keys)

    def active(self, t: int, k_prime: int) -> np.ndarray:
        return self.keys[self.last > t - k_prime]                # pipeline.py:54-58

    def prune(self, t: int) -> None:
        keep = self.last > t - self.k                            # pipeline.py:59-64
        self.keys, self.last = self.keys[keep], self.last[keep]


@dataclass
class OracleSlice:
    """Everything one slice produced, for comparison."""

    t: int
    reports: SoaReports | None
    pool_inactive: int | None
    g0: np.ndarray | None
    due: tuple
    visited: int
    cleared: int


class OraclePipeline:
    """scan -> estimate -> advance -> prune, per slice (pipeline.py:142-160).

    ``workers`` fans hashing and gathers out over threads the way the reference
    pipeline does (pipeline.py:102-138); results do not depend on it.
    """

    SCAN_CHUNK = 1 << 15   # pipeline.py:26

    def __init__(self, cfg: OracleConfig, k_prime: int, floor: float = 0.0,
                 workers: int = 1, kind: str = "at"):
        if not 1 <= k_prime <= cfg.k:
            raise ValueError(f"k'={k_prime} outside [1, {cfg.k}]")
        self.cfg = cfg
        self.pool = make_oracle_pool(kind, cfg.c, cfg.k, cfg.partition)
        self.hosts = OracleHosts(cfg.k)
        self.k_prime = k_prime
        self.floor = floor
        self.workers = workers
        self._ex = ThreadPoolExecutor(workers) if workers > 1 else None

    def close(self):
        if self._ex is not None:
            self._ex.shutdown()
            self._ex = None

    def scan(self, aips, bips) -> None:
        n = len(aips)
        spans = [(lo, min(lo + self.SCAN_CHUNK, n)) for lo in range(0, n, self.SCAN_CHUNK)]
        if self._ex is None:
            for lo, hi in spans:
                self.pool.set_cells(self.cfg.pair_cells(aips[lo:hi], bips[lo:hi]))
        else:
            futs = [self._ex.submit(self.cfg.pair_cells, aips[lo:hi], bips[lo:hi])
                    for lo, hi in spans]
            for f in futs:
                self.pool.set_cells(f.result())

    def g0(self, aips) -> np.ndarray:
        step = max(1, CELL_BUDGET // self.cfg.g)
        if self._ex is None or len(aips) <= step:
            return host_g0(self.pool, self.cfg, aips, self.k_prime)
        futs = [self._ex.submit(host_g0, self.pool, self.cfg, aips[lo:lo + step],
                                self.k_prime) for lo in range(0, len(aips), step)]
        return np.concatenate([f.result() for f in futs])

    def estimate(self, t: int):
        aips = self.hosts.active(t, self.k_prime)
        if len(aips) == 0:
            return None, None, None
        p = self.pool.count_inactive(self.k_prime)
        g0 = self.g0(aips)
        rep = reports_soa(self.cfg, aips, g0, p, t, self.k_prime)
        if self.floor > 0:
            rep = rep.select(rep.estimate >= self.floor)
        return rep, p, g0

    def process_slice(self, t: int, aips, bips) -> OracleSlice:
        aips = np.asarray(aips).astype(U64)
        bips = np.asarray(bips).astype(U64)
        self.scan(aips, bips)
        if len(aips):
            self.hosts.update(aips, t)
        rep, p, g0 = self.estimate(t)
        due, visited, cleared = self.pool.advance()
        if t % max(1, self.cfg.k) == 0:
            self.hosts.prune(t)
        return OracleSlice(t, rep, p, g0, due, visited, cleared)


# --------------------------------------------------------------------------
# synthetic traffic shared by bench.py (CPU arm) and the tests
# --------------------------------------------------------------------------

def synthetic_slice(t: int, n: int, hosts: int, base_aip: int = 0x0A000000,
                    trace_seed: int = 0):
    """Deterministic packets of slice ``t`` (SURVEY.md §8(d) cfg 2 shape).

    Integer-only so the CUDA generator (``csrc/vate_synth.cu``) reproduces it
    bit for bit.  Packet i of slice t draws x = mix64(stream + (t*2^32+i)*phi);
    its host rank is x mod hosts (aip = base_aip + rank) and its peer is one of
    that host's fixed peer set.  The set size is 1 + (r mod 8) + 2^min(lz, 12),
    with r a 24-bit per-host hash and lz its leading-zero count: heavy-tailed,
    mean about 11.5, at most 4104.  Bounding the distinct pairs per window keeps
    the pool load away from saturation (SURVEY.md §7 hard part 8).
    """
    stream = stream_of(trace_seed, SYNTH_SALT)
    i = np.arange(n, dtype=U64) + U64((t & 0xFFFFFFFF) << 32)
    with np.errstate(over="ignore"):
        x = mix64(U64(stream) + i * U64(PHI))
    rank = x % U64(hosts)
    r = mix64(rank ^ U64(SYNTH_HOST_SALT)) >> U64(40)          # 24 bits
    _, e = np.frexp(r.astype(np.float64))                      # bit_length, exact < 2^53
    lz = np.minimum(24 - e.astype(np.int64), 12)
    npeers = (U64(1) + (r & U64(7)) + (U64(1) << lz.astype(U64)))
    j = (x >> U64(32)) % npeers
    with np.errstate(over="ignore"):
        bip = mix64((rank << U64(20)) ^ j ^ U64(SYNTH_PEER_SALT)) & U64(0xFFFFFFFF)
    aip = (rank + U64(base_aip)) & U64(0xFFFFFFFF)
    return aip, bip


SYNTH_SALT = 0x51ED270B27C4DF1D
SYNTH_HOST_SALT = 0xA5A5A5A5A5A5A5A5
SYNTH_PEER_SALT = 0x3C6EF372FE94F82B


# --- cfg 3: Zipf host popularity + super-spreaders (SURVEY.md §8(d) cfg 3) -----------

ZIPF_Q = 40                            # CDF tables are fixed point with 40 fractional bits
SPREAD_BASE = 0x0B000000
SPREAD_BIP_SALT = 0x6A09E667F3BCC909
SPREAD_PEER_SALT = 0xBB67AE8584CAA73B


def zipf_cdf(hosts: int, s: float = 1.1) -> np.ndarray:
    """Upper-bound table: rank i is drawn for u in [cdf[i-1], cdf[i])."""
    w = 1.0 / np.arange(1, hosts + 1, dtype=np.float64) ** s
    c = np.floor(np.cumsum(w) / w.sum() * float(1 << ZIPF_Q)).astype(np.uint64)
    c[-1] = np.uint64(1 << ZIPF_Q)
    return c


def spreader_cdf(n: int = 64, seed: int = 0) -> np.ndarray:
    """Traffic share per spreader proportional to a log-uniform cardinality in [1e4, 1e6]."""
    u = (mix64(np.arange(n, dtype=U64) ^ U64(seed ^ 0x9E37)) >> U64(11)).astype(np.float64) / 2.0 ** 53
    w = 10.0 ** (4.0 + 2.0 * u)
    c = np.floor(np.cumsum(w) / w.sum() * float(1 << ZIPF_Q)).astype(np.uint64)
    c[-1] = np.uint64(1 << ZIPF_Q)
    return c


def synthetic_zipf_slice(t: int, n: int, hosts: int, zcdf: np.ndarray, scdf: np.ndarray,
                         spread_q16: int = 6554, base_aip: int = 0x0A000000, trace_seed: int = 0):
    """Packets of slice t for cfg 3; integer-only, equal to csrc k_synth_zipf.

    A packet is a spreader packet when the low 16 bits of its draw are below
    spread_q16 (6554/65536 ~ 10%): spreader s ~ scdf, random 32-bit peer.  Else
    a regular host rank ~ zcdf (Zipf s = 1.1) with the cfg-2 fixed peer sets.
    """
    stream = stream_of(trace_seed, SYNTH_SALT)
    i = np.arange(n, dtype=U64) + U64((t & 0xFFFFFFFF) << 32)
    with np.errstate(over="ignore"):
        x = mix64(U64(stream) + i * U64(PHI))
    u = x >> U64(24)
    spread = (x & U64(0xFFFF)) < U64(spread_q16)
    s_idx = np.searchsorted(scdf, u, side="right").astype(U64)
    rank = np.searchsorted(zcdf, u, side="right").astype(U64)
    r = mix64(rank ^ U64(SYNTH_HOST_SALT)) >> U64(40)
    _, e = np.frexp(r.astype(np.float64))
    lz = np.minimum(24 - e.astype(np.int64), 12)
    npeers = U64(1) + (r & U64(7)) + (U64(1) << lz.astype(U64))
    y = mix64(x ^ U64(SPREAD_PEER_SALT))
    j = (y >> U64(32)) % npeers
    with np.errstate(over="ignore"):
        bip_reg = mix64((rank << U64(20)) ^ j ^ U64(SYNTH_PEER_SALT)) & U64(0xFFFFFFFF)
    bip_spr = mix64(x ^ U64(SPREAD_BIP_SALT)) & U64(0xFFFFFFFF)
    aip = np.where(spread, U64(SPREAD_BASE) + s_idx, (rank + U64(base_aip)) & U64(0xFFFFFFFF))
    bip = np.where(spread, bip_spr, bip_reg)
    return aip.astype(U64), bip.astype(U64)
