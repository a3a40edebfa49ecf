"""Per-host estimation over the device pool (reference: estimator.py).

Same names, arguments, results and errors as the reference module; the pool
cells, the hashing, the g0 gathers and the float path all run on the GPU.

The float path reproduces the reference's numpy expression bit for bit
(estimator.py:146-155).  Its only transcendental inputs -- np.log of the
clamped virtual fraction for each possible g0 (g+1 values, once per g) and
np.log of the clamped pool fraction (one value per estimate) -- are taken with
numpy on the host, exactly as the reference computes them; the device applies
them per host with single IEEE-rounded subtract / multiply / divide.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np

from . import hashing
from ._lib import VATE_DEVICE, VATE_HOST, check, lib, ptr
from .errors import ConfigError
from .pools import TAIL_REMAINDER, AtPool, _DevicePool, make_pool

COUNTER_KINDS = ("at", "dr", "ts")


@dataclass(frozen=True)
class EstimatorConfig:
    """Virtual layout: g slots per host over a pool of 2**c counters (estimator.py:32-64)."""

    g: int
    c: int
    k: int
    seed: int = 0
    counter_kind: str = "at"
    partition: str = TAIL_REMAINDER

    def __post_init__(self):
        if self.g < 1:
            raise ConfigError(f"g must be at least 1, got {self.g}")
        if self.c < 1 or self.c > 32:
            raise ConfigError(f"c must be in [1, 32], got {self.c}")
        if self.g > (1 << self.c):
            raise ConfigError(f"g={self.g} exceeds the pool size 2^{self.c}")
        if not 0 <= self.seed < (1 << 64):
            raise ConfigError("seed must fit in 64 bits")
        if self.counter_kind not in COUNTER_KINDS:
            raise ConfigError(f"unknown counter kind {self.counter_kind!r}")
        object.__setattr__(self, "cell_stream",
                           hashing.derive_stream(self.seed, hashing.CELL_SALT))
        object.__setattr__(self, "group_stream",
                           hashing.derive_stream(self.seed, hashing.GROUP_SALT))

    def build_pool(self, device: int = 0):
        return make_pool(self.counter_kind, self.c, self.k, self.partition, device=device)


@dataclass(frozen=True)
class EstimateReport:
    """One host's estimate for the window of k' slices ending now (estimator.py:67-81)."""

    host: int
    window_start: int
    k_prime: int
    estimate: float
    z_v: float
    z_p: float
    saturated: bool

    @property
    def slice_end(self) -> int:
        return self.window_start + self.k_prime - 1


@dataclass
class HostReports:
    """Structure-of-arrays reports: the fast form of list[EstimateReport].

    Materialising 1M EstimateReport objects costs seconds of Python
    (SURVEY.md §7 hard part 6); the arrays are what the device produces.
    """

    host: np.ndarray        # uint64, ascending for pipeline output
    estimate: np.ndarray    # float64
    z_v: np.ndarray         # float64
    saturated: np.ndarray   # bool
    z_p: float
    window_start: int
    k_prime: int

    def __len__(self) -> int:
        return len(self.host)

    def to_list(self):
        return [EstimateReport(int(h), self.window_start, self.k_prime, float(e), float(z),
                               self.z_p, bool(s))
                for h, e, z, s in zip(self.host.tolist(), self.estimate.tolist(),
                                      self.z_v.tolist(), self.saturated.tolist())]


# --- the host-side log inputs of the float path ------------------------------------

_LOG_CACHE: dict = {}


def log_zv_table(g: int) -> np.ndarray:
    """np.log of the clamped virtual fraction for g0 = 0..g (estimator.py:147-150)."""
    tab = _LOG_CACHE.get(g)
    if tab is None:
        g0 = np.arange(g + 1, dtype=np.int64)
        z_v = g0 / np.float64(g)
        tab = np.ascontiguousarray(np.log(np.where(g0 == 0, 1.0 / (2 * g), z_v)))
        _LOG_CACHE[g] = tab
    return tab


def log_zp(pool_inactive: int, pool_size: int):
    """(np.log of the clamped pool fraction, z_p) (estimator.py:148-151)."""
    z_p = pool_inactive / np.float64(pool_size)
    zp_clamped = 1.0 / (2 * pool_size) if pool_inactive == 0 else z_p
    return float(np.log(zp_clamped)), float(z_p)


_LZP_CACHE: dict = {}
LZP_TABLE_MAX_C = 26   # 2^26+1 doubles = 512 MiB; larger pools take log_zp per slice


def log_zp_table(c: int):
    """np.log of the clamped pool fraction for every P in [0, 2^c] (estimator.py:148-151),
    elementwise identical to log_zp(P, 2^c); None above LZP_TABLE_MAX_C."""
    if c > LZP_TABLE_MAX_C:
        return None
    tab = _LZP_CACHE.get(c)
    if tab is None:
        size = 1 << c
        zp = np.arange(size + 1, dtype=np.int64) / np.float64(size)
        zp[0] = 1.0 / (2 * size)
        tab = np.ascontiguousarray(np.log(zp))
        _LZP_CACHE[c] = tab
    return tab


def _ensure_log_table(pool: AtPool, g: int) -> None:
    if getattr(pool, "_lzv_g", None) != g:
        tab = log_zv_table(g)
        check(lib.vate_set_log_table(pool.handle, g, ptr(tab)))
        pool._lzv_g = g


# --- a device context for the pool-less calls -------------------------------------

_CTX: dict = {}
_CTX_LOCK = threading.Lock()


def context_pool(device: int = 0) -> AtPool:
    """A 2-cell pool whose stream serves pool-less calls (pair_cells, ...)."""
    with _CTX_LOCK:
        pool = _CTX.get(device)
        if pool is None:
            pool = AtPool(1, 1, "low-dev", device=device)
            _CTX[device] = pool
        return pool


def _u64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x).astype(np.uint64, copy=False))


def _check_pool_cfg(pool, cfg) -> None:
    if not isinstance(pool, _DevicePool):
        raise TypeError("pool must be a device pool (AtPool, DrPool or TsPool)")
    if pool.c != cfg.c:
        raise ValueError(f"pool has c={pool.c} but the config has c={cfg.c}")


# --- hashing entry points (estimator.py:84-111) ------------------------------------

def virtual_slot(cfg: EstimatorConfig, bip: int) -> int:
    return hashing.group_index(bip, cfg.g, cfg.group_stream)


def cell_of(cfg: EstimatorConfig, aip: int, slot: int) -> int:
    if slot >= cfg.g:
        raise ValueError(f"virtual slot {slot} outside [0, {cfg.g})")
    return hashing.cell_index(aip, slot, cfg.c, cfg.cell_stream)


def pair_cells(cfg: EstimatorConfig, aips, bips, pool: AtPool | None = None) -> np.ndarray:
    """Pool cells touched by a batch of pairs (estimator.py:96-99), hashed on the device."""
    a, b = _u64(aips), _u64(bips)
    if a.shape != b.shape:
        raise ValueError("aips and bips must have the same length")
    out = np.empty(a.size, dtype=np.uint64)
    if a.size:
        ctx = pool if pool is not None else context_pool()
        check(lib.vate_pair_cells(ctx.handle, cfg.g, cfg.c, cfg.cell_stream, cfg.group_stream,
                                  ptr(a), ptr(b), a.size, VATE_HOST, ptr(out)))
    return out


def host_cells(cfg: EstimatorConfig, aips, pool: AtPool | None = None) -> np.ndarray:
    """All g cells of each host, host-major (estimator.py:107-111)."""
    a = _u64(aips)
    out = np.empty(a.size * cfg.g, dtype=np.uint64)
    if a.size:
        ctx = pool if pool is not None else context_pool()
        check(lib.vate_host_cells(ctx.handle, cfg.g, cfg.c, cfg.cell_stream, ptr(a), a.size,
                                  VATE_HOST, ptr(out)))
    return out


# --- scan (estimator.py:102-104) ------------------------------------------------------

def record_pairs(pool: AtPool, cfg: EstimatorConfig, aips, bips) -> None:
    """Record a batch of pairs into the pool (scan phase), fused hash + scatter."""
    _check_pool_cfg(pool, cfg)
    a, b = _u64(aips), _u64(bips)
    if a.shape != b.shape:
        raise ValueError("aips and bips must have the same length")
    if a.size:
        check(lib.vate_scan_pairs(pool.handle, cfg.g, cfg.cell_stream, cfg.group_stream,
                                  ptr(a), ptr(b), a.size, VATE_HOST, None, 0))


def record_packed(pool: AtPool, cfg: EstimatorConfig, pairs, n: int | None = None,
                  on_device: bool = False) -> None:
    """Scan packed {u32 aip, u32 bip} records: a uint32 array of shape (n, 2), or a
    device pointer (int) with ``on_device=True``."""
    _check_pool_cfg(pool, cfg)
    if on_device:
        check(lib.vate_scan_packed(pool.handle, cfg.g, cfg.cell_stream, cfg.group_stream,
                                   int(pairs), int(n), VATE_DEVICE, None, 0))
        return
    arr = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1)
    if arr.size:
        check(lib.vate_scan_packed(pool.handle, cfg.g, cfg.cell_stream, cfg.group_stream,
                                   ptr(arr), arr.size // 2, VATE_HOST, None, 0))


# --- estimate (estimator.py:114-181) ------------------------------------------------

def inactive_virtual_counts(pool: AtPool, cfg: EstimatorConfig, aips, k_prime: int) -> np.ndarray:
    """Per-host count of inactive virtual slots g0, as int64 (estimator.py:114-123)."""
    _check_pool_cfg(pool, cfg)
    pool._validate_width(k_prime)
    a = _u64(aips)
    out = np.empty(a.size, dtype=np.int32)
    if a.size:
        check(lib.vate_host_g0(pool.handle, cfg.g, cfg.cell_stream, ptr(a), a.size, k_prime,
                               ptr(out), VATE_HOST))
    return out.astype(np.int64)


def estimate_linear(g: int, g0: int):
    """Plain linear estimate -g*ln(g0/g) (estimator.py:126-135); scalar helper."""
    if not 0 <= g0 <= g:
        raise ValueError(f"g0={g0} outside [0, {g}]")
    saturated = g0 == 0
    clamped = max(g0, 1)
    return float(g * np.log(g / np.float64(clamped))), saturated


def reports_from_counts_soa(cfg: EstimatorConfig, aips, g0, pool_inactive: int,
                            slice_end: int, k_prime: int, pool: AtPool | None = None) -> HostReports:
    """Integer counts -> reports, as arrays, via the device float path."""
    a = _u64(aips)
    g0 = np.ascontiguousarray(np.asarray(g0), dtype=np.int32)
    if g0.shape != a.shape:
        raise ValueError("aips and g0 must have the same length")
    ctx = pool if pool is not None else context_pool()
    _ensure_log_table(ctx, cfg.g)
    lzp, z_p = log_zp(int(pool_inactive), 1 << cfg.c)
    est = np.empty(a.size, dtype=np.float64)
    zv = np.empty(a.size, dtype=np.float64)
    sat = np.empty(a.size, dtype=np.uint8)
    if a.size:
        check(lib.vate_reports_from_counts(ctx.handle, cfg.g, ptr(g0), a.size, int(pool_inactive),
                                           lzp, ptr(est), ptr(zv), ptr(sat)))
    return HostReports(a, est, zv, sat.view(bool), z_p, slice_end - k_prime + 1, k_prime)


def reports_from_counts(cfg: EstimatorConfig, aips, g0, pool_inactive: int,
                        slice_end: int, k_prime: int):
    """list[EstimateReport] in input order (estimator.py:138-162)."""
    return reports_from_counts_soa(cfg, aips, g0, pool_inactive, slice_end, k_prime).to_list()


def estimate_hosts_soa(pool: AtPool, cfg: EstimatorConfig, aips, slice_end: int,
                       k_prime: int, pool_inactive=None) -> HostReports:
    if pool_inactive is None:
        pool_inactive = pool.count_inactive(k_prime)
    g0 = inactive_virtual_counts(pool, cfg, aips, k_prime)
    return reports_from_counts_soa(cfg, aips, g0, pool_inactive, slice_end, k_prime, pool=pool)


def estimate_hosts(pool: AtPool, cfg: EstimatorConfig, aips, slice_end: int, k_prime: int,
                   pool_inactive=None):
    """Estimate every host in ``aips`` (estimator.py:165-174)."""
    return estimate_hosts_soa(pool, cfg, aips, slice_end, k_prime, pool_inactive).to_list()


def estimate_host(pool: AtPool, cfg: EstimatorConfig, aip: int, slice_end: int, k_prime: int,
                  pool_inactive=None) -> EstimateReport:
    """Single-host wrapper (estimator.py:177-181)."""
    return estimate_hosts(pool, cfg, np.array([aip], dtype=np.uint64), slice_end, k_prime,
                          pool_inactive)[0]
