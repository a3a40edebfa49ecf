"""The asynchronous-timestamp pool, resident on a B200 (reference: pools.py).

``AtPool`` keeps the reference's duck-typed pool protocol (pools.py:153-259:
set_many / set_one / check_one / inactive_mask / count_inactive /
inactive_fraction / advance_slice / bits_per_counter / memory_bytes) and the
AtPool extras (layout queries, bact0, snapshot_bytes / save / load), but the
2**c cells live in device memory and every data operation is a CUDA kernel in
libvate_b200.so.  Layout queries (block_of, block_range, ...) are closed-form
integer geometry answered on the host.

The DR and TS comparator pools (pools.py:301-410) run on the device too
(csrc/vate_compare.cu): ``DrPool`` (distance recorders, the VDRE baseline
whose every cell slides every slice) and ``TsPool`` (64-bit last-seen slice
indices).  They share the scan, host registry, g0 gather and float path with
``AtPool``; snapshots and the replica merge are AT-only, as in the reference.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import VATE_DEVICE, VATE_HOST, check, lib, ptr
from .errors import ConfigError

TAIL_REMAINDER = "tail"
LOW_DEVIATION = "low-dev"
PARTITIONS = (TAIL_REMAINDER, LOW_DEVIATION)
MAX_K = 1 << 15
_SNAPSHOT_HEADER = struct.Struct("<4sBBHH6x")   # pools.py:32
_SNAPSHOT_MAGIC = b"ATP1"


@dataclass(frozen=True)
class MaintenanceReport:
    """What one slice advance touched (pools.py:43-54)."""

    blocks: tuple
    cells_maintained: int
    cells_cleared: int


def _validate_pool_shape(c: int, k: int) -> None:
    """pools.py:57-64, same messages."""
    if not 1 <= k <= MAX_K:
        raise ConfigError(f"k must be in [1, {MAX_K}], got {k}")
    if c > 32:
        raise ConfigError(f"c must be at most 32, got {c}")
    if c < 1 or (1 << c) < 2 * k:
        raise ConfigError(
            f"pool of 2^{c} cells cannot hold 2k={2 * k} non-empty blocks")


def maintenance_blocks(b0: int, b1: int) -> tuple:
    """(b0, b1) for the AT pool; () for DR / TS (the library reports -1, -1)."""
    return () if b0 < 0 else (b0, b1)


def _as_u64(idx) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(idx).astype(np.uint64, copy=False))


class BlockLayout:
    """Closed-form geometry of the 2k blocks (pools.py:72-149), no device needed.

    tail: 2k-1 blocks of floor(S/(2k-1)) cells, the remainder in the last;
    low-dev: floor(S/2k) cells per block, the last S mod 2k blocks one more.
    """

    def __init__(self, c: int, k: int, partition: str = TAIL_REMAINDER):
        _validate_pool_shape(c, k)
        if partition not in PARTITIONS:
            raise ConfigError(f"unknown partition method {partition!r}")
        self.c, self.k, self.partition = c, k, partition
        self.size = 1 << c
        self.nblocks = 2 * k
        self.sentinel = 2 * k
        if partition == TAIL_REMAINDER:
            self._a = self.size // (self.nblocks - 1)
            self._b = self.size % (self.nblocks - 1)
            if self._b == 0:
                raise ConfigError(
                    "tail partition leaves the last block empty for "
                    f"c={c}, k={k}; use the {LOW_DEVIATION!r} partition")
        else:
            self._a2 = self.size // self.nblocks
            self._b2 = self.size % self.nblocks
            self._split = self._a2 * (self.nblocks - self._b2 + 1)

    def block_of(self, i: int) -> int:
        if not 0 <= i < self.size:
            raise ValueError(f"cell index {i} outside [0, {self.size})")
        if self.partition == TAIL_REMAINDER:
            return min(i // self._a, self.nblocks - 1)
        if i < self._split:
            return i // self._a2
        return (i + self.nblocks - self._b2) // (self._a2 + 1)

    def block_of_vec(self, idx: np.ndarray) -> np.ndarray:
        idx = np.asarray(idx).astype(np.uint64, copy=False)
        if self.partition == TAIL_REMAINDER:
            return np.minimum(idx // np.uint64(self._a), np.uint64(self.nblocks - 1))
        lead = idx // np.uint64(self._a2)
        tail = (idx + np.uint64(self.nblocks - self._b2)) // np.uint64(self._a2 + 1)
        return np.where(idx < np.uint64(self._split), lead, tail)

    def block_range(self, bi: int):
        if not 0 <= bi < self.nblocks:
            raise ValueError(f"block index {bi} outside [0, {self.nblocks})")
        if self.partition == TAIL_REMAINDER:
            start = bi * self._a
            return start, (self.size if bi == self.nblocks - 1 else start + self._a)
        narrow = self.nblocks - self._b2
        if bi < narrow:
            return bi * self._a2, (bi + 1) * self._a2
        base = narrow * self._a2 + (bi - narrow) * (self._a2 + 1)
        return base, base + self._a2 + 1

    def block_sizes(self):
        return [hi - lo for lo, hi in (self.block_range(b) for b in range(self.nblocks))]

    @property
    def max_block_size(self) -> int:
        if self.partition == TAIL_REMAINDER:
            return max(self._a, self.size - self._a * (self.nblocks - 1))
        return self._a2 + (1 if self._b2 else 0)


class _DevicePool:
    """Handle plumbing and the pool protocol shared by every device pool kind."""

    kind = "at"
    _kind_code = 0

    def _create(self, c: int, k: int, partition: str, device: int) -> None:
        self.device = device
        h = C.c_void_p()
        check(lib.vate_pool_create_kind(C.byref(h), self._kind_code, c, k,
                                        PARTITIONS.index(partition), device))
        self._h = h
        _lib.track(self)

    # --- handle -----------------------------------------------------------------
    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value and not _lib.shutting_down():
            lib.vate_pool_destroy(h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:   # interpreter shutdown
            pass

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def _info(self):
        bact0, cb, stream = C.c_int32(), C.c_int32(), C.c_void_p()
        check(lib.vate_pool_info(self._h, C.byref(bact0), C.byref(cb), C.byref(stream)))
        return bact0.value, cb.value, stream.value

    @property
    def cell_bytes(self) -> int:
        """Device bytes per cell: AT 1 (k <= 127), 2 (k <= 32767) or 4; DR 1 or 2; TS 8."""
        return self._info()[1]

    @property
    def stream(self) -> int:
        """The cudaStream_t all of this pool's kernels run on."""
        return self._info()[2]

    def synchronize(self) -> None:
        check(lib.vate_pool_sync(self._h))

    # --- counter access (device) -------------------------------------------------
    def set_one(self, i: int) -> None:
        if not 0 <= i < self.size:
            raise ValueError(f"cell index {i} outside [0, {self.size})")
        self.set_many(np.array([i], dtype=np.uint64))

    def set_many(self, idx) -> None:
        """Record activity on every cell in ``idx`` (pools.py:164-178, :314, :363)."""
        idx = _as_u64(idx)
        check(lib.vate_set_cells(self._h, ptr(idx), idx.size, VATE_HOST))

    def set_many_device(self, idx_ptr: int, n: int) -> None:
        """set_many on a device array of n uint64 indices (e.g. a torch tensor)."""
        check(lib.vate_set_cells(self._h, idx_ptr, n, VATE_DEVICE))

    def _validate_width(self, k_prime: int) -> None:
        if not 1 <= k_prime <= self.k:
            raise ValueError(f"k'={k_prime} outside [1, {self.k}]")

    def check_one(self, i: int, k_prime: int) -> bool:
        if not 0 <= i < self.size:
            raise ValueError(f"cell index {i} outside [0, {self.size})")
        return not bool(self.inactive_mask(np.array([i], dtype=np.uint64), k_prime)[0])

    def inactive_mask(self, idx, k_prime: int) -> np.ndarray:
        """True where the cell is inactive for width k' (pools.py:187-193, :326, :375)."""
        self._validate_width(k_prime)
        idx = _as_u64(idx)
        out = np.empty(idx.shape, dtype=np.uint8)
        if idx.size:
            check(lib.vate_inactive_mask(self._h, ptr(idx), idx.size, k_prime, ptr(out), VATE_HOST))
        return out.view(bool)

    def count_inactive(self, k_prime: int) -> int:
        """Pool cells inactive for width k' (pools.py:195-210)."""
        self._validate_width(k_prime)
        out = C.c_uint64()
        check(lib.vate_count_inactive(self._h, k_prime, C.byref(out)))
        return out.value

    def inactive_fraction(self, k_prime: int) -> float:
        return self.count_inactive(k_prime) / self.size

    # --- maintenance (pools.py:221-249, :339-349, :399-401) ---------------------------
    def advance_slice(self) -> MaintenanceReport:
        blocks = (C.c_int32 * 2)()
        maint, cleared = C.c_uint64(), C.c_uint64()
        check(lib.vate_advance(self._h, blocks, C.byref(maint), C.byref(cleared)))
        return MaintenanceReport(maintenance_blocks(blocks[0], blocks[1]), maint.value,
                                 cleared.value)

    @property
    def memory_bytes(self) -> int:
        """The reference's accounting of the pool (pools.py:257-259, :355-356,
        :409-410): its packed words (AT: plus the snapshot header)."""
        return self.packed_bytes

    def mode(self) -> dict:
        """The pool's storage mode: deferred scatter, bit-plane mode and its window."""
        out = (C.c_int32 * 5)()
        check(lib.vate_pool_mode(self._h, out))
        return {"deferred": bool(out[0]), "bitplane": bool(out[1]), "window": out[2],
                "ring_slots": out[3], "scan_filter": bool(out[4])}

    def scan_form(self) -> int:
        """1 if the last packed scan took the skewed-traffic form (stamp filter)."""
        return int(self.mode()["scan_filter"])

    @property
    def deferred(self) -> bool:
        """Scans mark the pending-set bitmap instead of storing cells (VATE_OPT_DEFERRED)."""
        return self.mode()["deferred"]

    @property
    def device_bytes(self) -> int:
        """What the pool occupies in HBM: unpacked cells (u8 / u16 / u32 / u64)
        plus the pending-set bitmap of a deferred AT pool."""
        pend = C.c_int64()
        check(lib.vate_pool_device_bytes(self._h, C.byref(pend)))
        return pend.value

    @property
    def cells(self) -> "DeviceCells":
        return DeviceCells(self)

    # --- instrumentation -----------------------------------------------------------
    def launches(self) -> int:
        n = C.c_uint64()
        check(lib.vate_pool_launches(self._h, C.byref(n)))
        return n.value

    OPTIONS = ("g0_kernel", "incremental", "scan_filter", "concurrent", "inc_sort",
               "fuse_sweep", "deferred", "bitplane", "l2_keep")

    def set_option(self, option: str, value: int) -> None:
        """Tuning switches (include/vate.h enum vate_option): 'g0_kernel' (0 auto,
        1 gather, 2 smem), 'incremental' (0/1), 'scan_filter' (-1 auto, 0, 1),
        'concurrent', 'inc_sort', 'fuse_sweep' (0/1), 'deferred' (-1 auto, 0, 1),
        'bitplane' (-1 auto, 0, 1), 'l2_keep' (-1 auto, 0, 1).
        Every setting leaves identical results."""
        check(lib.vate_pool_set_option(self._h, self.OPTIONS.index(option), int(value)))

    def inc_stats(self) -> dict:
        """Counters of the incremental estimate."""
        out = (C.c_uint64 * 11)()
        check(lib.vate_pool_inc_stats(self._h, out))
        keys = ("rebuilds", "delta_slices", "refresh_slices", "full_slices",
                "last_delta_cells", "last_delta_work", "identity_slices", "hosts_indexed",
                "rebuild_us_total", "miss_accum", "extends")
        return dict(zip(keys, list(out)))

    def sort_stats(self) -> dict:
        """How the sorted active set was produced: full sorts, merges, reuses."""
        out = (C.c_uint64 * 3)()
        check(lib.vate_pool_sort_stats(self._h, out))
        d = dict(zip(("full", "incremental", "reused"), list(out)))
        sz = (C.c_uint64 * 3)()
        check(lib.vate_pool_sort_sizes(self._h, sz))
        d["key_sorts"], d["keys_sorted"], d["largest_sort"] = list(sz)
        return d

    def timeline(self):
        """(kind, start ms, end ms) of every timed launch since set_timing(True)."""
        n = C.c_uint64()
        check(lib.vate_pool_timeline(self._h, None, 0, C.byref(n)))
        out = np.zeros(3 * n.value, dtype=np.float64)
        if n.value:
            check(lib.vate_pool_timeline(self._h, ptr(out), n.value, C.byref(n)))
        return [(_lib.KERNEL_KINDS[int(out[3 * i])], out[3 * i + 1], out[3 * i + 2])
                for i in range(len(out) // 3)]

    def set_latency(self, on: bool) -> None:
        """Per-slice estimate latency of the slice steps (CUDA events: end of the
        slice's scan -> its report rows in host memory); resets the counters."""
        check(lib.vate_pool_set_latency(self._h, int(on)))

    def latency(self) -> dict:
        out = (C.c_double * 4)()
        check(lib.vate_pool_latency(self._h, out))
        return {"slices": int(out[0]), "mean_ms": out[1], "max_ms": out[2], "last_ms": out[3]}

    def l2_ceilings(self, buf_bytes: int = 32 << 20, n: int = 20_000_000, reps: int = 5) -> dict:
        """L2 ceilings over an L2-resident buffer (vate_bench_l2; measurement only)."""
        out = (C.c_double * 4)()
        check(lib.vate_bench_l2(self._h, buf_bytes, n, reps, out))
        return {"buffer_bytes": buf_bytes, "random_sector_reads_G_per_s": out[0],
                "random_u16_stores_G_per_s": out[1], "random_red_or_G_per_s": out[2],
                "stream_read_GB_per_s": out[3]}

    def scan_skeleton_ms(self, mark_log2: int, table_bytes: int, n: int, reps: int = 5) -> float:
        """ms per launch of the scan's memory skeleton (vate_bench_scan_skeleton;
        measurement only): n streamed packets, each one random red.or into a
        2^mark_log2-bit bitmap and one random 32-B read of a table_bytes table."""
        ms = C.c_double()
        check(lib.vate_bench_scan_skeleton(self._h, int(mark_log2), int(table_bytes), int(n),
                                           int(reps), C.byref(ms)))
        return ms.value

    def set_timing(self, on: bool) -> None:
        check(lib.vate_pool_set_timing(self._h, int(on)))

    def kernel_time(self, kind: str):
        """(total ms, launches) recorded by CUDA events for one kernel kind."""
        ms, n = C.c_double(), C.c_uint64()
        check(lib.vate_pool_timing(self._h, _lib.KERNEL_KINDS.index(kind), C.byref(ms), C.byref(n)))
        return ms.value, n.value


class AtPool(BlockLayout, _DevicePool):
    """2**c asynchronous timestamps in 2k staggered-clock blocks, on the GPU."""

    kind = "at"
    _kind_code = 0

    def __init__(self, c: int, k: int, partition: str = TAIL_REMAINDER, device: int = 0):
        BlockLayout.__init__(self, c, k, partition)
        self._create(c, k, partition, device)

    @property
    def bact0(self) -> int:
        """Clock of block 0 in the current slice (pools.py:96)."""
        return self._info()[0]

    # --- layout: BlockLayout supplies block_of / block_range / block_sizes ---
    def block_act(self, bi: int) -> int:
        if not 0 <= bi < self.nblocks:
            raise ValueError(f"block index {bi} outside [0, {self.nblocks})")
        return (self.bact0 + bi) % self.nblocks

    # --- accounting and snapshots ---------------------------------------------------
    @property
    def bits_per_counter(self) -> int:
        return (2 * self.k).bit_length()   # counters.py:52-54

    @property
    def packed_bytes(self) -> int:
        """The reference's accounting: packed words + guard word + header (pools.py:256-259)."""
        return (-(-self.size * self.bits_per_counter // 64) + 1) * 8 + _SNAPSHOT_HEADER.size

    def snapshot_bytes(self) -> bytes:
        """ATP1 bytes identical to the reference's (pools.py:261-265)."""
        n = C.c_uint64()
        check(lib.vate_snapshot_size(self._h, C.byref(n)))
        buf = np.empty(n.value, dtype=np.uint8)
        used = C.c_uint64()
        check(lib.vate_snapshot(self._h, ptr(buf), buf.size, C.byref(used)))
        return buf.tobytes()

    def save(self, path) -> None:
        with open(path, "wb") as fh:
            fh.write(self.snapshot_bytes())

    @classmethod
    def from_bytes(cls, blob: bytes, device: int = 0, where: str = "pool snapshot") -> "AtPool":
        if len(blob) < _SNAPSHOT_HEADER.size:
            raise ConfigError(f"{where} is truncated")
        magic, c, part, k, bact0 = _SNAPSHOT_HEADER.unpack_from(blob)
        if magic != _SNAPSHOT_MAGIC:
            raise ConfigError(f"{where} is not a pool snapshot")
        if part >= len(PARTITIONS):
            raise ConfigError(f"snapshot has unknown partition code {part}")
        pool = cls(c, k, PARTITIONS[part], device=device)
        if bact0 >= pool.nblocks:
            raise ConfigError(f"snapshot clock {bact0} out of range")
        expected = 8 * -(-pool.size * pool.bits_per_counter // 64)
        if len(blob) - _SNAPSHOT_HEADER.size != expected:
            raise ConfigError(
                f"snapshot payload is {len(blob) - _SNAPSHOT_HEADER.size} bytes, "
                f"expected {expected}")
        arr = np.frombuffer(blob, dtype=np.uint8)
        check(lib.vate_load(pool._h, ptr(arr), arr.size))
        return pool

    @classmethod
    def load(cls, path, device: int = 0) -> "AtPool":
        """pools.py:271-298."""
        with open(path, "rb") as fh:
            blob = fh.read()
        return cls.from_bytes(blob, device=device, where=str(path))



class DeviceCells:
    """Read view of the cells mirroring PackedArray's read API (bitpack.py:26-140)."""

    def __init__(self, pool: _DevicePool):
        self._pool = pool
        self.size = pool.size
        self.width = pool.bits_per_counter
        self.mask = np.uint64((1 << self.width) - 1) if self.width < 64 else np.uint64(~0 & ((1 << 64) - 1))

    def __len__(self):
        return self.size

    def get(self, idx) -> np.ndarray:
        idx = _as_u64(idx)
        out = np.empty(idx.shape, dtype=np.uint64)
        if idx.size:
            check(lib.vate_get_cells64(self._pool.handle, ptr(idx), idx.size, ptr(out), VATE_HOST))
        return out

    def get_one(self, i: int) -> int:
        return int(self.get(np.array([i], dtype=np.uint64))[0])

    def get_range(self, start: int, stop: int) -> np.ndarray:
        return self.get(np.arange(start, stop, dtype=np.uint64))

    @property
    def data_words(self) -> np.ndarray:
        """The packed payload words of the ATP1 snapshot (bitpack.py:46-49)."""
        blob = self._pool.snapshot_bytes()
        return np.frombuffer(blob[_SNAPSHOT_HEADER.size:], dtype="<u8").copy()

    # --- write API (bitpack.py:57-78, :97-140), device kernels -------------------
    def set(self, idx, values) -> None:
        """cells[idx] = values & mask; duplicate indices must carry equal values."""
        idx = _as_u64(idx)
        vals = np.ascontiguousarray(np.broadcast_to(
            np.asarray(values, dtype=np.uint64), idx.shape)).reshape(-1)
        idx = np.ascontiguousarray(idx.reshape(-1))
        if idx.size:
            check(lib.vate_put_cells(self._pool.handle, ptr(idx), ptr(vals), idx.size, VATE_HOST))

    def set_one(self, i: int, value: int) -> None:
        if not 0 <= i < self.size:
            raise ValueError(f"cell index {i} outside [0, {self.size})")
        self.set(np.array([i], dtype=np.uint64), np.array([int(value) & int(self.mask)],
                                                           dtype=np.uint64))

    def set_range(self, start: int, values) -> None:
        values = np.asarray(values, dtype=np.uint64)
        self.set(np.arange(start, start + len(values), dtype=np.uint64), values)

    def fill(self, value: int) -> None:
        """Every cell = value (ValueError if it exceeds the width, bitpack.py:57-60)."""
        if int(value) >> self.width:
            raise ValueError(f"value {value} exceeds {self.width} bits")
        check(lib.vate_fill_cells(self._pool.handle, int(value)))

    @property
    def nbytes(self) -> int:
        """PackedArray.nbytes: packed words plus the guard word (bitpack.py:53-55)."""
        return (-(-self.size * self.width // 64) + 1) * 8 if self.width < 64 else self.size * 8


class DrPool(_DevicePool):
    """2**c distance recorders; every cell slides every slice (pools.py:301-353)."""

    kind = "dr"
    _kind_code = 1

    def __init__(self, c: int, k: int, device: int = 0):
        _validate_pool_shape(c, k)
        self.c, self.k, self.size = c, k, 1 << c
        self._create(c, k, TAIL_REMAINDER, device)

    @property
    def bits_per_counter(self) -> int:
        return self.k.bit_length()          # dr_bits, counters.py:132-134

    @property
    def packed_bytes(self) -> int:
        """The reference's PackedArray accounting (bitpack.py nbytes)."""
        return (-(-self.size * self.bits_per_counter // 64) + 1) * 8


class TsPool(_DevicePool):
    """2**c plain last-seen slice indices; no maintenance (pools.py:356-410)."""

    kind = "ts"
    _kind_code = 2

    def __init__(self, c: int, k: int, device: int = 0):
        _validate_pool_shape(c, k)
        self.c, self.k, self.size = c, k, 1 << c
        self._create(c, k, TAIL_REMAINDER, device)

    @property
    def t(self) -> int:
        """The pool's current slice index (advances taken, pools.py:360)."""
        kind, t = C.c_int(), C.c_uint64()
        check(lib.vate_pool_kind(self._h, C.byref(kind), C.byref(t)))
        return t.value

    @property
    def bits_per_counter(self) -> int:
        return 64

    @property
    def packed_bytes(self) -> int:
        return self.size * 8


def make_pool(kind: str, c: int, k: int, partition: str = TAIL_REMAINDER, device: int = 0):
    """Build a counter pool by kind name (pools.py:413-421)."""
    if kind == "at":
        return AtPool(c, k, partition, device=device)
    if kind == "dr":
        return DrPool(c, k, device=device)
    if kind == "ts":
        return TsPool(c, k, device=device)
    raise ConfigError(f"unknown counter kind {kind!r}")
