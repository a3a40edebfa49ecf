"""ctypes loader for oracle/vate_oracle_native.c -- TEST INFRASTRUCTURE ONLY.

The C half of the oracle (g0 over many hosts, ATP1 packing) for parity checks
at BASELINE sizes.  ``build()`` compiles it with gcc into ``oracle/_build/``
(git-ignored; the .so travels to the GPU box with the snapshot, and is rebuilt
on demand if missing).  Only ``tests/`` use it.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "vate_oracle_native.c")
OUT = os.path.join(HERE, "_build", "libvate_oracle.so")

_lib = None


def build() -> str:
    """gcc -O3 -fopenmp the oracle's C half (idempotent: skips an up-to-date .so)."""
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    if os.path.exists(OUT) and os.path.getmtime(OUT) >= os.path.getmtime(SRC):
        return OUT
    subprocess.run(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC",
                    "-o", OUT, SRC], check=True)
    return OUT


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        _lib.vo_host_g0.argtypes = [P, C.c_uint64, P, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                    C.c_uint64, P, C.c_uint64, P, C.c_int]
        _lib.vo_pack_cells.argtypes = [P, C.c_uint64, C.c_int, P, C.c_uint64, C.c_int]
        _lib.vo_pair_cells.argtypes = [P, P, C.c_uint64, C.c_uint64, C.c_int, C.c_uint64,
                                       C.c_uint64, P, C.c_int]
        _lib.vo_set_cells.argtypes = [P, C.c_uint64, P, C.c_int, C.c_int, P, C.c_uint64, P, P,
                                      C.c_int]
        _lib.vo_synthetic_slice.argtypes = [C.c_int64, C.c_uint64, C.c_uint64, C.c_uint64,
                                            C.c_uint64, C.c_uint64, C.c_uint64, P, P, C.c_int]
    return _lib


def _threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def host_g0(pool, cfg, aips, k_prime: int) -> np.ndarray:
    """oracle.host_g0 (estimator.py:114-123) for an OraclePool, in C."""
    pool._check_width(k_prime)
    cells = np.ascontiguousarray(pool.cells, dtype=np.uint32)
    starts = np.ascontiguousarray(pool.starts, dtype=np.int64)
    a = np.ascontiguousarray(np.asarray(aips).astype(np.uint64))
    out = np.empty(len(a), dtype=np.int64)
    lib().vo_host_g0(cells.ctypes.data, pool.size, starts.ctypes.data, pool.nblocks,
                     int(pool.bact0), int(k_prime), int(cfg.g), int(cfg.cell_stream),
                     a.ctypes.data, len(a), out.ctypes.data, _threads())
    return out


def pair_cells(cfg, aips, bips) -> np.ndarray:
    """OracleConfig.pair_cells (estimator.py:96-99) in C."""
    a = np.ascontiguousarray(np.asarray(aips).astype(np.uint64))
    b = np.ascontiguousarray(np.asarray(bips).astype(np.uint64))
    out = np.empty(len(a), dtype=np.uint64)
    lib().vo_pair_cells(a.ctypes.data, b.ctypes.data, len(a), int(cfg.g), int(cfg.c),
                        int(cfg.cell_stream), int(cfg.group_stream), out.ctypes.data, _threads())
    return out


def set_cells(pool, idx) -> None:
    """OraclePool.set_cells (pools.py:163-178), histogram included when tracked, in C."""
    i = np.ascontiguousarray(np.asarray(idx).astype(np.uint64))
    assert pool.cells.dtype == np.uint32 and pool.cells.flags.c_contiguous
    starts = np.ascontiguousarray(pool.starts, dtype=np.int64)
    hist = pool.hist
    if hist is not None:
        assert hist.dtype == np.int64 and hist.flags.c_contiguous
    blk = np.empty(len(i), dtype=np.int32)
    rc = lib().vo_set_cells(pool.cells.ctypes.data, pool.size, starts.ctypes.data, pool.nblocks,
                            int(pool.bact0), i.ctypes.data, len(i),
                            hist.ctypes.data if hist is not None else None, blk.ctypes.data,
                            _threads())
    if rc:
        raise ValueError("cell index out of range")


def synthetic_slice(t: int, n: int, hosts: int, base_aip: int = 0x0A000000, trace_seed: int = 0):
    """oracle.synthetic_slice in C (same packets, bit for bit)."""
    from .vate_oracle import SYNTH_HOST_SALT, SYNTH_PEER_SALT, SYNTH_SALT, stream_of
    a = np.empty(n, dtype=np.uint64)
    b = np.empty(n, dtype=np.uint64)
    lib().vo_synthetic_slice(int(t), n, hosts, base_aip, stream_of(trace_seed, SYNTH_SALT),
                             SYNTH_HOST_SALT, SYNTH_PEER_SALT, a.ctypes.data, b.ctypes.data,
                             _threads())
    return a, b


def pack_cells(cells: np.ndarray, width: int) -> bytes:
    """oracle.pack_cells (bitpack.py:26-78) in C."""
    c = np.ascontiguousarray(cells, dtype=np.uint32)
    nwords = -(-len(c) * width // 64)
    words = np.empty(nwords, dtype=np.uint64)
    lib().vo_pack_cells(c.ctypes.data, len(c), int(width), words.ctypes.data, nwords, _threads())
    return words.astype("<u8", copy=False).tobytes()


def snapshot_bytes(pool) -> bytes:
    """OraclePool.snapshot_bytes (pools.py:261-265) with the C packer."""
    from .vate_oracle import ATP1_HEADER, ATP1_MAGIC, PARTITION_CODES, at_width
    header = ATP1_HEADER.pack(ATP1_MAGIC, pool.c, PARTITION_CODES[pool.partition], pool.k,
                              pool.bact0)
    return header + pack_cells(pool.cells, at_width(pool.k))
