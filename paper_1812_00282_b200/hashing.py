"""Scalar hash helpers and constants (reference: hashing.py:18-67).

The data path hashes on the device (csrc/vate_internal.cuh: mix64, slot_of,
cell_of).  The host only needs the scalar finalizer to derive the two hash
streams of an EstimatorConfig once, and the scalar lookups for the
single-value API (virtual_slot / cell_of).
"""

_M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
CELL_SALT = 0x9D9E26B1D9C4F201
GROUP_SALT = 0x5C5D14FA8A33E96D


def mix64(z: int) -> int:
    """splitmix64 finalizer on a Python int, wrapping at 2**64."""
    z &= _M64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & _M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def derive_stream(seed: int, salt: int) -> int:
    """One hash family's stream from the user seed (hashing.py:43-45)."""
    return mix64((seed ^ salt) & _M64)


def cell_index(aip: int, vid: int, c: int, stream: int) -> int:
    """Scalar H(aip, slot); only the low 32 bits of aip reach the key."""
    return mix64(((((aip << 32) | vid) & _M64) * GOLDEN + stream) & _M64) & ((1 << c) - 1)


def group_index(bip: int, g: int, stream: int) -> int:
    """Scalar BH(bip) in [0, g)."""
    return mix64((bip * GOLDEN + stream) & _M64) % g
