"""Window shape and the AT width rule (reference: counters.py:27-54).

The per-cell AT rules (set / check / preserve, counters.py:57-127) are
implemented on the device: csrc/vate_internal.cuh (is_inactive) and
csrc/vate_pool.cu (k_sweep, the comparison-only preserve).
"""

from dataclasses import dataclass

MAX_K = 1 << 15
TS_UNSET = (1 << 64) - 1   # counters.py:159: a TS cell never set


@dataclass(frozen=True)
class WindowConfig:
    """Up to ``k`` slices of ``slice_us`` microseconds (counters.py:30-47)."""

    k: int
    slice_us: int

    def __post_init__(self):
        if not 1 <= self.k <= MAX_K:
            raise ValueError(f"k must be in [1, {MAX_K}], got {self.k}")
        if self.slice_us <= 0:
            raise ValueError(f"slice_us must be positive, got {self.slice_us}")

    def validate_width(self, k_prime: int) -> None:
        if not 1 <= k_prime <= self.k:
            raise ValueError(f"query width k'={k_prime} outside [1, {self.k}]")


def ats_bits(k: int) -> int:
    """Bits per asynchronous timestamp: ceil(log2(2k+1)) (counters.py:52-54)."""
    return (2 * k).bit_length()


def dr_bits(k: int) -> int:
    """Bits per distance recorder: ceil(log2(k+1)) (counters.py:132-134)."""
    return k.bit_length()
