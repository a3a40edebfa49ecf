// vate_cells.cuh -- register-level helpers on 32-cell words of unpacked cells,
// shared by the pool pass (vate_pool.cu) and the bit-plane mode's block
// materialisation (vate_bitplane.cu): the two-block sweep (pools.py:221-249,
// counters.py:113-127), pending marks taking their block clock
// (pools.py:164-178), whole-sector write-back.
#pragma once

#include "vate_internal.cuh"

namespace vate {

struct SweepSpec {
  uint64_t s0, e0, s1, e1;          // the two due ranges (e == s: none)
  uint32_t k, B;
  unsigned long long* cleared;      // nullptr: no fused sweep
};

// Register-free (re-reads the word's cells, L1-hot): words of u32 cells and the
// partial last word of a tiny pool.
template <typename T>
__device__ __forceinline__ unsigned sweep_word(T* __restrict__ cells, uint64_t i0, uint32_t cnt,
                                            uint64_t s0, uint64_t e0, uint64_t s1, uint64_t e1,
                                            uint32_t k, uint32_t B) {
  unsigned cleared = 0;
  for (uint32_t j = 0; j < cnt; ++j) {
    const uint64_t i = i0 + j;
    const bool due0 = i >= s0 && i < e0, due1 = i >= s1 && i < e1;
    if (!due0 && !due1) continue;
    const uint32_t v = cells[i];
    const bool stale = due0 ? v <= k : ((v >= k && v <= B - 1) || v == 0);
    if (stale) {
      cells[i] = (T)B;
      ++cleared;
    }
  }
  return cleared;
}

// Bits j of [i0, i0+32) that fall in [s, e).
__device__ __forceinline__ uint32_t range_bits(uint64_t i0, uint64_t s, uint64_t e) {
  const uint64_t lo = s > i0 ? s - i0 : 0, hi = e > i0 ? umin64(e - i0, 32) : 0;
  if (lo >= hi) return 0u;
  const uint32_t below_hi = hi >= 32 ? 0xffffffffu : (1u << hi) - 1u;
  return below_hi & ~((1u << lo) - 1u);
}

// The same sweep for a full word of u8/u16 cells, on the pass's register copy:
// stale cells are rewritten in the registers; bit v of `chg` marks a changed
// uint4.  (The scalar form re-reads each cell from L2 -- the pass's loads are
// evict-first -- and its 32 dependent round trips set the kernel's tail on
// small pools.)
template <typename T>
__device__ __forceinline__ unsigned sweep_regs(uint4 (&r)[(int)sizeof(T) * 2], uint64_t i0,
                                               const SweepSpec& SW, unsigned& chg) {
  static_assert(sizeof(T) <= 2, "u8/u16 cells");
  const uint32_t due0 = range_bits(i0, SW.s0, SW.e0), due1 = range_bits(i0, SW.s1, SW.e1);
  if (!(due0 | due1)) return 0;
  constexpr int kPer = 4 / (int)sizeof(T), kBits = 8 * (int)sizeof(T);
  constexpr uint32_t kMask = sizeof(T) == 1 ? 0xFFu : 0xFFFFu;
  uint32_t* x = reinterpret_cast<uint32_t*>(r);
  unsigned cleared = 0;
#pragma unroll
  for (int q = 0; q < 32 / kPer; ++q) {
#pragma unroll
    for (int h = 0; h < kPer; ++h) {
      const int j = q * kPer + h;
      const uint32_t v = (x[q] >> (h * kBits)) & kMask;
      const bool stale = ((due0 >> j) & 1u) ? v <= SW.k
                         : ((due1 >> j) & 1u) ? ((v >= SW.k && v <= SW.B - 1) || v == 0) : false;
      if (stale) {
        x[q] = (x[q] & ~(kMask << (h * kBits))) | (SW.B << (h * kBits));
        ++cleared;
        chg |= 1u << (q / 4);
      }
    }
  }
  return cleared;
}

// Pending-set marks of a word whose 32 cells share clock `act`, applied to the
// register copy (u8: 4 cells per 32-bit lane, u16: 2); bit v of the result
// marks a changed uint4.
template <typename T>
__device__ __forceinline__ unsigned apply_marks_regs(uint4 (&r)[(int)sizeof(T) * 2], uint32_t m,
                                                     uint32_t act) {
  static_assert(sizeof(T) <= 2, "u8/u16 cells");
  uint32_t* x = reinterpret_cast<uint32_t*>(r);
  unsigned chg = 0;
  if (sizeof(T) == 1) {
    const uint32_t a4 = act * 0x01010101u;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t nib = (m >> (4 * q)) & 0xFu;
      const uint32_t bm = ((nib * 0x00204081u) & 0x01010101u) * 0xFFu;  // bit j -> byte j
      x[q] = (x[q] & ~bm) | (a4 & bm);
    }
    chg = m ? 3u : 0u;  // (see below: a marked cell changes)
  } else {
    // lane masks by sign-replicating byte permutes: copy s[k] = m << k puts bit
    // 8j + 7 - k of m at the sign of byte j, and prmt with a selector nibble's
    // bit 3 set writes that sign into a whole byte -- one prmt per two cells
    const uint32_t a2 = act * 0x00010001u;
    uint32_t sh[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) sh[k] = m << k;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int j = (2 * q) >> 3, k = 7 - ((2 * q) & 7);  // bit 2q: byte j of sh[k]; 2q+1: of sh[k-1]
      const uint32_t sel = (8u | j) | ((8u | j) << 4) | ((12u | j) << 8) | ((12u | j) << 12);
      uint32_t bm;
      asm("prmt.b32 %0, %1, %2, %3;" : "=r"(bm) : "r"(sh[k]), "r"(sh[k - 1]), "r"(sel));
      x[q] = (x[q] & ~bm) | (a2 & bm);
    }
    // a marked cell never already holds its clock (it would have been set in
    // this slice, and this slice's sets are the marks): a sector with a mark
    // changed
    chg = ((m & 0xFFFFu) ? 3u : 0u) | ((m >> 16) ? 12u : 0u);
  }
  return chg;
}

// Marks of a word that straddles a block boundary (or holds u32 cells), in
// memory: each marked cell takes its own block's clock.
template <typename T>
__device__ __forceinline__ void apply_marks_scalar(T* __restrict__ cells, uint64_t i0, uint32_t cnt,
                                                   uint32_t m, const Layout& L, uint32_t bact0) {
  for_word_clocks(i0, cnt, L, bact0, [&](uint32_t j, uint32_t act) {
    if ((m >> j) & 1u) cells[i0 + j] = (T)act;
  });
}

// Changed 32-byte sectors of a word back to HBM (uint4 pairs, whole sectors).
template <typename T>
__device__ __forceinline__ void store_sectors(T* __restrict__ cells, uint64_t i0,
                                              const uint4 (&r)[(int)sizeof(T) * 2], unsigned chg) {
  constexpr int NV = (int)sizeof(T) * 2;
  uint4* dst = reinterpret_cast<uint4*>(cells + i0);
#pragma unroll
  for (int s = 0; s < NV / 2; ++s)
    if ((chg >> (2 * s)) & 3u) {
      dst[2 * s] = r[2 * s];
      dst[2 * s + 1] = r[2 * s + 1];
    }
}


}  // namespace vate
