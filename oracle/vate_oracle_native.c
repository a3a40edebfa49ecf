/* vate_oracle_native.c -- TEST INFRASTRUCTURE ONLY (the oracle's C half).
 *
 * Plain-C restatement of the oracle functions whose numpy form is too slow for
 * parity checks at BASELINE sizes (2^28 cells, 5M packets per slice, 1M hosts x
 * g = 1024):
 *
 *   vo_host_g0      per-host inactive virtual-slot count g0
 *                   (estimator.py:107-123 host_cells + inactive_virtual_counts,
 *                    with hashing.py:25-57 and pools.py:187-193)
 *   vo_pack_cells   ATP1 payload: w-bit cells LSB-first into little-endian u64
 *                   words (bitpack.py:26-78, pools.py:261-265)
 *   vo_pair_cells   estimator.py:96-99 (hashing.py:48-67)
 *   vo_set_cells    AtPool.set_many with its value histogram (pools.py:163-178)
 *   vo_synthetic_slice  the tests' synthetic traffic (oracle.synthetic_slice)
 *
 * Paths are relative to the reference package root pkg/src/slidecard/.  Only
 * tests/ (through oracle/native.py) may load this library; the product path is
 * the CUDA library.  Its results are pinned against oracle/vate_oracle.py (the
 * numpy restatement, itself pinned to the reference's golden vectors) by
 * tests/test_oracle_native.py.
 *
 * Cells are held unpacked as uint32 (one per cell), block lookup is a binary
 * search over the block start offsets (as the numpy oracle's searchsorted).
 */
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define PHI 0x9E3779B97F4A7C15ull  /* hashing.py:18 */
#define MUL1 0xBF58476D1CE4E5B9ull /* hashing.py:28 */
#define MUL2 0x94D049BB133111EBull /* hashing.py:29 */

static inline uint64_t mix64(uint64_t z) { /* hashing.py:25-30 */
  z ^= z >> 30;
  z *= MUL1;
  z ^= z >> 27;
  z *= MUL2;
  return z ^ (z >> 31);
}

/* block owning cell i: last b with starts[b] <= i (starts has nblocks + 1 entries) */
static inline int block_of(const int64_t* starts, int nblocks, int64_t i) {
  int lo = 0, hi = nblocks; /* invariant: starts[lo] <= i < starts[hi] */
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (starts[mid] <= i) lo = mid;
    else hi = mid;
  }
  return lo;
}

int vo_abi(void) { return 1; }

/* g0[h] = #{ j < g : cell(aip_h, j) inactive for k' }  (estimator.py:114-123).
 * cell(aip, j) = mix64(((aip << 32) | j) * phi + cell_stream) & (size - 1)
 * (hashing.py:48-57: aip bits >= 32 fall off the 64-bit key);
 * inactive: v == sentinel or (clock(block) - v) mod 2k >= k' (pools.py:187-193). */
int vo_host_g0(const uint32_t* cells, uint64_t size, const int64_t* starts, int nblocks,
               int bact0, int k_prime, uint64_t g, uint64_t cell_stream,
               const uint64_t* aips, uint64_t n, int64_t* out, int threads) {
  const uint64_t mask = size - 1;
  const uint32_t sentinel = (uint32_t)nblocks;
  (void)threads;
#pragma omp parallel for schedule(dynamic, 256) num_threads(threads > 0 ? threads : 1)
  for (int64_t h = 0; h < (int64_t)n; ++h) {
    const uint64_t hi = aips[h] << 32;
    int64_t cnt = 0;
    for (uint64_t j = 0; j < g; ++j) {
      const uint64_t cell = mix64((hi | j) * PHI + cell_stream) & mask;
      const uint32_t v = cells[cell];
      if (v == sentinel) {
        ++cnt;
        continue;
      }
      const int b = block_of(starts, nblocks, (int64_t)cell);
      const int64_t act = (int64_t)((bact0 + b) % nblocks);
      const int64_t dist = ((act - (int64_t)v) % nblocks + nblocks) % nblocks;
      cnt += dist >= k_prime;
    }
    out[h] = cnt;
  }
  return 0;
}

/* ATP1 payload (bitpack.py:26-78): cell i occupies bits [i*w, i*w + w) of the
 * little-endian u64 word array, LSB first; pad bits are zero.  Every group of 64
 * cells fills exactly w words, so groups are independent (parallel). */
int vo_pack_cells(const uint32_t* cells, uint64_t n, int width, uint64_t* words,
                  uint64_t nwords, int threads) {
  memset(words, 0, nwords * 8);
  const int64_t groups = (int64_t)((n + 63) / 64);
  (void)threads;
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
  for (int64_t q = 0; q < groups; ++q) {
    const uint64_t lo = (uint64_t)q * 64, hi = lo + 64 < n ? lo + 64 : n;
    for (uint64_t i = lo; i < hi; ++i) {
      const uint64_t v = cells[i] & ((1ull << width) - 1);
      const uint64_t bit = i * (uint64_t)width;
      const uint64_t w = bit >> 6;
      const unsigned s = (unsigned)(bit & 63);
      words[w] |= v << s;
      if (s + width > 64) words[w + 1] |= v >> (64 - s);
    }
  }
  return 0;
}

/* pair_cells (estimator.py:96-99): cell = H(aip, BH(bip)) with
 * BH(bip) = mix64(bip * phi + group_stream) mod g (hashing.py:60-67). */
int vo_pair_cells(const uint64_t* aips, const uint64_t* bips, uint64_t n, uint64_t g, int c,
                  uint64_t cell_stream, uint64_t group_stream, uint64_t* out, int threads) {
  const uint64_t mask = c >= 64 ? ~0ull : ((1ull << c) - 1);
  (void)threads;
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
  for (int64_t i = 0; i < (int64_t)n; ++i) {
    const uint64_t slot = mix64(bips[i] * PHI + group_stream) % g;
    out[i] = mix64(((aips[i] << 32) | slot) * PHI + cell_stream) & mask;
  }
  return 0;
}

/* AtPool.set_many with the per-block value histogram (pools.py:163-178): every
 * listed cell takes its block's clock (bact0 + block) mod 2k; hist[block][old]--
 * and hist[block][new]++ once per distinct cell (in list order: a repeat finds
 * the new value already stored and changes nothing, exactly like np.unique
 * first).  hist may be NULL.  Block ids are found in parallel; then each thread
 * applies the cells of its own contiguous block range (so cells and histogram
 * rows have one writer each).  blk is caller scratch of n int32. */
int vo_set_cells(uint32_t* cells, uint64_t size, const int64_t* starts, int nblocks, int bact0,
                 const uint64_t* idx, uint64_t n, int64_t* hist, int32_t* blk, int threads) {
  int bad = 0;
  const int nt = threads > 0 ? threads : 1;
#pragma omp parallel for schedule(static) num_threads(nt) reduction(| : bad)
  for (int64_t q = 0; q < (int64_t)n; ++q) {
    if (idx[q] >= size) { /* pools.py:106-107 */
      bad = 1;
      blk[q] = -1;
      continue;
    }
    blk[q] = block_of(starts, nblocks, (int64_t)idx[q]);
  }
  if (bad) return -1;
#pragma omp parallel num_threads(nt)
  {
#ifdef _OPENMP
    const int me = omp_get_thread_num(), all = omp_get_num_threads();
#else
    const int me = 0, all = 1;
#endif
    const int lo = (int)((int64_t)nblocks * me / all), hi = (int)((int64_t)nblocks * (me + 1) / all);
    for (uint64_t q = 0; q < n; ++q) {
      const int b = blk[q];
      if (b < lo || b >= hi) continue;
      const uint64_t i = idx[q];
      const uint32_t act = (uint32_t)((bact0 + b) % nblocks);
      const uint32_t old = cells[i];
      if (old == act) continue;
      if (hist) {
        hist[(int64_t)b * (nblocks + 1) + old] -= 1;
        hist[(int64_t)b * (nblocks + 1) + act] += 1;
      }
      cells[i] = act;
    }
  }
  return 0;
}

/* oracle.synthetic_slice (test traffic, not reference code): packet i of slice t
 * draws x = mix64(stream + (t * 2^32 + i) * phi); host rank = x mod hosts; peer j
 * of that host's fixed set of 1 + (r & 7) + 2^min(lz, 12) peers, r a 24-bit per
 * host hash with lz = 24 - bit_length(r). */
int vo_synthetic_slice(int64_t t, uint64_t n, uint64_t hosts, uint64_t base_aip, uint64_t stream,
                       uint64_t host_salt, uint64_t peer_salt, uint64_t* aips, uint64_t* bips,
                       int threads) {
  const uint64_t t_hi = ((uint64_t)t & 0xFFFFFFFFull) << 32;
  (void)threads;
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
  for (int64_t i = 0; i < (int64_t)n; ++i) {
    const uint64_t x = mix64(stream + ((uint64_t)i + t_hi) * PHI);
    const uint64_t rank = x % hosts;
    const uint64_t r = mix64(rank ^ host_salt) >> 40;
    const int bl = r ? 64 - __builtin_clzll(r) : 0;
    const int lz = 24 - bl < 12 ? 24 - bl : 12;
    const uint64_t npeers = 1 + (r & 7) + (1ull << lz);
    const uint64_t j = (x >> 32) % npeers;
    bips[i] = mix64((rank << 20) ^ j ^ peer_salt) & 0xFFFFFFFFull;
    aips[i] = (rank + base_aip) & 0xFFFFFFFFull;
  }
  return 0;
}
