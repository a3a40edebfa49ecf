// vate_bitplane.cu -- the AT pool's recent history as bit planes.
//
// A deferred pool's scan already writes one bit per packet into an
// L2-resident mark bitmap instead of the cell.  Bit-plane mode keeps those
// bitmaps, one per epoch (an epoch is the span between two advances, i.e. a
// slice), in a ring of R = k + L + 1 slots, and answers the per-slice
// estimate for k' = L without reading the 2^c cells:
//
//   a cell is active for k' at epoch e  <=>  it was set in one of the epochs
//   e-k'+1 .. e  (ats_check, counters.py:79-90, with the two-block sweep's
//   guarantee that no stale clock aliases: the reference's own AT == DR == TS
//   identity, test_estimator.py:233-255)
//
// so inactive = ~(OR of the last L mark bitmaps).  That sliding OR is kept in
// two pieces (the two-stacks trick): epochs are grouped in blocks of L; P is
// the OR of the current block's finished epochs, and S[j] (j = 1 .. L-1) the
// OR of the previous block's epochs j .. L-1, built once per block by one
// backward pass over its L bitmaps.  At epoch e = N*L + j the window is
// S[j+1] | P | M_e: the estimate's pool pass reads three 2^c/8-byte bitmaps
// and the previous bitmap instead of 2^c cells (cfg 4: 4 x 32 MiB instead of
// 512 MiB).
//
// The cells stay the reference's AT state (snapshots, point queries, other
// k'): each AT block remembers the last epoch whose marks it holds; when the
// two-block advance makes a block due (pools.py:221-249) its pending epochs
// are applied -- per cell the newest marking epoch's clock -- and then the
// sweep rule, exactly as the direct path would have left it.  Every block is
// due every k epochs, so no block is more than k epochs behind and the ring
// reaches back far enough; a read of the cells anywhere else first brings
// every block up to date (bp_materialize_all).
//
// Memory (cfg 4: c = 28, k = k' = 300): ring 601 x 32 MiB + S 299 x 32 MiB
// = 28 GiB of HBM, traded for ~0.5 GB less DRAM traffic per slice.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "vate_cells.cuh"
#include "vate_internal.cuh"

namespace vate {

__host__ __device__ __forceinline__ uint32_t slot_of_epoch(int64_t e, uint32_t R) {
  return (uint32_t)(((e % (int64_t)R) + (int64_t)R) % (int64_t)R);
}

__device__ __forceinline__ unsigned block_sum_bp(unsigned v) {
  __shared__ unsigned warp_sums[32];
  v = __reduce_add_sync(0xffffffffu, v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) warp_sums[wid] = v;
  __syncthreads();
  unsigned total = 0;
  if (wid == 0) {
    total = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0u;
    total = __reduce_add_sync(0xffffffffu, total);
  }
  return total;  // valid in thread 0
}

// Block clock at epoch ep, given the clock of block 0 at epoch e_hi.
__device__ __forceinline__ uint32_t clock_at(uint32_t bact0_hi, int64_t e_hi, int64_t ep,
                                             uint32_t b, uint32_t B) {
  const uint32_t back = (uint32_t)(e_hi - ep) % B;  // e_hi - ep < the ring length
  return (bact0_hi + B - back + b) % B;
}

// The estimate's pass: bits = ~(S | P | M) over valid cells, P's popcount,
// the incremental-g0 delta against the previous bitmap, and (fold) P | M as
// the new prefix.  Four words per thread (16-byte loads).
template <bool CS>
__global__ void __launch_bounds__(256) k_bp_window(const uint32_t* __restrict__ S,
                                                   const uint32_t* __restrict__ Pin,
                                                   const uint32_t* __restrict__ M,
                                                   uint32_t* __restrict__ Pout,
                                                   uint32_t* __restrict__ bitmap,
                                                   uint64_t nwords, uint64_t size,
                                                   unsigned long long* pool_inactive,
                                                   DeltaOut D, Publish pub) {
  __shared__ DeltaStage ds;
  delta_stage_init(ds);
  unsigned local = 0;
  const uint64_t nq = (nwords + 3) / 4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq; q += stride) {
    const uint64_t w0 = q * 4;
    uint32_t s[4] = {0, 0, 0, 0}, pv[4], m[4], prev[4] = {0, 0, 0, 0};
    if (w0 + 4 <= nwords) {
      const uint4 pp = __ldcs(reinterpret_cast<const uint4*>(Pin) + q);
      const uint4 mm = __ldcg(reinterpret_cast<const uint4*>(M) + q);
      pv[0] = pp.x; pv[1] = pp.y; pv[2] = pp.z; pv[3] = pp.w;
      m[0] = mm.x; m[1] = mm.y; m[2] = mm.z; m[3] = mm.w;
      if (S) {
        const uint4 ss = __ldcs(reinterpret_cast<const uint4*>(S) + q);
        s[0] = ss.x; s[1] = ss.y; s[2] = ss.z; s[3] = ss.w;
      }
      if (D.bprev) {
        const uint4 bb = __ldcs(reinterpret_cast<const uint4*>(D.bprev) + q);
        prev[0] = bb.x; prev[1] = bb.y; prev[2] = bb.z; prev[3] = bb.w;
      }
    } else {
      for (int i = 0; i < 4; ++i) {
        const uint64_t w = w0 + i;
        pv[i] = w < nwords ? Pin[w] : 0u;
        m[i] = w < nwords ? M[w] : 0u;
        if (S) s[i] = w < nwords ? S[w] : 0u;
        if (D.bprev) prev[i] = w < nwords ? D.bprev[w] : 0u;
      }
    }
    uint32_t bits[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint64_t w = w0 + i;
      const uint64_t i0 = w * 32;
      const uint32_t valid = i0 + 32 <= size ? 0xffffffffu
                             : (i0 < size ? (1u << (uint32_t)(size - i0)) - 1u : 0u);
      bits[i] = ~(s[i] | pv[i] | m[i]) & valid;
      local += __popc(bits[i]);
      if (D.bprev && w < nwords) delta_word(D, ds, bits[i], prev[i], i0);
    }
    if (w0 + 4 <= nwords) {
      const uint4 bv = make_uint4(bits[0], bits[1], bits[2], bits[3]);
      const uint4 pw = make_uint4(pv[0] | m[0], pv[1] | m[1], pv[2] | m[2], pv[3] | m[3]);
      if (CS) {  // evict-first: keep the registry and the marks in L2 for the next scan
        __stcs(reinterpret_cast<uint4*>(bitmap) + q, bv);
        if (Pout) __stcs(reinterpret_cast<uint4*>(Pout) + q, pw);
      } else {
        reinterpret_cast<uint4*>(bitmap)[q] = bv;
        if (Pout) reinterpret_cast<uint4*>(Pout)[q] = pw;
      }
    } else {
      for (int i = 0; i < 4; ++i)
        if (w0 + i < nwords) {
          bitmap[w0 + i] = bits[i];
          if (Pout) Pout[w0 + i] = pv[i] | m[i];
        }
    }
  }
  if (D.bprev) delta_flush(D, ds);
  const unsigned sum = block_sum_bp(local);
  if (threadIdx.x == 0 && sum) atomicAdd(pool_inactive, (unsigned long long)sum);
  publish_last_block(pub);
}

// P |= M (an advance with no estimate in its epoch).
__global__ void k_bp_fold(uint32_t* __restrict__ P, const uint32_t* __restrict__ M, uint64_t nwords) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += stride)
    P[w] |= M[w];
}

// S[j] = OR of the block's epochs j .. L-1 (j = L-1 down to 1), one word
// position per thread; loads of eight epochs are issued ahead of their ORs.
__global__ void __launch_bounds__(256) k_bp_suffix(const uint32_t* __restrict__ ring, uint32_t R,
                                                   int64_t base, uint32_t L,
                                                   uint32_t* __restrict__ S, uint64_t nwords) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += stride) {
    uint32_t acc = 0;
    int j = (int)L - 1;
    uint32_t slot = slot_of_epoch(base + j, R);
    while (j >= 1) {
      uint32_t v[8];
      const int n = j >= 8 ? 8 : j;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (u < n) {
          v[u] = __ldcs(ring + (uint64_t)slot * nwords + w);
          slot = slot ? slot - 1 : R - 1;
        }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (u < n) {
          acc |= v[u];
          S[(uint64_t)(j - u - 1) * nwords + w] = acc;  // S[j'] at index j' - 1
        }
      j -= n;
    }
  }
}

// Rebuilding the history from the cells (enable, load, put, fill): a cell of
// age a < L (a = (act - v) mod 2k, its epochs since the last set) is marked in
// the ring slot of epoch e - a; the sentinel and older cells are not.  A value
// above 2k (hand-made snapshots only) has no history: flagged, and the pool
// stays in the direct form.
template <typename T>
__global__ void k_bp_history(const T* __restrict__ cells, Layout L, uint32_t bact0,
                             uint32_t* __restrict__ ring, uint32_t R, int64_t e, uint32_t W,
                             uint64_t nwords, unsigned long long* bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += stride) {
    const uint64_t i0 = w * 32;
    const uint32_t cnt = (uint32_t)umin64(32, L.size - i0);
    for_word_clocks(i0, cnt, L, bact0, [&](uint32_t j, uint32_t act) {
      const uint32_t v = cells[i0 + j];
      if (v == L.B) return;
      if (v > L.B) {
        *bad = 1;
        return;
      }
      const uint32_t a = (act + L.B - v) % L.B;
      if (a < W) atomicOr(ring + (uint64_t)slot_of_epoch(e - (int64_t)a, R) * nwords + w, 1u << j);
    });
  }
}

// Bring cells up to date: for each word in [w_lo, w_hi) and each AT block it
// holds inside [s, e_): apply the block's pending epochs (applied[b], e_hi]
// newest first (a cell takes the clock of its newest marking epoch), then,
// with rule >= 0, the sweep of that due range (rule 0: clock 0, v <= k stale;
// rule 1: clock k, k <= v <= 2k-1 or v == 0 stale), counting cleared cells.
template <typename T>
__global__ void __launch_bounds__(256) k_bp_apply(T* __restrict__ cells, Layout L,
                                                  const uint32_t* __restrict__ ring, uint32_t R,
                                                  uint64_t nwords, int64_t e_hi, uint32_t bact0_hi,
                                                  const int64_t* __restrict__ applied,
                                                  uint64_t s, uint64_t e_, int rule,
                                                  unsigned long long* cleared) {
  constexpr int NV = (int)sizeof(T) * 2;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t w_lo = s / 32, w_hi = (e_ + 31) / 32;
  unsigned local = 0;
  for (uint64_t w = w_lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < w_hi; w += stride) {
    const uint64_t i0 = w * 32;
    const uint32_t cnt = (uint32_t)umin64(32, L.size - i0);
    const bool regs = sizeof(T) <= 2 && cnt == 32;
    uint4 r[NV];
    if (regs) {
#pragma unroll
      for (int v = 0; v < NV; ++v) r[v] = reinterpret_cast<const uint4*>(cells + i0)[v];
    }
    unsigned chg = 0;
    uint64_t seg = i0 > s ? i0 : s;
    const uint64_t word_end = umin64(i0 + cnt, e_);
    uint32_t b = block_of(seg, L);
    while (seg < word_end) {
      const uint64_t seg_end = umin64(block_start(b + 1, L), word_end);
      const uint32_t rm = range_bits(i0, seg, seg_end);
      const int64_t ap = applied[b];
      uint32_t acc = 0;
      int64_t ep = e_hi;
      uint32_t slot = slot_of_epoch(ep, R);
      while (ep > ap && acc != rm) {
        uint32_t v[8];
        const int n = (int)((ep - ap) >= 8 ? 8 : (ep - ap));
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (u < n) {
            v[u] = __ldcg(ring + (uint64_t)slot * nwords + w);
            slot = slot ? slot - 1 : R - 1;
          }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (u >= n) break;
          const uint32_t m = v[u] & rm & ~acc;
          if (m) {
            const uint32_t clk = clock_at(bact0_hi, e_hi, ep - u, b, L.B);
            if constexpr (sizeof(T) <= 2) {
              if (regs) {
                chg |= apply_marks_regs<T>(r, m, clk);
              } else {
                for (uint32_t j = 0; j < cnt; ++j)
                  if ((m >> j) & 1u) cells[i0 + j] = (T)clk;
              }
            } else {
              for (uint32_t j = 0; j < cnt; ++j)
                if ((m >> j) & 1u) cells[i0 + j] = (T)clk;
            }
            acc |= m;
          }
        }
        ep -= n;
      }
      if (rule >= 0) {
        SweepSpec SW{0, 0, 0, 0, L.k, L.B, cleared};
        if (rule == 0) { SW.s0 = seg; SW.e0 = seg_end; }
        else { SW.s1 = seg; SW.e1 = seg_end; }
        if constexpr (sizeof(T) <= 2) {
          if (regs) local += sweep_regs<T>(r, i0, SW, chg);
          else local += sweep_word(cells, i0, cnt, SW.s0, SW.e0, SW.s1, SW.e1, SW.k, SW.B);
        } else {
          local += sweep_word(cells, i0, cnt, SW.s0, SW.e0, SW.s1, SW.e1, SW.k, SW.B);
        }
      }
      seg = seg_end;
      ++b;
    }
    if constexpr (sizeof(T) <= 2) {
      if (regs && chg) store_sectors<T>(cells, i0, r, chg);
    }
  }
  if (rule >= 0) {
    local = __reduce_add_sync(0xffffffffu, local);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(cleared, (unsigned long long)local);
  }
}

// The due blocks at an advance, in two kernels with parallelism over epochs:
//  groups: one thread per (16-epoch group, word): which cells of the word were
//    marked in the group (acc) and, per cell, the offset of its newest marking
//    epoch in the group as four bit planes -- 16 independent loads per thread;
//  resolve: one thread per word: the newest group that marked each cell gives
//    its epoch, hence its clock (pools.py:164-178); then the sweep rule
//    (pools.py:221-249) and the whole word back to HBM.
constexpr int kGroup = 16;
struct DueRange {
  uint64_t s, e;      // cell range (one AT block)
  int64_t ap;         // epochs <= ap are already in its cells
  uint32_t b;         // the block
  int rule;           // 0: clock-0 sweep, 1: clock-k sweep
};

__global__ void __launch_bounds__(256) k_bp_groups(const uint32_t* __restrict__ ring, uint32_t R,
                                                   uint64_t nwords, DueRange r0, DueRange r1,
                                                   int64_t e_hi, uint32_t* __restrict__ acc_out,
                                                   uint4* __restrict__ planes_out,
                                                   uint64_t wstride, uint32_t gstride) {
  // grid: x over the range's words, y over 16-epoch groups, z over the two ranges
  const DueRange D = blockIdx.z ? r1 : r0;
  const uint64_t w0 = D.s / 32, W = (D.e + 31) / 32 - w0;
  const int64_t npend = e_hi - D.ap;
  const uint32_t g = blockIdx.y;
  if (npend <= (int64_t)g * kGroup) return;
  const int64_t newest = e_hi - (int64_t)g * kGroup;
  const int n = (int)((npend - (int64_t)g * kGroup) < kGroup ? (npend - (int64_t)g * kGroup) : kGroup);
  const uint32_t slot0 = slot_of_epoch(newest, R);  // one 64-bit modulo per thread
  for (uint64_t wi = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; wi < W;
       wi += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t v[kGroup];
    uint32_t slot = slot0;
#pragma unroll
    for (int u = 0; u < kGroup; ++u) {
      v[u] = u < n ? __ldcg(ring + (uint64_t)slot * nwords + w0 + wi) : 0u;
      slot = slot ? slot - 1 : R - 1;
    }
    uint32_t acc = 0, p0 = 0, p1 = 0, p2 = 0, p3 = 0;
#pragma unroll
    for (int u = 0; u < kGroup; ++u) {
      const uint32_t m = v[u] & ~acc;
      acc |= m;
      if (u & 1) p0 |= m;
      if (u & 2) p1 |= m;
      if (u & 4) p2 |= m;
      if (u & 8) p3 |= m;
    }
    const uint64_t o = ((uint64_t)blockIdx.z * gstride + g) * wstride + wi;
    acc_out[o] = acc;
    planes_out[o] = make_uint4(p0, p1, p2, p3);
  }
}

constexpr int kResolveThreads = 64;  // small CTAs: the few thousand words spread over every SM

template <typename T>
__global__ void __launch_bounds__(kResolveThreads) k_bp_resolve(T* __restrict__ cells, Layout L,
                                                    DueRange r0, DueRange r1, int range_base,
                                                    int64_t e_hi, uint32_t bact0_hi,
                                                    const uint32_t* __restrict__ acc_in,
                                                    const uint4* __restrict__ planes_in,
                                                    uint64_t wstride, uint32_t gstride,
                                                    unsigned long long* cleared) {
  constexpr int kChunk = 8;
  __shared__ uint32_t cs[kResolveThreads * 33];
  uint32_t* c = cs + threadIdx.x * 33;
  const int slot_y = range_base + (int)blockIdx.y;
  const DueRange D = slot_y ? r1 : r0;
  const uint64_t w0 = D.s / 32, W = (D.e + 31) / 32 - w0;
  const int64_t npend = e_hi - D.ap;
  const uint32_t G = npend > 0 ? (uint32_t)((npend + kGroup - 1) / kGroup) : 0u;
  const uint32_t B = L.B, k = L.k;
  const uint32_t act_hi = (bact0_hi + D.b) % B;  // the block's clock at epoch e_hi
  unsigned local = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t wi = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; wi < W; wi += stride) {
    const uint64_t w = w0 + wi, i0 = w * 32;
    const uint32_t cnt = (uint32_t)umin64(32, L.size - i0);
    const uint32_t rm = range_bits(i0, D.s, D.e);
    if (cnt == 32 && sizeof(T) <= 2) {  // 32 or 64 bytes: vector loads
      constexpr int NV = (int)sizeof(T) * 2;
      uint4 r[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) r[v] = reinterpret_cast<const uint4*>(cells + i0)[v];
      const T* e = reinterpret_cast<const T*>(r);
#pragma unroll
      for (int j = 0; j < 32; ++j) c[j] = e[j];
    } else {
      for (uint32_t j = 0; j < cnt; ++j) c[j] = cells[i0 + j];
    }
    uint32_t done = 0;
    bool changed = false;
    for (uint32_t g0 = 0; g0 < G && done != rm; g0 += kChunk) {
      // the chunk's group masks at once, then (ALU only) the cells each group
      // is the newest for, then those groups' epoch planes at once
      uint32_t m[kChunk];
      uint4 pl[kChunk];
#pragma unroll
      for (int u = 0; u < kChunk; ++u)
        m[u] = g0 + u < G ? acc_in[((uint64_t)slot_y * gstride + g0 + u) * wstride + wi] : 0u;
#pragma unroll
      for (int u = 0; u < kChunk; ++u) {
        m[u] &= rm & ~done;
        done |= m[u];
      }
#pragma unroll
      for (int u = 0; u < kChunk; ++u)
        if (m[u]) pl[u] = planes_in[((uint64_t)slot_y * gstride + g0 + u) * wstride + wi];
#pragma unroll
      for (int u = 0; u < kChunk; ++u) {
        uint32_t mm = m[u];
        if (!mm) continue;
        changed = true;
        while (mm) {
          const int j = __ffs(mm) - 1;
          mm &= mm - 1;
          const uint32_t off = (g0 + u) * kGroup + ((pl[u].x >> j) & 1u) +
                               2u * ((pl[u].y >> j) & 1u) + 4u * ((pl[u].z >> j) & 1u) +
                               8u * ((pl[u].w >> j) & 1u);
          c[j] = (act_hi + B - off % B) % B;  // the clock of its newest marking epoch
        }
      }
    }
    // the sweep of this due range (k_sweep's rule, pools.py:236-248)
    for (uint32_t j = 0; j < cnt; ++j) {
      if (!((rm >> j) & 1u)) continue;
      const uint32_t v = c[j];
      const bool stale = D.rule == 0 ? v <= k : ((v >= k && v <= B - 1) || v == 0);
      if (stale) {
        c[j] = B;
        ++local;
        changed = true;
      }
    }
    if (changed) {
      if (cnt == 32 && sizeof(T) <= 2) {
        constexpr int NV = (int)sizeof(T) * 2;
        uint4 r[NV];
        T* e = reinterpret_cast<T*>(r);
#pragma unroll
        for (int j = 0; j < 32; ++j) e[j] = (T)c[j];
#pragma unroll
        for (int v = 0; v < NV; ++v) reinterpret_cast<uint4*>(cells + i0)[v] = r[v];
      } else {
        for (uint32_t j = 0; j < cnt; ++j) cells[i0 + j] = (T)c[j];
      }
    }
  }
  local = __reduce_add_sync(0xffffffffu, local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(cleared, (unsigned long long)local);
}

template <typename F>
static int with_cell_bp(int bytes, F f) {
  switch (bytes) {
    case 1: return f(uint8_t{});
    case 2: return f(uint16_t{});
    default: return f(uint32_t{});
  }
}

static uint64_t bp_nwords(const vate_pool* p) { return (p->L.size + 31) / 32; }

static uint32_t* ring_slot(vate_pool* p, int64_t e) {
  return p->bp_ring.as<uint32_t>() + (uint64_t)slot_of_epoch(e, p->bp_R) * bp_nwords(p);
}

static int bp_upload_applied(vate_pool* p) {
  VATE_CUDA(cudaMemcpyAsync(p->bp_applied.ptr, p->bp_applied_h.data(),
                            p->bp_applied_h.size() * sizeof(int64_t), cudaMemcpyHostToDevice,
                            p->stream));
  // the host vector may change before the copy runs: wait for it (off the hot path
  // callers only; the advance path uploads two entries the same way)
  VATE_CUDA(cudaStreamSynchronize(p->stream));
  return VATE_OK;
}

// S of the block [base, base + L) and P = 0 (the next block starts).
static int bp_block_boundary(vate_pool* p, int64_t base) {
  const uint64_t nwords = bp_nwords(p);
  if (p->bp_L > 1)
    VATE_LAUNCH(p, VATE_K_OTHER, grid_for(nwords, 256, 148u * 32u), 256, 0, k_bp_suffix,
                p->bp_ring.as<const uint32_t>(), p->bp_R, base, p->bp_L, p->bp_S.as<uint32_t>(),
                nwords);
  VATE_CUDA(cudaMemsetAsync(p->bp_P.ptr, 0, nwords * 4, p->stream));
  return VATE_OK;
}

}  // namespace vate

using namespace vate;

namespace vate {

uint32_t* pend_ptr(vate_pool* p) {
  return p->bp ? ring_slot(p, p->bp_e) : p->pend.as<uint32_t>();
}

// Rebuild ring, S and P from the (up-to-date) cells at a block start.
static int bp_history(vate_pool* p) {
  int rc0 = bp_wait_aux(p);
  if (rc0) return rc0;
  const uint64_t nwords = bp_nwords(p);
  // a fresh block: e is a multiple of L; the previous block is epochs e-L .. e-1
  p->bp_e = (int64_t)p->bp_R * p->bp_L * 4;
  VATE_CUDA(cudaMemsetAsync(p->bp_ring.ptr, 0, p->bp_ring.bytes, p->stream));
  VATE_CUDA(cudaMemsetAsync(p->d_ctr + C_TRACE, 0, 8, p->stream));
  rc0 = with_cell_bp(p->cell_bytes, [&](auto tag) -> int {
    using T = decltype(tag);
    VATE_LAUNCH(p, VATE_K_OTHER, grid_for(nwords, 256, 148u * 32u), 256, 0, k_bp_history<T>,
                (const T*)p->cells, p->L, p->bact0, p->bp_ring.as<uint32_t>(), p->bp_R, p->bp_e,
                p->bp_L, nwords, p->d_ctr + C_TRACE);
    return VATE_OK;
  });
  if (rc0) return rc0;
  int rc = bp_block_boundary(p, p->bp_e - (int64_t)p->bp_L);
  if (rc) return rc;
  unsigned long long bad = 0;
  VATE_CUDA(cudaMemcpyAsync(&bad, p->d_ctr + C_TRACE, 8, cudaMemcpyDeviceToHost, p->stream));
  VATE_CUDA(cudaStreamSynchronize(p->stream));
  if (bad) return 1;  // values above 2k: no history
  p->bp_applied_h.assign(p->L.B, p->bp_e - 1);
  rc = bp_upload_applied(p);
  if (rc) return rc;
  p->bp_folded = false;
  p->bp_flushed_e = p->bp_e;
  p->pend_dirty = false;
  return VATE_OK;
}

static void bp_free(vate_pool* p) {
  p->bp_acc.release();
  p->bp_planes.release();
  p->bp_ring.release();
  p->bp_S.release();
  p->bp_P.release();
  p->bp_applied.release();
  p->bp = false;
}

int bp_maybe_enable(vate_pool* p, int k_prime) {
  if (p->bp || p->bp_failed || p->kind != VATE_AT) return VATE_OK;
  if (p->opt_bp == 0 || (p->opt_bp == -1 && !p->deferred)) return VATE_OK;
  if (p->adv_pending) return VATE_OK;  // enable between advances only
  int rc = p->deferred ? VATE_OK : set_deferred(p, true);  // scans must mark
  if (rc) return rc;
  rc = flush_pending(p);  // the deferred marks into the cells first
  if (rc) return rc;
  const uint64_t nwords = bp_nwords(p);
  p->bp_L = (uint32_t)k_prime;
  p->bp_R = (uint32_t)p->k + p->bp_L + 1;
  const uint64_t need = ((uint64_t)p->bp_R + p->bp_L + 1) * nwords * 4;
  size_t free_b = 0, total_b = 0;
  VATE_CUDA(cudaMemGetInfo(&free_b, &total_b));
  if (need + (4ull << 30) > free_b) {  // keep 4 GiB of headroom
    p->bp_failed = true;
    return VATE_OK;
  }
  // scratch of the due-block kernels: per range, groups x words of a block
  uint64_t wmax = 0;
  for (uint32_t b = 0; b < p->L.B; ++b)
    wmax = std::max<uint64_t>(wmax, (block_start(b + 1, p->L) - block_start(b, p->L) + 63) / 32);
  p->bp_wmax = wmax;
  p->bp_gmax = (p->bp_R + kGroup - 1) / kGroup;
  if (p->bp_acc.ensure(2ull * p->bp_gmax * wmax * 4) ||
      p->bp_planes.ensure(2ull * p->bp_gmax * wmax * 16) ||
      p->bp_ring.ensure((uint64_t)p->bp_R * nwords * 4) ||
      p->bp_S.ensure((uint64_t)std::max<uint32_t>(p->bp_L, 2) * nwords * 4) ||
      p->bp_P.ensure(nwords * 4) || p->bp_applied.ensure(p->L.B * sizeof(int64_t))) {
    bp_free(p);
    p->bp_failed = true;
    set_error(VATE_OK, "");
    return VATE_OK;
  }
  rc = bp_history(p);
  if (rc == 1) {  // hand-made values: stay direct
    bp_free(p);
    p->bp_failed = true;
    return VATE_OK;
  }
  if (rc) return rc;
  p->bp = true;
  return VATE_OK;
}

int bp_wait_aux(vate_pool* p) {
  if (!p->bp_join) return VATE_OK;
  VATE_CUDA(cudaStreamWaitEvent(p->stream, p->ev_bp, 0));
  p->bp_join = false;
  return VATE_OK;
}

int bp_materialize_all(vate_pool* p) {
  if (!p->bp) return VATE_OK;
  int rc0 = bp_wait_aux(p);
  if (rc0) return rc0;
  if (p->bp_flushed_e == p->bp_e && !p->pend_dirty) return VATE_OK;
  int rc = bp_upload_applied(p);
  if (rc) return rc;
  const uint64_t nwords = bp_nwords(p);
  rc = with_cell_bp(p->cell_bytes, [&](auto tag) -> int {
    using T = decltype(tag);
    VATE_LAUNCH(p, VATE_K_OTHER, grid_for(nwords, 256, 148u * 32u), 256, 0, k_bp_apply<T>,
                (T*)p->cells, p->L, p->bp_ring.as<const uint32_t>(), p->bp_R, nwords, p->bp_e,
                p->bact0, p->bp_applied.as<const int64_t>(), 0ull, p->L.size, -1, nullptr);
    return VATE_OK;
  });
  if (rc) return rc;
  // epoch e may still receive marks: everything through e-1 is now in the cells
  for (auto& a : p->bp_applied_h) a = std::max(a, p->bp_e - 1);
  p->bp_flushed_e = p->bp_e;
  p->pend_dirty = false;
  return bp_upload_applied(p);
}

int bp_disable(vate_pool* p) {
  if (!p->bp) return VATE_OK;
  int rc = bp_materialize_all(p);
  if (rc) return rc;
  VATE_CUDA(cudaStreamSynchronize(p->stream));
  bp_free(p);
  // back to the deferred form: its pending-set bitmap starts empty
  if (p->deferred) {
    const uint64_t bytes = bp_nwords(p) * 4;
    rc = p->pend.ensure(bytes);
    if (rc) return rc;
    VATE_CUDA(cudaMemsetAsync(p->pend.ptr, 0, bytes, p->stream));
  }
  p->pend_dirty = false;
  return VATE_OK;
}

int bp_rebuild(vate_pool* p) {
  if (!p->bp) return VATE_OK;
  int rc = bp_history(p);
  if (rc == 1) {  // the new contents have no history: leave bit-plane mode
    bp_free(p);
    p->bp_failed = true;
    if (p->deferred) {
      const uint64_t bytes = bp_nwords(p) * 4;
      rc = p->pend.ensure(bytes);
      if (rc) return rc;
      VATE_CUDA(cudaMemsetAsync(p->pend.ptr, 0, bytes, p->stream));
    }
    return VATE_OK;
  }
  return rc;
}

static int bp_due(vate_pool* p);
static int bp_next_epoch(vate_pool* p);

int bp_window(vate_pool* p, int k_prime, bool with_delta, bool fused_advance) {
  (void)k_prime;
  const uint64_t nwords = bp_nwords(p);
  int rc = p->bitmap.ensure(nwords * 4 + 16);
  if (rc) return rc;
  VATE_CUDA(cudaMemsetAsync(p->d_ctr + C_P, 0, 8, p->stream));
  DeltaOut D{};
  if (with_delta) {
    IncIndex& I = p->inc;
    VATE_CUDA(cudaMemsetAsync(p->d_ctr + C_DCNT, 0, 16, p->stream));
    D = DeltaOut{I.bprev.as<const uint32_t>(), I.off.as<const uint32_t>(),
                 I.dlist.as<unsigned long long>(), I.dlist_cap, p->d_ctr + C_DCNT,
                 p->d_ctr + C_DWORK};
  }
  const Publish pub{p->d_done, p->d_ctr, p->h_ctr_dev,
                    (1u << C_P) | (with_delta ? (1u << C_DCNT) | (1u << C_DWORK) : 0u)};
  const uint32_t j = (uint32_t)(p->bp_e % (int64_t)p->bp_L);
  const uint32_t* S = (j + 1 <= p->bp_L - 1) ? p->bp_S.as<const uint32_t>() + (uint64_t)j * nwords
                                             : nullptr;  // S[j+1] at index j
  const bool fold = fused_advance && !p->bp_folded;
  const uint32_t* M = pend_ptr(p);
  // the due blocks of the advance, on their own stream (forked from main)
  auto launch_due = [&]() -> int {
    // the due blocks on the aux stream beside the window pass (they read only
    // ring slots up to this epoch and write only cells, which the pass does
    // not touch); bp_wait_aux orders every later cell access after them.
    // cfg 4: 0.183 -> 0.169 ms per slice (profiles/r02l_ab_bp_aux.txt); beside
    // the next slice's scan instead they slowed both down (0.240 -> 0.268; again
    // at the L2-hint scan: 0.136 -> 0.172, profiles/r02g_ab_due_late.txt)
    if (p->adv_pending) return set_error(VATE_EVALUE, "previous advance not collected");
    if (!p->ev_bp) VATE_CUDA(cudaEventCreateWithFlags(&p->ev_bp, cudaEventDisableTiming));
    if (!p->ev_bp_fork) VATE_CUDA(cudaEventCreateWithFlags(&p->ev_bp_fork, cudaEventDisableTiming));
    if (!p->bp_stream) VATE_CUDA(cudaStreamCreateWithFlags(&p->bp_stream, cudaStreamNonBlocking));
    // their own stream: they start with the pass instead of queueing behind the
    // registry compaction on aux, so the advance result (which the next call
    // waits for) lands early
    VATE_CUDA(cudaEventRecord(p->ev_bp_fork, p->stream));
    VATE_CUDA(cudaStreamWaitEvent(p->bp_stream, p->ev_bp_fork, 0));
    cudaStream_t main_stream = p->stream;
    p->stream = p->bp_stream;
    rc = bp_due(p);
    if (rc == VATE_OK) {
      const cudaError_t ce = cudaEventRecord(p->ev_bp, p->stream);
      if (ce != cudaSuccess) rc = cuda_fail(ce, "bit-plane advance");
    }
    p->stream = main_stream;
    if (rc) return rc;
    p->bp_join = true;
    return VATE_OK;
  };
  if (fused_advance) {
    rc = launch_due();
    if (rc) return rc;
  }
  // evict-first stores: the registry and the marks stay in L2 for the next scan
  // 4 CTAs per SM, looping: the pass takes the same 47 us with 4 or 64, and the
  // due blocks and the registry compaction beside it get the SM room (cfg 4:
  // 0.149 -> 0.143 ms per slice, profiles/r02m_ab_window_grid.txt)
  VATE_LAUNCH(p, VATE_K_BITMAP, grid_for((nwords + 3) / 4, 256, 148u * 4u), 256, 0,
              k_bp_window<true>, S, p->bp_P.as<const uint32_t>(), M,
              fold ? p->bp_P.as<uint32_t>() : nullptr, p->bitmap.as<uint32_t>(), nwords,
              p->L.size, p->d_ctr + C_P, D, pub);
  if (fold) p->bp_folded = true;
  if (fused_advance) return bp_next_epoch(p);
  return VATE_OK;
}

// AtPool.advance_slice (pools.py:221-249) in bit-plane mode: fold the epoch's
// marks into P, advance the clock, bring the two due blocks up to date and
// sweep them, open the next epoch (its ring slot cleared) and, at a block
// boundary, build the suffix ORs.  The result is collected with
// vate_advance_result like the direct advance.
int bp_advance(vate_pool* p) {
  if (p->adv_pending) return set_error(VATE_EVALUE, "previous advance not collected");
  const uint64_t nwords = bp_nwords(p);
  if (!p->bp_folded)
    VATE_LAUNCH(p, VATE_K_OTHER, grid_for(nwords, 256, 148u * 16u), 256, 0, k_bp_fold,
                p->bp_P.as<uint32_t>(), pend_ptr(p), nwords);
  int rc = bp_due(p);
  if (rc) return rc;
  return bp_next_epoch(p);
}

// The clock advance and the two due blocks (their kernels on p->stream).
static int bp_due(vate_pool* p) {
  const uint64_t nwords = bp_nwords(p);
  const uint32_t B = p->L.B, k = p->L.k;
  const uint32_t old_bact0 = p->bact0;
  p->bact0 = (p->bact0 + 1) % B;  // pools.py:228
  const uint32_t z = (B - p->bact0) % B, q = (k + B - p->bact0) % B;  // pools.py:231-232
  const uint64_t s0 = block_start(z, p->L), e0 = block_start(z + 1, p->L);
  const uint64_t s1 = block_start(q, p->L), e1 = block_start(q + 1, p->L);
  p->adv_blocks[0] = (int32_t)z;
  p->adv_blocks[1] = (int32_t)q;
  p->adv_maint = (e0 - s0) + (e1 - s1);
  VATE_CUDA(cudaMemsetAsync(p->d_ctr + C_CLEARED, 0, 8, p->stream));
  // the due blocks' pending epochs (applied[b], e]: newest marking epoch per
  // cell by 16-epoch groups, then clocks and the sweep rule per range
  const int64_t e = p->bp_e;
  const DueRange r0{s0, e0, p->bp_applied_h[z], z, 0}, r1{s1, e1, p->bp_applied_h[q], q, 1};
  const uint64_t wstride = p->bp_wmax;
  const uint32_t gstride = p->bp_gmax;
  if ((uint64_t)((e - std::min(r0.ap, r1.ap) + kGroup - 1) / kGroup) > gstride ||
      (e0 - s0 + 63) / 32 > wstride || (e1 - s1 + 63) / 32 > wstride)
    return set_error(VATE_EVALUE, "bit-plane advance: a due block is further behind than the ring");
  const uint32_t gmax = (uint32_t)((e - std::min(r0.ap, r1.ap) + kGroup - 1) / kGroup);
  const uint64_t wmax = std::max((e0 + 31) / 32 - s0 / 32, (e1 + 31) / 32 - s1 / 32);
  VATE_LAUNCH(p, VATE_K_SWEEP, dim3(grid_for(wmax, 256, 148u * 4u), std::max(gmax, 1u), 2), 256, 0,
              k_bp_groups,
              p->bp_ring.as<const uint32_t>(), p->bp_R, nwords, r0, r1, e,
              p->bp_acc.as<uint32_t>(), p->bp_planes.as<uint4>(), wstride, gstride);
  int rc = with_cell_bp(p->cell_bytes, [&](auto tag) -> int {
    using T = decltype(tag);
    const uint64_t nw = std::max((e0 + 31) / 32 - s0 / 32, (e1 + 31) / 32 - s1 / 32);
    // both ranges in one launch unless they share a word (adjacent blocks: k = 1)
    const bool share = (e0 + 31) / 32 > s1 / 32 && (e1 + 31) / 32 > s0 / 32;
    for (int r = 0; r < (share ? 2 : 1); ++r)
      VATE_LAUNCH(p, VATE_K_SWEEP, dim3(grid_for(nw, kResolveThreads, 148u * 32u), share ? 1 : 2),
                  kResolveThreads, 0, k_bp_resolve<T>, (T*)p->cells, p->L, r0, r1, r, e, old_bact0,
                  p->bp_acc.as<const uint32_t>(), p->bp_planes.as<const uint4>(), wstride,
                  gstride, p->d_ctr + C_CLEARED);
    return VATE_OK;
  });
  if (rc == VATE_OK) {
    // the two blocks now hold every epoch through e (the host mirror; the device
    // copy is uploaded before its one reader, bp_materialize_all)
    p->bp_applied_h[z] = e;
    p->bp_applied_h[q] = e;
    cudaError_t ce = cudaMemcpyAsync(p->h_ctr + C_CLEARED, p->d_ctr + C_CLEARED, 8,
                                     cudaMemcpyDeviceToHost, p->stream);
    if (ce == cudaSuccess) ce = cudaEventRecord(p->ev_adv, p->stream);
    if (ce != cudaSuccess) rc = cuda_fail(ce, "bit-plane advance");
  }
  return rc;
}

// Open the next epoch: its ring slot (held epoch e + 1 - R, past every use)
// emptied; at a block boundary the suffix ORs of the finished block.
static int bp_next_epoch(vate_pool* p) {
  const uint64_t nwords = bp_nwords(p);
  int rc = VATE_OK;
  p->bp_e = p->bp_e + 1;
  p->bp_folded = false;
  VATE_CUDA(cudaMemsetAsync(ring_slot(p, p->bp_e), 0, nwords * 4, p->stream));
  if (p->bp_e % (int64_t)p->bp_L == 0) {
    rc = bp_block_boundary(p, p->bp_e - (int64_t)p->bp_L);
    if (rc) return rc;
  }
  p->adv_pending = true;
  p->sweeps_fused++;
  return VATE_OK;
}

}  // namespace vate

extern "C" int vate_pool_mode(const vate_pool* p, int32_t out[5]) {
  if (!p || !out) return set_error(VATE_EVALUE, "null argument");
  out[0] = p->deferred ? 1 : 0;
  out[1] = p->bp ? 1 : 0;
  out[2] = (int32_t)p->bp_L;
  out[3] = (int32_t)p->bp_R;
  out[4] = p->scan_form_used;
  return VATE_OK;
}
