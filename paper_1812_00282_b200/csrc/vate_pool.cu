// vate_pool.cu -- the AT pool on the device: lifecycle, ingest scan,
// two-block maintenance, whole-pool inactive bitmap / count, point queries,
// ATP1 snapshots, replica merge and the synthetic packet generator.
//
// Reference: pools.py:67-298 (AtPool), estimator.py:96-104 (pair_cells /
// record_pairs), bitpack.py:26-140 (the snapshot bit layout).
#include <cuda_profiler_api.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>

#include "vate_internal.cuh"
#include "vate_registry.cuh"
#include "vate_cells.cuh"

namespace vate {

// ---------------------------------------------------------------------------
// error plumbing, staging, timing
// ---------------------------------------------------------------------------

static thread_local std::string g_err;
thread_local unsigned long long g_api_calls = 0;

int set_error(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  // consume the runtime's last-error state: a non-sticky failure (a bad device
  // ordinal, a failed allocation) must not resurface at the next launch check
  (void)cudaGetLastError();
  return set_error(e == cudaErrorMemoryAllocation ? VATE_ENOMEM : VATE_ECUDA,
                   std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

int DevBuf::ensure(size_t want) {
  if (want <= bytes && ptr) return VATE_OK;
  size_t grow = std::max<size_t>(want, bytes + bytes / 2);
  grow = (grow + 255) & ~size_t(255);
  if (ptr) {
    cudaError_t e = cudaFree(ptr);  // device-synchronising: safe for in-flight work
    ptr = nullptr;
    bytes = 0;
    if (e != cudaSuccess) return cuda_fail(e, "cudaFree");
  }
  cudaError_t e = cudaMalloc(&ptr, grow);
  if (e != cudaSuccess) {
    ptr = nullptr;
    return cuda_fail(e, "cudaMalloc");
  }
  bytes = grow;
  return VATE_OK;
}

void DevBuf::release() {
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  bytes = 0;
}

int enter(vate_pool* p) {
  if (!p) return set_error(VATE_EVALUE, "null pool handle");
  VATE_CUDA(cudaSetDevice(p->device));
  return VATE_OK;
}

int stage_in(vate_pool* p, DevBuf& buf, const void* src, size_t bytes, int where,
             const void** dev) {
  if (where == VATE_DEVICE || bytes == 0) {
    *dev = src;
    return VATE_OK;
  }
  int rc = buf.ensure(bytes);
  if (rc) return rc;
  VATE_CUDA(cudaMemcpyAsync(buf.ptr, src, bytes, cudaMemcpyHostToDevice, p->stream));
  *dev = buf.ptr;
  return VATE_OK;
}

// The host round trip of a slice.  (Spinning on a mapped flag stored by a
// one-thread kernel was measured slower than the driver's wait and removed.)
static int wait_stream(vate_pool* p) {
  VATE_CUDA(cudaStreamSynchronize(p->stream));
  return VATE_OK;
}

int sync_small(vate_pool* p) {
  int wrc = wait_stream(p);
  if (wrc) return wrc;
  if (p->h_ctr && p->h_ctr[C_ERR]) {
    p->h_ctr[C_ERR] = 0;
    return set_error(VATE_EVALUE, "cell index outside the pool");
  }
  return VATE_OK;
}

static cudaEvent_t take_event(vate_pool* p) {
  if (!p->event_pool.empty()) {
    cudaEvent_t e = p->event_pool.back();
    p->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

void timing_begin(vate_pool* p, int kind, cudaEvent_t* a) {
  (void)kind;
  if (!p->timing) return;
  *a = take_event(p);
  cudaEventRecord(*a, p->stream);
}

void timing_end(vate_pool* p, int kind, cudaEvent_t a) {
  if (!p->timing || !a) return;
  cudaEvent_t b = take_event(p);
  cudaEventRecord(b, p->stream);
  p->timed_pending.push_back({kind, a, b});
}

int collect_timing(vate_pool* p) {
  if (p->timed_pending.empty()) return VATE_OK;
  VATE_CUDA(cudaStreamSynchronize(p->stream));
  if (p->aux_stream) VATE_CUDA(cudaStreamSynchronize(p->aux_stream));
  for (auto& t : p->timed_pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t.a, t.b);
    p->timed_ms[t.kind] += ms;
    p->timed_n[t.kind] += 1;
    if (p->timeline_ref && p->timeline.size() < 3 * 65536) {  // (kind, start, end) in ms
      float s0 = 0.f, s1 = 0.f;
      cudaEventElapsedTime(&s0, p->timeline_ref, t.a);
      cudaEventElapsedTime(&s1, p->timeline_ref, t.b);
      p->timeline.push_back((double)t.kind);
      p->timeline.push_back(s0);
      p->timeline.push_back(s1);
    }
    p->event_pool.push_back(t.a);
    p->event_pool.push_back(t.b);
  }
  p->timed_pending.clear();
  return VATE_OK;
}

uint32_t grid_for(uint64_t work, uint32_t per_block, uint32_t cap_blocks) {
  uint64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap_blocks) g = cap_blocks;
  return (uint32_t)g;
}

template <typename F>
static int with_cell(int bytes, F f) {
  switch (bytes) {
    case 1: return f(uint8_t{});
    case 2: return f(uint16_t{});
    default: return f(uint32_t{});
  }
}

// Cell type and store rule of a pool: AT stores its block clock; the DR / TS
// comparators store a constant per slice (0, or the slice index).
// A deferred AT pool marks the pending-set bitmap instead (MarkRule).
// L2 evict_last on the scan's registry and mark accesses (VATE_OPT_L2_KEEP):
// auto = deferred pools, whose slice also streams the bit-plane / cell passes
// through L2 between two scans.  No persisting set-aside is configured: with
// 16-96 MB set aside the window pass lost L2 room and the slice slowed (cfg 4
// 0.137 -> 0.142-0.191 ms); the bare hint keeps the scan's DRAM write-back at
// 17 vs 60 MB per launch and the slice 1.5 % faster (profiles/r02y_ab_l2keep.txt)
static int l2_keep(const vate_pool* p) {
  return p->opt_l2_keep == 1 || (p->opt_l2_keep == -1 && p->deferred) ? 1 : 0;
}

template <typename F>
static int with_store(vate_pool* p, F f) {
  if (p->kind == VATE_AT && p->deferred) {
    p->pend_dirty = true;
    return with_cell(p->cell_bytes,
                     [&](auto tag) { return f(tag, MarkRule{pend_ptr(p), l2_keep(p)}); });
  }
  if (p->kind == VATE_AT)
    return with_cell(p->cell_bytes, [&](auto tag) { return f(tag, AtRule{p->L, p->bact0}); });
  const ConstRule r{p->kind == VATE_DR ? 0ull : p->ts_now};
  if (p->kind == VATE_TS) return f(uint64_t{}, r);
  if (p->cell_bytes == 1) return f(uint8_t{}, r);
  return f(uint16_t{}, r);
}

__device__ __forceinline__ unsigned block_sum(unsigned v) {
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

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------

template <typename T>
__global__ void k_fill(T* cells, uint64_t n, T value) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    cells[i] = value;
}

// A batch of U packets per thread: BH, H, then the cell write (pools.py:153-178
// with estimator.py:96-99), then the host-registry touch.  Same-cell writers
// of a slice store the same clock, so plain stores suffice -- no atomics, no
// read-modify-write.  A deferred pool (MarkRule: cells beyond L2) instead
// sets the cell's bit in the L2-resident pending-set bitmap (one red.or) and
// the next pool pass writes the clock (store_cell).  The registry step issues
// all U first-probe loads (one 32-byte sector each) before resolving any, so
// a thread keeps U independent requests in flight; only misses take the
// probing insert.
// FILTER (skewed traffic): registry stamps are filtered per CTA by a small
// direct-mapped table of the slots this CTA already stamped with t in shared
// memory.  Loads of `last` come from L1 and are stale within a launch, so
// without it every packet of a heavy hitter would store into the same 8 bytes
// -- hundreds of thousands of same-address stores serialised at one L2 slice
// (cfg 3's Zipf head).
constexpr int kTouchSlots = 1024;

__device__ __forceinline__ void touch_filter_init(unsigned* filt) {
  for (int i = threadIdx.x; i < kTouchSlots; i += blockDim.x) filt[i] = 0u;
  __syncthreads();
}

__device__ __forceinline__ void touch_last(const RegRef& R, unsigned* filt, uint64_t slot,
                                           long long t) {
  const unsigned tag = (unsigned)slot + 1u;
  // one shared-memory exchange: exactly one thread of a racing group sees a
  // different previous tag and stamps (race-free under compute-sanitizer)
  if (atomicExch(filt + (slot & (kTouchSlots - 1)), tag) == tag) return;
  reg_stamp(R, slot, t);
}

// Registry misses of the home sector are deferred to a per-CTA shared-memory
// queue and inserted after the CTA's packets, by dense threads: in-line, a
// warp would run the probe loop as long as its slowest of 64 packets.
// A key is queued with bit 0 of `skip` set when the home sector held two other
// keys (the walk resumes at the next sector) -- the common case; a home
// sector with an empty slot means a new key, inserted from the home sector.
constexpr int kDeferCap = 1024;
struct DeferQ {
  unsigned long long keys[kDeferCap];
  unsigned char skip[kDeferCap];
  unsigned n;
};

__device__ __forceinline__ void defer_init(DeferQ* dq) {
  if (threadIdx.x == 0) dq->n = 0;
}

__device__ __forceinline__ void defer_drain(DeferQ* dq, const RegRef& R, long long t) {
  __syncthreads();
  const unsigned n = min(dq->n, (unsigned)kDeferCap);
  for (unsigned i = threadIdx.x; i < n; i += blockDim.x)
    reg_insert(R, dq->keys[i], t, false, dq->skip[i] != 0);
}

template <typename T, bool REG, int U, bool FILTER, typename Rule>
__device__ __forceinline__ void scan_batch(const uint64_t (&aip)[U], const uint64_t (&bip)[U],
                                           int m, T* __restrict__ cells, const HashParams& H,
                                           const Rule& rule, const RegRef& R, long long t,
                                           unsigned* filt, DeferQ* dq = nullptr) {
#pragma unroll
  for (int q = 0; q < U; ++q)
    if (q < m) store_cell<T, FILTER>(cells, cell_of(aip[q], slot_of(bip[q], H), H), rule);
  if (REG) {
    // all U first probes in flight before any is resolved: each reads the home
    // sector (two slots, one 256-bit load)
    uint64_t slot[U];
    RegEntry e[U], f[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      slot[q] = reg_home(aip[q], R.mask);
      if (q < m) ld_pair(R.table + slot[q], e[q], f[q], R.l2_keep);
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      if (q >= m) continue;
      if (aip[q] != kEmptyKey && e[q].key == aip[q]) {
        if (e[q].last != t) {
          if (FILTER) touch_last(R, filt, slot[q], t);
          else reg_stamp(R, slot[q], t);
        }
      } else if (aip[q] != kEmptyKey && f[q].key == aip[q]) {
        if (f[q].last != t) {
          if (FILTER) touch_last(R, filt, slot[q] + 1, t);
          else reg_stamp(R, slot[q] + 1, t);
        }
      } else {
        if (dq) {
          const unsigned pos = atomicAdd(&dq->n, 1u);
          if (pos < (unsigned)kDeferCap) {
            dq->keys[pos] = aip[q];
            dq->skip[pos] = (aip[q] != kEmptyKey && e[q].key != kEmptyKey && f[q].key != kEmptyKey);
            continue;
          }
        }
        reg_insert(R, aip[q], t, false);
      }
    }
  }
}

// The packed scan: one uint4 (two 8-byte packets) per thread per iteration,
// 8 CTAs per SM at <= 32 registers (measured best on cfg 2/3/4 against one
// packet, two or four uint4 per thread, and a TMA-fed persistent form).
template <typename T, bool REG, bool FILTER, typename Rule>
__global__ void __launch_bounds__(kThreads, 8) k_scan_packed16(
    const uint4* __restrict__ pairs2, uint64_t npairs2, T* __restrict__ cells, HashParams H,
    Rule rule, RegRef R, long long t) {
  __shared__ unsigned filt[REG && FILTER ? kTouchSlots : 1];
  __shared__ __align__(16) unsigned char dq_raw[REG ? sizeof(DeferQ) : 16];
  DeferQ* dq = REG ? reinterpret_cast<DeferQ*>(dq_raw) : nullptr;
  if (REG) defer_init(dq);
  if (REG && FILTER) touch_filter_init(filt);  // (its barrier also publishes dq->n = 0)
  else if (REG) __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < npairs2; i += stride) {
    const uint4 q = __ldcs(pairs2 + i);  // streamed once: evict-first
    const uint64_t a[2] = {q.x, q.z}, b[2] = {q.y, q.w};
    scan_batch<T, REG, 2, FILTER>(a, b, 2, cells, H, rule, R, t, filt, dq);
  }
  if (REG) defer_drain(dq, R, t);
}

// One 8-byte packet per thread: input that is not 16-byte aligned, and the odd
// last packet of a 16-byte aligned batch.
template <typename T, bool REG, bool FILTER, typename Rule>
__global__ void __launch_bounds__(kThreads) k_scan_packed8(
    const uint2* __restrict__ pairs, uint64_t n, T* __restrict__ cells, HashParams H,
    Rule rule, RegRef R, long long t) {
  __shared__ unsigned filt[REG && FILTER ? kTouchSlots : 1];
  __shared__ __align__(16) unsigned char dq_raw[REG ? sizeof(DeferQ) : 16];
  DeferQ* dq = REG ? reinterpret_cast<DeferQ*>(dq_raw) : nullptr;
  if (REG) defer_init(dq);
  if (REG && FILTER) touch_filter_init(filt);
  else if (REG) __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint2 q = __ldcs(pairs + i);  // streamed once: evict-first
    const uint64_t a[1] = {q.x}, b[1] = {q.y};
    scan_batch<T, REG, 1, FILTER>(a, b, 1, cells, H, rule, R, t, filt, dq);
  }
  if (REG) defer_drain(dq, R, t);
}

// The u64 form (record_pairs on u64 aips / bips, estimator.py:96-104).
template <typename T, bool REG, typename Rule>
__global__ void __launch_bounds__(kThreads) k_scan_u64(
    const uint64_t* __restrict__ aips, const uint64_t* __restrict__ bips, uint64_t n,
    T* __restrict__ cells, HashParams H, Rule rule, RegRef R, long long t) {
  constexpr int U = 4;
  unsigned* filt = nullptr;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += U * stride) {
    uint64_t a[U], b[U];
    int m = 0;
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const uint64_t j = i + q * stride;
      a[q] = b[q] = 0;
      if (j < n) {
        a[q] = __ldcs(aips + j);
        b[q] = __ldcs(bips + j);
        m = q + 1;
      }
    }
    scan_batch<T, REG, U, false>(a, b, m, cells, H, rule, R, t, filt);
  }
}

__global__ void k_pair_cells(const uint64_t* __restrict__ aips,
                             const uint64_t* __restrict__ bips, uint64_t n, HashParams H,
                             uint64_t* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = cell_of(aips[i], slot_of(bips[i], H), H);
}

__global__ void k_host_cells(const uint64_t* __restrict__ aips, uint64_t n, uint64_t g,
                             HashParams H, uint64_t* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n * g; i += stride)
    out[i] = cell_of(aips[i / g], i % g, H);
}

template <typename T, typename Rule>
__global__ void k_set_cells(const uint64_t* __restrict__ idx, uint64_t n, T* __restrict__ cells,
                            uint64_t size, Rule rule, unsigned long long* err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t c = idx[i];
    if (c >= size) {
      *err = 1;
      continue;
    }
    store_cell<T>(cells, c, rule);
  }
}

// Two due blocks after the clock advance (pools.py:221-249, counters.py:113-127):
// range 0 sits at clock 0 (stale: v <= k), range 1 at clock k (stale:
// k <= v <= 2k-1 or v == 0).  Stale cells become the sentinel 2k.
template <typename T>
__global__ void __launch_bounds__(kThreads) k_sweep(T* __restrict__ cells, uint64_t s0,
                                                    uint64_t n0, uint64_t s1, uint64_t n1,
                                                    uint32_t k, unsigned long long* cleared) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t total = n0 + n1;
  const uint32_t B = 2 * k;
  unsigned local = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
    const bool at_zero = i < n0;
    const uint64_t c = at_zero ? s0 + i : s1 + (i - n0);
    const uint32_t v = cells[c];
    const bool stale = at_zero ? (v <= k) : ((v >= k && v <= B - 1) || v == 0);
    if (stale) {
      cells[c] = (T)B;
      ++local;
    }
  }
  const unsigned s = block_sum(local);
  if (threadIdx.x == 0 && s) atomicAdd(cleared, (unsigned long long)s);
}

// Active bits of 32 cells that share one clock, SIMD-in-register for u8/u16
// cells: a cell is active iff its value lies in the cyclic interval
// [act-k'+1, act] (mod 2k) -- the predicate of pools.py:187-193 for values
// <= 2k.  Returns false if a value exceeds 2k (only a hand-made snapshot can
// hold one); the caller then takes the exact scalar path.
template <typename T>
__device__ __forceinline__ bool active_bits_simd(const uint4 (&r)[(int)sizeof(T) * 2], uint32_t act,
                                                 uint32_t B, uint32_t kp, uint32_t* active) {
  const int lo = (int)act - (int)kp + 1;
  const uint32_t* x = reinterpret_cast<const uint32_t*>(r);
  uint32_t bits = 0, bad = 0;
  if (sizeof(T) == 1 && B < 128) {
    // Guard-bit SWAR: with every lane below 128, ((x | H) - y) & H flags the
    // lanes where x >= y, and no borrow crosses a lane.  4 ops per 4 cells.
    const uint32_t H = 0x80808080u;
    const uint32_t AH = (act * 0x01010101u) | H;
    const uint32_t L4 = (uint32_t)(lo >= 0 ? lo : lo + (int)B) * 0x01010101u;
    const uint32_t B4 = B * 0x01010101u, Bp1 = (B + 1) * 0x01010101u;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t xh = x[q] | H;
      bad |= (x[q] & H) | ((xh - Bp1) & H);  // a byte >= 128 or > 2k
      const uint32_t ge_lo = (xh - L4) & H, le_act = (AH - x[q]) & H;
      const uint32_t m = lo >= 0 ? (ge_lo & le_act) : (le_act | (ge_lo & ~((xh - B4) & H)));
      bits |= ((((m >> 7) * 0x01020408u) >> 24) & 0xFu) << (4 * q);
    }
  } else if (sizeof(T) == 2 && B < 32768) {
    // Per 2-cell word: the guard-bit compares, then the two result bits (15, 31)
    // go to bit q (even cell 2q) and bit 16+q (odd cell 2q+1) of an interleaved
    // mask, un-interleaved once per 32 cells; the "value > 2k" check is one
    // lane-wise max per word, tested once.  (The cfg-4 bitmap pass is
    // issue-bound: this form retires ~35 % fewer instructions per cell.)
    // Every stored value fits the pool's width (<= 15 bits here), so each
    // lane is < 0x8000 and x | H == x + H: one add per compare.  The flags
    // (bits 15, 31) shift into the interleaved mask: after the 16 steps bit
    // 15 of step q sits at bit q and bit 31 at bit 16 + q.
    const uint32_t H = 0x80008000u;
    const uint32_t AH = (act * 0x00010001u) | H;
    const uint32_t GL = H - (uint32_t)(lo >= 0 ? lo : lo + (int)B) * 0x00010001u;
    const uint32_t GB = H - B * 0x00010001u;
    uint32_t mx = 0, inter = 0;
    if (lo >= 0) {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        mx = __vmaxu2(mx, x[q]);
        inter = (inter >> 1) | ((x[q] + GL) & (AH - x[q]) & H);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        mx = __vmaxu2(mx, x[q]);
        inter = (inter >> 1) | (((AH - x[q]) | ((x[q] + GL) & ~(x[q] + GB))) & H);
      }
    }
    bad = __vcmpgtu2(mx, B * 0x00010001u);
    // interleave: low 16 bits -> even positions, high 16 bits -> odd positions
    uint32_t e = inter & 0xFFFFu, o = inter >> 16;
    e = (e | (e << 8)) & 0x00FF00FFu; e = (e | (e << 4)) & 0x0F0F0F0Fu;
    e = (e | (e << 2)) & 0x33333333u; e = (e | (e << 1)) & 0x55555555u;
    o = (o | (o << 8)) & 0x00FF00FFu; o = (o | (o << 4)) & 0x0F0F0F0Fu;
    o = (o | (o << 2)) & 0x33333333u; o = (o | (o << 1)) & 0x55555555u;
    bits = e | (o << 1);
  } else if (sizeof(T) == 1) {
    const uint32_t B4 = B * 0x01010101u, A4 = act * 0x01010101u;
    const uint32_t L4 = (uint32_t)(lo >= 0 ? lo : lo + (int)B) * 0x01010101u;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      bad |= __vcmpgtu4(x[q], B4);
      const uint32_t m = lo >= 0 ? (__vcmpgeu4(x[q], L4) & __vcmpleu4(x[q], A4))
                                 : (__vcmpleu4(x[q], A4) | (__vcmpgeu4(x[q], L4) & __vcmpltu4(x[q], B4)));
      bits |= (((m & 0x01010101u) * 0x01020408u) >> 24) << (4 * q);
    }
  } else {
    return false;  // 2k >= 32768: the exact scalar path
  }
  *active = bits;
  return bad == 0;
}

// Whole-pool pass: inactive bitmap for width k' plus its popcount P
// (count_inactive, pools.py:195-210; predicate pools.py:187-193).  With
// `bprev` set it also emits the cells whose bit flipped against the previous
// estimate's bitmap (the incremental g0 delta, vate_incremental.cu), so the
// delta costs no second pass.
// Deferred pools (PEND): the pass first applies its word's pending-set marks
// -- marked cells take their block clock, the write set_many would have made
// (pools.py:164-178) -- and clears them, so the scan's scattered writes reach
// HBM as part of this streaming pass instead of one sector read + write per
// packet.
// The slice advance fused into the bitmap pass (vate_slice_step): the bits are
// taken with the slice's clocks, then the two blocks due under the advanced
// clock are swept exactly as k_sweep does (pools.py:221-249): range 0 at clock
// 0 (stale: v <= k), range 1 at clock k (stale: k <= v <= 2k-1 or v == 0).
// Each cell is read and rewritten by the one thread that owns its word, after
// its bit is taken, so the estimate sees the pre-advance pool as it must.
// Write-back: only the 32-byte sectors of a word that changed, always whole
// sectors -- a 16-byte store into a sector the pass read evict-first makes the
// L2 fill the other half from DRAM (scripts/probes/probe_marks.cu: 634 vs
// 165 us for a 512 MiB pass applying 5M marks).
// The rare words, entirely in memory (re-reads are L1/L2 hits): a word that
// straddles a block boundary (2k of them), u32 cells (k = 2^15), the partial
// last word of a pool smaller than 32 cells, and -- with m = 0, no sweep --
// the bits of a word holding values above 2k (hand-made snapshots only).
// Out of line, so the common path keeps its registers.
template <typename T>
__device__ __forceinline__ uint32_t slow_word(T* __restrict__ cells, uint32_t m, uint64_t i0,
                                           uint32_t cnt, Layout L, uint32_t bact0, uint32_t kp,
                                           SweepSpec SW, unsigned* swept) {
  uint32_t b = block_of(i0, L);
  uint64_t next = block_start(b + 1, L);
  uint32_t a = clock_of(bact0, b, L.B);
  uint32_t bits = 0;
#pragma unroll 1
  for (uint32_t j = 0; j < cnt; ++j) {
    while (i0 + j >= next) {
      ++b;
      next = block_start(b + 1, L);
      a = (a + 1 == L.B) ? 0 : a + 1;
    }
    if ((m >> j) & 1u) cells[i0 + j] = (T)a;
    bits |= (uint32_t)is_inactive(cells[i0 + j], a, L.B, kp) << j;
  }
  if (swept && SW.cleared && ((i0 < SW.e0 && i0 + cnt > SW.s0) || (i0 < SW.e1 && i0 + cnt > SW.s1)))
    *swept += sweep_word(cells, i0, cnt, SW.s0, SW.e0, SW.s1, SW.e1, SW.k, SW.B);
  return bits;
}

// One word of the pass: marks, bits, sweep, write-back.  Returns the inactive
// bits; adds the swept-clear count to `swept`.
template <typename T, bool PEND>
__device__ __forceinline__ uint32_t pass_word(T* __restrict__ cells, uint4 (&r)[(int)sizeof(T) * 2],
                                              uint32_t m, uint64_t i0, uint32_t cnt,
                                              uint64_t next, uint32_t act,
                                              const Layout& L, uint32_t bact0, uint32_t kp,
                                              const SweepSpec& SW, unsigned& swept) {
  if (sizeof(T) > 2 || cnt != 32 || i0 + 32 > next)
    return slow_word<T>(cells, PEND ? m : 0u, i0, cnt, L, bact0, kp, SW, &swept);
  if constexpr (sizeof(T) <= 2) {
    unsigned chg = 0;
    if (PEND && m) chg = apply_marks_regs<T>(r, m, act);
    uint32_t active, bits;
    if (active_bits_simd<T>(r, act, L.B, kp, &active)) {
      bits = ~active;
    } else {  // a value above 2k: the exact scalar predicate, from memory
      if (chg) store_sectors<T>(cells, i0, r, chg);
      chg = 0;
      bits = slow_word<T>(cells, 0u, i0, 32, L, bact0, kp, SW, nullptr);
    }
    if (SW.cleared && ((i0 < SW.e0 && i0 + 32 > SW.s0) || (i0 < SW.e1 && i0 + 32 > SW.s1)))
      swept += sweep_regs<T>(r, i0, SW, chg);
    if (chg) store_sectors<T>(cells, i0, r, chg);
    return bits;
  }
  return 0u;
}

// One 32-cell word per thread per iteration; its 16-byte cell loads, the
// previous bitmap word and the pending marks are all issued before any
// predicate, for memory-level parallelism.  Each CTA walks a contiguous run
// of words (256 consecutive words per step, coalesced), so a thread stays in
// one block for many steps and recomputes the block and its clock (a 64-bit
// division) only when it crosses a block boundary.
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <typename T, bool PEND, int PF = 0>
__global__ void __launch_bounds__(kThreads, sizeof(T) == 1 ? 5 : 4) k_bitmap(T* __restrict__ cells, Layout L,
                                                     uint32_t bact0, uint32_t kp,
                                                     uint32_t* __restrict__ bitmap,
                                                     uint64_t nwords,
                                                     unsigned long long* pool_inactive,
                                                     DeltaOut D, Publish pub, SweepSpec SW,
                                                     uint32_t* __restrict__ pend) {
  constexpr int NV = (int)sizeof(T) * 2;
  __shared__ DeltaStage ds;
  delta_stage_init(ds);
  const uint64_t per_cta = ((nwords + gridDim.x - 1) / gridDim.x + kThreads - 1) / kThreads * kThreads;
  const uint64_t w_lo = blockIdx.x * per_cta, w_hi = umin64(nwords, w_lo + per_cta);
  unsigned local = 0, swept = 0;
  uint64_t bnext = 0;  // end of the cached block (words only move forward)
  uint32_t act = 0;
  if (PF && threadIdx.x == 0) {  // the first PF steps' cells into L2
    for (int q = 0; q < PF; ++q) {
      const uint64_t f = w_lo + (uint64_t)q * kThreads;
      if (f + kThreads <= w_hi) prefetch_l2(cells + f * 32, kThreads * 32 * sizeof(T));
    }
  }
  for (uint64_t w = w_lo + threadIdx.x; w < w_hi; w += kThreads) {
    if (PF && threadIdx.x == 0) {  // L2 bulk prefetch PF steps ahead (one instruction)
      const uint64_t f = w + (uint64_t)PF * kThreads;
      if (f + kThreads <= w_hi) {
        prefetch_l2(cells + f * 32, kThreads * 32 * sizeof(T));
        if (PEND) prefetch_l2(pend + f, kThreads * 4);
        if (D.bprev) prefetch_l2(D.bprev + f, kThreads * 4);
      }
    }
    uint4 r[NV];
    const uint32_t prev = D.bprev ? __ldcs(D.bprev + w) : 0u;
    const uint32_t m = PEND ? __ldcg(pend + w) : 0u;
    const uint64_t i0 = w * 32;
    const uint32_t cnt = (uint32_t)umin64(32, L.size - i0);
    if (cnt == 32) {
#pragma unroll
      for (int v = 0; v < NV; ++v) r[v] = __ldcs(reinterpret_cast<const uint4*>(cells + i0) + v);
    }
    if (i0 >= bnext) {
      const uint32_t b = block_of(i0, L);
      bnext = block_start(b + 1, L);
      act = clock_of(bact0, b, L.B);
    }
    const uint32_t bits = pass_word<T, PEND>(cells, r, m, i0, cnt, bnext, act, L, bact0, kp, SW,
                                             swept);
    if (PEND && m) pend[w] = 0u;
    bitmap[w] = bits;
    local += __popc(bits);
    if (D.bprev) delta_word(D, ds, bits, prev, i0);
  }
  if (D.bprev) delta_flush(D, ds);
  if (SW.cleared) {
    const unsigned ws = __reduce_add_sync(0xffffffffu, swept);
    if ((threadIdx.x & 31) == 0 && ws) atomicAdd(SW.cleared, (unsigned long long)ws);
  }
  const unsigned s = block_sum(local);
  if (threadIdx.x == 0 && s) atomicAdd(pool_inactive, (unsigned long long)s);
  publish_last_block(pub);  // P (and the delta / sweep counts) straight into pinned memory
}

// flush_pending: the marks alone (no bitmap), reading only the 2^c/8-byte
// pending-set bitmap and the words it marks -- for the point queries,
// snapshots and standalone advances that read cells outside the slice step.
template <typename T>
__global__ void __launch_bounds__(kThreads) k_apply_pending(T* __restrict__ cells, Layout L,
                                                            uint32_t bact0,
                                                            uint32_t* __restrict__ pend,
                                                            uint64_t nwords) {
  constexpr int NV = (int)sizeof(T) * 2;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += stride) {
    const uint32_t m = __ldcg(pend + w);
    if (!m) continue;
    const uint64_t i0 = w * 32;
    const uint32_t cnt = (uint32_t)umin64(32, L.size - i0);
    const uint32_t b = block_of(i0, L);
    bool done = false;
    if constexpr (sizeof(T) <= 2) {
      if (cnt == 32 && i0 + 32 <= block_start(b + 1, L)) {
        uint4 r[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) r[v] = reinterpret_cast<const uint4*>(cells + i0)[v];
        const unsigned chg = apply_marks_regs<T>(r, m, clock_of(bact0, b, L.B));
        store_sectors<T>(cells, i0, r, chg);
        done = true;
      }
    }
    if (!done) apply_marks_scalar<T>(cells, i0, cnt, m, L, bact0);
    pend[w] = 0u;
  }
}

template <typename T>
__global__ void k_mask(const T* __restrict__ cells, const uint64_t* __restrict__ idx, uint64_t n,
                       Layout L, uint32_t bact0, uint32_t kp, uint8_t* __restrict__ out,
                       unsigned long long* err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t c = idx[i];
    if (c >= L.size) {
      *err = 1;
      out[i] = 0;
      continue;
    }
    out[i] = is_inactive(cells[c], clock_of(bact0, block_of(c, L), L.B), L.B, kp);
  }
}

template <typename T>
__global__ void k_get(const T* __restrict__ cells, const uint64_t* __restrict__ idx, uint64_t n,
                      uint64_t size, uint32_t* __restrict__ out, unsigned long long* err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t c = idx[i];
    if (c >= size) {
      *err = 1;
      out[i] = 0;
      continue;
    }
    out[i] = cells[c];
  }
}

// ATP1 payload: cell i occupies bits [i*w, i*w+w) of a little-endian stream of
// u64 words, LSB first; pad bits are zero (bitpack.py:26-78, pools.py:261-265).
template <typename T>
__global__ void k_pack(const T* __restrict__ cells, uint64_t size, uint32_t width,
                       unsigned long long* __restrict__ words, uint64_t nwords) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += stride) {
    const uint64_t bit0 = w * 64;
    const uint64_t i0 = bit0 / width;
    const uint64_t i1 = umin64((bit0 + 63) / width, size - 1);
    unsigned long long acc = 0;
    for (uint64_t i = i0; i <= i1; ++i) {
      const unsigned long long v = cells[i];
      const long long sh = (long long)(i * width) - (long long)bit0;
      acc |= sh >= 0 ? (v << sh) : (v >> (-sh));
    }
    words[w] = acc;
  }
}

template <typename T>
__global__ void k_unpack(const unsigned long long* __restrict__ words, uint64_t nwords,
                         uint64_t size, uint32_t width, T* __restrict__ cells) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const unsigned long long mask = (1ull << width) - 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < size; i += stride) {
    const uint64_t bit = i * width;
    const uint64_t w0 = bit >> 6;
    const uint32_t off = (uint32_t)(bit & 63);
    unsigned long long v = words[w0] >> off;
    if (off + width > 64 && w0 + 1 < nwords) v |= words[w0 + 1] << (64 - off);
    cells[i] = (T)(v & mask);
  }
}

// Replica merge, step 1: bit per cell, set iff the cell holds its block's
// current clock, i.e. was set in this slice (maintenance leaves no cell at its
// own clock: ats_preserve, counters.py:92-110).
template <typename T>
__global__ void k_dirty(const T* __restrict__ cells, Layout L, uint32_t bact0,
                        uint32_t* __restrict__ bitmap, uint64_t nwords) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += stride) {
    const uint64_t i0 = w * 32;
    const uint32_t cnt = (uint32_t)umin64(32, L.size - i0);
    uint32_t bits = 0;
    for_word_clocks(i0, cnt, L, bact0, [&](uint32_t j, uint32_t act) {
      bits |= (uint32_t)((uint32_t)cells[i0 + j] == act) << j;
    });
    bitmap[w] = bits;
  }
}

// Replica merge, step 2: OR of every rank's dirty bitmap; dirty cells take
// their block clock.  Equals the newest-timestamp max of SURVEY.md §8e.
template <typename T>
__global__ void k_merge(T* __restrict__ cells, Layout L, uint32_t bact0,
                        const uint32_t* __restrict__ bitmaps, uint64_t nwords, int nranks,
                        uint32_t* __restrict__ pend) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += stride) {
    uint32_t bits = 0;
    for (int r = 0; r < nranks; ++r) bits |= bitmaps[(uint64_t)r * nwords + w];
    if (pend) {  // deferred pool: the union becomes the pending marks
      pend[w] = bits;
      continue;
    }
    if (!bits) continue;
    const uint64_t i0 = w * 32;
    const uint32_t cnt = (uint32_t)umin64(32, L.size - i0);
    for_word_clocks(i0, cnt, L, bact0, [&](uint32_t j, uint32_t act) {
      if ((bits >> j) & 1u) cells[i0 + j] = (T)act;
    });
  }
}

// Synthetic packets; must equal oracle/vate_oracle.py:synthetic_slice.
constexpr uint64_t kSynthSalt = 0x51ED270B27C4DF1Dull;
constexpr uint64_t kSynthHostSalt = 0xA5A5A5A5A5A5A5A5ull;
constexpr uint64_t kSynthPeerSalt = 0x3C6EF372FE94F82Bull;

__global__ void k_synth(long long t, uint64_t n, DivU64 dh, uint64_t base_aip, uint64_t stream,
                        uint2* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t hi = ((uint64_t)t & 0xFFFFFFFFull) << 32;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t x = mix64(stream + (hi + i) * kPhi);
    uint64_t rank;
    div_u64(x, dh, &rank);
    const uint32_t r = (uint32_t)(mix64(rank ^ kSynthHostSalt) >> 40);
    const uint32_t lz = min(__clz(r) - 8, 12);
    const uint32_t npeers = 1u + (r & 7u) + (1u << lz);
    const uint32_t j = (uint32_t)((x >> 32) % npeers);
    const uint32_t bip = (uint32_t)mix64((rank << 20) ^ (uint64_t)j ^ kSynthPeerSalt);
    out[i] = make_uint2((uint32_t)(rank + base_aip), bip);
  }
}

// cfg 3 packets; must equal oracle/vate_oracle.py:synthetic_zipf_slice.
constexpr uint64_t kSpreadBase = 0x0B000000ull;
constexpr uint64_t kSpreadBipSalt = 0x6A09E667F3BCC909ull;
constexpr uint64_t kSpreadPeerSalt = 0xBB67AE8584CAA73Bull;

__device__ __forceinline__ uint64_t upper_bound_u64(const uint64_t* __restrict__ v, uint64_t n,
                                                    uint64_t key) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (v[mid] <= key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void k_synth_zipf(long long t, uint64_t n, uint64_t base_aip, uint64_t stream,
                             const uint64_t* __restrict__ zcdf, uint64_t hosts,
                             const uint64_t* __restrict__ scdf, uint64_t nspread,
                             uint32_t spread_q16, uint2* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t hi = ((uint64_t)t & 0xFFFFFFFFull) << 32;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t x = mix64(stream + (hi + i) * kPhi);
    const uint64_t u = x >> 24;
    if ((x & 0xFFFFull) < spread_q16) {
      const uint64_t s = upper_bound_u64(scdf, nspread, u);
      out[i] = make_uint2((uint32_t)(kSpreadBase + s), (uint32_t)mix64(x ^ kSpreadBipSalt));
    } else {
      const uint64_t rank = upper_bound_u64(zcdf, hosts, u);
      const uint32_t r = (uint32_t)(mix64(rank ^ kSynthHostSalt) >> 40);
      const uint32_t lz = min(__clz(r) - 8, 12);
      const uint32_t npeers = 1u + (r & 7u) + (1u << lz);
      const uint32_t j = (uint32_t)((mix64(x ^ kSpreadPeerSalt) >> 32) % npeers);
      const uint32_t bip = (uint32_t)mix64((rank << 20) ^ (uint64_t)j ^ kSynthPeerSalt);
      out[i] = make_uint2((uint32_t)(rank + base_aip), bip);
    }
  }
}

}  // namespace vate

using namespace vate;

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------

namespace vate {
// comparator pools (vate_compare.cu)
int cmp_fill(vate_pool* p);
int cmp_build_bitmap(vate_pool* p, int k_prime, bool with_delta);
int cmp_advance_async(vate_pool* p);
int cmp_inactive_mask(vate_pool* p, const uint64_t* d_idx, uint64_t n, int k_prime,
                      uint8_t* out_dev);

static int require_at(const vate_pool* p, const char* what) {
  if (!p) return set_error(VATE_EVALUE, "null pool handle");
  if (p->kind != VATE_AT)
    return set_error(VATE_ECONFIG, std::string(what) + " is defined for the AT pool only");
  return VATE_OK;
}

// Build the k' inactive bitmap and enqueue P into h_ctr[C_P] (not synced).
int build_bitmap(vate_pool* p, int k_prime, bool with_delta, bool fused_advance) {
  if (p->kind != VATE_AT) return cmp_build_bitmap(p, k_prime, with_delta);
  int rc = bp_maybe_enable(p, k_prime);
  if (rc) return rc;
  if (p->bp) {
    if ((uint32_t)k_prime == p->bp_L) return bp_window(p, k_prime, with_delta, fused_advance);
    // another width: the cells, brought up to date, through the direct pass;
    // the advance keeps the bit-plane bookkeeping
    rc = bp_materialize_all(p);
    if (rc) return rc;
    rc = build_bitmap_direct(p, k_prime, with_delta, false);
    if (rc || !fused_advance) return rc;
    return bp_advance(p);
  }
  return build_bitmap_direct(p, k_prime, with_delta, fused_advance);
}

int build_bitmap_direct(vate_pool* p, int k_prime, bool with_delta, bool fused_advance) {
  const uint64_t nwords = (p->L.size + 31) / 32;
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
  // the fused advance: due blocks under the advanced clock (pools.py:228-232)
  SweepSpec SW{};
  uint32_t z = 0, qb = 0;
  if (fused_advance) {
    if (p->adv_pending) return set_error(VATE_EVALUE, "previous advance not collected");
    const uint32_t B = p->L.B, k = p->L.k;
    const uint32_t nb = (p->bact0 + 1) % B;
    z = (B - nb) % B;
    qb = (k + B - nb) % B;
    SW = SweepSpec{block_start(z, p->L), block_start(z + 1, p->L), block_start(qb, p->L),
                   block_start(qb + 1, p->L), k, B, p->d_ctr + C_CLEARED};
    VATE_CUDA(cudaMemsetAsync(p->d_ctr + C_CLEARED, 0, 8, p->stream));
  }
  // counters published by the last CTA (zero-copy)
  const Publish pub{p->d_done, p->d_ctr, p->h_ctr_dev,
                    (1u << C_P) | (with_delta ? (1u << C_DCNT) | (1u << C_DWORK) : 0u) |
                        (fused_advance ? (1u << C_CLEARED) : 0u)};
  const bool pend = p->pend_dirty;
  uint32_t* pend_words = pend_ptr(p);
  rc = with_cell(p->cell_bytes, [&](auto tag) -> int {
    using T = decltype(tag);
    // pools beyond L2 stream from HBM: each CTA bulk-prefetches its cells two
    // steps ahead into L2 (one instruction per step), which takes the pass
    // from 177 to 166 us at cfg 4 (profiles/r02c_ab_pass.txt); an L2-resident
    // pool gains nothing from it
    const uint32_t grid = grid_for(nwords, kThreads, p->cap_bitmap);
    if (p->L.size * (uint64_t)sizeof(T) > (64ull << 20)) {
      if (pend)
        VATE_LAUNCH(p, VATE_K_BITMAP, grid, kThreads, 0, (k_bitmap<T, true, 2>), (T*)p->cells,
                    p->L, p->bact0, (uint32_t)k_prime, p->bitmap.as<uint32_t>(), nwords,
                    p->d_ctr + C_P, D, pub, SW, pend_words);
      else
        VATE_LAUNCH(p, VATE_K_BITMAP, grid, kThreads, 0, (k_bitmap<T, false, 2>), (T*)p->cells,
                    p->L, p->bact0, (uint32_t)k_prime, p->bitmap.as<uint32_t>(), nwords,
                    p->d_ctr + C_P, D, pub, SW, pend_words);
      return VATE_OK;
    }
    if (pend)
      VATE_LAUNCH(p, VATE_K_BITMAP, grid, kThreads, 0, (k_bitmap<T, true>), (T*)p->cells, p->L,
                  p->bact0, (uint32_t)k_prime, p->bitmap.as<uint32_t>(), nwords, p->d_ctr + C_P,
                  D, pub, SW, pend_words);
    else
      VATE_LAUNCH(p, VATE_K_BITMAP, grid, kThreads, 0, (k_bitmap<T, false>), (T*)p->cells, p->L,
                  p->bact0, (uint32_t)k_prime, p->bitmap.as<uint32_t>(), nwords, p->d_ctr + C_P,
                  D, pub, SW, pend_words);
    return VATE_OK;
  });
  if (rc) return rc;
  p->pend_dirty = false;
  // P (and the delta counts) reach the host with the estimate's one round trip,
  // written into pinned memory by the kernel's last CTA
  if (fused_advance) {  // AtPool.advance_slice bookkeeping; result via vate_advance_result
    p->bact0 = (p->bact0 + 1) % p->L.B;
    p->adv_blocks[0] = (int32_t)z;
    p->adv_blocks[1] = (int32_t)qb;
    p->adv_maint = (SW.e0 - SW.s0) + (SW.e1 - SW.s1);
    VATE_CUDA(cudaEventRecord(p->ev_adv, p->stream));
    p->adv_pending = true;
    p->sweeps_fused++;
  }
  return VATE_OK;
}

int flush_pending(vate_pool* p) {
  if (p->bp) return bp_materialize_all(p);
  if (!p->pend_dirty) return VATE_OK;
  const uint64_t nwords = (p->L.size + 31) / 32;
  int rc = with_cell(p->cell_bytes, [&](auto tag) -> int {
    using T = decltype(tag);
    VATE_LAUNCH(p, VATE_K_OTHER, grid_for(nwords, kThreads, p->cap_bitmap), kThreads, 0,
                k_apply_pending<T>, (T*)p->cells, p->L, p->bact0, p->pend.as<uint32_t>(), nwords);
    return VATE_OK;
  });
  if (rc) return rc;
  p->pend_dirty = false;
  return VATE_OK;
}

// Auto: defer (and keep the bit-plane history) when the cells take 16 MiB or
// more: cfg 2 (16 MiB, L2-resident: 0.140 -> 0.117 ms per slice), cfg 3 (64
// MiB: 0.380 -> 0.314) and cfg 4 / 5 (512 MiB); a small pool is faster with
// direct stores and the fused sweep (cfg 1, 1 MiB: 0.050 vs 0.070;
// profiles/r02h_ab_modes.txt, r02n_ab_modes.txt).
bool default_deferred(const vate_pool* p) {
  return p->kind == VATE_AT && p->L.size * (uint64_t)p->cell_bytes >= kDeferBytes;
}

int set_deferred(vate_pool* p, bool on) {
  if (on && p->kind != VATE_AT) on = false;  // the comparators store constants directly
  if (on == p->deferred) return VATE_OK;
  if (!on) {
    int rc = bp_disable(p);  // bit-plane mode needs marks
    if (rc) return rc;
    rc = flush_pending(p);
    if (rc) return rc;
    p->deferred = false;
    return VATE_OK;
  }
  const uint64_t bytes = ((p->L.size + 31) / 32) * 4;
  if (p->pend.bytes < bytes) {
    int rc = p->pend.ensure(bytes);
    if (rc) return rc;
    VATE_CUDA(cudaMemsetAsync(p->pend.ptr, 0, bytes, p->stream));
  }
  p->deferred = true;
  return VATE_OK;
}

static int lat_harvest(vate_pool* p, int slot) {
  if (!p->lat_b_set[slot]) return VATE_OK;
  VATE_CUDA(cudaEventSynchronize(p->lat_b[slot]));
  float ms = 0.f;
  VATE_CUDA(cudaEventElapsedTime(&ms, p->lat_a[slot], p->lat_b[slot]));
  p->lat_n++;
  p->lat_sum_ms += ms;
  p->lat_last_ms = ms;
  if (ms > p->lat_max_ms) p->lat_max_ms = ms;
  p->lat_b_set[slot] = false;
  p->lat_t[slot] = -1;
  return VATE_OK;
}

int lat_scan_end(vate_pool* p, int64_t t) {
  if (!p->lat_on) return VATE_OK;
  const int slot = (int)(t & 1);
  int rc = lat_harvest(p, slot);
  if (rc) return rc;
  VATE_CUDA(cudaEventRecord(p->lat_a[slot], p->stream));
  p->lat_t[slot] = t;
  return VATE_OK;
}

int lat_rows(vate_pool* p, int64_t t) {
  if (!p->lat_on) return VATE_OK;
  const int slot = (int)(t & 1);
  if (p->lat_t[slot] != t) return VATE_OK;
  VATE_CUDA(cudaEventRecord(p->lat_b[slot], p->d2h_stream));
  p->lat_b_set[slot] = true;
  return VATE_OK;
}

int check_width(vate_pool* p, int k_prime) {
  if (k_prime < 1 || k_prime > p->k)
    return set_error(VATE_EVALUE, "k'=" + std::to_string(k_prime) + " outside [1, " +
                                      std::to_string(p->k) + "]");
  return VATE_OK;
}
}  // namespace vate

extern "C" {

const char* vate_last_error(void) { return vate::g_err.c_str(); }
int vate_abi_version(void) { return VATE_ABI_VERSION; }

int vate_device_count(int* n) {
  VATE_CUDA(cudaGetDeviceCount(n));
  return VATE_OK;
}

static int pool_create(vate_pool** out, int kind, int c, int k, int partition, int device) {
  if (!out) return set_error(VATE_EVALUE, "null output pointer");
  *out = nullptr;
  if (kind != VATE_AT && kind != VATE_DR && kind != VATE_TS)
    return set_error(VATE_ECONFIG, "unknown counter kind " + std::to_string(kind));
  // _validate_pool_shape (pools.py:57-64) and AtPool.__init__ (pools.py:72-95)
  if (k < 1 || k > kMaxK)
    return set_error(VATE_ECONFIG, "k must be in [1, 32768], got " + std::to_string(k));
  if (c > 32) return set_error(VATE_ECONFIG, "c must be at most 32, got " + std::to_string(c));
  if (c < 1 || (1ull << c) < 2ull * (uint64_t)k)
    return set_error(VATE_ECONFIG, "pool of 2^" + std::to_string(c) +
                                       " cells cannot hold 2k=" + std::to_string(2 * k) +
                                       " non-empty blocks");
  if (partition != VATE_TAIL && partition != VATE_LOWDEV)
    return set_error(VATE_ECONFIG, "unknown partition method");
  if (kind != VATE_AT) partition = VATE_TAIL;  // make_pool passes it to AtPool only
  const uint64_t S = 1ull << c;
  const uint32_t B = 2u * (uint32_t)k;
  Layout L{};
  L.size = S;
  L.B = B;
  L.k = (uint32_t)k;
  L.part = partition;
  if (kind != VATE_AT) {  // no blocks: only the size is used
    L.da = make_div(1);
    L.da1 = make_div(1);
  } else if (partition == VATE_TAIL) {
    const uint64_t a = S / (B - 1), b = S % (B - 1);
    if (b == 0)
      return set_error(VATE_ECONFIG,
                       "tail partition leaves the last block empty for c=" + std::to_string(c) +
                           ", k=" + std::to_string(k) + "; use the 'low-dev' partition");
    L.da = make_div(a);
    L.da1 = make_div(a);
  } else {
    const uint64_t a2 = S / B, b2 = S % B;
    L.da = make_div(a2);
    L.da1 = make_div(a2 + 1);
    L.split = a2 * (B - b2 + 1);
    L.narrow = B - b2;
  }
  vate_pool* p = new vate_pool();
  p->device = device;
  p->c = c;
  p->k = k;
  p->partition = partition;
  p->kind = kind;
  p->width = 32u - (uint32_t)__builtin_clz(B);  // (2k).bit_length()
  if (kind == VATE_DR) p->width = 32u - (uint32_t)__builtin_clz((uint32_t)k);  // dr_bits
  if (kind == VATE_TS) p->width = 64;
  p->cell_bytes = p->width <= 8 ? 1 : (p->width <= 16 ? 2 : (p->width <= 32 ? 4 : 8));

  p->L = L;
  int rc = VATE_OK;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&p->cells, S * (uint64_t)p->cell_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_ctr, C_N * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMallocHost(&p->h_ctr, C_N * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaHostGetDevicePointer((void**)&p->h_ctr_dev, p->h_ctr, 0);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_done, 64);
  if (e == cudaSuccess) e = cudaMemset(p->d_done, 0, 64);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_small, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_adv, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->d2h_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->aux_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->h2d_stream, cudaStreamNonBlocking);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    for (cudaEvent_t* ev : {&p->ev_fin[i], &p->ev_d2h[i], &p->ev_h2d[i], &p->ev_used[i]})
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
  }
  if (e == cudaSuccess)
    e = cudaMemsetAsync(p->d_ctr, 0, C_N * sizeof(unsigned long long), p->stream);
  if (e != cudaSuccess) rc = cuda_fail(e, "vate_pool_create");
  if (rc == VATE_OK) {
    memset(p->h_ctr, 0, C_N * sizeof(unsigned long long));
    // every cell starts at the sentinel 2k (ats_init, counters.py:57-59)
    if (kind != VATE_AT)
      rc = cmp_fill(p);
    else
      rc = with_cell(p->cell_bytes, [&](auto tag) -> int {
        using T = decltype(tag);
        VATE_LAUNCH(p, VATE_K_OTHER, grid_for(S, kThreads), kThreads, 0, k_fill<T>, (T*)p->cells,
                    S, (T)B);
        return VATE_OK;
      });
  }
  // grid caps of the kernels that share SMs in the slice step (round-1 A/B
  // runs at cfg 2-4): a pool of <= 64 MiB gets a one-wave bitmap pass (its
  // launch bound: 5 CTAs per SM for u8 cells, 4 for u16, looping), leaving SM
  // slots to the registry compaction and the delta apply beside it; a larger,
  // HBM-bound pool a contiguous run of ~1800 words per CTA; the compaction 3
  // CTAs per SM.
  const uint64_t pool_bytes = S * (uint64_t)p->cell_bytes;
  p->cap_bitmap = pool_bytes <= (64ull << 20) ? 148u * (p->cell_bytes == 1 ? 5u : 4u) : 148u * 32u;
  p->cap_active = 148u * 3u;
  p->cap_inc = 148u * 16u;
  p->cap_final = 148u * 16u;
  if (rc == VATE_OK) rc = set_deferred(p, default_deferred(p));
  if (rc == VATE_OK) rc = sync_small(p);
  if (rc != VATE_OK) {
    vate_pool_destroy(p);
    return rc;
  }
  *out = p;
  return VATE_OK;
}

int vate_pool_create(vate_pool** out, int c, int k, int partition, int device) {
  return pool_create(out, VATE_AT, c, k, partition, device);
}

int vate_pool_create_kind(vate_pool** out, int kind, int c, int k, int partition, int device) {
  return pool_create(out, kind, c, k, partition, device);
}

int vate_pool_destroy(vate_pool* p) {
  if (!p) return VATE_OK;
  cudaSetDevice(p->device);
  if (p->stream) cudaStreamSynchronize(p->stream);
  if (p->d2h_stream) cudaStreamSynchronize(p->d2h_stream);
  if (p->h2d_stream) cudaStreamSynchronize(p->h2d_stream);
  if (p->aux_stream) cudaStreamSynchronize(p->aux_stream);
  if (p->bp_stream) cudaStreamSynchronize(p->bp_stream);
  for (DevBuf* b : {&p->bitmap, &p->in_a, &p->in_b, &p->out_buf, &p->hosts_sorted, &p->hosts_tmp,
                    &p->g0, &p->flags, &p->sel_idx, &p->cub_tmp, &p->lzv})
    b->release();
  for (int i = 0; i < 2; ++i) {
    for (DevBuf* b : {&p->est_out[i], &p->zv_out[i], &p->sat_out[i], &p->host_out[i], &p->stage[i]})
      b->release();
    for (cudaEvent_t ev : {p->ev_fin[i], p->ev_d2h[i], p->ev_h2d[i], p->ev_used[i]})
      if (ev) cudaEventDestroy(ev);
  }
  if (p->d2h_stream) cudaStreamDestroy(p->d2h_stream);
  if (p->h2d_stream) cudaStreamDestroy(p->h2d_stream);
  if (p->aux_stream) cudaStreamDestroy(p->aux_stream);
  if (p->bp_stream) cudaStreamDestroy(p->bp_stream);
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  if (p->ev_counts) cudaEventDestroy(p->ev_counts);
  if (p->ev_post) cudaEventDestroy(p->ev_post);
  if (p->timeline_ref) cudaEventDestroy(p->timeline_ref);
  p->pend.release();
  p->bp_ring.release();
  p->bp_S.release();
  p->bp_P.release();
  p->bp_applied.release();
  p->bp_acc.release();
  p->bp_planes.release();
  for (int i = 0; i < 2; ++i) {
    if (p->lat_a[i]) cudaEventDestroy(p->lat_a[i]);
    if (i == 0 && p->ev_bp) cudaEventDestroy(p->ev_bp);
    if (i == 0 && p->ev_bp_fork) cudaEventDestroy(p->ev_bp_fork);
    if (p->lat_b[i]) cudaEventDestroy(p->lat_b[i]);
  }
  if (p->d_done) cudaFree(p->d_done);
  if (p->ev_join) cudaEventDestroy(p->ev_join);
  inc_release(p);
  if (p->cells) cudaFree(p->cells);
  if (p->d_ctr) cudaFree(p->d_ctr);
  if (p->h_ctr) cudaFreeHost(p->h_ctr);
  if (p->ev_small) cudaEventDestroy(p->ev_small);
  if (p->ev_adv) cudaEventDestroy(p->ev_adv);
  for (auto& t : p->timed_pending) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (auto e : p->event_pool) cudaEventDestroy(e);
  for (auto e : p->marks)
    if (e) cudaEventDestroy(e);
  if (p->stream) cudaStreamDestroy(p->stream);
  delete p;
  return VATE_OK;
}

int vate_pool_info(const vate_pool* p, int32_t* bact0, int32_t* cell_bytes, void** stream) {
  if (!p) return set_error(VATE_EVALUE, "null pool handle");
  if (bact0) *bact0 = (int32_t)p->bact0;
  if (cell_bytes) *cell_bytes = p->cell_bytes;
  if (stream) *stream = (void*)p->stream;
  return VATE_OK;
}

int vate_pool_device_bytes(const vate_pool* p, int64_t* bytes) {
  if (!p || !bytes) return set_error(VATE_EVALUE, "null argument");
  const uint64_t cb = p->kind == VATE_TS ? 8 : (uint64_t)p->cell_bytes;
  *bytes = (int64_t)(p->L.size * cb + (p->deferred ? p->pend.bytes : 0) +
                     (p->bp ? p->bp_ring.bytes + p->bp_S.bytes + p->bp_P.bytes : 0));
  return VATE_OK;
}

int vate_pool_set_latency(vate_pool* p, int on) {
  int rc = enter(p);
  if (rc) return rc;
  for (int i = 0; i < 2; ++i) {
    if (!p->lat_a[i]) VATE_CUDA(cudaEventCreate(&p->lat_a[i]));
    if (!p->lat_b[i]) VATE_CUDA(cudaEventCreate(&p->lat_b[i]));
    p->lat_t[i] = -1;
    p->lat_b_set[i] = false;
  }
  p->lat_on = on != 0;
  p->lat_n = 0;
  p->lat_sum_ms = p->lat_max_ms = p->lat_last_ms = 0;
  return VATE_OK;
}

int vate_pool_lat_mark(vate_pool* p, int64_t t, int which) {
  int rc = enter(p);
  if (rc) return rc;
  return which == 0 ? lat_scan_end(p, t) : lat_rows(p, t);
}

int vate_pool_latency(vate_pool* p, double out[4]) {
  int rc = enter(p);
  if (rc) return rc;
  for (int i = 0; i < 2; ++i) {
    rc = lat_harvest(p, i);
    if (rc) return rc;
  }
  out[0] = (double)p->lat_n;
  out[1] = p->lat_n ? p->lat_sum_ms / (double)p->lat_n : 0.0;
  out[2] = p->lat_max_ms;
  out[3] = p->lat_last_ms;
  return VATE_OK;
}

int vate_pool_sync(vate_pool* p) {
  int rc = enter(p);
  if (rc) return rc;
  VATE_CUDA(cudaStreamSynchronize(p->h2d_stream));
  VATE_CUDA(cudaStreamSynchronize(p->d2h_stream));
  for (cudaStream_t s : {p->aux_stream, p->bp_stream})
    if (s) VATE_CUDA(cudaStreamSynchronize(s));
  return sync_small(p);
}

int vate_api_calls(uint64_t* n) {
  if (!n) return set_error(VATE_EVALUE, "null argument");
  *n = vate::g_api_calls;
  return VATE_OK;
}

int vate_pool_launches(const vate_pool* p, uint64_t* n) {
  if (!p) return set_error(VATE_EVALUE, "null pool handle");
  *n = p->launches;
  return VATE_OK;
}

int vate_pool_set_timing(vate_pool* p, int on) {
  int rc = enter(p);
  if (rc) return rc;
  rc = collect_timing(p);
  if (rc) return rc;
  p->timing = on != 0;
  p->timeline.clear();
  if (p->timing) {
    if (!p->timeline_ref) VATE_CUDA(cudaEventCreate(&p->timeline_ref));
    VATE_CUDA(cudaEventRecord(p->timeline_ref, p->stream));
  }
  for (int i = 0; i < VATE_K_COUNT; ++i) {
    p->timed_ms[i] = 0;
    p->timed_n[i] = 0;
  }
  return VATE_OK;
}

int vate_pool_timing(vate_pool* p, int kind, double* total_ms, uint64_t* launches) {
  int rc = enter(p);
  if (rc) return rc;
  if (kind < 0 || kind >= VATE_K_COUNT) return set_error(VATE_EVALUE, "bad kernel kind");
  rc = collect_timing(p);
  if (rc) return rc;
  *total_ms = p->timed_ms[kind];
  *launches = p->timed_n[kind];
  return VATE_OK;
}

int vate_pool_set_option(vate_pool* p, int option, int64_t value) {
  if (!p) return set_error(VATE_EVALUE, "null pool handle");
  if (option == VATE_OPT_G0 && value >= 0 && value <= 2) {
    p->opt_g0 = (int)value;
    return VATE_OK;
  }
  if (option == VATE_OPT_FUSE_SWEEP && (value == 0 || value == 1)) {
    p->opt_fuse_sweep = (int)value;
    return VATE_OK;
  }
  if (option == VATE_OPT_INC_SORT && (value == 0 || value == 1)) {
    p->opt_inc_sort = (int)value;
    return VATE_OK;
  }
  if (option == VATE_OPT_CONCURRENT && (value == 0 || value == 1)) {
    p->opt_concurrent = (int)value;
    return VATE_OK;
  }
  if (option == VATE_OPT_L2_KEEP && value >= -1 && value <= 1) {
    p->opt_l2_keep = (int)value;
    return VATE_OK;
  }
  if (option == VATE_OPT_SCAN_FILTER && value >= -1 && value <= 1) {
    p->opt_scan_check = (int)value;
    return VATE_OK;
  }
  if (option == VATE_OPT_INCREMENTAL && (value == 0 || value == 1)) {
    p->opt_inc = (int)value;
    if (!value) p->inc.valid = false;
    return VATE_OK;
  }

  if (option == VATE_OPT_BITPLANE && value >= -1 && value <= 1) {
    int rc = enter(p);
    if (rc) return rc;
    p->opt_bp = (int)value;
    p->bp_failed = false;
    if (value == 0) return bp_disable(p);
    return VATE_OK;  // enabled at the next estimate (its k' is the window)
  }
  if (option == VATE_OPT_DEFERRED && value >= -1 && value <= 1) {
    int rc = enter(p);
    if (rc) return rc;
    p->opt_deferred = (int)value;
    return set_deferred(p, value == 1 || (value == -1 && default_deferred(p)));
  }
  return set_error(VATE_EVALUE, "unknown option or value");
}

int vate_pool_timeline(vate_pool* p, double* out, uint64_t cap, uint64_t* n) {
  int rc = enter(p);
  if (rc) return rc;
  rc = collect_timing(p);
  if (rc) return rc;
  const uint64_t m = p->timeline.size() / 3;
  *n = m;
  for (uint64_t i = 0; i < 3 * std::min<uint64_t>(m, cap); ++i) out[i] = p->timeline[i];
  return VATE_OK;
}

int vate_pool_sort_stats(const vate_pool* p, uint64_t out[3]) {
  if (!p) return set_error(VATE_EVALUE, "null pool handle");
  out[0] = p->sorts_full;
  out[1] = p->sorts_incremental;
  out[2] = p->sorts_skipped;
  return VATE_OK;
}

int vate_pool_sort_sizes(const vate_pool* p, uint64_t out[3]) {
  if (!p) return set_error(VATE_EVALUE, "null pool handle");
  out[0] = p->sort_calls;
  out[1] = p->sort_keys_n;
  out[2] = p->sort_max_n;
  return VATE_OK;
}

int vate_pool_inc_stats(vate_pool* p, uint64_t out[11]) {
  int rc = enter(p);
  if (rc) return rc;
  IncIndex& I = p->inc;
  if (I.rb_timing) {  // the last rebuild's device time
    float ms = 0.f;
    VATE_CUDA(cudaEventSynchronize(I.ev_rb[1]));
    VATE_CUDA(cudaEventElapsedTime(&ms, I.ev_rb[0], I.ev_rb[1]));
    I.rebuild_ms += ms;
    I.rb_timing = false;
  }
  const uint64_t v[11] = {I.rebuilds, I.delta_slices, I.refresh_slices, I.full_slices,
                          I.last_delta_cells, I.last_delta_work, I.identity_slices,
                          I.valid ? I.m : 0, (uint64_t)(I.rebuild_ms * 1000.0), I.miss_accum,
                          I.extends};
  for (int i = 0; i < 11; ++i) out[i] = v[i];
  return VATE_OK;
}

int vate_profiler(int on) {
  VATE_CUDA(on ? cudaProfilerStart() : cudaProfilerStop());
  return VATE_OK;
}

int vate_mark(vate_pool* p, int id) {
  int rc = enter(p);
  if (rc) return rc;
  if (id < 0 || id >= 16) return set_error(VATE_EVALUE, "mark id outside [0, 16)");
  if (!p->marks[id]) VATE_CUDA(cudaEventCreate(&p->marks[id]));
  VATE_CUDA(cudaEventRecord(p->marks[id], p->stream));
  return VATE_OK;
}

int vate_mark_elapsed(vate_pool* p, int id0, int id1, double* ms) {
  int rc = enter(p);
  if (rc) return rc;
  if (id0 < 0 || id0 >= 16 || id1 < 0 || id1 >= 16 || !p->marks[id0] || !p->marks[id1])
    return set_error(VATE_EVALUE, "unrecorded mark");
  VATE_CUDA(cudaEventSynchronize(p->marks[id1]));
  float f = 0.f;
  VATE_CUDA(cudaEventElapsedTime(&f, p->marks[id0], p->marks[id1]));
  *ms = f;
  return VATE_OK;
}

// ---- ingest -----------------------------------------------------------------

int vate_set_cells(vate_pool* p, const uint64_t* idx, uint64_t n, int where) {
  int rc = enter(p);
  if (rc || n == 0) return rc;
  if (where == VATE_HOST) {
    for (uint64_t i = 0; i < n; ++i)
      if (idx[i] >= p->L.size)
        return set_error(VATE_EVALUE, "cell index " + std::to_string(idx[i]) + " outside [0, " +
                                          std::to_string(p->L.size) + ")");
  }
  const void* d_idx;
  rc = stage_in(p, p->in_a, idx, n * 8, where, &d_idx);
  if (rc) return rc;
  return with_store(p, [&](auto tag, auto rule) -> int {
    using T = decltype(tag);
    VATE_LAUNCH(p, VATE_K_SCAN, grid_for(n, kThreads), kThreads, 0,
                (k_set_cells<T, decltype(rule)>), (const uint64_t*)d_idx, n, (T*)p->cells,
                p->L.size, rule, p->d_ctr + C_ERR);
    return VATE_OK;
  });
}

static int scan_common(vate_pool* p, HashParams H, const uint64_t* aips, const uint64_t* bips,
                       const uint32_t* pairs, uint64_t n, int where, vate_hosts* hosts,
                       int64_t t) {
  int rc = enter(p);
  if (rc || n == 0) return rc;
  if (H.g < 1 || H.g > p->L.size) return set_error(VATE_ECONFIG, "g must be in [1, 2^c]");
  RegRef R{};
  if (hosts) {
    if (hosts->pool != p) return set_error(VATE_EVALUE, "host registry belongs to another pool");
    rc = hosts_prepare_insert(hosts, n);
    if (rc) return rc;
    R = hosts->ref();
    R.stamp_max = hosts->note_t(t) ? 1 : 0;
    R.l2_keep = l2_keep(p);
  }
  // registry-stamp filter: auto takes it for skewed traffic -- when the last
  // compacted slice saw 8 or more packets per distinct host (Zipf-like heads
  // whose same-address stamps serialise); plain stamps otherwise
  int filt = p->opt_scan_check;
  if (filt < 0) filt = (hosts && hosts->last_touched && n >= 8 * hosts->last_touched) ? 1 : 0;
  p->scan_form_used = filt;
  if (pairs) {
    const void* d_pairs;
    rc = stage_in(p, p->in_a, pairs, n * 8, where, &d_pairs);
    if (rc) return rc;
    const bool aligned16 = ((uintptr_t)d_pairs & 15u) == 0;
    return with_store(p, [&](auto tag, auto rule) -> int {
      using T = decltype(tag);
      using Rl = decltype(rule);
      T* cells = (T*)p->cells;
      uint64_t done = 0;
      if (aligned16 && n >= 2) {  // one uint4 (two packets) per thread
        const uint64_t n2 = n / 2;
        // about four uint4 per thread, between 16 and 64 CTAs per SM: cfg 4
        // (2.5M uint4) 0.185 -> 0.178 ms per slice over one per thread; cfg 5
        // (50M) collapses with 16 per SM (3.6 vs 1.2 ms: its per-CTA stamp filter
        // and deferred queue are per launch slice of packets)
        const uint64_t want = std::max<uint64_t>(148ull * 16u, n2 / (4ull * kThreads));
        const uint32_t grid = grid_for(n2, kThreads, (uint32_t)std::min<uint64_t>(want, 148ull * 64u));
        const uint4* src = (const uint4*)d_pairs;
        if (hosts && filt)
          VATE_LAUNCH(p, VATE_K_SCAN, grid, kThreads, 0, (k_scan_packed16<T, true, true, Rl>),
                      src, n2, cells, H, rule, R, (long long)t);
        else if (hosts)
          VATE_LAUNCH(p, VATE_K_SCAN, grid, kThreads, 0, (k_scan_packed16<T, true, false, Rl>),
                      src, n2, cells, H, rule, R, (long long)t);
        else
          VATE_LAUNCH(p, VATE_K_SCAN, grid, kThreads, 0, (k_scan_packed16<T, false, false, Rl>),
                      src, n2, cells, H, rule, R, (long long)t);
        done = 2 * n2;
      }
      if (done < n) {  // unaligned input, or the odd last packet: one packet per thread
        const uint64_t m = n - done;
        const uint32_t grid = grid_for(m, kThreads, 148u * 64u);
        const uint2* src = (const uint2*)d_pairs + done;
        if (hosts && filt)
          VATE_LAUNCH(p, VATE_K_SCAN, grid, kThreads, 0, (k_scan_packed8<T, true, true, Rl>),
                      src, m, cells, H, rule, R, (long long)t);
        else if (hosts)
          VATE_LAUNCH(p, VATE_K_SCAN, grid, kThreads, 0, (k_scan_packed8<T, true, false, Rl>),
                      src, m, cells, H, rule, R, (long long)t);
        else
          VATE_LAUNCH(p, VATE_K_SCAN, grid, kThreads, 0, (k_scan_packed8<T, false, false, Rl>),
                      src, m, cells, H, rule, R, (long long)t);
      }
      return VATE_OK;
    });
  }
  const void *d_a, *d_b;
  rc = stage_in(p, p->in_a, aips, n * 8, where, &d_a);
  if (rc) return rc;
  rc = stage_in(p, p->in_b, bips, n * 8, where, &d_b);
  if (rc) return rc;
  const uint32_t grid = grid_for(n, kThreads, 148u * 16u);
  return with_store(p, [&](auto tag, auto rule) -> int {
    using T = decltype(tag);
    using Rl = decltype(rule);
    if (hosts)
      VATE_LAUNCH(p, VATE_K_SCAN, grid, kThreads, 0, (k_scan_u64<T, true, Rl>), (const uint64_t*)d_a,
                  (const uint64_t*)d_b, n, (T*)p->cells, H, rule, R, (long long)t);
    else
      VATE_LAUNCH(p, VATE_K_SCAN, grid, kThreads, 0, (k_scan_u64<T, false, Rl>), (const uint64_t*)d_a,
                  (const uint64_t*)d_b, n, (T*)p->cells, H, rule, R, (long long)t);
    return VATE_OK;
  });
}

int vate_scan_pairs(vate_pool* p, uint64_t g, uint64_t cell_stream, uint64_t group_stream,
                    const uint64_t* aips, const uint64_t* bips, uint64_t n, int where,
                    vate_hosts* hosts, int64_t t) {
  if (!p) return set_error(VATE_EVALUE, "null pool handle");
  return scan_common(p, make_hash(g, p->c, cell_stream, group_stream), aips, bips, nullptr, n,
                     where, hosts, t);
}

int vate_scan_packed(vate_pool* p, uint64_t g, uint64_t cell_stream, uint64_t group_stream,
                     const uint32_t* pairs, uint64_t n, int where, vate_hosts* hosts,
                     int64_t t) {
  if (!p) return set_error(VATE_EVALUE, "null pool handle");
  return scan_common(p, make_hash(g, p->c, cell_stream, group_stream), nullptr, nullptr, pairs,
                     n, where, hosts, t);
}

int vate_stage_packed(vate_pool* p, const uint32_t* pairs, uint64_t n, int* slot) {
  int rc = enter(p);
  if (rc) return rc;
  const int s = p->stage_slot;
  p->stage_slot ^= 1;
  if (p->stage[s].bytes < n * 8) {
    VATE_CUDA(cudaEventSynchronize(p->ev_used[s]));
    rc = p->stage[s].ensure(n * 8 + 16);
    if (rc) return rc;
  }
  VATE_CUDA(cudaStreamWaitEvent(p->h2d_stream, p->ev_used[s], 0));  // last scan of this buffer
  if (n) VATE_CUDA(cudaMemcpyAsync(p->stage[s].ptr, pairs, n * 8, cudaMemcpyHostToDevice, p->h2d_stream));
  VATE_CUDA(cudaEventRecord(p->ev_h2d[s], p->h2d_stream));
  *slot = s;
  return VATE_OK;
}

int vate_scan_staged(vate_pool* p, uint64_t g, uint64_t cell_stream, uint64_t group_stream,
                     int slot, uint64_t n, vate_hosts* hosts, int64_t t) {
  int rc = enter(p);
  if (rc) return rc;
  if (slot < 0 || slot > 1 || p->stage[slot].bytes < n * 8)
    return set_error(VATE_EVALUE, "bad staging slot");
  VATE_CUDA(cudaStreamWaitEvent(p->stream, p->ev_h2d[slot], 0));
  rc = scan_common(p, make_hash(g, p->c, cell_stream, group_stream), nullptr, nullptr,
                   (const uint32_t*)p->stage[slot].ptr, n, VATE_DEVICE, hosts, t);
  if (rc) return rc;
  VATE_CUDA(cudaEventRecord(p->ev_used[slot], p->stream));
  return VATE_OK;
}

int vate_pair_cells(vate_pool* p, uint64_t g, int c, uint64_t cell_stream,
                    uint64_t group_stream, const uint64_t* aips, const uint64_t* bips,
                    uint64_t n, int where, uint64_t* out_cells) {
  int rc = enter(p);
  if (rc || n == 0) return rc;
  if (c < 1 || c > 32 || g < 1 || g > (1ull << c))
    return set_error(VATE_ECONFIG, "bad g/c for pair_cells");
  const void *d_a, *d_b;
  rc = stage_in(p, p->in_a, aips, n * 8, where, &d_a);
  if (rc) return rc;
  rc = stage_in(p, p->in_b, bips, n * 8, where, &d_b);
  if (rc) return rc;
  rc = p->out_buf.ensure(n * 8);
  if (rc) return rc;
  VATE_LAUNCH(p, VATE_K_OTHER, grid_for(n, kThreads), kThreads, 0, k_pair_cells,
              (const uint64_t*)d_a, (const uint64_t*)d_b, n, make_hash(g, c, cell_stream, group_stream),
              p->out_buf.as<uint64_t>());
  VATE_CUDA(cudaMemcpyAsync(out_cells, p->out_buf.ptr, n * 8, cudaMemcpyDeviceToHost, p->stream));
  return sync_small(p);
}

int vate_host_cells(vate_pool* p, uint64_t g, int c, uint64_t cell_stream, const uint64_t* aips,
                    uint64_t n, int where, uint64_t* out_cells) {
  int rc = enter(p);
  if (rc || n == 0) return rc;
  if (c < 1 || c > 32 || g < 1 || g > (1ull << c))
    return set_error(VATE_ECONFIG, "bad g/c for host_cells");
  const void* d_a;
  rc = stage_in(p, p->in_a, aips, n * 8, where, &d_a);
  if (rc) return rc;
  rc = p->out_buf.ensure(n * g * 8);
  if (rc) return rc;
  VATE_LAUNCH(p, VATE_K_OTHER, grid_for(n * g, kThreads), kThreads, 0, k_host_cells,
              (const uint64_t*)d_a, n, g, make_hash(g, c, cell_stream, 0), p->out_buf.as<uint64_t>());
  VATE_CUDA(cudaMemcpyAsync(out_cells, p->out_buf.ptr, n * g * 8, cudaMemcpyDeviceToHost, p->stream));
  return sync_small(p);
}

// ---- maintenance --------------------------------------------------------------

int vate_advance_async(vate_pool* p) {
  int rc = enter(p);
  if (rc) return rc;
  if (p->adv_pending) return set_error(VATE_EVALUE, "previous advance not collected");
  if (p->kind != VATE_AT) return cmp_advance_async(p);
  if (p->bp) return bp_advance(p);
  rc = flush_pending(p);  // marks take the clocks of the slice that made them
  if (rc) return rc;
  const uint32_t B = p->L.B, k = p->L.k;
  p->bact0 = (p->bact0 + 1) % B;  // pools.py:228
  const uint32_t z = (B - p->bact0) % B, q = (k + B - p->bact0) % B;  // pools.py:231-232
  const uint64_t s0 = block_start(z, p->L), e0 = block_start(z + 1, p->L);
  const uint64_t s1 = block_start(q, p->L), e1 = block_start(q + 1, p->L);
  p->adv_blocks[0] = (int32_t)z;
  p->adv_blocks[1] = (int32_t)q;
  p->adv_maint = (e0 - s0) + (e1 - s1);
  VATE_CUDA(cudaMemsetAsync(p->d_ctr + C_CLEARED, 0, 8, p->stream));
  rc = with_cell(p->cell_bytes, [&](auto tag) -> int {
    using T = decltype(tag);
    VATE_LAUNCH(p, VATE_K_SWEEP, grid_for(p->adv_maint, kThreads, 148u * 8u), kThreads, 0,
                k_sweep<T>, (T*)p->cells, s0, e0 - s0, s1, e1 - s1, k, p->d_ctr + C_CLEARED);
    return VATE_OK;
  });
  if (rc) return rc;
  VATE_CUDA(cudaMemcpyAsync(p->h_ctr + C_CLEARED, p->d_ctr + C_CLEARED, 8, cudaMemcpyDeviceToHost,
                            p->stream));
  VATE_CUDA(cudaEventRecord(p->ev_adv, p->stream));
  p->adv_pending = true;
  return VATE_OK;
}

int vate_advance_result(vate_pool* p, int32_t blocks[2], uint64_t* maintained,
                        uint64_t* cleared) {
  int rc = enter(p);
  if (rc) return rc;
  if (!p->adv_pending) return set_error(VATE_EVALUE, "no advance pending");
  VATE_CUDA(cudaEventSynchronize(p->ev_adv));  // only the sweep's counter, not later work
  p->adv_pending = false;
  if (blocks) {
    blocks[0] = p->adv_blocks[0];
    blocks[1] = p->adv_blocks[1];
  }
  if (maintained) *maintained = p->adv_maint;
  if (cleared) *cleared = p->h_ctr[C_CLEARED];
  return VATE_OK;
}

int vate_advance(vate_pool* p, int32_t blocks[2], uint64_t* maintained, uint64_t* cleared) {
  int rc = vate_advance_async(p);
  if (rc) return rc;
  return vate_advance_result(p, blocks, maintained, cleared);
}

// ---- queries ------------------------------------------------------------------


int vate_count_inactive(vate_pool* p, int k_prime, uint64_t* out) {
  int rc = enter(p);
  if (rc) return rc;
  rc = check_width(p, k_prime);
  if (rc) return rc;
  rc = build_bitmap(p, k_prime);
  if (rc) return rc;
  rc = sync_small(p);
  if (rc) return rc;
  *out = p->h_ctr[C_P];
  return VATE_OK;
}

int vate_inactive_mask(vate_pool* p, const uint64_t* idx, uint64_t n, int k_prime, uint8_t* out,
                       int where) {
  int rc = enter(p);
  if (rc) return rc;
  rc = check_width(p, k_prime);
  if (rc || n == 0) return rc;
  const void* d_idx;
  rc = stage_in(p, p->in_a, idx, n * 8, where, &d_idx);
  if (rc) return rc;
  rc = p->out_buf.ensure(n);
  if (rc) return rc;
  rc = flush_pending(p);
  if (rc) return rc;
  if (p->kind != VATE_AT)
    rc = cmp_inactive_mask(p, (const uint64_t*)d_idx, n, k_prime, p->out_buf.as<uint8_t>());
  else rc = with_cell(p->cell_bytes, [&](auto tag) -> int {
    using T = decltype(tag);
    VATE_LAUNCH(p, VATE_K_OTHER, grid_for(n, kThreads), kThreads, 0, k_mask<T>, (const T*)p->cells,
                (const uint64_t*)d_idx, n, p->L, p->bact0, (uint32_t)k_prime,
                p->out_buf.as<uint8_t>(), p->d_ctr + C_ERR);
    return VATE_OK;
  });
  if (rc) return rc;
  VATE_CUDA(cudaMemcpyAsync(p->h_ctr + C_ERR, p->d_ctr + C_ERR, 8, cudaMemcpyDeviceToHost, p->stream));
  VATE_CUDA(cudaMemsetAsync(p->d_ctr + C_ERR, 0, 8, p->stream));
  VATE_CUDA(cudaMemcpyAsync(out, p->out_buf.ptr, n, cudaMemcpyDeviceToHost, p->stream));
  return sync_small(p);
}

int vate_get_cells(vate_pool* p, const uint64_t* idx, uint64_t n, uint32_t* out, int where) {
  int rc = enter(p);
  if (rc || n == 0) return rc;
  if (p->kind == VATE_TS) return set_error(VATE_EVALUE, "TS cells are 64-bit: use vate_get_cells64");
  const void* d_idx;
  rc = stage_in(p, p->in_a, idx, n * 8, where, &d_idx);
  if (rc) return rc;
  rc = p->out_buf.ensure(n * 4);
  if (rc) return rc;
  rc = flush_pending(p);
  if (rc) return rc;
  rc = with_cell(p->cell_bytes, [&](auto tag) -> int {
    using T = decltype(tag);
    VATE_LAUNCH(p, VATE_K_OTHER, grid_for(n, kThreads), kThreads, 0, k_get<T>, (const T*)p->cells,
                (const uint64_t*)d_idx, n, p->L.size, p->out_buf.as<uint32_t>(), p->d_ctr + C_ERR);
    return VATE_OK;
  });
  if (rc) return rc;
  VATE_CUDA(cudaMemcpyAsync(p->h_ctr + C_ERR, p->d_ctr + C_ERR, 8, cudaMemcpyDeviceToHost, p->stream));
  VATE_CUDA(cudaMemsetAsync(p->d_ctr + C_ERR, 0, 8, p->stream));
  VATE_CUDA(cudaMemcpyAsync(out, p->out_buf.ptr, n * 4, cudaMemcpyDeviceToHost, p->stream));
  return sync_small(p);
}

// ---- snapshots ----------------------------------------------------------------

static uint64_t payload_words(const vate_pool* p) {
  return (p->L.size * p->width + 63) / 64;  // bitpack.py:36
}

int vate_snapshot_size(const vate_pool* p, uint64_t* nbytes) {
  int rc = require_at(p, "snapshot_bytes");
  if (rc) return rc;
  *nbytes = 16 + 8 * payload_words(p);
  return VATE_OK;
}

int vate_snapshot(vate_pool* p, uint8_t* buf, uint64_t cap, uint64_t* len) {
  int rc = require_at(p, "snapshot_bytes");
  if (rc) return rc;
  rc = enter(p);
  if (rc) return rc;
  const uint64_t nwords = payload_words(p), need = 16 + 8 * nwords;
  if (len) *len = need;
  if (cap < need) return set_error(VATE_EVALUE, "snapshot buffer too small");
  // header <4sBBHH6x>: magic, c, partition, k, bact0 (pools.py:32, :261-265)
  memset(buf, 0, 16);
  memcpy(buf, "ATP1", 4);
  buf[4] = (uint8_t)p->c;
  buf[5] = (uint8_t)p->partition;
  buf[6] = (uint8_t)(p->k & 0xFF);
  buf[7] = (uint8_t)((p->k >> 8) & 0xFF);
  buf[8] = (uint8_t)(p->bact0 & 0xFF);
  buf[9] = (uint8_t)((p->bact0 >> 8) & 0xFF);
  rc = p->out_buf.ensure(nwords * 8);
  if (rc) return rc;
  rc = flush_pending(p);
  if (rc) return rc;
  rc = with_cell(p->cell_bytes, [&](auto tag) -> int {
    using T = decltype(tag);
    VATE_LAUNCH(p, VATE_K_OTHER, grid_for(nwords, kThreads), kThreads, 0, k_pack<T>,
                (const T*)p->cells, p->L.size, p->width, p->out_buf.as<unsigned long long>(), nwords);
    return VATE_OK;
  });
  if (rc) return rc;
  VATE_CUDA(cudaMemcpyAsync(buf + 16, p->out_buf.ptr, nwords * 8, cudaMemcpyDeviceToHost, p->stream));
  return sync_small(p);
}

int vate_load(vate_pool* p, const uint8_t* buf, uint64_t len) {
  int rc = require_at(p, "load");
  if (rc) return rc;
  rc = enter(p);
  if (rc) return rc;
  // pools.py:271-298
  if (len < 16) return set_error(VATE_ECONFIG, "pool snapshot is truncated");
  if (memcmp(buf, "ATP1", 4) != 0) return set_error(VATE_ECONFIG, "not a pool snapshot");
  const int c = buf[4], part = buf[5];
  const int k = buf[6] | (buf[7] << 8);
  const uint32_t bact0 = buf[8] | (buf[9] << 8);
  if (part > 1) return set_error(VATE_ECONFIG, "snapshot has unknown partition code " + std::to_string(part));
  if (c != p->c || k != p->k || part != p->partition)
    return set_error(VATE_ECONFIG, "snapshot shape differs from this pool");
  if (bact0 >= p->L.B)
    return set_error(VATE_ECONFIG, "snapshot clock " + std::to_string(bact0) + " out of range");
  const uint64_t nwords = payload_words(p);
  if (len - 16 != nwords * 8)
    return set_error(VATE_ECONFIG, "snapshot payload is " + std::to_string(len - 16) +
                                       " bytes, expected " + std::to_string(nwords * 8));
  rc = p->in_a.ensure(nwords * 8 + 8);
  if (rc) return rc;
  VATE_CUDA(cudaMemcpyAsync(p->in_a.ptr, buf + 16, nwords * 8, cudaMemcpyHostToDevice, p->stream));
  if (p->pend_dirty && !p->bp) {  // every cell is overwritten: earlier marks are void
    VATE_CUDA(cudaMemsetAsync(p->pend.ptr, 0, p->pend.bytes, p->stream));
    p->pend_dirty = false;
  }
  rc = bp_wait_aux(p);
  if (rc) return rc;
  rc = with_cell(p->cell_bytes, [&](auto tag) -> int {
    using T = decltype(tag);
    VATE_LAUNCH(p, VATE_K_OTHER, grid_for(p->L.size, kThreads), kThreads, 0, k_unpack<T>,
                p->in_a.as<const unsigned long long>(), nwords, p->L.size, p->width, (T*)p->cells);
    return VATE_OK;
  });
  if (rc) return rc;
  rc = sync_small(p);
  if (rc) return rc;
  p->bact0 = bact0;
  return bp_rebuild(p);  // bit-plane mode: the history of the loaded cells
}

// ---- replica merge --------------------------------------------------------------

int vate_dirty_bitmap(vate_pool* p, uint32_t* bitmap_dev) {
  int rc = require_at(p, "the replica merge");
  if (rc) return rc;
  rc = enter(p);
  if (rc) return rc;
  const uint64_t nw = (p->L.size + 31) / 32;
  if (p->deferred) {  // the pending marks are exactly the cells this rank set
    if (!p->pend_dirty) VATE_CUDA(cudaMemsetAsync(bitmap_dev, 0, nw * 4, p->stream));
    else VATE_CUDA(cudaMemcpyAsync(bitmap_dev, pend_ptr(p), nw * 4, cudaMemcpyDeviceToDevice, p->stream));
    return VATE_OK;
  }
  rc = flush_pending(p);
  if (rc) return rc;
  const uint64_t nwords = (p->L.size + 31) / 32;
  return with_cell(p->cell_bytes, [&](auto tag) -> int {
    using T = decltype(tag);
    VATE_LAUNCH(p, VATE_K_OTHER, grid_for(nwords, kThreads), kThreads, 0, k_dirty<T>,
                (const T*)p->cells, p->L, p->bact0, bitmap_dev, nwords);
    return VATE_OK;
  });
}

int vate_merge_dirty(vate_pool* p, const uint32_t* bitmaps_dev, int nranks) {
  int rc = require_at(p, "the replica merge");
  if (rc) return rc;
  rc = enter(p);
  if (rc) return rc;
  if (nranks < 1) return set_error(VATE_EVALUE, "nranks must be >= 1");
  const uint64_t nwords = (p->L.size + 31) / 32;
  return with_cell(p->cell_bytes, [&](auto tag) -> int {
    using T = decltype(tag);
    VATE_LAUNCH(p, VATE_K_OTHER, grid_for(nwords, kThreads), kThreads, 0, k_merge<T>, (T*)p->cells,
                p->L, p->bact0, bitmaps_dev, nwords, nranks,
                p->deferred ? pend_ptr(p) : nullptr);
    if (p->deferred) p->pend_dirty = true;
    return VATE_OK;
  });
}

// ---- synthetic traffic ------------------------------------------------------------

int vate_synth_zipf(vate_pool* p, int64_t t, uint64_t n, uint64_t hosts, uint64_t base_aip,
                    uint64_t trace_seed, const uint64_t* zipf_cdf_dev, const uint64_t* spread_cdf_dev,
                    uint64_t nspread, uint32_t spread_q16, uint32_t* pairs_dev) {
  int rc = enter(p);
  if (rc || n == 0) return rc;
  if (hosts < 1 || nspread < 1) return set_error(VATE_EVALUE, "empty CDF table");
  VATE_LAUNCH(p, VATE_K_OTHER, grid_for(n, kThreads), kThreads, 0, k_synth_zipf, (long long)t, n,
              base_aip, mix64(trace_seed ^ kSynthSalt), zipf_cdf_dev, hosts, spread_cdf_dev, nspread,
              spread_q16, (uint2*)pairs_dev);
  return VATE_OK;
}

int vate_synth_packets(vate_pool* p, int64_t t, uint64_t n, uint64_t hosts, uint64_t base_aip,
                       uint64_t trace_seed, uint32_t* pairs_dev) {
  int rc = enter(p);
  if (rc || n == 0) return rc;
  if (hosts < 1) return set_error(VATE_EVALUE, "hosts must be >= 1");
  VATE_LAUNCH(p, VATE_K_OTHER, grid_for(n, kThreads), kThreads, 0, k_synth, (long long)t, n,
              make_div(hosts), base_aip, mix64(trace_seed ^ kSynthSalt), (uint2*)pairs_dev);
  return VATE_OK;
}

}  // extern "C"
