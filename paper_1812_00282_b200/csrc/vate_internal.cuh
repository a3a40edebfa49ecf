// vate_internal.cuh -- shared device helpers and the pool handle.
//
// Data layout in HBM:
//   cells    : 2^c unpacked ATs, one uint8 (k <= 127), uint16 (k <= 32767) or
//              uint32 (k = 32768) each.  The reference packs w-bit cells into
//              u64 words (bitpack.py:26-56); unpacked cells make every scan
//              write a plain byte/short store with no read-modify-write, and the
//              ATP1 packed form is produced only for snapshots.
//   bitmap   : 1 bit per cell, "inactive for k'" (pools.py:187-193), rebuilt
//              per estimate; 2^c/8 bytes, L2-resident up to c = 29.
//   registry : open-addressing table of {u64 aip, i64 last-seen slice}.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <climits>

#include <string>
#include <vector>

#include "../../include/vate.h"

namespace vate {

constexpr uint64_t kPhi = 0x9E3779B97F4A7C15ull;   // hashing.py:18
constexpr uint64_t kMul1 = 0xBF58476D1CE4E5B9ull;  // hashing.py:28
constexpr uint64_t kMul2 = 0x94D049BB133111EBull;  // hashing.py:29
constexpr uint64_t kEmptyKey = ~0ull;               // registry empty-slot marker
constexpr int kMaxK = 1 << 15;                      // counters.py:27
constexpr int kThreads = 256;

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// splitmix64 finalizer (hashing.py:25-30); u64 arithmetic wraps like numpy's.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= kMul1;
  z ^= z >> 27;
  z *= kMul2;
  return z ^ (z >> 31);
}

// Exact x / d for any 64-bit x and d >= 1: q = hi64(x * floor((2^64-1)/d)) is
// at most 2 below the true quotient; two conditional corrections fix it.
struct DivU64 {
  uint64_t d, m;
};
inline DivU64 make_div(uint64_t d) { return DivU64{d, d ? ~0ull / d : 0ull}; }
__device__ __forceinline__ uint64_t div_u64(uint64_t x, DivU64 D, uint64_t* rem) {
  uint64_t q = __umul64hi(x, D.m);
  uint64_t r = x - q * D.d;
  if (r >= D.d) { ++q; r -= D.d; }
  if (r >= D.d) { ++q; r -= D.d; }
  if (rem) *rem = r;
  return q;
}

// EstimatorConfig hash parameters (estimator.py:32-61).
struct HashParams {
  uint64_t g;
  DivU64 dg;
  uint64_t gmask;      // g - 1 when g is a power of two
  int gpow2;
  uint64_t cs, gs;     // cell_stream, group_stream
  uint64_t cmask;      // 2^c - 1
};
inline HashParams make_hash(uint64_t g, int c, uint64_t cs, uint64_t gs) {
  HashParams H;
  H.g = g;
  H.dg = make_div(g);
  H.gpow2 = (g & (g - 1)) == 0;
  H.gmask = g - 1;
  H.cs = cs;
  H.gs = gs;
  H.cmask = (c >= 64) ? ~0ull : ((1ull << c) - 1);
  return H;
}

// BH(bip) = mix64(bip*phi + group_stream) mod g   (hashing.py:60-67)
__device__ __forceinline__ uint64_t slot_of(uint64_t bip, const HashParams& H) {
  uint64_t h = mix64(bip * kPhi + H.gs);
  if (H.gpow2) return h & H.gmask;
  uint64_t r;
  div_u64(h, H.dg, &r);
  return r;
}
// H(aip, slot) = mix64(((aip<<32)|slot)*phi + cell_stream) & (2^c-1)  (hashing.py:48-57)
__device__ __forceinline__ uint64_t cell_of(uint64_t aip, uint64_t slot, const HashParams& H) {
  return mix64(((aip << 32) | slot) * kPhi + H.cs) & H.cmask;
}

// Block layout of the 2k staggered-clock blocks (pools.py:80-95, :104-136).
struct Layout {
  uint64_t size;      // 2^c
  uint32_t B;         // nblocks = 2k (also the sentinel value)
  uint32_t k;
  int part;           // 0 tail, 1 low-dev
  DivU64 da;          // tail: a = S/(B-1); low-dev: a' = S/B
  DivU64 da1;         // low-dev: a'+1
  uint64_t split;     // low-dev: a'*(B-b'+1)
  uint64_t narrow;    // low-dev: B-b'
};

__host__ __device__ __forceinline__ uint32_t clock_of(uint32_t bact0, uint32_t blk, uint32_t B) {
  uint32_t s = bact0 + blk;
  return s >= B ? s - B : s;
}

__device__ __forceinline__ uint32_t block_of(uint64_t i, const Layout& L) {
  if (L.part == 0) {
    uint64_t q = div_u64(i, L.da, nullptr);
    return q < (uint64_t)(L.B - 1) ? (uint32_t)q : L.B - 1;
  }
  if (i < L.split) return (uint32_t)div_u64(i, L.da, nullptr);
  return (uint32_t)div_u64(i + L.narrow, L.da1, nullptr);
}

__host__ __device__ __forceinline__ uint64_t block_start(uint32_t b, const Layout& L) {
  if (b >= L.B) return L.size;
  if (L.part == 0) return (uint64_t)b * L.da.d;
  if (b < L.narrow) return (uint64_t)b * L.da.d;
  return L.narrow * L.da.d + (uint64_t)(b - L.narrow) * L.da1.d;
}

// Calls f(j, act) for the cells i0+j, j < cnt, walking block boundaries.
template <typename F>
__device__ __forceinline__ void for_word_clocks(uint64_t i0, uint32_t cnt, const Layout& L,
                                                uint32_t bact0, F f) {
  uint32_t b = block_of(i0, L);
  uint64_t next = block_start(b + 1, L);
  uint32_t act = clock_of(bact0, b, L.B);
  if (i0 + cnt <= next) {
#pragma unroll
    for (uint32_t j = 0; j < 32; ++j)
      if (j < cnt) f(j, act);
    return;
  }
  for (uint32_t j = 0; j < cnt; ++j) {
    while (i0 + j >= next) {
      ++b;
      next = block_start(b + 1, L);
      act = (act + 1 == L.B) ? 0 : act + 1;
    }
    f(j, act);
  }
}

// L2 eviction-priority policy for loads / reds that should outlive streaming
// traffic (createpolicy: fraction 1.0 of the accessed lines get evict_last).
__device__ __forceinline__ uint64_t l2_keep_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// What a scan / set_many stores into a cell: the AT pool stores the clock of
// the cell's block (pools.py:164-178); the comparators store a constant.
struct AtRule {
  Layout L;
  uint32_t bact0;
  static constexpr bool kMark = false, kSkip = false;
  template <typename T>
  __device__ __forceinline__ T value(uint64_t cell) const {
    return (T)clock_of(bact0, block_of(cell, L), L.B);
  }
};
struct ConstRule {
  unsigned long long v;  // DrPool: 0 (pools.py:314-315); TsPool: the slice index (:363-364)
  static constexpr bool kMark = false, kSkip = false;
  template <typename T>
  __device__ __forceinline__ T value(uint64_t) const { return (T)v; }
};
// A deferred AT pool (cells beyond L2): the write is one bit in the
// L2-resident pending-set bitmap; the next pool pass (k_bitmap, or
// flush_pending) stores the block clock into every marked cell.  Same result:
// nothing reads or re-clocks a cell between the two (flush_pending runs
// before any other cell access and before every advance).
struct MarkRule {
  uint32_t* pend;
  int keep = 0;  // L2 evict_last on the marks (VATE_OPT_L2_KEEP)
  static constexpr bool kMark = true, kSkip = false;
};
// No cell write (a registry-only pass).
struct SkipRule {
  static constexpr bool kMark = false, kSkip = true;
};

// CHECK (skewed traffic, the scan's stamp-filter form): a mark is first read
// from L2 and the red issued only if the bit is not yet set -- reads of a hot
// word are served in parallel, reds to one word serialise in the L2 atomic
// unit (cfg 3's Zipf head: ~460 marks per word of its top host's 1024 cells).
template <typename T, bool CHECK = false, typename Rule>
__device__ __forceinline__ void store_cell(T* __restrict__ cells, uint64_t c, const Rule& rule) {
  if constexpr (Rule::kSkip)
    return;
  else if constexpr (Rule::kMark) {  // fire-and-forget: a red (the compiler's atomicOr was a
    // returning atomic here; red: cfg 4 scan 94 -> 87 us, cfg 5 1.21 -> 1.13 ms)
    const uint32_t bit = 1u << (uint32_t)(c & 31);
    if (CHECK && (__ldcg(rule.pend + (c >> 5)) & bit)) return;
    if (rule.keep)
      asm volatile("red.relaxed.gpu.global.or.L2::cache_hint.b32 [%0], %1, %2;"
                   ::"l"(rule.pend + (c >> 5)), "r"(bit), "l"(l2_keep_policy()) : "memory");
    else
      asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(rule.pend + (c >> 5)), "r"(bit)
                   : "memory");
  }
  else
    cells[c] = rule.template value<T>(c);
}

// The incremental-g0 delta of a bitmap pass (vate_incremental.cu): with
// `bprev` set, every word's bits are XORed with the previous estimate's bitmap
// and the flipped cells are emitted, staged per CTA in shared memory with one
// global reservation per CTA.  Shared by the AT and the comparator passes.
struct DeltaOut {
  const uint32_t* bprev;       // nullptr: no delta
  const uint32_t* off;         // inverse-index offsets
  unsigned long long* list;    // cell | (now_inactive << 32)
  uint64_t cap;
  unsigned long long* count;
  unsigned long long* work;
};
constexpr unsigned kDeltaStage = 1024;
struct DeltaStage {
  unsigned long long delta[kDeltaStage];
  unsigned nd;
  unsigned long long work, base;
};
__device__ __forceinline__ void delta_stage_init(DeltaStage& ds) {
  if (threadIdx.x == 0) {
    ds.nd = 0;
    ds.work = 0;
  }
  __syncthreads();
}
// prev: D.bprev[w], loaded by the caller (the bitmap pass issues it with the
// cell loads so its latency overlaps theirs)
__device__ __forceinline__ void delta_word(const DeltaOut& D, DeltaStage& ds, uint32_t bits,
                                           uint32_t prev, uint64_t i0) {
  uint32_t x = bits ^ prev;
  if (!x) return;
  unsigned long long wsum = 0;
  while (x) {
    const int j = __ffs(x) - 1;
    x &= x - 1;
    const uint64_t cell = i0 + j;
    wsum += D.off[cell + 1] - D.off[cell];
    const unsigned long long v = cell | ((unsigned long long)((bits >> j) & 1u) << 32);
    const unsigned slot = atomicAdd(&ds.nd, 1u);
    if (slot < kDeltaStage) {
      ds.delta[slot] = v;
    } else {  // stage full: straight to the global list
      const unsigned long long pos = atomicAdd(D.count, 1ull);
      if (pos < D.cap) D.list[pos] = v;
    }
  }
  atomicAdd(&ds.work, wsum);
}
__device__ __forceinline__ void delta_flush(const DeltaOut& D, DeltaStage& ds) {
  __syncthreads();
  const unsigned nd = ds.nd < kDeltaStage ? ds.nd : kDeltaStage;
  if (threadIdx.x == 0) {
    ds.base = nd ? atomicAdd(D.count, (unsigned long long)nd) : 0ull;
    if (ds.work) atomicAdd(D.work, ds.work);
  }
  __syncthreads();
  for (unsigned i = threadIdx.x; i < nd; i += blockDim.x)
    if (ds.base + i < D.cap) D.list[ds.base + i] = ds.delta[i];
}

// Zero-copy publication of a kernel's counters for the slice's host round
// trip: the last CTA to finish copies n device counters into pinned host
// memory (mapped; UVA), replacing a small D2H memcpy whose copy-engine latency
// sat on the round trip.  Called by every thread at the very end of a kernel,
// after the CTA's atomics on src; done[0] must be 0 at launch and is reset.
struct Publish {
  unsigned int* done;
  const unsigned long long* src;
  unsigned long long* dst;  // device alias of pinned host memory (nullptr: off)
  unsigned mask;            // counters i with bit i set are copied
};
__device__ __forceinline__ void publish_last_block(const Publish& P) {
  if (!P.dst) return;
  __shared__ unsigned s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(P.done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  // the last CTA's first warp copies the counters, one lane each (their L2
  // round trips overlap instead of chaining)
  if (s_last && threadIdx.x < 32) {
    __threadfence();
    const int i = threadIdx.x;
    if ((P.mask >> i) & 1u) P.dst[i] = *((volatile const unsigned long long*)P.src + i);
    __threadfence_system();
    __syncwarp();
    if (i == 0) *P.done = 0u;
  }
}

// Inactive for width k' (pools.py:187-193): sentinel, or (act + 2k - v) mod 2k
// >= k'.  For stored values above 2k (only reachable through a hand-made
// snapshot) the reference's uint64 wraparound is reproduced exactly.
__device__ __forceinline__ bool is_inactive(uint32_t v, uint32_t act, uint32_t B, uint32_t kp) {
  if (v == B) return true;
  uint32_t d;
  if (v <= act) d = act - v;
  else if (v < B) d = act + B - v;
  else d = (uint32_t)(((uint64_t)act + B - (uint64_t)v) % B);
  return d >= kp;
}

// Registry entry: one 16-byte sector-aligned record per host.
struct __align__(16) RegEntry {
  unsigned long long key;
  long long last;
};

struct RegRef {
  RegEntry* table;        // cap entries + 1 special entry (key == kEmptyKey)
  uint64_t mask;          // cap - 1
  unsigned long long* count;      // distinct keys stored
  RegEntry* ovf;          // overflow list (probe limit hit)
  unsigned long long* ovf_n;
  uint64_t ovf_cap;
  unsigned int* special;  // 1 if the special entry is present
  int enabled;
  // stamps as red.max (fire-and-forget; a plain store costs the scan more in L2):
  // set only when this call's t is at least every slice the registry has seen,
  // where max and the reference's overwrite (pipeline.py:50-52) agree
  int stamp_max;
  // registry sector loads and stamps with the L2 evict_last policy
  // (VATE_OPT_L2_KEEP): the table stays in L2 across the slice's streaming passes
  int l2_keep;
};


// A growable device buffer (one stream per pool, so growth may sync).
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  int ensure(size_t want);
  void release();
  template <typename T> T* as() const { return static_cast<T*>(ptr); }
};

}  // namespace vate

struct vate_hosts;

namespace vate {
// Incremental g0 state (vate_incremental.cu): an inverse index cell -> host
// slots over a host set X, g0 of every host of X for the previous inactive
// bitmap, and that bitmap.  Invariant: g0x[i] == #inactive slots of X[i] in bprev.
struct IncIndex {
  bool valid = false;
  bool early_apply = false;               // this slice's delta was launched before the round trip
  uint64_t early_nhosts = 0;              // the active count that launch's guard read
  cudaEvent_t ev_apply = nullptr;
  uint64_t g = 0, cs = 0;
  int kp = 0;
  uint64_t m = 0;                         // hosts in X
  DevBuf X, g0x, off, ent, cursor, bprev, dlist, miss, scan_tmp;
  // extension (merge the previous slice's misses into X): staging + double buffers
  DevBuf Ykeys, Yg0, Ys, Yg0s, remap, posY, Xn, g0xn, off2, offY, ent2, sort_tmp;
  uint64_t extends = 0, extend_accum = 0;
  bool want_extend = false;
  uint64_t dlist_cap = 0;
  bool delta_launched = false;
  bool want_rebuild = false;
  uint64_t last_n = 0;                    // active hosts of the previous estimate
  uint64_t req_g = 0, req_cs = 0;         // previous request (rebuild on repeat)
  int req_kp = 0;
  uint64_t rebuilds = 0, delta_slices = 0, refresh_slices = 0, full_slices = 0;
  uint64_t last_delta_cells = 0, last_delta_work = 0, last_misses = 0;
  // identity fast path: the active list equals X (same sorted version), so g0x
  // *is* the g0 array and no lookup is needed
  bool identity_ok = false;
  uint64_t identity_version = 0, lookup_version = 0;
  bool lookup_pending = false;
  uint64_t identity_slices = 0;
  uint64_t miss_accum = 0;                // misses gathered since the last rebuild
  cudaEvent_t ev_rb[2] = {nullptr, nullptr};
  bool rb_timing = false;
  double rebuild_ms = 0;
};
}  // namespace vate

struct vate_pool {
  int device = 0;
  int kind = 0;            // VATE_AT, or a comparator: VATE_DR / VATE_TS (vate_compare.cu)
  uint64_t ts_now = 0;     // TsPool.t: advances taken (pools.py:360)
  cudaStream_t stream = nullptr;
  int c = 0, k = 0, partition = 0;
  uint32_t width = 0;      // ats_bits(k) (counters.py:52-54)
  int cell_bytes = 1;
  vate::Layout L{};
  uint32_t bact0 = 0;
  void* cells = nullptr;
  // deferred scatter (AT pools whose cells exceed L2): the
  // pending-set bitmap, one bit per cell, L2-resident; set by scans and
  // set_many, applied and cleared by the next pool pass
  vate::DevBuf pend;
  bool deferred = false;     // scans mark pend instead of storing into cells
  bool pend_dirty = false;   // pend may hold marks
  int opt_deferred = -1;     // -1 auto (cells >= kDeferBytes), 0 off, 1 on
  // bit-plane mode (vate_bitplane.cu): the pool's recent
  // history as one mark bitmap per epoch (advance) in a ring, a prefix OR of
  // the current L-epoch block and suffix ORs of the previous one, so the
  // estimate's inactive bitmap for k' = L is ~(S | P | M_e) -- three bitmaps
  // instead of the 2^c cells; cells are brought up to date block by block
  // when a block is due for its sweep (and wholesale before any other read)
  int opt_bp = -1;           // -1 auto (on for deferred pools), 0 off, 1 on
  bool bp = false;
  uint32_t bp_L = 0, bp_R = 0;   // window width (epochs), ring slots
  int64_t bp_e = 0;              // current epoch
  bool bp_folded = false;        // M_e already ORed into P in this epoch
  bool bp_failed = false;        // enabling was refused (memory, values > 2k)
  int64_t bp_flushed_e = -1;     // epoch of the last whole-pool materialization
  vate::DevBuf bp_ring, bp_S, bp_P, bp_applied, bp_acc, bp_planes;
  cudaEvent_t ev_bp = nullptr;  // the last due-block work (bp_stream)
  cudaEvent_t ev_bp_fork = nullptr;
  cudaStream_t bp_stream = nullptr;  // the due blocks, beside the window pass
  bool bp_join = false;         // cell accesses must wait for ev_bp
  uint64_t bp_wmax = 0;      // words of the largest block (+1), scratch row length
  uint32_t bp_gmax = 0;      // 16-epoch groups the ring spans
  std::vector<int64_t> bp_applied_h;  // per block: epochs <= this are in the cells
  // grid caps of the kernels that share the SMs in the slice step, fixed at
  // pool creation from its shape (co-scheduling)
  uint32_t cap_bitmap = 0, cap_active = 0, cap_inc = 0, cap_final = 0;
  // per-slice estimate latency (vate_pool_set_latency): CUDA events at the end
  // of slice t's scan (main stream) and after its report rows' D2H (copy
  // stream), one pair per slice parity
  bool lat_on = false;
  cudaEvent_t lat_a[2] = {nullptr, nullptr}, lat_b[2] = {nullptr, nullptr};
  int64_t lat_t[2] = {-1, -1};
  bool lat_b_set[2] = {false, false};
  uint64_t lat_n = 0;
  double lat_sum_ms = 0, lat_max_ms = 0, lat_last_ms = 0;

  vate::DevBuf bitmap;      // (S+31)/32 words
  vate::DevBuf in_a, in_b;  // staging for host inputs
  vate::DevBuf out_buf;     // staging for device outputs
  vate::DevBuf hosts_sorted, hosts_tmp, g0, flags, sel_idx, cub_tmp;
  vate::DevBuf est_out[2], zv_out[2], sat_out[2], host_out[2];  // double-buffered reports
  int out_slot = 0;
  vate::DevBuf stage[2];    // double-buffered packet staging (H2D prefetch)
  int stage_slot = 0;
  cudaStream_t d2h_stream = nullptr, h2d_stream = nullptr;
  cudaEvent_t ev_fin[2] = {nullptr, nullptr}, ev_d2h[2] = {nullptr, nullptr};
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};
  vate::DevBuf lzv;         // log table, g+1 doubles
  uint64_t lzv_g = 0;

  unsigned long long* d_ctr = nullptr;  // device counters (see enum in .cu)
  unsigned long long* h_ctr = nullptr;  // pinned mirror
  unsigned long long* h_ctr_dev = nullptr;  // its device alias (zero-copy publication)
  unsigned int* d_done = nullptr;       // last-block tickets: [0] bitmap, [1] registry
  cudaEvent_t ev_small = nullptr;
  cudaEvent_t marks[16] = {nullptr};

  // fused-estimate state between begin/finish
  uint64_t est_n = 0;
  const uint64_t* est_keys = nullptr;  // the hosts est_n counts (a share of hosts_sorted)
  int est_kp = 0;
  uint64_t est_g = 0;

  // pending async advance
  bool adv_pending = false;
  int32_t adv_blocks[2] = {0, 0};
  uint64_t adv_maint = 0;

  // options
  int opt_g0 = 0;
  int opt_inc = 1;            // incremental g0 through the inverse index
  int opt_l2_keep = -1;      // L2 evict_last on registry + marks in the scan: -1 auto, 0, 1
  int opt_scan_check = -1;   // registry-stamp filter: -1 auto, 0 off, 1 on
  int scan_form_used = 0;     // the form the last packed scan ran (auto resolved)
  int opt_concurrent = 1;     // fork independent estimate phases onto aux_stream
  int opt_fuse_sweep = 1;     // slice step: the advance sweep inside the bitmap pass
  cudaStream_t aux_stream = nullptr;   // second compute stream (fork/join with events)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // lagged slice step: the slice whose results the next call completes
  bool lag_pending = false;      // a slice awaits completion (lag_t, lag_kp)
  bool lag_completing = false;   // begin ran for it; end must follow
  int64_t lag_t = 0;
  int lag_kp = 0;
  bool lag_has_next = false;     // the slice begin announced (lag_next_*)
  int64_t lag_next_t = 0;
  int lag_next_kp = 0;
  bool lag_deferred_scan = false;  // its scan waits for the previous slice's end
  const uint32_t* lag_scan_pairs = nullptr;
  uint64_t lag_scan_n = 0;
  int lag_scan_where = 0;
  cudaEvent_t ev_counts = nullptr;
  cudaEvent_t ev_post = nullptr;       // the completed slice's post-round-trip work
  // multi-GPU lagged step (vate_pool_set_peer): the replica exchange runs
  // between each slice's scan and its pool pass, and this rank estimates its
  // share `lag_part` of `lag_nparts` of the sorted active set
  vate_peer* lag_peer = nullptr;
  int lag_part = 0, lag_nparts = 1;
  bool post_recorded = false;
  const void* sorted_owner = nullptr;  // registry whose active set hosts_sorted holds
  uint64_t sorted_n = 0;
  uint64_t sorts_skipped = 0;
  uint64_t sort_calls = 0, sort_keys_n = 0, sort_max_n = 0;  // key sorts: calls, keys, largest
  uint64_t sorts_full = 0, sorts_incremental = 0;
  uint64_t sweeps_fused = 0;
  int opt_inc_sort = 1;       // merge membership flips into the sorted active set
  uint64_t sorted_version = 1;         // bumps whenever hosts_sorted changes content
  const int32_t* g0_src = nullptr;     // g0 array the float path reads (p->g0 or inc.g0x)
  cudaEvent_t ev_adv = nullptr;        // advance counters landed in h_ctr
  vate::IncIndex inc;
  int dsmem_clusters = -1;   // cached max active clusters for the DSMEM gather (-1 unknown)

  // instrumentation
  uint64_t launches = 0;
  bool timing = false;
  struct Timed {
    int kind;
    cudaEvent_t a, b;
  };
  std::vector<Timed> timed_pending;
  std::vector<cudaEvent_t> event_pool;
  cudaEvent_t timeline_ref = nullptr;  // recorded when timing is switched on
  std::vector<double> timeline;        // (kind, start ms, end ms) per timed launch
  double timed_ms[VATE_K_COUNT] = {0};
  uint64_t timed_n[VATE_K_COUNT] = {0};
};

struct vate_hosts {
  vate_pool* pool = nullptr;
  unsigned long long prev_maxkey = ~0ull;  // largest active key of the previous compaction
  int k = 1;
  uint64_t cap = 0;
  vate::DevBuf table, ovf, scratch;
  unsigned long long* d_count = nullptr;  // [0] count, [1] ovf_n, [2] special flag, [3] maxkey, [4] nout
  unsigned long long* h_count = nullptr;  // pinned mirror of d_count
  unsigned long long* h_count_dev = nullptr;  // its device alias (k_active publishes)
  uint64_t ovf_cap = 0;
  uint64_t pending = 0;    // registry inserts enqueued since the last drain
  uint64_t count_hint = 0; // last count read back
  bool needs_grow = false; // load factor passed 1/2: grow at the next drain point
  bool lagged = false;     // completing a slice while the next one's scan may run
  uint64_t last_touched = 0;  // hosts seen in the last compacted slice (scan-form heuristic)
  vate::DevBuf member;     // u8 per slot: in the active set of the last compaction
  bool member_valid = false;
  vate::DevBuf flips;      // arrivals, departures and their sorted copies (4 x flip_cap)
  uint64_t flip_cap = 0;
  long long t_hi = LLONG_MIN;  // largest slice index any write path has stamped

  vate::RegRef ref() const;
  // Record a write with slice t; true when t >= every earlier one (stamp_max ok).
  bool note_t(long long t) {
    const bool mono = t >= t_hi;
    if (mono) t_hi = t;
    return mono;
  }
};

namespace vate {

int build_bitmap(vate_pool* p, int k_prime, bool with_delta = false, bool fused_advance = false);
int build_bitmap_direct(vate_pool* p, int k_prime, bool with_delta, bool fused_advance);
// Apply and clear the pending-set marks of a deferred pool (no-op otherwise):
// every cell access other than the bitmap pass calls it first.
int flush_pending(vate_pool* p);
// estimate-latency marks (no-ops unless vate_pool_set_latency(p, 1))
int lat_scan_end(vate_pool* p, int64_t t);
int lat_rows(vate_pool* p, int64_t t);
// Start or stop deferring for the pool (flushes first when stopping).
int set_deferred(vate_pool* p, bool on);
// bit-plane mode (vate_bitplane.cu)
uint32_t* pend_ptr(vate_pool* p);       // where this epoch's marks go
int bp_maybe_enable(vate_pool* p, int k_prime);
int bp_disable(vate_pool* p);
int bp_materialize_all(vate_pool* p);
int bp_window(vate_pool* p, int k_prime, bool with_delta, bool fused_advance);
int bp_advance(vate_pool* p);
int bp_rebuild(vate_pool* p);           // after cells were overwritten (load, put, fill)
int bp_wait_aux(vate_pool* p);          // order a cell access after the due-block work
uint64_t peer_key_cap(const vate_peer* x);
constexpr uint64_t kDeferBytes = 16ull << 20;
bool default_deferred(const vate_pool* p);

// error plumbing (thread-local message)
int set_error(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
extern thread_local unsigned long long g_api_calls;  // CUDA runtime calls (host-cost accounting)
#define VATE_CUDA(call)                                  \
  do {                                                   \
    ++::vate::g_api_calls;                               \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return ::vate::cuda_fail(_e, #call); \
  } while (0)

int enter(vate_pool* p);                  // cudaSetDevice + sticky-error check
int stage_in(vate_pool* p, DevBuf& buf, const void* src, size_t bytes, int where,
             const void** dev);           // host -> device staging
int sync_small(vate_pool* p);             // wait for the stream
void timing_begin(vate_pool* p, int kind, cudaEvent_t* a);
void timing_end(vate_pool* p, int kind, cudaEvent_t a);
int collect_timing(vate_pool* p);
uint32_t grid_for(uint64_t work, uint32_t per_block, uint32_t cap_blocks = 148u * 64u);
// A/B knob: the CTA cap named by env var `name` if set, else dflt.

// counters in vate_pool::d_ctr
enum Ctr { C_P = 0, C_CLEARED = 1, C_NSEL = 2, C_ERR = 3, C_DCNT = 4, C_DWORK = 5, C_MISS = 6,
           C_TRACE = 7, C_N = 8 };

// estimate helpers (vate_estimate.cu / vate_incremental.cu)
int launch_g0(vate_pool* p, const uint64_t* hosts_dev, uint64_t n, HashParams H, int32_t* g0_dev);
int launch_g0_list(vate_pool* p, const uint64_t* hosts_dev, const uint32_t* idx_dev,
                   const unsigned long long* count_dev, uint64_t cap, HashParams H, int32_t* g0_dev,
                   uint64_t* yk = nullptr, int32_t* yg = nullptr);
bool inc_delta_ready(vate_pool* p, uint64_t g, uint64_t cs, int kp);
int inc_compute_g0(vate_pool* p, const uint64_t* hosts_dev, uint64_t n, HashParams H, int kp);
int inc_apply_early(vate_pool* p, const unsigned long long* nhosts_dev, uint64_t g);
void inc_release(vate_pool* p);

// registry helpers (vate_hosts.cu)
int hosts_drain(vate_hosts* h);
int hosts_prepare_insert(vate_hosts* h, uint64_t n);
int hosts_touched_launch(vate_hosts* h, int64_t t, uint64_t* out_dev, uint64_t cap,
                         unsigned long long* nout_dev);
int hosts_ovf_state(vate_hosts* h, uint64_t* novf, uint64_t* cap);
int hosts_ovf_reset(vate_hosts* h, uint64_t n);
int hosts_compact_active(vate_hosts* h, int64_t t, int k_prime, uint64_t** keys_dev,
                         uint64_t* n);
// split form: launch (no sync; counters -> pinned), the caller syncs, finish sorts
int hosts_active_launch(vate_hosts* h, int64_t t, int k_prime);
const unsigned long long* hosts_nactive_dev(const vate_hosts* h);  // k_active's count
uint64_t hosts_nactive_host(const vate_hosts* h);                  // its pinned copy
int hosts_active_finish(vate_hosts* h, int64_t t, int k_prime, uint64_t** keys_dev, uint64_t* n);

}  // namespace vate

// RAII-free launch accounting: count every kernel, optionally time it.
#define VATE_LAUNCH(p, kind, grid, block, smem, kernel, ...)               \
  do {                                                                     \
    cudaEvent_t _ta = nullptr;                                             \
    ::vate::timing_begin((p), (kind), &_ta);                               \
    kernel<<<(grid), (block), (smem), (p)->stream>>>(__VA_ARGS__);        \
    (p)->launches++;                                                       \
    ::vate::timing_end((p), (kind), _ta);                                  \
    cudaError_t _le = cudaGetLastError();                                  \
    if (_le != cudaSuccess) return ::vate::cuda_fail(_le, #kernel);        \
  } while (0)
