// vate_hosts.cu -- the host registry on the device (SlidingHostSet,
// pipeline.py:43-64): last-seen slice per host, the sorted active set of a
// window, and pruning.
//
// Layout: open addressing with linear probing over 16-byte {key, last}
// entries (one sector per probe), kept at load factor <= 1/2 by growing at
// every drain.  Inserts that exceed the probe limit are parked in an
// overflow list and re-inserted at the next drain, which every read of the
// registry performs first, so no update is ever lost.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include <string>
#include <utility>

#include "vate_internal.cuh"
#include "vate_registry.cuh"

namespace vate {

enum HCtr { H_COUNT = 0, H_OVF = 1, H_SPECIAL = 2, H_MAXKEY = 3, H_NOUT = 4, H_CHANGES = 5, H_NOUT2 = 6,
            H_ARR = 7, H_DEP = 8, H_TOUCHED = 9, H_N = 10 };

// Membership flips of one compaction, for the incremental sorted-set update:
// keys that joined (arrivals) and left (departures) the window's active set.
struct FlipLists {
  unsigned long long* arr;
  unsigned long long* dep;
  uint64_t cap;            // entries per list; a list that overflows forces a full sort
  unsigned long long* n_arr;
  unsigned long long* n_dep;
};

RegRef make_ref(const vate_hosts* h, const DevBuf& table, uint64_t cap) {
  RegRef R{};
  R.table = table.as<RegEntry>();
  R.mask = cap - 1;
  R.count = h->d_count + H_COUNT;
  R.ovf = h->ovf.as<RegEntry>();
  R.ovf_n = h->d_count + H_OVF;
  R.ovf_cap = h->ovf_cap;
  R.special = reinterpret_cast<unsigned int*>(h->d_count + H_SPECIAL);
  R.enabled = 1;
  return R;
}

__global__ void k_insert_keys(const uint64_t* __restrict__ keys, uint64_t n, RegRef R,
                              long long t) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    reg_insert(R, keys[i], t, false);
}

// Re-insert whole entries (rehash, overflow drain, prune rebuild).  n may live
// on the device (n_dev) when the host has not read it back.
__global__ void k_insert_entries(const RegEntry* __restrict__ src, uint64_t n,
                                 const unsigned long long* n_dev, RegRef R, int skip_empty) {
  const uint64_t total = n_dev ? *n_dev : n;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
    const RegEntry e = src[i];
    if (skip_empty && e.key == kEmptyKey) continue;
    reg_insert(R, e.key, e.last, true);
  }
}

// Keys whose last-seen slice is > cut, appended in arbitrary order (the caller
// sorts).  Each CTA handles tiles of 1024 entries (4 per thread) and reserves
// its output range with one atomic per tile.
constexpr int kActTile = 1024;

// Pass 1 (every estimate): membership of every slot for the window (last > cut),
// recorded in member[]; counts the active keys, the slots whose membership
// flipped since the previous compaction, and the largest active key.  One
// global atomic per CTA for each counter.
__global__ void __launch_bounds__(256) k_active(const RegEntry* __restrict__ table, uint64_t cap,
                                                const unsigned long long* special, long long cut,
                                                uint8_t* __restrict__ member,
                                                unsigned long long* nout,
                                                unsigned long long* maxkey,
                                                unsigned long long* changes, FlipLists F,
                                                Publish pub, long long t_now,
                                                unsigned long long* touched) {
  __shared__ unsigned s_n, s_flips;
  __shared__ unsigned long long s_max;
  if (threadIdx.x == 0) {
    s_n = 0;
    s_flips = 0;
    s_max = 0;
  }
  __syncthreads();
  const uint64_t total = cap + 1;
  const bool special_present = (*special & 0xFFFFFFFFull) != 0;
  unsigned long long kmax = 0;
  unsigned mine = 0, flips = 0, now = 0;
  // each warp takes tiles of 128 consecutive slots, lane l slots l, l+32, l+64,
  // l+96: every load instruction moves 512 contiguous bytes (entries) or 32
  // (membership flags), all four entry loads in flight before any is used
  const int lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i0 = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 128; i0 < total;
       i0 += warps * 128) {
    RegEntry ev[4];
    uint8_t mv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t i = i0 + lane + 32 * q;
      if (i < total) {
        ev[q] = table[i];
        mv[q] = member[i];
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t i = i0 + lane + 32 * q;
      if (i >= total) break;
      const RegEntry e = ev[q];
      const bool tk = (i < cap) ? (e.key != kEmptyKey && e.last > cut)
                                : (special_present && e.last > cut);
      if ((mv[q] != 0) != tk) {
        member[i] = tk;
        ++flips;
        if (F.arr) {  // rare in steady traffic: one atomic per flip
          const unsigned long long pos = atomicAdd(tk ? F.n_arr : F.n_dep, 1ull);
          if (pos < F.cap) (tk ? F.arr : F.dep)[pos] = e.key;
        }
      }
      if (tk) {
        ++mine;
        now += e.last == t_now;  // hosts seen in this very slice (scan-form heuristic)
        kmax = e.key > kmax ? e.key : kmax;
      }
    }
  }
  mine = __reduce_add_sync(0xffffffffu, mine);
  flips = __reduce_add_sync(0xffffffffu, flips);
  now = __reduce_add_sync(0xffffffffu, now);
  if ((threadIdx.x & 31) == 0 && now) atomicAdd(touched, (unsigned long long)now);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, kmax, o);
    kmax = other > kmax ? other : kmax;
  }
  if ((threadIdx.x & 31) == 0) {
    if (mine) atomicAdd(&s_n, mine);
    if (flips) atomicAdd(&s_flips, flips);
    if (kmax) atomicMax(&s_max, kmax);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_n) atomicAdd(nout, (unsigned long long)s_n);
    if (s_flips) atomicAdd(changes, (unsigned long long)s_flips);
    if (s_max) atomicMax(maxkey, s_max);
  }
  publish_last_block(pub);  // every registry counter straight into pinned memory
}

// Pass 2 (only when membership changed): the member keys, appended in arbitrary
// order (the caller sorts); one reservation per 1024-slot tile.
__global__ void __launch_bounds__(256) k_active_keys(const RegEntry* __restrict__ table,
                                                     uint64_t cap,
                                                     const uint8_t* __restrict__ member,
                                                     uint64_t* __restrict__ out,
                                                     unsigned long long* nout) {
  __shared__ unsigned warp_tot[8];
  __shared__ unsigned long long base_s;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t total = cap + 1;
  for (uint64_t tile = (uint64_t)blockIdx.x * kActTile; tile < total;
       tile += (uint64_t)gridDim.x * kActTile) {
    const uint64_t i0 = tile + threadIdx.x * 4;
    unsigned long long key[4];
    unsigned mine = 0, take = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t i = i0 + q;
      key[q] = 0;
      if (i < total && member[i]) {
        key[q] = table[i].key;
        take |= 1u << q;
        ++mine;
      }
    }
    unsigned incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned tot = 0;
      for (int w = 0; w < 8; ++w) tot += warp_tot[w];
      base_s = tot ? atomicAdd(nout, (unsigned long long)tot) : 0ull;
    }
    __syncthreads();
    unsigned before = 0;
    for (int w = 0; w < wid; ++w) before += warp_tot[w];
    unsigned long long pos = base_s + before + incl - mine;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if ((take >> q) & 1u) out[pos++] = key[q];
    __syncthreads();
  }
}

// Entries with last > horizon (prune keeps them), appended with one
// reservation per 1024-slot tile; count_only just counts the expired ones.
__global__ void __launch_bounds__(256) k_keep(const RegEntry* __restrict__ table, uint64_t cap,
                                              long long horizon, RegEntry* __restrict__ out,
                                              unsigned long long* nout, int count_only) {
  __shared__ unsigned warp_tot[8];
  __shared__ unsigned long long base_s;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned expired = 0;
  for (uint64_t tile = (uint64_t)blockIdx.x * kActTile; tile < cap;
       tile += (uint64_t)gridDim.x * kActTile) {
    const uint64_t i0 = tile + threadIdx.x * 4;
    RegEntry e[4];
    unsigned take = 0, mine = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t i = i0 + q;
      if (i < cap) {
        e[q] = table[i];
        if (e[q].key != kEmptyKey) {
          if (e[q].last > horizon) {
            take |= 1u << q;
            ++mine;
          } else {
            ++expired;
          }
        }
      }
    }
    if (count_only) continue;
    unsigned incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned tot = 0;
      for (int w = 0; w < 8; ++w) tot += warp_tot[w];
      base_s = tot ? atomicAdd(nout, (unsigned long long)tot) : 0ull;
    }
    __syncthreads();
    unsigned before = 0;
    for (int w = 0; w < wid; ++w) before += warp_tot[w];
    unsigned long long pos = base_s + before + incl - mine;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if ((take >> q) & 1u) out[pos++] = e[q];
    __syncthreads();
  }
  if (count_only) {
    expired = __reduce_add_sync(0xffffffffu, expired);
    if (lane == 0 && expired) atomicAdd(nout, (unsigned long long)expired);
  }
}

// Keys last seen exactly in slice t (the hosts this rank registered this slice).
__global__ void k_touched(const RegEntry* __restrict__ table, uint64_t cap, long long t,
                          const unsigned long long* special, uint64_t* __restrict__ out,
                          uint64_t out_cap, unsigned long long* nout) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base <= cap; base += stride) {
    const uint64_t i = base + threadIdx.x;
    bool take = false;
    unsigned long long key = 0;
    if (i <= cap) {
      const RegEntry e = table[i];
      key = i < cap ? e.key : kEmptyKey;
      take = (i < cap ? key != kEmptyKey : (*special & 0xFFFFFFFFull) != 0) && e.last == t;
    }
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (m) {
      unsigned long long pos = 0;
      if (lane == 0) pos = atomicAdd(nout, (unsigned long long)__popc(m));
      pos = __shfl_sync(0xffffffffu, pos, 0) + __popc(m & ((1u << lane) - 1u));
      if (take && pos < out_cap) out[pos] = key;
    }
  }
}

static int ensure_table(DevBuf& buf, uint64_t cap, cudaStream_t s) {
  int rc = buf.ensure((cap + 1) * sizeof(RegEntry));
  if (rc) return rc;
  VATE_CUDA(cudaMemsetAsync(buf.ptr, 0xFF, (cap + 1) * sizeof(RegEntry), s));
  return VATE_OK;
}

static uint64_t pow2_at_least(uint64_t x) {
  uint64_t c = 1;
  while (c < x) c <<= 1;
  return c;
}

int hosts_read_counters(vate_hosts* h, unsigned long long out[H_N]) {
  vate_pool* p = h->pool;
  VATE_CUDA(cudaMemcpyAsync(h->h_count, h->d_count, H_N * 8, cudaMemcpyDeviceToHost, p->stream));
  VATE_CUDA(cudaStreamSynchronize(p->stream));
  for (int i = 0; i < H_N; ++i) out[i] = h->h_count[i];
  return VATE_OK;
}

int hosts_drain(vate_hosts* h) {
  vate_pool* p = h->pool;
  unsigned long long c[H_N];
  int rc = hosts_read_counters(h, c);
  if (rc) return rc;
  const uint64_t count = c[H_COUNT], novf = c[H_OVF];
  const bool special = (c[H_SPECIAL] & 0xFFFFFFFFull) != 0;
  if (novf > h->ovf_cap)
    return set_error(VATE_ECUDA, "host registry overflow list overran its capacity");
  // Grow on parked inserts or load > 1/2; shrink when load < 1/16.  The parked
  // list repeats a key once per packet, so it only forces "at least double";
  // the recursion below grows again if re-insertion still overflows.
  const bool shrink = novf == 0 && h->cap > (1u << 16) && count * 16 < h->cap;
  // load kept <= 0.6: the table stays small enough to live in L2 next to the
  // pool (every packet probes it once)
  if (novf > 0 || count * 5 > h->cap * 3 || shrink) {
    uint64_t new_cap = pow2_at_least(2 * count + 64);
    if (novf > 0 || count * 5 > h->cap * 3) new_cap = std::max<uint64_t>(new_cap, 2 * h->cap);
    new_cap = std::max<uint64_t>(new_cap, 1u << 12);
    // rehash the live table: copy entries out first (rebuild consumes `src`)
    DevBuf old;
    old.ptr = h->table.ptr;
    old.bytes = h->table.bytes;
    const uint64_t old_cap = h->cap;
    h->table.ptr = nullptr;
    h->table.bytes = 0;
    // new table in h->table via scratch swap
    rc = ensure_table(h->scratch, new_cap, p->stream);
    if (rc) return rc;
    VATE_CUDA(cudaMemcpyAsync(h->scratch.as<RegEntry>() + new_cap, old.as<RegEntry>() + old_cap,
                              sizeof(RegEntry), cudaMemcpyDeviceToDevice, p->stream));
    VATE_CUDA(cudaMemsetAsync(h->d_count + H_COUNT, 0, 8, p->stream));
    VATE_CUDA(cudaMemsetAsync(h->d_count + H_OVF, 0, 8, p->stream));
    unsigned long long one = special ? 1ull : 0ull;
    VATE_CUDA(cudaMemcpyAsync(h->d_count + H_COUNT, &one, 8, cudaMemcpyHostToDevice, p->stream));
    RegRef R = make_ref(h, h->scratch, new_cap);
    VATE_LAUNCH(p, VATE_K_REGISTRY, grid_for(old_cap, kThreads, 148u * 16u), kThreads, 0,
                k_insert_entries, old.as<RegEntry>(), old_cap, (const unsigned long long*)nullptr,
                R, 1);
    if (novf) {
      // overflow entries go after the rehash; keep a copy since inserts may park again
      DevBuf tmp;
      rc = tmp.ensure(novf * sizeof(RegEntry));
      if (rc) { old.release(); return rc; }
      VATE_CUDA(cudaMemcpyAsync(tmp.ptr, h->ovf.ptr, novf * sizeof(RegEntry),
                                cudaMemcpyDeviceToDevice, p->stream));
      VATE_LAUNCH(p, VATE_K_REGISTRY, grid_for(novf, kThreads, 148u * 16u), kThreads, 0,
                  k_insert_entries, tmp.as<RegEntry>(), novf, (const unsigned long long*)nullptr,
                  R, 0);
      VATE_CUDA(cudaStreamSynchronize(p->stream));
      tmp.release();
    }
    VATE_CUDA(cudaStreamSynchronize(p->stream));
    old.release();
    h->table.ptr = h->scratch.ptr;
    h->table.bytes = h->scratch.bytes;
    h->scratch.ptr = nullptr;
    h->scratch.bytes = 0;
    h->cap = new_cap;
    h->member_valid = false;  // slots moved
    rc = hosts_read_counters(h, c);
    if (rc) return rc;
    if (c[H_OVF]) return hosts_drain(h);  // pathological: grow again
  }
  h->pending = 0;
  h->count_hint = c[H_COUNT];
  return VATE_OK;
}

// Stream-ordered touched-key compaction into caller memory (the multi-GPU peer
// window): parked inserts are drained first (host sync); *nout_dev receives the
// count, keys beyond cap are dropped (the caller checks the count).
int hosts_touched_launch(vate_hosts* h, int64_t t, uint64_t* out_dev, uint64_t cap,
                         unsigned long long* nout_dev) {
  vate_pool* p = h->pool;
  int rc = hosts_drain(h);
  if (rc) return rc;
  VATE_CUDA(cudaMemsetAsync(nout_dev, 0, 8, p->stream));
  VATE_LAUNCH(p, VATE_K_REGISTRY, grid_for(h->cap + 1, kThreads, 148u * 16u), kThreads, 0, k_touched,
              h->table.as<const RegEntry>(), h->cap, (long long)t, h->d_count + H_SPECIAL, out_dev,
              cap, nout_dev);
  return VATE_OK;
}

// Parked-insert count and capacity (syncs the stream).
int hosts_ovf_state(vate_hosts* h, uint64_t* novf, uint64_t* cap) {
  unsigned long long c[H_N];
  int rc = hosts_read_counters(h, c);
  if (rc) return rc;
  *novf = c[H_OVF];
  *cap = h->ovf_cap;
  return VATE_OK;
}

// Make room for n parked inserts and forget the parked ones (they are redone).
int hosts_ovf_reset(vate_hosts* h, uint64_t n) {
  int rc = h->ovf.ensure(n * sizeof(RegEntry));
  if (rc) return rc;
  h->ovf_cap = h->ovf.bytes / sizeof(RegEntry);
  VATE_CUDA(cudaMemsetAsync(h->d_count + H_OVF, 0, 8, h->pool->stream));
  return VATE_OK;
}

int hosts_prepare_insert(vate_hosts* h, uint64_t n) {
  if (h->pending + n > h->ovf_cap) {
    if (h->pending) {
      int rc = hosts_drain(h);
      if (rc) return rc;
    }
    if (n > h->ovf_cap) {
      int rc = h->ovf.ensure(n * sizeof(RegEntry));
      if (rc) return rc;
      h->ovf_cap = h->ovf.bytes / sizeof(RegEntry);
    }
  }
  h->pending += n;
  return VATE_OK;
}

// lower_bound in a sorted device array
__device__ __forceinline__ uint64_t lower_bound_u64(const unsigned long long* a, uint64_t n,
                                                    unsigned long long x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Incremental sorted-set update: new = (old \ dep) U arr, all sorted, arr and
// old disjoint, dep a subset of old.  Every element's final rank is found by
// binary search, so the merge is one scatter pass.
// Both halves in one launch: threads [0, n_old) place the old keys, the rest
// the arrivals (one launch fewer in the churn tail).
__global__ void k_merge_both(const unsigned long long* __restrict__ old, uint64_t n_old,
                             const unsigned long long* __restrict__ dep, uint64_t n_dep,
                             const unsigned long long* __restrict__ arr, uint64_t n_arr,
                             unsigned long long* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_old + n_arr;
       i += stride) {
    if (i < n_old) {
      const unsigned long long x = old[i];
      const uint64_t d = lower_bound_u64(dep, n_dep, x);
      if (d < n_dep && dep[d] == x) continue;  // departed
      out[i - d + lower_bound_u64(arr, n_arr, x)] = x;
    } else {
      const uint64_t j = i - n_old;
      const unsigned long long y = arr[j];
      out[j + lower_bound_u64(old, n_old, y) - lower_bound_u64(dep, n_dep, y)] = y;
    }
  }
}

// Small sorts (the slice's arrivals / departures, typically a few hundred
// keys): one CTA, a bitonic network in shared memory -- one launch instead of
// the radix sort's histogram + digit passes (~20 us of launch-bound work each).
constexpr uint32_t kSmallSort = 4096;

struct SmallSort {
  const unsigned long long* in;
  unsigned long long* out;
  uint32_t n, np2;
};

__global__ void __launch_bounds__(512) k_sort_small(SmallSort a, SmallSort b) {
  const SmallSort& x = blockIdx.x == 0 ? a : b;
  const unsigned long long* __restrict__ in = x.in;
  unsigned long long* __restrict__ out = x.out;
  const uint32_t n = x.n, np2 = x.np2;
  extern __shared__ unsigned long long sk[];
  for (uint32_t i = threadIdx.x; i < np2; i += blockDim.x) sk[i] = i < n ? in[i] : ~0ull;
  __syncthreads();
  for (uint32_t k = 2; k <= np2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < np2; i += blockDim.x) {
        const uint32_t ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long a = sk[i], b = sk[ixj];
          if ((a > b) == ((i & k) == 0)) {
            sk[i] = b;
            sk[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) out[i] = sk[i];
}

static int sort_keys(vate_pool* p, uint64_t* in, uint64_t* out, uint64_t n, int end_bit) {
  p->sort_keys_n += n;
  p->sort_calls++;
  p->sort_max_n = std::max<uint64_t>(p->sort_max_n, n);
  if (n <= kSmallSort) {
    uint32_t np2 = 2;
    while (np2 < n) np2 <<= 1;
    const SmallSort a{(const unsigned long long*)in, (unsigned long long*)out, (uint32_t)n, np2};
    VATE_LAUNCH(p, VATE_K_SORT, 1, std::min<uint32_t>(512u, np2 / 2), np2 * 8, k_sort_small, a, a);
    return VATE_OK;
  }
  size_t bytes = 0;
  VATE_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, (const unsigned long long*)in,
                                           (unsigned long long*)out, (int64_t)n, 0, end_bit,
                                           p->stream));
  int rc = p->cub_tmp.ensure(bytes + 256);
  if (rc) return rc;
  cudaEvent_t ta = nullptr;
  timing_begin(p, VATE_K_SORT, &ta);
  VATE_CUDA(cub::DeviceRadixSort::SortKeys(p->cub_tmp.ptr, bytes, (const unsigned long long*)in,
                                           (unsigned long long*)out, (int64_t)n, 0, end_bit,
                                           p->stream));
  timing_end(p, VATE_K_SORT, ta);
  p->launches += 1 + (uint64_t)(end_bit + 7) / 8;  // histogram + one pass per 8-bit digit
  return VATE_OK;
}

// Launch the active-set compaction; counters land in h_count after a sync.
int hosts_active_launch(vate_hosts* h, int64_t t, int k_prime) {
  vate_pool* p = h->pool;
  int rc;
  if (h->needs_grow) {
    rc = hosts_drain(h);
    if (rc) return rc;
    h->needs_grow = false;
  }
  rc = p->hosts_tmp.ensure((h->cap + 2) * 8);
  if (rc) return rc;
  if (p->hosts_sorted.bytes < (h->cap + 2) * 8) p->sorted_owner = nullptr;  // realloc loses it
  rc = p->hosts_sorted.ensure((h->cap + 2) * 8);
  if (rc) return rc;
  if (!h->member_valid || h->member.bytes < h->cap + 1) {
    rc = h->member.ensure(h->cap + 1);
    if (rc) return rc;
    VATE_CUDA(cudaMemsetAsync(h->member.ptr, 0, h->cap + 1, p->stream));
    h->member_valid = false;  // first compaction after a (re)layout always sorts
  }
  VATE_CUDA(cudaMemsetAsync(h->d_count + H_MAXKEY, 0, 8 * (H_N - H_MAXKEY), p->stream));
  FlipLists F{};
  h->flip_cap = std::max<uint64_t>(4096, h->cap / 16);
  rc = h->flips.ensure(4 * h->flip_cap * 8);
  if (rc) return rc;
  F.arr = h->flips.as<unsigned long long>();
  F.dep = F.arr + h->flip_cap;
  F.cap = h->flip_cap;
  F.n_arr = h->d_count + H_ARR;
  F.n_dep = h->d_count + H_DEP;
  // 3 CTAs per SM, looping: the compaction runs beside the bitmap pass and
  // leaves it SM slots (scripts/xp_aux_caps.sh: cfg 2 0.137 -> 0.134 ms/slice)
  VATE_LAUNCH(p, VATE_K_REGISTRY, grid_for((h->cap + 4) / 4, 256, p->cap_active), 256, 0, k_active,
              h->table.as<const RegEntry>(), h->cap, h->d_count + H_SPECIAL,
              (long long)(t - k_prime), h->member.as<uint8_t>(), h->d_count + H_NOUT,
              h->d_count + H_MAXKEY, h->d_count + H_CHANGES, F,
              Publish{p->d_done + 1, h->d_count, h->h_count_dev, (1u << H_N) - 1u}, (long long)t,
              h->d_count + H_TOUCHED);
  return VATE_OK;
}

const unsigned long long* hosts_nactive_dev(const vate_hosts* h) { return h->d_count + H_NOUT; }
uint64_t hosts_nactive_host(const vate_hosts* h) { return h->h_count[H_NOUT]; }

// After the caller's sync: handle parked inserts, then sort the active keys.
// Lagged slice step (vate_slice_step_lagged): the next slice's scan may already
// be running, so the table must not be rehashed and membership cannot be
// recomputed.  Inserts parked by this slice's scans are the first novf entries
// of the overflow list (the compaction's counter snapshot) and all were seen in
// this slice: the active set is the compaction's members plus those keys,
// sorted and deduplicated.  The table grows at the next compaction launch.
__global__ void k_ovf_keys(const RegEntry* __restrict__ ovf, uint64_t n,
                           unsigned long long* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = ovf[i].key;
}

static int active_with_parked(vate_hosts* h, uint64_t novf, uint64_t** keys_dev, uint64_t* n) {
  vate_pool* p = h->pool;
  const uint64_t members = h->h_count[H_NOUT];
  int rc = p->hosts_tmp.ensure((members + novf + 2) * 8);
  if (rc) return rc;
  rc = p->hosts_sorted.ensure((members + novf + 2) * 8);
  if (rc) return rc;
  if (members)
    VATE_LAUNCH(p, VATE_K_REGISTRY, grid_for(h->cap + 1, kActTile, 148u * 8u), 256, 0,
                k_active_keys, h->table.as<const RegEntry>(), h->cap,
                h->member.as<const uint8_t>(), p->hosts_tmp.as<uint64_t>(),
                h->d_count + H_NOUT2);
  VATE_LAUNCH(p, VATE_K_REGISTRY, grid_for(novf, kThreads, 148u * 8u), kThreads, 0, k_ovf_keys,
              h->ovf.as<const RegEntry>(), novf, p->hosts_tmp.as<unsigned long long>() + members);
  const uint64_t total = members + novf;
  rc = sort_keys(p, p->hosts_tmp.as<uint64_t>(), p->hosts_sorted.as<uint64_t>(), total, 64);
  if (rc) return rc;
  size_t bytes = 0;
  VATE_CUDA(cub::DeviceSelect::Unique(nullptr, bytes, p->hosts_sorted.as<unsigned long long>(),
                                      p->hosts_tmp.as<unsigned long long>(),
                                      h->d_count + H_NOUT2, (int64_t)total, p->stream));
  rc = p->cub_tmp.ensure(bytes + 256);
  if (rc) return rc;
  VATE_CUDA(cub::DeviceSelect::Unique(p->cub_tmp.ptr, bytes,
                                      p->hosts_sorted.as<unsigned long long>(),
                                      p->hosts_tmp.as<unsigned long long>(),
                                      h->d_count + H_NOUT2, (int64_t)total, p->stream));
  p->launches += 2;
  unsigned long long uniq = 0;
  VATE_CUDA(cudaMemcpyAsync(&uniq, h->d_count + H_NOUT2, 8, cudaMemcpyDeviceToHost, p->stream));
  VATE_CUDA(cudaStreamSynchronize(p->stream));
  std::swap(p->hosts_sorted.ptr, p->hosts_tmp.ptr);
  std::swap(p->hosts_sorted.bytes, p->hosts_tmp.bytes);
  *keys_dev = p->hosts_sorted.as<uint64_t>();
  *n = uniq;
  h->member_valid = false;  // the list is not member[]'s set: the next compaction sorts
  h->needs_grow = true;     // drain (grow + re-insert) before the next compaction
  p->sorted_owner = h;
  p->sorted_n = uniq;
  p->sorted_version++;
  p->sorts_full++;
  return VATE_OK;
}

int hosts_active_finish(vate_hosts* h, int64_t t, int k_prime, uint64_t** keys_dev, uint64_t* n) {
  vate_pool* p = h->pool;
  int rc;
  if (h->h_count[H_OVF] && h->lagged) {
    h->count_hint = h->h_count[H_COUNT];
    return active_with_parked(h, h->h_count[H_OVF], keys_dev, n);
  }
  if (h->h_count[H_OVF]) {  // inserts hit the probe limit: grow, re-insert, recompute
    rc = hosts_drain(h);
    if (rc) return rc;
    rc = hosts_active_launch(h, t, k_prime);
    if (rc) return rc;
    VATE_CUDA(cudaStreamSynchronize(p->stream));
  }
  h->pending = 0;
  h->count_hint = h->h_count[H_COUNT];
  h->last_touched = h->h_count[H_TOUCHED];
  if (h->count_hint * 5 > h->cap * 3 || (h->cap > (1u << 16) && h->count_hint * 16 < h->cap))
    h->needs_grow = true;
  *n = h->h_count[H_NOUT];
  *keys_dev = p->hosts_sorted.as<uint64_t>();
  // same membership as the last compaction, whose sorted list is still in place
  const bool was_valid = h->member_valid;  // member[] held the previous compaction's set
  const bool reuse = h->member_valid && h->h_count[H_CHANGES] == 0 && p->sorted_owner == h &&
                     p->sorted_n == *n;
  h->member_valid = true;
  if (reuse) {
    p->sorts_skipped++;
    return VATE_OK;
  }
  // membership changed by a few keys: merge them into the previous sorted list
  const uint64_t na = h->h_count[H_ARR], nd = h->h_count[H_DEP];
  const bool incremental = p->opt_inc_sort && was_valid &&
                           p->sorted_owner == h && na <= h->flip_cap && nd <= h->flip_cap &&
                           p->sorted_n + na - nd == *n && (na + nd) * 8 <= *n;
  // radix-sort only the key bits in use: arrivals are at most this compaction's
  // largest active key, departures at most the previous one's (u32 addresses:
  // 4 digit passes instead of 8)
  const unsigned long long maxkey_now = h->h_count[H_MAXKEY];
  const unsigned long long maxkey_both = std::max(maxkey_now, h->prev_maxkey);
  h->prev_maxkey = maxkey_now;
  int inc_bits = 64;
  while (inc_bits > 1 && !((maxkey_both >> (inc_bits - 1)) & 1ull)) --inc_bits;
  if (incremental) {
    unsigned long long* arr = h->flips.as<unsigned long long>();
    unsigned long long* dep = arr + h->flip_cap;
    unsigned long long* arr_s = dep + h->flip_cap;
    unsigned long long* dep_s = arr_s + h->flip_cap;
    if (na && nd && na <= kSmallSort && nd <= kSmallSort) {
      // both lists in one launch (one CTA each; a single key sorts as itself)
      uint32_t pa = 2, pd = 2;
      while (pa < na) pa <<= 1;
      while (pd < nd) pd <<= 1;
      const uint32_t np2 = std::max(pa, pd);
      p->sort_keys_n += na + nd;
      p->sort_calls += 2;
      p->sort_max_n = std::max<uint64_t>(p->sort_max_n, std::max(na, nd));
      VATE_LAUNCH(p, VATE_K_SORT, 2, std::min<uint32_t>(512u, np2 / 2), np2 * 8, k_sort_small,
                  SmallSort{arr, arr_s, (uint32_t)na, pa}, SmallSort{dep, dep_s, (uint32_t)nd, pd});
    } else {
      if (na > 1) {
        rc = sort_keys(p, (uint64_t*)arr, (uint64_t*)arr_s, na, inc_bits);
        if (rc) return rc;
      } else if (na == 1) {
        VATE_CUDA(cudaMemcpyAsync(arr_s, arr, 8, cudaMemcpyDeviceToDevice, p->stream));
      }
      if (nd > 1) {
        rc = sort_keys(p, (uint64_t*)dep, (uint64_t*)dep_s, nd, inc_bits);
        if (rc) return rc;
      } else if (nd == 1) {
        VATE_CUDA(cudaMemcpyAsync(dep_s, dep, 8, cudaMemcpyDeviceToDevice, p->stream));
      }
    }
    const auto* old = p->hosts_sorted.as<const unsigned long long>();
    auto* out = p->hosts_tmp.as<unsigned long long>();
    VATE_LAUNCH(p, VATE_K_SORT, grid_for(p->sorted_n + na, 256, 148u * 16u), 256, 0,
                k_merge_both, old, p->sorted_n, dep_s, nd, arr_s, na, out);
    std::swap(p->hosts_sorted.ptr, p->hosts_tmp.ptr);
    std::swap(p->hosts_sorted.bytes, p->hosts_tmp.bytes);
    *keys_dev = p->hosts_sorted.as<uint64_t>();
    p->sorted_n = *n;
    p->sorted_version++;
    p->sorts_incremental++;
    return VATE_OK;
  }
  // membership changed: write the member keys (same predicate, from member[])
  if (*n) {
    VATE_LAUNCH(p, VATE_K_REGISTRY, grid_for(h->cap + 1, kActTile, 148u * 8u), 256, 0,
                k_active_keys, h->table.as<const RegEntry>(), h->cap,
                h->member.as<const uint8_t>(), p->hosts_tmp.as<uint64_t>(),
                h->d_count + H_NOUT2);
  }
  const unsigned long long maxkey = h->h_count[H_MAXKEY];
  int end_bit = 64;
  while (end_bit > 1 && !((maxkey >> (end_bit - 1)) & 1ull)) --end_bit;
  if (*n > 1) {
    rc = sort_keys(p, p->hosts_tmp.as<uint64_t>(), p->hosts_sorted.as<uint64_t>(), *n, end_bit);
    if (rc) return rc;
  } else if (*n == 1) {
    VATE_CUDA(cudaMemcpyAsync(p->hosts_sorted.ptr, p->hosts_tmp.ptr, 8, cudaMemcpyDeviceToDevice,
                              p->stream));
  }
  p->sorted_owner = h;
  p->sorted_n = *n;
  p->sorted_version++;
  p->sorts_full++;
  return VATE_OK;
}

// Sorted keys with last > t - k' into pool->hosts_sorted.
int hosts_compact_active(vate_hosts* h, int64_t t, int k_prime, uint64_t** keys_dev,
                         uint64_t* n) {
  int rc = hosts_active_launch(h, t, k_prime);
  if (rc) return rc;
  VATE_CUDA(cudaStreamSynchronize(h->pool->stream));
  return hosts_active_finish(h, t, k_prime, keys_dev, n);
}

}  // namespace vate

vate::RegRef vate_hosts::ref() const { return vate::make_ref(this, table, cap); }

using namespace vate;

extern "C" {

int vate_hosts_create(vate_hosts** out, vate_pool* p, int k) {
  if (!out) return set_error(VATE_EVALUE, "null output pointer");
  *out = nullptr;
  int rc = enter(p);
  if (rc) return rc;
  vate_hosts* h = new vate_hosts();
  h->pool = p;
  h->k = k;
  h->cap = 1 << 12;
  cudaError_t e = cudaMalloc(&h->d_count, H_N * 8);
  if (e == cudaSuccess) e = cudaMallocHost(&h->h_count, H_N * 8);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer((void**)&h->h_count_dev, h->h_count, 0);
  if (e != cudaSuccess) {
    delete h;
    return cuda_fail(e, "cudaMalloc");
  }
  e = cudaMemsetAsync(h->d_count, 0, H_N * 8, p->stream);
  if (e == cudaSuccess) rc = ensure_table(h->table, h->cap, p->stream);
  else rc = cuda_fail(e, "cudaMemsetAsync");
  if (rc == VATE_OK) {
    rc = h->ovf.ensure(4096 * sizeof(RegEntry));
    h->ovf_cap = h->ovf.bytes / sizeof(RegEntry);
  }
  if (rc == VATE_OK) rc = sync_small(p);
  if (rc) {
    vate_hosts_destroy(h);
    return rc;
  }
  *out = h;
  return VATE_OK;
}

int vate_hosts_destroy(vate_hosts* h) {
  if (!h) return VATE_OK;
  cudaSetDevice(h->pool->device);
  cudaStreamSynchronize(h->pool->stream);
  if (h->pool->sorted_owner == h) h->pool->sorted_owner = nullptr;
  h->table.release();
  h->member.release();
  h->ovf.release();
  h->scratch.release();
  if (h->d_count) cudaFree(h->d_count);
  if (h->h_count) cudaFreeHost(h->h_count);
  delete h;
  return VATE_OK;
}

int vate_hosts_update(vate_hosts* h, const uint64_t* aips, uint64_t n, int64_t t, int where) {
  if (!h) return set_error(VATE_EVALUE, "null registry handle");
  vate_pool* p = h->pool;
  int rc = enter(p);
  if (rc || n == 0) return rc;
  rc = hosts_prepare_insert(h, n);
  if (rc) return rc;
  h->note_t(t);
  const void* d_keys;
  rc = stage_in(p, p->in_a, aips, n * 8, where, &d_keys);
  if (rc) return rc;
  VATE_LAUNCH(p, VATE_K_REGISTRY, grid_for(n, kThreads, 148u * 16u), kThreads, 0, k_insert_keys,
              (const uint64_t*)d_keys, n, h->ref(), (long long)t);
  return VATE_OK;
}

int vate_hosts_active(vate_hosts* h, int64_t t, int k_prime, uint64_t* out, uint64_t cap,
                      uint64_t* n) {
  if (!h) return set_error(VATE_EVALUE, "null registry handle");
  vate_pool* p = h->pool;
  int rc = enter(p);
  if (rc) return rc;
  uint64_t* keys = nullptr;
  rc = hosts_compact_active(h, t, k_prime, &keys, n);
  if (rc) return rc;
  const uint64_t m = *n < cap ? *n : cap;
  if (m) VATE_CUDA(cudaMemcpyAsync(out, keys, m * 8, cudaMemcpyDeviceToHost, p->stream));
  return sync_small(p);
}

int vate_hosts_prune(vate_hosts* h, int64_t t) {
  if (!h) return set_error(VATE_EVALUE, "null registry handle");
  vate_pool* p = h->pool;
  int rc = enter(p);
  if (rc) return rc;
  rc = hosts_drain(h);
  if (rc) return rc;
  const long long horizon = (long long)(t - h->k);
  // count the expired first: in steady traffic nothing expires and the table
  // stays as it is (slots, membership flags and the sorted active list intact)
  unsigned long long c[H_N];
  VATE_CUDA(cudaMemsetAsync(h->d_count + H_NOUT, 0, 8, p->stream));
  VATE_LAUNCH(p, VATE_K_REGISTRY, grid_for(h->cap, kActTile, 148u * 8u), 256, 0, k_keep,
              h->table.as<const RegEntry>(), h->cap, horizon, (RegEntry*)nullptr,
              h->d_count + H_NOUT, 1);
  RegEntry special_entry;
  VATE_CUDA(cudaMemcpyAsync(&special_entry, h->table.as<RegEntry>() + h->cap, sizeof(RegEntry),
                            cudaMemcpyDeviceToHost, p->stream));
  rc = hosts_read_counters(h, c);
  if (rc) return rc;
  const bool special_present = (c[H_SPECIAL] & 0xFFFFFFFFull) != 0;
  if (c[H_NOUT] == 0 && !(special_present && special_entry.last <= horizon)) return VATE_OK;
  // keep list -> fresh table of the same capacity
  DevBuf& keep = h->scratch;
  rc = keep.ensure((h->count_hint + 1) * sizeof(RegEntry));
  if (rc) return rc;
  VATE_CUDA(cudaMemsetAsync(h->d_count + H_NOUT, 0, 8, p->stream));
  VATE_LAUNCH(p, VATE_K_REGISTRY, grid_for(h->cap, kActTile, 148u * 8u), 256, 0, k_keep,
              h->table.as<const RegEntry>(), h->cap, horizon, keep.as<RegEntry>(),
              h->d_count + H_NOUT, 0);
  // special entry: keep iff present and last > horizon
  rc = hosts_read_counters(h, c);
  if (rc) return rc;
  const bool special = special_present && special_entry.last > horizon;
  rc = ensure_table(h->table, h->cap, p->stream);
  if (rc) return rc;
  if (special) {
    VATE_CUDA(cudaMemcpyAsync(h->table.as<RegEntry>() + h->cap, &special_entry, sizeof(RegEntry),
                              cudaMemcpyHostToDevice, p->stream));
  }
  unsigned long long init[3] = {special ? 1ull : 0ull, 0ull, special ? 1ull : 0ull};
  VATE_CUDA(cudaMemcpyAsync(h->d_count, init, 24, cudaMemcpyHostToDevice, p->stream));
  VATE_LAUNCH(p, VATE_K_REGISTRY, grid_for(c[H_NOUT], kThreads, 148u * 16u), kThreads, 0,
              k_insert_entries, keep.as<const RegEntry>(), (uint64_t)c[H_NOUT],
              (const unsigned long long*)nullptr, h->ref(), 1);
  VATE_CUDA(cudaStreamSynchronize(p->stream));
  h->member_valid = false;  // slots moved
  h->count_hint = c[H_NOUT] + (special ? 1 : 0);
  h->pending = 0;
  return VATE_OK;
}

int vate_hosts_touched(vate_hosts* h, int64_t t, uint64_t* out_dev, uint64_t cap, uint64_t* n) {
  if (!h) return set_error(VATE_EVALUE, "null registry handle");
  vate_pool* p = h->pool;
  int rc = enter(p);
  if (rc) return rc;
  rc = hosts_drain(h);  // parked inserts first
  if (rc) return rc;
  VATE_CUDA(cudaMemsetAsync(h->d_count + H_NOUT, 0, 8, p->stream));
  VATE_LAUNCH(p, VATE_K_REGISTRY, grid_for(h->cap + 1, kThreads, 148u * 16u), kThreads, 0, k_touched,
              h->table.as<const RegEntry>(), h->cap, (long long)t, h->d_count + H_SPECIAL, out_dev,
              cap, h->d_count + H_NOUT);
  unsigned long long c[H_N];
  rc = hosts_read_counters(h, c);
  if (rc) return rc;
  *n = c[H_NOUT];
  if (*n > cap) return set_error(VATE_EVALUE, "touched-host buffer too small");
  return VATE_OK;
}

int vate_hosts_size(vate_hosts* h, uint64_t* n) {
  if (!h) return set_error(VATE_EVALUE, "null registry handle");
  int rc = enter(h->pool);
  if (rc) return rc;
  rc = hosts_drain(h);
  if (rc) return rc;
  *n = h->count_hint;
  return VATE_OK;
}

}  // extern "C"
