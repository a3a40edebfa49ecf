// vate_peer.cu -- the multi-GPU slice exchange over peer memory (SURVEY.md §8e,
// "Option P2P (preferred)"): no NCCL on the data path.
//
// One process per GPU, each with a private replica pool.  Replicas share bact0
// and hold identical cells at slice start, so the only state that crosses
// NVLink per slice is "which cells did some rank set" (1 bit per cell) plus the
// hosts each rank registered (SlidingHostSet.update, pipeline.py:50-52, over a
// sharded stream).  Every rank owns one exchange window in its own HBM,
// exported with cudaIpcGetMemHandle and mapped by every peer:
//
//   arrive[2][world]  u64 flags: peer r stores the epoch into slot r (phase 0/1)
//   count[2]          touched-key count of the slice of that parity
//   bits[2][nwords]   this rank's dirty bitmap (cells holding their block clock)
//   keys[2][key_cap]  this rank's touched keys
//   red[2][seg]       two-shot: the OR of every rank's bitmap over this rank's
//                     segment of words
//
// Buffers alternate by slice parity.  A rank rewrites parity p at epoch e+2
// only after waiting for every peer's epoch-(e+1) arrival, which each peer
// signals after (stream order) its epoch-e reads -- so one barrier per phase
// suffices and nothing is overwritten while a peer still reads it.
//
// Merge kernels (the fused collective): the dirty-bit OR is computed from the
// peers' windows directly by the kernel that applies it to the cells, word by
// word, so the NVLink transfer overlaps the cell stores.
//   one-shot: every rank reads all world bitmaps           -> (world-1)*S/8 B in
//   two-shot: rank r ORs its 1/world segment from everyone, publishes it, then
//             reads the other segments' ORs                -> 2(world-1)/world*S/8 B in
// The result is the reference's single-pool state exactly (newest-timestamp max
// of the replicas).  Barriers spin on ld.acquire.sys with a
// globaltimer bound, so a missing peer becomes an error, not a hang.
#include <cstring>
#include <string>

#include "vate_internal.cuh"
#include "vate_registry.cuh"

struct vate_peer {
  vate_pool* pool = nullptr;
  vate_hosts* hosts = nullptr;
  int rank = 0, world = 1, mode = 0;
  uint64_t key_cap = 0, nwords = 0, seg = 0;
  uint64_t epoch = 0;
  uint8_t* win = nullptr;           // own window (cudaMalloc, IPC-exported)
  size_t win_bytes = 0;
  uint8_t** d_bases = nullptr;      // device table: window base of every rank
  uint8_t* bases[64] = {nullptr};   // host copy (own = win, peers = IPC mappings)
  bool opened = false;
  unsigned long long* d_err = nullptr;  // [0] barrier timeout
  unsigned long long* h_mirror = nullptr;  // pinned: [0] err, [1] own touched count
  uint64_t last_touched_total = 0;
  uint64_t nvlink_bytes = 0;        // bytes this rank read from peers (last exchange)
};

namespace vate {

constexpr int kMaxWorld = 64;
constexpr unsigned long long kBarrierTimeoutNs = 20ull * 1000 * 1000 * 1000;

struct WinLayout {
  uint64_t arrive, count, bits[2], keys[2], red[2], total;
};

static uint64_t up256(uint64_t x) { return (x + 255) & ~uint64_t(255); }

static WinLayout win_layout(int world, uint64_t nwords, uint64_t seg, uint64_t key_cap) {
  WinLayout w{};
  uint64_t o = 0;
  w.arrive = o; o = up256(o + 2ull * kMaxWorld * 8);
  w.count = o;  o = up256(o + 2 * 8);
  for (int q = 0; q < 2; ++q) { w.bits[q] = o; o = up256(o + nwords * 4); }
  for (int q = 0; q < 2; ++q) { w.keys[q] = o; o = up256(o + key_cap * 8); }
  for (int q = 0; q < 2; ++q) { w.red[q] = o; o = up256(o + seg * 4); }
  w.total = o;
  (void)world;
  return w;
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Thread 0 of every CTA waits until all ranks stored >= epoch into this rank's
// arrive[phase][*]; the CTA barrier then orders the CTA's later loads.
__device__ __forceinline__ void wait_arrivals(const unsigned long long* arrive, int world,
                                              unsigned long long epoch,
                                              unsigned long long* err) {
  if (threadIdx.x == 0) {
    const unsigned long long t0 = globaltimer();
    for (int r = 0; r < world; ++r) {
      while (ld_acquire_sys(arrive + r) < epoch) {
        if (globaltimer() - t0 > kBarrierTimeoutNs) {
          atomicExch(err, 1ull);
          break;
        }
        __nanosleep(64);
      }
    }
  }
  __syncthreads();
}

// Lane r publishes this rank's arrival (epoch) into rank r's window.
__global__ void k_arrive(uint8_t* const* bases, uint64_t off_arrive, int phase, int me, int world,
                         unsigned long long epoch) {
  const int r = threadIdx.x;
  __threadfence_system();
  if (r < world) {
    auto* slot = reinterpret_cast<unsigned long long*>(bases[r] + off_arrive) +
                 (uint64_t)phase * kMaxWorld + me;
    st_release_sys(slot, epoch);
  }
}

template <typename T>
__global__ void k_dirty_into(const T* __restrict__ cells, Layout L, uint32_t bact0,
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

// Dirty cells take their block clock; on a deferred pool (pend set) the
// union becomes the pending marks instead, which the bitmap pass applies.
template <typename T>
__device__ __forceinline__ void apply_word(T* __restrict__ cells, const Layout& L, uint32_t bact0,
                                           uint64_t w, uint32_t bits, uint32_t* pend) {
  if (pend) {
    pend[w] = bits;
    return;
  }
  if (!bits) return;
  const uint64_t i0 = w * 32;
  const uint32_t cnt = (uint32_t)umin64(32, L.size - i0);
  for_word_clocks(i0, cnt, L, bact0, [&](uint32_t j, uint32_t act) {
    if ((bits >> j) & 1u) cells[i0 + j] = (T)act;
  });
}

// one-shot: OR of all world windows' bitmaps, applied to own cells
template <typename T>
__global__ void __launch_bounds__(256) k_merge_oneshot(
    T* __restrict__ cells, Layout L, uint32_t bact0, uint8_t* const* __restrict__ bases,
    uint64_t off_bits, int world, uint64_t nwords, unsigned long long epoch,
    const unsigned long long* arrive, unsigned long long* err, uint32_t* __restrict__ pend) {
  wait_arrivals(arrive, world, epoch, err);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += stride) {
    uint32_t bits = 0;
    for (int r = 0; r < world; ++r)
      bits |= __ldcg(reinterpret_cast<const uint32_t*>(bases[r] + off_bits) + w);
    apply_word(cells, L, bact0, w, bits, pend);
  }
}

// two-shot, phase 1: OR of everyone's bitmap over own segment -> red, applied
template <typename T>
__global__ void __launch_bounds__(256) k_merge_reduce(
    T* __restrict__ cells, Layout L, uint32_t bact0, uint8_t* const* __restrict__ bases,
    uint64_t off_bits, uint64_t off_red, int me, int world, uint64_t nwords, uint64_t seg,
    unsigned long long epoch, const unsigned long long* arrive, unsigned long long* err,
    uint32_t* __restrict__ pend) {
  wait_arrivals(arrive, world, epoch, err);
  const uint64_t lo = (uint64_t)me * seg, hi = umin64(nwords, lo + seg);
  uint32_t* red = reinterpret_cast<uint32_t*>(bases[me] + off_red);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < hi; w += stride) {
    uint32_t bits = 0;
    for (int r = 0; r < world; ++r)
      bits |= __ldcg(reinterpret_cast<const uint32_t*>(bases[r] + off_bits) + w);
    red[w - lo] = bits;
    apply_word(cells, L, bact0, w, bits, pend);
  }
}

// two-shot, phase 2: the other segments' ORs from their owners, applied
template <typename T>
__global__ void __launch_bounds__(256) k_merge_gather(
    T* __restrict__ cells, Layout L, uint32_t bact0, uint8_t* const* __restrict__ bases,
    uint64_t off_red, int me, int world, uint64_t nwords, uint64_t seg,
    unsigned long long epoch, const unsigned long long* arrive, unsigned long long* err,
    uint32_t* __restrict__ pend) {
  wait_arrivals(arrive, world, epoch, err);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t lo_me = (uint64_t)me * seg, hi_me = umin64(nwords, lo_me + seg);
  const uint64_t others = nwords - (hi_me - lo_me);
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < others; q += stride) {
    const uint64_t w = q < lo_me ? q : q + (hi_me - lo_me);
    const uint64_t owner = w / seg;
    const uint32_t bits = __ldcg(
        reinterpret_cast<const uint32_t*>(bases[owner] + off_red) + (w - owner * seg));
    apply_word(cells, L, bact0, w, bits, pend);
  }
}

// Every peer's touched keys of this slice into the registry (last-seen = t).
__global__ void k_absorb_peers(uint8_t* const* __restrict__ bases, uint64_t off_count,
                               uint64_t off_keys, int me, int world, uint64_t key_cap, RegRef R,
                               long long t) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (int r = 0; r < world; ++r) {
    if (r == me) continue;
    const uint64_t n = umin64(
        __ldcg(reinterpret_cast<const unsigned long long*>(bases[r] + off_count)), key_cap);
    const uint64_t* keys = reinterpret_cast<const uint64_t*>(bases[r] + off_keys);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
      reg_insert(R, __ldcg(keys + i), t, false);
  }
}

template <typename F>
static int with_cell_t(int bytes, F f) {
  switch (bytes) {
    case 1: return f(uint8_t{});
    case 2: return f(uint16_t{});
    default: return f(uint32_t{});
  }
}

}  // namespace vate

namespace vate {
uint64_t peer_key_cap(const vate_peer* x) { return x->key_cap; }
}  // namespace vate

using namespace vate;

extern "C" {

int vate_peer_create(vate_peer** out, vate_pool* p, vate_hosts* h, int rank, int world,
                     uint64_t key_cap, uint8_t* handle_out) {
  if (!out || !handle_out) return set_error(VATE_EVALUE, "null output pointer");
  *out = nullptr;
  int rc = enter(p);
  if (rc) return rc;
  if (!h || h->pool != p) return set_error(VATE_EVALUE, "registry does not belong to the pool");
  if (p->kind != VATE_AT) return set_error(VATE_ECONFIG, "the replica merge is defined for the AT pool only");
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
    return set_error(VATE_EVALUE, "rank/world out of range (world <= 64)");
  if (key_cap < 1) return set_error(VATE_EVALUE, "key_cap must be >= 1");
  vate_peer* x = new vate_peer();
  x->pool = p;
  x->hosts = h;
  x->rank = rank;
  x->world = world;
  x->key_cap = key_cap;
  x->nwords = (p->L.size + 31) / 32;
  x->seg = (x->nwords + world - 1) / world;
  x->seg = (x->seg + 31) & ~uint64_t(31);  // 128-B aligned segments
  const WinLayout W = win_layout(world, x->nwords, x->seg, key_cap);
  x->win_bytes = W.total;
  cudaError_t e = cudaMalloc(&x->win, x->win_bytes);
  if (e == cudaSuccess) e = cudaMemset(x->win, 0, x->win_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&x->d_bases, kMaxWorld * sizeof(uint8_t*));
  if (e == cudaSuccess) e = cudaMalloc(&x->d_err, 64);
  if (e == cudaSuccess) e = cudaMemset(x->d_err, 0, 64);
  if (e == cudaSuccess) e = cudaHostAlloc(&x->h_mirror, 64, cudaHostAllocDefault);
  cudaIpcMemHandle_t ipc;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&ipc, x->win);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    rc = cuda_fail(e, "peer window allocation / IPC export");
    vate_peer_destroy(x);
    return rc;
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle is 64 bytes");
  memcpy(handle_out, &ipc, 64);
  x->bases[rank] = x->win;
  *out = x;
  return VATE_OK;
}

int vate_peer_open(vate_peer* x, const uint8_t* handles) {
  if (!x || !handles) return set_error(VATE_EVALUE, "null peer handle");
  int rc = enter(x->pool);
  if (rc) return rc;
  if (x->opened) return set_error(VATE_EVALUE, "peer windows already opened");
  for (int r = 0; r < x->world; ++r) {
    if (r == x->rank) continue;
    cudaIpcMemHandle_t ipc;
    memcpy(&ipc, handles + 64 * r, 64);
    void* ptr = nullptr;
    VATE_CUDA(cudaIpcOpenMemHandle(&ptr, ipc, cudaIpcMemLazyEnablePeerAccess));
    x->bases[r] = static_cast<uint8_t*>(ptr);
  }
  VATE_CUDA(cudaMemcpy(x->d_bases, x->bases, kMaxWorld * sizeof(uint8_t*),
                       cudaMemcpyHostToDevice));
  x->opened = true;
  return VATE_OK;
}

int vate_peer_set_mode(vate_peer* x, int mode) {
  if (!x) return set_error(VATE_EVALUE, "null peer handle");
  if (mode < 0 || mode > 2) return set_error(VATE_EVALUE, "mode must be 0 (auto), 1 or 2");
  x->mode = mode;
  return VATE_OK;
}

int vate_peer_destroy(vate_peer* x) {
  if (!x) return VATE_OK;
  cudaSetDevice(x->pool->device);
  if (x->opened) {
    cudaStreamSynchronize(x->pool->stream);
    for (int r = 0; r < x->world; ++r)
      if (r != x->rank && x->bases[r]) cudaIpcCloseMemHandle(x->bases[r]);
  }
  if (x->win) cudaFree(x->win);
  if (x->d_bases) cudaFree(x->d_bases);
  if (x->d_err) cudaFree(x->d_err);
  if (x->h_mirror) cudaFreeHost(x->h_mirror);
  delete x;
  return VATE_OK;
}

// One slice's exchange; see the file comment.  Called after this rank's scans
// of slice t and before its estimate; returns once the merged cells and the
// union host registry are in place (one host sync for the registry drain, one
// at the end).
int vate_peer_exchange(vate_peer* x, int64_t t, uint64_t* touched_total) {
  if (!x) return set_error(VATE_EVALUE, "null peer handle");
  vate_pool* p = x->pool;
  vate_hosts* h = x->hosts;
  int rc = enter(p);
  if (rc) return rc;
  if (!x->opened) return set_error(VATE_EVALUE, "peer windows not opened (vate_peer_open)");
  const unsigned long long epoch = ++x->epoch;
  const int par = (int)(epoch & 1);
  const WinLayout W = win_layout(x->world, x->nwords, x->seg, x->key_cap);
  auto* own_arrive = reinterpret_cast<const unsigned long long*>(x->win + W.arrive);
  auto* own_count = reinterpret_cast<unsigned long long*>(x->win + W.count) + par;
  const bool two_shot = x->mode == 2 || (x->mode == 0 && x->world > 2);
  const uint32_t grid = 148u * 8u;

  // 1. this rank's dirty bitmap and touched keys into its window: a deferred
  // pool's pending marks are exactly the cells it set (a 2^c/8-byte copy); a
  // direct-store pool derives them from a pass over its cells
  uint32_t* pend = p->deferred ? pend_ptr(p) : nullptr;
  if (pend) {
    if (p->pend_dirty)
      VATE_CUDA(cudaMemcpyAsync(x->win + W.bits[par], pend, x->nwords * 4,
                                cudaMemcpyDeviceToDevice, p->stream));
    else
      VATE_CUDA(cudaMemsetAsync(x->win + W.bits[par], 0, x->nwords * 4, p->stream));
  } else {
    rc = with_cell_t(p->cell_bytes, [&](auto tag) -> int {
      using T = decltype(tag);
      VATE_LAUNCH(p, VATE_K_OTHER, grid_for(x->nwords, kThreads), kThreads, 0, k_dirty_into<T>,
                  (const T*)p->cells, p->L, p->bact0,
                  reinterpret_cast<uint32_t*>(x->win + W.bits[par]), x->nwords);
      return VATE_OK;
    });
    if (rc) return rc;
  }
  rc = hosts_touched_launch(h, t, reinterpret_cast<uint64_t*>(x->win + W.keys[par]), x->key_cap,
                            own_count);
  if (rc) return rc;
  VATE_CUDA(cudaMemcpyAsync(x->h_mirror + 1, own_count, 8, cudaMemcpyDeviceToHost, p->stream));

  // 2. arrive, then the fused OR-and-apply over peer memory
  VATE_LAUNCH(p, VATE_K_OTHER, 1, 64, 0, k_arrive, x->d_bases, W.arrive, 0, x->rank, x->world,
              epoch);
  rc = with_cell_t(p->cell_bytes, [&](auto tag) -> int {
    using T = decltype(tag);
    if (!two_shot) {
      VATE_LAUNCH(p, VATE_K_OTHER, grid, 256, 0, k_merge_oneshot<T>, (T*)p->cells, p->L, p->bact0,
                  x->d_bases, W.bits[par], x->world, x->nwords, epoch, own_arrive, x->d_err, pend);
    } else {
      VATE_LAUNCH(p, VATE_K_OTHER, grid, 256, 0, k_merge_reduce<T>, (T*)p->cells, p->L, p->bact0,
                  x->d_bases, W.bits[par], W.red[par], x->rank, x->world, x->nwords, x->seg, epoch, own_arrive,
                  x->d_err, pend);
      VATE_LAUNCH(p, VATE_K_OTHER, 1, 64, 0, k_arrive, x->d_bases, W.arrive, 1, x->rank, x->world,
                  epoch);
      VATE_LAUNCH(p, VATE_K_OTHER, grid, 256, 0, k_merge_gather<T>, (T*)p->cells, p->L, p->bact0,
                  x->d_bases, W.red[par], x->rank, x->world, x->nwords, x->seg, epoch,
                  own_arrive + kMaxWorld, x->d_err, pend);
    }
    return VATE_OK;
  });
  if (rc) return rc;
  if (pend) p->pend_dirty = true;
  const uint64_t wb = x->nwords * 4;
  x->nvlink_bytes = two_shot ? 2 * (wb / x->world) * (x->world - 1) : wb * (x->world - 1);

  // 3. the peers' touched hosts into this registry (the barrier above ordered them)
  h->note_t(t);
  for (int attempt = 0; attempt < 3; ++attempt) {
    VATE_LAUNCH(p, VATE_K_REGISTRY, 148u * 16u, kThreads, 0, k_absorb_peers, x->d_bases,
                W.count + 8 * par, W.keys[par], x->rank, x->world, x->key_cap, h->ref(), (long long)t);
    VATE_CUDA(cudaMemcpyAsync(x->h_mirror, x->d_err, 8, cudaMemcpyDeviceToHost, p->stream));
    uint64_t novf = 0, ovf_cap = 0;
    rc = hosts_ovf_state(h, &novf, &ovf_cap);  // syncs the stream
    if (rc) return rc;
    if (x->h_mirror[0]) {
      cudaMemsetAsync(x->d_err, 0, 8, p->stream);
      return set_error(VATE_ECUDA, "peer exchange: timed out waiting for a peer's arrival");
    }
    if (x->h_mirror[1] > x->key_cap)
      return set_error(VATE_EVALUE, "peer exchange: touched hosts exceed key_cap");
    if (novf <= ovf_cap) break;
    // parked inserts overran the list: enlarge it and redo the (idempotent) absorb
    rc = hosts_ovf_reset(h, novf);
    if (rc) return rc;
  }
  rc = hosts_drain(h);  // parked inserts, growth past the load bound
  if (rc) return rc;
  if (touched_total) {
    // own count is in the mirror; the peers' counts are read from their windows
    uint64_t total = x->h_mirror[1];
    for (int r = 0; r < x->world; ++r) {
      if (r == x->rank) continue;
      unsigned long long c = 0;
      VATE_CUDA(cudaMemcpy(&c, x->bases[r] + W.count + 8 * par, 8, cudaMemcpyDeviceToHost));
      total += c;
    }
    *touched_total = total;
  }
  return VATE_OK;
}

int vate_peer_info(const vate_peer* x, uint64_t* window_bytes, uint64_t* nvlink_bytes,
                   int* two_shot) {
  if (!x) return set_error(VATE_EVALUE, "null peer handle");
  if (window_bytes) *window_bytes = x->win_bytes;
  if (nvlink_bytes) *nvlink_bytes = x->nvlink_bytes;
  if (two_shot) *two_shot = x->mode == 2 || (x->mode == 0 && x->world > 2);
  return VATE_OK;
}

}  // extern "C"
