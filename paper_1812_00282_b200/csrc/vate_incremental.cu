// vate_incremental.cu -- exact incremental g0 for the fused per-slice estimate.
//
// g0(h) = #{ j < g : inactive(H(h, j)) } (estimator.py:114-123) is recomputed
// from scratch by the reference every slice: H*g hashed gathers (1.02 G at 1M
// hosts).  Between consecutive slices only the cells whose inactive bit flipped
// can change any g0, and in steady traffic that is a tiny fraction of the pool
// (DESIGN.md §4b measures ~0.07% per slice on the cfg-2 trace).  So:
//
//   * an inverse index (CSR: off[cell] .. off[cell+1] -> host ids) over a host
//     set X holds every (host, slot) pair once, duplicates included;
//   * g0x[i] is g0 of X[i] for the previous bitmap bprev;
//   * per slice: delta = bitmap XOR bprev; each flipped cell adds +-1 to the g0x
//     of every (host, slot) pair that maps to it; hosts of the active set found
//     in X read g0x, the rest ("misses", e.g. new hosts) take the full gather.
//
// All integer arithmetic: the result equals the full recompute exactly, which
// the GPU parity tests check slice by slice against the oracle.  When the delta
// touches more than 1/4 of a full recompute, g0x is refreshed by one full
// gather over X instead; X is rebuilt from the active set when misses exceed
// 5% or X grows past twice the active set.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <string>

#include <utility>

#include "vate_internal.cuh"

namespace vate {

__device__ __forceinline__ uint64_t host_base(uint64_t aip, const HashParams& H) {
  return ((uint64_t)((uint32_t)aip * (uint32_t)kPhi) << 32) + H.cs;  // ((aip<<32)*phi + cs)
}

// entries per cell over all (host, slot) pairs of X
__global__ void k_inc_count(const uint64_t* __restrict__ X, uint64_t total, DivU64 dg,
                            HashParams H, uint32_t* __restrict__ cnt) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
    uint64_t j;
    const uint64_t h = div_u64(i, dg, &j);
    const uint64_t cell = mix64(host_base(X[h], H) + j * kPhi) & H.cmask;
    atomicAdd(cnt + cell, 1u);
  }
}

__global__ void k_inc_fill(const uint64_t* __restrict__ X, uint64_t total, DivU64 dg, HashParams H,
                           uint32_t* __restrict__ cursor, uint32_t* __restrict__ ent) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
    uint64_t j;
    const uint64_t h = div_u64(i, dg, &j);
    const uint64_t cell = mix64(host_base(X[h], H) + j * kPhi) & H.cmask;
    ent[atomicAdd(cursor + cell, 1u)] = (uint32_t)h;
  }
}

// One warp per flipped cell: +1 to every pair that became inactive, -1 otherwise.
// Early form (guard != nullptr, launched before the slice's host round trip):
// the kernel itself takes the host's delta-vs-refresh decision from the same
// counters -- the delta list is complete (count <= cap) and its work is at most
// a quarter of a full recompute (work <= nhosts * g / 4) -- and does nothing
// otherwise; the host repeats the decision after the round trip.
struct ApplyGuard {
  const unsigned long long* work;
  const unsigned long long* nhosts;
  uint64_t g;
};
__device__ __forceinline__ bool apply_allowed(const unsigned long long* count, uint64_t cap,
                                              const ApplyGuard& G) {
  return *count <= cap && *G.work <= (*G.nhosts * G.g) / 4;
}

__global__ void k_inc_apply(const unsigned long long* __restrict__ list,
                            const unsigned long long* count, uint64_t cap,
                            const uint32_t* __restrict__ off, const uint32_t* __restrict__ ent,
                            int32_t* __restrict__ g0x, ApplyGuard G) {
  if (G.work && !apply_allowed(count, cap, G)) return;
  const uint64_t n = umin64(*count, cap);
  const int lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    const unsigned long long v = list[i];
    const uint64_t cell = v & 0xFFFFFFFFull;
    const int d = (v >> 32) ? 1 : -1;
    const uint32_t e1 = off[cell + 1];
    for (uint32_t e = off[cell] + lane; e < e1; e += 32) atomicAdd(g0x + ent[e], d);
  }
}

// Sorted active hosts A -> g0 from the index where present, else a miss.
// Both lists are ascending, so each thread takes a run of kRun consecutive
// hosts: one binary search places the first, the rest advance linearly
// (typically one step per host), falling back to a search on long gaps.
constexpr int kRun = 8;
__global__ void k_inc_lookup(const uint64_t* __restrict__ A, uint64_t n,
                             const uint64_t* __restrict__ X, uint64_t m,
                             const int32_t* __restrict__ g0x, int32_t* __restrict__ g0,
                             uint32_t* __restrict__ miss, unsigned long long* nmiss) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * kRun;
  for (uint64_t i0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * kRun; i0 < n; i0 += stride) {
    uint64_t lo = 0;
    bool placed = false;
    for (int r = 0; r < kRun && i0 + r < n; ++r) {
      const uint64_t i = i0 + r;
      const uint64_t a = A[i];
      int walked = 0;
      while (placed && lo < m && X[lo] < a && walked < 16) {
        ++lo;
        ++walked;
      }
      if (!placed || (lo < m && X[lo] < a)) {  // first host of the run, or a long gap
        uint64_t hi = m;
        while (lo < hi) {
          const uint64_t mid = (lo + hi) >> 1;
          if (X[mid] < a) lo = mid + 1;
          else hi = mid;
        }
        placed = true;
      }
      if (lo < m && X[lo] == a) g0[i] = g0x[lo];
      else miss[atomicAdd(nmiss, 1ull)] = (uint32_t)i;
    }
  }
}

__device__ __forceinline__ uint64_t lower_bound_u64(const uint64_t* __restrict__ v, uint64_t n,
                                                    uint64_t key) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (v[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Merge positions of X (m, sorted) and Y (y, sorted, disjoint from X) in X u Y.
__global__ void k_ext_positions(const uint64_t* __restrict__ X, uint64_t m,
                                const int32_t* __restrict__ g0x, const uint64_t* __restrict__ Ys,
                                uint64_t y, const int32_t* __restrict__ Yg0s,
                                uint32_t* __restrict__ remapX, uint32_t* __restrict__ posY,
                                uint64_t* __restrict__ Xn, int32_t* __restrict__ g0xn) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m + y; i += stride) {
    if (i < m) {
      const uint64_t a = X[i];
      const uint64_t p = i + lower_bound_u64(Ys, y, a);
      remapX[i] = (uint32_t)p;
      Xn[p] = a;
      g0xn[p] = g0x[i];
    } else {
      const uint64_t j = i - m, b = Ys[j];
      const uint64_t p = j + lower_bound_u64(X, m, b);
      posY[j] = (uint32_t)p;
      Xn[p] = b;
      g0xn[p] = Yg0s[j];
    }
  }
}

__global__ void k_ext_offsets(const uint32_t* __restrict__ offX, const uint32_t* __restrict__ offY,
                              uint64_t n, uint32_t* __restrict__ off2) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < n; c += stride)
    off2[c] = offX[c] + offY[c];
}

// X's entries into the merged CSR (renumbered), one warp per run of cells.
__global__ void k_ext_copy(const uint32_t* __restrict__ offX, const uint32_t* __restrict__ entX,
                           const uint32_t* __restrict__ off2, const uint32_t* __restrict__ remapX,
                           uint64_t ncells, uint32_t* __restrict__ ent2) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t c = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; c < ncells; c += warps) {
    const uint32_t a = offX[c], b = offX[c + 1], d = off2[c];
    for (uint32_t e = a + lane; e < b; e += 32) ent2[d + (e - a)] = remapX[entX[e]];
  }
}

// Y's (host, slot) pairs after X's entries of each cell.
__global__ void k_ext_fill_y(const uint64_t* __restrict__ Ys, uint64_t total, DivU64 dg,
                             HashParams H, const uint32_t* __restrict__ offX,
                             const uint32_t* __restrict__ off2, const uint32_t* __restrict__ posY,
                             uint32_t* __restrict__ cursor, uint32_t* __restrict__ ent2) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
    uint64_t j;
    const uint64_t h = div_u64(i, dg, &j);
    const uint64_t cell = mix64(host_base(Ys[h], H) + j * kPhi) & H.cmask;
    const uint32_t at = off2[cell] + (offX[cell + 1] - offX[cell]) + atomicAdd(cursor + cell, 1u);
    ent2[at] = posY[h];
  }
}

void inc_release(vate_pool* p) {
  IncIndex& I = p->inc;
  for (cudaEvent_t& e : I.ev_rb)
    if (e) {
      cudaEventDestroy(e);
      e = nullptr;
    }
  for (DevBuf* b : {&I.X, &I.g0x, &I.off, &I.ent, &I.cursor, &I.bprev, &I.dlist, &I.miss, &I.scan_tmp,
                    &I.Ykeys, &I.Yg0, &I.Ys, &I.Yg0s, &I.remap, &I.posY, &I.Xn, &I.g0xn, &I.off2,
                    &I.offY, &I.ent2, &I.sort_tmp})
    b->release();
  I.valid = false;
  I.m = 0;
}

static void swap_buf(DevBuf& a, DevBuf& b) {
  std::swap(a.ptr, b.ptr);
  std::swap(a.bytes, b.bytes);
}

// Whether the coming bitmap pass should also emit the delta against bprev
// (index live and built for these parameters).
bool inc_delta_ready(vate_pool* p, uint64_t g, uint64_t cs, int kp) {
  IncIndex& I = p->inc;
  I.delta_launched = p->opt_inc && I.valid && !I.want_rebuild && I.g == g && I.cs == cs &&
                     I.kp == kp;
  return I.delta_launched;
}

// Build the inverse index over X = hosts (sorted, n), with g0x = g0_dev (already
// computed on the current bitmap), and take the current bitmap as bprev.
static int inc_rebuild(vate_pool* p, const uint64_t* hosts, uint64_t n, HashParams H, int kp,
                       const int32_t* g0_dev) {
  IncIndex& I = p->inc;
  I.valid = false;
  const uint64_t total = n * H.g;
  const uint64_t S = p->L.size, nwords = (S + 31) / 32;
  if (n == 0 || total >= (1ull << 32)) return VATE_OK;  // u32 offsets only
  // memory: ent 4*total, off/cursor 4*(S+1) each; keep a quarter of free memory spare
  size_t free_b = 0, tot_b = 0;
  VATE_CUDA(cudaMemGetInfo(&free_b, &tot_b));
  const uint64_t need = 4 * total + 8 * (S + 2) + 8 * n * 2 + 4 * nwords;
  if (need + tot_b / 4 > free_b + I.ent.bytes + I.off.bytes + I.cursor.bytes) return VATE_OK;
  int rc;
  if ((rc = I.X.ensure(n * 8 + 8)) || (rc = I.g0x.ensure(n * 4 + 4)) ||
      (rc = I.off.ensure((S + 2) * 4)) || (rc = I.cursor.ensure((S + 2) * 4)) ||
      (rc = I.ent.ensure(total * 4 + 4)) || (rc = I.bprev.ensure(nwords * 4 + 16)) ||
      (rc = I.miss.ensure(n * 4 + 4)))
    return rc;
  I.dlist_cap = S / 8 + 1024;
  if ((rc = I.dlist.ensure(I.dlist_cap * 8))) return rc;
  for (cudaEvent_t& e : I.ev_rb)
    if (!e) VATE_CUDA(cudaEventCreate(&e));
  if (I.rb_timing) {  // fold in a previous rebuild not yet read
    float ms = 0.f;
    VATE_CUDA(cudaEventSynchronize(I.ev_rb[1]));
    VATE_CUDA(cudaEventElapsedTime(&ms, I.ev_rb[0], I.ev_rb[1]));
    I.rebuild_ms += ms;
  }
  VATE_CUDA(cudaEventRecord(I.ev_rb[0], p->stream));
  VATE_CUDA(cudaMemcpyAsync(I.X.ptr, hosts, n * 8, cudaMemcpyDeviceToDevice, p->stream));
  VATE_CUDA(cudaMemcpyAsync(I.g0x.ptr, g0_dev, n * 4, cudaMemcpyDeviceToDevice, p->stream));
  VATE_CUDA(cudaMemsetAsync(I.cursor.ptr, 0, (S + 1) * 4, p->stream));
  const DivU64 dg = make_div(H.g);
  VATE_LAUNCH(p, VATE_K_OTHER, grid_for(total, kThreads, 148u * 32u), kThreads, 0, k_inc_count,
              I.X.as<const uint64_t>(), total, dg, H, I.cursor.as<uint32_t>());
  size_t tmp = 0;
  VATE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, I.cursor.as<uint32_t>(),
                                          I.off.as<uint32_t>(), (int64_t)(S + 1), p->stream));
  if ((rc = I.scan_tmp.ensure(tmp + 256))) return rc;
  VATE_CUDA(cub::DeviceScan::ExclusiveSum(I.scan_tmp.ptr, tmp, I.cursor.as<uint32_t>(),
                                          I.off.as<uint32_t>(), (int64_t)(S + 1), p->stream));
  p->launches += 2;
  VATE_CUDA(cudaMemcpyAsync(I.cursor.ptr, I.off.ptr, (S + 1) * 4, cudaMemcpyDeviceToDevice,
                            p->stream));
  VATE_LAUNCH(p, VATE_K_OTHER, grid_for(total, kThreads, 148u * 32u), kThreads, 0, k_inc_fill,
              I.X.as<const uint64_t>(), total, dg, H, I.cursor.as<uint32_t>(),
              I.ent.as<uint32_t>());
  VATE_CUDA(cudaMemcpyAsync(I.bprev.ptr, p->bitmap.ptr, nwords * 4, cudaMemcpyDeviceToDevice,
                            p->stream));
  VATE_CUDA(cudaEventRecord(I.ev_rb[1], p->stream));
  I.rb_timing = true;
  I.miss_accum = 0;
  I.extend_accum = 0;
  I.want_extend = false;
  I.m = n;
  I.g = H.g;
  I.cs = H.cs;
  I.kp = kp;
  I.valid = true;
  I.want_rebuild = false;
  I.rebuilds++;
  I.identity_ok = true;  // X is exactly this active list
  I.identity_version = p->sorted_version;
  return VATE_OK;
}

// Merge the y hosts captured by the previous lookup (Ykeys/Yg0, valid for
// bprev) into X: sorted union, renumbered CSR with their (host, slot) pairs.
// One streaming pass over the index (~8 B per entry) instead of a rebuild.
static int inc_extend(vate_pool* p, uint64_t y, HashParams H) {
  IncIndex& I = p->inc;
  const uint64_t m = I.m, S = p->L.size, mn = m + y, total_new = mn * H.g;
  if (y == 0 || total_new >= (1ull << 32)) return VATE_OK;
  int rc;
  if ((rc = I.Ys.ensure(y * 8 + 8)) || (rc = I.Yg0s.ensure(y * 4 + 4)) ||
      (rc = I.remap.ensure(m * 4 + 4)) || (rc = I.posY.ensure(y * 4 + 4)) ||
      (rc = I.Xn.ensure(mn * 8 + 8)) || (rc = I.g0xn.ensure(mn * 4 + 4)) ||
      (rc = I.off2.ensure((S + 2) * 4)) || (rc = I.offY.ensure((S + 2) * 4)) ||
      (rc = I.ent2.ensure(total_new * 4 + 4)) || (rc = I.miss.ensure(mn * 4 + 4)))
    return rc;
  size_t tmp = 0;
  VATE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, I.Ykeys.as<const unsigned long long>(),
                                            I.Ys.as<unsigned long long>(), I.Yg0.as<const int32_t>(),
                                            I.Yg0s.as<int32_t>(), (int64_t)y, 0, 64, p->stream));
  if ((rc = I.sort_tmp.ensure(tmp + 256))) return rc;
  VATE_CUDA(cub::DeviceRadixSort::SortPairs(I.sort_tmp.ptr, tmp, I.Ykeys.as<const unsigned long long>(),
                                            I.Ys.as<unsigned long long>(), I.Yg0.as<const int32_t>(),
                                            I.Yg0s.as<int32_t>(), (int64_t)y, 0, 64, p->stream));
  p->launches += 9;
  VATE_LAUNCH(p, VATE_K_OTHER, grid_for(mn, kThreads, 148u * 32u), kThreads, 0, k_ext_positions,
              I.X.as<const uint64_t>(), m, I.g0x.as<const int32_t>(), I.Ys.as<const uint64_t>(), y,
              I.Yg0s.as<const int32_t>(), I.remap.as<uint32_t>(), I.posY.as<uint32_t>(),
              I.Xn.as<uint64_t>(), I.g0xn.as<int32_t>());
  // Y's CSR offsets: count, scan; merged offsets = X's + Y's
  const DivU64 dg = make_div(H.g);
  VATE_CUDA(cudaMemsetAsync(I.cursor.ptr, 0, (S + 1) * 4, p->stream));
  VATE_LAUNCH(p, VATE_K_OTHER, grid_for(y * H.g, kThreads, 148u * 32u), kThreads, 0, k_inc_count,
              I.Ys.as<const uint64_t>(), y * H.g, dg, H, I.cursor.as<uint32_t>());
  tmp = 0;
  VATE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, I.cursor.as<uint32_t>(), I.offY.as<uint32_t>(),
                                          (int64_t)(S + 1), p->stream));
  if ((rc = I.scan_tmp.ensure(tmp + 256))) return rc;
  VATE_CUDA(cub::DeviceScan::ExclusiveSum(I.scan_tmp.ptr, tmp, I.cursor.as<uint32_t>(),
                                          I.offY.as<uint32_t>(), (int64_t)(S + 1), p->stream));
  p->launches += 2;
  VATE_LAUNCH(p, VATE_K_OTHER, grid_for(S + 1, kThreads, 148u * 32u), kThreads, 0, k_ext_offsets,
              I.off.as<const uint32_t>(), I.offY.as<const uint32_t>(), S + 1, I.off2.as<uint32_t>());
  VATE_LAUNCH(p, VATE_K_OTHER, grid_for(S * 32, kThreads, 148u * 32u), kThreads, 0, k_ext_copy,
              I.off.as<const uint32_t>(), I.ent.as<const uint32_t>(), I.off2.as<const uint32_t>(),
              I.remap.as<const uint32_t>(), S, I.ent2.as<uint32_t>());
  VATE_CUDA(cudaMemsetAsync(I.cursor.ptr, 0, (S + 1) * 4, p->stream));
  VATE_LAUNCH(p, VATE_K_OTHER, grid_for(y * H.g, kThreads, 148u * 32u), kThreads, 0, k_ext_fill_y,
              I.Ys.as<const uint64_t>(), y * H.g, dg, H, I.off.as<const uint32_t>(),
              I.off2.as<const uint32_t>(), I.posY.as<const uint32_t>(), I.cursor.as<uint32_t>(),
              I.ent2.as<uint32_t>());
  swap_buf(I.X, I.Xn);
  swap_buf(I.g0x, I.g0xn);
  swap_buf(I.off, I.off2);
  swap_buf(I.ent, I.ent2);
  I.m = mn;
  I.identity_ok = false;
  I.extend_accum = 0;
  I.extends++;
  return VATE_OK;
}

// g0 of the sorted active hosts into p->g0 (after the estimate's round trip).
int inc_compute_g0(vate_pool* p, const uint64_t* hosts, uint64_t n, HashParams H, int kp) {
  IncIndex& I = p->inc;
  int rc;
  if ((rc = p->g0.ensure(n * 4 + 4))) return rc;
  const bool same_req = I.req_g == H.g && I.req_cs == H.cs && I.req_kp == kp;
  I.req_g = H.g;
  I.req_cs = H.cs;
  I.req_kp = kp;
  if (I.delta_launched) {
    I.delta_launched = false;
    if (I.want_extend) {  // last slice's misses join X before this slice's delta
      I.want_extend = false;
      if ((rc = inc_extend(p, I.last_misses, H))) return rc;
    }
    const uint64_t dcells = p->h_ctr[C_DCNT], dwork = p->h_ctr[C_DWORK];
    I.last_delta_cells = dcells;
    I.last_delta_work = dwork;
    // the early kernel (if launched) decided on the same counters and on the
    // active count of the first compaction (begin_complete made the stream wait
    // for it before anything could reset that count)
    const bool applied = I.early_apply && dcells <= I.dlist_cap &&
                         dwork <= I.early_nhosts * H.g / 4;
    I.early_apply = false;
    if (dcells <= I.dlist_cap && dwork <= n * H.g / 4) {
      if (!applied)
        VATE_LAUNCH(p, VATE_K_G0, grid_for(umin64(dcells, 1u << 20) * 32 + 32, kThreads,
                                           148u * 16u),
                    kThreads, 0, k_inc_apply, I.dlist.as<const unsigned long long>(),
                    p->d_ctr + C_DCNT, I.dlist_cap, I.off.as<const uint32_t>(),
                    I.ent.as<const uint32_t>(), I.g0x.as<int32_t>(), ApplyGuard{});
      I.delta_slices++;
    } else {  // too much churn for the delta: refresh every host of X in one gather
      if ((rc = launch_g0(p, I.X.as<const uint64_t>(), I.m, H, I.g0x.as<int32_t>()))) return rc;
      I.refresh_slices++;
    }
    if (I.identity_ok && I.identity_version == p->sorted_version && I.m == n) {
      p->g0_src = I.g0x.as<const int32_t>();  // the active list is X itself
      I.identity_slices++;
    } else {
      I.identity_ok = false;
      if ((rc = I.miss.ensure(n * 4 + 4))) return rc;
      VATE_CUDA(cudaMemsetAsync(p->d_ctr + C_MISS, 0, 8, p->stream));
      VATE_LAUNCH(p, VATE_K_G0, grid_for((n + kRun - 1) / kRun, kThreads, 148u * 16u), kThreads, 0,
                  k_inc_lookup, hosts,
                  n, I.X.as<const uint64_t>(), I.m, I.g0x.as<const int32_t>(), p->g0.as<int32_t>(),
                  I.miss.as<uint32_t>(), p->d_ctr + C_MISS);
      // the misses' g0 gather also captures them (keys + g0, list order) so the
      // next slice can merge them into X
      if ((rc = I.Ykeys.ensure(n * 8 + 8)) || (rc = I.Yg0.ensure(n * 4 + 4))) return rc;
      if ((rc = launch_g0_list(p, hosts, I.miss.as<const uint32_t>(), p->d_ctr + C_MISS, n, H,
                               p->g0.as<int32_t>(), I.Ykeys.as<uint64_t>(), I.Yg0.as<int32_t>())))
        return rc;
      VATE_CUDA(cudaMemcpyAsync(p->h_ctr + C_MISS, p->d_ctr + C_MISS, 8, cudaMemcpyDeviceToHost,
                                p->stream));
      I.lookup_pending = true;
      I.lookup_version = p->sorted_version;
      p->g0_src = p->g0.as<const int32_t>();
    }
    swap_buf(p->bitmap, I.bprev);  // g0x now matches this slice's bitmap
    I.last_n = n;
    if (I.m > 2 * n) I.want_rebuild = true;
    return VATE_OK;
  }
  // full recompute; then (re)build the index over this active set
  if ((rc = launch_g0(p, hosts, n, H, p->g0.as<int32_t>()))) return rc;
  p->g0_src = p->g0.as<const int32_t>();
  I.full_slices++;
  if (p->opt_inc && (same_req || !I.valid)) {
    if ((rc = inc_rebuild(p, hosts, n, H, kp, p->g0.as<const int32_t>()))) return rc;
  }
  I.last_n = n;
  return VATE_OK;
}

}  // namespace vate

namespace vate {
// Launch the delta apply right behind the bitmap pass, on the aux stream, so it
// overlaps the slice's host round trip (see k_inc_apply).  Only in steady
// state: the index is live, no previous lookup is pending (its misses could
// extend X, which must precede the delta) and the whole active set is this
// pool's (no multi-GPU share).  nhosts_dev is the registry's active count.
int inc_apply_early(vate_pool* p, const unsigned long long* nhosts_dev, uint64_t g) {
  IncIndex& I = p->inc;
  if (!I.delta_launched || I.lookup_pending || I.want_extend || !p->opt_concurrent) return VATE_OK;
  if (!I.ev_apply) VATE_CUDA(cudaEventCreateWithFlags(&I.ev_apply, cudaEventDisableTiming));
  VATE_CUDA(cudaEventRecord(I.ev_apply, p->stream));           // bitmap + delta list done
  VATE_CUDA(cudaStreamWaitEvent(p->aux_stream, I.ev_apply, 0));
  std::swap(p->stream, p->aux_stream);
  cudaEvent_t ta = nullptr;
  timing_begin(p, VATE_K_G0, &ta);
  k_inc_apply<<<p->cap_inc, kThreads, 0, p->stream>>>(
      I.dlist.as<const unsigned long long>(), p->d_ctr + C_DCNT, I.dlist_cap,
      I.off.as<const uint32_t>(), I.ent.as<const uint32_t>(), I.g0x.as<int32_t>(),
      ApplyGuard{p->d_ctr + C_DWORK, nhosts_dev, g});
  p->launches++;
  timing_end(p, VATE_K_G0, ta);
  const cudaError_t le = cudaGetLastError();
  std::swap(p->stream, p->aux_stream);
  if (le != cudaSuccess) return cuda_fail(le, "k_inc_apply (early)");
  VATE_CUDA(cudaEventRecord(I.ev_apply, p->aux_stream));
  I.early_apply = true;
  return VATE_OK;
}
}  // namespace vate
