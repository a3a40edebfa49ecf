// vate_estimate.cu -- the per-host estimate: g0 gather over the inactive
// bitmap, the float path, the floor filter, and the fused per-slice driver.
//
// Reference: estimator.py:107-181 (host_cells, inactive_virtual_counts,
// reports_from_counts, estimate_hosts), pipeline.py:120-138 (_estimate).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include <utility>

#include "vate_internal.cuh"

namespace vate {

int check_width(vate_pool* p, int k_prime);    // vate_pool.cu

// g0[h] = #{ j < g : bitmap bit of H(aip_h, j) is set }  (estimator.py:107-123)
//
// LPH lanes cooperate on one host.  Keys of one host differ only in the low
// word, so ((aip<<32)|j)*phi + cs = base + j*phi with
// base = ((uint32(aip) * uint32(phi)) << 32) + cs, and each lane walks its
// slots with one 64-bit add.  The bitmap (2^c/8 bytes) stays L2-resident.
// LIST: gather only the hosts hosts[idx[i]], i < min(*count, n) (the misses of
// the incremental path), writing g0[idx[i]].
template <int LPH, bool LIST = false>
__global__ void __launch_bounds__(kThreads) k_g0(const uint64_t* __restrict__ hosts, uint64_t n,
                                                 const uint32_t* __restrict__ bitmap,
                                                 HashParams H, int32_t* __restrict__ g0,
                                                 const uint32_t* __restrict__ idx = nullptr,
                                                 const unsigned long long* count = nullptr,
                                                 uint64_t* __restrict__ yk = nullptr,
                                                 int32_t* __restrict__ yg = nullptr) {
  if (LIST) n = umin64(n, *count);
  const int lane = threadIdx.x & 31;
  const int sub = lane & (LPH - 1);
  const unsigned gmask = LPH == 32 ? 0xffffffffu : (((1u << LPH) - 1u) << (lane & ~(LPH - 1)));
  const uint64_t groups = ((uint64_t)gridDim.x * blockDim.x) / LPH;
  const uint64_t step = (uint64_t)LPH * kPhi;
  const uint64_t g = H.g;
  for (uint64_t h = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / LPH; h < n; h += groups) {
    const uint64_t hi = LIST ? idx[h] : h;
    const uint64_t aip = hosts[hi];
    uint64_t x = ((uint64_t)((uint32_t)aip * (uint32_t)kPhi) << 32) + H.cs + (uint64_t)sub * kPhi;
    uint32_t cnt = 0;
    uint64_t j = sub;
    // four independent gathers in flight per lane
    for (; j + 3 * LPH < g; j += 4 * LPH) {
      const uint64_t c0 = mix64(x) & H.cmask;
      const uint64_t c1 = mix64(x + step) & H.cmask;
      const uint64_t c2 = mix64(x + 2 * step) & H.cmask;
      const uint64_t c3 = mix64(x + 3 * step) & H.cmask;
      const uint32_t w0 = __ldg(bitmap + (c0 >> 5));
      const uint32_t w1 = __ldg(bitmap + (c1 >> 5));
      const uint32_t w2 = __ldg(bitmap + (c2 >> 5));
      const uint32_t w3 = __ldg(bitmap + (c3 >> 5));
      cnt += ((w0 >> (c0 & 31)) & 1u) + ((w1 >> (c1 & 31)) & 1u) + ((w2 >> (c2 & 31)) & 1u) +
             ((w3 >> (c3 & 31)) & 1u);
      x += 4 * step;
    }
    for (; j < g; j += LPH) {
      const uint64_t c0 = mix64(x) & H.cmask;
      cnt += (__ldg(bitmap + (c0 >> 5)) >> (c0 & 31)) & 1u;
      x += step;
    }
#pragma unroll
    for (int o = LPH / 2; o; o >>= 1) cnt += __shfl_xor_sync(gmask, cnt, o);
    if (sub == 0) {
      g0[hi] = (int32_t)cnt;
      if (LIST && yk) {  // the list's hosts and g0 in list order (the index capture)
        yk[h] = aip;
        yg[h] = (int32_t)cnt;
      }
    }
  }
}

// The same gather with the inactive bitmap in shared memory.  For c <= 20 one
// CTA holds the whole bitmap (<= 128 KB); for 20 < c <= 24 a thread-block
// cluster of 2^(c-20) CTAs holds it, 128 KB per CTA, and a gather of cell x
// reads word (x mod 2^20)/32 of CTA x >> 20 through distributed shared memory
// (mapa + ld.shared::cluster).  Random 4-byte LDGs are bound by the L1TEX
// wavefront rate (one 128-B line per cycle per SM); shared-memory loads are
// bound by bank conflicts instead.
__device__ __forceinline__ uint32_t ld_dsmem(uint32_t local_addr, uint32_t rank) {
  uint32_t remote, v;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(rank));
  asm("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(remote));
  return v;
}

constexpr int kDsmemLog2Bits = 20;  // bits held per CTA (128 KB)
constexpr int kDsmemThreads = 1024;

template <int LPH, bool CLUSTER>
__global__ void __launch_bounds__(kDsmemThreads, 1) k_g0_smem(
    const uint64_t* __restrict__ hosts, uint64_t n, const uint32_t* __restrict__ bitmap,
    uint32_t words_per_cta, HashParams H, int32_t* __restrict__ g0) {
  extern __shared__ uint4 smem4[];
  namespace cg = cooperative_groups;
  uint32_t rank = 0;
  if (CLUSTER) rank = cg::this_cluster().block_rank();
  {
    const uint4* src = reinterpret_cast<const uint4*>(bitmap + (uint64_t)rank * words_per_cta);
    for (uint32_t i = threadIdx.x; i < words_per_cta / 4; i += blockDim.x) smem4[i] = __ldcg(src + i);
    const uint32_t* s1 = bitmap + (uint64_t)rank * words_per_cta;
    for (uint32_t i = (words_per_cta / 4) * 4 + threadIdx.x; i < words_per_cta; i += blockDim.x)
      reinterpret_cast<uint32_t*>(smem4)[i] = s1[i];
  }
  if (CLUSTER) cg::this_cluster().sync();
  else __syncthreads();
  const uint32_t* sbits = reinterpret_cast<const uint32_t*>(smem4);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sbits);
  const uint64_t local_mask = (1ull << kDsmemLog2Bits) - 1;
  const int lane = threadIdx.x & 31;
  const int sub = lane & (LPH - 1);
  const unsigned gmask = LPH == 32 ? 0xffffffffu : (((1u << LPH) - 1u) << (lane & ~(LPH - 1)));
  const uint64_t groups = ((uint64_t)gridDim.x * blockDim.x) / LPH;
  const uint64_t step = (uint64_t)LPH * kPhi;
  const uint64_t g = H.g;
  auto bit = [&](uint64_t c) -> uint32_t {
    uint32_t w;
    if (CLUSTER) w = ld_dsmem(sbase + (uint32_t)((c & local_mask) >> 5) * 4u,
                              (uint32_t)(c >> kDsmemLog2Bits));
    else w = sbits[c >> 5];
    return (w >> (c & 31)) & 1u;
  };
  for (uint64_t h = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / LPH; h < n; h += groups) {
    const uint64_t aip = hosts[h];
    uint64_t x = ((uint64_t)((uint32_t)aip * (uint32_t)kPhi) << 32) + H.cs + (uint64_t)sub * kPhi;
    uint32_t cnt = 0;
    uint64_t j = sub;
    for (; j + 3 * LPH < g; j += 4 * LPH) {
      const uint64_t c0 = mix64(x) & H.cmask;
      const uint64_t c1 = mix64(x + step) & H.cmask;
      const uint64_t c2 = mix64(x + 2 * step) & H.cmask;
      const uint64_t c3 = mix64(x + 3 * step) & H.cmask;
      cnt += bit(c0) + bit(c1) + bit(c2) + bit(c3);
      x += 4 * step;
    }
    for (; j < g; j += LPH) {
      cnt += bit(mix64(x) & H.cmask);
      x += step;
    }
#pragma unroll
    for (int o = LPH / 2; o; o >>= 1) cnt += __shfl_xor_sync(gmask, cnt, o);
    if (sub == 0) g0[h] = (int32_t)cnt;
  }
  if (CLUSTER) cg::this_cluster().sync();  // peers may still read this CTA's bits
}

template <int LPH>
static int launch_g0_smem(vate_pool* p, const uint64_t* hosts_dev, uint64_t n, HashParams H,
                          int32_t* g0_dev) {
  const uint64_t nbits = p->L.size;
  const uint32_t cs = nbits > (1ull << kDsmemLog2Bits) ? (uint32_t)(nbits >> kDsmemLog2Bits) : 1u;
  const uint32_t words = (uint32_t)((nbits / cs + 31) / 32);
  const size_t smem = ((size_t)words * 4 + 15) & ~size_t(15);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.blockDim = dim3(kDsmemThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = p->stream;
  if (cs > 1) {
    auto kern = k_g0_smem<LPH, true>;
    VATE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (cs > 8) VATE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (p->dsmem_clusters < 0) {
      int nc = 0;
      cfg.gridDim = dim3(cs);
      VATE_CUDA(cudaOccupancyMaxActiveClusters(&nc, kern, &cfg));
      p->dsmem_clusters = nc;
    }
    if (p->dsmem_clusters < 1) return set_error(VATE_ECUDA, "no room for a DSMEM cluster");
    cfg.gridDim = dim3((uint32_t)p->dsmem_clusters * cs);
    cudaEvent_t ta = nullptr;
    timing_begin(p, VATE_K_G0, &ta);
    VATE_CUDA(cudaLaunchKernelEx(&cfg, kern, hosts_dev, n, p->bitmap.as<const uint32_t>(), words, H,
                                 g0_dev));
    timing_end(p, VATE_K_G0, ta);
  } else {
    auto kern = k_g0_smem<LPH, false>;
    VATE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
    cfg.gridDim = dim3((uint32_t)sms);
    cfg.numAttrs = 0;
    cudaEvent_t ta = nullptr;
    timing_begin(p, VATE_K_G0, &ta);
    VATE_CUDA(cudaLaunchKernelEx(&cfg, kern, hosts_dev, n, p->bitmap.as<const uint32_t>(), words, H,
                                 g0_dev));
    timing_end(p, VATE_K_G0, ta);
  }
  p->launches++;
  return VATE_OK;
}

int launch_g0(vate_pool* p, const uint64_t* hosts_dev, uint64_t n, HashParams H,
              int32_t* g0_dev) {
  // lanes per host: the next power of two >= g, at most a warp
  int lph = 1;
  while (lph < 32 && (uint64_t)lph < H.g) lph <<= 1;
  const uint64_t threads = n * (uint64_t)lph;
  const uint32_t grid = grid_for(threads, kThreads, 148u * 64u);
  const uint32_t* bm = p->bitmap.as<const uint32_t>();
  // the smem/DSMEM gather needs the whole bitmap in <= 16 CTAs of 128 KB
  const bool smem_ok = p->c <= kDsmemLog2Bits + 4 && p->c >= 5;
  // auto: only when one CTA holds the whole bitmap (c <= 20); the cluster/DSMEM
  // form measured 4x slower than the L2 gather on B200 (profiles/)
  const bool use_smem = smem_ok && (p->opt_g0 == 2 || (p->opt_g0 == 0 && p->c <= kDsmemLog2Bits));
  if (use_smem) {
    switch (lph) {
      case 1: return launch_g0_smem<1>(p, hosts_dev, n, H, g0_dev);
      case 2: return launch_g0_smem<2>(p, hosts_dev, n, H, g0_dev);
      case 4: return launch_g0_smem<4>(p, hosts_dev, n, H, g0_dev);
      case 8: return launch_g0_smem<8>(p, hosts_dev, n, H, g0_dev);
      case 16: return launch_g0_smem<16>(p, hosts_dev, n, H, g0_dev);
      default: return launch_g0_smem<32>(p, hosts_dev, n, H, g0_dev);
    }
  }
  switch (lph) {
    case 1: VATE_LAUNCH(p, VATE_K_G0, grid, kThreads, 0, k_g0<1>, hosts_dev, n, bm, H, g0_dev); break;
    case 2: VATE_LAUNCH(p, VATE_K_G0, grid, kThreads, 0, k_g0<2>, hosts_dev, n, bm, H, g0_dev); break;
    case 4: VATE_LAUNCH(p, VATE_K_G0, grid, kThreads, 0, k_g0<4>, hosts_dev, n, bm, H, g0_dev); break;
    case 8: VATE_LAUNCH(p, VATE_K_G0, grid, kThreads, 0, k_g0<8>, hosts_dev, n, bm, H, g0_dev); break;
    case 16: VATE_LAUNCH(p, VATE_K_G0, grid, kThreads, 0, k_g0<16>, hosts_dev, n, bm, H, g0_dev); break;
    default: VATE_LAUNCH(p, VATE_K_G0, grid, kThreads, 0, k_g0<32>, hosts_dev, n, bm, H, g0_dev); break;
  }
  return VATE_OK;
}

int launch_g0_list(vate_pool* p, const uint64_t* hosts_dev, const uint32_t* idx_dev,
                   const unsigned long long* count_dev, uint64_t cap, HashParams H,
                   int32_t* g0_dev, uint64_t* yk, int32_t* yg) {
  int lph = 1;
  while (lph < 32 && (uint64_t)lph < H.g) lph <<= 1;
  // the count lives on the device: size the grid for a modest list, grid-stride beyond
  const uint32_t grid = grid_for(umin64(cap, 1u << 16) * (uint64_t)lph, kThreads, 148u * 16u);
  const uint32_t* bm = p->bitmap.as<const uint32_t>();
  switch (lph) {
    case 1: VATE_LAUNCH(p, VATE_K_G0, grid, kThreads, 0, (k_g0<1, true>), hosts_dev, cap, bm, H, g0_dev, idx_dev, count_dev, yk, yg); break;
    case 2: VATE_LAUNCH(p, VATE_K_G0, grid, kThreads, 0, (k_g0<2, true>), hosts_dev, cap, bm, H, g0_dev, idx_dev, count_dev, yk, yg); break;
    case 4: VATE_LAUNCH(p, VATE_K_G0, grid, kThreads, 0, (k_g0<4, true>), hosts_dev, cap, bm, H, g0_dev, idx_dev, count_dev, yk, yg); break;
    case 8: VATE_LAUNCH(p, VATE_K_G0, grid, kThreads, 0, (k_g0<8, true>), hosts_dev, cap, bm, H, g0_dev, idx_dev, count_dev, yk, yg); break;
    case 16: VATE_LAUNCH(p, VATE_K_G0, grid, kThreads, 0, (k_g0<16, true>), hosts_dev, cap, bm, H, g0_dev, idx_dev, count_dev, yk, yg); break;
    default: VATE_LAUNCH(p, VATE_K_G0, grid, kThreads, 0, (k_g0<32, true>), hosts_dev, cap, bm, H, g0_dev, idx_dev, count_dev, yk, yg); break;
  }
  return VATE_OK;
}

// The single float path (estimator.py:138-162), per host:
//   z_v = g0/g;  raw = g * (log_zp - log_zv[g0]);  est = max(raw, 0)
//   saturated = g0 == 0 | raw < 0 | P == 0
// log_zv / log_zp come from numpy on the host (see vate.h), and the
// subtraction and product are single IEEE roundings with no contraction, so
// the results are bit-identical to the reference's numpy expression.
struct FloatPath {
  const double* lzv;
  double lzp;
  double gd;
  int pool_empty;  // P == 0
  double floor;    // keep iff floor <= 0 or est >= floor (pipeline.py:136-137)
};

__device__ __forceinline__ void float_path(int32_t g0, const FloatPath& F, double* est, double* zv,
                                           uint8_t* sat, bool* keep) {
  const double raw = __dmul_rn(F.gd, __dsub_rn(F.lzp, F.lzv[g0]));
  *zv = __ddiv_rn((double)g0, F.gd);
  *sat = (g0 == 0) | (raw < 0.0) | F.pool_empty;
  *est = raw < 0.0 ? 0.0 : raw;
  *keep = !(F.floor > 0.0) || *est >= F.floor;
}

constexpr int kFinTile = 1024;  // hosts per CTA in the filter passes (256 threads x 4)

// Pass 1: per-tile kept counts (only when a floor is set).
__global__ void __launch_bounds__(256) k_final_count(const int32_t* __restrict__ g0, uint64_t n,
                                                     FloatPath F, unsigned* __restrict__ tile_cnt) {
  __shared__ unsigned s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kFinTile + threadIdx.x * 4;
  unsigned local = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (base + q < n) {
      double e, z;
      uint8_t st;
      bool keep;
      float_path(g0[base + q], F, &e, &z, &st, &keep);
      local += keep;
    }
  }
  local = __reduce_add_sync(0xffffffffu, local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(&s, local);
  __syncthreads();
  if (threadIdx.x == 0) tile_cnt[blockIdx.x] = s;
}

// Pass 2: exclusive scan of tile counts in one CTA; total -> *nsel.
__global__ void __launch_bounds__(1024) k_final_scan(unsigned* __restrict__ tile_cnt, uint64_t ntiles,
                                                     unsigned long long* nsel) {
  __shared__ unsigned long long warp_tot[32];
  __shared__ unsigned long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint64_t base = 0; base < ntiles; base += blockDim.x) {
    const uint64_t i = base + threadIdx.x;
    const unsigned long long v = i < ntiles ? tile_cnt[i] : 0;
    unsigned long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      unsigned long long w = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long u = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += u;
      }
      warp_tot[lane] = w;  // inclusive prefix over warps
    }
    __syncthreads();
    const unsigned long long before = (wid ? warp_tot[wid - 1] : 0) + carry;
    if (i < ntiles) tile_cnt[i] = (unsigned)(before + incl - v);
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = before + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *nsel = carry;
}

// Pass 3 (or the only pass without a floor): values for every host; kept
// rows are written in host order at their stable compacted position.
__global__ void __launch_bounds__(256) k_final_write(const uint64_t* __restrict__ hosts,
                                                     const int32_t* __restrict__ g0, uint64_t n,
                                                     FloatPath F, const unsigned* __restrict__ tile_off,
                                                     uint64_t* __restrict__ out_host,
                                                     double* __restrict__ out_est,
                                                     double* __restrict__ out_zv,
                                                     uint8_t* __restrict__ out_sat) {
  __shared__ unsigned warp_tot[8];
  const uint64_t base = (uint64_t)blockIdx.x * kFinTile + threadIdx.x * 4;
  double e[4], z[4];
  uint8_t st[4];
  bool keep[4];
  unsigned mine = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    keep[q] = false;
    if (base + q < n) {
      float_path(g0[base + q], F, &e[q], &z[q], &st[q], &keep[q]);
      mine += keep[q];
    }
  }
  uint64_t pos = base;
  if (tile_off) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    unsigned before = 0;
    for (int w = 0; w < wid; ++w) before += warp_tot[w];
    pos = (uint64_t)tile_off[blockIdx.x] + before + incl - mine;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (keep[q]) {
      out_host[pos] = hosts ? hosts[base + q] : 0;
      out_est[pos] = e[q];
      out_zv[pos] = z[q];
      out_sat[pos] = st[q];
      ++pos;
    }
  }
}

// Writes report set `slot`; the D2H that last read that set must be done first.
// No floor: every host is kept at its own position, so a plain grid-stride
// loop gives fully coalesced loads and stores.
__global__ void __launch_bounds__(256) k_final_all(const uint64_t* __restrict__ hosts,
                                                   const int32_t* __restrict__ g0, uint64_t n,
                                                   FloatPath F, uint64_t* __restrict__ out_host,
                                                   double* __restrict__ out_est,
                                                   double* __restrict__ out_zv,
                                                   uint8_t* __restrict__ out_sat) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    double e, z;
    uint8_t st;
    bool keep;
    float_path(__ldcs(g0 + i), F, &e, &z, &st, &keep);
    if (hosts) __stcs(out_host + i, __ldcs(hosts + i));
    __stcs(out_est + i, e);
    __stcs(out_zv + i, z);
    out_sat[i] = st;
  }
}

static int run_float_path(vate_pool* p, const uint64_t* hosts_dev, const int32_t* g0_dev,
                          uint64_t n, FloatPath F, int slot, uint64_t* nkept) {
  const uint64_t ntiles = (n + kFinTile - 1) / kFinTile;
  int rc;
  VATE_CUDA(cudaStreamWaitEvent(p->stream, p->ev_d2h[slot], 0));
  for (DevBuf* b : {&p->host_out[slot], &p->est_out[slot], &p->zv_out[slot]}) {
    rc = b->ensure(n * 8 + 8);
    if (rc) return rc;
  }
  rc = p->sat_out[slot].ensure(n + 8);
  if (rc) return rc;
  const unsigned* tile_off = nullptr;
  if (F.floor > 0.0) {
    rc = p->flags.ensure(ntiles * 4 + 16);
    if (rc) return rc;
    VATE_LAUNCH(p, VATE_K_FINAL, (uint32_t)ntiles, 256, 0, k_final_count, g0_dev, n, F,
                p->flags.as<unsigned>());
    VATE_LAUNCH(p, VATE_K_FINAL, 1, 1024, 0, k_final_scan, p->flags.as<unsigned>(), ntiles,
                p->d_ctr + C_NSEL);
    VATE_CUDA(cudaMemcpyAsync(p->h_ctr + C_NSEL, p->d_ctr + C_NSEL, 8, cudaMemcpyDeviceToHost,
                              p->stream));
    tile_off = p->flags.as<const unsigned>();
  }
  if (tile_off)
    VATE_LAUNCH(p, VATE_K_FINAL, (uint32_t)ntiles, 256, 0, k_final_write, hosts_dev, g0_dev, n, F,
                tile_off, p->host_out[slot].as<uint64_t>(), p->est_out[slot].as<double>(),
                p->zv_out[slot].as<double>(), p->sat_out[slot].as<uint8_t>());
  else
    VATE_LAUNCH(p, VATE_K_FINAL, grid_for(n, 256, p->cap_final), 256, 0, k_final_all, hosts_dev,
                g0_dev, n, F, p->host_out[slot].as<uint64_t>(), p->est_out[slot].as<double>(),
                p->zv_out[slot].as<double>(), p->sat_out[slot].as<uint8_t>());
  if (F.floor > 0.0) {
    rc = sync_small(p);
    if (rc) return rc;
    *nkept = p->h_ctr[C_NSEL];
  } else {
    *nkept = n;
  }
  return VATE_OK;
}

// Report rows of set `slot` -> host, on the D2H stream once the float path is
// done; overlaps the next slice's kernels.  ev_d2h[slot] marks completion.
static int copy_rows_out(vate_pool* p, int slot, uint64_t m, bool with_hosts, uint64_t* out_host,
                         double* out_est, double* out_zv, uint8_t* out_sat) {
  VATE_CUDA(cudaEventRecord(p->ev_fin[slot], p->stream));
  VATE_CUDA(cudaStreamWaitEvent(p->d2h_stream, p->ev_fin[slot], 0));
  if (m) {
    cudaStream_t s = p->d2h_stream;
    if (with_hosts && out_host)
      VATE_CUDA(cudaMemcpyAsync(out_host, p->host_out[slot].ptr, m * 8, cudaMemcpyDeviceToHost, s));
    if (out_est)
      VATE_CUDA(cudaMemcpyAsync(out_est, p->est_out[slot].ptr, m * 8, cudaMemcpyDeviceToHost, s));
    if (out_zv)
      VATE_CUDA(cudaMemcpyAsync(out_zv, p->zv_out[slot].ptr, m * 8, cudaMemcpyDeviceToHost, s));
    if (out_sat)
      VATE_CUDA(cudaMemcpyAsync(out_sat, p->sat_out[slot].ptr, m, cudaMemcpyDeviceToHost, s));
  }
  VATE_CUDA(cudaEventRecord(p->ev_d2h[slot], p->d2h_stream));
  return VATE_OK;
}

static int wait_rows(vate_pool* p, int slot) {
  VATE_CUDA(cudaEventSynchronize(p->ev_d2h[slot]));
  return VATE_OK;
}

static int float_params(vate_pool* p, uint64_t g, uint64_t pool_inactive, double log_zp,
                        double floor, FloatPath* F) {
  if (p->lzv_g != g || !p->lzv.ptr)
    return set_error(VATE_EVALUE, "log table not set for g=" + std::to_string(g));
  F->lzv = p->lzv.as<const double>();
  F->lzp = log_zp;
  F->gd = (double)g;
  F->pool_empty = pool_inactive == 0;
  F->floor = floor;
  return VATE_OK;
}

}  // namespace vate

using namespace vate;

extern "C" {

int vate_host_g0(vate_pool* p, uint64_t g, uint64_t cell_stream, const uint64_t* aips, uint64_t n,
                 int k_prime, int32_t* g0, int where) {
  int rc = enter(p);
  if (rc) return rc;
  rc = check_width(p, k_prime);
  if (rc || n == 0) return rc;
  if (g < 1 || g > p->L.size) return set_error(VATE_ECONFIG, "g must be in [1, 2^c]");
  rc = build_bitmap(p, k_prime);
  if (rc) return rc;
  const void* d_aips;
  rc = stage_in(p, p->in_a, aips, n * 8, where, &d_aips);
  if (rc) return rc;
  rc = p->g0.ensure(n * 4 + 4);
  if (rc) return rc;
  rc = launch_g0(p, (const uint64_t*)d_aips, n, make_hash(g, p->c, cell_stream, 0), p->g0.as<int32_t>());
  if (rc) return rc;
  VATE_CUDA(cudaMemcpyAsync(g0, p->g0.ptr, n * 4, cudaMemcpyDeviceToHost, p->stream));
  return sync_small(p);
}

int vate_set_log_table(vate_pool* p, uint64_t g, const double* log_zv) {
  int rc = enter(p);
  if (rc) return rc;
  rc = p->lzv.ensure((g + 1) * 8);
  if (rc) return rc;
  VATE_CUDA(cudaMemcpyAsync(p->lzv.ptr, log_zv, (g + 1) * 8, cudaMemcpyHostToDevice, p->stream));
  rc = sync_small(p);
  if (rc) return rc;
  p->lzv_g = g;
  return VATE_OK;
}

int vate_reports_from_counts(vate_pool* p, uint64_t g, const int32_t* g0, uint64_t n,
                             uint64_t pool_inactive, double log_zp, double* est, double* z_v,
                             uint8_t* saturated) {
  int rc = enter(p);
  if (rc || n == 0) return rc;
  for (uint64_t i = 0; i < n; ++i)
    if (g0[i] < 0 || (uint64_t)g0[i] > g)
      return set_error(VATE_EVALUE, "g0=" + std::to_string(g0[i]) + " outside [0, " + std::to_string(g) + "]");
  FloatPath F;
  rc = float_params(p, g, pool_inactive, log_zp, 0.0, &F);
  if (rc) return rc;
  const void* d_g0;
  rc = stage_in(p, p->in_a, g0, n * 4, VATE_HOST, &d_g0);
  if (rc) return rc;
  uint64_t kept = 0;
  const int slot = p->out_slot;
  p->out_slot ^= 1;
  rc = run_float_path(p, nullptr, (const int32_t*)d_g0, n, F, slot, &kept);
  if (rc) return rc;
  rc = copy_rows_out(p, slot, n, false, nullptr, est, z_v, saturated);
  if (rc) return rc;
  return wait_rows(p, slot);
}

// The estimate in two halves around its single host round trip.
// enqueue: the bitmap pass (P, and the flipped cells when the index is live)
// and the active-set compaction; their counters are copied to pinned memory.
// with_advance: slice t's advance follows its bitmap pass on the main stream --
// fused into the pass for the AT pool (no separate sweep launch), a separate
// kernel for the comparators; collected with vate_advance_result.
static int bitmap_and_advance(vate_pool* p, int k_prime, bool delta, bool with_advance) {
  const bool fuse = with_advance && p->kind == VATE_AT && p->opt_fuse_sweep;
  int rc = build_bitmap(p, k_prime, delta, fuse);
  if (rc || !with_advance || fuse) return rc;
  return vate_advance_async(p);
}

static int begin_enqueue(vate_pool* p, vate_hosts* hosts, uint64_t g, uint64_t cell_stream,
                         int64_t t, int k_prime, bool whole_set = true,
                         bool with_advance = false) {
  if (!hosts || hosts->pool != p) return set_error(VATE_EVALUE, "registry does not belong to pool");
  int rc = check_width(p, k_prime);
  if (rc) return rc;
  if (g < 1 || g > p->L.size) return set_error(VATE_ECONFIG, "g must be in [1, 2^c]");
  p->est_n = 0;
  if (!p->opt_concurrent) {
    rc = bitmap_and_advance(p, k_prime, inc_delta_ready(p, g, cell_stream, k_prime), with_advance);
    if (rc) return rc;
    return hosts_active_launch(hosts, t, k_prime);  // pipeline.py:121
  }
  // fork: the registry compaction (reads the registry) runs on the aux stream
  // beside the bitmap pass (reads the cells); joined before the round trip
  VATE_CUDA(cudaEventRecord(p->ev_fork, p->stream));
  VATE_CUDA(cudaStreamWaitEvent(p->aux_stream, p->ev_fork, 0));
  std::swap(p->stream, p->aux_stream);
  rc = hosts_active_launch(hosts, t, k_prime);  // pipeline.py:121
  std::swap(p->stream, p->aux_stream);
  if (rc) return rc;
  VATE_CUDA(cudaEventRecord(p->ev_join, p->aux_stream));
  const bool delta = inc_delta_ready(p, g, cell_stream, k_prime);
  rc = build_bitmap(p, k_prime, delta,
                    with_advance && p->kind == VATE_AT && p->opt_fuse_sweep);
  if (rc) return rc;
  if (whole_set) {  // the delta apply overlaps the round trip (behind active on aux)
    rc = inc_apply_early(p, hosts_nactive_dev(hosts), g);
    if (rc) return rc;
  }
  if (with_advance && !(p->kind == VATE_AT && p->opt_fuse_sweep)) {
    rc = vate_advance_async(p);  // comparators: the separate advance kernel
    if (rc) return rc;
  }
  VATE_CUDA(cudaStreamWaitEvent(p->stream, p->ev_join, 0));
  return VATE_OK;
}

// complete (after the caller's sync): the sorted active set, P, and g0 of
// every active host (incremental or full); the g0 kernels are left running.
static int begin_complete(vate_pool* p, vate_hosts* hosts, uint64_t g, uint64_t cell_stream,
                          int64_t t, int k_prime, uint64_t* nhosts, uint64_t* pool_inactive,
                          int part = 0, int nparts = 1) {
  IncIndex& I = p->inc;
  if (I.lookup_pending) {  // misses of the previous lookup (landed before this sync)
    I.lookup_pending = false;
    I.last_misses = p->h_ctr[C_MISS];
    I.miss_accum += I.last_misses;
    I.extend_accum += I.last_misses;
    // Policy (ski rental on measured costs, profiles/): the captured misses of
    // the last lookup join X by a streaming CSR merge (~8 B per index entry)
    // once the misses gathered since the last merge reach 1/4 of |X|
    // (a miss costs g sector gathers, 32 B each); X is rebuilt from scratch only
    // when most of the active set is new or X has gone stale (> 2x active).
    if (I.valid && I.last_n && I.last_misses * 2 > I.last_n) I.want_rebuild = true;
    else if (I.valid && I.last_misses && I.extend_accum * 4 >= I.m) I.want_extend = true;
    if (I.valid && I.last_misses == 0 && I.m == I.last_n) {  // that active list == X
      I.identity_ok = true;
      I.identity_version = I.lookup_version;
    }
  }
  if (I.early_apply) {
    // the guard of the early delta apply read the registry's first active count
    // (now in the pinned counters); a relaunch below may reset it on the device,
    // so this stream waits for the apply first
    I.early_nhosts = hosts_nactive_host(hosts);
    VATE_CUDA(cudaStreamWaitEvent(p->stream, I.ev_apply, 0));
  }
  uint64_t* keys = nullptr;
  uint64_t n = 0;
  int rc = hosts_active_finish(hosts, t, k_prime, &keys, &n);
  if (rc) return rc;
  if (nparts > 1) {  // this rank's contiguous share of the sorted active set
    const uint64_t lo = n * (uint64_t)part / nparts, hi = n * (uint64_t)(part + 1) / nparts;
    keys += lo;
    n = hi - lo;
  }
  *nhosts = n;
  *pool_inactive = 0;
  if (n == 0) {  // no hosts: no report (pipeline.py:122-123); the index stays as it was
    I.delta_launched = false;
    return VATE_OK;
  }
  *pool_inactive = p->h_ctr[C_P];
  rc = inc_compute_g0(p, keys, n, make_hash(g, p->c, cell_stream, 0), k_prime);
  if (rc) return rc;
  p->est_n = n;
  p->est_keys = keys;
  p->est_kp = k_prime;
  p->est_g = g;
  return VATE_OK;
}

int vate_estimate_begin(vate_pool* p, vate_hosts* hosts, uint64_t g, uint64_t cell_stream,
                        int64_t t, int k_prime, uint64_t* nhosts, uint64_t* pool_inactive) {
  int rc = enter(p);
  if (rc) return rc;
  rc = begin_enqueue(p, hosts, g, cell_stream, t, k_prime);
  if (rc) return rc;
  rc = sync_small(p);
  if (rc) return rc;
  return begin_complete(p, hosts, g, cell_stream, t, k_prime, nhosts, pool_inactive);
}

int vate_estimate_begin_part(vate_pool* p, vate_hosts* hosts, uint64_t g, uint64_t cell_stream,
                             int64_t t, int k_prime, int part, int nparts, uint64_t* nhosts,
                             uint64_t* pool_inactive) {
  int rc = enter(p);
  if (rc) return rc;
  if (nparts < 1 || part < 0 || part >= nparts) return set_error(VATE_EVALUE, "bad part");
  rc = begin_enqueue(p, hosts, g, cell_stream, t, k_prime, nparts == 1);
  if (rc) return rc;
  rc = sync_small(p);
  if (rc) return rc;
  return begin_complete(p, hosts, g, cell_stream, t, k_prime, nhosts, pool_inactive, part, nparts);
}

int vate_estimate_begin_hosts(vate_pool* p, const uint64_t* hosts, uint64_t n, int where,
                              uint64_t g, uint64_t cell_stream, int k_prime,
                              uint64_t* pool_inactive) {
  int rc = enter(p);
  if (rc) return rc;
  rc = check_width(p, k_prime);
  if (rc) return rc;
  if (g < 1 || g > p->L.size) return set_error(VATE_ECONFIG, "g must be in [1, 2^c]");
  p->est_n = 0;
  *pool_inactive = 0;
  p->sorted_owner = nullptr;  // hosts_sorted no longer holds a registry's active set
  p->sorted_version++;
  p->g0_src = nullptr;
  rc = p->hosts_sorted.ensure(n * 8 + 8);
  if (rc) return rc;
  if (n) {
    if (where == VATE_DEVICE)
      VATE_CUDA(cudaMemcpyAsync(p->hosts_sorted.ptr, hosts, n * 8, cudaMemcpyDeviceToDevice, p->stream));
    else
      VATE_CUDA(cudaMemcpyAsync(p->hosts_sorted.ptr, hosts, n * 8, cudaMemcpyHostToDevice, p->stream));
  }
  rc = build_bitmap(p, k_prime);
  if (rc) return rc;
  VATE_CUDA(cudaEventRecord(p->ev_small, p->stream));
  if (n) {
    rc = p->g0.ensure(n * 4 + 4);
    if (rc) return rc;
    rc = launch_g0(p, p->hosts_sorted.as<uint64_t>(), n, make_hash(g, p->c, cell_stream, 0),
                   p->g0.as<int32_t>());
    if (rc) return rc;
  }
  VATE_CUDA(cudaEventSynchronize(p->ev_small));
  *pool_inactive = p->h_ctr[C_P];
  p->est_n = n;
  p->est_keys = p->hosts_sorted.as<const uint64_t>();
  p->est_kp = k_prime;
  p->est_g = g;
  return VATE_OK;
}

static int estimate_finish_impl(vate_pool* p, uint64_t g, uint64_t pool_inactive, double log_zp,
                                double floor, uint64_t* out_host, double* out_est,
                                double* out_zv, uint8_t* out_sat, uint64_t cap, uint64_t* nkept,
                                bool wait) {
  int rc = enter(p);
  if (rc) return rc;
  if (g != p->est_g) return set_error(VATE_EVALUE, "estimate_finish: g differs from begin");
  const uint64_t n = p->est_n;
  *nkept = 0;
  if (n == 0) return VATE_OK;
  FloatPath F;
  rc = float_params(p, g, pool_inactive, log_zp, floor, &F);
  if (rc) return rc;
  uint64_t kept = 0;
  const int slot = p->out_slot;
  p->out_slot ^= 1;
  rc = run_float_path(p, p->est_keys,
                      p->g0_src ? p->g0_src : p->g0.as<const int32_t>(), n, F, slot, &kept);
  if (rc) return rc;
  *nkept = kept;
  p->est_n = 0;
  rc = copy_rows_out(p, slot, kept < cap ? kept : cap, true, out_host, out_est, out_zv, out_sat);
  if (rc || !wait) return rc;
  return wait_rows(p, slot);
}

int vate_estimate_finish(vate_pool* p, uint64_t g, uint64_t pool_inactive, double log_zp,
                         double floor, uint64_t* out_host, double* out_est, double* out_zv,
                         uint8_t* out_sat, uint64_t cap, uint64_t* nkept) {
  return estimate_finish_impl(p, g, pool_inactive, log_zp, floor, out_host, out_est, out_zv,
                              out_sat, cap, nkept, true);
}

int vate_estimate_finish_async(vate_pool* p, uint64_t g, uint64_t pool_inactive, double log_zp,
                               double floor, uint64_t* out_host, double* out_est,
                               double* out_zv, uint8_t* out_sat, uint64_t cap, uint64_t* nkept) {
  return estimate_finish_impl(p, g, pool_inactive, log_zp, floor, out_host, out_est, out_zv,
                              out_sat, cap, nkept, false);
}

int vate_slice_step(vate_pool* p, vate_hosts* hosts, uint64_t g, uint64_t cell_stream,
                    uint64_t group_stream, const uint32_t* pairs, uint64_t n, int where,
                    int64_t t, int k_prime, double floor, const double* log_zp_table,
                    uint64_t* out_host, double* out_est, double* out_zv, uint8_t* out_sat,
                    uint64_t cap, vate_step_result* res) {
  int rc = enter(p);
  if (rc) return rc;
  if (!res || !log_zp_table) return set_error(VATE_EVALUE, "null result or log table");
  memset(res, 0, sizeof(*res));
  // scan (pipeline.py:144-147)
  if (where == VATE_STAGED) {
    rc = vate_scan_staged(p, g, cell_stream, group_stream, (int)(uintptr_t)pairs, n, hosts, t);
  } else if (n) {
    rc = vate_scan_packed(p, g, cell_stream, group_stream, pairs, n, where, hosts, t);
  }
  if (rc) return rc;
  rc = lat_scan_end(p, t);
  if (rc) return rc;
  if (p->adv_pending) {  // the previous slice's advance (its bitmap pass) is long done
    res->prev_collected = 1;
    rc = vate_advance_result(p, res->prev_blocks, &res->prev_maintained, &res->prev_cleared);
    if (rc) return rc;
  }
  // estimate, first half, with this slice's advance fused into the bitmap pass
  // (it touches cells, which nothing after the pass reads); then the slice's
  // one host round trip
  rc = begin_enqueue(p, hosts, g, cell_stream, t, k_prime, true, true);
  if (rc) return rc;
  rc = sync_small(p);
  if (rc) return rc;
  uint64_t nh = 0, pin = 0;
  rc = begin_complete(p, hosts, g, cell_stream, t, k_prime, &nh, &pin);
  if (rc) return rc;
  res->nhosts = nh;
  res->pool_inactive = pin;
  uint64_t kept = 0;
  if (nh) {
    rc = vate_estimate_finish_async(p, g, pin, log_zp_table[pin], floor, out_host, out_est,
                                    out_zv, out_sat, cap, &kept);
    res->nkept = kept;
    if (rc == VATE_OK) rc = lat_rows(p, t);
  }
  return rc;
}

// ---- lagged (software-pipelined) slice step ----------------------------------
// The step for slice t enqueues slice t's scan first, then completes the
// PREVIOUS slice (its round trip has long landed; its g0 lookups, float path
// and report copies run on the aux stream beside this scan), then enqueues
// slice t's bitmap pass, registry compaction, early delta apply and sweep.  The
// GPU goes from one slice's sweep straight into the next slice's scan; the
// results of slice t arrive with the call for slice t+1 (or the flush).
// Two halves around the previous slice's P (the float path needs np.log of the
// pool fraction, taken on the host when no table is given): begin (scan t,
// previous slice up to g0) and end (previous slice's float path, prune; slice
// t up to its sweep).  Falls back to completing the previous slice before the
// scan when the registry's parked-insert list could fill (a drain must not
// rehash the table under a running scan).
static int lagged_begin_prev(vate_pool* p, vate_hosts* hosts, uint64_t g, uint64_t cell_stream,
                             vate_step_result* res) {
  if (!p->lag_pending) return VATE_OK;
  p->lag_pending = false;
  p->lag_completing = true;
  const int64_t t = p->lag_t;
  const int kp = p->lag_kp;
  res->prev_t = t;
  res->prev_valid = 1;
  VATE_CUDA(cudaEventSynchronize(p->ev_counts));  // its bitmap + compaction counters landed
  if (p->adv_pending) {  // its sweep (right behind its bitmap pass)
    res->prev_collected = 1;
    int rc = vate_advance_result(p, res->prev_blocks, &res->prev_maintained, &res->prev_cleared);
    if (rc) return rc;
  }
  // post-round-trip work of slice t on the aux stream, beside the next scan
  std::swap(p->stream, p->aux_stream);
  hosts->lagged = true;
  uint64_t nh = 0, pin = 0;
  int rc = begin_complete(p, hosts, g, cell_stream, t, kp, &nh, &pin, p->lag_part, p->lag_nparts);
  hosts->lagged = false;
  std::swap(p->stream, p->aux_stream);
  res->nhosts = nh;
  res->pool_inactive = pin;
  return rc;
}

static int lagged_end_prev(vate_pool* p, vate_hosts* hosts, uint64_t g, double floor,
                           double log_zp, uint64_t* out_host, double* out_est, double* out_zv,
                           uint8_t* out_sat, uint64_t cap, vate_step_result* res) {
  if (!p->lag_completing) return VATE_OK;
  p->lag_completing = false;
  const int64_t t = p->lag_t;
  std::swap(p->stream, p->aux_stream);
  int rc = VATE_OK;
  if (res->nhosts) {
    uint64_t kept = 0;
    rc = vate_estimate_finish_async(p, g, res->pool_inactive, log_zp, floor, out_host, out_est,
                                    out_zv, out_sat, cap, &kept);
    res->nkept = kept;
    if (rc == VATE_OK) rc = lat_rows(p, t);
  }
  // everything above (g0 delta / lookups read the delta list and bitmap buffers
  // the next bitmap pass rewrites) must finish before slice t+1's bitmap pass
  if (rc == VATE_OK) {
    const cudaError_t e = cudaEventRecord(p->ev_post, p->stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaEventRecord (post)");
    else p->post_recorded = true;
  }
  std::swap(p->stream, p->aux_stream);
  // SlidingHostSet.prune (pipeline.py:59-64, at t % k == 0) after slice t's
  // reports: the next slice's scan may have stamped hosts already, which the
  // prune keeps (last > t - k), exactly as if it had run first.  The post work
  // above reads registry slots the prune's rebuild moves: wait for it first.
  if (rc == VATE_OK && t % (int64_t)(hosts->k > 0 ? hosts->k : 1) == 0) {
    const cudaError_t e = cudaStreamSynchronize(p->aux_stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize (prune)");
    rc = vate_hosts_prune(hosts, t);
  }
  return rc;
}

int vate_slice_lagged_begin(vate_pool* p, vate_hosts* hosts, uint64_t g, uint64_t cell_stream,
                            uint64_t group_stream, const uint32_t* pairs, uint64_t n, int where,
                            int64_t t, int k_prime, vate_step_result* res) {
  int rc = enter(p);
  if (rc) return rc;
  if (!res || !hosts) return set_error(VATE_EVALUE, "null argument");
  if (p->lag_completing) return set_error(VATE_EVALUE, "lagged step: end of the previous call missing");
  memset(res, 0, sizeof(*res));
  rc = check_width(p, k_prime);
  if (rc) return rc;
  if (!p->ev_counts) VATE_CUDA(cudaEventCreateWithFlags(&p->ev_counts, cudaEventDisableTiming));
  if (!p->ev_post) VATE_CUDA(cudaEventCreateWithFlags(&p->ev_post, cudaEventDisableTiming));
  if (p->lag_peer && n > peer_key_cap(p->lag_peer))  // before the scan: replicas stay equal
    return set_error(VATE_EVALUE, std::to_string(n) + " packets exceed the peer key_cap " +
                                      std::to_string(peer_key_cap(p->lag_peer)));
  p->lag_next_t = t;
  p->lag_next_kp = k_prime;
  p->lag_has_next = true;
  // a scan that might have to drain the registry waits for the previous slice
  p->lag_deferred_scan = hosts->pending + n > hosts->ovf_cap;
  if (p->lag_deferred_scan) {
    p->lag_scan_pairs = pairs;
    p->lag_scan_n = n;
    p->lag_scan_where = where;
    return lagged_begin_prev(p, hosts, g, cell_stream, res);  // scan after the end
  }
  if (where == VATE_STAGED) {
    rc = vate_scan_staged(p, g, cell_stream, group_stream, (int)(uintptr_t)pairs, n, hosts, t);
  } else if (n) {
    rc = vate_scan_packed(p, g, cell_stream, group_stream, pairs, n, where, hosts, t);
  }
  if (rc) return rc;
  rc = lat_scan_end(p, t);
  if (rc) return rc;
  return lagged_begin_prev(p, hosts, g, cell_stream, res);
}

int vate_slice_lagged_end(vate_pool* p, vate_hosts* hosts, uint64_t g, uint64_t cell_stream,
                          uint64_t group_stream, double floor, double log_zp, uint64_t* out_host,
                          double* out_est, double* out_zv, uint8_t* out_sat, uint64_t cap,
                          vate_step_result* res) {
  int rc = enter(p);
  if (rc) return rc;
  if (!res || !hosts) return set_error(VATE_EVALUE, "null argument");
  rc = lagged_end_prev(p, hosts, g, floor, log_zp, out_host, out_est, out_zv, out_sat, cap, res);
  if (rc) return rc;
  if (!p->lag_has_next) {  // a flush: nothing follows
    VATE_CUDA(cudaStreamSynchronize(p->aux_stream));
    return VATE_OK;
  }
  p->lag_has_next = false;
  const int64_t t = p->lag_next_t;
  const int k_prime = p->lag_next_kp;
  if (p->lag_deferred_scan) {  // the previous slice is complete: drain, grow, scan
    p->lag_deferred_scan = false;
    VATE_CUDA(cudaStreamSynchronize(p->aux_stream));
    rc = hosts_drain(hosts);
    if (rc) return rc;
    rc = hosts->ovf.ensure(2 * (p->lag_scan_n + 1) * sizeof(RegEntry));  // two slices' parks
    if (rc) return rc;
    hosts->ovf_cap = hosts->ovf.bytes / sizeof(RegEntry);
    if (p->lag_scan_where == VATE_STAGED) {
      rc = vate_scan_staged(p, g, cell_stream, group_stream, (int)(uintptr_t)p->lag_scan_pairs,
                            p->lag_scan_n, hosts, t);
    } else if (p->lag_scan_n) {
      rc = vate_scan_packed(p, g, cell_stream, group_stream, p->lag_scan_pairs, p->lag_scan_n,
                            p->lag_scan_where, hosts, t);
    }
    if (rc) return rc;
    rc = lat_scan_end(p, t);
    if (rc) return rc;
  }
  // multi-GPU: merge the replicas and absorb the peers' hosts of slice t
  if (p->lag_peer) {
    rc = vate_peer_exchange(p->lag_peer, t, nullptr);
    if (rc) return rc;
  }
  // slice t up to its counters; then its sweep (it reads no g0, only cells already counted)
  if (p->post_recorded) {
    VATE_CUDA(cudaStreamWaitEvent(p->stream, p->ev_post, 0));
    p->post_recorded = false;
  }
  rc = begin_enqueue(p, hosts, g, cell_stream, t, k_prime, p->lag_nparts == 1, true);  // + advance(t)
  if (rc) return rc;
  VATE_CUDA(cudaEventRecord(p->ev_counts, p->stream));
  p->lag_pending = true;
  p->lag_t = t;
  p->lag_kp = k_prime;
  return VATE_OK;
}

int vate_slice_lagged_flush_begin(vate_pool* p, vate_hosts* hosts, uint64_t g,
                                  uint64_t cell_stream, vate_step_result* res) {
  int rc = enter(p);
  if (rc) return rc;
  if (!res || !hosts) return set_error(VATE_EVALUE, "null argument");
  memset(res, 0, sizeof(*res));
  p->lag_has_next = false;
  p->lag_deferred_scan = false;
  return lagged_begin_prev(p, hosts, g, cell_stream, res);
}

int vate_slice_step_lagged(vate_pool* p, vate_hosts* hosts, uint64_t g, uint64_t cell_stream,
                           uint64_t group_stream, const uint32_t* pairs, uint64_t n, int where,
                           int64_t t, int k_prime, double floor, const double* log_zp_table,
                           uint64_t* out_host, double* out_est, double* out_zv,
                           uint8_t* out_sat, uint64_t cap, vate_step_result* res) {
  if (!log_zp_table) return set_error(VATE_EVALUE, "null log table");
  int rc = vate_slice_lagged_begin(p, hosts, g, cell_stream, group_stream, pairs, n, where, t,
                                   k_prime, res);
  if (rc) return rc;
  return vate_slice_lagged_end(p, hosts, g, cell_stream, group_stream, floor,
                               log_zp_table[res->pool_inactive], out_host, out_est, out_zv,
                               out_sat, cap, res);
}

int vate_slice_flush(vate_pool* p, vate_hosts* hosts, uint64_t g, uint64_t cell_stream,
                     double floor, const double* log_zp_table, uint64_t* out_host,
                     double* out_est, double* out_zv, uint8_t* out_sat, uint64_t cap,
                     vate_step_result* res) {
  if (!log_zp_table) return set_error(VATE_EVALUE, "null log table");
  int rc = vate_slice_lagged_flush_begin(p, hosts, g, cell_stream, res);
  if (rc) return rc;
  return vate_slice_lagged_end(p, hosts, g, cell_stream, 0, floor,
                               log_zp_table[res->pool_inactive], out_host, out_est, out_zv,
                               out_sat, cap, res);
}

int vate_pool_set_peer(vate_pool* p, vate_peer* x, int part, int nparts) {
  int rc = enter(p);
  if (rc) return rc;
  if (p->lag_pending || p->lag_completing)
    return set_error(VATE_EVALUE, "set the peer between lagged runs (flush first)");
  if (nparts < 1 || part < 0 || part >= nparts) return set_error(VATE_EVALUE, "bad part");
  p->lag_peer = x;
  p->lag_part = x ? part : 0;
  p->lag_nparts = x ? nparts : 1;
  return VATE_OK;
}

int vate_reports_device(vate_pool* p, uint64_t** host, double** est, double** zv,
                        uint8_t** sat) {
  if (!p) return set_error(VATE_EVALUE, "null pool handle");
  const int slot = p->out_slot ^ 1;  // the set the last finish wrote
  if (host) *host = p->host_out[slot].as<uint64_t>();
  if (est) *est = p->est_out[slot].as<double>();
  if (zv) *zv = p->zv_out[slot].as<double>();
  if (sat) *sat = p->sat_out[slot].as<uint8_t>();
  return VATE_OK;
}

int vate_reports_copy(vate_pool* p, uint64_t first, uint64_t n, uint64_t* host, double* est,
                      double* zv, uint8_t* sat) {
  int rc = enter(p);
  if (rc) return rc;
  const int slot = p->out_slot ^ 1;  // the set the last finish wrote
  const uint64_t avail = p->host_out[slot].bytes / 8;
  if (first + n > avail)
    return set_error(VATE_EVALUE, "report rows [" + std::to_string(first) + ", " +
                                      std::to_string(first + n) + ") beyond the last slice's " +
                                      std::to_string(avail) + "-row buffer");
  VATE_CUDA(cudaEventSynchronize(p->ev_fin[slot]));
  if (n == 0) return VATE_OK;
  if (host) VATE_CUDA(cudaMemcpy(host, p->host_out[slot].as<uint64_t>() + first, n * 8, cudaMemcpyDeviceToHost));
  if (est) VATE_CUDA(cudaMemcpy(est, p->est_out[slot].as<double>() + first, n * 8, cudaMemcpyDeviceToHost));
  if (zv) VATE_CUDA(cudaMemcpy(zv, p->zv_out[slot].as<double>() + first, n * 8, cudaMemcpyDeviceToHost));
  if (sat) VATE_CUDA(cudaMemcpy(sat, p->sat_out[slot].as<uint8_t>() + first, n, cudaMemcpyDeviceToHost));
  return VATE_OK;
}

int vate_estimate_wait(vate_pool* p) {
  int rc = enter(p);
  if (rc) return rc;
  VATE_CUDA(cudaStreamSynchronize(p->d2h_stream));
  return VATE_OK;
}

}  // extern "C"
