// vate_probe.cu -- ceilings for the rooflines bench.py reports (no reference
// counterpart: measurement infrastructure).
//
// vate_bench_l2: the L2 ceilings of the access patterns the L2-resident
// kernels are made of, over an L2-resident buffer: random 32-byte sector
// reads, random 2-byte stores (one sector each), random 32-bit red.or, and a
// streaming 16-byte read.  Addresses come from a 32-bit multiply-xorshift of
// the thread's counter (a few ALU ops, no index stream), so the probes measure
// the memory system, not an input array.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "vate_internal.cuh"

namespace vate {

__device__ __forceinline__ uint32_t rnd32(uint32_t x) {
  x *= 0x9E3779B1u;
  x ^= x >> 15;
  x *= 0x85EBCA77u;
  return x ^ (x >> 13);
}

// Four independent accesses per thread per step (memory-level parallelism as
// the scan has it: two packets, each a registry read and a cell write).
__global__ void __launch_bounds__(256) k_l2_gather(const uint4* __restrict__ buf, uint32_t nsec_mask,
                                                   uint64_t n, uint32_t seed, unsigned* out) {
  unsigned acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 4; i < n; i += 4 * stride) {
    uint32_t v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      v[u] = i + u < n ? __ldcg(buf + 2 * (uint64_t)(rnd32((uint32_t)(i + u) ^ seed) & nsec_mask)).x : 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u];
  }
  if (acc == 0x9E3779B9u) *out = acc;
}

__global__ void __launch_bounds__(256) k_l2_store(uint16_t* __restrict__ buf, uint32_t cell_mask,
                                                  uint64_t n, uint32_t seed) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 4; i < n; i += 4 * stride) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u < n) buf[rnd32((uint32_t)(i + u) ^ seed) & cell_mask] = (uint16_t)i;
  }
}

__global__ void __launch_bounds__(256) k_l2_red(uint32_t* __restrict__ buf, uint32_t bit_mask,
                                                uint64_t n, uint32_t seed) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 4; i < n; i += 4 * stride) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (i + u >= n) break;
      const uint32_t b = rnd32((uint32_t)(i + u) ^ seed) & bit_mask;
      asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(buf + (b >> 5)),
                   "r"(1u << (b & 31))
                   : "memory");
    }
  }
}

__global__ void __launch_bounds__(256) k_l2_stream(const uint4* __restrict__ buf, uint64_t n16,
                                                   unsigned* out) {
  unsigned acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
    const uint4 q = __ldcg(buf + i);
    acc ^= q.x ^ q.y ^ q.z ^ q.w;
  }
  if (acc == 0x9E3779B9u) *out = acc;
}

// The scan's memory skeleton: per 16-byte input (two packets, streamed
// evict-first) two red.or into a mark bitmap of 2^mark_log2 bits and two 32-B
// home-sector reads of a table of 2^tab_log2 sectors, in the scan's order and
// grid, with no hashing or compare chain -- what k_scan_packed16 would cost if
// only its memory operations counted.
//
// Ablation flags (scripts/scan_ablation.py): bit 0 the scan's 64-bit hashing
// (three splitmix64 per packet instead of one 32-bit mix), bit 1 a stamp store
// into the read sector for one packet in four, bit 2 a dependent second sector
// read for one packet in nine (a registry key outside its home sector), bit 3
// 256-bit sector loads as the registry lookup issues them, bit 4 (with bit 1)
// the stamp as a red.max instead of a store, bit 5 (with bit 1) the stamp as a
// red.or into a touched-slot bitmap.
template <int F>
__global__ void __launch_bounds__(256, 8) k_l2_scan_skeleton(
    const uint4* __restrict__ in, uint64_t n2, uint32_t* __restrict__ marks, uint32_t bit_mask,
    uint4* __restrict__ tab, uint32_t sec_mask, unsigned* out) {
  unsigned acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
    const uint4 q = __ldcs(in + i);
    uint32_t h0, h1, r0, r1;
    if (F & 1) {
      const uint64_t a0 = q.x + i, a1 = q.z + 3 * i;
      const uint64_t s0 = mix64(q.y * kPhi + 77), s1 = mix64(q.w * kPhi + 77 + i);
      h0 = (uint32_t)mix64(((a0 << 32) | (s0 & 1023)) * kPhi + 99);
      h1 = (uint32_t)mix64(((a1 << 32) | (s1 & 1023)) * kPhi + 99);
      r0 = (uint32_t)mix64(a0 ^ 0x2545F4914F6CDD1Dull);
      r1 = (uint32_t)mix64(a1 ^ 0x2545F4914F6CDD1Dull);
    } else {
      h0 = rnd32(q.x ^ (uint32_t)i);
      h1 = rnd32(q.z ^ (uint32_t)i ^ 0x9E37u);
      r0 = rnd32(h0);
      r1 = rnd32(h1);
    }
    const uint32_t b0 = h0 & bit_mask, b1 = h1 & bit_mask;
    asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(marks + (b0 >> 5)),
                 "r"(1u << (b0 & 31)) : "memory");
    asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(marks + (b1 >> 5)),
                 "r"(1u << (b1 & 31)) : "memory");
    uint4* p0 = tab + 2 * (uint64_t)(r0 & sec_mask);
    uint4* p1 = tab + 2 * (uint64_t)(r1 & sec_mask);
    uint32_t v0, v1;
    if (F & 8) {
      unsigned long long k0, l0, k1, l1, m0, n0, m1, n1;
      asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(k0), "=l"(l0), "=l"(k1), "=l"(l1) : "l"(p0));
      asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(m0), "=l"(n0), "=l"(m1), "=l"(n1) : "l"(p1));
      v0 = (uint32_t)(k0 ^ l0 ^ k1 ^ l1);
      v1 = (uint32_t)(m0 ^ n0 ^ m1 ^ n1);
    } else {
      v0 = __ldcg(p0).x;
      v1 = __ldcg(p1).x;
    }
    if ((F & 2) && !(F & 48)) {
      if ((r0 >> 28) < 4 && v0 != (uint32_t)i) reinterpret_cast<uint32_t*>(p0)[2] = (uint32_t)i;
      if ((r1 >> 28) < 4 && v1 != (uint32_t)i) reinterpret_cast<uint32_t*>(p1)[2] = (uint32_t)i;
    }
    if ((F & 2) && (F & 32)) {  // the stamp as one bit per slot in a touched bitmap
      // (the table has sec_mask + 1 sectors of two slots: 2 * (sec_mask + 1) bits
      // live in the mark buffer's first words)
      if ((r0 >> 28) < 4) {
        const uint32_t b = (r0 & sec_mask) * 2;
        asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(marks + (b >> 5)),
                     "r"(1u << (b & 31)) : "memory");
      }
      if ((r1 >> 28) < 4) {
        const uint32_t b = (r1 & sec_mask) * 2;
        asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(marks + (b >> 5)),
                     "r"(1u << (b & 31)) : "memory");
      }
    } else if ((F & 2) && (F & 16)) {  // the stamp as a fire-and-forget red.max
      if ((r0 >> 28) < 4 && v0 != (uint32_t)i)
        asm volatile("red.relaxed.gpu.global.max.s64 [%0], %1;" ::"l"(reinterpret_cast<long long*>(p0) + 1),
                     "l"((long long)i) : "memory");
      if ((r1 >> 28) < 4 && v1 != (uint32_t)i)
        asm volatile("red.relaxed.gpu.global.max.s64 [%0], %1;" ::"l"(reinterpret_cast<long long*>(p1) + 1),
                     "l"((long long)i) : "memory");
    }
    if (F & 4) {
      if ((r0 >> 24) % 9 == 0) v0 += __ldcg(tab + 2 * (uint64_t)((v0 + r0 + 1) & sec_mask)).x;
      if ((r1 >> 24) % 9 == 0) v1 += __ldcg(tab + 2 * (uint64_t)((v1 + r1 + 1) & sec_mask)).x;
    }
    acc += v0 + v1;
  }
  if (acc == 0x9E3779B9u) *out = acc;
}

template <int F>
static void launch_skeleton(vate_pool* p, uint32_t grid, const uint4* in, uint64_t n2,
                            uint32_t* marks, uint32_t bit_mask, uint4* tab, uint32_t sec_mask) {
  k_l2_scan_skeleton<F><<<grid, 256, 0, p->stream>>>(in, n2, marks, bit_mask, tab, sec_mask,
                                                      (unsigned*)p->d_ctr + 2 * C_TRACE);
}

}  // namespace vate

using namespace vate;

extern "C" int vate_bench_scan_ablation(vate_pool* p, int mark_log2, uint64_t table_bytes,
                                        uint64_t n, int reps, int flags, double* ms_out);

// ms per launch of k_l2_scan_skeleton over n packets (n even) with a mark
// bitmap of 2^mark_log2 bits and a table of table_bytes (power of two), on the
// scan's grid (vate_pool.cu: scan_packed dispatch).
extern "C" int vate_bench_scan_skeleton(vate_pool* p, int mark_log2, uint64_t table_bytes,
                                        uint64_t n, int reps, double* ms_out) {
  return vate_bench_scan_ablation(p, mark_log2, table_bytes, n, reps, 0, ms_out);
}

// The skeleton with the ablation flags above (measurement only).
extern "C" int vate_bench_scan_ablation(vate_pool* p, int mark_log2, uint64_t table_bytes,
                                        uint64_t n, int reps, int flags, double* ms_out) {
  int rc = enter(p);
  if (rc) return rc;
  if (flags < 0 || flags > 47) return set_error(VATE_EVALUE, "flags must be in [0, 47]");
  if (mark_log2 < 10 || mark_log2 > 32 || table_bytes < 4096 ||
      (table_bytes & (table_bytes - 1)) || table_bytes > (1ull << 36) || n < 2 || reps < 1)
    return set_error(VATE_EVALUE, "bad skeleton shape");
  DevBuf in, marks, tab;
  const uint64_t n2 = n / 2;
  if ((rc = in.ensure(n2 * 16)) || (rc = marks.ensure((1ull << mark_log2) / 8)) ||
      (rc = tab.ensure(table_bytes)))
    return rc;
  VATE_CUDA(cudaMemsetAsync(in.ptr, 0x5a, n2 * 16, p->stream));
  VATE_CUDA(cudaMemsetAsync(marks.ptr, 0, (1ull << mark_log2) / 8, p->stream));
  VATE_CUDA(cudaMemsetAsync(tab.ptr, 0, table_bytes, p->stream));
  const uint64_t want = std::max<uint64_t>(148ull * 16u, n2 / (4ull * 256u));
  const uint32_t grid = (uint32_t)std::min<uint64_t>(std::min<uint64_t>(want, 148ull * 64u),
                                                     (n2 + 255) / 256);
  cudaEvent_t a, b;
  VATE_CUDA(cudaEventCreate(&a));
  VATE_CUDA(cudaEventCreate(&b));
  for (int r = -1; r < reps; ++r) {
    if (r == 0) VATE_CUDA(cudaEventRecord(a, p->stream));
    static void (*const fns[48])(vate_pool*, uint32_t, const uint4*, uint64_t, uint32_t*,
                                 uint32_t, uint4*, uint32_t) = {
        launch_skeleton<0>, launch_skeleton<1>, launch_skeleton<2>, launch_skeleton<3>,
        launch_skeleton<4>, launch_skeleton<5>, launch_skeleton<6>, launch_skeleton<7>,
        launch_skeleton<8>, launch_skeleton<9>, launch_skeleton<10>, launch_skeleton<11>,
        launch_skeleton<12>, launch_skeleton<13>, launch_skeleton<14>, launch_skeleton<15>,
        launch_skeleton<16>, launch_skeleton<17>, launch_skeleton<18>, launch_skeleton<19>,
        launch_skeleton<20>, launch_skeleton<21>, launch_skeleton<22>, launch_skeleton<23>,
        launch_skeleton<24>, launch_skeleton<25>, launch_skeleton<26>, launch_skeleton<27>,
        launch_skeleton<28>, launch_skeleton<29>, launch_skeleton<30>, launch_skeleton<31>,
        launch_skeleton<32>, launch_skeleton<33>, launch_skeleton<34>, launch_skeleton<35>,
        launch_skeleton<36>, launch_skeleton<37>, launch_skeleton<38>, launch_skeleton<39>,
        launch_skeleton<40>, launch_skeleton<41>, launch_skeleton<42>, launch_skeleton<43>,
        launch_skeleton<44>, launch_skeleton<45>, launch_skeleton<46>, launch_skeleton<47>};
    fns[flags](p, grid, in.as<const uint4>(), n2, marks.as<uint32_t>(),
               (uint32_t)((1ull << mark_log2) - 1), tab.as<uint4>(),
               (uint32_t)(table_bytes / 32 - 1));
    VATE_CUDA(cudaGetLastError());
  }
  VATE_CUDA(cudaEventRecord(b, p->stream));
  VATE_CUDA(cudaEventSynchronize(b));
  float t = 0.f;
  VATE_CUDA(cudaEventElapsedTime(&t, a, b));
  *ms_out = t / reps;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  in.release();
  marks.release();
  tab.release();
  return VATE_OK;
}

// out[0] random 32-B sector reads (G sectors/s), out[1] random 2-byte stores
// (G stores/s = G sectors/s), out[2] random red.or (G ops/s, the scan's mark),
// out[3] streaming read (GB/s), all over a buf_bytes (power of two) buffer.
extern "C" int vate_bench_l2(vate_pool* p, uint64_t buf_bytes, uint64_t n, int reps,
                             double out[4]) {
  int rc = enter(p);
  if (rc) return rc;
  if (buf_bytes < 4096 || (buf_bytes & (buf_bytes - 1)) || buf_bytes > (1ull << 32))
    return set_error(VATE_EVALUE, "buf_bytes must be a power of two in [4 KiB, 4 GiB]");
  if (reps < 1 || n < 1) return set_error(VATE_EVALUE, "reps and n must be >= 1");
  DevBuf buf;
  rc = buf.ensure(buf_bytes);
  if (rc) return rc;
  VATE_CUDA(cudaMemsetAsync(buf.ptr, 0, buf_bytes, p->stream));
  cudaEvent_t a, b;
  VATE_CUDA(cudaEventCreate(&a));
  VATE_CUDA(cudaEventCreate(&b));
  const uint32_t grid = 148u * 32u;
  const uint32_t nsec = (uint32_t)(buf_bytes / 32);
  double ms[4] = {0, 0, 0, 0};
  for (int probe = 0; probe < 4; ++probe) {
    for (int r = -1; r < reps; ++r) {  // r = -1: warm-up (the buffer into L2)
      if (r == 0) VATE_CUDA(cudaEventRecord(a, p->stream));
      const uint32_t seed = 0x5bd1e995u * (uint32_t)(r + 2);
      switch (probe) {
        case 0:
          VATE_LAUNCH(p, VATE_K_OTHER, grid, 256, 0, k_l2_gather, buf.as<const uint4>(), nsec - 1,
                      n, seed, (unsigned*)p->d_ctr + 2 * C_TRACE);
          break;
        case 1:
          VATE_LAUNCH(p, VATE_K_OTHER, grid, 256, 0, k_l2_store, buf.as<uint16_t>(),
                      (uint32_t)(buf_bytes / 2 - 1), n, seed);
          break;
        case 2:
          VATE_LAUNCH(p, VATE_K_OTHER, grid, 256, 0, k_l2_red, buf.as<uint32_t>(),
                      (uint32_t)(buf_bytes * 8 - 1), n, seed);
          break;
        default:
          VATE_LAUNCH(p, VATE_K_OTHER, grid, 256, 0, k_l2_stream, buf.as<const uint4>(),
                      buf_bytes / 16, (unsigned*)p->d_ctr + 2 * C_TRACE);
          break;
      }
    }
    VATE_CUDA(cudaEventRecord(b, p->stream));
    VATE_CUDA(cudaEventSynchronize(b));
    float t = 0.f;
    VATE_CUDA(cudaEventElapsedTime(&t, a, b));
    ms[probe] = t / reps;
  }
  out[0] = (double)n / (ms[0] * 1e-3) / 1e9;
  out[1] = (double)n / (ms[1] * 1e-3) / 1e9;
  out[2] = (double)n / (ms[2] * 1e-3) / 1e9;
  out[3] = (double)buf_bytes / (ms[3] * 1e-3) / 1e9;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  buf.release();
  return VATE_OK;
}
