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

}  // namespace vate

using namespace vate;

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
