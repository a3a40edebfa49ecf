// Probe: the deferred scatter for pools beyond L2.  Instead of a random u16
// store into the 512 MiB cell array (a DRAM sector read + write per packet),
// the scan sets one bit per packet in an L2-resident 32 MiB mark bitmap
// (red.global.or), and the next whole-pool pass applies the marks while it
// streams the cells anyway.  Times: random stores into 512 MiB vs random
// red.or into 32 MiB (5M and 100M per launch), and a streaming pass over the
// u16 cells that applies marks and writes back only changed 16-B vectors.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a probe_marks.cu
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s %d %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 27; z *= 0x94D049BB133111EBull; return z ^ (z >> 31);
}

__global__ void k_gen(uint32_t* idx, uint64_t n, uint64_t seed, uint32_t mask) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    idx[i] = (uint32_t)(mix64(seed * 0x9E3779B97F4A7C15ull + i) & mask);
}

__global__ void __launch_bounds__(256) k_store(const uint4* __restrict__ idx, uint64_t n4, uint16_t* __restrict__ cells, uint16_t v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 q = __ldcs(idx + i);
    cells[q.x] = v; cells[q.y] = v; cells[q.z] = v; cells[q.w] = v;
  }
}
__global__ void __launch_bounds__(256) k_mark(const uint4* __restrict__ idx, uint64_t n4, uint32_t* __restrict__ marks) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 q = __ldcs(idx + i);
    atomicOr(marks + (q.x >> 5), 1u << (q.x & 31));
    atomicOr(marks + (q.y >> 5), 1u << (q.y & 31));
    atomicOr(marks + (q.z >> 5), 1u << (q.z & 31));
    atomicOr(marks + (q.w >> 5), 1u << (q.w & 31));
  }
}
// whole-pool pass: 32 u16 cells per thread-word; marked cells take v; changed
// vectors are stored; marks cleared; an "active" bitmap word written.
__global__ void __launch_bounds__(256) k_apply(uint16_t* __restrict__ cells, uint32_t* __restrict__ marks,
                                               uint32_t* __restrict__ bits, uint64_t nwords, uint16_t v) {
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += (uint64_t)gridDim.x * blockDim.x) {
    uint4 r[4];
    const uint4* src = reinterpret_cast<const uint4*>(cells + w * 32);
    const uint32_t m = __ldcg(marks + w);
#pragma unroll
    for (int q = 0; q < 4; ++q) r[q] = __ldcs(src + q);
    uint32_t* x = reinterpret_cast<uint32_t*>(r);
    unsigned changed = 0, act = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      uint32_t lo = x[q] & 0xFFFF, hi = x[q] >> 16;
      if ((m >> (2 * q)) & 1) lo = v;
      if ((m >> (2 * q + 1)) & 1) hi = v;
      const uint32_t y = lo | (hi << 16);
      if (y != x[q]) changed |= 1u << (q / 4);
      x[q] = y;
      act |= (uint32_t)(lo == v) << (2 * q) | (uint32_t)(hi == v) << (2 * q + 1);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if ((changed >> q) & 1) reinterpret_cast<uint4*>(cells + w * 32)[q] = r[q];
    if (m) marks[w] = 0;
    bits[w] = act;
  }
}
__global__ void __launch_bounds__(256) k_readpass(const uint16_t* __restrict__ cells, uint32_t* __restrict__ bits, uint64_t nwords, uint16_t v) {
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += (uint64_t)gridDim.x * blockDim.x) {
    uint4 r[4];
    const uint4* src = reinterpret_cast<const uint4*>(cells + w * 32);
#pragma unroll
    for (int q = 0; q < 4; ++q) r[q] = __ldcs(src + q);
    const uint32_t* x = reinterpret_cast<const uint32_t*>(r);
    uint32_t act = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) act |= (uint32_t)((x[q] & 0xFFFF) == v) << (2 * q) | (uint32_t)((x[q] >> 16) == v) << (2 * q + 1);
    bits[w] = act;
  }
}


template <bool EF, bool WHOLE>
__global__ void __launch_bounds__(256) k_apply2(uint16_t* __restrict__ cells, uint32_t* __restrict__ marks,
                                                uint32_t* __restrict__ bits, uint64_t nwords, uint16_t v) {
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += (uint64_t)gridDim.x * blockDim.x) {
    uint4 r[4];
    const uint4* src = reinterpret_cast<const uint4*>(cells + w * 32);
    uint32_t m;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(m) : "l"(marks + w));
#pragma unroll
    for (int q = 0; q < 4; ++q) r[q] = EF ? __ldcs(src + q) : __ldcg(src + q);
    uint32_t x[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) { x[4*q] = r[q].x; x[4*q+1] = r[q].y; x[4*q+2] = r[q].z; x[4*q+3] = r[q].w; }
    unsigned changed = 0, act = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      uint32_t lo = x[q] & 0xFFFF, hi = x[q] >> 16;
      if ((m >> (2 * q)) & 1) lo = v;
      if ((m >> (2 * q + 1)) & 1) hi = v;
      const uint32_t y = lo | (hi << 16);
      if (y != x[q]) changed |= 1u << (q / 4);
      x[q] = y;
      act |= (uint32_t)(lo == v) << (2 * q) | (uint32_t)(hi == v) << (2 * q + 1);
    }
    if (WHOLE && changed) changed = 0xF;
    uint4* dst = reinterpret_cast<uint4*>(cells + w * 32);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if ((changed >> q) & 1) dst[q] = make_uint4(x[4*q], x[4*q+1], x[4*q+2], x[4*q+3]);
    if (m) asm volatile("st.global.u32 [%0], %1;" :: "l"(marks + w), "r"(0u) : "memory");
    bits[w] = act;
  }
}

template <typename F>
static float time_it(int iters, F launch) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  for (int i = 0; i < 3; ++i) launch(i);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int i = 0; i < iters; ++i) launch(i + 3);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  return ms / iters;
}

int main() {
  const int c = 28;
  const uint64_t S = 1ull << c, nwords = S / 32;
  const uint32_t mask = (uint32_t)(S - 1);
  const int NSETS = 8;
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  uint16_t* cells; CK(cudaMalloc(&cells, S * 2)); CK(cudaMemset(cells, 0, S * 2));
  uint32_t *marks, *bits; CK(cudaMalloc(&marks, S / 8)); CK(cudaMalloc(&bits, S / 8));
  CK(cudaMemset(marks, 0, S / 8));
  for (uint64_t n : {5000000ull, 100000000ull}) {
    const int nsets = n > 10000000ull ? 2 : NSETS;
    uint32_t* sets; CK(cudaMalloc(&sets, nsets * n * 4));
    for (int s = 0; s < nsets; ++s) k_gen<<<sms * 8, 256>>>(sets + s * n, n, 1000 + s, mask);
    CK(cudaDeviceSynchronize());
    const int grid = sms * 8, iters = n > 10000000ull ? 4 : 20;
    float t = time_it(iters, [&](int i) { k_store<<<grid, 256>>>((const uint4*)(sets + (i % nsets) * n), n / 4, cells, (uint16_t)(i & 511)); });
    printf("{\"variant\": \"random u16 stores into 512 MiB\", \"n\": %llu, \"us\": %.2f, \"Gpps\": %.2f}\n", (unsigned long long)n, t * 1e3, n / (t * 1e-3) / 1e9);
    t = time_it(iters, [&](int i) { k_mark<<<grid, 256>>>((const uint4*)(sets + (i % nsets) * n), n / 4, marks); });
    printf("{\"variant\": \"random red.or into 32 MiB marks (no clear)\", \"n\": %llu, \"us\": %.2f, \"Gpps\": %.2f}\n", (unsigned long long)n, t * 1e3, n / (t * 1e-3) / 1e9);
    // mark + apply pass pairs
    float tm = 0, ta = 0;
    cudaEvent_t e0, e1, e2; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1)); CK(cudaEventCreate(&e2));
    CK(cudaMemset(marks, 0, S / 8));
    for (int i = 0; i < iters + 2; ++i) {
      CK(cudaEventRecord(e0));
      k_mark<<<grid, 256>>>((const uint4*)(sets + (i % nsets) * n), n / 4, marks);
      CK(cudaEventRecord(e1));
      k_apply<<<sms * 32, 256>>>(cells, marks, bits, nwords, (uint16_t)(i & 511));
      CK(cudaEventRecord(e2));
      CK(cudaEventSynchronize(e2));
      float a, b; CK(cudaEventElapsedTime(&a, e0, e1)); CK(cudaEventElapsedTime(&b, e1, e2));
      if (i >= 2) { tm += a; ta += b; }
    }
    printf("{\"variant\": \"mark (marks cleared by the pass) + apply pass\", \"n\": %llu, \"mark_us\": %.2f, \"apply_us\": %.2f}\n",
           (unsigned long long)n, tm / iters * 1e3, ta / iters * 1e3);
    auto pair = [&](const char* name, auto apply) {
      float tm2 = 0, ta2 = 0;
      for (int i = 0; i < iters + 2; ++i) {
        CK(cudaEventRecord(e0));
        k_mark<<<grid, 256>>>((const uint4*)(sets + (i % nsets) * n), n / 4, marks);
        CK(cudaEventRecord(e1));
        apply(i);
        CK(cudaEventRecord(e2));
        CK(cudaEventSynchronize(e2));
        float a, b; CK(cudaEventElapsedTime(&a, e0, e1)); CK(cudaEventElapsedTime(&b, e1, e2));
        if (i >= 2) { tm2 += a; ta2 += b; }
      }
      printf("{\"variant\": \"%s\", \"n\": %llu, \"mark_us\": %.2f, \"apply_us\": %.2f}\n", name,
             (unsigned long long)n, tm2 / iters * 1e3, ta2 / iters * 1e3);
    };
    pair("apply2 EF partial", [&](int i) { k_apply2<true, false><<<sms * 32, 256>>>(cells, marks, bits, nwords, (uint16_t)(i & 511)); });
    pair("apply2 EF whole", [&](int i) { k_apply2<true, true><<<sms * 32, 256>>>(cells, marks, bits, nwords, (uint16_t)(i & 511)); });
    pair("apply2 CG partial", [&](int i) { k_apply2<false, false><<<sms * 32, 256>>>(cells, marks, bits, nwords, (uint16_t)(i & 511)); });
    pair("apply2 CG whole", [&](int i) { k_apply2<false, true><<<sms * 32, 256>>>(cells, marks, bits, nwords, (uint16_t)(i & 511)); });
    pair("apply2 EF whole, grid 148x8", [&](int i) { k_apply2<true, true><<<sms * 8, 256>>>(cells, marks, bits, nwords, (uint16_t)(i & 511)); });
    pair("apply2 EF whole, 1 word/thread", [&](int i) { k_apply2<true, true><<<(unsigned)(nwords / 256), 256>>>(cells, marks, bits, nwords, (uint16_t)(i & 511)); });

    CK(cudaFree(sets));
  }
  float t = time_it(10, [&](int i) { k_readpass<<<sms * 32, 256>>>(cells, bits, nwords, (uint16_t)i); });
  printf("{\"variant\": \"read-only pass over 512 MiB u16 + bitmap write\", \"us\": %.2f, \"GBps\": %.1f}\n", t * 1e3, (S * 2 + S / 8) / (t * 1e-3) / 1e9);
  return 0;
}
