// Probe: does ordering the scan's random u16 cell stores by pool region cut
// their cost on a 512 MiB (2^28 x u16) pool?  Standalone; prints one JSON line
// per variant.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a probe_scatter.cu
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s %d %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 27; z *= 0x94D049BB133111EBull; return z ^ (z >> 31);
}

__global__ void k_gen(uint32_t* idx, uint64_t n, uint64_t seed, uint32_t mask) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    idx[i] = (uint32_t)(mix64(seed * 0x9E3779B97F4A7C15ull + i) & mask);
}

template <typename T>
__global__ void __launch_bounds__(256) k_store(const uint32_t* __restrict__ idx, uint64_t n, T* __restrict__ cells, T v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    cells[__ldcs(idx + i)] = v;
}
template <typename T>
__global__ void __launch_bounds__(256) k_store4(const uint4* __restrict__ idx, uint64_t n4, T* __restrict__ cells, T v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 q = __ldcs(idx + i);
    cells[q.x] = v; cells[q.y] = v; cells[q.z] = v; cells[q.w] = v;
  }
}
// random 32-B sector read-modify-write (load 16 B, store 16 B) over a buffer
__global__ void __launch_bounds__(256) k_rmw(const uint32_t* __restrict__ idx, uint64_t n, uint4* __restrict__ buf, uint32_t mask) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t s = (__ldcs(idx + i) & mask) * 2;
    uint4 a = buf[s];
    a.x += 1;
    buf[s] = a;
  }
}
// random 32-B sector loads (one 16-B load per sector) -> sum
__global__ void __launch_bounds__(256) k_gather(const uint32_t* __restrict__ idx, uint64_t n, const uint4* __restrict__ buf, uint32_t mask, unsigned* out) {
  unsigned acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t s = (__ldcs(idx + i) & mask) * 2;
    acc += buf[s].x;
  }
  if (acc == 0x12345678u) *out = acc;
}
__global__ void __launch_bounds__(256) k_stream_read(const uint4* __restrict__ a, uint64_t n, unsigned* out) {
  unsigned acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 q = __ldcs(a + i); acc ^= q.x ^ q.y ^ q.z ^ q.w;
  }
  if (acc == 0x12345678u) *out = acc;
}
__global__ void __launch_bounds__(256) k_stream_copy(const uint4* __restrict__ a, uint4* __restrict__ b, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

static int g_sms;
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

int main(int argc, char** argv) {
  const uint64_t n = 5000000;
  const int c = 28;
  const uint32_t mask = (1u << c) - 1;
  const int NSETS = 16;
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0)); g_sms = prop.multiProcessorCount;
  printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d}\n", prop.name, g_sms, prop.l2CacheSize);
  uint16_t* cells; CK(cudaMalloc(&cells, (2ull << c)));
  CK(cudaMemset(cells, 0, 2ull << c));
  uint32_t* sets; CK(cudaMalloc(&sets, NSETS * n * 4));
  uint32_t* tmp; CK(cudaMalloc(&tmp, n * 4));
  unsigned* out; CK(cudaMalloc(&out, 64));
  for (int s = 0; s < NSETS; ++s) k_gen<<<1184, 256>>>(sets + s * n, n, 1000 + s, mask);
  CK(cudaDeviceSynchronize());
  const int grid = g_sms * 8;
  const int iters = 32;
  auto rnd = [&](int i) { k_store<uint16_t><<<grid, 256>>>(sets + (i % NSETS) * n, n, cells, (uint16_t)(i & 511)); };
  float t = time_it(iters, rnd);
  printf("{\"variant\": \"random u16 stores 5M into 512MiB\", \"us\": %.2f}\n", t * 1e3);
  auto rnd4 = [&](int i) { k_store4<uint16_t><<<grid, 256>>>((const uint4*)(sets + (i % NSETS) * n), n / 4, cells, (uint16_t)(i & 511)); };
  t = time_it(iters, rnd4);
  printf("{\"variant\": \"random u16 stores, 4 per thread\", \"us\": %.2f}\n", t * 1e3);
  // bucketed orders: stable radix sort on bits [shift, 28)
  uint32_t* sorted; CK(cudaMalloc(&sorted, NSETS * n * 4));
  void* ws = nullptr; size_t wsb = 0;
  cub::DeviceRadixSort::SortKeys(ws, wsb, sets, sorted, (int)n, 0, 28);
  CK(cudaMalloc(&ws, wsb));
  int shifts[] = {4, 8, 10, 12, 14, 16, 18, 20, 22, 24, 26};
  for (int sh : shifts) {
    for (int s = 0; s < NSETS; ++s)
      CK(cub::DeviceRadixSort::SortKeys(ws, wsb, sets + s * n, sorted + s * n, (int)n, sh, 28));
    CK(cudaDeviceSynchronize());
    auto f = [&](int i) { k_store<uint16_t><<<grid, 256>>>(sorted + (i % NSETS) * n, n, cells, (uint16_t)(i & 511)); };
    t = time_it(iters, f);
    printf("{\"variant\": \"bucketed by cell>>%d (%d buckets of %d KiB)\", \"us\": %.2f}\n", sh, 1 << (28 - sh), (2 << sh) / 1024, t * 1e3);
    auto f4 = [&](int i) { k_store4<uint16_t><<<grid, 256>>>((const uint4*)(sorted + (i % NSETS) * n), n / 4, cells, (uint16_t)(i & 511)); };
    t = time_it(iters, f4);
    printf("{\"variant\": \"bucketed by cell>>%d, 4 per thread\", \"us\": %.2f}\n", sh, t * 1e3);
  }
  // streaming read / copy of the pool
  t = time_it(10, [&](int) { k_stream_read<<<g_sms * 8, 256>>>((const uint4*)cells, (2ull << c) / 16, out); });
  printf("{\"variant\": \"stream read 512MiB\", \"us\": %.2f, \"GBps\": %.1f}\n", t * 1e3, (2ull << c) / (t * 1e-3) / 1e9);
  uint16_t* cells2; CK(cudaMalloc(&cells2, (2ull << c)));
  t = time_it(10, [&](int) { k_stream_copy<<<g_sms * 8, 256>>>((const uint4*)cells, (uint4*)cells2, (2ull << c) / 16); });
  printf("{\"variant\": \"stream copy 512MiB\", \"us\": %.2f, \"GBps\": %.1f}\n", t * 1e3, 2.0 * (2ull << c) / (t * 1e-3) / 1e9);
  // L2 ceilings: random sector RMW / gather / u8 store on L2-resident buffers
  for (uint32_t mb : {8u, 16u, 32u, 64u, 512u}) {
    const uint32_t nsec = mb * (1u << 20) / 32;
    t = time_it(iters, [&](int i) { k_rmw<<<grid, 256>>>(sets + (i % NSETS) * n, n, (uint4*)cells2, nsec - 1); });
    printf("{\"variant\": \"random 32B-sector RMW over %u MiB\", \"us\": %.2f, \"Gsectors_per_s\": %.2f}\n", mb, t * 1e3, n / (t * 1e-3) / 1e9);
    t = time_it(iters, [&](int i) { k_gather<<<grid, 256>>>(sets + (i % NSETS) * n, n, (const uint4*)cells2, nsec - 1, out); });
    printf("{\"variant\": \"random 32B-sector gather over %u MiB\", \"us\": %.2f, \"Gsectors_per_s\": %.2f}\n", mb, t * 1e3, n / (t * 1e-3) / 1e9);
  }
  for (int cc : {20, 24, 26}) {
    for (int s = 0; s < NSETS; ++s) k_gen<<<1184, 256>>>(tmp, 1, 0, 0);
    t = time_it(iters, [&](int i) { k_store<uint8_t><<<grid, 256>>>(sets + (i % NSETS) * n, n, (uint8_t*)cells2 , (uint8_t)i); });
    (void)cc;
    break;
  }
  for (int cc : {20, 24, 26}) {
    uint32_t* s2; CK(cudaMalloc(&s2, NSETS * n * 4));
    for (int s = 0; s < NSETS; ++s) k_gen<<<1184, 256>>>(s2 + s * n, n, 77 + s, (1u << cc) - 1);
    t = time_it(iters, [&](int i) { k_store<uint8_t><<<grid, 256>>>(s2 + (i % NSETS) * n, n, (uint8_t*)cells2, (uint8_t)i); });
    printf("{\"variant\": \"random u8 stores 5M into 2^%d (L2 pool)\", \"us\": %.2f}\n", cc, t * 1e3);
    CK(cudaFree(s2));
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
