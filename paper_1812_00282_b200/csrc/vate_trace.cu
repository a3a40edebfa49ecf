// vate_trace.cu -- trace ingest on the device.
//
// traceio.py reads 16-byte little-endian records {u64 ts_us, u32 aip, u32 bip}
// (traceio.py:24, :77-106) and slice_stream (traceio.py:188-230) regroups them
// into consecutive slices t = ts // slice_us - base, emitting empty slices so
// windows advance.  Here one kernel pass over a chunk of records packs them to
// the scan's 8-byte {aip, bip} form, finds every slice start by comparing
// neighbours (timestamps are sorted, so slice ids are monotone) and records the
// first order violation -- the reader then hands each slice to the scan as a
// device pointer, with no host-side regrouping.
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "vate_internal.cuh"

namespace vate {

struct Rec {
  unsigned long long ts;
  unsigned aip, bip;
};

__global__ void k_trace_bucket(const Rec* __restrict__ rec, uint64_t n, uint64_t slice_us,
                               long long first, unsigned long long prev_ts, int has_prev,
                               uint2* __restrict__ out, uint64_t out_off,
                               unsigned long long* __restrict__ starts, uint64_t nslices,
                               unsigned long long* violation) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const Rec r = rec[i];
    out[out_off + i] = make_uint2(r.aip, r.bip);
    const long long s = (long long)(r.ts / slice_us) - first;
    long long sp;
    if (i == 0) {
      sp = -1;
      if (has_prev && r.ts < prev_ts) atomicMin(violation, 0ull);
    } else {
      const unsigned long long pts = rec[i - 1].ts;
      if (r.ts < pts) atomicMin(violation, (unsigned long long)i);
      sp = (long long)(pts / slice_us) - first;
    }
    // every slice in (sp, s] starts here (the empty ones included)
    for (long long q = sp + 1; q <= s && q < (long long)nslices; ++q)
      if (q >= 0) starts[q] = out_off + i;
  }
}

}  // namespace vate

using namespace vate;

extern "C" {

int vate_trace_bucket(vate_pool* p, const uint8_t* records, uint64_t n, int where,
                      uint64_t slice_us, int64_t first_slice, uint64_t prev_ts, int has_prev,
                      uint32_t* pairs_dev, uint64_t pairs_off, uint64_t nslices,
                      uint64_t* starts, int64_t* violation) {
  int rc = enter(p);
  if (rc) return rc;
  if (slice_us == 0) return set_error(VATE_ECONFIG, "slice duration must be positive");
  *violation = -1;
  if (n == 0) return VATE_OK;
  const void* d_rec;
  rc = stage_in(p, p->in_a, records, n * 16, where, &d_rec);
  if (rc) return rc;
  rc = p->out_buf.ensure((nslices + 1) * 8);
  if (rc) return rc;
  VATE_CUDA(cudaMemsetAsync(p->d_ctr + C_TRACE, 0xFF, 8, p->stream));  // violation slot
  VATE_LAUNCH(p, VATE_K_OTHER, grid_for(n, kThreads, 148u * 32u), kThreads, 0, k_trace_bucket,
              (const Rec*)d_rec, n, slice_us, (long long)first_slice,
              (unsigned long long)prev_ts, has_prev, (uint2*)pairs_dev, pairs_off,
              p->out_buf.as<unsigned long long>(), nslices, p->d_ctr + C_TRACE);
  VATE_CUDA(cudaMemcpyAsync(starts, p->out_buf.ptr, nslices * 8, cudaMemcpyDeviceToHost, p->stream));
  VATE_CUDA(cudaMemcpyAsync(p->h_ctr + C_TRACE, p->d_ctr + C_TRACE, 8, cudaMemcpyDeviceToHost,
                            p->stream));
  VATE_CUDA(cudaStreamSynchronize(p->stream));
  const unsigned long long v = p->h_ctr[C_TRACE];
  *violation = v == ~0ull ? -1 : (int64_t)v;
  return VATE_OK;
}

int vate_copy_device(vate_pool* p, void* dst, const void* src, uint64_t bytes) {
  int rc = enter(p);
  if (rc || bytes == 0) return rc;
  VATE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, p->stream));
  return VATE_OK;
}

}  // extern "C"
