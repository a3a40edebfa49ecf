// vate_trace.cu -- trace ingest on the device.
//
// traceio.py reads 16-byte little-endian records {u64 ts_us, u32 aip, u32 bip}
// (traceio.py:24, :77-106) and slice_stream (traceio.py:188-230) regroups them
// into consecutive slices t = ts // slice_us - base, emitting empty slices so
// windows advance.  Here one kernel pass over a chunk of records packs them to
// the scan's 8-byte {aip, bip} form, records one run per slice change
// (timestamps are sorted, so slice ids are monotone) and the first order
// violation -- the reader then hands each slice to the scan as a device
// pointer, with no host-side regrouping.
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "vate_internal.cuh"

namespace vate {

struct Rec {
  unsigned long long ts;
  unsigned aip, bip;
};

}  // namespace vate

using namespace vate;

extern "C" {

}  // extern "C"

// ---------------------------------------------------------------------------
// Line-rate ingest (traceio.DeviceSlices): a tracer owns two pinned host
// staging buffers the reader fills straight from the file, two device record
// buffers, two packed-pair buffers and its own stream.  Per chunk: H2D of the
// records (async, from pinned memory), the carried tail of the previous chunk's
// last slice copied to the pair buffer's start, then k_trace_runs packs the
// records and appends one (slice, offset) run per slice change -- runs, not a
// dense per-slice table, so an idle gap costs nothing (empty slices are
// emitted lazily by the reader) -- and the runs, their count and the first
// order violation come back to pinned memory.  The pool's compute stream waits
// for the chunk by event; a pair buffer is rewritten only after the scans that
// read it (vate_tracer_release records when they were enqueued).
// ---------------------------------------------------------------------------
namespace vate {

__global__ void k_trace_runs(const Rec* __restrict__ rec, uint64_t n, uint64_t slice_us,
                             long long first, unsigned long long prev_ts, int has_prev,
                             uint2* __restrict__ out, uint64_t out_off,
                             unsigned long long* __restrict__ runs, unsigned long long* nruns,
                             unsigned long long* violation) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const Rec r = rec[i];
    out[out_off + i] = make_uint2(r.aip, r.bip);
    const long long s = (long long)(r.ts / slice_us) - first;
    bool change;
    if (i == 0) {
      change = true;
      if (has_prev && r.ts < prev_ts) atomicMin(violation, 0ull);
    } else {
      const unsigned long long pts = rec[i - 1].ts;
      if (r.ts < pts) atomicMin(violation, (unsigned long long)i);
      change = (long long)(pts / slice_us) - first != s;
    }
    if (change) {
      const unsigned long long k = atomicAdd(nruns, 1ull);
      runs[2 * k] = (unsigned long long)s;
      runs[2 * k + 1] = out_off + i;
    }
  }
}

}  // namespace vate

struct vate_tracer {
  vate_pool* pool = nullptr;
  int device = 0;                                    // (the pool may be gone at destroy)
  uint64_t chunk = 0, slice_us = 1;
  cudaStream_t stream = nullptr;
  uint8_t* host[2] = {nullptr, nullptr};            // pinned record staging
  unsigned long long* h_meta[2] = {nullptr, nullptr};  // pinned: [0] nruns, [1] violation, runs...
  vate::DevBuf rec[2], pairs[2], meta[2];
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr},
              ev_release[2] = {nullptr, nullptr};
};

extern "C" {

int vate_tracer_create(vate_tracer** out, vate_pool* p, uint64_t chunk, uint64_t slice_us) {
  int rc = enter(p);
  if (rc) return rc;
  if (!out || chunk == 0) return set_error(VATE_EVALUE, "null output or empty chunk");
  if (slice_us == 0) return set_error(VATE_ECONFIG, "slice duration must be positive");
  vate_tracer* x = new vate_tracer();
  x->pool = p;
  x->device = p->device;
  x->chunk = chunk;
  x->slice_us = slice_us;
  cudaError_t e = cudaStreamCreateWithFlags(&x->stream, cudaStreamNonBlocking);
  for (int s = 0; s < 2 && e == cudaSuccess; ++s) {
    e = cudaHostAlloc((void**)&x->host[s], chunk * 16, cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaHostAlloc((void**)&x->h_meta[s], (2 * chunk + 2) * 8, cudaHostAllocDefault);
    for (cudaEvent_t* ev : {&x->ev_h2d[s], &x->ev_done[s], &x->ev_release[s]})
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(x->ev_release[s], x->stream);
    if (e == cudaSuccess) e = cudaEventRecord(x->ev_h2d[s], x->stream);
  }
  if (e == cudaSuccess) {
    for (int s = 0; s < 2 && rc == VATE_OK; ++s) {
      rc = x->rec[s].ensure(chunk * 16);
      if (!rc) rc = x->pairs[s].ensure(chunk * 8);
      if (!rc) rc = x->meta[s].ensure((2 * chunk + 2) * 8);
    }
  } else {
    rc = cuda_fail(e, "vate_tracer_create");
  }
  if (rc) {
    vate_tracer_destroy(x);
    return rc;
  }
  *out = x;
  return VATE_OK;
}

int vate_tracer_destroy(vate_tracer* x) {
  if (!x) return VATE_OK;
  cudaSetDevice(x->device);
  if (x->stream) cudaStreamSynchronize(x->stream);
  for (int s = 0; s < 2; ++s) {
    if (x->host[s]) cudaFreeHost(x->host[s]);
    if (x->h_meta[s]) cudaFreeHost(x->h_meta[s]);
    x->rec[s].release();
    x->pairs[s].release();
    x->meta[s].release();
    for (cudaEvent_t ev : {x->ev_h2d[s], x->ev_done[s], x->ev_release[s]})
      if (ev) cudaEventDestroy(ev);
  }
  if (x->stream) cudaStreamDestroy(x->stream);
  delete x;
  return VATE_OK;
}

// The pinned staging buffer of a slot, once its previous H2D has finished.
int vate_tracer_buffer(vate_tracer* x, int slot, uint8_t** host) {
  if (!x || slot < 0 || slot > 1) return set_error(VATE_EVALUE, "bad tracer slot");
  int rc = enter(x->pool);
  if (rc) return rc;
  VATE_CUDA(cudaEventSynchronize(x->ev_h2d[slot]));
  *host = x->host[slot];
  return VATE_OK;
}

// Submit n records (in the slot's staging buffer): H2D, the carried pairs
// (carry_n pairs at carry_off of the other slot's pair buffer) to the start of
// this slot's pair buffer, then the packing / run kernel.  Asynchronous.
int vate_tracer_submit(vate_tracer* x, int slot, uint64_t n, int64_t first_slice,
                       uint64_t prev_ts, int has_prev, uint64_t carry_off, uint64_t carry_n) {
  if (!x || slot < 0 || slot > 1) return set_error(VATE_EVALUE, "bad tracer slot");
  vate_pool* p = x->pool;
  int rc = enter(p);
  if (rc) return rc;
  if (n > x->chunk) return set_error(VATE_EVALUE, "chunk larger than the tracer's buffers");
  if (carry_n + n > x->chunk) {  // a slice longer than a chunk: grow this pair buffer
    VATE_CUDA(cudaEventSynchronize(x->ev_release[slot]));
    rc = x->pairs[slot].ensure((carry_n + n) * 8);
    if (rc) return rc;
  }
  cudaStream_t s = x->stream;
  VATE_CUDA(cudaMemcpyAsync(x->rec[slot].ptr, x->host[slot], n * 16, cudaMemcpyHostToDevice, s));
  VATE_CUDA(cudaEventRecord(x->ev_h2d[slot], s));
  VATE_CUDA(cudaStreamWaitEvent(s, x->ev_release[slot], 0));  // scans of its last chunk enqueued
  if (carry_n)
    VATE_CUDA(cudaMemcpyAsync(x->pairs[slot].ptr, x->pairs[slot ^ 1].as<uint8_t>() + carry_off * 8,
                              carry_n * 8, cudaMemcpyDeviceToDevice, s));
  unsigned long long* meta = x->meta[slot].as<unsigned long long>();
  VATE_CUDA(cudaMemsetAsync(meta, 0, 8, s));
  VATE_CUDA(cudaMemsetAsync(meta + 1, 0xFF, 8, s));
  if (n) {
    k_trace_runs<<<grid_for(n, kThreads, 148u * 32u), kThreads, 0, s>>>(
        x->rec[slot].as<const Rec>(), n, x->slice_us, (long long)first_slice,
        (unsigned long long)prev_ts, has_prev, x->pairs[slot].as<uint2>(), carry_n, meta + 2,
        meta, meta + 1);
    p->launches++;
    VATE_CUDA(cudaGetLastError());
  }
  // the counters, then the runs (their count is known only on the device: copy
  // the capacity's worth lazily -- collect copies the used part)
  VATE_CUDA(cudaMemcpyAsync(x->h_meta[slot], meta, 16, cudaMemcpyDeviceToHost, s));
  VATE_CUDA(cudaEventRecord(x->ev_done[slot], s));
  return VATE_OK;
}

// Wait for a submitted chunk: its runs (slice relative to first_slice, pair
// offset; unsorted), their count, the first order violation (-1 none), and its
// pair buffer; the pool's compute stream is ordered after it.
int vate_tracer_collect(vate_tracer* x, int slot, uint64_t* runs, uint64_t cap, uint64_t* nruns,
                        int64_t* violation, uint32_t** pairs_dev) {
  if (!x || slot < 0 || slot > 1) return set_error(VATE_EVALUE, "bad tracer slot");
  vate_pool* p = x->pool;
  int rc = enter(p);
  if (rc) return rc;
  VATE_CUDA(cudaEventSynchronize(x->ev_done[slot]));
  const uint64_t nr = x->h_meta[slot][0];
  const unsigned long long v = x->h_meta[slot][1];
  *violation = v == ~0ull ? -1 : (int64_t)v;
  *nruns = nr;
  if (nr > cap) return set_error(VATE_EVALUE, "run buffer too small");
  if (nr)
    VATE_CUDA(cudaMemcpy(runs, x->meta[slot].as<unsigned long long>() + 2, nr * 16,
                         cudaMemcpyDeviceToHost));
  VATE_CUDA(cudaStreamWaitEvent(p->stream, x->ev_done[slot], 0));
  *pairs_dev = x->pairs[slot].as<uint32_t>();
  return VATE_OK;
}

// Every scan reading the slot's pair buffer has been enqueued on the pool's
// stream: the next submit into that slot waits for them.
int vate_tracer_release(vate_tracer* x, int slot) {
  if (!x || slot < 0 || slot > 1) return set_error(VATE_EVALUE, "bad tracer slot");
  int rc = enter(x->pool);
  if (rc) return rc;
  VATE_CUDA(cudaEventRecord(x->ev_release[slot], x->pool->stream));
  return VATE_OK;
}

}  // extern "C"
