// vate_compare.cu -- the comparator pools of the reference on the device
// (pools.py:301-410): DrPool (VDRE distance recorders)
// and TsPool (plain last-seen slice indices).  They exist to reproduce the
// paper's VATE-vs-VDRE maintenance contrast and the
// reference's AT == DR == TS estimate identity (test_estimator.py:233-255),
// so they share the AT pool's handle, scan kernels (ConstRule store), host
// registry, g0 gather and float path; only the cell predicate, the slice
// advance and the cell type differ:
//
//   DR: dr_bits(k) = k.bit_length() bits (counters.py:132-134) -> u8 / u16
//       cells, filled with k; set -> 0; advance -> v = min(v+1, k) for EVERY
//       cell (the whole-pool sweep VATE avoids), cleared = cells reaching k;
//       inactive(k') <=> v >= k'                           (pools.py:301-353)
//   TS: u64 cells, filled with TS_UNSET = 2^64-1 (counters.py:159); set -> t
//       (the pool's own slice index); advance -> t += 1, nothing maintained;
//       inactive(k') <=> v == TS_UNSET or t - v >= k' (u64)  (pools.py:356-410)
#include <string>

#include "vate_internal.cuh"

namespace vate {

constexpr unsigned long long kTsUnset = ~0ull;  // counters.py:159

struct CmpPred {
  int kind;
  uint32_t kp;
  unsigned long long now;
  template <typename T>
  __device__ __forceinline__ bool inactive(T v) const {
    if (kind == VATE_DR) return (uint64_t)v >= kp;
    const unsigned long long x = (unsigned long long)v;
    return x == kTsUnset || now - x >= (unsigned long long)kp;
  }
};

template <typename T>
__global__ void k_cmp_fill(T* __restrict__ cells, uint64_t n, T value) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    cells[i] = value;
}

// Inactive bitmap + P for the comparators: one 32-cell word per thread, 16-byte
// loads (32 cells = 32 / 64 / 256 bytes for u8 / u16 / u64).
template <typename T>
__global__ void __launch_bounds__(256) k_cmp_bitmap(const T* __restrict__ cells, uint64_t size,
                                                    CmpPred P, uint32_t* __restrict__ bitmap,
                                                    uint64_t nwords,
                                                    unsigned long long* pool_inactive,
                                                    DeltaOut D) {
  constexpr int NV = (int)sizeof(T) * 2;  // uint4 per 32 cells
  __shared__ DeltaStage ds;
  if (D.bprev) delta_stage_init(ds);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned local = 0;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += stride) {
    const uint64_t i0 = w * 32;
    uint32_t bits = 0;
    if (i0 + 32 <= size) {
      uint4 r[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) r[v] = __ldcs(reinterpret_cast<const uint4*>(cells + i0) + v);
      const T* e = reinterpret_cast<const T*>(r);
#pragma unroll
      for (int j = 0; j < 32; ++j) bits |= (uint32_t)P.inactive(e[j]) << j;
    } else {
      for (uint64_t j = 0; i0 + j < size; ++j) bits |= (uint32_t)P.inactive(cells[i0 + j]) << j;
    }
    bitmap[w] = bits;
    local += __popc(bits);
    if (D.bprev) delta_word(D, ds, bits, D.bprev[w], i0);
  }
  if (D.bprev) delta_flush(D, ds);
  local = __reduce_add_sync(0xffffffffu, local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(pool_inactive, (unsigned long long)local);
}

template <typename T>
__global__ void k_cmp_mask(const T* __restrict__ cells, uint64_t size,
                           const uint64_t* __restrict__ idx, uint64_t n, CmpPred P,
                           uint8_t* __restrict__ out, unsigned long long* err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t c = idx[i];
    if (c >= size) {
      *err = 1;
      out[i] = 0;
      continue;
    }
    out[i] = P.inactive(cells[c]);
  }
}

template <typename T>
__global__ void k_get64(const T* __restrict__ cells, uint64_t size, const uint64_t* __restrict__ idx,
                        uint64_t n, unsigned long long* __restrict__ out, unsigned long long* err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t c = idx[i];
    if (c >= size) {
      *err = 1;
      out[i] = 0;
      continue;
    }
    out[i] = (unsigned long long)cells[c];
  }
}

// PackedArray.set / set_one / set_range (bitpack.py:97-140): cells[idx] =
// value & mask; duplicate indices carry equal values (the reference's contract).
template <typename T>
__global__ void k_put64(T* __restrict__ cells, uint64_t size, const uint64_t* __restrict__ idx,
                        const unsigned long long* __restrict__ vals, uint64_t n,
                        unsigned long long mask, unsigned long long* err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t c = idx[i];
    if (c >= size) {
      *err = 1;
      continue;
    }
    cells[c] = (T)(vals[i] & mask);
  }
}

// DrPool.advance_slice (pools.py:339-349): every recorder slides by one,
// saturating at k; a streaming read-modify-write of the whole pool, 16 bytes
// per thread per step (HBM-bound: 2 * cell_bytes * 2^c per slice).
template <typename T>
__global__ void __launch_bounds__(256) k_dr_slide(T* __restrict__ cells, uint64_t size, uint32_t k,
                                                  unsigned long long* cleared) {
  constexpr int PER = 16 / (int)sizeof(T);
  const uint64_t nvec = size / PER;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned local = 0;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nvec; q += stride) {
    uint4 r = __ldcs(reinterpret_cast<const uint4*>(cells) + q);
    T* e = reinterpret_cast<T*>(&r);
    bool any = false;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const uint32_t v = e[j];
      if (v < k) {
        local += (v + 1 == k);
        e[j] = (T)(v + 1);
        any = true;
      }
    }
    if (any) __stcs(reinterpret_cast<uint4*>(cells) + q, r);
  }
  // tail (size < PER only happens for tiny pools)
  for (uint64_t i = nvec * PER + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < size;
       i += stride) {
    const uint32_t v = cells[i];
    if (v < k) {
      local += (v + 1 == k);
      cells[i] = (T)(v + 1);
    }
  }
  local = __reduce_add_sync(0xffffffffu, local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(cleared, (unsigned long long)local);
}

template <typename F>
static int with_cmp_cell(const vate_pool* p, F f) {
  if (p->kind == VATE_TS) return f(uint64_t{});
  if (p->cell_bytes == 1) return f(uint8_t{});
  return f(uint16_t{});
}

int cmp_fill(vate_pool* p) {
  const uint64_t S = p->L.size;
  return with_cmp_cell(p, [&](auto tag) -> int {
    using T = decltype(tag);
    const T init = p->kind == VATE_DR ? (T)p->k : (T)kTsUnset;
    VATE_LAUNCH(p, VATE_K_OTHER, grid_for(S, kThreads), kThreads, 0, k_cmp_fill<T>, (T*)p->cells,
                S, init);
    return VATE_OK;
  });
}

int cmp_build_bitmap(vate_pool* p, int k_prime, bool with_delta) {
  const uint64_t nwords = (p->L.size + 31) / 32;
  int rc = p->bitmap.ensure(nwords * 4 + 16);
  if (rc) return rc;
  VATE_CUDA(cudaMemsetAsync(p->d_ctr + C_P, 0, 8, p->stream));
  DeltaOut D{};
  if (with_delta) {  // the incremental g0's flipped cells, as in the AT pass
    IncIndex& I = p->inc;
    VATE_CUDA(cudaMemsetAsync(p->d_ctr + C_DCNT, 0, 16, p->stream));
    D = DeltaOut{I.bprev.as<const uint32_t>(), I.off.as<const uint32_t>(),
                 I.dlist.as<unsigned long long>(), I.dlist_cap, p->d_ctr + C_DCNT,
                 p->d_ctr + C_DWORK};
  }
  const CmpPred P{p->kind, (uint32_t)k_prime, p->ts_now};
  rc = with_cmp_cell(p, [&](auto tag) -> int {
    using T = decltype(tag);
    VATE_LAUNCH(p, VATE_K_BITMAP, grid_for(nwords, 256, 148u * 16u), 256, 0, k_cmp_bitmap<T>,
                (const T*)p->cells, p->L.size, P, p->bitmap.as<uint32_t>(), nwords,
                p->d_ctr + C_P, D);
    return VATE_OK;
  });
  if (rc) return rc;
  VATE_CUDA(cudaMemcpyAsync(p->h_ctr + C_P, p->d_ctr + C_P, 8, cudaMemcpyDeviceToHost, p->stream));
  if (with_delta)
    VATE_CUDA(cudaMemcpyAsync(p->h_ctr + C_DCNT, p->d_ctr + C_DCNT, 16, cudaMemcpyDeviceToHost,
                              p->stream));
  return VATE_OK;
}

// Blocks are reported as (-1, -1): the reference's MaintenanceReport(()) for
// DR / TS (pools.py:349, :401).
int cmp_advance_async(vate_pool* p) {
  p->adv_blocks[0] = p->adv_blocks[1] = -1;
  VATE_CUDA(cudaMemsetAsync(p->d_ctr + C_CLEARED, 0, 8, p->stream));
  if (p->kind == VATE_DR) {
    p->adv_maint = p->L.size;
    int rc = with_cmp_cell(p, [&](auto tag) -> int {
      using T = decltype(tag);
      VATE_LAUNCH(p, VATE_K_SWEEP, grid_for(p->L.size / (16 / sizeof(T)) + 1, 256, 148u * 16u), 256,
                  0, k_dr_slide<T>, (T*)p->cells, p->L.size, (uint32_t)p->k, p->d_ctr + C_CLEARED);
      return VATE_OK;
    });
    if (rc) return rc;
  } else {
    p->adv_maint = 0;
    p->ts_now += 1;  // TsPool.advance_slice (pools.py:399-401)
  }
  VATE_CUDA(cudaMemcpyAsync(p->h_ctr + C_CLEARED, p->d_ctr + C_CLEARED, 8, cudaMemcpyDeviceToHost,
                            p->stream));
  VATE_CUDA(cudaEventRecord(p->ev_adv, p->stream));
  p->adv_pending = true;
  return VATE_OK;
}

int cmp_inactive_mask(vate_pool* p, const uint64_t* d_idx, uint64_t n, int k_prime,
                      uint8_t* out_dev) {
  const CmpPred P{p->kind, (uint32_t)k_prime, p->ts_now};
  return with_cmp_cell(p, [&](auto tag) -> int {
    using T = decltype(tag);
    VATE_LAUNCH(p, VATE_K_OTHER, grid_for(n, kThreads), kThreads, 0, k_cmp_mask<T>,
                (const T*)p->cells, p->L.size, d_idx, n, P, out_dev, p->d_ctr + C_ERR);
    return VATE_OK;
  });
}

template <typename F>
static int with_any_cell(vate_pool* p, F f) {
  if (p->kind == VATE_TS) return f(uint64_t{});
  if (p->cell_bytes == 1) return f(uint8_t{});
  if (p->cell_bytes == 2) return f(uint16_t{});
  return f(uint32_t{});
}

static unsigned long long width_mask(const vate_pool* p) {
  return p->width >= 64 ? ~0ull : ((1ull << p->width) - 1);
}

}  // namespace vate

using namespace vate;

extern "C" {

int vate_put_cells(vate_pool* p, const uint64_t* idx, const uint64_t* values, uint64_t n,
                   int where) {
  int rc = enter(p);
  if (rc || n == 0) return rc;
  if (where == VATE_HOST) {
    for (uint64_t i = 0; i < n; ++i)
      if (idx[i] >= p->L.size)
        return set_error(VATE_EVALUE, "cell index " + std::to_string(idx[i]) + " outside [0, " +
                                          std::to_string(p->L.size) + ")");
  }
  const void *d_idx, *d_val;
  rc = stage_in(p, p->in_a, idx, n * 8, where, &d_idx);
  if (rc) return rc;
  rc = stage_in(p, p->in_b, values, n * 8, where, &d_val);
  if (rc) return rc;
  rc = flush_pending(p);  // an older mark must not overwrite the value
  if (rc) return rc;
  rc = with_any_cell(p, [&](auto tag) -> int {
    using T = decltype(tag);
    VATE_LAUNCH(p, VATE_K_OTHER, grid_for(n, kThreads), kThreads, 0, k_put64<T>, (T*)p->cells,
                p->L.size, (const uint64_t*)d_idx, (const unsigned long long*)d_val, n,
                width_mask(p), p->d_ctr + C_ERR);
    return VATE_OK;
  });
  if (rc) return rc;
  rc = sync_small(p);
  if (rc) return rc;
  return bp_rebuild(p);  // bit-plane mode: the new values' history
}

int vate_fill_cells(vate_pool* p, uint64_t value) {
  int rc = enter(p);
  if (rc) return rc;
  if (p->width < 64 && (value >> p->width))  // PackedArray.fill (bitpack.py:57-60)
    return set_error(VATE_EVALUE, "value " + std::to_string(value) + " exceeds " +
                                      std::to_string(p->width) + " bits");
  if (p->pend_dirty && !p->bp) {  // every cell is overwritten: earlier marks are void
    VATE_CUDA(cudaMemsetAsync(p->pend.ptr, 0, p->pend.bytes, p->stream));
    p->pend_dirty = false;
  }
  rc = bp_wait_aux(p);
  if (rc) return rc;
  const uint64_t S = p->L.size;
  rc = with_any_cell(p, [&](auto tag) -> int {
    using T = decltype(tag);
    VATE_LAUNCH(p, VATE_K_OTHER, grid_for(S, kThreads), kThreads, 0, k_cmp_fill<T>, (T*)p->cells,
                S, (T)value);
    return VATE_OK;
  });
  if (rc) return rc;
  rc = sync_small(p);
  if (rc) return rc;
  return bp_rebuild(p);
}

int vate_get_cells64(vate_pool* p, const uint64_t* idx, uint64_t n, uint64_t* out, int where) {
  int rc = enter(p);
  if (rc || n == 0) return rc;
  const void* d_idx;
  rc = stage_in(p, p->in_a, idx, n * 8, where, &d_idx);
  if (rc) return rc;
  rc = p->out_buf.ensure(n * 8);
  if (rc) return rc;
  rc = flush_pending(p);
  if (rc) return rc;
  auto launch = [&](auto tag) -> int {
    using T = decltype(tag);
    VATE_LAUNCH(p, VATE_K_OTHER, grid_for(n, kThreads), kThreads, 0, k_get64<T>, (const T*)p->cells,
                p->L.size, (const uint64_t*)d_idx, n, p->out_buf.as<unsigned long long>(),
                p->d_ctr + C_ERR);
    return VATE_OK;
  };
  if (p->kind == VATE_TS) rc = launch(uint64_t{});
  else if (p->cell_bytes == 1) rc = launch(uint8_t{});
  else if (p->cell_bytes == 2) rc = launch(uint16_t{});
  else rc = launch(uint32_t{});
  if (rc) return rc;
  VATE_CUDA(cudaMemcpyAsync(p->h_ctr + C_ERR, p->d_ctr + C_ERR, 8, cudaMemcpyDeviceToHost, p->stream));
  VATE_CUDA(cudaMemsetAsync(p->d_ctr + C_ERR, 0, 8, p->stream));
  VATE_CUDA(cudaMemcpyAsync(out, p->out_buf.ptr, n * 8, cudaMemcpyDeviceToHost, p->stream));
  return sync_small(p);
}

int vate_pool_kind(const vate_pool* p, int* kind, uint64_t* slice_index) {
  if (!p) return set_error(VATE_EVALUE, "null pool handle");
  if (kind) *kind = p->kind;
  if (slice_index) *slice_index = p->ts_now;
  return VATE_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Speed-of-light probe for the scan's memory pattern (bench only): per
// "packet", one random 32-byte sector load from a table of table_bytes and one
// random 1-byte store into a buffer of cell_bytes, addresses from a counter
// hash (no input stream, no dependency between them).  Both buffers sized as
// the scan's registry and pool, so this is the L2 (or HBM) random-access
// ceiling the scan kernel is measured against.
// ---------------------------------------------------------------------------
namespace vate {
__global__ void __launch_bounds__(256) k_sol_scatter(const uint4* __restrict__ table,
                                                     uint64_t table_mask,
                                                     uint8_t* __restrict__ cells,
                                                     uint64_t cell_mask, uint64_t n,
                                                     unsigned long long* sink) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t h = mix64(i * kPhi + 12345);
    cells[h & cell_mask] = (uint8_t)i;
    const uint4 v = table[(h >> 32) & table_mask];
    acc += v.x ^ v.w;
  }
  if (acc == 0x9E3779B97F4A7C15ull) *sink = acc;  // keeps the loads alive
}
}  // namespace vate

extern "C" int vate_bench_sol_scatter(vate_pool* p, uint64_t n, uint64_t table_bytes,
                                      int reps, double* ms_per_rep) {
  int rc = enter(p);
  if (rc) return rc;
  const uint64_t cell_bytes = p->L.size * (uint64_t)p->cell_bytes;
  DevBuf table;
  rc = table.ensure(table_bytes);
  if (rc) return rc;
  VATE_CUDA(cudaMemsetAsync(table.ptr, 0, table_bytes, p->stream));
  cudaEvent_t a, b;
  VATE_CUDA(cudaEventCreate(&a));
  VATE_CUDA(cudaEventCreate(&b));
  const uint32_t grid = grid_for(n, 256, 148u * 64u);
  uint64_t tmask = 1;
  while (tmask * 2 * 16 <= table_bytes) tmask *= 2;
  VATE_LAUNCH(p, VATE_K_OTHER, grid, 256, 0, k_sol_scatter, table.as<const uint4>(), tmask - 1,
              (uint8_t*)p->cells, cell_bytes - 1, n, p->d_ctr + C_TRACE);  // warm-up
  VATE_CUDA(cudaEventRecord(a, p->stream));
  for (int r = 0; r < reps; ++r)
    VATE_LAUNCH(p, VATE_K_OTHER, grid, 256, 0, k_sol_scatter, table.as<const uint4>(), tmask - 1,
                (uint8_t*)p->cells, cell_bytes - 1, n, p->d_ctr + C_TRACE);
  VATE_CUDA(cudaEventRecord(b, p->stream));
  VATE_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  VATE_CUDA(cudaEventElapsedTime(&ms, a, b));
  *ms_per_rep = ms / reps;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  table.release();
  return VATE_OK;
}
