// N4 / N5 / N7: SM-driven peer copy kernels.
//
//   kb_copy_pages   KV exchange and dissolve-time consolidation: the moves
//                   are the device image of plan_exchange's tasks
//                   (pkg/src/dropsim/exchange.py:146-205) executed at
//                   engine.py:690-726 / 1211-1239.  Page addresses come from
//                   the two pools' block tables ON DEVICE; the host never
//                   sees page ids.
//   kb_copy_slabs   parameter restore / merge-time fetch: the device image of
//                   plan_restore_transfers (exchange.py:208-249) used at
//                   engine.py:762-783 and 1127-1141.
//   kb_copy_bytes   activation hand-off between pipeline stages
//                   (engine.py:428-448).
// Source and destination may live on different GPUs: pools map every slab
// with cuMemSetAccess for all peers, so a plain ld.global/st.global on the
// peer VA travels over NVLink.  All kernels move 16-byte vectors with 8
// loads in flight per thread and a grid of 148 x k blocks.
#include <cstring>

#include "kb_common.cuh"

namespace kb {

constexpr int kThreads = 256;
constexpr int kUnroll = 8;
constexpr int64_t kPiece = 32768;  // bytes of one page handled by one block pass

// Grid of the bulk copies.  One CTA per 32 KiB piece (a short-lived CTA:
// one 8-deep load / store round per thread), not a persistent grid: a
// burst then never holds the SMs for its whole duration, so work on a
// higher-priority stream -- the pipeline's activation hand-off, the
// reference's _PRIO (exchange.py:27-28) -- gets the next free CTA slots
// within microseconds instead of waiting for a multi-GB burst to drain.
// KB_COPY_PERSISTENT=1 builds the r1 grid (148 x 8 CTAs striding over the
// pieces) for A/B runs.
#ifndef KB_COPY_PERSISTENT
#define KB_COPY_PERSISTENT 0
#endif
inline int copy_grid(int64_t pieces) {
  return KB_COPY_PERSISTENT ? grid_for(pieces, 1, 148 * 8) : grid_for(pieces, 1, 1 << 30);
}

__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(int4* p, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// Copy `nvec` int4 from s to d with the whole block, kUnroll loads in flight.
__device__ __forceinline__ void block_copy(int4* __restrict__ d, const int4* __restrict__ s,
                                           int64_t nvec) {
  for (int64_t v0 = threadIdx.x; v0 < nvec; v0 += (int64_t)kThreads * kUnroll) {
    int4 r[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      int64_t v = v0 + (int64_t)u * kThreads;
      if (v < nvec) r[u] = ld_stream(s + v);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      int64_t v = v0 + (int64_t)u * kThreads;
      if (v < nvec) st_stream(d + v, r[u]);
    }
  }
}

struct PoolView {
  const int32_t* bt;
  uint8_t* kv;
  int L;
  int maxp;
};

// Moves travel by value in kernel parameter space (no staging copy, no sync).
constexpr int kMoveBatch = 256;
struct MoveBatch {
  kb_move mv[kMoveBatch];
  int64_t cum[kMoveBatch];
};

__global__ void __launch_bounds__(kThreads)
copy_pages_kernel(PoolView dst, PoolView src, const __grid_constant__ MoveBatch batch, int n,
                  int64_t total_pages, int64_t page_bytes, int64_t pieces) {
  const kb_move* moves = batch.mv;
  const int64_t* cum = batch.cum;
  const int64_t piece_bytes = page_bytes / pieces;
  for (int64_t job = blockIdx.x; job < total_pages * pieces; job += gridDim.x) {
    const int64_t pg = job / pieces, pc = job % pieces;
    int lo = 0, hi = n - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (cum[mid] <= pg) lo = mid; else hi = mid - 1;
    }
    const kb_move mv = moves[lo];
    const int64_t flat = mv.flat_lo + (pg - cum[lo]);
    const int layer = mv.layer_lo + (int)(flat / mv.npages);
    const int idx = (int)(flat % mv.npages);
    const int32_t sp = src.bt[((int64_t)mv.src_slot * src.L + layer) * src.maxp + idx];
    const int32_t dp = dst.bt[((int64_t)mv.dst_slot * dst.L + layer) * dst.maxp + idx];
    const int4* s = reinterpret_cast<const int4*>(src.kv + (int64_t)sp * page_bytes + pc * piece_bytes);
    int4* d = reinterpret_cast<int4*>(dst.kv + (int64_t)dp * page_bytes + pc * piece_bytes);
    block_copy(d, s, piece_bytes / 16);
  }
}

// Pages of one (slot, layer range) <-> a flat host buffer (pinned, mapped
// into the device VA): flattened page f = (layer - lo) * npages + i sits at
// host + f * page_bytes.  The SMs drive the PCIe / C2C transfer with 16-byte
// loads and stores, like the peer copies.
__global__ void __launch_bounds__(kThreads)
copy_pages_host_kernel(PoolView pool, uint8_t* __restrict__ host, kb_move mv, int64_t total_pages,
                       int64_t page_bytes, int64_t pieces, int to_host) {
  const int64_t piece_bytes = page_bytes / pieces;
  for (int64_t job = blockIdx.x; job < total_pages * pieces; job += gridDim.x) {
    const int64_t f = mv.flat_lo + job / pieces, pc = job % pieces;
    const int layer = mv.layer_lo + (int)(f / mv.npages);
    const int idx = (int)(f % mv.npages);
    const int32_t pg = pool.bt[((int64_t)mv.src_slot * pool.L + layer) * pool.maxp + idx];
    uint8_t* dev = pool.kv + (int64_t)pg * page_bytes + pc * piece_bytes;
    uint8_t* hst = host + f * page_bytes + pc * piece_bytes;
    if (to_host)
      block_copy(reinterpret_cast<int4*>(hst), reinterpret_cast<const int4*>(dev), piece_bytes / 16);
    else
      block_copy(reinterpret_cast<int4*>(dev), reinterpret_cast<const int4*>(hst), piece_bytes / 16);
  }
}

__global__ void __launch_bounds__(kThreads)
copy_flat_kernel(int4* __restrict__ d, const int4* __restrict__ s, int64_t nvec) {
  // grid-stride over 32 KiB pieces
  const int64_t per = kPiece / 16;
  const int64_t pieces = (nvec + per - 1) / per;
  for (int64_t pc = blockIdx.x; pc < pieces; pc += gridDim.x) {
    const int64_t beg = pc * per;
    const int64_t cnt = nvec - beg < per ? nvec - beg : per;
    block_copy(d + beg, s + beg, cnt);
  }
}

__global__ void copy_tail_kernel(uint8_t* __restrict__ d, const uint8_t* __restrict__ s, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}

static int launch_flat(uint64_t dst, uint64_t src, int64_t nbytes, cudaStream_t st) {
  if (nbytes <= 0) return KB_OK;
  const bool aligned = ((dst | src) & 15) == 0;
  int64_t body = aligned ? (nbytes & ~(int64_t)15) : 0;
  if (body) {
    int64_t pieces = ceil_div(body / 16, kPiece / 16);
    int grid = copy_grid(pieces);
    copy_flat_kernel<<<grid, kThreads, 0, st>>>(reinterpret_cast<int4*>(dst),
                                                reinterpret_cast<const int4*>(src), body / 16);
    KB_LAUNCH_CHECK();
  }
  if (nbytes > body) {
    int64_t rest = nbytes - body;
    copy_tail_kernel<<<grid_for(rest, 256, 1024), 256, 0, st>>>(
        reinterpret_cast<uint8_t*>(dst + body), reinterpret_cast<const uint8_t*>(src + body), rest);
    KB_LAUNCH_CHECK();
  }
  return KB_OK;
}

}  // namespace kb

using namespace kb;

extern "C" int kb_copy_pages(kb_pool* dst, kb_pool* src, const kb_move* moves, int32_t n,
                             uintptr_t stream) {
  if (!dst || !src) return fail(KB_EINVAL, "null pool");
  if (dst->view) return fail(KB_EINVAL, "copy destination must be a pool this process owns (pull from views)");
  if (n <= 0) return KB_OK;
  if (dst->m.page_bytes != src->m.page_bytes || dst->m.num_layers != src->m.num_layers)
    return fail(KB_EINVAL, "pools disagree on page geometry");
  const int L = src->m.num_layers;
  std::vector<int64_t> cum(n);
  int64_t total = 0;
  for (int i = 0; i < n; ++i) {
    const kb_move& mv = moves[i];
    if (mv.layer_lo < 0 || mv.layer_hi > L || mv.layer_hi <= mv.layer_lo || mv.npages < 0 ||
        mv.flat_lo < 0 || mv.flat_hi < mv.flat_lo ||
        mv.flat_hi > (mv.layer_hi - mv.layer_lo) * mv.npages || mv.src_slot < 0 ||
        mv.src_slot >= src->max_slots || mv.dst_slot < 0 || mv.dst_slot >= dst->max_slots)
      return fail(KB_EINVAL, "bad move " + std::to_string(i));
    for (int l = mv.layer_lo; l < mv.layer_hi; ++l) {
      if (src->h_np[(int64_t)mv.src_slot * L + l] < mv.npages ||
          dst->h_np[(int64_t)mv.dst_slot * L + l] < mv.npages)
        return fail(KB_EINVAL, "move " + std::to_string(i) + " names pages that are not allocated");
    }
    cum[i] = total;
    total += mv.flat_hi - mv.flat_lo;
  }
  if (total == 0) return KB_OK;
  KB_RT(cudaSetDevice(src->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t pieces = src->m.page_bytes > kPiece ? src->m.page_bytes / kPiece : 1;
  PoolView dv{dst->d_bt, reinterpret_cast<uint8_t*>(dst->kva), L, dst->maxp};
  PoolView sv{src->d_bt, reinterpret_cast<uint8_t*>(src->kva), L, src->maxp};
  int rc;
  if ((rc = pool_enter(dst, st)) || (rc = pool_enter(src, st))) return rc;
  MoveBatch batch;
  for (int b0 = 0; b0 < n; b0 += kMoveBatch) {
    const int nb = std::min(kMoveBatch, n - b0);
    int64_t sub = 0;
    for (int i = 0; i < nb; ++i) {
      batch.mv[i] = moves[b0 + i];
      batch.cum[i] = sub;
      sub += moves[b0 + i].flat_hi - moves[b0 + i].flat_lo;
    }
    if (sub == 0) continue;
    int grid = copy_grid(sub * pieces);
    copy_pages_kernel<<<grid, kThreads, 0, st>>>(dv, sv, batch, nb, sub, src->m.page_bytes,
                                                 pieces);
    KB_LAUNCH_CHECK();
  }
  (void)cum;
  if ((rc = pool_leave(dst, st)) || (rc = pool_leave(src, st))) return rc;
  return KB_OK;
}

extern "C" int kb_copy_slabs(kb_pool* dst, kb_pool* src, int32_t lo, int32_t hi, int64_t byte_lo,
                             int64_t byte_hi, uintptr_t stream) {
  if (!dst || !src) return fail(KB_EINVAL, "null pool");
  if (dst->view) return fail(KB_EINVAL, "copy destination must be a pool this process owns (pull from views)");
  if (dst->m.slab_bytes != src->m.slab_bytes) return fail(KB_EINVAL, "pools disagree on slab size");
  const int64_t slab = src->m.slab_bytes;
  if (hi <= lo || byte_lo < 0 || byte_hi < byte_lo || byte_hi > (int64_t)(hi - lo) * slab)
    return fail(KB_EINVAL, "bad slab byte range");
  for (int l = lo; l < hi; ++l) {
    if (src->layer_state[l] != kLayerHeld)
      return fail(KB_ESTATE, "source does not hold layer " + std::to_string(l));
    if (dst->layer_state[l] == kLayerDropped)
      return fail(KB_ESTATE, "destination layer " + std::to_string(l) + " is not reserved for a pull");
  }
  KB_RT(cudaSetDevice(dst->device));
  uint64_t d = (uint64_t)dst->wva + (uint64_t)lo * slab + byte_lo;
  uint64_t s = (uint64_t)src->wva + (uint64_t)lo * slab + byte_lo;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if ((rc = pool_enter(dst, st)) || (rc = pool_enter(src, st))) return rc;
  if ((rc = launch_flat(d, s, byte_hi - byte_lo, st))) return rc;
  if ((rc = pool_leave(dst, st)) || (rc = pool_leave(src, st))) return rc;
  return KB_OK;
}

extern "C" int kb_copy_slabs_from_host(kb_pool* dst, const void* host_src, int32_t lo, int32_t hi,
                                       int64_t byte_lo, int64_t byte_hi, uintptr_t stream) {
  if (!dst || !host_src) return fail(KB_EINVAL, "null argument");
  if (dst->view) return refuse_view();
  const int64_t slab = dst->m.slab_bytes;
  if (hi <= lo || byte_lo < 0 || byte_hi < byte_lo || byte_hi > (int64_t)(hi - lo) * slab)
    return fail(KB_EINVAL, "bad slab byte range");
  for (int l = lo; l < hi; ++l)
    if (dst->layer_state[l] == kLayerDropped)
      return fail(KB_ESTATE, "destination layer " + std::to_string(l) + " is not reserved for a pull");
  KB_RT(cudaSetDevice(dst->device));
  cudaStream_t st = (cudaStream_t)stream;
  int rc = pool_enter(dst, st);
  if (rc) return rc;
  KB_RT(cudaMemcpyAsync(reinterpret_cast<void*>(dst->wva + (uint64_t)lo * slab + byte_lo),
                        static_cast<const char*>(host_src) + byte_lo, byte_hi - byte_lo,
                        cudaMemcpyHostToDevice, st));
  return pool_leave(dst, st);
}

extern "C" int kb_copy_bytes(uint64_t dst, uint64_t src, int64_t nbytes, uintptr_t stream) {
  if (nbytes < 0) return fail(KB_EINVAL, "negative size");
  return launch_flat(dst, src, nbytes, (cudaStream_t)stream);
}

extern "C" int kb_copy_pages_host(kb_pool* p, const kb_move* mv, void* host, int32_t to_host,
                                  uintptr_t stream) {
  if (!p || !mv || !host) return fail(KB_EINVAL, "null argument");
  if (p->view) return refuse_view();
  const int L = p->m.num_layers;
  if (mv->layer_lo < 0 || mv->layer_hi > L || mv->layer_hi <= mv->layer_lo || mv->npages < 0 ||
      mv->flat_lo < 0 || mv->flat_hi < mv->flat_lo ||
      mv->flat_hi > (mv->layer_hi - mv->layer_lo) * mv->npages || mv->src_slot < 0 ||
      mv->src_slot >= p->max_slots)
    return fail(KB_EINVAL, "bad host move");
  for (int l = mv->layer_lo; l < mv->layer_hi; ++l)
    if (p->h_np[(int64_t)mv->src_slot * L + l] < mv->npages)
      return fail(KB_EINVAL, "host move names pages that are not allocated");
  const int64_t total = mv->flat_hi - mv->flat_lo;
  if (total == 0) return KB_OK;
  KB_RT(cudaSetDevice(p->device));
  void* dhost = nullptr;
  // pinned host memory is mapped into the device VA (UVA): same address
  KB_RT(cudaHostGetDevicePointer(&dhost, host, 0));
  if ((reinterpret_cast<uintptr_t>(dhost) & 15) != 0) return fail(KB_EINVAL, "host buffer must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t pieces = p->m.page_bytes > kPiece ? p->m.page_bytes / kPiece : 1;
  PoolView pv{p->d_bt, reinterpret_cast<uint8_t*>(p->kva), L, p->maxp};
  int rc = pool_enter(p, st);
  if (rc) return rc;
  // PCIe-bound: 16 CTAs keep ~0.5 MB in flight -- enough for the host link --
  // and leave the other SMs to the compute the swap overlaps with
  copy_pages_host_kernel<<<grid_for(total * pieces, 1, 16), kThreads, 0, st>>>(
      pv, static_cast<uint8_t*>(dhost), *mv, total, p->m.page_bytes, pieces, to_host);
  KB_LAUNCH_CHECK();
  return pool_leave(p, st);
}

// ------------------------------------------------ cross-process activation buffers
// The stage s -> s+1 hand-off of a pipeline group whose members live in
// different processes (engine.py:428-448): the receiving stage owns a
// device buffer, the sending stage maps it through CUDA IPC and writes the
// activation rows into it with the copy kernel above (NVLink stores).

extern "C" int kb_device_alloc(int32_t device, int64_t nbytes, uint64_t* ptr) {
  if (!ptr || nbytes <= 0) return fail(KB_EINVAL, "bad allocation request");
  KB_RT(cudaSetDevice(device));
  void* p = nullptr;
  KB_RT(cudaMalloc(&p, (size_t)nbytes));
  *ptr = reinterpret_cast<uint64_t>(p);
  return KB_OK;
}

extern "C" int kb_device_free(uint64_t ptr) {
  if (ptr) KB_RT(cudaFree(reinterpret_cast<void*>(ptr)));
  return KB_OK;
}

extern "C" int kb_ipc_mem_export(uint64_t ptr, uint8_t* handle) {
  if (!ptr || !handle) return fail(KB_EINVAL, "null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) <= 64, "ipc handle size");
  cudaIpcMemHandle_t h;
  KB_RT(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(ptr)));
  std::memset(handle, 0, 64);
  std::memcpy(handle, &h, sizeof(h));
  return KB_OK;
}

extern "C" int kb_ipc_mem_import(int32_t device, const uint8_t* handle, uint64_t* ptr) {
  if (!handle || !ptr) return fail(KB_EINVAL, "null argument");
  KB_RT(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  KB_RT(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *ptr = reinterpret_cast<uint64_t>(p);
  return KB_OK;
}

extern "C" int kb_ipc_mem_close(uint64_t ptr) {
  if (ptr) KB_RT(cudaIpcCloseMemHandle(reinterpret_cast<void*>(ptr)));
  return KB_OK;
}
