// N1 + N2 + N3: VMM slab pool, device page allocator / block tables, and the
// restore-time page compaction.
//
// Reference semantics followed (pkg/src/dropsim/):
//   build_instance   memory.py:132-144   -> kb_pool_create
//   drop_layers      memory.py:147-172   -> kb_drop_layers
//   restore_layers   memory.py:175-197   -> kb_restore_begin
//   complete_restore memory.py:200-212   -> kb_restore_complete
//   KVAllocator      memory.py:70-129    -> kb_pages_grow / kb_pages_release
//
// B200 design: every layer slab is ONE physical VMM allocation mapped at TWO
// virtual addresses from pool creation on -- under the weight VA (layer l at
// l * slab) and as a fixed page range of the KV VA (after the head segment).
// Dropping a layer is therefore no driver call at all: a kernel flips the
// slab's pages from "reserved" to "free" in the page bitmap, and the next
// block-table growth can hand them out.  Restoring vacates the slab's page
// range (device compaction: live pages move to the lowest free pages outside
// it, block tables rewritten through the owner map) and marks it reserved
// again, so the parameter pull can land under the weight VA.  The paper's
// "5 ms per remap" (map_latency_us, config.py:40) becomes a
// few microseconds of kernel time.
//
// The reference is token-granular and position-free; pages, block tables
// and compaction are the device layer underneath.  Every
// allocation choice is deterministic (lowest free page id first) so the CPU
// restatement in oracle/kvpool.py reproduces block tables bit for bit.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <mutex>
#include <set>
#include <tuple>

#include "kb_common.cuh"

namespace kb {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

Driver& drv() {
  static Driver d;
  return d;
}

int ensure_driver() {
  Driver& d = drv();
  if (d.ready) return KB_OK;
  KB_RT(cudaFree(nullptr));
  auto get = [](const char* name, void** fn) -> bool {
    cudaDriverEntryPointQueryResult q;
    return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
           q == cudaDriverEntryPointSuccess && *fn != nullptr;
  };
  bool ok = get("cuMemCreate", (void**)&d.MemCreate) && get("cuMemRelease", (void**)&d.MemRelease) &&
            get("cuMemMap", (void**)&d.MemMap) && get("cuMemUnmap", (void**)&d.MemUnmap) &&
            get("cuMemSetAccess", (void**)&d.MemSetAccess) &&
            get("cuMemAddressReserve", (void**)&d.MemAddressReserve) &&
            get("cuMemAddressFree", (void**)&d.MemAddressFree) &&
            get("cuMemGetAllocationGranularity", (void**)&d.MemGetAllocationGranularity) &&
            get("cuTensorMapEncodeTiled", (void**)&d.TensorMapEncodeTiled) &&
            get("cuGetErrorString", (void**)&d.GetErrorString) &&
            get("cuMemExportToShareableHandle", (void**)&d.MemExport) &&
            get("cuMemImportFromShareableHandle", (void**)&d.MemImport);
  if (!ok) return fail(KB_ECUDA, "cannot resolve CUDA driver entry points");
  d.ready = true;
  return KB_OK;
}

int refuse_view() {
  return fail(KB_EINVAL, "pool is a read-only peer view: its owner process performs this operation");
}

int ensure_smem_attr(const void* fn, int bytes, int device) {
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, int>> done;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(fn, device, bytes);
  if (done.count(key)) return KB_OK;
  KB_RT(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.insert(key);
  return KB_OK;
}

int ensure_scratch(kb_pool* p, int64_t bytes) {
  if (p->scratch_bytes >= bytes) return KB_OK;
  if (p->d_scratch) cudaFree(p->d_scratch);
  p->d_scratch = nullptr;
  int64_t want = round_up(bytes < (1 << 20) ? (1 << 20) : bytes * 2, 256);
  KB_RT(cudaMalloc(&p->d_scratch, want));
  p->scratch_bytes = want;
  return KB_OK;
}

// Inside a CUDA graph capture the graph's own edges order the work (events
// recorded outside the capture cannot be waited on): no-ops there.
static bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}

int pool_enter(kb_pool* p, cudaStream_t st) {
  if (capturing(st)) return KB_OK;
  if (p->meta_set) KB_RT(cudaStreamWaitEvent(st, p->meta_ev, 0));
  return KB_OK;
}

int pool_leave(kb_pool* p, cudaStream_t st) {
  if (capturing(st)) return KB_OK;
  for (auto& se : p->op_ev)
    if (se.first == st) {
      KB_RT(cudaEventRecord(se.second, st));
      return KB_OK;
    }
  if (p->op_ev.size() >= 32) {
    // many short-lived streams: fold them into this one ON THE DEVICE -- st
    // waits for every other stream's last pool op, so the event recorded
    // below stands for all of them (no host synchronization)
    for (auto& se : p->op_ev) {
      KB_RT(cudaStreamWaitEvent(st, se.second, 0));
      cudaEventDestroy(se.second);  // released once the wait has resolved
    }
    p->op_ev.clear();
  }
  cudaEvent_t ev;
  KB_RT(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  p->op_ev.emplace_back(st, ev);
  KB_RT(cudaEventRecord(ev, st));
  return KB_OK;
}

int pool_meta_begin(kb_pool* p, cudaStream_t st, bool wait_all_streams) {
  if (capturing(st)) return KB_OK;
  if (wait_all_streams)
    for (auto& se : p->op_ev)
      if (se.first != st) KB_RT(cudaStreamWaitEvent(st, se.second, 0));
  return pool_enter(p, st);
}

int pool_meta_end(kb_pool* p, cudaStream_t st) {
  if (!capturing(st)) {
    KB_RT(cudaEventRecord(p->meta_ev, st));
    p->meta_set = true;
  }
  return pool_leave(p, st);
}

// ---------------------------------------------------------------- kernels

constexpr int kScanThreads = 1024;
constexpr int32_t kReserved = -2;  // owner[] of a slab page holding live weights

// Block-wide exclusive scan of one int per thread (1024 threads).
__device__ __forceinline__ int block_exclusive_scan(int v, int* total, int* warp_sums) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = warp_sums[lane];
    int s = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    warp_sums[lane] = s - w;
    if (lane == 31) *total = s;
  }
  __syncthreads();
  int r = warp_sums[warp] + x - v;
  __syncthreads();
  return r;
}

// Enumerate, in ascending order, the set (want_live) or clear bits of the
// pages in [lo, hi) and hand the k-th one to emit(base_k + k, page) for
// k < limit.  Tiles of kScanThreads * kWordsPerThread words; stops early
// once `limit` pages were found.  *found_out = min(found, limit).
template <int kWordsPerThread, typename Emit>
__device__ void scan_pages(const uint32_t* __restrict__ bitmap, int64_t lo, int64_t hi,
                           bool want_live, int64_t limit, Emit emit, int64_t* found_out) {
  __shared__ int warp_sums[32];
  __shared__ int tile_total;
  int64_t found = 0;
  const int64_t w_lo = lo >> 5, w_hi = (hi + 31) >> 5;
  const int64_t tile_words = (int64_t)kScanThreads * kWordsPerThread;
  for (int64_t t0 = w_lo; t0 < w_hi && found < limit; t0 += tile_words) {
    uint32_t bits[kWordsPerThread];
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < kWordsPerThread; ++j) {
      int64_t w = t0 + (int64_t)threadIdx.x * kWordsPerThread + j;
      uint32_t b = 0;
      if (w < w_hi) {
        uint32_t raw = bitmap[w];
        b = want_live ? raw : ~raw;
        int64_t base = w << 5;
        if (base < lo) b &= ~0u << (lo - base);
        if (base + 32 > hi) {
          int64_t keep = hi - base;
          b &= keep <= 0 ? 0u : (keep >= 32 ? ~0u : ((1u << keep) - 1u));
        }
      }
      bits[j] = b;
      cnt += __popc(b);
    }
    int off = block_exclusive_scan(cnt, &tile_total, warp_sums);
    int64_t k = found + off;
#pragma unroll
    for (int j = 0; j < kWordsPerThread; ++j) {
      uint32_t b = bits[j];
      int64_t base = (t0 + (int64_t)threadIdx.x * kWordsPerThread + j) << 5;
      while (b && k < limit) {
        int bit = __ffs(b) - 1;
        b &= b - 1;
        emit(k, base + bit);
        ++k;
      }
    }
    found += tile_total;
    __syncthreads();
  }
  if (found_out) *found_out = found < limit ? found : limit;
}

// Grow: a batch of requests passed by value (kernel parameter space, no
// host->device copy) with exclusive prefix `cum` (pages per request); the
// k-th lowest free page goes to flattened slot k (reserved slab pages are
// set in the bitmap, so they are never free).
constexpr int kGrowBatch = 256;
struct GrowBatch {
  kb_grow r[kGrowBatch];
  int64_t cum[kGrowBatch];
};

__global__ void __launch_bounds__(kScanThreads)
grow_kernel(uint32_t* __restrict__ bitmap, int32_t* __restrict__ owner, int32_t* __restrict__ bt,
            int32_t* __restrict__ np, const __grid_constant__ GrowBatch batch, int n,
            int64_t total, int64_t max_pages, int L, int maxp) {
  constexpr int kW = 4;                       // bitmap words per thread per tile
  constexpr int kTileWords = kScanThreads * kW;
  __shared__ int warp_sums[32];
  __shared__ int tile_total;
  __shared__ int s_pref[kTileWords];          // free pages before each word (tile-local)
  __shared__ uint32_t s_bits[kTileWords];     // free bits of each word
  __shared__ int64_t s_cum[kGrowBatch];
  for (int i = threadIdx.x; i < n; i += blockDim.x) s_cum[i] = batch.cum[i];
  const int64_t w_hi = (max_pages + 31) >> 5;
  int64_t found = 0;
  for (int64_t t0 = 0; t0 < w_hi && found < total; t0 += kTileWords) {
    uint32_t bits[kW];
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      const int64_t w = t0 + (int64_t)threadIdx.x * kW + j;
      uint32_t b = 0;
      if (w < w_hi) {
        b = ~bitmap[w];
        const int64_t keep = max_pages - (w << 5);
        if (keep < 32) b &= (1u << keep) - 1u;
      }
      bits[j] = b;
      cnt += __popc(b);
    }
    int off = block_exclusive_scan(cnt, &tile_total, warp_sums);
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      s_pref[threadIdx.x * kW + j] = off;
      s_bits[threadIdx.x * kW + j] = bits[j];
      off += __popc(bits[j]);
    }
    __syncthreads();
    const int take = (int)min((int64_t)tile_total, total - found);
    // balanced emission: the e-th free page of the tile goes to flattened
    // slot found + e; consecutive threads take consecutive slots, so the
    // block-table and owner writes coalesce
    for (int e = threadIdx.x; e < take; e += blockDim.x) {
      int lo = 0, hi = kTileWords - 1;  // last word with s_pref <= e
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_pref[mid] <= e) lo = mid; else hi = mid - 1;
      }
      const int64_t page = ((t0 + lo) << 5) + __fns(s_bits[lo], 0, e - s_pref[lo] + 1);
      const int64_t k = found + e;
      int a = 0, b = n - 1;  // last request with cum <= k
      while (a < b) {
        const int mid = (a + b + 1) >> 1;
        if (s_cum[mid] <= k) a = mid; else b = mid - 1;
      }
      const kb_grow r = batch.r[a];
      const int64_t rem = k - s_cum[a];
      const int layer = r.layer_lo + (int)(rem / r.add_pages);
      const int idx = np[(int64_t)r.slot * L + layer] + (int)(rem % r.add_pages);
      const int64_t cell = ((int64_t)r.slot * L + layer) * maxp + idx;
      bt[cell] = (int32_t)page;
      owner[page] = (int32_t)cell;
    }
    // mark the taken pages: the lowest (take - pref) free bits of each word
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      const int wl = threadIdx.x * kW + j;
      const int got = min(max(take - s_pref[wl], 0), __popc(bits[j]));
      if (got > 0) {
        const uint32_t upto = got == __popc(bits[j]) ? bits[j]
                              : bits[j] & ((1u << __fns(bits[j], 0, got + 1)) - 1u);
        bitmap[t0 + wl] |= upto;
      }
    }
    found += take;
    __syncthreads();
  }
  // page counts: every (request, layer) cell is distinct (host-checked)
  for (int c = threadIdx.x; c < n * L; c += blockDim.x) {
    const kb_grow r = batch.r[c / L];
    const int l = c % L;
    if (l >= r.layer_lo && l < r.layer_hi) np[(int64_t)r.slot * L + l] += r.add_pages;
  }
}

// Release all pages of (slot, layer) for layers in [lo, hi): one block per pair.
constexpr int kReleaseBatch = 1024;
struct SlotBatch {
  int32_t s[kReleaseBatch];
};

__global__ void release_kernel(uint32_t* __restrict__ bitmap, int32_t* __restrict__ owner,
                               int32_t* __restrict__ bt, int32_t* __restrict__ np,
                               const __grid_constant__ SlotBatch slots, int lo, int hi, int L,
                               int maxp) {
  const int span = hi - lo;
  const int slot = slots.s[blockIdx.x / span];
  const int layer = lo + blockIdx.x % span;
  int32_t* row = bt + ((int64_t)slot * L + layer) * maxp;
  const int cnt = np[(int64_t)slot * L + layer];
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    int32_t page = row[i];
    atomicAnd(&bitmap[page >> 5], ~(1u << (page & 31)));
    owner[page] = -1;
    row[i] = -1;
  }
  __syncthreads();
  if (threadIdx.x == 0) np[(int64_t)slot * L + layer] = 0;
}

// Mark a page range reserved for weights (set) or free for KV (clear).
__global__ void range_mark_kernel(uint32_t* __restrict__ bitmap, int32_t* __restrict__ owner,
                                  int64_t lo, int64_t hi, int set) {
  for (int64_t p = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < hi;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (set) {
      atomicOr(&bitmap[p >> 5], 1u << (p & 31));
      owner[p] = kReserved;
    } else {
      atomicAnd(&bitmap[p >> 5], ~(1u << (p & 31)));
      owner[p] = -1;
    }
  }
}

// Compaction plan for vacating [r_lo, r_hi): its live pages ascending ->
// src[]; the same number of lowest free pages outside the range -> dst[].
__global__ void __launch_bounds__(kScanThreads)
compact_plan_kernel(const uint32_t* __restrict__ bitmap, int64_t r_lo, int64_t r_hi,
                    int64_t max_pages, int32_t* __restrict__ src, int32_t* __restrict__ dst,
                    int64_t cap, int64_t* __restrict__ counts) {
  int64_t m = 0;
  scan_pages<4>(bitmap, r_lo, r_hi, true, cap,
                [&](int64_t k, int64_t page) { src[k] = (int32_t)page; }, &m);
  __syncthreads();
  int64_t f1 = 0, f2 = 0;
  scan_pages<4>(bitmap, 0, r_lo, false, m,
                [&](int64_t k, int64_t page) { dst[k] = (int32_t)page; }, &f1);
  __syncthreads();
  if (f1 < m) {
    scan_pages<4>(bitmap, r_hi, max_pages, false, m - f1,
                  [&](int64_t k, int64_t page) { dst[f1 + k] = (int32_t)page; }, &f2);
  }
  if (threadIdx.x == 0) {
    counts[0] = m;
    counts[1] = f1 + f2;
  }
}

// Move page contents src[i] -> dst[i] within one pool (HBM read+write).
constexpr int kPieceBytes = 32768;
constexpr int kCopyThreads = 256;

__global__ void __launch_bounds__(kCopyThreads)
compact_copy_kernel(uint8_t* __restrict__ kv, const int32_t* __restrict__ src,
                    const int32_t* __restrict__ dst, const int64_t* __restrict__ counts,
                    int64_t page_bytes) {
  const int64_t pieces = page_bytes / kPieceBytes > 0 ? page_bytes / kPieceBytes : 1;
  const int64_t piece_bytes = page_bytes / pieces;
  const int64_t m = counts[0];
  for (int64_t job = blockIdx.x; job < m * pieces; job += gridDim.x) {
    const int64_t i = job / pieces, pc = job % pieces;
    const int4* s = reinterpret_cast<const int4*>(kv + (int64_t)src[i] * page_bytes + pc * piece_bytes);
    int4* d = reinterpret_cast<int4*>(kv + (int64_t)dst[i] * page_bytes + pc * piece_bytes);
    const int64_t nvec = piece_bytes / 16;
    for (int64_t v0 = threadIdx.x; v0 < nvec; v0 += (int64_t)kCopyThreads * 8) {
      int4 r[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        int64_t v = v0 + (int64_t)u * kCopyThreads;
        if (v < nvec) r[u] = s[v];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        int64_t v = v0 + (int64_t)u * kCopyThreads;
        if (v < nvec) d[v] = r[u];
      }
    }
  }
}

// Rewrite block tables / owners / bitmap for the moved pages.
__global__ void compact_fixup_kernel(uint32_t* __restrict__ bitmap, int32_t* __restrict__ owner,
                                     int32_t* __restrict__ bt, const int32_t* __restrict__ src,
                                     const int32_t* __restrict__ dst,
                                     const int64_t* __restrict__ counts) {
  const int64_t m = counts[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = src[i], d = dst[i];
    const int32_t cell = owner[s];
    bt[cell] = d;
    owner[d] = cell;
    owner[s] = -1;
    atomicOr(&bitmap[d >> 5], 1u << (d & 31));
    atomicAnd(&bitmap[s >> 5], ~(1u << (s & 31)));
  }
}

// ---------------------------------------------------------------- VMM helpers

static int make_handle(int device, int64_t bytes, CUmemGenericAllocationHandle* out) {
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  KB_CU(drv().MemCreate(out, (size_t)bytes, &prop, 0));
  return KB_OK;
}

static int map_at(kb_pool* p, CUdeviceptr va, int64_t bytes, CUmemGenericAllocationHandle h) {
  KB_CU(drv().MemMap(va, (size_t)bytes, 0, h, 0));
  std::vector<CUmemAccessDesc> acc(p->access.size());
  for (size_t i = 0; i < p->access.size(); ++i) {
    acc[i].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc[i].location.id = p->access[i];
    acc[i].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  }
  KB_CU(drv().MemSetAccess(va, (size_t)bytes, acc.data(), acc.size()));
  return KB_OK;
}

static int set_device(int device) {
  KB_RT(cudaSetDevice(device));
  KB_RT(cudaFree(nullptr));  // materialise the primary context
  return ensure_driver();
}

static int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

static inline int64_t slab_pages(const kb_pool* p) { return p->m.slab_bytes / p->m.page_bytes; }
static inline int64_t slab_first_page(const kb_pool* p, int layer) {
  return p->head_pages + (int64_t)layer * slab_pages(p);
}

}  // namespace kb

using namespace kb;

// ------------------------------------------------------------------ C ABI

extern "C" const char* kb_last_error(void) { return g_err.c_str(); }
extern "C" int kb_version(void) { return 1; }

extern "C" int kb_init(int32_t device, const int32_t* peers, int32_t n_peers) {
  int rc = set_device(device);
  if (rc) return rc;
  for (int i = 0; i < n_peers; ++i) {
    if (peers[i] == device) continue;
    int can = 0;
    KB_RT(cudaDeviceCanAccessPeer(&can, device, peers[i]));
    if (!can) return fail(KB_EINVAL, "device " + std::to_string(device) +
                                         " cannot access peer " + std::to_string(peers[i]));
    cudaError_t e = cudaDeviceEnablePeerAccess(peers[i], 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
      return fail(KB_ECUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
    cudaGetLastError();
  }
  return KB_OK;
}

extern "C" int kb_vmm_granularity(int32_t device, int64_t* out_bytes) {
  int rc = set_device(device);
  if (rc) return rc;
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g = 0;
  KB_CU(drv().MemGetAllocationGranularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  *out_bytes = (int64_t)g;
  return KB_OK;
}

extern "C" int kb_pool_create(int32_t device, const kb_model_desc* model, int64_t hbm_bytes,
                              int32_t max_slots, int32_t max_pages_per_seq, int32_t slack_pages,
                              const int32_t* peers, int32_t n_peers, kb_pool** out) {
  *out = nullptr;
  const kb_model_desc m = *model;
  const int64_t param = (int64_t)m.num_layers * m.slab_bytes;
  if (m.num_layers < 1 || m.slab_bytes < 1 || m.page_bytes < 1 || m.block_tokens < 1)
    return fail(KB_EINVAL, "model byte sizes must be positive");
  if (m.page_bytes != (int64_t)m.block_tokens * 2 * m.n_kv_heads * m.head_dim * 2)
    return fail(KB_EINVAL, "page_bytes != block_tokens * 2 * n_kv_heads * head_dim * 2");
  if (hbm_bytes <= param)
    return fail(KB_EINVAL, "HBM " + std::to_string(hbm_bytes) + " cannot hold one parameter copy");
  int64_t gran = 0;
  int rc = kb_vmm_granularity(device, &gran);
  if (rc) return rc;
  if (m.slab_bytes % gran) return fail(KB_EINVAL, "slab_bytes must be a multiple of the VMM granularity");
  if (gran % m.page_bytes) return fail(KB_EINVAL, "page_bytes must divide the VMM granularity");
  if (max_slots < 1 || max_pages_per_seq < 1 || slack_pages < 0)
    return fail(KB_EINVAL, "bad slot / page limits");

  kb_pool* p = new kb_pool();
  p->device = device;
  p->m = m;
  p->hbm_bytes = hbm_bytes;
  p->gran = gran;
  p->access.push_back(device);
  for (int i = 0; i < n_peers; ++i)
    if (peers[i] != device) p->access.push_back(peers[i]);
  p->max_slots = max_slots;
  p->maxp = max_pages_per_seq;

  auto bail = [&](int code) {
    kb_pool_destroy(p);
    return code;
  };
  const int64_t head = round_up((int64_t)slack_pages * m.page_bytes + (hbm_bytes - param), gran);
  p->wva_size = (size_t)param;
  p->kva_size = (size_t)(head + param);
  CUresult r = drv().MemAddressReserve(&p->wva, p->wva_size, (size_t)gran, 0, 0);
  if (r != CUDA_SUCCESS) return bail(fail(KB_ECUDA, "cuMemAddressReserve(weights) failed"));
  r = drv().MemAddressReserve(&p->kva, p->kva_size, (size_t)gran, 0, 0);
  if (r != CUDA_SUCCESS) return bail(fail(KB_ECUDA, "cuMemAddressReserve(kv) failed"));
  {
    CUmemGenericAllocationHandle h;
    if ((rc = make_handle(device, head, &h))) return bail(rc);
    p->kv_segs.push_back({h, head, false});
    if ((rc = map_at(p, p->kva, head, h))) return bail(rc);
  }
  // each layer slab: one physical allocation, two views
  p->layer_handle.assign(m.num_layers, 0);
  p->layer_state.assign(m.num_layers, kLayerHeld);
  for (int l = 0; l < m.num_layers; ++l) {
    CUmemGenericAllocationHandle h;
    if ((rc = make_handle(device, m.slab_bytes, &h))) return bail(rc);
    p->layer_handle[l] = h;
    if ((rc = map_at(p, p->wva + (CUdeviceptr)l * m.slab_bytes, m.slab_bytes, h))) return bail(rc);
    if ((rc = map_at(p, p->kva + head + (CUdeviceptr)l * m.slab_bytes, m.slab_bytes, h)))
      return bail(rc);
  }
  p->head_pages = head / m.page_bytes;
  p->slack_pages = slack_pages;
  p->usable_pages = p->head_pages;
  p->max_pages = (int64_t)p->kva_size / m.page_bytes;
  if (m.head_dim == 128 && (m.block_tokens == 64 || m.block_tokens == 128)) {
    cuuint64_t dims[2] = {128, (cuuint64_t)(p->kva_size / 256)};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {64, (cuuint32_t)m.block_tokens};
    cuuint32_t estr[2] = {1, 1};
    r = drv().TensorMapEncodeTiled(&p->kv_tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                   reinterpret_cast<void*>(p->kva), dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return bail(fail(KB_ECUDA, "cuTensorMapEncodeTiled(kv) failed"));
  }
  if (p->max_pages >= (int64_t)1 << 31) return bail(fail(KB_EINVAL, "too many pages for int32 ids"));
  p->n_words = ceil_div(p->max_pages, 32);
  const int64_t cells = (int64_t)max_slots * m.num_layers;
  if (cells * max_pages_per_seq >= (int64_t)1 << 31)
    return bail(fail(KB_EINVAL, "block table too large for int32 cells"));
  if (cudaMalloc(&p->d_bitmap, p->n_words * 4) != cudaSuccess ||
      cudaMalloc(&p->d_owner, p->max_pages * 4) != cudaSuccess ||
      cudaMalloc(&p->d_bt, cells * max_pages_per_seq * 4) != cudaSuccess ||
      cudaMalloc(&p->d_np, cells * 4) != cudaSuccess)
    return bail(fail(KB_ECUDA, "cudaMalloc(pool metadata) failed"));
  cudaMemset(p->d_bitmap, 0, p->n_words * 4);
  cudaMemset(p->d_owner, 0xff, p->max_pages * 4);
  cudaMemset(p->d_bt, 0xff, cells * max_pages_per_seq * 4);
  cudaMemset(p->d_np, 0, cells * 4);
  p->h_np.assign(cells, 0);
  if (cudaMallocHost(&p->h_pinned, 64) != cudaSuccess)
    return bail(fail(KB_ECUDA, "cudaMallocHost failed"));
  if (cudaHostAlloc(&p->h_status, 64, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(reinterpret_cast<void**>(&p->d_status), p->h_status, 0) != cudaSuccess)
    return bail(fail(KB_ECUDA, "cudaHostAlloc(status) failed"));
  p->h_status[0] = 0;  // KB_KV_V_OVERFLOW seen
  p->h_status[1] = 0;  // KB_KV_V_UNDERFLOW seen
  p->h_status[2] = 0;  // KB_KV_NO_PAGE seen
  if (cudaStreamCreateWithFlags(&p->own_stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(KB_ECUDA, "cudaStreamCreate failed"));
  if (cudaEventCreateWithFlags(&p->counts_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->meta_ev, cudaEventDisableTiming) != cudaSuccess)
    return bail(fail(KB_ECUDA, "cudaEventCreate failed"));
  // sized for vacating every slab at once: never reallocated under a
  // compaction in flight
  if ((rc = ensure_scratch(p, 2 * (p->max_pages - p->head_pages) * 4 + 64 + (1 << 20))))
    return bail(rc);
  // every slab page starts reserved: the layer's weights live there
  range_mark_kernel<<<grid_for(p->max_pages - p->head_pages, 256, 1024), 256, 0, p->own_stream>>>(
      p->d_bitmap, p->d_owner, p->head_pages, p->max_pages, 1);
  if (cudaDeviceSynchronize() != cudaSuccess) return bail(fail(KB_ECUDA, "pool init sync failed"));
  *out = p;
  return KB_OK;
}

extern "C" int kb_pool_destroy(kb_pool* p) {
  if (!p) return KB_OK;
  cudaSetDevice(p->device);
  cudaDeviceSynchronize();
  const int64_t head = p->kv_segs.empty() ? 0 : p->kv_segs[0].bytes;
  for (int l = 0; l < (int)p->layer_handle.size(); ++l) {
    if (p->layer_handle[l]) {
      drv().MemUnmap(p->wva + (CUdeviceptr)l * p->m.slab_bytes, p->m.slab_bytes);
      drv().MemUnmap(p->kva + head + (CUdeviceptr)l * p->m.slab_bytes, p->m.slab_bytes);
      drv().MemRelease(p->layer_handle[l]);
    }
  }
  for (auto& s : p->kv_segs) {
    drv().MemUnmap(p->kva, s.bytes);
    drv().MemRelease(s.h);
  }
  if (p->wva) drv().MemAddressFree(p->wva, p->wva_size);
  if (p->kva) drv().MemAddressFree(p->kva, p->kva_size);
  if (p->d_bitmap) cudaFree(p->d_bitmap);
  if (p->d_owner) cudaFree(p->d_owner);
  if (p->view) {
    if (p->d_bt) cudaIpcCloseMemHandle(p->d_bt);
    if (p->d_np) cudaIpcCloseMemHandle(p->d_np);
  } else {
    if (p->d_bt) cudaFree(p->d_bt);
    if (p->d_np) cudaFree(p->d_np);
  }
  if (p->d_scratch) cudaFree(p->d_scratch);
  if (p->h_pinned) cudaFreeHost(p->h_pinned);
  if (p->h_status) cudaFreeHost(p->h_status);
  if (p->own_stream) cudaStreamDestroy(p->own_stream);
  for (auto& se : p->op_ev) cudaEventDestroy(se.second);
  if (p->counts_ev) cudaEventDestroy(p->counts_ev);
  if (p->meta_ev) cudaEventDestroy(p->meta_ev);
  delete p;
  return KB_OK;
}

extern "C" int kb_pool_query(kb_pool* p, kb_pool_info* o) {
  if (!p || !o) return fail(KB_EINVAL, "null pool");
  o->extent_pages = p->usable_pages;
  o->live_pages = p->live_pages;
  o->slack_pages = p->slack_pages;
  o->max_pages = p->max_pages;
  int held = 0;
  for (auto s : p->layer_state) held += s != kLayerDropped;
  o->layers_mapped = held;
  o->device = p->device;
  o->weight_base = (uint64_t)p->wva;
  o->kv_base = (uint64_t)p->kva;
  o->block_table = (uint64_t)p->d_bt;
  o->npages = (uint64_t)p->d_np;
  o->max_slots = p->max_slots;
  o->max_pages_per_seq = p->maxp;
  return KB_OK;
}

extern "C" uint64_t kb_weight_ptr(kb_pool* p, int32_t layer) {
  if (!p || layer < 0 || layer >= p->m.num_layers || p->layer_state[layer] == kLayerDropped)
    return 0;
  return (uint64_t)(p->wva + (CUdeviceptr)layer * p->m.slab_bytes);
}

// Land the last compaction's (moved, free-found) counts from pinned memory.
static int collect_counts(kb_pool* p) {
  if (!p->counts_pending) return KB_OK;
  KB_RT(cudaEventSynchronize(p->counts_ev));
  p->counts_pending = false;
  const int64_t* c = reinterpret_cast<const int64_t*>(p->h_pinned);
  p->last_moved = c[0];
  if (c[1] < c[0])  // cannot happen after restore_begin's capacity check
    return fail(KB_ESTATE, "compaction found too few free pages");
  return KB_OK;
}

extern "C" int kb_drop_layers(kb_pool* p, int32_t lo, int32_t hi, int64_t* remap_ns) {
  if (!p) return fail(KB_EINVAL, "null pool");
  if (p->view) return refuse_view();
  if (hi <= lo) return fail(KB_EINVAL, "empty layer range");
  for (int l = lo; l < hi; ++l) {
    if (l < 0 || l >= p->m.num_layers) return fail(KB_EINVAL, "layer " + std::to_string(l) + " absent from segment table");
    if (p->layer_state[l] != kLayerHeld)
      return fail(KB_ESTATE, "layer " + std::to_string(l) + " absent on device pool");
  }
  KB_RT(cudaSetDevice(p->device));
  const int64_t t0 = now_ns();
  // the slab pages of [lo, hi) become free KV pages; no driver call, the
  // slabs were mapped into the KV VA at creation.  A bitmap op: ordered
  // after every earlier one and before every later grow on any stream,
  // without blocking the host.
  const int64_t a = slab_first_page(p, lo), b = slab_first_page(p, hi);
  int rc = pool_meta_begin(p, p->own_stream, false);
  if (rc) return rc;
  range_mark_kernel<<<grid_for(b - a, 256, 1024), 256, 0, p->own_stream>>>(p->d_bitmap, p->d_owner,
                                                                           a, b, 0);
  KB_LAUNCH_CHECK();
  if ((rc = pool_meta_end(p, p->own_stream))) return rc;
  for (int l = lo; l < hi; ++l) p->layer_state[l] = kLayerDropped;
  p->usable_pages += b - a;
  if (remap_ns) *remap_ns = now_ns() - t0;
  return KB_OK;
}

extern "C" int kb_restore_begin(kb_pool* p, int32_t lo, int32_t hi, uintptr_t stream,
                                int64_t* moved_pages, int64_t* remap_ns) {
  if (!p) return fail(KB_EINVAL, "null pool");
  if (p->view) return refuse_view();
  if (hi <= lo) return fail(KB_EINVAL, "empty layer range");
  for (int l = lo; l < hi; ++l) {
    if (l < 0 || l >= p->m.num_layers) return fail(KB_EINVAL, "layer " + std::to_string(l) + " absent from segment table");
    if (p->layer_state[l] != kLayerDropped)
      return fail(KB_ESTATE, "layer " + std::to_string(l) + " already held on device pool");
  }
  const int64_t a = slab_first_page(p, lo), b = slab_first_page(p, hi);
  // every live page must fit outside the returned range
  if (p->live_pages > p->usable_pages - (b - a))
    return fail(KB_REFUSED, "restore blocked: " + std::to_string(p->live_pages) +
                                " live pages do not fit in " +
                                std::to_string(p->usable_pages - (b - a)) + " remaining pages");
  KB_RT(cudaSetDevice(p->device));
  const int64_t t0 = now_ns();
  cudaStream_t st = (cudaStream_t)stream;
  int rc = collect_counts(p);  // an earlier compaction's count, if unread
  if (rc) return rc;
  // releases / grows / copies in flight on other streams: the plan must see
  // them -- ordered on the device, the host does not block
  if ((rc = pool_meta_begin(p, st, true))) return rc;
  const int64_t cap = b - a;
  int64_t* d_counts = reinterpret_cast<int64_t*>(p->d_scratch);
  int32_t* d_src = reinterpret_cast<int32_t*>((char*)p->d_scratch + 64);
  int32_t* d_dst = d_src + cap;
  compact_plan_kernel<<<1, kScanThreads, 0, st>>>(p->d_bitmap, a, b, p->max_pages, d_src, d_dst,
                                                   cap, d_counts);
  KB_LAUNCH_CHECK();
  const int64_t pieces = p->m.page_bytes / kPieceBytes > 0 ? p->m.page_bytes / kPieceBytes : 1;
  compact_copy_kernel<<<grid_for(cap * pieces, 1, 148 * 16), kCopyThreads, 0, st>>>(
      reinterpret_cast<uint8_t*>(p->kva), d_src, d_dst, d_counts, p->m.page_bytes);
  KB_LAUNCH_CHECK();
  compact_fixup_kernel<<<grid_for(cap, 256, 1024), 256, 0, st>>>(p->d_bitmap, p->d_owner, p->d_bt,
                                                                  d_src, d_dst, d_counts);
  KB_LAUNCH_CHECK();
  range_mark_kernel<<<grid_for(cap, 256, 1024), 256, 0, st>>>(p->d_bitmap, p->d_owner, a, b, 1);
  KB_LAUNCH_CHECK();
  // the moved-page count travels back asynchronously (kb_pool_last_moved)
  KB_RT(cudaMemcpyAsync(p->h_pinned, d_counts, 16, cudaMemcpyDeviceToHost, st));
  KB_RT(cudaEventRecord(p->counts_ev, st));
  if ((rc = pool_meta_end(p, st))) return rc;
  p->counts_pending = true;
  for (int l = lo; l < hi; ++l) p->layer_state[l] = kLayerRestoring;
  p->usable_pages -= b - a;
  if (moved_pages) {
    if ((rc = collect_counts(p))) return rc;
    *moved_pages = p->last_moved;
  }
  if (remap_ns) *remap_ns = now_ns() - t0;
  return KB_OK;
}

extern "C" int kb_pool_last_moved(kb_pool* p, int64_t* moved_pages) {
  if (!p || !moved_pages) return fail(KB_EINVAL, "null argument");
  KB_RT(cudaSetDevice(p->device));
  int rc = collect_counts(p);
  if (rc) return rc;
  *moved_pages = p->last_moved;
  return KB_OK;
}

extern "C" int kb_restore_complete(kb_pool* p, int32_t lo, int32_t hi) {
  if (!p) return fail(KB_EINVAL, "null pool");
  if (p->view) return refuse_view();
  for (int l = lo; l < hi; ++l) {
    if (l < 0 || l >= p->m.num_layers || p->layer_state[l] != kLayerRestoring)
      return fail(KB_ESTATE, "layer " + std::to_string(l) + " not awaiting restore");
  }
  for (int l = lo; l < hi; ++l) p->layer_state[l] = kLayerHeld;
  return KB_OK;
}

extern "C" int kb_pages_grow(kb_pool* p, const kb_grow* reqs, int32_t n, uintptr_t stream) {
  if (!p) return fail(KB_EINVAL, "null pool");
  if (p->view) return refuse_view();
  if (n <= 0) return KB_OK;
  const int L = p->m.num_layers;
  int64_t total = 0;
  for (int i = 0; i < n; ++i) {
    const kb_grow& r = reqs[i];
    if (r.slot < 0 || r.slot >= p->max_slots || r.layer_lo < 0 || r.layer_hi > L ||
        r.layer_hi <= r.layer_lo || r.add_pages < 1)
      return fail(KB_EINVAL, "bad grow request " + std::to_string(i));
    for (int l = r.layer_lo; l < r.layer_hi; ++l) {
      int64_t c = (int64_t)r.slot * L + l;
      if (p->h_np[c] + r.add_pages > p->maxp)
        return fail(KB_EINVAL, "slot " + std::to_string(r.slot) + " exceeds max_pages_per_seq");
    }
    total += (int64_t)(r.layer_hi - r.layer_lo) * r.add_pages;
  }
  if (n > 1) {
    std::vector<int64_t> cells;
    for (int i = 0; i < n; ++i)
      for (int l = reqs[i].layer_lo; l < reqs[i].layer_hi; ++l)
        cells.push_back((int64_t)reqs[i].slot * L + l);
    std::sort(cells.begin(), cells.end());
    for (size_t i = 1; i < cells.size(); ++i)
      if (cells[i] == cells[i - 1]) return fail(KB_EINVAL, "duplicate (slot, layer) in one grow batch");
  }
  if (total > p->usable_pages - p->live_pages)
    return fail(KB_REFUSED, "out of KV pages: need " + std::to_string(total) + ", free " +
                                std::to_string(p->usable_pages - p->live_pages));
  KB_RT(cudaSetDevice(p->device));
  cudaStream_t st = (cudaStream_t)stream;
  // batches travel in kernel parameter space: no staging copy, no host
  // synchronization; ordered after the pool's earlier bitmap ops
  int rc = pool_meta_begin(p, st, false);
  if (rc) return rc;
  GrowBatch batch;
  for (int b0 = 0; b0 < n; b0 += kGrowBatch) {
    const int nb = std::min(kGrowBatch, n - b0);
    int64_t sub = 0;
    for (int i = 0; i < nb; ++i) {
      batch.r[i] = reqs[b0 + i];
      batch.cum[i] = sub;
      sub += (int64_t)(reqs[b0 + i].layer_hi - reqs[b0 + i].layer_lo) * reqs[b0 + i].add_pages;
    }
    grow_kernel<<<1, kScanThreads, 0, st>>>(p->d_bitmap, p->d_owner, p->d_bt, p->d_np, batch, nb,
                                            sub, p->max_pages, L, p->maxp);
    KB_LAUNCH_CHECK();
  }
  if ((rc = pool_meta_end(p, st))) return rc;
  for (int i = 0; i < n; ++i)
    for (int l = reqs[i].layer_lo; l < reqs[i].layer_hi; ++l)
      p->h_np[(int64_t)reqs[i].slot * L + l] += reqs[i].add_pages;
  p->live_pages += total;
  return KB_OK;
}

extern "C" int kb_pages_release(kb_pool* p, const int32_t* slots, int32_t n, int32_t lo,
                                int32_t hi, uintptr_t stream) {
  if (!p) return fail(KB_EINVAL, "null pool");
  if (p->view) return refuse_view();
  const int L = p->m.num_layers;
  if (n <= 0 || hi <= lo) return KB_OK;
  if (lo < 0 || hi > L) return fail(KB_EINVAL, "bad layer range");
  int64_t freed = 0;
  for (int i = 0; i < n; ++i) {
    if (slots[i] < 0 || slots[i] >= p->max_slots) return fail(KB_EINVAL, "bad slot");
    for (int l = lo; l < hi; ++l) freed += p->h_np[(int64_t)slots[i] * L + l];
  }
  KB_RT(cudaSetDevice(p->device));
  cudaStream_t st = (cudaStream_t)stream;
  // after every stream's last op: no reader may still be on these pages
  int rc = pool_meta_begin(p, st, true);
  if (rc) return rc;
  SlotBatch batch;
  for (int b0 = 0; b0 < n; b0 += kReleaseBatch) {
    const int nb = std::min(kReleaseBatch, n - b0);
    for (int i = 0; i < nb; ++i) batch.s[i] = slots[b0 + i];
    release_kernel<<<nb * (hi - lo), 128, 0, st>>>(p->d_bitmap, p->d_owner, p->d_bt, p->d_np,
                                                    batch, lo, hi, L, p->maxp);
    KB_LAUNCH_CHECK();
  }
  if ((rc = pool_meta_end(p, st))) return rc;
  for (int i = 0; i < n; ++i)
    for (int l = lo; l < hi; ++l) p->h_np[(int64_t)slots[i] * L + l] = 0;
  p->live_pages -= freed;
  return KB_OK;
}

extern "C" int64_t kb_pages_per_layer_count(kb_pool* p, int32_t slot, int32_t layer) {
  if (!p || slot < 0 || slot >= p->max_slots || layer < 0 || layer >= p->m.num_layers) return -1;
  return p->h_np[(int64_t)slot * p->m.num_layers + layer];
}

extern "C" int kb_read_block_table(kb_pool* p, int32_t slot, int32_t layer, int32_t* out,
                                   int32_t cap, int32_t* n_out) {
  if (!p || slot < 0 || slot >= p->max_slots || layer < 0 || layer >= p->m.num_layers)
    return fail(KB_EINVAL, "bad slot/layer");
  KB_RT(cudaSetDevice(p->device));
  KB_RT(cudaDeviceSynchronize());
  int cnt = 0;
  KB_RT(cudaMemcpy(&cnt, p->d_np + (int64_t)slot * p->m.num_layers + layer, 4, cudaMemcpyDeviceToHost));
  if (cnt > cap) return fail(KB_EINVAL, "output buffer too small");
  if (cnt)
    KB_RT(cudaMemcpy(out, p->d_bt + ((int64_t)slot * p->m.num_layers + layer) * p->maxp,
                     (size_t)cnt * 4, cudaMemcpyDeviceToHost));
  *n_out = cnt;
  return KB_OK;
}

extern "C" int kb_read_bitmap(kb_pool* p, uint32_t* out, int64_t n_words) {
  if (!p || n_words > p->n_words) return fail(KB_EINVAL, "bad bitmap read");
  if (p->view) return refuse_view();
  KB_RT(cudaSetDevice(p->device));
  KB_RT(cudaDeviceSynchronize());
  KB_RT(cudaMemcpy(out, p->d_bitmap, (size_t)n_words * 4, cudaMemcpyDeviceToHost));
  return KB_OK;
}

extern "C" int kb_read_owner(kb_pool* p, int32_t* out, int64_t n) {
  if (!p || n > p->max_pages) return fail(KB_EINVAL, "bad owner read");
  if (p->view) return refuse_view();
  KB_RT(cudaSetDevice(p->device));
  KB_RT(cudaDeviceSynchronize());
  KB_RT(cudaMemcpy(out, p->d_owner, (size_t)n * 4, cudaMemcpyDeviceToHost));
  return KB_OK;
}

// ------------------------------------------------------- cross-process views
// One process per GPU: the owner exports its VMM handles as POSIX file
// descriptors and its block table / page counts as CUDA IPC handles; a peer
// imports them as a read-only view in its own VA with access for its own
// device, and pulls pages and slabs over NVLink with the same copy kernels.

extern "C" int kb_pool_export(kb_pool* p, kb_export_desc* o, int32_t* fds, int32_t cap) {
  if (!p || !o || !fds) return fail(KB_EINVAL, "null argument");
  if (p->view) return refuse_view();
  const int n = 1 + p->m.num_layers;
  if (cap < n) return fail(KB_EINVAL, "fd buffer holds " + std::to_string(cap) + " < " +
                                          std::to_string(n) + " handles");
  KB_RT(cudaSetDevice(p->device));
  std::memset(o, 0, sizeof(*o));
  o->model = p->m;
  o->hbm_bytes = p->hbm_bytes;
  o->head_bytes = p->kv_segs.empty() ? 0 : p->kv_segs[0].bytes;
  o->slack_pages = p->slack_pages;
  o->device = p->device;
  o->max_slots = p->max_slots;
  o->max_pages_per_seq = p->maxp;
  o->n_handles = n;
  static_assert(sizeof(cudaIpcMemHandle_t) <= 64, "ipc handle size");
  cudaIpcMemHandle_t hb, hn;
  KB_RT(cudaIpcGetMemHandle(&hb, p->d_bt));
  KB_RT(cudaIpcGetMemHandle(&hn, p->d_np));
  std::memcpy(o->bt_ipc, &hb, sizeof(hb));
  std::memcpy(o->np_ipc, &hn, sizeof(hn));
  for (int i = 0; i < n; ++i) fds[i] = -1;
  for (int i = 0; i < n; ++i) {
    CUmemGenericAllocationHandle h = i == 0 ? p->kv_segs[0].h : p->layer_handle[i - 1];
    int fd = -1;
    CUresult r = drv().MemExport(&fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    if (r != CUDA_SUCCESS) return fail(KB_ECUDA, "cuMemExportToShareableHandle failed for handle " +
                                                     std::to_string(i));
    fds[i] = fd;
  }
  return KB_OK;
}

extern "C" int kb_pool_import(int32_t device, const kb_export_desc* d, const int32_t* fds,
                              int32_t n_fds, kb_pool** out) {
  if (!d || !fds || !out) return fail(KB_EINVAL, "null argument");
  *out = nullptr;
  const kb_model_desc m = d->model;
  if (m.num_layers < 1 || m.slab_bytes < 1 || m.page_bytes < 1 || d->head_bytes < 0)
    return fail(KB_EINVAL, "bad export descriptor");
  if (n_fds != 1 + m.num_layers || d->n_handles != n_fds)
    return fail(KB_EINVAL, "export carries " + std::to_string(n_fds) + " handles, want " +
                               std::to_string(1 + m.num_layers));
  int rc = set_device(device);
  if (rc) return rc;
  kb_pool* p = new kb_pool();
  p->view = true;
  p->device = device;
  p->m = m;
  p->hbm_bytes = d->hbm_bytes;
  p->access.push_back(device);
  p->max_slots = d->max_slots;
  p->maxp = d->max_pages_per_seq;
  auto bail = [&](int code) {
    kb_pool_destroy(p);
    return code;
  };
  int64_t gran = 0;
  if ((rc = kb_vmm_granularity(device, &gran))) return bail(rc);
  p->gran = gran;
  const int64_t param = (int64_t)m.num_layers * m.slab_bytes;
  const int64_t head = d->head_bytes;
  p->wva_size = (size_t)param;
  p->kva_size = (size_t)(head + param);
  if (drv().MemAddressReserve(&p->wva, p->wva_size, (size_t)gran, 0, 0) != CUDA_SUCCESS ||
      drv().MemAddressReserve(&p->kva, p->kva_size, (size_t)gran, 0, 0) != CUDA_SUCCESS)
    return bail(fail(KB_ECUDA, "cuMemAddressReserve(view) failed"));
  auto import = [&](int32_t fd, CUmemGenericAllocationHandle* h) -> int {
    CUresult r = drv().MemImport(h, reinterpret_cast<void*>((uintptr_t)fd),
                                 CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    if (r != CUDA_SUCCESS) return fail(KB_ECUDA, "cuMemImportFromShareableHandle failed");
    return KB_OK;
  };
  {
    CUmemGenericAllocationHandle h;
    if ((rc = import(fds[0], &h))) return bail(rc);
    p->kv_segs.push_back({h, head, false});
    if ((rc = map_at(p, p->kva, head, h))) return bail(rc);
  }
  p->layer_handle.assign(m.num_layers, 0);
  p->layer_state.assign(m.num_layers, kLayerHeld);
  for (int l = 0; l < m.num_layers; ++l) {
    CUmemGenericAllocationHandle h;
    if ((rc = import(fds[1 + l], &h))) return bail(rc);
    p->layer_handle[l] = h;
    if ((rc = map_at(p, p->wva + (CUdeviceptr)l * m.slab_bytes, m.slab_bytes, h))) return bail(rc);
    if ((rc = map_at(p, p->kva + head + (CUdeviceptr)l * m.slab_bytes, m.slab_bytes, h)))
      return bail(rc);
  }
  p->head_pages = head / m.page_bytes;
  p->slack_pages = d->slack_pages;
  p->max_pages = (int64_t)p->kva_size / m.page_bytes;
  p->usable_pages = p->head_pages;
  cudaIpcMemHandle_t hb, hn;
  std::memcpy(&hb, d->bt_ipc, sizeof(hb));
  std::memcpy(&hn, d->np_ipc, sizeof(hn));
  void* bt = nullptr;
  void* np = nullptr;
  if (cudaIpcOpenMemHandle(&bt, hb, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return bail(fail(KB_ECUDA, "cudaIpcOpenMemHandle(block table) failed"));
  p->d_bt = static_cast<int32_t*>(bt);
  if (cudaIpcOpenMemHandle(&np, hn, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return bail(fail(KB_ECUDA, "cudaIpcOpenMemHandle(page counts) failed"));
  p->d_np = static_cast<int32_t*>(np);
  p->h_np.assign((size_t)p->max_slots * m.num_layers, 0);
  if (cudaStreamCreateWithFlags(&p->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->meta_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->counts_ev, cudaEventDisableTiming) != cudaSuccess)
    return bail(fail(KB_ECUDA, "view stream/event creation failed"));
  *out = p;
  return KB_OK;
}

extern "C" int kb_pool_view_refresh(kb_pool* p, const uint8_t* layer_held, int32_t n_layers) {
  if (!p || !layer_held) return fail(KB_EINVAL, "null argument");
  if (!p->view) return fail(KB_EINVAL, "not a peer view");
  if (n_layers != p->m.num_layers) return fail(KB_EINVAL, "layer count mismatch");
  KB_RT(cudaSetDevice(p->device));
  KB_RT(cudaMemcpy(p->h_np.data(), p->d_np, p->h_np.size() * 4, cudaMemcpyDeviceToHost));
  int64_t live = 0, usable = p->head_pages;
  const int64_t sp = p->m.slab_bytes / p->m.page_bytes;
  for (auto c : p->h_np) live += c;
  for (int l = 0; l < n_layers; ++l) {
    p->layer_state[l] = layer_held[l] ? kLayerHeld : kLayerDropped;
    if (!layer_held[l]) usable += sp;
  }
  p->live_pages = live;
  p->usable_pages = usable;
  return KB_OK;
}

extern "C" int kb_pool_is_view(kb_pool* p) { return p && p->view ? 1 : 0; }

// Work the pool cannot see (a CUDA graph replay: captures record no pool
// events) brackets itself with these, so the replay waits for the last
// bitmap op and later releases / compactions wait for the replay.
extern "C" int kb_pool_stream_begin(kb_pool* p, uintptr_t stream) {
  if (!p) return fail(KB_EINVAL, "null pool");
  KB_RT(cudaSetDevice(p->device));
  return pool_enter(p, (cudaStream_t)stream);
}

extern "C" int kb_pool_stream_end(kb_pool* p, uintptr_t stream) {
  if (!p) return fail(KB_EINVAL, "null pool");
  KB_RT(cudaSetDevice(p->device));
  return pool_leave(p, (cudaStream_t)stream);
}
