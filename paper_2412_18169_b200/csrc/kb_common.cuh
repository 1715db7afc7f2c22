// Shared internals of the kunserve_b200 C-ABI library (sm_100a).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/kunserve_b200.h"

namespace kb {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

// CUDA driver entry points, resolved at run time through the runtime's
// cudaGetDriverEntryPoint so the library has no link-time libcuda
// dependency (it loads -- and exports its ABI -- on a host without a GPU).
struct Driver {
  PFN_cuMemCreate MemCreate = nullptr;
  PFN_cuMemRelease MemRelease = nullptr;
  PFN_cuMemMap MemMap = nullptr;
  PFN_cuMemUnmap MemUnmap = nullptr;
  PFN_cuMemSetAccess MemSetAccess = nullptr;
  PFN_cuMemAddressReserve MemAddressReserve = nullptr;
  PFN_cuMemAddressFree MemAddressFree = nullptr;
  PFN_cuMemGetAllocationGranularity MemGetAllocationGranularity = nullptr;
  PFN_cuTensorMapEncodeTiled TensorMapEncodeTiled = nullptr;
  PFN_cuGetErrorString GetErrorString = nullptr;
  PFN_cuMemExportToShareableHandle MemExport = nullptr;
  PFN_cuMemImportFromShareableHandle MemImport = nullptr;
  bool ready = false;
};
Driver& drv();
int ensure_driver();

#define KB_CU(call)                                                           \
  do {                                                                        \
    CUresult _r = (call);                                                     \
    if (_r != CUDA_SUCCESS) {                                                 \
      const char* _s = nullptr;                                               \
      if (::kb::drv().GetErrorString) ::kb::drv().GetErrorString(_r, &_s);     \
      return ::kb::fail(KB_ECUDA, std::string(#call) + ": " + (_s ? _s : "?")); \
    }                                                                         \
  } while (0)

#define KB_RT(call)                                                           \
  do {                                                                        \
    cudaError_t _e = (call);                                                  \
    if (_e != cudaSuccess) {                                                  \
      return ::kb::fail(KB_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    }                                                                         \
  } while (0)

#define KB_LAUNCH_CHECK()                                                     \
  do {                                                                        \
    cudaError_t _e = cudaGetLastError();                                      \
    if (_e != cudaSuccess) {                                                  \
      return ::kb::fail(KB_ECUDA, std::string("launch: ") + cudaGetErrorString(_e)); \
    }                                                                         \
  } while (0)

// Stream ordering of pool operations (see kb_pool::op_ev), all on the
// device -- the host never blocks.  Program order of the API calls is the
// order that counts:
//  * bitmap ops (grow, release, drop, compaction) run after the previous
//    bitmap op, whatever streams the two were issued on; release and
//    compaction also run after the last op of every stream that touched
//    the pool (no page is freed or moved under a reader or writer);
//  * data ops (page copies, appends, attention) run after the last bitmap
//    op, so they see every block-table change issued before them.
int pool_enter(kb_pool* p, cudaStream_t st);
int pool_leave(kb_pool* p, cudaStream_t st);
int pool_meta_begin(kb_pool* p, cudaStream_t st, bool wait_all_streams);
int pool_meta_end(kb_pool* p, cudaStream_t st);

struct KvSeg {
  CUmemGenericAllocationHandle h;
  int64_t bytes;
  bool slab;
};

constexpr uint8_t kLayerHeld = 0;       // weights valid under the weight VA
constexpr uint8_t kLayerDropped = 1;    // slab pages belong to the KV pool
constexpr uint8_t kLayerRestoring = 2;  // slab vacated, parameter pull pending

}  // namespace kb

struct kb_pool {
  int device = 0;
  kb_model_desc m{};
  int64_t hbm_bytes = 0;
  int64_t gran = 0;
  std::vector<int> access;  // devices granted RW on every mapping (self first)

  CUdeviceptr wva = 0;
  size_t wva_size = 0;
  CUdeviceptr kva = 0;
  size_t kva_size = 0;
  std::vector<CUmemGenericAllocationHandle> layer_handle;  // slab l (mapped twice)
  std::vector<uint8_t> layer_state;                        // kLayerHeld / Dropped / Restoring
  std::vector<kb::KvSeg> kv_segs;                          // head segment

  int64_t head_pages = 0;    // slack + residual pages at the head of the KV VA
  int64_t usable_pages = 0;  // head + pages of every dropped slab
  int64_t slack_pages = 0;
  int64_t max_pages = 0;
  int64_t live_pages = 0;
  int64_t n_words = 0;

  int max_slots = 0;
  int maxp = 0;  // max pages per (slot, layer)
  uint32_t* d_bitmap = nullptr;
  int32_t* d_owner = nullptr;
  int32_t* d_bt = nullptr;
  int32_t* d_np = nullptr;
  std::vector<int32_t> h_np;  // host mirror of npages

  // scratch: device buffer for request lists and compaction pairs
  void* d_scratch = nullptr;
  int64_t scratch_bytes = 0;
  int32_t* h_pinned = nullptr;  // small pinned readback buffer
  // sticky KV status, pinned + mapped: word 0 = a V value overflowed fp16,
  // word 1 = a V row underflowed; appends set them from the device with
  // plain stores, the host reads them without a copy (kb_pool_kv_status)
  uint32_t* h_status = nullptr;
  uint32_t* d_status = nullptr;
  cudaStream_t own_stream = nullptr;
  // Cross-stream ordering without host synchronization (kb::pool_enter /
  // pool_leave / pool_meta_begin / pool_meta_end): the last pool operation
  // of every stream that touched the pool, the last bitmap op and the last
  // compaction.
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> op_ev;
  cudaEvent_t meta_ev = nullptr;    // last bitmap op
  cudaEvent_t counts_ev = nullptr;  // last compaction's counts in h_pinned
  bool meta_set = false;
  bool counts_pending = false;  // compaction counts still in flight to h_pinned
  int64_t last_moved = 0;
  // TMA descriptor over the whole KV VA viewed as [rows][head_dim] bf16
  // (row = one token of one kv head of K or V), box = [block_tokens][64].
  alignas(64) CUtensorMap kv_tmap;
  // Imported from another process (kb_pool_import): slabs mapped from the
  // owner's exported handles, block table / page counts opened through CUDA
  // IPC.  Only a copy source; every mutating entry point refuses a view.
  bool view = false;
};

namespace kb {
// cudaFuncAttributeMaxDynamicSharedMemorySize is a property of (kernel,
// device): opt `fn` in on `device` once (thread-safe; every template
// instantiation is its own kernel pointer).
int ensure_smem_attr(const void* fn, int bytes, int device);
int ensure_scratch(kb_pool* p, int64_t bytes);
int refuse_view();
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }
inline int grid_for(int64_t work, int per_block, int max_blocks) {
  int64_t g = ceil_div(work, per_block);
  if (g > max_blocks) g = max_blocks;
  if (g < 1) g = 1;
  return (int)g;
}
}  // namespace kb
