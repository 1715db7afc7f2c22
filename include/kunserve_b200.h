/*
 * kunserve_b200.h -- C ABI of the B200 data plane for KunServe's
 * parameter-centric overload path (arXiv 2412.18169).
 *
 * The reference (pkg/src/dropsim, pure Python) has no FFI: its "device"
 * is a segment table and a link model.  Each entry point below is the
 * device implementation behind one reference call site; the citation on
 * every declaration names the reference function whose semantics it
 * implements (file:line under /root/reference/pkg/src/dropsim/).
 *
 * Conventions
 *   - plain pointers and sizes only; no torch / CUDA runtime types.
 *     Streams are passed as `uintptr_t` (a cudaStream_t / CUstream value).
 *   - status: 0 = ok, 1 = expected refusal (out of pages, restore cannot
 *     vacate), < 0 = error.  kb_last_error() returns the thread-local text.
 *     The Python shim maps refusals to the reference's False returns and
 *     errors to ValueError/RuntimeError with the same text.
 *   - single driver thread (reference SPEC.md:100); device work is async on
 *     the caller's stream unless the function says it synchronizes.
 *
 * Device layout
 *   weight VA : num_layers x slab_bytes, layer l at l*slab_bytes; one
 *               physical VMM handle (cuMemCreate) per layer slab, mapped at
 *               pool creation under the weight VA AND under its alias in
 *               the KV VA (drop / restore flip page availability; no
 *               cuMemMap / cuMemUnmap on the hot path).
 *   KV VA     : [slack pages | residual | alias of slab 0 | ... slab L-1]
 *               (a slab's alias pages are free for KV only while its layer
 *               is dropped; reserved otherwise)
 *               page p at kv_base + p*page_bytes; a page holds one layer of
 *               `block_tokens` tokens of one request:
 *               [K|V][n_kv_heads][block_tokens][head_dim], K bf16, V fp16
 *               (V converted on append; range-guarded, see kb_pool_kv_status).
 *   metadata  : page bitmap (1 = live), owner[page] (reverse map),
 *               block_table[slot][layer][max_pages_per_seq] (int32, -1 empty),
 *               npages[slot][layer].
 */
#ifndef KUNSERVE_B200_H
#define KUNSERVE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KB_OK 0
#define KB_REFUSED 1
#define KB_EINVAL (-1)
#define KB_ECUDA (-2)
#define KB_ESTATE (-3)

typedef struct kb_pool kb_pool; /* opaque: one instance's HBM on one GPU */

typedef struct kb_model_desc {
    int32_t num_layers;      /* ModelSpec.num_layers (ref core.py:50-68) */
    int32_t n_kv_heads;
    int32_t head_dim;        /* 128 for every BASELINE model */
    int32_t block_tokens;    /* tokens per page */
    int64_t slab_bytes;      /* ModelSpec.bytes_per_layer, 2 MiB multiple */
    int64_t page_bytes;      /* block_tokens * 2 * n_kv_heads * head_dim * 2 */
} kb_model_desc;

typedef struct kb_pool_info {
    int64_t extent_pages;    /* mapped KV pages (slack + residual + dropped) */
    int64_t live_pages;
    int64_t slack_pages;
    int64_t max_pages;       /* KV VA capacity in pages */
    int32_t layers_mapped;   /* layers whose slab is mapped at the weight VA */
    int32_t device;
    uint64_t weight_base;    /* device VA of layer 0's slab */
    uint64_t kv_base;        /* device VA of page 0 */
    uint64_t block_table;    /* device pointer, int32 [max_slots][L][max_pages_per_seq] */
    uint64_t npages;         /* device pointer, int32 [max_slots][L] */
    int32_t max_slots;
    int32_t max_pages_per_seq;
} kb_pool_info;

/* One block-table growth request: every layer in [layer_lo, layer_hi) of
 * `slot` gains `add_pages` pages (lowest free page ids first, assigned in
 * request order, then layer order, then page order). */
typedef struct kb_grow {
    int32_t slot;
    int32_t layer_lo;
    int32_t layer_hi;
    int32_t add_pages;
} kb_grow;

/* One KV move: flattened page range [flat_lo, flat_hi) of the layer range
 * [layer_lo, layer_hi) of a request, flat = (layer - layer_lo) * npages + i,
 * from src_slot in the source pool to dst_slot in the destination pool. */
typedef struct kb_move {
    int32_t src_slot;
    int32_t dst_slot;
    int32_t layer_lo;
    int32_t layer_hi;
    int32_t npages;
    int32_t flat_lo;
    int32_t flat_hi;
    int32_t _pad;
} kb_move;

/* ---- context / errors ------------------------------------------------- */
const char* kb_last_error(void);
int kb_version(void);
/* Initialise the CUDA primary context of `device` and enable peer access
 * to the listed peers (NVSwitch: every pair).  Idempotent. */
int kb_init(int32_t device, const int32_t* peers, int32_t n_peers);
int kb_vmm_granularity(int32_t device, int64_t* out_bytes);

/* ---- N1: VMM slab pool ------------------------------------------------ */
/* build_instance (memory.py:132-144): one cuMemCreate slab per layer mapped
 * into the weight VA, residual budget (hbm_bytes - param_bytes, rounded up
 * to the granularity) plus `slack_pages` of fragmentation headroom at the
 * head of the KV VA.  Refuses (KB_EINVAL) when hbm_bytes <= param_bytes. */
int kb_pool_create(int32_t device, const kb_model_desc* model, int64_t hbm_bytes,
                   int32_t max_slots, int32_t max_pages_per_seq, int32_t slack_pages,
                   const int32_t* peers, int32_t n_peers, kb_pool** out);
int kb_pool_destroy(kb_pool* pool);
int kb_pool_query(kb_pool* pool, kb_pool_info* out);

/* drop_layers (memory.py:147-172) + the caller's remap charge
 * (engine.py:796-807).  Every layer slab is mapped at creation under both
 * the weight VA and a fixed page range of the KV VA, so a drop is one
 * bitmap kernel: the slab pages of [lo, hi) turn from reserved into free KV
 * pages.  Asynchronous; ordered before every later page operation on any
 * stream (see "Stream ordering" below).  remap_ns receives the host time. */
int kb_drop_layers(kb_pool* pool, int32_t lo, int32_t hi, int64_t* remap_ns);

/* restore_layers (memory.py:175-197): vacate the slab page range of
 * [lo, hi) -- live pages there move to the lowest free pages outside it
 * (device compaction, block tables rewritten on device through the owner
 * map) -- and mark it reserved again so the parameter pull can land under
 * the weight VA.  KB_REFUSED (nothing changed) if the live pages cannot
 * fit.  Runs on `stream` after every earlier page operation of the pool on
 * any stream, before every later one; the host does not block.  With a
 * non-NULL moved_pages the call waits for the compaction and reports its
 * size; otherwise read it later with kb_pool_last_moved. */
int kb_restore_begin(kb_pool* pool, int32_t lo, int32_t hi, uintptr_t stream,
                     int64_t* moved_pages, int64_t* remap_ns);
/* pages moved by the pool's last compaction (waits for it) */
int kb_pool_last_moved(kb_pool* pool, int64_t* moved_pages);
/* complete_restore (memory.py:200-212): bookkeeping only; validates that
 * [lo, hi) is mapped at the weight VA awaiting the pull. */
int kb_restore_complete(kb_pool* pool, int32_t lo, int32_t hi);
/* device pointer of layer `layer`'s slab in the weight VA (0 if unmapped) */
uint64_t kb_weight_ptr(kb_pool* pool, int32_t layer);

/* Stream ordering.  Page operations may be issued on any streams without
 * host synchronization; the order of the calls is the order on the device.
 * Grows, releases, drops and compactions run after the pool's previous one
 * of those; releases and compactions also after the last operation of
 * every stream that touched the pool (no page is freed or moved under a
 * reader); copies, appends and attention after the last grow / release /
 * drop / compaction.  Inside a CUDA graph capture the graph's own edges are
 * the ordering; a REPLAY of such a graph is invisible to the pool, so the
 * caller brackets it with kb_pool_stream_begin / kb_pool_stream_end on the
 * replay stream (wait for the last bitmap op; later releases and
 * compactions wait for the replay). */
int kb_pool_stream_begin(kb_pool* pool, uintptr_t stream);
int kb_pool_stream_end(kb_pool* pool, uintptr_t stream);

/* ---- N2: paged KV block tables (KVAllocator, memory.py:70-129) ---------- */
/* Grow block tables on device: the kernel takes the K lowest free page ids
 * below the extent (K = sum of (layer_hi-layer_lo)*add_pages) and appends
 * them.  KB_REFUSED if fewer than K pages are free (nothing changed). */
int kb_pages_grow(kb_pool* pool, const kb_grow* reqs, int32_t n, uintptr_t stream);
/* Release every page of layers [lo, hi) of each listed slot (free / shrink
 * of a request's allocation on this member, and the source side of an
 * exchange once its last chunk lands). */
int kb_pages_release(kb_pool* pool, const int32_t* slots, int32_t n, int32_t lo,
                     int32_t hi, uintptr_t stream);
/* Host copies of device state, for parity checks (synchronizing). */
int kb_read_block_table(kb_pool* pool, int32_t slot, int32_t layer, int32_t* out,
                        int32_t cap, int32_t* n_out);
int kb_read_bitmap(kb_pool* pool, uint32_t* out, int64_t n_words);
int kb_read_owner(kb_pool* pool, int32_t* out, int64_t n);
int64_t kb_pages_per_layer_count(kb_pool* pool, int32_t slot, int32_t layer);

/* ---- N1 across processes: peer views over NVLink ------------------------ */
/* One process per GPU (torchrun): a pool is exported once as POSIX file
 * descriptors of its VMM handles (head segment, then slab 0..L-1) plus CUDA
 * IPC handles of its block table and page counts; a peer process imports
 * them as a read-only VIEW mapped into its own VA with access for its own
 * device, so kb_copy_pages / kb_copy_slabs with the view as `src` pull the
 * owner's pages and slabs over NVLink (plan_exchange / plan_restore_transfers
 * flows whose source lives on another rank, exchange.py:146-249).  A view
 * refuses every mutating call (grow, release, drop, restore, append,
 * attention); the owner performs those, and the two processes order them
 * (a view's copies complete before the owner releases or compacts).
 * kb_pool_export fills `fds[0 .. 1+L)` with new descriptors the caller
 * passes on (SCM_RIGHTS) and closes. */
typedef struct kb_export_desc {
    kb_model_desc model;
    int64_t hbm_bytes;
    int64_t head_bytes;      /* KV VA head segment (slack + residual), bytes */
    int64_t slack_pages;
    int32_t device;          /* owner's device ordinal */
    int32_t max_slots;
    int32_t max_pages_per_seq;
    int32_t n_handles;       /* 1 + num_layers */
    uint8_t bt_ipc[64];      /* cudaIpcMemHandle_t of block_table */
    uint8_t np_ipc[64];      /* cudaIpcMemHandle_t of npages */
} kb_export_desc;
int kb_pool_export(kb_pool* pool, kb_export_desc* out, int32_t* fds, int32_t cap);
int kb_pool_import(int32_t device, const kb_export_desc* desc, const int32_t* fds,
                   int32_t n_fds, kb_pool** out);
/* Refresh a view's host mirrors before planning against it: page counts
 * from the owner's device array (synchronizing), layer states from the
 * caller's mirror of the owner's segment table (1 = held). */
int kb_pool_view_refresh(kb_pool* view, const uint8_t* layer_held, int32_t n_layers);
/* 1 if `pool` is an imported view, 0 if this process owns it. */
int kb_pool_is_view(kb_pool* pool);

/* ---- N4/N5/N7: NVLink peer copy kernels --------------------------------- */
/* KV exchange / consolidation (exchange.py:146-205, engine.py:690-726,
 * 1211-1239): copy whole pages named by the two pools' block tables. */
int kb_copy_pages(kb_pool* dst, kb_pool* src, const kb_move* moves, int32_t n,
                  uintptr_t stream);
/* Parameter restore / fetch (exchange.py:208-249): bytes [byte_lo, byte_hi)
 * of the weight range of layers [lo, hi) from src's weight VA to dst's. */
int kb_copy_slabs(kb_pool* dst, kb_pool* src, int32_t lo, int32_t hi, int64_t byte_lo,
                  int64_t byte_hi, uintptr_t stream);
/* HOST replica source (exchange.py:18, 224-233): pinned host -> weight VA. */
int kb_copy_slabs_from_host(kb_pool* dst, const void* host_src, int32_t lo, int32_t hi,
                            int64_t byte_lo, int64_t byte_hi, uintptr_t stream);
/* Swap baseline (engine.py:906-970, KV to / from the HOST pseudo instance):
 * the pages of move->src_slot, layers [layer_lo, layer_hi), flattened pages
 * [flat_lo, flat_hi) to (to_host = 1) or from (0) a pinned host buffer
 * holding flattened page f at host + f * page_bytes (dst_slot unused). */
int kb_copy_pages_host(kb_pool* pool, const kb_move* move, void* host, int32_t to_host,
                       uintptr_t stream);
/* Activation hand-off between pipeline stages (engine.py:428-448) and any
 * other flat device-to-device (peer) copy: 16-byte vector kernel. */
int kb_copy_bytes(uint64_t dst, uint64_t src, int64_t nbytes, uintptr_t stream);

/* ---- N7 across processes: activation hand-off buffers ------------------- */
/* The receiving stage of a pipeline group (engine.py:428-448) allocates its
 * activation slots with kb_device_alloc and exports them (CUDA IPC); the
 * sending stage maps them (kb_ipc_mem_import) and writes each microbatch's
 * rows with kb_copy_bytes -- stores over NVLink into the peer's HBM. */
int kb_device_alloc(int32_t device, int64_t nbytes, uint64_t* ptr);
int kb_device_free(uint64_t ptr);
/* ptr must be a kb_device_alloc pointer (CUDA IPC names whole allocations) */
int kb_ipc_mem_export(uint64_t ptr, uint8_t* handle /* 64 bytes */);
int kb_ipc_mem_import(int32_t device, const uint8_t* handle, uint64_t* ptr);
int kb_ipc_mem_close(uint64_t ptr);

/* ---- N8: paged attention over the pool --------------------------------- */
/* Write the new tokens' K/V into their pages.  k, v: [ntok][n_kv_heads][head_dim]
 * bf16; token t belongs to slot slots[t] at position pos[t]; its page must
 * already be in the block table.  row_stride: elements between consecutive
 * tokens' rows of k and v (0 = contiguous, n_kv_heads * head_dim), so the
 * K and V column blocks of a fused QKV projection can be passed in place. */
int kb_kv_append(kb_pool* pool, int32_t layer, uint64_t k, uint64_t v,
                 uint64_t slots, uint64_t pos, int32_t ntok, int64_t row_stride,
                 uintptr_t stream);
/* The V cache is fp16: exact for bf16 V values of magnitude in [2^-14,
 * 65504] (or 0).  Appends flag, in the pool's sticky status word,
 * KB_KV_V_OVERFLOW for any |v| >= 2^16 (inf, NaN included) and
 * KB_KV_V_UNDERFLOW for a V row (one token, one kv head) whose largest |v|
 * is nonzero and below 2^-14 (the whole row would be fp16-subnormal; small
 * entries beside a normal row maximum keep the normal range's 2^-11 error
 * bound relative to it), and still store the fp16 rounding.
 * kb_pool_kv_status returns the flags of every append that has completed
 * (synchronize the appending stream first for an exact answer) and clears
 * them when `clear` != 0; the host shims raise ValueError on any flag.
 * KB_KV_NO_PAGE: a row whose slot or position lies outside the block table,
 * or whose page was never grown (kb_pages_grow), was skipped -- nothing is
 * written outside the pool. */
#define KB_KV_V_OVERFLOW 1u
#define KB_KV_V_UNDERFLOW 2u
#define KB_KV_NO_PAGE 4u
int kb_pool_kv_status(kb_pool* pool, uint32_t* flags, int32_t clear);
/* Decode: q [nseq][n_q_heads][head_dim] bf16, one query token per sequence
 * attending to ctx_lens[i] cached tokens of slot slots[i] (including its
 * own, already appended).  out [nseq][n_q_heads][head_dim] bf16.
 * workspace: workspace_bytes >= kb_decode_workspace_bytes(nseq, ...) bytes of
 * device scratch (KB_EINVAL otherwise: its layout grows with nseq).  The work
 * plan (KV splits, item order) depends only on ctx_lens and
 * slots: with flags & KB_DECODE_REUSE_PLAN the plan already in `workspace`
 * (from an earlier call with the same ctx_lens and slots, e.g. the previous
 * layer of the same decode step) is reused and no plan kernel runs.  Such a
 * launch (programmatic dependent launch) reads the plan, the block tables
 * and every K/V row but each sequence's newest token BEFORE its
 * griddepcontrol.wait: those must have been written by work that completed
 * before the immediately preceding kernel on `stream` started -- true for
 * any ordinary kernel, memcpy or event wait in between; of this library's
 * kernels that let their successor start early, kv_append writes only the
 * newest token's row and decode / combine write only their outputs and
 * workspace.  q, slots and ctx_lens are read after the wait. */
#define KB_DECODE_REUSE_PLAN 1
/* The KV splits of a (sequence, kv head) merge inside the attention kernel
 * (a dedicated merge warp) from half a pair per SM up, and in a combine
 * launch for smaller batches;
 * flags & KB_DECODE_COMBINE / KB_DECODE_FUSE force either (A/B, tests). */
#define KB_DECODE_COMBINE 2
#define KB_DECODE_FUSE 4
int64_t kb_decode_workspace_bytes(int32_t nseq, int32_t n_q_heads, int32_t max_splits);
int kb_paged_decode(kb_pool* pool, int32_t layer, int32_t n_q_heads, uint64_t q,
                    uint64_t slots, uint64_t ctx_lens, int32_t nseq, int32_t max_ctx,
                    float scale, uint64_t out, uint64_t workspace, int64_t workspace_bytes,
                    int32_t max_splits, int32_t flags, uintptr_t stream);
/* Chunked prefill: for sequence i, q rows [q_off[i], q_off[i]+q_len[i]) are
 * positions [prefix[i], prefix[i]+q_len[i]) of slot slots[i]; they attend
 * causally over pages [0, prefix[i]+q_len[i]) (the chunk's K/V must be
 * appended first).  q/out: [total_q][n_q_heads][head_dim] bf16.
 * kv_splits > 1 splits every (sequence, 256-row tile, head) unit's key range
 * into that many CTAs (wave balance on 148 SMs) whose partials a combine
 * kernel merges; it needs kb_prefill_workspace_bytes() of device scratch. */
int64_t kb_prefill_workspace_bytes(int32_t nseq, int32_t n_q_heads, int32_t max_q_len,
                                   int32_t kv_splits);
int kb_paged_prefill(kb_pool* pool, int32_t layer, int32_t n_q_heads, uint64_t q,
                     uint64_t slots, uint64_t q_off, uint64_t q_len, uint64_t prefix,
                     int32_t nseq, int32_t max_q_len, float scale, uint64_t out,
                     uint64_t workspace, int32_t kv_splits, uintptr_t stream);

/* ---- parity at production sizes -------------------------------------- */
/* Position-sensitive content hash of nseg device segments of seg_bytes
 * bytes (16-byte aligned, multiple of 16): segment i starts at
 * base + seg_index[i] * seg_bytes (seg_index: device int64 array, or 0 for
 * i itself).  out (device uint64[nseg]) receives
 *   H = fmix(S ^ seg_bytes),  S = sum_j fmix(w_j ^ j * 0x9E3779B97F4A7C15)
 * over the segment's little-endian uint64 words w_j (fmix = splitmix64's
 * finalizer).  Used to compare whole slabs and every KV page against their
 * expected contents without host copies; oracle/kvpool.py restates it. */
int kb_hash_segments(uint64_t base, int64_t seg_bytes, uint64_t seg_index, int32_t nseg,
                     uint64_t out, uintptr_t stream);

/* ---- decoder-layer elementwise ops for the device-backed engine --------- */
/* Stage execution of a pipeline member (engine.py:389-397 charges its time):
 * x (+)= res in place (res may be 0), out = rmsnorm(x) * w; bf16 rows of
 * `hidden` elements.  And the SwiGLU: out[r, :] = silu(gu[r, :F]) * gu[r, F:]. */
int kb_add_rmsnorm(uint64_t x, uint64_t res, uint64_t w, uint64_t out, int32_t n,
                   int32_t hidden, float eps, uintptr_t stream);
int kb_silu_mul(uint64_t gu, uint64_t out, int32_t n, int32_t ffn, uintptr_t stream);

#ifdef __cplusplus
}
#endif
#endif /* KUNSERVE_B200_H */
