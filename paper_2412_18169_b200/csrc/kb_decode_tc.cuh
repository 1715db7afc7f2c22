// tcgen05 / TMA paged decode attention: persistent CTAs over length-sorted
// (sequence, kv head, KV split) work items.
//
// Orientation: tokens on the MMA M dimension so the tensor core sees a real
// 128-row tile even though a GQA group has only 4-5 query heads:
//   S^T[128 tok x 16]  = K_tile[128 tok x 128 d] . Q^T[128 d x 16 heads]
//   O^T[128 d x 16]   += V^T[128 d x 128 tok] . P^T[128 tok x 16 heads]
// Query heads >= G are padding.  The V cache is fp16 (kb_append.cu), so P
// enters P.V as fp16 (11-bit mantissa).
// K/V tiles are two 64-token pages (block_tokens 64) or one 128-token page,
// staged by TMA with 128-byte swizzle straight from the pool pages named by
// the block table; V is read as an MN-major operand (no transpose pass).
// S and O live in TMEM (double-buffered); the online softmax runs on 4
// warps, one token (for S) and one head_dim lane (for O) per thread.
//
// Scheduling: a one-CTA plan kernel (kb_decode.cu) splits long sequences so
// every work item has at most T tiles -- T balancing the work over two items
// per persistent CTA -- and orders items longest first.  CTA b starts with
// item b, then fetches the next index from a per-layer counter (greedy
// longest-processing-time) three tiles before its current item's last
// load, so the CTAs that finish first take the next items; the producer
// copies each item into a shared-memory ring for the MMA and softmax warps.  The TMA -> MMA ->
// softmax pipeline runs continuously across items (the next item's Q is
// staged one tile into the current one, and an item's epilogue runs after
// the next item's first P is out), so HBM streaming never drains between
// sequences.  With a reused plan the first item's loads start before
// griddepcontrol.wait.
//
// Warp roles (192 threads): 0-3 softmax / epilogue, 4 TMA producer,
// 5 MMA issuer + TMEM owner; the merge-warp build adds 6 split merger and
// 7 work-item claims (256 threads).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "kb_common.cuh"
#include "kb_sm100.cuh"

namespace kb {

constexpr int kDecStages = 3;
// Two instantiations per page size: kMW (the batch merges its KV splits in
// the kernel) adds a seventh warp that does the merging -- the fence, the
// counter round trip and the partial loads leave the softmax warps, and no
// combine launch follows the layer; without it (small batches, where a
// combine launch is cheaper than merges in the kernel's tail) the CTA keeps
// its six warps and register budget (r4: the 224-thread build was 2-6%
// slower at 4-16 sequences in combine mode).
// KB_DEC_CLAIM_WARP (merge-warp builds): an eighth warp takes the lazy
// claims (counter atomic + item load) off the TMA producer, which only
// signals a request -- the producer never blocks on a claim's round trips
// (r5 A/B, us per Llama layer at 16 / 32 / 64 / 147 sequences: 24.25 /
// 33.80 / 70.62 / 177.04 without, 24.05 / 33.65 / 70.41 / 177.17 with)
#ifndef KB_DEC_CLAIM_WARP
#define KB_DEC_CLAIM_WARP 1
#endif
constexpr int dec_threads(bool mw) { return mw ? (KB_DEC_CLAIM_WARP ? 256 : 224) : 192; }
constexpr int kMRing = 8;  // merge jobs in flight per CTA
constexpr int kTileTok = 128;
constexpr int kStageBytes = 65536;       // K (32 KiB) + V (32 KiB) for 128 tokens
constexpr int kHalfBytes = 16384;        // one 64-wide d-half of a 128-token tile
constexpr int kQBytes = 4096;            // 16 rows x 128 d bf16, SW128 K-major
constexpr int kPBytes = 4096;            // 16 rows x 128 tok bf16, SW128 K-major
constexpr int kDecMiscBytes = 2048;
constexpr int kDecSmem = kDecStages * kStageBytes + 2 * kQBytes + 2 * kPBytes + kDecMiscBytes + 1024;
constexpr uint32_t kDecTmemCols = 64;    // S0 S1 O0 O1, 16 columns each
constexpr int kRing = 16;                // work items published ahead per CTA
// KB_DEC_LAZY_D > 0: claim item r+1 at item r's tile nt - D (producer) and
// read it / load its Q at tile nt - DS (softmax); 0: the round-4 scheme
// (item 1 claimed at the start, then two items ahead).  r5 A/B, us per
// Llama layer at 4 / 16 / 32 / 64 / 147 sequences: 0: 10.59 / 25.09 /
// 34.61 / 72.47 / 178.78; D = DS = 3: 10.54 / 24.33 / 33.96 / 70.99 /
// 178.00 (kept); 4: 10.53 / 24.37 / 34.16 / 70.85 / 177.22; 5: 10.52 /
// 24.98 / 34.10 / 71.19 / 177.64; 1: 10.39 / 24.62 / 35.05 / 72.95 / 180.63
// KB_DEC_BT_PREFETCH: prefetch a published item's first block-table line
// into L1 (r5 A/B: within +-0.2% at 4-147 sequences -- the border's page
// lookup is not what an extra item costs; off)
#ifndef KB_DEC_BT_PREFETCH
#define KB_DEC_BT_PREFETCH 0
#endif
#ifndef KB_DEC_LAZY_D
#define KB_DEC_LAZY_D 3
#endif
#ifndef KB_DEC_LAZY_DS
#define KB_DEC_LAZY_DS KB_DEC_LAZY_D
#endif

// one KV split of a (sequence, kv head) pair: tiles [t_beg, t_beg + nt);
// the slot, context length and the pair's split count ride along (no
// dependent global load before the item's first TMA or in its epilogue)
struct DecodeItem {
  int32_t seq, h, split, t_beg, nt, slot, ctx, ns;
};

struct DecodeMisc {
  uint64_t full[kDecStages];
  uint64_t empty[kDecStages];
  uint64_t s_full[2];
  uint64_t o_full[2];
  uint64_t p_full[2];
  uint64_t q_full[2];
  uint64_t ring_full[kRing];   // item index published by the producer
  uint64_t ring_empty[kRing];  // MMA warp + softmax done with the item
  DecodeItem ring_it[kRing];   // the published items (nt < 0: no more work)
  uint64_t m_full[kMRing];   // merge job published by the softmax warps
  uint64_t m_empty[kMRing];  // merge warp has read the job
  int4 m_job[kMRing];        // {seq, h, ns, 1}; {.., 0}: no more jobs
  uint64_t creq;             // claim requests, producer -> claim warp
  uint32_t tmem_base;
  int32_t last;  // this CTA finished the last split of its (sequence, kv head)
  float red[2][4][8];
  float lred[4][8];
};

// KB_DEC_TRACE (variant builds only, tools/decode_trace_probe.py): per-CTA
// %globaltimer stamps of the kernel's phases, read back by kb_debug_dec_trace
#ifdef KB_DEC_TRACE
constexpr int kTraceSlots = 16;
__device__ unsigned long long g_dec_trace[1024 * kTraceSlots];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#ifdef KB_DEC_TRACE_CHAIN
// chain mode (tools/decode_chain_trace.py): one row of CTAs per layer 0..5
#define DEC_TRACE_ROW (((layer % 6) * (int)gridDim.x + (int)blockIdx.x) * kTraceSlots)
#else
#define DEC_TRACE_ROW ((int)blockIdx.x * kTraceSlots)
#endif
#define DEC_TRACE(slot) (g_dec_trace[DEC_TRACE_ROW + (slot)] = gtimer())
#define DEC_TRACE_VAL(slot, v) (g_dec_trace[DEC_TRACE_ROW + (slot)] = (v))
#else
#define DEC_TRACE(slot) ((void)0)
#define DEC_TRACE_VAL(slot, v) ((void)0)
#endif

template <int kB, bool kMW>
__global__ void __launch_bounds__(dec_threads(kMW), 1)
decode_tc_kernel(const __grid_constant__ CUtensorMap tmap, const __nv_bfloat16* __restrict__ q,
                 const int32_t* __restrict__ bt, const DecodeItem* __restrict__ items,
                 const int32_t* __restrict__ n_items_ptr, int32_t* __restrict__ item_counter,
                 const int32_t* __restrict__ nsplit_of, int32_t* __restrict__ split_done,
                 int nseq, int fuse_merge, __nv_bfloat16* __restrict__ out,
                 float* __restrict__ part_o,
                 float* __restrict__ part_ml, int Hkv, int G, int Hq, int L, int maxp, int layer,
                 int max_splits, float scale_log2, int early_loads) {
  using namespace sm100;
  // Work items are sorted longest first and handed out dynamically: CTA b
  // starts with item b, then its producer warp takes the next index from a
  // per-layer global counter (a greedy longest-processing-time schedule, so
  // the CTAs finish within one short item of each other) and publishes it
  // to the MMA and softmax warps through a small shared-memory ring.
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) DEC_TRACE(0);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem + kDecStages * kStageBytes;  // two buffers (item parity)
  uint8_t* sP = sQ + 2 * kQBytes;  // two buffers (tile parity)
  DecodeMisc* misc = reinterpret_cast<DecodeMisc*>(sP + 2 * kPBytes);
  static_assert(sizeof(DecodeMisc) <= kDecMiscBytes, "DecodeMisc outgrew its smem slot");

  if (warp == 5) {
    if (lane == 0) {
      for (int s = 0; s < kDecStages; ++s) {
        mbar_init(&misc->full[s], 1);
        mbar_init(&misc->empty[s], 1);
      }
      for (int b = 0; b < 2; ++b) {
        mbar_init(&misc->s_full[b], 1);
        mbar_init(&misc->o_full[b], 1);
        mbar_init(&misc->q_full[b], 128);
        mbar_init(&misc->p_full[b], 128);
      }
      for (int r = 0; r < kRing; ++r) {
        mbar_init(&misc->ring_full[r], 1);
        mbar_init(&misc->ring_empty[r], 2);
      }
      for (int r = 0; r < kMRing; ++r) {
        mbar_init(&misc->m_full[r], 1);
        mbar_init(&misc->m_empty[r], 1);
      }
      mbar_init(&misc->creq, 1);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(&misc->tmem_base, kDecTmemCols);
  }
  if (warp == 4 && lane == 0) tma_prefetch_desc(&tmap);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = misc->tmem_base;
  constexpr int kPPT = kTileTok / kB;  // pages per tile
  // issue the TMA loads of tile t of item `it` into stage j % kDecStages
  auto issue_tile = [&](const DecodeItem& it, int t, int j) {
    const int stage = j % kDecStages;
    const int tile = it.t_beg + t;
    const int32_t* bt_row = bt + ((int64_t)it.slot * L + layer) * maxp;
    int npg = 0;
    int32_t pages[kPPT];
#pragma unroll
    for (int k = 0; k < kPPT; ++k) {
      const int pi = tile * kPPT + k;
      pages[k] = (pi * kB < it.ctx) ? bt_row[pi] : -1;
      npg += pages[k] >= 0;
    }
    mbar_arrive_expect_tx(&misc->full[stage], (uint32_t)(npg * kB * 512));
    uint8_t* sK = smem + stage * kStageBytes;
    uint8_t* sV = sK + 2 * kHalfBytes;
#pragma unroll
    for (int k = 0; k < kPPT; ++k) {
      if (pages[k] < 0) continue;
      const int rk = ((pages[k] * 2 + 0) * Hkv + it.h) * kB;
      const int rv = ((pages[k] * 2 + 1) * Hkv + it.h) * kB;
      const int off = k * kB * 128;
      tma_load_2d(sK + off, &tmap, 0, rk, &misc->full[stage]);
      tma_load_2d(sK + kHalfBytes + off, &tmap, 64, rk, &misc->full[stage]);
      tma_load_2d(sV + off, &tmap, 0, rv, &misc->full[stage]);
      tma_load_2d(sV + kHalfBytes + off, &tmap, 64, rv, &misc->full[stage]);
    }
  };
  // item r of this CTA (every role reads the ring in the same order; the
  // producer copies each item into the ring, so no role loads an item from
  // global memory at an item border)
  auto get_item = [&](int r, DecodeItem& it) -> bool {
    const int slot = r % kRing;
    mbar_wait(&misc->ring_full[slot], (r / kRing) & 1);
    it = misc->ring_it[slot];
    return it.nt > 0;
  };
  // Producer state: items are published two ahead of the loads, so the
  // softmax can stage the next item's Q early.
  const bool producer = warp == 4 && lane == 0;
  int n_items = 0, npre = 0, published = 0;
  bool exhausted = false;
  // pre: the static first item, when the caller already loaded it
  auto publish = [&](const DecodeItem* pre = nullptr) {
    if (exhausted) return;
    const int r = published++;
    const int slot = r % kRing;
    if (r >= kRing) mbar_wait(&misc->ring_empty[slot], ((r / kRing) - 1) & 1);
    // the first item is static (no atomic round trip before the first
    // load); every CTA then makes exactly one failing fetch, and the last
    // of those re-arms the counter (a reused plan)
    const int grid = (int)gridDim.x;
    int idx = r == 0 ? (int)blockIdx.x : -1;
    if (idx < 0 || idx >= n_items) {
      const int raw = atomicAdd(item_counter + layer, 1);
      if (idx < 0) idx = grid + raw;
      if (idx >= n_items) {
        if (raw == max(n_items - grid, 0) + grid - 1) item_counter[layer] = 0;
        idx = -1;
        exhausted = true;
      }
    }
    DecodeItem v{};
    v.nt = -1;
    if (idx >= 0) v = pre ? *pre : items[idx];
    misc->ring_it[slot] = v;
    mbar_arrive(&misc->ring_full[slot]);
#if KB_DEC_BT_PREFETCH
    // the item's first block-table entries into L1 now: its first tile's
    // page lookup at the item border is then an L1 hit, not an L2 round
    // trip behind a saturated memory system
    if (idx >= 0 && r > 0) {
      const int32_t* row = bt + ((int64_t)v.slot * L + layer) * maxp + v.t_beg * (kTileTok / kB);
      asm volatile("prefetch.global.L1 [%0];" ::"l"(row));
    }
#endif
  };
  // Launched with programmatic stream serialization: the prologue above
  // overlapped the previous kernel's tail.  With a reused plan
  // (early_loads) the producer also publishes its static first item and
  // starts that item's loads before griddepcontrol.wait: the plan, the
  // block tables and every K/V row but the newest token's were written by
  // grids that completed before the previous launch could start (only
  // kv_append, the usual predecessor, writes K/V -- the newest token's row,
  // which no tile loaded here holds).  q and the counters are read after it.
  if (early_loads && producer) {
    // the item count and the static first item load together (one global
    // round trip less before the first TMA); the plan never holds more than
    // nseq * Hkv * max_splits items, so the speculative read stays in it
    const bool spec = (int)blockIdx.x < nseq * Hkv * max_splits;
    DecodeItem first{};
    if (spec) first = items[blockIdx.x];
    n_items = *n_items_ptr;
    if ((int)blockIdx.x < n_items) {
      publish(spec ? &first : nullptr);
      DecodeItem it0;
      get_item(0, it0);
      // tiles [0, nsafe) end before the newest token (position ctx - 1)
      const int nsafe = (it0.ctx - 1) / kTileTok - it0.t_beg;
      npre = min(min(it0.nt, kDecStages), max(nsafe, 0));
      for (int t = 0; t < npre; ++t) issue_tile(it0, t, t);
      if (npre) DEC_TRACE(3);
    }
  }
  // everything below may read what the previous grid wrote (q, the newest
  // K/V rows, the previous layer's workspace use, a fresh plan)
  pdl_wait();
  pdl_launch_dependents();
  if (tid == 0) DEC_TRACE(1);
  if (producer && published == 0) n_items = *n_items_ptr;

  if (warp == 4) {
    // ------------------------------------------------ TMA producer
    if (lane == 0 && KB_DEC_LAZY_D > 0) {
      // Lazy claims: item r+1 is claimed and published while item r's tile
      // nt - KB_DEC_LAZY_D is issued -- one item ahead, late in the current
      // one -- so the CTAs that finish first take the next items (a
      // longest-processing-time queue), instead of every CTA holding two
      // items claimed at its start.
      if (published == 0) publish();  // item 0
      int j = 0;
      for (int r = 0;; ++r) {
        DecodeItem it;
        if (!get_item(r, it)) break;
        if (r == 0) DEC_TRACE(2);
        const int pub_t = max(it.nt - KB_DEC_LAZY_D, 0);
        for (int t = 0; t < it.nt; ++t, ++j) {
          if (!(r == 0 && t < npre)) {  // else issued before griddepcontrol.wait
            const int stage = j % kDecStages;
            if (j >= kDecStages) mbar_wait(&misc->empty[stage], ((j / kDecStages) - 1) & 1);
            issue_tile(it, t, j);
            if (j == 0) DEC_TRACE(3);
          }
          if (t == pub_t) {  // item r + 1
            if (kMW && KB_DEC_CLAIM_WARP)
              mbar_arrive(&misc->creq);
            else
              publish();
          }
        }
      }
    } else if (lane == 0) {
      if (published == 0) publish();  // item 0; item 1 once item 0's first loads are out
      bool second = npre > 0;
      if (second) publish();
      int j = 0;  // global tile counter of this CTA
      for (int r = 0;; ++r) {
        DecodeItem it;
        if (!get_item(r, it)) break;
        if (r == 0) DEC_TRACE(2);
        for (int t = 0; t < it.nt; ++t, ++j) {
          if (r == 0 && t < npre) continue;  // issued before griddepcontrol.wait
          const int stage = j % kDecStages;
          if (j >= kDecStages) mbar_wait(&misc->empty[stage], ((j / kDecStages) - 1) & 1);
          issue_tile(it, t, j);
          if (j == 0) DEC_TRACE(3);
          if (!second) {
            second = true;
            publish();
          }
        }
        publish();
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------ MMA issuer
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);  // warp-uniform MMA operands
    constexpr uint32_t kIdQK = idesc_bf16_f32(128, 16, false, false);
    constexpr uint32_t kIdPV = idesc_f16_f32(128, 16, true, false);  // V^T fp16, P^T fp16
    const uint32_t p_base = smem_u32(sP);
    // QK cursor runs one tile ahead of the PV cursor, across item borders
    int qr = 0, qt = 0, qj = 0;
    DecodeItem qit;
    bool qvalid = get_item(0, qit);
    auto issue_next_qk = [&]() -> bool {
      while (qvalid && qt >= qit.nt) {
        ++qr;
        qt = 0;
        qvalid = get_item(qr, qit);
      }
      if (!qvalid) return false;
      if (qt == 0) mbar_wait(&misc->q_full[qr & 1], (qr >> 1) & 1);
      const int stage = qj % kDecStages;
      mbar_wait(&misc->full[stage], (qj / kDecStages) & 1);
      tc_fence_after();
      if (lane == 0 && qj == 0) DEC_TRACE(4);
      if (lane == 0) {
        // A = K tile (d-halves 16 KiB apart), B = Q (d-halves 2 KiB apart)
        mma_ss_8<2, 4, 6, 1024, 1026, 1028, 1030, 2, 4, 6, 128, 130, 132, 134>(
            tm + (qj & 1) * 16, sw128_desc(smem_u32(smem + stage * kStageBytes), 16, 1024),
            sw128_desc(smem_u32(sQ + (qr & 1) * kQBytes), 16, 1024), kIdQK, 0u);
        mma_commit(&misc->s_full[qj & 1]);
      }
      __syncwarp();
      ++qt;
      ++qj;
      return true;
    };
    issue_next_qk();
    int j = 0;
    for (int r = 0;; ++r) {
      DecodeItem cur;
      if (!get_item(r, cur)) break;
      const int nt = cur.nt;
      for (int t = 0; t < nt; ++t, ++j) {
        issue_next_qk();
        mbar_wait(&misc->p_full[j & 1], (j >> 1) & 1);
        tc_fence_after();
        if (lane == 0) {
          const int stage = j % kDecStages;
          // A = V^T, MN-major (16 tokens = 2 KiB per step); B = P^T (halves 2 KiB apart)
          mma_ss_8<128, 256, 384, 512, 640, 768, 896, 2, 4, 6, 128, 130, 132, 134>(
              tm + 32 + (j & 1) * 16,
              sw128_desc(smem_u32(smem + stage * kStageBytes + 2 * kHalfBytes), kHalfBytes, 1024),
              sw128_desc(p_base + (j & 1) * kPBytes, 16, 1024), kIdPV, 0u);
          mma_commit(&misc->o_full[j & 1]);
          mma_commit(&misc->empty[stage]);
        }
        __syncwarp();
      }
      if (lane == 0) mbar_arrive(&misc->ring_empty[r % kRing]);  // done with item r
      __syncwarp();
    }
  } else if (kMW && KB_DEC_CLAIM_WARP && warp == 7) {
    // ------------------------------------------------ claims (items >= 1)
    if (lane == 0 && KB_DEC_LAZY_D > 0) {
      n_items = *n_items_ptr;
      published = 1;  // item 0 is the producer's
      mbar_wait(&misc->ring_full[0], 0);
      if (misc->ring_it[0].nt > 0) {
        for (int k = 0;; ++k) {
          mbar_wait(&misc->creq, k & 1);
          publish();
          if (exhausted) break;
        }
      }
    }
  } else if (kMW && warp == 6) {
    // ------------------------------------------------ split merger
    // Jobs come from the softmax warps once a split's partial (O / l, m, l
    // rows) is written.  Lane 0 publishes it GPU-wide and counts the pair's
    // finished splits (threadfence-reduction: the fence is cumulative over
    // the softmax threads' stores, ordered before it by their named barrier
    // and the job's mbarrier); the CTA that finishes the last split merges
    // the pair, one float4 of the 128 head-dim lanes per lane, and re-arms
    // the counter for the next layer.
    for (int k = 0;; ++k) {
      const int slot = k % kMRing;
      mbar_wait(&misc->m_full[slot], (k / kMRing) & 1);
      const int4 job = misc->m_job[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&misc->m_empty[slot]);
      if (!job.w) break;
      const int seq = job.x, h = job.y, ns = job.z;
      int32_t* done = split_done + seq * Hkv + h;
      int last = 0;
      if (lane == 0) {
#ifdef KB_DEC_MERGE_FENCES
        __threadfence();
        last = atomicAdd(done, 1) == ns - 1;
#else
        // one acq_rel atomic instead of fence / relaxed add / fence: its
        // release half publishes the split's partial rows (cumulative over
        // the softmax threads' stores, ordered before this lane by their
        // barrier and the job's mbarrier), its acquire half makes the other
        // splits' rows visible to the merger
        int old;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                     : "=r"(old) : "l"(done) : "memory");
        last = old == ns - 1;
#endif
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (!last) continue;
#ifdef KB_DEC_MERGE_FENCES
      __threadfence();
#else
      __syncwarp();  // lanes 1-31 read after lane 0's acquire (warp-synchronous)
#endif
      // every load of the merge is issued before its first use: the (m, l)
      // of split s for all G rows by lane s, then the partial O rows four
      // splits at a time -- two or three L2 round trips, not one per split
      const int64_t row0 = ((int64_t)seq * Hq + h * G) * max_splits;  // row of (g=0, split 0)
      float mg[8], wl[8];
      float mstar[8], lsum[8];
      float4 acc[8];
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        mstar[g] = -INFINITY;
        lsum[g] = 0.f;
        acc[g] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      for (int s0 = 0; s0 < ns; s0 += 32) {
        const int sidx = s0 + lane;
        float lg[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          mg[g] = -INFINITY;
          lg[g] = 0.f;
          if (g < G && sidx < ns) {
            const float2 ml = __ldcg(reinterpret_cast<const float2*>(
                part_ml + (row0 + (int64_t)g * max_splits + sidx) * 2));
            mg[g] = ml.x;
            lg[g] = ml.y;
          }
        }
        // this chunk's maxima, then weights relative to the running max
        // (chunks of 32 splits only when max_splits > 32)
        float cm[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          float v = mg[g];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
          cm[g] = v;
        }
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          const float mn = fmaxf(mstar[g], cm[g]);
          const float sc = (mn == -INFINITY) ? 1.f : exp2f(mstar[g] - mn);  // rescale what we have
          lsum[g] *= sc;
          acc[g].x *= sc;
          acc[g].y *= sc;
          acc[g].z *= sc;
          acc[g].w *= sc;
          mstar[g] = mn;
          wl[g] = (mg[g] == -INFINITY) ? 0.f : exp2f(mg[g] - mn);
          float lw = wl[g] * lg[g];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) lw += __shfl_xor_sync(0xffffffffu, lw, o);
          lsum[g] += lw;
        }
        const int cnt = min(32, ns - s0);
        for (int i0 = 0; i0 < cnt; i0 += 4) {
          float4 v[4][8];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int g = 0; g < 8; ++g)
              v[i][g] = (g < G && i0 + i < cnt)
                            ? __ldcg(reinterpret_cast<const float4*>(
                                  part_o + (row0 + (int64_t)g * max_splits + s0 + i0 + i) * 128) +
                                     lane)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int g = 0; g < 8; ++g) {
              const float wi = __shfl_sync(0xffffffffu, wl[g], (i0 + i) & 31);
              acc[g].x += wi * v[i][g].x;
              acc[g].y += wi * v[i][g].y;
              acc[g].z += wi * v[i][g].z;
              acc[g].w += wi * v[i][g].w;
            }
        }
      }
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        if (g >= G) break;
        const int64_t hrow = (int64_t)seq * Hq + h * G + g;
        const float inv = lsum[g] > 0.f ? 1.f / lsum[g] : 0.f;
        __nv_bfloat162 b01 = __floats2bfloat162_rn(acc[g].x * inv, acc[g].y * inv);
        __nv_bfloat162 b23 = __floats2bfloat162_rn(acc[g].z * inv, acc[g].w * inv);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&b01);
        pk.y = *reinterpret_cast<uint32_t*>(&b23);
        reinterpret_cast<uint2*>(out + hrow * 128)[lane] = pk;
      }
      if (lane == 0) *done = 0;
    }
  } else {
    // ------------------------------------------------ softmax / epilogue (tid < 128)
    // Q of an item: G rows (<= 8) x 16 chunks of 16 bytes, two per thread;
    // loaded into registers early, stored (SW128 K-major) when the buffer
    // is free, so the global load never sits on the softmax's critical path
    int4 qv[2];
    auto load_q = [&](const DecodeItem& it) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int c = tid + k * 128, g = c >> 4, chunk = c & 15;
        qv[k] = g < G ? reinterpret_cast<const int4*>(
                            q + ((int64_t)it.seq * Hq + it.h * G + g) * 128)[chunk]
                      : make_int4(0, 0, 0, 0);
      }
    };
    auto store_q = [&](int r) {
      uint8_t* dst = sQ + (r & 1) * kQBytes;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int c = tid + k * 128, g = c >> 4, chunk = c & 15;
        const uint32_t off = (chunk >> 3) * 2048 + g * 128 + ((((chunk & 7) ^ (g & 7)) & 7) << 4);
        *reinterpret_cast<int4*>(dst + off) = qv[k];
      }
      fence_proxy_async_smem();
      mbar_arrive(&misc->q_full[r & 1]);
    };
    // both P buffers start zero: rows >= 8 (GQA padding) are never written
    for (int c = tid; c < 2 * kPBytes / 16; c += 128)
      reinterpret_cast<int4*>(sP)[c] = make_int4(0, 0, 0, 0);
    int mjobs = 0;  // merge jobs handed to the merge warp (tid 0 counts)
    DecodeItem it, nxt;
    bool have = get_item(0, it), nhave = false;
    if (have) {
      load_q(it);
      store_q(0);
    }
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    int j = 0;
    // Running state of the current item and of the previous ("pending")
    // item, whose epilogue is deferred until the next item's first P is
    // out: the tensor core and the TMA loads never wait on an item border.
    float m_run[8], l_part[8], o_acc[8], alpha0[8], alpha1[8];  // alpha by tile parity
    float pm[8], pl[8], po[8];
    bool pend = false;
    DecodeItem pit{};
    int pr = 0;
    // O of tile x is folded two tiles later (or at the item's end), so the
    // softmax never waits on the P.V it has just released:
    //   acc = acc * alpha_x + O_x,  alpha_x = exp2(m_{x-1} - m_x)
    auto fold = [&](int x, float (&acc)[8]) {
      mbar_wait(&misc->o_full[x & 1], (x >> 1) & 1);
      tc_fence_after();
      float ov[8];
      tmem_ld_32x32b_x8(tmem + lane_base + 32 + (x & 1) * 16, ov);
#pragma unroll
      for (int g = 0; g < 8; ++g) acc[g] = acc[g] * ((x & 1) ? alpha1[g] : alpha0[g]) + ov[g];
    };
    // the pending item's epilogue (its O fully folded): normalise or write
    // the split partials, merge (fused mode), release its ring slot
    auto finalize = [&]() {
      // l = sum over the 128 token lanes
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        float v = pl[g];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) misc->lred[warp][g] = v;
      }
      named_bar_sync(1, 128);
      const int ns = pit.ns;  // (a global load here sat on the softmax's path)
      for (int g = 0; g < G; ++g) {
        const float l = misc->lred[0][g] + misc->lred[1][g] + misc->lred[2][g] + misc->lred[3][g];
        const int64_t hrow = (int64_t)pit.seq * Hq + pit.h * G + g;
        if (ns == 1) {  // no merge needed
          out[hrow * 128 + tid] = __float2bfloat16(l > 0.f ? po[g] / l : 0.f);
        } else {
          const int64_t row = hrow * max_splits + pit.split;
          part_o[row * 128 + tid] = po[g];
          if (tid == 0) {
            part_ml[row * 2] = pm[g];
            part_ml[row * 2 + 1] = l;
          }
        }
      }
      if (kMW && ns > 1) {
        // hand the split to the merge warp (its partial rows are written)
        named_bar_sync(1, 128);
        if (tid == 0) {
          const int slot = mjobs % kMRing;
          if (mjobs >= kMRing) mbar_wait(&misc->m_empty[slot], ((mjobs / kMRing) - 1) & 1);
          misc->m_job[slot] = make_int4(pit.seq, pit.h, ns, 1);
          mbar_arrive(&misc->m_full[slot]);
        }
        ++mjobs;
      }
      named_bar_sync(1, 128);  // lred / last are reused by the next item
      if (tid == 0) {
        if (pr < 3) DEC_TRACE(6 + pr);
        DEC_TRACE(9);
        DEC_TRACE_VAL(11, (unsigned long long)(pr + 1));
        mbar_arrive(&misc->ring_empty[pr % kRing]);  // done with item pr
      }
      pend = false;
    };
    auto to_pending = [&](int r) {
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        pm[g] = m_run[g];
        pl[g] = l_part[g];
        po[g] = o_acc[g];
      }
      pit = it;
      pr = r;
      pend = true;
    };
    for (int r = 0; have; ++r) {
      // Q of item r+1 goes into the buffer item r-1 used (its QKs are done):
      // the item is read from the ring after this item's first tile (the
      // producer publishes it once this item's loads are out, so the
      // softmax never waits on it), Q loaded then and stored one tile later
      int q_state = 0;  // 0: item r+1 not read yet, 1: Q loaded, 2: stored / none
      const int ctx = it.ctx;
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        m_run[g] = -INFINITY;
        l_part[g] = 0.f;
        o_acc[g] = 0.f;
      }
      for (int t = 0; t < it.nt; ++t, ++j) {
        const int tile = it.t_beg + t;
        const int valid = min(kTileTok, ctx - tile * kTileTok);
        mbar_wait(&misc->s_full[j & 1], (j >> 1) & 1);
        tc_fence_after();
        if (tid == 0 && j == 0) DEC_TRACE(5);
        float s[8];
        tmem_ld_32x32b_x8(tmem + lane_base + (j & 1) * 16, s);
        const bool ok = tid < valid;
#pragma unroll
        for (int g = 0; g < 8; ++g) s[g] = (ok && g < G) ? s[g] * scale_log2 : -INFINITY;
        float mx[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          float v = s[g];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
          mx[g] = v;
        }
        if (lane == 0) {
#pragma unroll
          for (int g = 0; g < 8; ++g) misc->red[j & 1][warp][g] = mx[g];
        }
        named_bar_sync(1, 128);
        // O of tile j-2 (same TMEM O / P buffers as tile j): fold it first
        // (the pending item's second-to-last tile at this item's start)
        if (t >= 2)
          fold(j - 2, o_acc);
        else if (t == 0 && pend && pit.nt >= 2)
          fold(j - 2, po);
        float p[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          const float tm = fmaxf(fmaxf(misc->red[j & 1][0][g], misc->red[j & 1][1][g]),
                                 fmaxf(misc->red[j & 1][2][g], misc->red[j & 1][3][g]));
          const float m_new = fmaxf(m_run[g], tm);
          float alpha;
          if (m_new == -INFINITY) {
            alpha = 1.f;
            p[g] = 0.f;
          } else {
            alpha = exp2f(m_run[g] - m_new);
            p[g] = exp2f(s[g] - m_new);
          }
          if (j & 1)
            alpha1[g] = alpha;
          else
            alpha0[g] = alpha;
          l_part[g] = l_part[g] * alpha + p[g];
          m_run[g] = m_new;
        }
        if (valid < kTileTok) {
          // partial last tile: zero V rows past the context so 0 * garbage
          // cannot reach the accumulator
          const int stage = j % kDecStages;
          mbar_wait(&misc->full[stage], (j / kDecStages) & 1);
          if (tid >= valid) {
            uint8_t* sV = smem + stage * kStageBytes + 2 * kHalfBytes;
            int4* r0 = reinterpret_cast<int4*>(sV + tid * 128);
            int4* r1 = reinterpret_cast<int4*>(sV + kHalfBytes + tid * 128);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              r0[c] = make_int4(0, 0, 0, 0);
              r1[c] = make_int4(0, 0, 0, 0);
            }
          }
        }
        // P^T -> SW128 K-major image in buffer j&1, fp16 (rows 8..15 stay
        // zero).  PV of tile j-2 (same buffer) is done: it was folded above.
        uint8_t* pbuf = sP + (j & 1) * kPBytes + (tid >> 6) * 2048;
#pragma unroll
        for (int g = 0; g < 8; ++g)
          *reinterpret_cast<__half*>(pbuf + sw128_offset(g, tid & 63)) = __float2half_rn(p[g]);
        fence_proxy_async_smem();
        mbar_arrive(&misc->p_full[j & 1]);
        // the previous item's last O, then its epilogue, while P.V of this
        // tile runs
        if (t == 0 && pend) {
          fold(j - 1, po);
          finalize();
        }
        if (q_state == 1) {
          store_q(r + 1);
          q_state = 2;
        }
        if (q_state == 0 && t >= (KB_DEC_LAZY_D > 0 ? max(it.nt - KB_DEC_LAZY_DS, 0) : 0)) {
          nhave = get_item(r + 1, nxt);
          q_state = 2;
          if (nhave) {
            load_q(nxt);
            q_state = 1;
            if (t == it.nt - 1) {  // a one-tile item: store right away
              store_q(r + 1);
              q_state = 2;
            }
          }
        }
      }
      if (tid == 0) DEC_TRACE_VAL(12, (unsigned long long)j);
      to_pending(r);
      if (!nhave) {  // the CTA's last item: no next P to hide the epilogue behind
        if (it.nt >= 2) fold(j - 2, po);
        fold(j - 1, po);
        finalize();
      }
      it = nxt;  // item r+1, read from the ring during item r
      have = nhave;
    }
    if (kMW && tid == 0) {  // no more jobs
      const int slot = mjobs % kMRing;
      if (mjobs >= kMRing) mbar_wait(&misc->m_empty[slot], ((mjobs / kMRing) - 1) & 1);
      misc->m_job[slot] = make_int4(0, 0, 0, 0);
      mbar_arrive(&misc->m_full[slot]);
    }
    // sequences with no context have no item: their rows are zero
    for (int sq = blockIdx.x; sq < nseq; sq += gridDim.x)
      if (nsplit_of[sq] == 0)
        for (int h = 0; h < Hq; ++h) out[((int64_t)sq * Hq + h) * 128 + tid] = __float2bfloat16(0.f);
  }
  tc_fence_before();
  __syncthreads();
  if (tid == 0) DEC_TRACE(10);
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tmem, kDecTmemCols);
  }
}

inline int launch_decode_tc(kb_pool* p, int layer, int Hq, uint64_t q, int grid, float scale, float* part_o,
                            float* part_ml, const DecodeItem* items, const int32_t* n_items,
                            int32_t* item_counter, const int32_t* nsplit, int32_t* split_done,
                            int nseq, int fuse_merge, uint64_t out,
                            int max_splits, int early_loads, cudaStream_t st) {
  const int Hkv = p->m.n_kv_heads, B = p->m.block_tokens;
  const float scale_log2 = scale * 1.4426950408889634f;
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(dec_threads(fuse_merge != 0));
  cfg.dynamicSmemBytes = kDecSmem;
  cfg.stream = st;
  cfg.attrs = pdl;
  cfg.numAttrs = 1;
  auto go = [&](auto kernel) -> int {
    int rc = ensure_smem_attr(reinterpret_cast<const void*>(kernel), kDecSmem, p->device);
    if (rc) return rc;
    KB_RT(cudaLaunchKernelEx(&cfg, kernel,
        p->kv_tmap, reinterpret_cast<const __nv_bfloat16*>(q), p->d_bt, items, n_items, item_counter, nsplit, split_done, nseq, fuse_merge,
        reinterpret_cast<__nv_bfloat16*>(out), part_o,
        part_ml, Hkv,
        Hq / Hkv, Hq, p->m.num_layers, p->maxp, layer, max_splits, scale_log2, early_loads));
    return KB_OK;
  };
  int rc;
  if (B == 64) rc = fuse_merge ? go(decode_tc_kernel<64, true>) : go(decode_tc_kernel<64, false>);
  else rc = fuse_merge ? go(decode_tc_kernel<128, true>) : go(decode_tc_kernel<128, false>);
  if (rc) return rc;
  KB_LAUNCH_CHECK();
  return KB_OK;
}

}  // namespace kb
