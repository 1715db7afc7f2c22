// N8 (decode): paged decode attention over the (enlarged, non-contiguous)
// KV pool, GQA, head_dim 128, bf16 in / fp32 accumulate.
//
// The reference has no attention: its only trace is the
// cost proxy attention_units(c, p) = p*c + (c^2+c)/2
// (pkg/src/dropsim/costmodel.py:50-57).  Parity is against the fp32 CPU
// restatement oracle/attention.py with max-abs <= 2e-2, mean-rel <= 1e-3.
//
// Per layer: the persistent tcgen05 kernel (kb_decode_tc.cuh), which for
// large batches also merges the KV splits, else a split-KV combine launch;
// plus one plan launch (work items) per decode step, reused by every layer.
#include "kb_common.cuh"
#include "kb_decode_tc.cuh"

namespace kb {

constexpr int kPlanThreads = 1024;
constexpr int kMaxLayers = 256;  // per-layer work-item counters in the workspace
constexpr int kLenBuckets = 1024;
#ifndef KB_DEC_ITEMS_PER_CTA
#define KB_DEC_ITEMS_PER_CTA 2  // swept 1-8 on B200 with dynamic fetching: 1-2 best
#endif
constexpr int kItemsPerCta = KB_DEC_ITEMS_PER_CTA;  // target work items per persistent CTA
// ...except when the batch has 1.5-2.8 (sequence, kv head) pairs per CTA:
// two rounds then leave the pairs nearly unsplit and their lognormal lengths
// unbalanced; three items per CTA split the long ones (B200 sweep over four
// context draws, r3p: 32 sequences +1 to +9 pt of HBM, 40 about even; two
// stay better at <= 24 and >= 48 sequences)
#ifndef KB_DEC_ADAPT_IPC
#define KB_DEC_ADAPT_IPC 1
#endif
// lower bound of that range in eighths of a pair per CTA: 12 = 1.5 (r5:
// before the lazy claims 1.25 measured 3.3% faster at 24 Llama sequences
// over seven context draws; with them 1.5 is 2-10% faster there again)
#ifndef KB_DEC_IPC3_LO_X8
#define KB_DEC_IPC3_LO_X8 12
#endif
// upper bound in fifths of a pair per CTA: 14 = 2.8 (r5, with lazy claims:
// 48 Llama sequences (2.6 pairs per CTA) 0.6-5% faster with 3 items, 56
// (3.0) 2-3% slower; was 12 = 2.4)
#ifndef KB_DEC_IPC3_HI_X5
#define KB_DEC_IPC3_HI_X5 14
#endif
// ...and one item per CTA below half a pair per CTA (<= 9 Llama sequences:
// the items are then whole pairs of similar length, and a second round only
// adds a merge; r3r: +2 to +6 pt at 4-8 sequences, 2 items stay better at
// 12-24).  Twice the items-per-CTA target there, an A/B knob:
#ifndef KB_DEC_TINY_IPC_X2
#define KB_DEC_TINY_IPC_X2 2
#endif
// ...and between half a pair and one pair per CTA (A/B knob, doubled)
#ifndef KB_DEC_SUB1_IPC_X2
#define KB_DEC_SUB1_IPC_X2 (2 * KB_DEC_ITEMS_PER_CTA)
#endif
#ifndef KB_DEC_MIN_TILES
#define KB_DEC_MIN_TILES 2
#endif
constexpr int kMinTiles = KB_DEC_MIN_TILES;  // shortest split (128-token tiles)
#ifndef KB_DEC_UNEVEN
#define KB_DEC_UNEVEN 0
#endif
#ifndef KB_DEC_TSEARCH
#define KB_DEC_TSEARCH 1
#endif
// piece k of a pair of `tiles` tiles cut into s splits of target length T:
// even (k*tiles/s) or, KB_DEC_UNEVEN, T-long pieces and a short remainder
__device__ __forceinline__ void piece(int tiles, int s, int T, int k, int& beg, int& len) {
  if (KB_DEC_UNEVEN && s * T >= tiles) {
    beg = k * T;
    len = min(T, tiles - beg);
  } else {
    beg = k * tiles / s;
    len = (k + 1) * tiles / s - beg;
  }
}

// Split-KV combine for small batches: one CTA per (sequence, q head),
// thread = head_dim lane.  Sequences with 0 splits (no context) get a zero
// row, with 1 split the attention kernel wrote the row itself.
__global__ void decode_combine_kernel(const float* __restrict__ part_o,
                                      const float* __restrict__ part_ml,
                                      const int32_t* __restrict__ nsplit_of,
                                      __nv_bfloat16* __restrict__ out, int Hq, int max_splits) {
  // the next launch (the following layer's attention) may start its
  // prologue and its plan-safe early loads at once: they touch nothing this
  // grid or the attention grid before it writes, and its own
  // griddepcontrol.wait orders the rest after this grid
  sm100::pdl_launch_dependents();
  sm100::pdl_wait();  // the attention kernel's partials
  const int sh = blockIdx.x;  // seq * Hq + head
  const int seq = sh / Hq;
  const int ns = nsplit_of[seq];
  if (ns <= 1) return;
  const float* ml = part_ml + (int64_t)sh * max_splits * 2;
  float mstar = -INFINITY;
  for (int s = 0; s < ns; ++s) mstar = fmaxf(mstar, ml[2 * s]);
  float l = 0.f, o = 0.f;
  for (int s = 0; s < ns; ++s) {
    const float ms = ml[2 * s];
    const float w = ms == -INFINITY ? 0.f : exp2f(ms - mstar);
    l += w * ml[2 * s + 1];
    o += w * part_o[((int64_t)sh * max_splits + s) * 128 + threadIdx.x];
  }
  out[(int64_t)sh * 128 + threadIdx.x] = __float2bfloat16(l > 0.f ? o / l : 0.f);
}

// KB_DEC_REFINE: hand the item budget T leaves unused to the sequences with
// the longest pieces (one more split each).  Measured slower on B200 (r2y:
// 16 sequences 25.9 vs 25.6 us per layer, 4 sequences up to +2.5 us over
// three context draws) -- off; kept for A/B.
#ifndef KB_DEC_REFINE
#define KB_DEC_REFINE 0
#endif

// Block-wide inclusive scan (1024 threads); warp_sum is 32 ints of smem.
__device__ __forceinline__ int block_incl_scan(int v, int* warp_sum) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sum[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = warp_sum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_sum[lane] = t;
  }
  __syncthreads();
  const int r = (w ? warp_sum[w - 1] : 0) + x;
  __syncthreads();  // warp_sum is reused by the next call
  return r;
}

// KB_DEC_SPLITS_FIRST: the pieces of split pairs are handed out before every
// unsplit pair (each group longest first), so the in-kernel merges of the
// last splits run mid-kernel on the merge warp, not in the kernel's tail;
// 0: one longest-first order over all items.
#ifndef KB_DEC_SPLITS_FIRST
#define KB_DEC_SPLITS_FIRST 1
#endif
// histogram bucket of an item (bucket 0 is handed out first); sf: splits
// first (below two (sequence, kv head) pairs per CTA: r4 A/B 32 sequences
// 34.8 vs 36.0 us per Llama layer, 16: 25.1 vs 25.2; at 64 the plain order
// stays ahead, 72.6 vs 73.3)
__device__ __forceinline__ int item_bucket(int len, int nsplits, bool sf) {
  if (sf) {
    const int key = (nsplits > 1 ? kLenBuckets / 2 : 0) + min(len, kLenBuckets / 2 - 1);
    return kLenBuckets - 1 - key;
  }
  return kLenBuckets - 1 - min(len, kLenBuckets - 1);
}

// Work items: sequence i is cut into s_i = clamp(ceil(tiles_i / T), 1,
// max_splits) splits per kv head, T chosen so the items spread ~kItemsPerCta
// per persistent CTA; items are bucket-sorted longest first.  Sequences with
// no context get neutral partials here and no item.
__global__ void __launch_bounds__(kPlanThreads)
decode_plan_kernel(const int32_t* __restrict__ ctx, const int32_t* __restrict__ slots, int nseq, int Hkv, int Hq, int max_splits,
                   int grid_ctas, int min_tiles, int32_t* __restrict__ nsplit_of,
                   DecodeItem* __restrict__ items, int32_t* __restrict__ n_items,
                   float* __restrict__ part_ml, int32_t* __restrict__ item_counter,
                   int32_t* __restrict__ split_done) {
  __shared__ int hist[kLenBuckets];
  __shared__ int cursor[kLenBuckets];
  __shared__ unsigned long long total_tiles;
  __shared__ int T;
  const int tid = threadIdx.x;
  const long long pairs = (long long)nseq * Hkv;
  const bool splits_first = KB_DEC_SPLITS_FIRST && pairs < 2LL * grid_ctas;
  // items per CTA, doubled (the small-batch knob allows halves)
  const int ipc2 = !KB_DEC_ADAPT_IPC ? 2 * kItemsPerCta
                   : (8 * pairs >= (long long)KB_DEC_IPC3_LO_X8 * grid_ctas &&
                      5 * pairs <= (long long)KB_DEC_IPC3_HI_X5 * grid_ctas) ? 6
                   : (2 * pairs < (long long)grid_ctas) ? KB_DEC_TINY_IPC_X2
                   : (pairs < (long long)grid_ctas) ? KB_DEC_SUB1_IPC_X2
                   : 2 * kItemsPerCta;
  if (tid == 0) total_tiles = 0;
  for (int i = tid; i < kMaxLayers; i += blockDim.x) item_counter[i] = 0;
  for (int i = tid; i < nseq * Hkv; i += blockDim.x) split_done[i] = 0;
  for (int b = tid; b < kLenBuckets; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  unsigned long long local = 0;
  for (int i = tid; i < nseq; i += blockDim.x) local += (ctx[i] + kTileTok - 1) / kTileTok;
  atomicAdd(&total_tiles, local);
  __syncthreads();
  if (tid == 0) {
    const unsigned long long work = total_tiles * (unsigned long long)Hkv;
    const unsigned long long tgt = ((unsigned long long)grid_ctas * ipc2 + 1) / 2;
    const unsigned long long per = (work + tgt - 1) / tgt;
    T = (int)(per > (unsigned long long)min_tiles ? per : min_tiles);
  }
  __syncthreads();
  // ceil() per sequence makes the item count overshoot kItemsPerCta per CTA;
  // the few items past grid * kItemsPerCta then run as a third round on a
  // handful of CTAs (a 6 us tail at 16 sequences).  Warp w counts the items
  // T + w would give; the smallest T that fits the rounds wins.
  if (KB_DEC_TSEARCH) {
    __shared__ long long cnt_w[32];
    const int w = tid >> 5, lane = tid & 31;
    const int Tc = T + w;
    long long c = 0;
    for (int i = lane; i < nseq; i += 32) {
      const int tiles = (ctx[i] + kTileTok - 1) / kTileTok;
      if (tiles) c += min(max((tiles + Tc - 1) / Tc, 1), max_splits);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt_w[w] = c * Hkv;
    __syncthreads();
    if (tid == 0) {
      const long long target = ((long long)grid_ctas * ipc2 + 1) / 2;
      for (int k = 0; k < 32; ++k)
        if (cnt_w[k] <= target) {
          T += k;
          break;
        }
    }
    __syncthreads();
  }
  auto splits_of = [&](int tiles) {
    int s = (tiles + T - 1) / T;
    return s < 1 ? 1 : (s > max_splits ? max_splits : s);
  };
  // split counts per sequence (no context: no item, 0 splits -- the
  // attention kernel writes a zero row)
  for (int i = tid; i < nseq; i += blockDim.x) {
    const int tiles = (ctx[i] + kTileTok - 1) / kTileTok;
    nsplit_of[i] = tiles == 0 ? 0 : splits_of(tiles);
  }
  __syncthreads();
  if (KB_DEC_REFINE) {
    // The item budget T leaves under grid * kItemsPerCta (the counts move in
    // steps of Hkv per sequence, so a T one smaller overshoots) goes to the
    // sequences whose pieces are longest: one more split each, longest
    // first, ties by index -- shorter last items, a tighter LPT tail.
    __shared__ unsigned long long cnt_all;
    __shared__ int thr, take, carry;
    __shared__ int scan_ws[32];
    if (tid == 0) {
      cnt_all = 0;
      carry = 0;
    }
    __syncthreads();
    unsigned long long c = 0;
    for (int i = tid; i < nseq; i += blockDim.x) {
      const int tiles = (ctx[i] + kTileTok - 1) / kTileTok, sp = nsplit_of[i];
      c += sp;
      if (tiles >= 2 && sp < max_splits && sp < tiles)
        atomicAdd(&hist[min((tiles + sp - 1) / sp, kLenBuckets - 1)], 1);
    }
    atomicAdd(&cnt_all, c);
    __syncthreads();
    if (tid == 0) {
      const long long target = ((long long)grid_ctas * ipc2 + 1) / 2;
      const long long cnt = (long long)cnt_all * Hkv;
      const long long extra = cnt <= target ? (target - cnt) / Hkv : 0;
      thr = 1 << 30;
      take = 0;
      long long acc = 0;
      for (int L = kLenBuckets - 1; L >= 2 && extra > 0; --L) {
        if (acc + hist[L] >= extra) {
          thr = L;
          take = (int)(extra - acc);
          break;
        }
        acc += hist[L];
      }
      if (extra > 0 && thr == (1 << 30)) thr = 1;  // every eligible sequence
    }
    __syncthreads();
    hist[tid] = 0;  // re-armed for the item histogram below
    for (int base = 0; base < nseq; base += blockDim.x) {
      const int i = base + tid;
      int L = 0, sp = 0;
      bool elig = false;
      if (i < nseq) {
        const int tiles = (ctx[i] + kTileTok - 1) / kTileTok;
        sp = nsplit_of[i];
        elig = tiles >= 2 && sp < max_splits && sp < tiles;
        L = elig ? (tiles + sp - 1) / sp : 0;
        L = min(L, kLenBuckets - 1);
      }
      const int f = elig && L == thr;
      const int incl = block_incl_scan(f, scan_ws);
      if (elig && (L > thr || (f && carry + incl - 1 < take))) nsplit_of[i] = sp + 1;
      __syncthreads();
      if (tid == kPlanThreads - 1) carry += incl;
      __syncthreads();
    }
  }
  for (int i = tid; i < nseq; i += blockDim.x) {
    const int tiles = (ctx[i] + kTileTok - 1) / kTileTok;
    const int s = nsplit_of[i];
    if (tiles == 0) continue;
    for (int k = 0; k < s; ++k) {
      int beg, len;
      piece(tiles, s, T, k, beg, len);
      atomicAdd(&hist[item_bucket(len, s, splits_first)], Hkv);
    }
  }
  __syncthreads();
  // exclusive scan of the (descending-length) histogram, one bucket per
  // thread: warp shuffles, then the 32 warp totals (a serial scan by one
  // thread cost ~30 us per decode step)
  static_assert(kLenBuckets == kPlanThreads && kPlanThreads == 1024, "one bucket per thread");
  __shared__ int warp_sum[32];
  {
    const int lane = tid & 31, w = tid >> 5;
    const int v = hist[tid];
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sum[w] = x;
    __syncthreads();
    if (w == 0) {
      int t = warp_sum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      warp_sum[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    const int before = (w ? warp_sum[w - 1] : 0) + x - v;
    cursor[tid] = before;
    if (tid == kLenBuckets - 1) *n_items = before + v;
  }
  __syncthreads();
  for (int i = tid; i < nseq; i += blockDim.x) {
    const int tiles = (ctx[i] + kTileTok - 1) / kTileTok;
    if (tiles == 0) continue;
    const int s = nsplit_of[i];
    for (int k = 0; k < s; ++k) {
      int beg, len;
      piece(tiles, s, T, k, beg, len);
      const int b = item_bucket(len, s, splits_first);
      for (int h = 0; h < Hkv; ++h) {
        const int pos = atomicAdd(&cursor[b], 1);
        items[pos] = DecodeItem{i, h, k, beg, len, slots[i], ctx[i], s};
      }
    }
  }
}

static int64_t ws_part_o(int64_t sh) { return round_up(sh * 128 * 4, 256); }
static int64_t ws_part_ml(int64_t sh) { return round_up(sh * 2 * 4, 256); }

}  // namespace kb

using namespace kb;

extern "C" int64_t kb_decode_workspace_bytes(int32_t nseq, int32_t n_q_heads, int32_t max_splits) {
  const int64_t sh = (int64_t)nseq * n_q_heads * max_splits;
  // items: at most nseq * n_kv_heads * max_splits <= sh
  return ws_part_o(sh) + ws_part_ml(sh) + round_up((int64_t)nseq * 4, 256) +
         round_up(sh * (int64_t)sizeof(DecodeItem), 256) + 256 + kMaxLayers * 4 +
         (int64_t)nseq * n_q_heads * 4;  // per-(sequence, kv head) split counters
}

extern "C" int kb_paged_decode(kb_pool* p, int32_t layer, int32_t n_q_heads, uint64_t q,
                               uint64_t slots, uint64_t ctx_lens, int32_t nseq, int32_t max_ctx,
                               float scale, uint64_t out, uint64_t workspace,
                               int64_t workspace_bytes, int32_t max_splits, int32_t flags,
                               uintptr_t stream) {
  if (!p) return fail(KB_EINVAL, "null pool");
  if (p->view) return refuse_view();
  const int Hkv = p->m.n_kv_heads, B = p->m.block_tokens;
  if (p->m.head_dim != 128) return fail(KB_EINVAL, "head_dim must be 128");
  if (n_q_heads % Hkv || n_q_heads / Hkv > 8) return fail(KB_EINVAL, "GQA group must be <= 8");
  if (B != 64 && B != 128) return fail(KB_EINVAL, "block_tokens must be 64 or 128");
  if (layer < 0 || layer >= p->m.num_layers || layer >= kMaxLayers) return fail(KB_EINVAL, "bad layer");
  if (max_splits < 1 || max_splits > 64) return fail(KB_EINVAL, "max_splits out of range");
  if (nseq <= 0) return KB_OK;
  (void)max_ctx;
  // the plan, the split partials and the counters all grow with nseq: a
  // workspace sized for fewer sequences would be overrun silently
  const int64_t need = kb_decode_workspace_bytes(nseq, n_q_heads, max_splits);
  if (!workspace || workspace_bytes < need)
    return fail(KB_EINVAL, "decode workspace holds " + std::to_string(workspace_bytes) + " < " +
                               std::to_string(need) + " bytes for " + std::to_string(nseq) +
                               " sequences");
  KB_RT(cudaSetDevice(p->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t sh = (int64_t)nseq * n_q_heads * max_splits;
  char* ws = reinterpret_cast<char*>(workspace);
  float* part_o = reinterpret_cast<float*>(ws);
  float* part_ml = reinterpret_cast<float*>(ws + ws_part_o(sh));
  int32_t* nsplit = reinterpret_cast<int32_t*>(ws + ws_part_o(sh) + ws_part_ml(sh));
  DecodeItem* items = reinterpret_cast<DecodeItem*>(ws + ws_part_o(sh) + ws_part_ml(sh) +
                                                     round_up((int64_t)nseq * 4, 256));
  int32_t* n_items = reinterpret_cast<int32_t*>(
      reinterpret_cast<char*>(items) + round_up(sh * (int64_t)sizeof(DecodeItem), 256));
  int32_t* item_counter = n_items + 64;  // kMaxLayers ints after the 256-byte n_items slot
  int32_t* split_done = item_counter + kMaxLayers;  // nseq * Hkv finished-split counters
  int dev_sms = 148;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, p->device);
  const int grid = dev_sms;  // persistent: one CTA per SM (the kernel needs ~210 KB smem)
  int rc = pool_enter(p, st);
  if (rc) return rc;
  if (!(flags & KB_DECODE_REUSE_PLAN)) {
    decode_plan_kernel<<<1, kPlanThreads, 0, st>>>(reinterpret_cast<const int32_t*>(ctx_lens),
                                                   reinterpret_cast<const int32_t*>(slots), nseq, Hkv, n_q_heads, max_splits, grid, kMinTiles,
                                                   nsplit, items, n_items, part_ml,
                                                   item_counter, split_done);
    KB_LAUNCH_CHECK();
  }
  #ifndef KB_DEC_FUSE_MIN_PAIRS_PER_SM_X4
#define KB_DEC_FUSE_MIN_PAIRS_PER_SM_X4 2
#endif
  // the merge warp makes the in-kernel merge cheap: it wins from about half
  // a (sequence, kv head) pair per SM up (r4 A/B against the combine launch,
  // us per Llama layer: 64 sequences 72.6 vs 76.2, 32: 36.1 vs 37.4, 16:
  // 25.2 vs 25.5); below, the few pairs' last merges sit in the kernel's
  // tail, where the combine launch is cheaper (4 sequences: 10.8 vs 11.8)
  int fuse = (int64_t)nseq * Hkv >= (int64_t)KB_DEC_FUSE_MIN_PAIRS_PER_SM_X4 * grid / 4;
  if (flags & KB_DECODE_COMBINE) fuse = 0;
  if (flags & KB_DECODE_FUSE) fuse = 1;
  rc = launch_decode_tc(p, layer, n_q_heads, q, grid, scale, part_o, part_ml,
                        items, n_items, item_counter, nsplit, split_done, nseq, fuse, out,
                        max_splits, (flags & KB_DECODE_REUSE_PLAN) ? 1 : 0, st);
  if (rc) return rc;
  if (!fuse) {
    // programmatic dependent launch: the combine CTAs start while the
    // attention kernel drains and wait for its memory (griddepcontrol.wait)
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nseq * n_q_heads);
    cfg.blockDim = dim3(128);
    cfg.stream = st;
    cfg.attrs = pdl;
    cfg.numAttrs = 1;
    KB_RT(cudaLaunchKernelEx(&cfg, decode_combine_kernel, (const float*)part_o,
                             (const float*)part_ml, (const int32_t*)nsplit,
                             reinterpret_cast<__nv_bfloat16*>(out), (int)n_q_heads, (int)max_splits));
    KB_LAUNCH_CHECK();
  }
  return pool_leave(p, st);
}

#ifdef KB_DEC_TRACE
extern "C" int kb_debug_dec_trace(unsigned long long* out, int32_t n) {
  if (n > 1024 * kb::kTraceSlots) n = 1024 * kb::kTraceSlots;
  return cudaMemcpyFromSymbol(out, kb::g_dec_trace, (size_t)n * 8) == cudaSuccess ? 0 : -1;
}
#endif
