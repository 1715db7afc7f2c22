// N8 (decode): paged decode attention over the (enlarged, non-contiguous)
// KV pool, GQA, head_dim 128, bf16 in / fp32 accumulate.
//
// The reference has no attention: its only trace is the
// cost proxy attention_units(c, p) = p*c + (c^2+c)/2
// (pkg/src/dropsim/costmodel.py:50-57).  Parity is against the fp32 CPU
// restatement oracle/attention.py with max-abs <= 2e-2, mean-rel <= 1e-3.
//
// Work split: one CTA per (sequence, kv head, KV split); the split's partial
// (o, m, l) go to a workspace and a combine kernel merges them.
#include "kb_common.cuh"
#include "kb_decode_tc.cuh"

namespace kb {

// Split-KV combine: one CTA per (sequence, q head), thread = head_dim lane.
__global__ void decode_combine_kernel(const float* __restrict__ part_o,
                                      const float* __restrict__ part_ml,
                                      const int32_t* __restrict__ nsplit_of,
                                      __nv_bfloat16* __restrict__ out, int Hq, int max_splits) {
  const int sh = blockIdx.x;  // seq * Hq + head
  const int seq = sh / Hq;
  const int ns = nsplit_of[seq];
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

// Per-sequence split count: pages of the sequence spread over at most
// max_splits CTAs, at least `min_pages` pages each.
__global__ void decode_plan_kernel(const int32_t* __restrict__ ctx, int nseq, int B,
                                   int max_splits, int min_pages, int32_t* __restrict__ nsplit_of) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nseq) return;
  int pages = (ctx[i] + B - 1) / B;
  int s = (pages + min_pages - 1) / min_pages;
  if (s > max_splits) s = max_splits;
  if (s < 1) s = 1;
  nsplit_of[i] = s;
}

}  // namespace kb

using namespace kb;

extern "C" int64_t kb_decode_workspace_bytes(int32_t nseq, int32_t n_q_heads, int32_t max_splits) {
  const int64_t sh = (int64_t)nseq * n_q_heads * max_splits;
  return round_up(sh * 128 * 4, 256) + round_up(sh * 2 * 4, 256) + round_up((int64_t)nseq * 4, 256);
}

extern "C" int kb_paged_decode(kb_pool* p, int32_t layer, int32_t n_q_heads, uint64_t q,
                               uint64_t slots, uint64_t ctx_lens, int32_t nseq, int32_t max_ctx,
                               float scale, uint64_t out, uint64_t workspace, int32_t max_splits,
                               uintptr_t stream) {
  if (!p) return fail(KB_EINVAL, "null pool");
  const int Hkv = p->m.n_kv_heads, B = p->m.block_tokens;
  if (p->m.head_dim != 128) return fail(KB_EINVAL, "head_dim must be 128");
  if (n_q_heads % Hkv || n_q_heads / Hkv > 8) return fail(KB_EINVAL, "GQA group must be <= 8");
  if (B != 64 && B != 128) return fail(KB_EINVAL, "block_tokens must be 64 or 128");
  if (layer < 0 || layer >= p->m.num_layers) return fail(KB_EINVAL, "bad layer");
  if (max_splits < 1 || max_splits > 64) return fail(KB_EINVAL, "max_splits out of range");
  if (nseq <= 0) return KB_OK;
  KB_RT(cudaSetDevice(p->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t sh = (int64_t)nseq * n_q_heads * max_splits;
  float* part_o = reinterpret_cast<float*>(workspace);
  float* part_ml = reinterpret_cast<float*>(workspace + round_up(sh * 128 * 4, 256));
  int32_t* nsplit = reinterpret_cast<int32_t*>(workspace + round_up(sh * 128 * 4, 256) +
                                               round_up(sh * 2 * 4, 256));
  // Aim for >= 2 waves of CTAs over 148 SMs; a split covers >= 2 tiles.
  const int64_t tiles_max = ceil_div(max_ctx, 128);
  int64_t base_ctas = (int64_t)nseq * Hkv;
  int min_tiles = (int)ceil_div(tiles_max * base_ctas, 148 * 4);
  if (min_tiles < 2) min_tiles = 2;
  const int min_pages = min_tiles * (128 / B);
  decode_plan_kernel<<<(int)ceil_div(nseq, 128), 128, 0, st>>>(
      reinterpret_cast<const int32_t*>(ctx_lens), nseq, B, max_splits, min_pages, nsplit);
  KB_LAUNCH_CHECK();
  int rc = launch_decode_tc(p, layer, n_q_heads, q, slots, ctx_lens, nseq, max_ctx, scale,
                            part_o, part_ml, nsplit, max_splits, st);
  if (rc) return rc;
  decode_combine_kernel<<<nseq * n_q_heads, 128, 0, st>>>(part_o, part_ml, nsplit,
                                                          reinterpret_cast<__nv_bfloat16*>(out),
                                                          n_q_heads, max_splits);
  KB_LAUNCH_CHECK();
  return KB_OK;
}
