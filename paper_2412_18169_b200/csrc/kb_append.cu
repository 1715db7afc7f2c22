// KV append: scatter the new tokens' K/V rows into their pages.
//
// Page layout (one layer, one request, block_tokens tokens):
//   [K|V][n_kv_heads][block_tokens][head_dim], K bf16, V fp16
// so one kv head's K (or V) for a page is a contiguous block_tokens x 256 B
// tile: the unit the attention kernels stage through TMA.
// The page is found through the pool's block table ON DEVICE:
//   page = bt[slot][layer][pos / block_tokens], row = pos % block_tokens.
#include <cuda_fp16.h>

#include "kb_common.cuh"

namespace kb {

// bf16 -> fp16 for 8 packed values (exact for |x| in fp16's normal range
// [2^-14, 65504]; V activations live far inside it).  Storing V as fp16 lets
// the attention kernels feed P as fp16 (11-bit mantissa) into the P.V
// tcgen05 MMA, which needs both operands in the same format.
//
// The range is GUARDED, not assumed.  A bf16 value's magnitude bits
// (b & 0x7FFF) order like its magnitude, so with M = the largest magnitude
// of one token's V row (128 values of one kv head):
//   KB_KV_V_OVERFLOW   any |v| >= 2^16 (M >= 0x4780; inf / NaN included):
//                      fp16 would hold inf;
//   KB_KV_V_UNDERFLOW  0 < M < 2^-14 (0x3880): the whole row sits in fp16's
//                      subnormal range, where its relative precision is lost.
// A row whose max is a normal fp16 keeps every element within 2^-11 of M
// (subnormal elements err by <= 2^-25 <= 2^-11 M), the same bound the normal
// range gives -- so small entries next to normal ones are fine.  The append
// kernel sets the flags' sticky words (pinned, mapped host memory; one word
// per flag, plain stores), which kb_pool_kv_status reports and the host
// raises on.
__device__ __forceinline__ int4 bf16x8_to_f16x8(int4 v) {
  uint32_t w[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float lo = __uint_as_float(w[i] << 16), hi = __uint_as_float(w[i] & 0xFFFF0000u);
    const __half2 h = __floats2half2_rn(lo, hi);
    w[i] = *reinterpret_cast<const uint32_t*>(&h);
  }
  return make_int4((int)w[0], (int)w[1], (int)w[2], (int)w[3]);
}

// largest bf16 magnitude field of 8 packed values
__device__ __forceinline__ uint32_t max_mag8(int4 v) {
  const uint32_t w[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) m = max(m, max(w[i] & 0x7FFFu, (w[i] >> 16) & 0x7FFFu));
  return m;
}

// one warp per (token, kv head): lanes 0-15 move K (bf16), lanes 16-31 move
// V (bf16 in, fp16 stored), 16 bytes each (head_dim 128 = 256 B per row).
__global__ void kv_append_kernel(uint8_t* __restrict__ kv, const int32_t* __restrict__ bt,
                                 const int4* __restrict__ k, const int4* __restrict__ v,
                                 const int32_t* __restrict__ slots, const int32_t* __restrict__ pos,
                                 int ntok, int Hkv, int B, int L, int maxp, int max_slots,
                                 int layer, int64_t page_bytes, int64_t row_vec,
                                 uint32_t* __restrict__ status) {
  // the attention launch that follows (programmatic dependent launch) may
  // run its prologue now; it waits for this grid's writes before reading
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= ntok * Hkv) return;
  const int t = warp / Hkv, h = warp % Hkv;
  const int slot = slots[t], p = pos[t];
  // a slot or position the block table does not cover, or a position whose
  // page was never grown, would write outside the pool: skip the row and
  // raise the sticky KB_KV_NO_PAGE word (warp-uniform: t and h are)
  const bool in_table = slot >= 0 && slot < max_slots && p >= 0 && p / B < maxp;
  const int32_t page = in_table ? bt[((int64_t)slot * L + layer) * maxp + p / B] : -1;
  if (page < 0) {
    if (lane == 0) *(volatile uint32_t*)(status + 2) = 1u;
    return;
  }
  const int row = p % B;
  const int which = lane >> 4;  // 0 = K, 1 = V
  const int4* src = (which ? v : k) + (int64_t)t * row_vec + h * 16 + (lane & 15);
  const int64_t half = page_bytes / 2;
  int4* dst = reinterpret_cast<int4*>(kv + (int64_t)page * page_bytes + which * half +
                                      ((int64_t)h * B + row) * 256) + (lane & 15);
  const int4 val = *src;
  *dst = which ? bf16x8_to_f16x8(val) : val;
  // V-row range guard: max magnitude over lanes 16-31 (xor shuffles stay
  // inside each 16-lane half)
  uint32_t m = max_mag8(val);
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  const uint32_t bad = !which ? 0u
                       : (m >= 0x4780u ? KB_KV_V_OVERFLOW : 0u) |
                             (m > 0u && m < 0x3880u ? KB_KV_V_UNDERFLOW : 0u);
  // rare: one store per offending row, one word per flag -- plain stores of
  // the same value (no read-modify-write: atomics on pinned host memory are
  // not native over PCIe)
  if (lane == 16 && bad) {
    volatile uint32_t* st = status;
    if (bad & KB_KV_V_OVERFLOW) st[0] = 1u;
    if (bad & KB_KV_V_UNDERFLOW) st[1] = 1u;
  }
}

}  // namespace kb

using namespace kb;

extern "C" int kb_kv_append(kb_pool* p, int32_t layer, uint64_t k, uint64_t v, uint64_t slots,
                            uint64_t pos, int32_t ntok, int64_t row_stride, uintptr_t stream) {
  if (!p) return fail(KB_EINVAL, "null pool");
  if (p->view) return refuse_view();
  if (p->m.head_dim != 128) return fail(KB_EINVAL, "head_dim must be 128");
  if (layer < 0 || layer >= p->m.num_layers) return fail(KB_EINVAL, "bad layer");
  if (ntok <= 0) return KB_OK;
  const int64_t stride = row_stride > 0 ? row_stride : (int64_t)p->m.n_kv_heads * 128;
  if (stride % 8 || ((k | v) & 15)) return fail(KB_EINVAL, "K/V rows must be 16-byte aligned");
  KB_RT(cudaSetDevice(p->device));
  const int64_t warps = (int64_t)ntok * p->m.n_kv_heads;
  int rc = pool_enter(p, (cudaStream_t)stream);
  if (rc) return rc;
  kv_append_kernel<<<(int)ceil_div(warps * 32, 256), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<uint8_t*>(p->kva), p->d_bt, reinterpret_cast<const int4*>(k),
      reinterpret_cast<const int4*>(v), reinterpret_cast<const int32_t*>(slots),
      reinterpret_cast<const int32_t*>(pos), ntok, p->m.n_kv_heads, p->m.block_tokens,
      p->m.num_layers, p->maxp, p->max_slots, layer, p->m.page_bytes, stride / 8, p->d_status);
  KB_LAUNCH_CHECK();
  return pool_leave(p, (cudaStream_t)stream);
}

extern "C" int kb_pool_kv_status(kb_pool* p, uint32_t* flags, int32_t clear) {
  if (!p || !flags) return fail(KB_EINVAL, "null argument");
  if (p->view) return refuse_view();
  volatile uint32_t* h = p->h_status;
  *flags = (h[0] ? KB_KV_V_OVERFLOW : 0u) | (h[1] ? KB_KV_V_UNDERFLOW : 0u) |
           (h[2] ? KB_KV_NO_PAGE : 0u);
  if (clear) {
    h[0] = 0;
    h[1] = 0;
    h[2] = 0;
  }
  return KB_OK;
}
