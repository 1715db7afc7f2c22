// Elementwise pieces of a decoder layer for the device-backed engine's stage
// execution (serving.StageRunner): the residual add fused into the RMSNorm
// that follows it, and the SwiGLU activation.  Not on the overload path
// itself; they keep the measured stage times (which drive the reference's
// scheduler clock, engine.py:389-397) free of a dozen tiny launches per layer.
#include <cuda_bf16.h>

#include "kb_common.cuh"

namespace kb {

// One warp per row: x (+)= res (bf16, in place); out = bf16(x * rsqrt(mean(x^2) + eps)) * w.
__global__ void __launch_bounds__(256)
add_rmsnorm_kernel(__nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ res,
                   const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ out, int n,
                   int H, float eps) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n) return;
  __nv_bfloat162* xr = reinterpret_cast<__nv_bfloat162*>(x + (int64_t)warp * H);
  const __nv_bfloat162* rr = res ? reinterpret_cast<const __nv_bfloat162*>(res + (int64_t)warp * H)
                                 : nullptr;
  const int H2 = H / 2;
  float ss = 0.f;
  for (int i = lane; i < H2; i += 32) {
    __nv_bfloat162 v = xr[i];
    if (rr) {
      v = __hadd2(v, rr[i]);
      xr[i] = v;
    }
    const float2 f = __bfloat1622float2(v);
    ss += f.x * f.x + f.y * f.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float inv = rsqrtf(ss / H + eps);
  const __nv_bfloat162* wr = reinterpret_cast<const __nv_bfloat162*>(w);
  __nv_bfloat162* orow = reinterpret_cast<__nv_bfloat162*>(out + (int64_t)warp * H);
  for (int i = lane; i < H2; i += 32) {
    const float2 f = __bfloat1622float2(xr[i]);
    const __nv_bfloat162 nrm = __floats2bfloat162_rn(f.x * inv, f.y * inv);
    orow[i] = __hmul2(nrm, wr[i]);
  }
}

// out[r, j] = silu(gu[r, j]) * gu[r, F + j], bf16 in / out, fp32 math.
__global__ void __launch_bounds__(256)
silu_mul_kernel(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ out, int n,
                int F) {
  const int64_t F2 = F / 2, total = (int64_t)n * F2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / F2, c = i % F2;
    const __nv_bfloat162* row = reinterpret_cast<const __nv_bfloat162*>(gu + r * 2 * F);
    const float2 g = __bfloat1622float2(row[c]);
    const float2 u = __bfloat1622float2(row[F2 + c]);
    const float a = g.x / (1.f + __expf(-g.x)) * u.x;
    const float b = g.y / (1.f + __expf(-g.y)) * u.y;
    reinterpret_cast<__nv_bfloat162*>(out + r * F)[c] = __floats2bfloat162_rn(a, b);
  }
}

}  // namespace kb

using namespace kb;

extern "C" int kb_add_rmsnorm(uint64_t x, uint64_t res, uint64_t w, uint64_t out, int32_t n,
                              int32_t hidden, float eps, uintptr_t stream) {
  if (!x || !w || !out || n < 0 || hidden <= 0 || (hidden & 1))
    return fail(KB_EINVAL, "bad add_rmsnorm arguments");
  if (n == 0) return KB_OK;
  add_rmsnorm_kernel<<<(int)ceil_div((int64_t)n * 32, 256), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<__nv_bfloat16*>(x), reinterpret_cast<const __nv_bfloat16*>(res),
      reinterpret_cast<const __nv_bfloat16*>(w), reinterpret_cast<__nv_bfloat16*>(out), n, hidden,
      eps);
  KB_LAUNCH_CHECK();
  return KB_OK;
}

extern "C" int kb_silu_mul(uint64_t gu, uint64_t out, int32_t n, int32_t ffn, uintptr_t stream) {
  if (!gu || !out || n < 0 || ffn <= 0 || (ffn & 1)) return fail(KB_EINVAL, "bad silu_mul arguments");
  if (n == 0) return KB_OK;
  const int64_t work = (int64_t)n * (ffn / 2);
  silu_mul_kernel<<<grid_for(work, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(gu), reinterpret_cast<__nv_bfloat16*>(out), n, ffn);
  KB_LAUNCH_CHECK();
  return KB_OK;
}
