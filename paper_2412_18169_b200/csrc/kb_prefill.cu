// N8 (prefill): chunked paged prefill attention on tcgen05.
//
// A chunk of c new tokens of one request attends over its p cached prefix
// tokens plus itself causally -- the work the reference's cost model counts
// as attention_units(c, p) = p*c + (c^2 + c)/2 token pairs
// (pkg/src/dropsim/costmodel.py:50-57, used for stage time at
// engine.py:389-397).  FLOPs per layer = 4 * Hq * head_dim * attention_units.
//
// CTA = (128-row query tile, query head).  Per 128-key tile:
//   S[128 q x 128 k]  = Q[128 x 128 d] . K^T        (K-major A and B)
//   O_t[128 q x 128 d] = P[128 q x 128 k] . V        (V is an MN-major B)
// S double-buffered in TMEM, P staged bf16 in smem (SW128), O folded into
// registers with the online-softmax rescale.  Warp roles (192 threads):
// 0-3 softmax / epilogue (thread = query row), 4 TMA producer (K/V pages
// named by the block table), 5 MMA issuer + TMEM owner.
#include <cuda_bf16.h>

#include "kb_common.cuh"
#include "kb_sm100.cuh"

namespace kb {

constexpr int kPfStages = 2;
constexpr int kPfThreads = 192;
constexpr int kPfTile = 128;
constexpr int kPfHalf = 16384;                     // 128 rows x 64 el x 2 B
constexpr int kPfKV = 4 * kPfHalf;                 // K + V for one 128-key tile
constexpr int kPfQ = 2 * kPfHalf;
constexpr int kPfP = 4 * kPfHalf;                  // P_hi + P_lo
constexpr int kPfSmem = kPfStages * kPfKV + kPfQ + kPfP + 1024 + 1024;
constexpr uint32_t kPfTmemCols = 512;               // S0 | S1 | O

struct PrefillMisc {
  uint64_t full[kPfStages];
  uint64_t empty[kPfStages];
  uint64_t s_full[2];
  uint64_t o_full;
  uint64_t p_full;
  uint64_t q_full;
  uint32_t tmem_base;
};

template <int kB>
__global__ void __launch_bounds__(kPfThreads, 1)
prefill_tc_kernel(const __grid_constant__ CUtensorMap tmap, const __nv_bfloat16* __restrict__ q,
                  const int32_t* __restrict__ bt, const int32_t* __restrict__ slots,
                  const int32_t* __restrict__ q_off, const int32_t* __restrict__ q_len,
                  const int32_t* __restrict__ prefix, int mtiles,
                  __nv_bfloat16* __restrict__ out, int Hkv, int Hq, int L, int maxp, int layer,
                  float scale_log2) {
  using namespace sm100;
  constexpr int kPPT = kPfTile / kB;
  const int hq = blockIdx.y;
  const int seq = blockIdx.x / mtiles, mt = blockIdx.x % mtiles;
  const int h = hq / (Hq / Hkv);
  const int qlen = q_len[seq], pre = prefix[seq], qo = q_off[seq];
  const int row0 = mt * kPfTile;
  if (row0 >= qlen) return;  // grid is sized for the longest chunk
  const int rows = min(kPfTile, qlen - row0);
  const int kv_len = pre + row0 + rows;  // keys visible to the last row
  const int nt = (kv_len + kPfTile - 1) / kPfTile;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem + kPfStages * kPfKV;
  uint8_t* sP = sQ + kPfQ;
  PrefillMisc* misc = reinterpret_cast<PrefillMisc*>(sP + kPfP);

  if (warp == 5) {
    if (lane == 0) {
      for (int s = 0; s < kPfStages; ++s) {
        mbar_init(&misc->full[s], 1);
        mbar_init(&misc->empty[s], 1);
      }
      mbar_init(&misc->s_full[0], 1);
      mbar_init(&misc->s_full[1], 1);
      mbar_init(&misc->o_full, 1);
      mbar_init(&misc->p_full, 128);
      mbar_init(&misc->q_full, 128);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(&misc->tmem_base, kPfTmemCols);
  }
  if (warp == 4 && lane == 0) tma_prefetch_desc(&tmap);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = misc->tmem_base;
  const int32_t* bt_row = bt + ((int64_t)slots[seq] * L + layer) * maxp;

  if (warp == 4) {
    if (lane == 0) {
      for (int j = 0; j < nt; ++j) {
        const int stage = j % kPfStages;
        if (j >= kPfStages) mbar_wait(&misc->empty[stage], ((j / kPfStages) - 1) & 1);
        int32_t pages[kPPT];
        int npg = 0;
#pragma unroll
        for (int k = 0; k < kPPT; ++k) {
          const int pi = j * kPPT + k;
          pages[k] = (pi * kB < kv_len) ? bt_row[pi] : -1;
          npg += pages[k] >= 0;
        }
        mbar_arrive_expect_tx(&misc->full[stage], (uint32_t)(npg * kB * 512));
        uint8_t* sK = smem + stage * kPfKV;
        uint8_t* sV = sK + 2 * kPfHalf;
#pragma unroll
        for (int k = 0; k < kPPT; ++k) {
          if (pages[k] < 0) continue;
          const int rk = ((pages[k] * 2 + 0) * Hkv + h) * kB;
          const int rv = ((pages[k] * 2 + 1) * Hkv + h) * kB;
          const int off = k * kB * 128;
          tma_load_2d(sK + off, &tmap, 0, rk, &misc->full[stage]);
          tma_load_2d(sK + kPfHalf + off, &tmap, 64, rk, &misc->full[stage]);
          tma_load_2d(sV + off, &tmap, 0, rv, &misc->full[stage]);
          tma_load_2d(sV + kPfHalf + off, &tmap, 64, rv, &misc->full[stage]);
        }
      }
    }
  } else if (warp == 5) {
    constexpr uint32_t kIdQK = idesc_bf16_f32(128, 128, false, false);
    constexpr uint32_t kIdPV = idesc_bf16_f32(128, 128, false, true);
    const uint32_t q_addr = smem_u32(sQ), p_addr = smem_u32(sP);
    auto issue_qk = [&](int j) {
      const int stage = j % kPfStages;
      mbar_wait(&misc->full[stage], (j / kPfStages) & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t k_addr = smem_u32(smem + stage * kPfKV);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t a = sw128_desc(q_addr + (kk >> 2) * kPfHalf + (kk & 3) * 32, 16, 1024);
          const uint64_t b = sw128_desc(k_addr + (kk >> 2) * kPfHalf + (kk & 3) * 32, 16, 1024);
          mma_f16_ss(tmem + (j & 1) * 128, a, b, kIdQK, kk > 0);
        }
        mma_commit(&misc->s_full[j & 1]);
      }
      __syncwarp();
    };
    mbar_wait(&misc->q_full, 0);
    issue_qk(0);
    for (int j = 0; j < nt; ++j) {
      if (j + 1 < nt) issue_qk(j + 1);
      mbar_wait(&misc->p_full, j & 1);
      tc_fence_after();
      if (lane == 0) {
        const int stage = j % kPfStages;
        const uint32_t v_addr = smem_u32(smem + stage * kPfKV + 2 * kPfHalf);
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
          const int k8 = kk & 7;  // kk < 8: P_hi, kk >= 8: P_lo; both against V
          const uint64_t a = sw128_desc(p_addr + (kk >> 3) * 2 * kPfHalf + (k8 >> 2) * kPfHalf +
                                            (k8 & 3) * 32, 16, 1024);
          const uint64_t b = sw128_desc(v_addr + k8 * 2048, kPfHalf, 1024);  // MN-major V
          mma_f16_ss(tmem + 256, a, b, kIdPV, kk > 0);
        }
        mma_commit(&misc->o_full);
        mma_commit(&misc->empty[stage]);
      }
      __syncwarp();
    }
  } else {
    // Q tile -> SW128 K-major image (row = query row, 2 d-halves)
    {
      const int r = tid;
      const int4* src = reinterpret_cast<const int4*>(q + ((int64_t)(qo + row0 + r) * Hq + hq) * 128);
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        int4 v = r < rows ? src[c] : make_int4(0, 0, 0, 0);
        const uint32_t off = (c >> 3) * kPfHalf + r * 128 + ((((c & 7) ^ (r & 7)) & 7) << 4);
        *reinterpret_cast<int4*>(sQ + off) = v;
      }
    }
    fence_proxy_async_smem();
    mbar_arrive(&misc->q_full);

    const int qpos = pre + row0 + tid;  // this thread's query position
    const bool row_ok = tid < rows;
    float o[128];
#pragma unroll
    for (int i = 0; i < 128; ++i) o[i] = 0.f;
    float m_run = -INFINITY, l_run = 0.f, alpha_prev = 1.f;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    for (int j = 0; j < nt; ++j) {
      mbar_wait(&misc->s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      // pass 1: row max over this key tile (S re-read from TMEM in pass 2)
      const int kbase = j * kPfTile;
      const uint32_t s_addr = tmem + lane_base + (j & 1) * 128;
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float part[32];
        tmem_ld_32x32b_x32(s_addr + c * 32, part);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const bool ok = row_ok && (kbase + c * 32 + i) <= qpos;
          mx = fmaxf(mx, ok ? part[i] * scale_log2 : -INFINITY);
        }
      }
      const float m_new = fmaxf(m_run, mx);
      const float alpha = m_new == -INFINITY ? 1.f : exp2f(m_run - m_new);
      if (j > 0) {  // fold the previous tile's O (frees the P buffer)
        mbar_wait(&misc->o_full, (j - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float part[32];
          tmem_ld_32x32b_x32(tmem + lane_base + 256 + c * 32, part);
#pragma unroll
          for (int i = 0; i < 32; ++i) o[c * 32 + i] = o[c * 32 + i] * alpha_prev + part[i];
        }
      }
      alpha_prev = alpha;
      if (kbase + kPfTile > kv_len) {  // partial tile: zero V rows past kv_len
        const int stage = j % kPfStages;
        mbar_wait(&misc->full[stage], (j / kPfStages) & 1);
        if (kbase + tid >= kv_len) {
          uint8_t* sV = smem + stage * kPfKV + 2 * kPfHalf;
          int4* r0 = reinterpret_cast<int4*>(sV + tid * 128);
          int4* r1 = reinterpret_cast<int4*>(sV + kPfHalf + tid * 128);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            r0[c] = make_int4(0, 0, 0, 0);
            r1[c] = make_int4(0, 0, 0, 0);
          }
        }
      }
      // pass 2: P = exp2(S*scale - m) -> bf16 SW128 K-major image (row = query row)
      float rs = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float part[32];
        tmem_ld_32x32b_x32(s_addr + c * 32, part);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const bool ok = row_ok && (kbase + c * 32 + i) <= qpos && m_new != -INFINITY;
          part[i] = ok ? exp2f(part[i] * scale_log2 - m_new) : 0.f;
          rs += part[i];
        }
#pragma unroll
        for (int q8 = 0; q8 < 4; ++q8) {
          const int ch = c * 4 + q8;  // 16-byte chunk (8 keys) of the 128-key row
          // P = P_hi + P_lo, both bf16: the PV chain runs over K = 256
          // ([P_hi | P_lo] . [V ; V]) so P carries ~16 mantissa bits.
          __nv_bfloat162 hi[4], lo[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float x0 = part[q8 * 8 + 2 * e], x1 = part[q8 * 8 + 2 * e + 1];
            hi[e] = __floats2bfloat162_rn(x0, x1);
            const float2 hf = __bfloat1622float2(hi[e]);
            lo[e] = __floats2bfloat162_rn(x0 - hf.x, x1 - hf.y);
          }
          const uint32_t off = (ch >> 3) * kPfHalf + tid * 128 + ((((ch & 7) ^ (tid & 7)) & 7) << 4);
          *reinterpret_cast<int4*>(sP + off) = *reinterpret_cast<int4*>(hi);
          *reinterpret_cast<int4*>(sP + 2 * kPfHalf + off) = *reinterpret_cast<int4*>(lo);
        }
      }
      l_run = l_run * alpha + rs;
      m_run = m_new;
      fence_proxy_async_smem();
      mbar_arrive(&misc->p_full);
    }
    mbar_wait(&misc->o_full, (nt - 1) & 1);
    tc_fence_after();
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float part[32];
      tmem_ld_32x32b_x32(tmem + lane_base + 256 + c * 32, part);
#pragma unroll
      for (int i = 0; i < 32; ++i) o[c * 32 + i] = o[c * 32 + i] * alpha_prev + part[i];
    }
    if (row_ok) {
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      int4* dst = reinterpret_cast<int4*>(out + ((int64_t)(qo + row0 + tid) * Hq + hq) * 128);
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        __nv_bfloat162 pk[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          pk[e] = __floats2bfloat162_rn(o[c * 8 + 2 * e] * inv, o[c * 8 + 2 * e + 1] * inv);
        dst[c] = *reinterpret_cast<int4*>(pk);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tmem, kPfTmemCols);
  }
}

}  // namespace kb

using namespace kb;

extern "C" int kb_paged_prefill(kb_pool* p, int32_t layer, int32_t n_q_heads, uint64_t q,
                                uint64_t slots, uint64_t q_off, uint64_t q_len, uint64_t prefix,
                                int32_t nseq, int32_t max_q_len, float scale, uint64_t out,
                                uintptr_t stream) {
  if (!p) return fail(KB_EINVAL, "null pool");
  const int Hkv = p->m.n_kv_heads, B = p->m.block_tokens;
  if (p->m.head_dim != 128) return fail(KB_EINVAL, "head_dim must be 128");
  if (n_q_heads % Hkv) return fail(KB_EINVAL, "n_q_heads must be a multiple of n_kv_heads");
  if (B != 64 && B != 128) return fail(KB_EINVAL, "block_tokens must be 64 or 128");
  if (layer < 0 || layer >= p->m.num_layers) return fail(KB_EINVAL, "bad layer");
  if (nseq <= 0) return KB_OK;
  KB_RT(cudaSetDevice(p->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (max_q_len <= 0) return KB_OK;
  // grid = (seq x m-tiles of the longest chunk) x q heads; CTAs past their
  // sequence's chunk exit at once, so no host copy of q_len is needed
  const int mtiles = (int)ceil_div(max_q_len, kPfTile);
  const float scale_log2 = scale * 1.4426950408889634f;
  dim3 grid((unsigned)(nseq * mtiles), n_q_heads);
  if (B == 64) {
    static bool attr = false;
    if (!attr) {
      KB_RT(cudaFuncSetAttribute(prefill_tc_kernel<64>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kPfSmem));
      attr = true;
    }
    prefill_tc_kernel<64><<<grid, kPfThreads, kPfSmem, st>>>(
        p->kv_tmap, reinterpret_cast<const __nv_bfloat16*>(q), p->d_bt,
        reinterpret_cast<const int32_t*>(slots), reinterpret_cast<const int32_t*>(q_off),
        reinterpret_cast<const int32_t*>(q_len), reinterpret_cast<const int32_t*>(prefix), mtiles,
        reinterpret_cast<__nv_bfloat16*>(out), Hkv, n_q_heads, p->m.num_layers, p->maxp,
        layer, scale_log2);
  } else {
    static bool attr = false;
    if (!attr) {
      KB_RT(cudaFuncSetAttribute(prefill_tc_kernel<128>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kPfSmem));
      attr = true;
    }
    prefill_tc_kernel<128><<<grid, kPfThreads, kPfSmem, st>>>(
        p->kv_tmap, reinterpret_cast<const __nv_bfloat16*>(q), p->d_bt,
        reinterpret_cast<const int32_t*>(slots), reinterpret_cast<const int32_t*>(q_off),
        reinterpret_cast<const int32_t*>(q_len), reinterpret_cast<const int32_t*>(prefix), mtiles,
        reinterpret_cast<__nv_bfloat16*>(out), Hkv, n_q_heads, p->m.num_layers, p->maxp,
        layer, scale_log2);
  }
  KB_LAUNCH_CHECK();
  return KB_OK;
}
