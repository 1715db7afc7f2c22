// tcgen05 / TMA paged decode attention (one CTA per (seq, kv head, split)).
//
// Orientation: tokens on the MMA M dimension so the tensor core sees a real
// 128-row tile even though a GQA group has only 4-5 query heads:
//   S^T[128 tok x 16]  = K_tile[128 tok x 128 d] . Q^T[128 d x 16 heads]
//   O^T[128 d x 16]   += V^T[128 d x 128 tok] . P^T[128 tok x 16 heads]
// (query heads >= G are zero padding).  K/V tiles are two 64-token pages
// (block_tokens 64) or one 128-token page, staged by TMA with 128-byte
// swizzle straight from the pool pages named by the block table; V is read
// as an MN-major operand, so no transpose pass exists.  S and O live in
// TMEM (double-buffered); the online softmax runs on 4 warps, one token
// (for S) and one head_dim lane (for O) per thread.
//
// Warp roles (192 threads): 0-3 softmax / epilogue, 4 TMA producer,
// 5 MMA issuer + TMEM owner.
#pragma once
#include <cuda_bf16.h>

#include "kb_common.cuh"
#include "kb_sm100.cuh"

namespace kb {

constexpr int kDecStages = 3;
constexpr int kDecThreads = 192;
constexpr int kTileTok = 128;
constexpr int kStageBytes = 65536;       // K (32 KiB) + V (32 KiB) for 128 tokens
constexpr int kHalfBytes = 16384;        // one 64-wide d-half of a 128-token tile
constexpr int kQBytes = 4096;            // 16 rows x 128 d bf16, SW128 K-major
constexpr int kPBytes = 4096;            // 16 rows x 128 tok bf16, SW128 K-major
constexpr int kDecSmem = kDecStages * kStageBytes + kQBytes + kPBytes + 1024 /*misc*/ + 1024 /*align*/;
constexpr uint32_t kDecTmemCols = 64;    // S0 S1 O0 O1, 16 columns each

struct DecodeMisc {
  uint64_t full[kDecStages];
  uint64_t empty[kDecStages];
  uint64_t s_full[2];
  uint64_t o_full[2];
  uint64_t p_full;
  uint64_t q_full;
  uint32_t tmem_base;
  uint32_t _pad;
  float red[2][4][8];
  float lred[4][8];
};

template <int kB>
__global__ void __launch_bounds__(kDecThreads, 1)
decode_tc_kernel(const __grid_constant__ CUtensorMap tmap, const __nv_bfloat16* __restrict__ q,
                 const int32_t* __restrict__ bt, const int32_t* __restrict__ slots,
                 const int32_t* __restrict__ ctx_lens, const int32_t* __restrict__ nsplit_of,
                 float* __restrict__ part_o, float* __restrict__ part_ml, int Hkv, int G, int Hq,
                 int L, int maxp, int layer, int max_splits, float scale_log2) {
  using namespace sm100;
  constexpr int kPPT = kTileTok / kB;  // pages per tile
  const int split = blockIdx.x % max_splits;
  const int sh = blockIdx.x / max_splits;
  const int seq = sh / Hkv, h = sh % Hkv;
  const int ns = nsplit_of[seq];
  if (split >= ns) return;
  const int ctx = ctx_lens[seq];
  const int tiles = (ctx + kTileTok - 1) / kTileTok;
  const int t_beg = (int)((int64_t)split * tiles / ns);
  const int nt = (int)((int64_t)(split + 1) * tiles / ns) - t_beg;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem + kDecStages * kStageBytes;
  uint8_t* sP = sQ + kQBytes;
  DecodeMisc* misc = reinterpret_cast<DecodeMisc*>(sP + kPBytes);

  if (nt <= 0) {  // empty split (ctx == 0): neutral partials
    for (int g = 0; g < G; ++g) {
      const int64_t row = ((int64_t)(seq * Hq + h * G + g) * max_splits + split);
      if (tid < 128) part_o[row * 128 + tid] = 0.f;
      if (tid == 0) {
        part_ml[row * 2] = -INFINITY;
        part_ml[row * 2 + 1] = 0.f;
      }
    }
    return;
  }

  if (warp == 5) {
    if (lane == 0) {
      for (int s = 0; s < kDecStages; ++s) {
        mbar_init(&misc->full[s], 1);
        mbar_init(&misc->empty[s], 1);
      }
      for (int b = 0; b < 2; ++b) {
        mbar_init(&misc->s_full[b], 1);
        mbar_init(&misc->o_full[b], 1);
      }
      mbar_init(&misc->p_full, 128);
      mbar_init(&misc->q_full, 128);
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
  const int slot = slots[seq];
  const int32_t* bt_row = bt + ((int64_t)slot * L + layer) * maxp;

  if (warp == 4) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      for (int j = 0; j < nt; ++j) {
        const int stage = j % kDecStages;
        if (j >= kDecStages) mbar_wait(&misc->empty[stage], ((j / kDecStages) - 1) & 1);
        const int tile = t_beg + j;
        int npg = 0;
        int32_t pages[kPPT];
#pragma unroll
        for (int k = 0; k < kPPT; ++k) {
          const int pi = tile * kPPT + k;
          pages[k] = (pi * kB < ctx) ? bt_row[pi] : -1;
          npg += pages[k] >= 0;
        }
        mbar_arrive_expect_tx(&misc->full[stage], (uint32_t)(npg * kB * 512));
        uint8_t* sK = smem + stage * kStageBytes;
        uint8_t* sV = sK + 2 * kHalfBytes;
#pragma unroll
        for (int k = 0; k < kPPT; ++k) {
          if (pages[k] < 0) continue;
          const int rk = ((pages[k] * 2 + 0) * Hkv + h) * kB;
          const int rv = ((pages[k] * 2 + 1) * Hkv + h) * kB;
          const int off = k * kB * 128;
          tma_load_2d(sK + off, &tmap, 0, rk, &misc->full[stage]);
          tma_load_2d(sK + kHalfBytes + off, &tmap, 64, rk, &misc->full[stage]);
          tma_load_2d(sV + off, &tmap, 0, rv, &misc->full[stage]);
          tma_load_2d(sV + kHalfBytes + off, &tmap, 64, rv, &misc->full[stage]);
        }
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------ MMA issuer
    constexpr uint32_t kIdQK = idesc_bf16_f32(128, 16, false, false);
    constexpr uint32_t kIdPV = idesc_bf16_f32(128, 16, true, false);
    const uint32_t q_addr = smem_u32(sQ), p_addr = smem_u32(sP);
    auto issue_qk = [&](int j) {
      const int stage = j % kDecStages;
      mbar_wait(&misc->full[stage], (j / kDecStages) & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t k_addr = smem_u32(smem + stage * kStageBytes);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t a = sw128_desc(k_addr + (kk >> 2) * kHalfBytes + (kk & 3) * 32, 16, 1024);
          const uint64_t b = sw128_desc(q_addr + (kk >> 2) * 2048 + (kk & 3) * 32, 16, 1024);
          mma_f16_ss(tmem + (j & 1) * 16, a, b, kIdQK, kk > 0);
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
        const int stage = j % kDecStages;
        const uint32_t v_addr = smem_u32(smem + stage * kStageBytes + 2 * kHalfBytes);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          // A = V^T, MN-major: LBO = d-half stride, SBO = 8-token group stride
          const uint64_t a = sw128_desc(v_addr + kk * 2048, kHalfBytes, 1024);
          const uint64_t b = sw128_desc(p_addr + (kk >> 2) * 2048 + (kk & 3) * 32, 16, 1024);
          mma_f16_ss(tmem + 32 + (j & 1) * 16, a, b, kIdPV, kk > 0);
        }
        mma_commit(&misc->o_full[j & 1]);
        mma_commit(&misc->empty[stage]);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------ softmax / epilogue (tid < 128)
    // Q -> SW128 K-major smem image, rows >= G zero.
    for (int c = tid; c < 16 * 16; c += 128) {
      const int g = c >> 4, chunk = c & 15;  // 16-byte chunk of 8 d values
      int4 val = make_int4(0, 0, 0, 0);
      if (g < G)
        val = reinterpret_cast<const int4*>(q + ((int64_t)seq * Hq + h * G + g) * 128)[chunk];
      const uint32_t off = (chunk >> 3) * 2048 + g * 128 + ((((chunk & 7) ^ (g & 7)) & 7) << 4);
      *reinterpret_cast<int4*>(sQ + off) = val;
    }
    fence_proxy_async_smem();
    mbar_arrive(&misc->q_full);

    float m_run[8], l_part[8], o_acc[8], alpha_prev[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      m_run[g] = -INFINITY;
      l_part[g] = 0.f;
      o_acc[g] = 0.f;
      alpha_prev[g] = 1.f;
    }
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    for (int j = 0; j < nt; ++j) {
      const int tile = t_beg + j;
      const int valid = min(kTileTok, ctx - tile * kTileTok);
      mbar_wait(&misc->s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
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
      float alpha[8], p[8];
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        float tm = fmaxf(fmaxf(misc->red[j & 1][0][g], misc->red[j & 1][1][g]),
                         fmaxf(misc->red[j & 1][2][g], misc->red[j & 1][3][g]));
        const float m_new = fmaxf(m_run[g], tm);
        if (m_new == -INFINITY) {
          alpha[g] = 1.f;
          p[g] = 0.f;
        } else {
          alpha[g] = exp2f(m_run[g] - m_new);  // m_run = -inf -> 0
          p[g] = exp2f(s[g] - m_new);          // masked -> 0
        }
        l_part[g] = l_part[g] * alpha[g] + p[g];
        m_run[g] = m_new;
      }
      if (j > 0) {  // fold in O of the previous tile (also frees the P buffer)
        mbar_wait(&misc->o_full[(j - 1) & 1], ((j - 1) >> 1) & 1);
        tc_fence_after();
        float ov[8], ol[8];
        tmem_ld_32x32b_x8(tmem + lane_base + 32 + ((j - 1) & 1) * 16, ov);
        tmem_ld_32x32b_x8(tmem + lane_base + 40 + ((j - 1) & 1) * 16, ol);
#pragma unroll
        for (int g = 0; g < 8; ++g) o_acc[g] = o_acc[g] * alpha_prev[g] + (ov[g] + ol[g]);
      }
#pragma unroll
      for (int g = 0; g < 8; ++g) alpha_prev[g] = alpha[g];
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
      // P^T -> SW128 K-major smem image (rows = heads, K = tokens).  The
      // N=16 MMA has room for 16 columns but a GQA group uses <= 8, so the
      // spare rows carry the bf16 residual of P: row g = bf16(p), row 8+g =
      // bf16(p - bf16(p)).  O^T columns g and 8+g sum to a ~16-bit-mantissa
      // P.V at no extra MMA cost (the kernel is HBM-bound).
      const uint32_t tbase = (tid >> 6) * 2048;
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const __nv_bfloat16 hi = __float2bfloat16(p[g]);
        const __nv_bfloat16 lo = __float2bfloat16(p[g] - __bfloat162float(hi));
        *reinterpret_cast<__nv_bfloat16*>(sP + tbase + sw128_offset(g, tid & 63)) = hi;
        *reinterpret_cast<__nv_bfloat16*>(sP + tbase + sw128_offset(g + 8, tid & 63)) = lo;
      }
      fence_proxy_async_smem();
      mbar_arrive(&misc->p_full);
    }
    {
      const int j = nt - 1;
      mbar_wait(&misc->o_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      float ov[8], ol[8];
      tmem_ld_32x32b_x8(tmem + lane_base + 32 + (j & 1) * 16, ov);
      tmem_ld_32x32b_x8(tmem + lane_base + 40 + (j & 1) * 16, ol);
#pragma unroll
      for (int g = 0; g < 8; ++g) o_acc[g] = o_acc[g] * alpha_prev[g] + (ov[g] + ol[g]);
    }
    // l = sum over the 128 token lanes
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      float v = l_part[g];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) misc->lred[warp][g] = v;
    }
    named_bar_sync(1, 128);
    for (int g = 0; g < G; ++g) {
      const int64_t row = ((int64_t)(seq * Hq + h * G + g) * max_splits + split);
      part_o[row * 128 + tid] = o_acc[g];
      if (tid == 0) {
        part_ml[row * 2] = m_run[g];
        part_ml[row * 2 + 1] =
            misc->lred[0][g] + misc->lred[1][g] + misc->lred[2][g] + misc->lred[3][g];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tmem, kDecTmemCols);
  }
}

inline int launch_decode_tc(kb_pool* p, int layer, int Hq, uint64_t q, uint64_t slots,
                            uint64_t ctx_lens, int nseq, int max_ctx, float scale, float* part_o,
                            float* part_ml, int32_t* nsplit, int max_splits, cudaStream_t st) {
  (void)max_ctx;
  const int Hkv = p->m.n_kv_heads, B = p->m.block_tokens;
  const float scale_log2 = scale * 1.4426950408889634f;
  dim3 grid((unsigned)((int64_t)nseq * Hkv * max_splits));
  if (B == 64) {
    static bool attr = false;
    if (!attr) {
      KB_RT(cudaFuncSetAttribute(decode_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kDecSmem));
      attr = true;
    }
    decode_tc_kernel<64><<<grid, kDecThreads, kDecSmem, st>>>(
        p->kv_tmap, reinterpret_cast<const __nv_bfloat16*>(q), p->d_bt,
        reinterpret_cast<const int32_t*>(slots), reinterpret_cast<const int32_t*>(ctx_lens),
        nsplit, part_o, part_ml, Hkv, Hq / Hkv, Hq, p->m.num_layers, p->maxp, layer, max_splits,
        scale_log2);
  } else {
    static bool attr = false;
    if (!attr) {
      KB_RT(cudaFuncSetAttribute(decode_tc_kernel<128>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kDecSmem));
      attr = true;
    }
    decode_tc_kernel<128><<<grid, kDecThreads, kDecSmem, st>>>(
        p->kv_tmap, reinterpret_cast<const __nv_bfloat16*>(q), p->d_bt,
        reinterpret_cast<const int32_t*>(slots), reinterpret_cast<const int32_t*>(ctx_lens),
        nsplit, part_o, part_ml, Hkv, Hq / Hkv, Hq, p->m.num_layers, p->maxp, layer, max_splits,
        scale_log2);
  }
  KB_LAUNCH_CHECK();
  return KB_OK;
}

}  // namespace kb
