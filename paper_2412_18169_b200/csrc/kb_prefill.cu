// N8 (prefill): chunked paged prefill attention on tcgen05.
//
// A chunk of c new tokens of one request attends over its p cached prefix
// tokens plus itself causally -- the work the reference's cost model counts
// as attention_units(c, p) = p*c + (c^2 + c)/2 token pairs
// (pkg/src/dropsim/costmodel.py:50-57, used for stage time at
// engine.py:389-397).  FLOPs per layer = 4 * Hq * head_dim * attention_units.
//
// CTA = two 128-row query tiles of one head (256 query rows) sharing every
// K/V tile.  Per 128-key tile j and query tile t:
//   S_t = Q_t . K_j^T                 (tcgen05, A and B from smem, K-major)
//   P_t = exp2(S_t*scale - m_t)       (softmax warpgroup t, one row per thread)
//   O_t += P_t . V_j                  (A = P from TMEM, B = V MN-major)
// S, P and O live in TMEM (S0 | S1 | O0 | O1 = 512 columns); P overwrites S
// as fp16 pairs -- the V cache is stored fp16 (kb_append.cu) so P can be
// fp16 (11-bit mantissa) in the same-format P.V MMA, where a bf16 P alone
// costs ~1.1e-3 relative error.  The two tiles
// ping-pong: the MMA warp issues QK0(j) QK1(j) PV0(j) QK0(j+1) PV1(j)
// QK1(j+1) ..., so the tensor pipe works on one tile while the other tile's
// softmax runs.  O is rescaled lazily, only when a row max grows by more
// than 2^8 (the probabilities stay bounded by 256, exact in bf16 / fp32).
//
// Warp roles (320 threads): 0-3 softmax tile 0, 4-7 softmax tile 1, 8 TMA
// producer (K/V pages named by the block table), 9 MMA issuer + TMEM owner.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "kb_common.cuh"
#include "kb_sm100.cuh"

namespace kb {

constexpr int kPfStages = 2;
constexpr int kPfThreads = 320;
constexpr int kPfTile = 128;
constexpr int kPfHalf = 16384;                     // 128 rows x 64 el x 2 B
constexpr int kPfKV = 4 * kPfHalf;                 // K + V for one 128-key tile
constexpr int kPfQ = 2 * kPfHalf;                  // one 128-row Q tile
constexpr int kPfSmem = kPfStages * kPfKV + 2 * kPfQ + 1024 + 1024;
constexpr uint32_t kPfTmemCols = 512;              // S0 | S1 | O0 | O1
constexpr float kRescaleLog2 = 8.0f;               // lazy-rescale threshold

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct PrefillMisc {
  uint64_t full[kPfStages];
  uint64_t empty[kPfStages];
  uint64_t s_full[2];
  uint64_t p_ready[2];
  uint64_t o_done[2];
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
  const int seq = blockIdx.x / mtiles, mt = blockIdx.x % mtiles;  // mt: 256-row CTA tile
  const int h = hq / (Hq / Hkv);
  const int qlen = q_len[seq], pre = prefix[seq], qo = q_off[seq];
  const int row0 = mt * 2 * kPfTile;
  if (row0 >= qlen) return;  // grid is sized for the longest chunk
  const int rows = min(2 * kPfTile, qlen - row0);
  const int kv_len = pre + row0 + rows;  // keys visible to the last row
  const int nt = (kv_len + kPfTile - 1) / kPfTile;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem + kPfStages * kPfKV;  // Q0 then Q1
  PrefillMisc* misc = reinterpret_cast<PrefillMisc*>(sQ + 2 * kPfQ);

  if (warp == 9) {
    if (lane == 0) {
      for (int s = 0; s < kPfStages; ++s) {
        mbar_init(&misc->full[s], 1);
        mbar_init(&misc->empty[s], 1);
      }
      for (int t = 0; t < 2; ++t) {
        mbar_init(&misc->s_full[t], 1);
        mbar_init(&misc->p_ready[t], 128);
        mbar_init(&misc->o_done[t], 1);
      }
      mbar_init(&misc->q_full, 256);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(&misc->tmem_base, kPfTmemCols);
  }
  if (warp == 8 && lane == 0) tma_prefetch_desc(&tmap);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = misc->tmem_base;
  const int32_t* bt_row = bt + ((int64_t)slots[seq] * L + layer) * maxp;

  if (warp == 8) {
    // ------------------------------------------------ TMA producer
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
  } else if (warp == 9) {
    // ------------------------------------------------ MMA issuer
    constexpr uint32_t kIdQK = idesc_bf16_f32(128, 128, false, false);
    constexpr uint32_t kIdPV = idesc_f16_f32(128, 128, false, true);  // P fp16, V fp16
    auto issue_qk = [&](int t, int j) {
      const int stage = j % kPfStages;
      if (t == 0) {
        mbar_wait(&misc->full[stage], (j / kPfStages) & 1);
        tc_fence_after();
      }
      if (lane == 0) {
        const uint32_t q_addr = smem_u32(sQ + t * kPfQ);
        const uint32_t k_addr = smem_u32(smem + stage * kPfKV);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t a = sw128_desc(q_addr + (kk >> 2) * kPfHalf + (kk & 3) * 32, 16, 1024);
          const uint64_t b = sw128_desc(k_addr + (kk >> 2) * kPfHalf + (kk & 3) * 32, 16, 1024);
          mma_f16_ss(tmem + t * 128, a, b, kIdQK, kk > 0);
        }
        mma_commit(&misc->s_full[t]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int t, int j) {
      mbar_wait(&misc->p_ready[t], j & 1);
      tc_fence_after();
      if (lane == 0) {
        const int stage = j % kPfStages;
        const uint32_t v_addr = smem_u32(smem + stage * kPfKV + 2 * kPfHalf);
        const uint32_t p_base = tmem + t * 128;
        // 16-key group m: P (fp16 pairs) at TMEM column 8m, V rows 16m..16m+15
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const uint64_t b = sw128_desc(v_addr + m * 2048, kPfHalf, 1024);  // MN-major V
          mma_f16_ts(tmem + 256 + t * 128, p_base + 8 * m, b, kIdPV, (j > 0 || m > 0) ? 1u : 0u);
        }
        // O_t is read only by the epilogue: signal once, after the last tile
        if (j == nt - 1) mma_commit(&misc->o_done[t]);
        if (t == 1) mma_commit(&misc->empty[stage]);
      }
      __syncwarp();
    };
    mbar_wait(&misc->q_full, 0);
    tc_fence_after();
    issue_qk(0, 0);
    issue_qk(1, 0);
    for (int j = 0; j < nt; ++j) {
      issue_pv(0, j);
      if (j + 1 < nt) issue_qk(0, j + 1);
      issue_pv(1, j);
      if (j + 1 < nt) issue_qk(1, j + 1);
    }
  } else {
    // ------------------------------------------------ softmax warpgroup t
    const int t = warp >> 2;              // query tile of this warpgroup
    const int r = tid & 127;              // row within the tile (= TMEM lane)
    const int qrow = row0 + t * kPfTile + r;  // row within the chunk
    const bool row_ok = qrow < qlen;
    const int qpos = pre + qrow;
    {  // Q tile t -> SW128 K-major image
      const int4* src = reinterpret_cast<const int4*>(q + ((int64_t)(qo + qrow) * Hq + hq) * 128);
      uint8_t* dst = sQ + t * kPfQ;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        int4 v = row_ok ? src[c] : make_int4(0, 0, 0, 0);
        const uint32_t off = (c >> 3) * kPfHalf + r * 128 + ((((c & 7) ^ (r & 7)) & 7) << 4);
        *reinterpret_cast<int4*>(dst + off) = v;
      }
    }
    fence_proxy_async_smem();
    mbar_arrive(&misc->q_full);
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t s_addr = tmem + lane_base + t * 128;
    const uint32_t o_addr = tmem + lane_base + 256 + t * 128;
    float m_ref = -INFINITY, l_run = 0.f;
    for (int j = 0; j < nt; ++j) {
      mbar_wait(&misc->s_full[t], j & 1);
      tc_fence_after();
      const int kbase = j * kPfTile;
      // Tiles wholly below the warp's first query position need no mask
      // (warp-uniform); diagonal / tail tiles take the masked path.
      const int warp_q0 = pre + row0 + t * kPfTile + (warp & 3) * 32;
      const bool full_tile = kbase + kPfTile - 1 <= warp_q0 &&
                             row0 + t * kPfTile + (warp & 3) * 32 + 31 < qlen;
      // S row in two halves of 64 columns (two loads, one wait each)
      float mraw = -INFINITY;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t sr[2][32];
        tmem_ld_32x32b_x32_async(s_addr + hh * 64, sr[0]);
        tmem_ld_32x32b_x32_async(s_addr + hh * 64 + 32, sr[1]);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (full_tile) {
#pragma unroll
            for (int i = 0; i < 32; ++i) mraw = fmaxf(mraw, __uint_as_float(sr[c][i]));
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const bool ok = row_ok && (kbase + hh * 64 + c * 32 + i) <= qpos;
              mraw = fmaxf(mraw, ok ? __uint_as_float(sr[c][i]) : -INFINITY);
            }
          }
        }
      }
      const float mx = mraw * scale_log2;
      // lazy rescale: move the reference max only when it grows by > 2^8.
      // TMEM ld/st are warp-collective, so the whole warp rescales when any
      // of its rows needs it (alpha = 1 for the others).
      const bool need = mx > m_ref + kRescaleLog2;
      if (__any_sync(0xffffffffu, need)) {
        const float alpha = !need ? 1.f : (m_ref == -INFINITY ? 0.f : exp2f(m_ref - mx));
        if (j > 0) {
          // O_t += P.V of tile j-1 completed before QK_t(j) (in-order pipe,
          // and s_full tracks every earlier MMA of the issuer)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float part[32];
            tmem_ld_32x32b_x32(o_addr + c * 32, part);
            uint32_t w[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) w[i] = __float_as_uint(part[i] * alpha);
            tmem_st_32x32b_x32(o_addr + c * 32, w);
          }
        }
        if (need) {
          l_run *= alpha;
          m_ref = mx;
        }
      }
      if (kbase + kPfTile > kv_len && t == 0) {  // partial tile: zero V rows past kv_len
        const int stage = j % kPfStages;
        mbar_wait(&misc->full[stage], (j / kPfStages) & 1);
        if (kbase + r >= kv_len) {
          uint8_t* sV = smem + stage * kPfKV + 2 * kPfHalf;
          int4* r0 = reinterpret_cast<int4*>(sV + r * 128);
          int4* r1 = reinterpret_cast<int4*>(sV + kPfHalf + r * 128);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            r0[c] = make_int4(0, 0, 0, 0);
            r1[c] = make_int4(0, 0, 0, 0);
          }
        }
        fence_proxy_async_smem();
      }
      // pass 2: P = exp2(S*scale - m_ref) as fp16 pairs (the V cache is
      // fp16, kb_append.cu), written over S: the 64 keys of S half hh land in
      // P columns [32hh, 32hh + 32) -- columns whose S values were consumed.
      float rs = 0.f;
      const bool live = m_ref != -INFINITY;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t sr[2][32];
        tmem_ld_32x32b_x32_async(s_addr + hh * 64, sr[0]);
        tmem_ld_32x32b_x32_async(s_addr + hh * 64 + 32, sr[1]);
        tmem_ld_wait();
        uint32_t w[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          float x[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = 2 * i + e;  // 0..63 within the half
            float v = fast_exp2(fmaf(__uint_as_float(sr[col >> 5][col & 31]), scale_log2, -m_ref));
            if (!full_tile) {
              const int key = kbase + hh * 64 + col;
              v = (row_ok && key <= qpos && live) ? v : 0.f;
            }
            x[e] = v;
          }
          rs += x[0] + x[1];
          const __half2 hp = __floats2half2_rn(x[0], x[1]);
          w[i] = *reinterpret_cast<const uint32_t*>(&hp);
        }
        tmem_st_32x32b_x32(s_addr + hh * 32, w);
      }
      tmem_st_wait();
      l_run += rs;
      tc_fence_before();
      mbar_arrive(&misc->p_ready[t]);
    }
    // epilogue: O_t / l -> bf16 rows
    mbar_wait(&misc->o_done[t], 0);
    tc_fence_after();
    {
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      int4* dst = reinterpret_cast<int4*>(out + ((int64_t)(qo + qrow) * Hq + hq) * 128);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float part[32];
        tmem_ld_32x32b_x32(o_addr + c * 32, part);  // warp-collective: every lane
        if (!row_ok) continue;
#pragma unroll
        for (int q8 = 0; q8 < 4; ++q8) {
          __nv_bfloat162 pk[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            pk[e] = __floats2bfloat162_rn(part[q8 * 8 + 2 * e] * inv, part[q8 * 8 + 2 * e + 1] * inv);
          dst[c * 4 + q8] = *reinterpret_cast<int4*>(pk);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
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
  if (p->view) return refuse_view();
  const int Hkv = p->m.n_kv_heads, B = p->m.block_tokens;
  if (p->m.head_dim != 128) return fail(KB_EINVAL, "head_dim must be 128");
  if (n_q_heads % Hkv) return fail(KB_EINVAL, "n_q_heads must be a multiple of n_kv_heads");
  if (B != 64 && B != 128) return fail(KB_EINVAL, "block_tokens must be 64 or 128");
  if (layer < 0 || layer >= p->m.num_layers) return fail(KB_EINVAL, "bad layer");
  if (nseq <= 0) return KB_OK;
  KB_RT(cudaSetDevice(p->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (max_q_len <= 0) return KB_OK;
  // grid = (seq x 256-row tiles of the longest chunk) x q heads; CTAs past
  // their sequence's chunk exit at once, so no host copy of q_len is needed
  const int mtiles = (int)ceil_div(max_q_len, 2 * kPfTile);
  const float scale_log2 = scale * 1.4426950408889634f;
  dim3 grid((unsigned)(nseq * mtiles), n_q_heads);
  auto launch = [&](auto kernel) -> int {
    static bool attr = false;
    if (!attr) {
      KB_RT(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPfSmem));
      attr = true;
    }
    kernel<<<grid, kPfThreads, kPfSmem, st>>>(
        p->kv_tmap, reinterpret_cast<const __nv_bfloat16*>(q), p->d_bt,
        reinterpret_cast<const int32_t*>(slots), reinterpret_cast<const int32_t*>(q_off),
        reinterpret_cast<const int32_t*>(q_len), reinterpret_cast<const int32_t*>(prefix), mtiles,
        reinterpret_cast<__nv_bfloat16*>(out), Hkv, n_q_heads, p->m.num_layers, p->maxp, layer,
        scale_log2);
    KB_LAUNCH_CHECK();
    return KB_OK;
  };
  int rc = pool_enter(p, st);
  if (rc) return rc;
  rc = B == 64 ? launch(prefill_tc_kernel<64>) : launch(prefill_tc_kernel<128>);
  if (rc) return rc;
  return pool_leave(p, st);
}
