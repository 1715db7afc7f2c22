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
// Warp roles (384 threads): 0-3 softmax tile 0, 4-7 softmax tile 1, 8 TMA
// producer (K/V pages named by the block table), 9 MMA issuer + TMEM owner,
// 10-11 idle; warpgroup 2 gives its registers to the softmax warpgroups
// (setmaxnreg) so a thread holds its full 128-column S row.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "kb_common.cuh"
#include "kb_sm100.cuh"

namespace kb {

constexpr int kPfStages = 2;
constexpr int kPfThreads = 384;  // 2 softmax warpgroups + 1 producer/MMA warpgroup
constexpr int kPfTile = 128;
constexpr int kPfHalf = 16384;                     // 128 rows x 64 el x 2 B
constexpr int kPfKV = 4 * kPfHalf;                 // K + V for one 128-key tile
constexpr int kPfQ = 2 * kPfHalf;                  // one 128-row Q tile
constexpr int kPfSmem = kPfStages * kPfKV + 2 * kPfQ + 1024 + 1024;
constexpr uint32_t kPfTmemCols = 512;              // S0 | S1 | O0 | O1
constexpr float kRescaleLog2 = 8.0f;               // lazy-rescale threshold
#ifndef KB_PF_REGS_SOFTMAX
#define KB_PF_REGS_SOFTMAX 216
#endif
// per SMSP: 2 softmax warps x 216 + 1 warpgroup-2 warp x 64 = 496 regs/lane.
// setmaxnreg.inc draws from the CTA's launch allocation (3 warps x 168 = 504
// per SMSP), so 2 x 224 + 64 = 512 never gets its registers and hangs.
// (A 640-thread variant -- two softmax warpgroups per Q tile splitting the
// columns -- measured 57-58% against this version's 61%: its pool of
// 5 x 96 per SMSP caps the softmax at 104 registers.)
constexpr int kPfRegsSoftmax = KB_PF_REGS_SOFTMAX;
constexpr int kPfRegsProducer = 64;

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed f32x2 FMA / add (sm_100a): two softmax elements per instruction.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

// exp2 on the FMA pipe (FA4's trick): the MUFU unit does 16 ex2 per clock
// per SM -- exactly the tensor pipe's pace for a 128x128 tile -- so a share
// of the exponentials is computed as 2^j * p(f), j = round(x),
// f = x - j in [-0.5, 0.5], p a degree-3 fit of 2^f (max rel. error 7.5e-5,
// below the fp16 rounding of P), 2^j added into the exponent bits.
__device__ __forceinline__ float2 exp2_fma2(float2 x) {
  const float kMagic = 12582912.0f;  // 1.5 * 2^23: round-to-nearest
  x.x = fmaxf(x.x, -127.f);
  x.y = fmaxf(x.y, -127.f);
  const float2 t = fadd2(x, make_float2(kMagic, kMagic));
  const float2 jf = fadd2(t, make_float2(-kMagic, -kMagic));
  const float2 f = fadd2(x, make_float2(-jf.x, -jf.y));
  float2 p = ffma2(make_float2(0.0551716685f, 0.0551716685f), f,
                   make_float2(0.2426111549f, 0.2426111549f));
  p = ffma2(p, f, make_float2(0.6932609677f, 0.6932609677f));
  p = ffma2(p, f, make_float2(0.9999280572f, 0.9999280572f));
  // bits(t) << 23 == j << 23 (mod 2^32): the magic's low 9 bits are zero
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}
// pairs i with i % kEmuEvery == kEmuEvery - 1 use exp2_fma2
#ifndef KB_PF_EMU_EVERY
#define KB_PF_EMU_EVERY 4
#endif
constexpr int kEmuEvery = KB_PF_EMU_EVERY;
// P key pairs published with p_lo (the rest with p_hi): 32 = halves; 48 =
// keys 0-95 first, so only the P.V of keys 96-127 and the next QK separate
// a tile's softmax from the next one -- measured 0.5% slower on the config-4
// layer (the loop is bound by the softmax, not by that tail; r4 pf_ab)
#ifndef KB_PF_PSPLIT
#define KB_PF_PSPLIT 32
#endif
constexpr int kPSplit = KB_PF_PSPLIT;
#ifdef KB_PF_THREAD_ARRIVE
constexpr int kPArrivals = 128;  // every softmax thread arrives on p_lo / p_hi
#else
constexpr int kPArrivals = 4;    // one elected lane per softmax warp
#endif
static_assert(kPSplit == 32 || kPSplit == 48, "P publish split: 32 or 48 pairs");
// (Issuing the QK of keys 64-127 early -- those S columns never hold P --
// as N=64 MMAs measured 52% against 67%: the half-width MMAs re-read Q for
// every half and double the QK instruction count.)
// (ex2.approx.f16x2 for a pair -- one MUFU op instead of two -- keeps the
// error at 3e-4 mean-rel but costs conversions: 50-61% of peak, so the pass
// is bound by instruction latency, not by the MUFU units.)
// (Strictly alternating the two tiles' exponential passes through an
// mbarrier token measured 64.4% vs 65.7% without: the pass is latency-bound
// per warp, not only MUFU-bound.)

// kSteps K=16 steps of O (+)= P.V: P (fp16 pairs) from TMEM columns 8m
// onward, V rows 16m onward (the SW128 MN-major descriptor advances 2 KiB,
// 128 in 16-byte units, per 16 rows)
template <int kSteps>
__device__ __forceinline__ void mma_ts_steps(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                             uint32_t idesc, uint32_t acc_first) {
#pragma unroll
  for (int m = 0; m < kSteps; ++m)
    sm100::mma_f16_ts(tmem_d, tmem_a + 8 * m, bdesc + 128 * m, idesc, m == 0 ? acc_first : 1u);
}

#ifdef KB_PF_CTA_TRACE
// per-CTA %globaltimer stamps of one launch (tools/pf_cta_trace.py): 0 entry,
// 1 first S seen (softmax warp 0), 2 last P published (warp 0), 3 exit; 4 SM id
__device__ unsigned long long g_pf_cta[8192][5];
__device__ __forceinline__ unsigned long long pf_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PF_CTA(slot)                                                                       \
  do {                                                                                     \
    const unsigned cta_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);  \
    if (cta_ < 8192) g_pf_cta[cta_][slot] = pf_gtimer();                                   \
  } while (0)
#else
#define PF_CTA(slot) \
  do {               \
  } while (0)
#endif

#ifdef KB_PF_TRACE
// per-tile clock64 stamps of one CTA (grid (0,0,0)), printed at its end:
// [t][j][slot] -- 0 S ready (softmax), 1 p_lo published, 2 p_hi published,
// 3 MMA saw p_lo, 4 PV_lo issued, 5 MMA saw p_hi, 6 PV_hi issued,
// 7 QK(t, j) issued
__device__ long long g_pft[2][128][8];
#define PFT(slot, t, j)                                                                   \
  do {                                                                                    \
    if (lane == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 128) \
      g_pft[t][j][slot] = clock64();                                                      \
  } while (0)
#else
#define PFT(slot, t, j) \
  do {                  \
  } while (0)
#endif

struct PrefillMisc {
  uint64_t full[kPfStages];
  uint64_t empty[kPfStages];
  uint64_t s_full[2];
  uint64_t p_lo[2];   // P of keys 0-63 of tile t stored (PV may start on them)
  uint64_t p_hi[2];   // P of keys 64-127 stored
  uint64_t pv_lo[2];  // the PV K-steps over keys 0-63 of tile t completed
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
                  float scale_log2, uint8_t* __restrict__ part) {
  using namespace sm100;
  constexpr int kPPT = kPfTile / kB;
  const int hq = blockIdx.y;
#ifndef KB_PF_LIGHT_FIRST
  // the causal row tiles furthest down see the most keys: dispatch them first
  const int seq = blockIdx.x / mtiles, mt = mtiles - 1 - (int)(blockIdx.x % mtiles);
#else
  const int seq = blockIdx.x / mtiles, mt = blockIdx.x % mtiles;  // mt: 256-row CTA tile
#endif
  const int64_t unit_x = (int64_t)seq * mtiles + mt;  // partials index (prefill_combine_kernel)
  const int split = blockIdx.z, splits = gridDim.z;
  const int h = hq / (Hq / Hkv);
  const int qlen = q_len[seq], pre = prefix[seq], qo = q_off[seq];
  const int row0 = mt * 2 * kPfTile;
  if (row0 >= qlen) return;  // grid is sized for the longest chunk
  const int rows = min(2 * kPfTile, qlen - row0);
  const int kv_len = pre + row0 + rows;  // keys visible to the last row
  const int nt_all = (kv_len + kPfTile - 1) / kPfTile;
  // KV split (flash-decoding style, for wave balance): this CTA takes key
  // tiles [j0, j0 + nt); the partial (O, m, l) goes to `part` and
  // prefill_combine_kernel merges the splits
  const int j0 = (int)((int64_t)split * nt_all / splits);
  const int nt = (int)((int64_t)(split + 1) * nt_all / splits) - j0;
  if (nt <= 0) {
    if (splits > 1 && threadIdx.x < 2 * kPfTile) {  // empty split: l = 0
      const int64_t u = (unit_x * Hq + hq) * splits + split;
      float* ml = reinterpret_cast<float*>(part + (int64_t)gridDim.x * Hq * splits * 2 * kPfTile * 256) +
                  (u * 2 * kPfTile + threadIdx.x) * 2;
      ml[0] = -INFINITY;
      ml[1] = 0.f;
    }
    return;
  }
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) PF_CTA(0);
#ifdef KB_PF_CTA_TRACE
  if (tid == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const unsigned cta_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    if (cta_ < 8192) g_pf_cta[cta_][4] = smid;
  }
#endif

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
        mbar_init(&misc->p_lo[t], kPArrivals);
        mbar_init(&misc->p_hi[t], kPArrivals);
        mbar_init(&misc->pv_lo[t], 1);
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
  // register rebalancing (per SMSP: 2 softmax warps + 1 warp of warpgroup 2):
  // the softmax rows keep all 128 S values in registers
  if (warp >= 8) {
#ifndef KB_PF_NO_SETMAXNREG
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kPfRegsProducer));
#endif
  if (warp >= 10) {
    // spare warps of warpgroup 2: nothing to do until the final barrier
  } else if (warp == 8) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      for (int j = 0; j < nt; ++j) {
        const int stage = j % kPfStages;
        if (j >= kPfStages) mbar_wait(&misc->empty[stage], ((j / kPfStages) - 1) & 1);
        int32_t pages[kPPT];
        int npg = 0;
#pragma unroll
        for (int k = 0; k < kPPT; ++k) {
          const int pi = (j0 + j) * kPPT + k;
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
    // warp-uniform TMEM base: with the shuffle the compiler keeps the MMA
    // operands in uniform registers (no per-MMA ELECT / R2UR.BROADCAST loop)
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    constexpr uint32_t kIdQK = idesc_bf16_f32(128, 128, false, false);
    constexpr uint32_t kIdPV = idesc_f16_f32(128, 128, false, true);  // P fp16, V fp16
#ifdef KB_PF_TIMING
    long long w_full = 0, w_p = 0, w_all = 0, w_iqk = 0, w_ipv = 0;
    const long long w_start = clock64();
#endif
    auto issue_qk = [&](int t, int j) {
      const int stage = j % kPfStages;
      if (t == 0) {
#ifdef KB_PF_TIMING
        const long long c0 = clock64();
#endif
        mbar_wait(&misc->full[stage], (j / kPfStages) & 1);
#ifdef KB_PF_TIMING
        w_full += clock64() - c0;
#endif
        tc_fence_after();
      }
#ifdef KB_PF_TIMING
      const long long ci = clock64();
#endif
#ifdef KB_PF_LANE0_MMA
      if (lane == 0) {
        mma_ss_k128(tm + t * 128, sw128_desc(smem_u32(sQ + t * kPfQ), 16, 1024),
                    sw128_desc(smem_u32(smem + stage * kPfKV), 16, 1024), kIdQK);
        mma_commit(&misc->s_full[t]);
      }
#else
      mma_ss_k128_w(tm + t * 128, sw128_desc(smem_u32(sQ + t * kPfQ), 16, 1024),
                    sw128_desc(smem_u32(smem + stage * kPfKV), 16, 1024), kIdQK);
      mma_commit_w(&misc->s_full[t]);
#endif
      __syncwarp();
      PFT(7, t, j);
#ifdef KB_PF_TIMING
      w_iqk += clock64() - ci;
#endif
    };
    auto issue_pv = [&](int t, int j) {
      // keys 0-63 as soon as their P is stored, keys 64-127 after the rest:
      // the first half of P.V overlaps the second half of the softmax
      const int stage = j % kPfStages;
      const uint64_t vdesc = sw128_desc(smem_u32(smem + stage * kPfKV + 2 * kPfHalf), kPfHalf, 1024);
#ifdef KB_PF_TIMING
      const long long c0 = clock64();
#endif
      mbar_wait(&misc->p_lo[t], j & 1);
      PFT(3, t, j);
#ifdef KB_PF_TIMING
      w_p += clock64() - c0;
#endif
      tc_fence_after();
#ifdef KB_PF_TIMING
      const long long ci = clock64();
#endif
#ifdef KB_PF_LANE0_MMA
      if (lane == 0) {
        // 16-key group m: P (fp16 pairs) at TMEM column 8m, V rows 16m..16m+15
        mma_ts_steps<kPSplit / 8>(tm + 256 + t * 128, tm + t * 128, vdesc, kIdPV, j > 0 ? 1u : 0u);
        mma_commit(&misc->pv_lo[t]);
      }
#else
      if constexpr (kPSplit == 32) {
        mma_ts_k64_w(tm + 256 + t * 128, tm + t * 128, vdesc, kIdPV, j > 0 ? 1u : 0u);
      } else if (lane == 0) {
        mma_ts_steps<kPSplit / 8>(tm + 256 + t * 128, tm + t * 128, vdesc, kIdPV, j > 0 ? 1u : 0u);
      }
      mma_commit_w(&misc->pv_lo[t]);
#endif
      __syncwarp();
      PFT(4, t, j);
      mbar_wait(&misc->p_hi[t], j & 1);
      PFT(5, t, j);
      tc_fence_after();
#ifdef KB_PF_LANE0_MMA
      if (lane == 0) {
        mma_ts_steps<(64 - kPSplit) / 8>(tm + 256 + t * 128, tm + t * 128 + kPSplit,
                                         vdesc + 16 * kPSplit, kIdPV, 1u);
        // O_t is read only by the epilogue: signal once, after the last tile
        if (j == nt - 1) mma_commit(&misc->o_done[t]);
        if (t == 1) mma_commit(&misc->empty[stage]);
      }
#else
      if constexpr (kPSplit == 32) {
        mma_ts_k64_w(tm + 256 + t * 128, tm + t * 128 + kPSplit, vdesc + 16 * kPSplit, kIdPV, 1u);
      } else if (lane == 0) {
        mma_ts_steps<(64 - kPSplit) / 8>(tm + 256 + t * 128, tm + t * 128 + kPSplit,
                                         vdesc + 16 * kPSplit, kIdPV, 1u);
      }
      // O_t is read only by the epilogue: signal once, after the last tile
      if (j == nt - 1) mma_commit_w(&misc->o_done[t]);
      if (t == 1) mma_commit_w(&misc->empty[stage]);
#endif
      __syncwarp();
      PFT(6, t, j);
#ifdef KB_PF_TIMING
      w_ipv += clock64() - ci;
#endif
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
#ifdef KB_PF_TIMING
    w_all = clock64() - w_start;
    if (lane == 0 && blockIdx.x == 7 && blockIdx.y == 0 && blockIdx.z == 0)
      printf("pf-timing mma: tiles %d wait-full %lld wait-p %lld issue-qk %lld issue-pv %lld "
             "total %lld per tile\n", nt, w_full / nt, w_p / nt, w_iqk / nt, w_ipv / nt,
             w_all / nt);
#endif
  }
  } else {
    // ------------------------------------------------ softmax warpgroup t
#ifndef KB_PF_NO_SETMAXNREG
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kPfRegsSoftmax));
#endif
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
#ifdef KB_PF_TIMING
    long long t_wait = 0, t_soft = 0, t_a = 0, t_b = 0, t_c = 0;
#endif
    for (int j = 0; j < nt; ++j) {
#ifdef KB_PF_TIMING
      const long long tw0 = clock64();
#endif
      mbar_wait(&misc->s_full[t], j & 1);
      // observe the previous tile's pv_lo phase (complete: its P.V ran before
      // this QK on the in-order tensor pipe).  Only the rare rescale path
      // needs the barrier, but every phase is waited so that no arrival
      // lands on a completed, unobserved phase (compute-sanitizer synccheck)
      if (j > 0) mbar_wait(&misc->pv_lo[t], (j - 1) & 1);
      if ((warp & 3) == 0) PFT(0, t, j);
      if (tid == 0 && j == 0) PF_CTA(1);
#ifdef KB_PF_TIMING
      const long long tw1 = clock64();
      t_wait += tw1 - tw0;
      t_a -= tw1; t_b -= tw1; t_c -= tw1;
#endif
      tc_fence_after();
      const int kbase = (j0 + j) * kPfTile;
      // Tiles wholly below the warp's first query position need no mask
      // (warp-uniform); diagonal / tail tiles take the masked path.
      const int warp_q0 = pre + row0 + t * kPfTile + (warp & 3) * 32;
      const bool full_tile = kbase + kPfTile - 1 <= warp_q0 &&
                             row0 + t * kPfTile + (warp & 3) * 32 + 31 < qlen;
      // the whole S row (128 columns) in registers: one TMEM round trip per
      // tile, the max and the exponentials both read the registers
      uint32_t sr[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32_async(s_addr + c * 32, sr[c]);
      tmem_ld_wait();
#ifdef KB_PF_TIMING
      t_a += clock64();
#endif
      // Once every row of the warp has a reference max, the tile goes
      // straight to the exponentials and the row max rides along (one pass
      // over the registers); only when some x = s*scale - m_ref exceeds the
      // lazy-rescale bound does the warp rescale and recompute P.  The first
      // tile of a row takes the max pass first.
      const bool fast = __all_sync(0xffffffffu, m_ref != -INFINITY);
      auto rescale_o = [&](float alpha) {
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
      };
      if (!fast) {
        float mr8[8];  // eight independent 3-input max chains
#pragma unroll
        for (int k = 0; k < 8; ++k) mr8[k] = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (full_tile) {
#pragma unroll
            for (int i = 0; i < 32; i += 2)
              mr8[(i >> 1) & 7] = fmaxf(mr8[(i >> 1) & 7], fmaxf(__uint_as_float(sr[c][i]),
                                                                 __uint_as_float(sr[c][i + 1])));
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const bool ok = row_ok && (kbase + c * 32 + i) <= qpos;
              mr8[i & 7] = fmaxf(mr8[i & 7], ok ? __uint_as_float(sr[c][i]) : -INFINITY);
            }
          }
        }
        const float mraw = fmaxf(fmaxf(fmaxf(mr8[0], mr8[1]), fmaxf(mr8[2], mr8[3])),
                                 fmaxf(fmaxf(mr8[4], mr8[5]), fmaxf(mr8[6], mr8[7])));
        const float mx = mraw * scale_log2;
        // lazy rescale: move the reference max only when it grows by > 2^8.
        // TMEM ld/st are warp-collective, so the whole warp rescales when any
        // of its rows needs it (alpha = 1 for the others).
        const bool need = mx > m_ref + kRescaleLog2;
        if (__any_sync(0xffffffffu, need)) {
          const float alpha = !need ? 1.f : (m_ref == -INFINITY ? 0.f : exp2f(m_ref - mx));
          rescale_o(alpha);
          if (need) {
            l_run *= alpha;
            m_ref = mx;
          }
        }
      }
#ifdef KB_PF_TIMING
      t_b += clock64();
#endif
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
      // fp16, kb_append.cu), written over S: key pair p lands in P column p
      // (columns [0, 64)) -- columns whose S values were consumed.  The first
      // kPSplit pairs are published together (p_lo: their P.V starts), the
      // rest after (p_hi), so only the tail's P.V and the next QK sit between
      // this tile's softmax and the next one.
      float2 rs2[4] = {};  // four partial sums: no 64-long dependent add chain
      const bool live = m_ref != -INFINITY;
      const float2 sc2 = make_float2(scale_log2, scale_log2);
      float2 nm2 = make_float2(-m_ref, -m_ref);
      // one straight-line body per case: unmasked tiles carry no selects
      auto p_chunk = [&](auto masked, auto p0, auto np, auto& w) {
        constexpr bool kMasked = decltype(masked)::value;
        constexpr int P0 = decltype(p0)::value, NP = decltype(np)::value;
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          const int p = P0 + i;
          const int col = 2 * p;  // key within the tile
          const float2 sv = make_float2(__uint_as_float(sr[col >> 5][col & 31]),
                                        __uint_as_float(sr[col >> 5][(col & 31) + 1]));
          const float2 xv = ffma2(sv, sc2, nm2);
          float2 v;
          if ((p & 31) % kEmuEvery == kEmuEvery - 1) {
            v = exp2_fma2(xv);
          } else {
            v.x = fast_exp2(xv.x);
            v.y = fast_exp2(xv.y);
          }
          if (kMasked) {
            const int key = kbase + col;
            const bool ok0 = row_ok && key <= qpos && live, ok1 = row_ok && key + 1 <= qpos && live;
            v.x = ok0 ? v.x : 0.f;
            v.y = ok1 ? v.y : 0.f;
          }
          rs2[p & 3] = fadd2(rs2[p & 3], v);
          const __half2 hp = __floats2half2_rn(v.x, v.y);
          w[i] = *reinterpret_cast<const uint32_t*>(&hp);
        }
      };
      auto store_chunk = [&](auto p0, auto np) {
        constexpr int P0 = decltype(p0)::value, NP = decltype(np)::value;
        static_assert(NP == 16 || NP == 32, "P chunks are 16 or 32 columns");
        uint32_t w[NP];
        if (full_tile) p_chunk(std::false_type{}, p0, np, w);
        else p_chunk(std::true_type{}, p0, np, w);
        if constexpr (NP == 32) tmem_st_32x32b_x32(s_addr + P0, w);
        else tmem_st_32x32b_x16(s_addr + P0, w);
      };
      auto take_rs = [&]() {
        const float r = (rs2[0].x + rs2[0].y) + (rs2[1].x + rs2[1].y) + (rs2[2].x + rs2[2].y) +
                        (rs2[3].x + rs2[3].y);
#pragma unroll
        for (int k = 0; k < 4; ++k) rs2[k] = make_float2(0.f, 0.f);
        return r;
      };
      auto publish = [&](uint64_t* bar) {
        tmem_st_wait();
        tc_fence_before();
#ifdef KB_PF_THREAD_ARRIVE
        mbar_arrive(bar);
#else
        // one arrive per warp once every lane's stores have landed (128
        // single-thread arrives on one barrier serialise in the SYNCS unit)
        __syncwarp();
        if (lane == 0) mbar_arrive(bar);
#endif
      };
      using I0 = std::integral_constant<int, 0>;
      using I16 = std::integral_constant<int, 16>;
      using I32 = std::integral_constant<int, 32>;
      using I48 = std::integral_constant<int, 48>;
      // the two publish groups: pairs [0, kPSplit) and [kPSplit, 64)
      auto store_lo = [&]() {
        store_chunk(I0{}, I32{});
        if constexpr (kPSplit == 48) store_chunk(I32{}, I16{});
      };
      auto store_hi = [&]() {
        if constexpr (kPSplit == 48) store_chunk(I48{}, I16{});
        else store_chunk(I32{}, I32{});
      };
      // max of x = s*scale - m_ref over the valid keys [k0, k1) (registers)
      auto range_xmax = [&](auto k0c, auto k1c) {
        constexpr int K0 = decltype(k0c)::value, K1 = decltype(k1c)::value;
        float m = -INFINITY;
#pragma unroll
        for (int k = K0; k < K1; ++k) {
          const bool ok = full_tile || (row_ok && (kbase + k) <= qpos);
          m = fmaxf(m, ok ? __uint_as_float(sr[k >> 5][k & 31]) : -INFINITY);
        }
        return m * scale_log2 - m_ref;
      };
      using KS = std::integral_constant<int, 2 * kPSplit>;
      using K128 = std::integral_constant<int, 128>;
      // Fast path overflow guard: a group's row sum above 2^14 means some P
      // may have left the lazily-rescaled range (and fp16's, at 2^16): take
      // the real max then, rescale, and recompute.  No per-element max
      // tracking; the comparison also catches inf / NaN sums.
      constexpr float kSumBound = 16384.f;
      store_lo();
      float rs = take_rs();
      if (fast && __any_sync(0xffffffffu, !(rs <= kSumBound))) {  // rare
        const float xmax = range_xmax(I0{}, KS{});
        const bool need = !(rs <= kSumBound);
        const float alpha = need ? exp2f(-xmax) : 1.f;  // 2^(m_ref - (m_ref + xmax))
        rescale_o(alpha);
        if (need) {
          l_run *= alpha;
          m_ref += xmax;
        }
        nm2 = make_float2(-m_ref, -m_ref);
        store_lo();  // P again with the new reference
        rs = take_rs();
      }
      l_run += rs;
      publish(&misc->p_lo[t]);
      if ((warp & 3) == 0) PFT(1, t, j);
      // the remaining keys (the P.V of the first group may already be running)
      store_hi();
      rs = take_rs();
      if (fast && __any_sync(0xffffffffu, !(rs <= kSumBound))) {
        // rare: O already holds this tile's first-group P.V under the old
        // reference -- let it land, then rescale everything so far
        const float xmax = range_xmax(KS{}, K128{});
        const bool need = !(rs <= kSumBound);
        mbar_wait(&misc->pv_lo[t], j & 1);
        tc_fence_after();
        const float alpha = need ? exp2f(-xmax) : 1.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float part[32];
          tmem_ld_32x32b_x32(o_addr + c * 32, part);
          uint32_t w[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) w[i] = __float_as_uint(part[i] * alpha);
          tmem_st_32x32b_x32(o_addr + c * 32, w);
        }
        if (need) {
          l_run *= alpha;
          m_ref += xmax;
        }
        nm2 = make_float2(-m_ref, -m_ref);
        store_hi();
        rs = take_rs();
      }
      l_run += rs;
#ifdef KB_PF_TIMING
      t_c += clock64();
#endif
      publish(&misc->p_hi[t]);
      if ((warp & 3) == 0) PFT(2, t, j);
      if (tid == 0 && j == nt - 1) PF_CTA(2);
#ifdef KB_PF_TIMING
      t_soft += clock64() - tw1;
#endif
    }
#ifdef KB_PF_TIMING
    if (lane == 0 && blockIdx.x == 7 && blockIdx.y == 0 && blockIdx.z == 0)
      printf("pf-timing warp %d tiles %d wait %lld soft %lld | ld %lld max %lld exp+st %lld\n",
             warp, nt, t_wait / nt, t_soft / nt, t_a / nt, t_b / nt, t_c / nt);
#endif
    // epilogue: O_t / l -> bf16 rows, or the split's partial (O, m, l)
    mbar_wait(&misc->o_done[t], 0);
    mbar_wait(&misc->pv_lo[t], (nt - 1) & 1);  // the last tile's phase, for synccheck
    tc_fence_after();
    if (splits > 1) {
      const int64_t u = (unit_x * Hq + hq) * splits + split;
      const int prow = t * kPfTile + r;  // row within the CTA's 256
      // partial O normalised by its own l, as fp16 (|O/l| <= max |v|; the
      // combine re-weights by l * 2^(m - M))
      int4* po = reinterpret_cast<int4*>(part + (u * 2 * kPfTile + prow) * 256);
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float part_o[32];
        tmem_ld_32x32b_x32(o_addr + c * 32, part_o);  // warp-collective
#pragma unroll
        for (int q8 = 0; q8 < 4; ++q8) {
          __half2 pk[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            pk[e] = __floats2half2_rn(part_o[q8 * 8 + 2 * e] * inv, part_o[q8 * 8 + 2 * e + 1] * inv);
          po[c * 4 + q8] = *reinterpret_cast<int4*>(pk);
        }
      }
      float* ml = reinterpret_cast<float*>(part + (int64_t)gridDim.x * Hq * splits * 2 * kPfTile * 256) +
                  (u * 2 * kPfTile + prow) * 2;
      ml[0] = l_run > 0.f ? m_ref : -INFINITY;
      ml[1] = l_run;
    } else {
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      int4* dst = reinterpret_cast<int4*>(out + ((int64_t)(qo + qrow) * Hq + hq) * 128);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float part_o[32];
        tmem_ld_32x32b_x32(o_addr + c * 32, part_o);  // warp-collective: every lane
        if (!row_ok) continue;
#pragma unroll
        for (int q8 = 0; q8 < 4; ++q8) {
          __nv_bfloat162 pk[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            pk[e] = __floats2bfloat162_rn(part_o[q8 * 8 + 2 * e] * inv,
                                          part_o[q8 * 8 + 2 * e + 1] * inv);
          dst[c * 4 + q8] = *reinterpret_cast<int4*>(pk);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tid == 0) PF_CTA(3);
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, kPfTmemCols);
  }
#ifdef KB_PF_TRACE
  if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
    __threadfence();
    const long long b = g_pft[0][0][0];
    for (int j = 0; j < min(nt, 128); ++j)
      for (int t = 0; t < 2; ++t)
        printf("pft %d %d %lld %lld %lld %lld %lld %lld %lld %lld\n", j, t, g_pft[t][j][0] - b,
               g_pft[t][j][1] - b, g_pft[t][j][2] - b, g_pft[t][j][3] - b, g_pft[t][j][4] - b,
               g_pft[t][j][5] - b, g_pft[t][j][6] - b, g_pft[t][j][7] - b);
  }
#endif
}

// Merge the KV splits of every (sequence, 256-row tile, q head) unit:
// O = sum_i O_i 2^(m_i - M) / sum_i l_i 2^(m_i - M), M = max_i m_i.
// One CTA per 64 rows of a unit (blockIdx.y = row quarter): 4x the CTAs of
// one-per-unit, so the HBM-bound merge fills the 148 SMs.
constexpr int kCombRows = 64;
__global__ void __launch_bounds__(256)
prefill_combine_kernel(const uint8_t* __restrict__ part, const int32_t* __restrict__ q_off,
                       const int32_t* __restrict__ q_len, int mtiles, int Hq, int splits,
                       __nv_bfloat16* __restrict__ out) {
  constexpr int kRows = 2 * kPfTile;
  __shared__ float s_w[kCombRows][8];
  const int unit = blockIdx.x;  // (seq * mtiles + mt) * Hq + hq
  const int hq = unit % Hq, cta = unit / Hq;
  const int seq = cta / mtiles, mt = cta % mtiles;
  const int qlen = q_len[seq], qo = q_off[seq];
  const int rbase = blockIdx.y * kCombRows;  // first row of this CTA within the unit
  const int row0 = mt * kRows + rbase;
  if (row0 >= qlen) return;
  const int64_t units = (int64_t)gridDim.x;
  const float* ml = reinterpret_cast<const float*>(part + units * splits * kRows * 256);
  if (threadIdx.x < kCombRows) {
    const int r = rbase + threadIdx.x;
    float m = -INFINITY;
    for (int s = 0; s < splits; ++s)
      m = fmaxf(m, ml[(((int64_t)unit * splits + s) * kRows + r) * 2]);
    float wsum = 0.f;
    for (int s = 0; s < splits; ++s) {
      const float* e = ml + (((int64_t)unit * splits + s) * kRows + r) * 2;
      const float w = (m == -INFINITY || e[0] == -INFINITY) ? 0.f : e[1] * exp2f(e[0] - m);
      s_w[threadIdx.x][s] = w;
      wsum += w;
    }
    const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
    for (int s = 0; s < splits; ++s) s_w[threadIdx.x][s] *= inv;
  }
  __syncthreads();
  const int rows = min(kCombRows, qlen - row0);
  // 16 threads per row, 8 fp16 (16 B) each; every split's 16 bytes of a
  // (row, chunk) are loaded before the first is used (up to 8 loads in
  // flight per thread instead of one per split in turn)
  const uint8_t* base = part + ((int64_t)unit * splits * kRows + rbase) * 256;
  const int64_t split_stride = (int64_t)kRows * 256;
  for (int i = threadIdx.x; i < rows * 16; i += blockDim.x) {
    const int r = i >> 4, c8 = i & 15;
    int4 v[8];
#pragma unroll
    for (int s = 0; s < 8; ++s)
      if (s < splits)
        v[s] = __ldcs(reinterpret_cast<const int4*>(base + s * split_stride + (int64_t)r * 256) + c8);
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      if (s >= splits) break;
      const float w = s_w[r][s];
      if (w == 0.f) continue;  // a split with no keys for this row: never written
      const __half2* h = reinterpret_cast<const __half2*>(&v[s]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __half22float2(h[e]);
        acc[2 * e] += f.x * w;
        acc[2 * e + 1] += f.y * w;
      }
    }
    __nv_bfloat162 pk[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) pk[e] = __floats2bfloat162_rn(acc[2 * e], acc[2 * e + 1]);
    reinterpret_cast<int4*>(out + ((int64_t)(qo + row0 + r) * Hq + hq) * 128)[c8] =
        *reinterpret_cast<int4*>(pk);
  }
}

}  // namespace kb

using namespace kb;

extern "C" int64_t kb_prefill_workspace_bytes(int32_t nseq, int32_t n_q_heads, int32_t max_q_len,
                                              int32_t kv_splits) {
  if (kv_splits <= 1 || nseq <= 0 || max_q_len <= 0) return 0;
  const int64_t units = (int64_t)nseq * ceil_div(max_q_len, 2 * kPfTile) * n_q_heads * kv_splits;
  return units * 2 * kPfTile * (128 * 2 + 2 * 4);  // fp16 O/l + (m, l) per row
}

extern "C" int kb_paged_prefill(kb_pool* p, int32_t layer, int32_t n_q_heads, uint64_t q,
                                uint64_t slots, uint64_t q_off, uint64_t q_len, uint64_t prefix,
                                int32_t nseq, int32_t max_q_len, float scale, uint64_t out,
                                uint64_t workspace, int32_t kv_splits, uintptr_t stream) {
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
  const int splits = kv_splits < 1 ? 1 : kv_splits;
  if (splits > 8) return fail(KB_EINVAL, "kv_splits must be <= 8");
  if (splits > 1 && !workspace) return fail(KB_EINVAL, "kv_splits > 1 needs a workspace");
  dim3 grid((unsigned)(nseq * mtiles), n_q_heads, splits);
  auto launch = [&](auto kernel) -> int {
    // per (instantiation, device): <64> and <128> share this lambda's type
    int arc = ensure_smem_attr(reinterpret_cast<const void*>(kernel), kPfSmem, p->device);
    if (arc) return arc;
    kernel<<<grid, kPfThreads, kPfSmem, st>>>(
        p->kv_tmap, reinterpret_cast<const __nv_bfloat16*>(q), p->d_bt,
        reinterpret_cast<const int32_t*>(slots), reinterpret_cast<const int32_t*>(q_off),
        reinterpret_cast<const int32_t*>(q_len), reinterpret_cast<const int32_t*>(prefix), mtiles,
        reinterpret_cast<__nv_bfloat16*>(out), Hkv, n_q_heads, p->m.num_layers, p->maxp, layer,
        scale_log2, reinterpret_cast<uint8_t*>(workspace));
    KB_LAUNCH_CHECK();
    return KB_OK;
  };
  int rc = pool_enter(p, st);
  if (rc) return rc;
  rc = B == 64 ? launch(prefill_tc_kernel<64>) : launch(prefill_tc_kernel<128>);
  if (rc) return rc;
  if (splits > 1) {
    prefill_combine_kernel<<<dim3(nseq * mtiles * n_q_heads, 2 * kPfTile / kCombRows), 256, 0,
                             st>>>(
        reinterpret_cast<const uint8_t*>(workspace), reinterpret_cast<const int32_t*>(q_off),
        reinterpret_cast<const int32_t*>(q_len), mtiles, n_q_heads, splits,
        reinterpret_cast<__nv_bfloat16*>(out));
    KB_LAUNCH_CHECK();
  }
  return pool_leave(p, st);
}

#ifdef KB_PF_CTA_TRACE
extern "C" int kb_debug_pf_cta_trace(unsigned long long* out, int32_t n) {
  if (n > 8192 * 5) n = 8192 * 5;
  return cudaMemcpyFromSymbol(out, kb::g_pf_cta, (size_t)n * 8) == cudaSuccess ? 0 : -1;
}
#endif
