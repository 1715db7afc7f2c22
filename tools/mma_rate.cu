// Tensor-pipe rate microbenchmark (measurement tool, not on the product
// path): one CTA per SM issues back-to-back tcgen05.mma kind::f16 of one
// shape from one thread and times them with clock64 -- cycles per MMA
// instruction and the implied dense TFLOP/s at the SM clock the run saw.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        tools/mma_rate.cu -o tools/var/mma_rate -lcuda && tools/var/mma_rate
//
// Shapes: the prefill's QK (SS, M128 N128 K16) and P.V (TS: A from TMEM),
// the decode's QK (SS, M128 N16), and N=256 for comparison.  Operands are
// zero tiles (the rate does not depend on values).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include "../paper_2412_18169_b200/csrc/kb_sm100.cuh"

using namespace kb::sm100;

constexpr int kIters = 4096;

// kBg (background work on warps 1-3 while thread 0 issues MMAs): 0 none,
// 1 TMEM loads (the softmax's S reads), 2 TMEM stores (P writes), 3 bulk
// async copies global -> shared (the K/V TMA traffic), 4 st.shared
template <int kMode, int N, bool kRand, int kBg>  // kMode 0: SS, 1: TS (A in TMEM)
__global__ void __launch_bounds__(128, 1) mma_rate(long long* cycles, const uint8_t* gsrc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint64_t bulk_bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  // operands: zeros, or random bf16 in [-2, 2) (the tensor pipe's power
  // draw depends on the data)
  for (int i = tid; i < 96 * 1024 / 4; i += 128) {
    uint32_t h = (uint32_t)i * 2654435761u;
    h ^= h >> 15;
    const uint32_t lo = 0x3f80u | ((h & 0x7f) << 0) | ((h >> 7 & 1) << 15);
    const uint32_t hi = 0x3f80u | ((h >> 8 & 0x7f) << 0) | ((h >> 15 & 1) << 15);
    reinterpret_cast<uint32_t*>(smem)[i] = kRand ? (lo | (hi << 16)) : 0u;
  }
  if (tid < 32) tmem_alloc(&tbase, 512);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bulk_bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, N, false, false);
    const uint64_t a = sw128_desc(smem_u32(smem), 16, 1024);
    const uint64_t b = sw128_desc(smem_u32(smem + 32768), 16, 1024);
    // warm-up
    for (int i = 0; i < 64; ++i) {
      if (kMode == 0) mma_f16_ss(tm, a, b, idesc, 1u);
      else mma_f16_ts(tm, tm + 256, b, idesc, 1u);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long c0 = clock64();
    for (int i = 0; i < kIters; ++i) {
      if (kMode == 0) mma_f16_ss(tm + (i & 1) * 128 * (N <= 128), a, b, idesc, 1u);
      else mma_f16_ts(tm + (i & 1) * 128 * (N <= 128), tm + 256 + 64 * (i & 1), b, idesc, 1u);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 1);
    const long long c1 = clock64();
    cycles[blockIdx.x] = c1 - c0;
    *reinterpret_cast<volatile uint32_t*>(&tbase) = 0xffffffffu;  // stop the loaders
  }
  if (kBg == 1 && tid >= 32) {
    // warps 1-3: TMEM loads of 32 columns in a loop, the softmax's S reads
    // (lanes of warp w read TMEM lanes 32w..32w+31)
    const uint32_t lane_base = (uint32_t)((tid >> 5) * 32) << 16;
    float sink = 0.f;
    while (*reinterpret_cast<volatile uint32_t*>(&tbase) != 0xffffffffu) {
      float v[32];
      tmem_ld_32x32b_x32(tm + lane_base + 384, v);
      sink += v[0];
    }
    if (sink == 12345.f) cycles[0] = 0;
  }
  if (kBg == 2 && tid >= 32) {
    const uint32_t lane_base = (uint32_t)((tid >> 5) * 32) << 16;
    uint32_t w[32];
    for (int i = 0; i < 32; ++i) w[i] = tid * 32 + i;
    while (*reinterpret_cast<volatile uint32_t*>(&tbase) != 0xffffffffu) {
      tmem_st_32x32b_x32(tm + lane_base + 448, w);
      tmem_st_wait();
    }
  }
  if (kBg == 3 && tid == 32) {
    // 32 KiB bulk copies into smem [64 KiB, 96 KiB), one in flight
    uint32_t ph = 0;
    int k = 0;
    while (*reinterpret_cast<volatile uint32_t*>(&tbase) != 0xffffffffu) {
      mbar_arrive_expect_tx(&bulk_bar, 32768);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(smem + 65536)),
          "l"(gsrc + (size_t)((blockIdx.x * 64 + (k++ & 63)) & 8191) * 32768), "r"(32768),
          "r"(smem_u32(&bulk_bar))
          : "memory");
      mbar_wait(&bulk_bar, ph);
      ph ^= 1;
    }
  }
  if (kBg == 4 && tid >= 32) {
    int4* p = reinterpret_cast<int4*>(smem + 65536) + (tid - 32);
    int i = 0;
    while (*reinterpret_cast<volatile uint32_t*>(&tbase) != 0xffffffffu) {
      p[(i & 31) * 96] = make_int4(i, i, i, i);
      ++i;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc(tm, 512);
  }
}

// The prefill's MMA stream without the softmax: per tile QK0 QK1 (SS, K-major,
// into S0 / S1) and PV0 PV1 (TS, A = P in the S columns, B = V; kVmn: V
// MN-major as the kernel stores it, else K-major), a commit after each group.
template <bool kVmn>
__global__ void __launch_bounds__(128, 1) pattern_rate(long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < 96 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (tid < 32) tmem_alloc(&tbase, 512);
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint32_t idqk = idesc_bf16_f32(128, 128, false, false);
    const uint32_t idpv = idesc_f16_f32(128, 128, false, kVmn);
    const uint64_t q0 = sw128_desc(smem_u32(smem), 16, 1024);
    const uint64_t q1 = sw128_desc(smem_u32(smem + 32768), 16, 1024);
    const uint64_t kd = sw128_desc(smem_u32(smem + 65536), 16, 1024);
    const uint64_t vd = kVmn ? sw128_desc(smem_u32(smem + 65536), 16384, 1024)
                             : sw128_desc(smem_u32(smem + 65536), 16, 1024);
    const int tiles = 256;
    long long c0 = 0;
    for (int j = 0; j < tiles + 8; ++j) {
      if (j == 8) c0 = clock64();
      for (int t = 0; t < 2; ++t) {  // QK_t: 8 K=16 steps over d (SW128 halves 16 KiB apart)
        const uint64_t qa = t ? q1 : q0;
        for (int k = 0; k < 8; ++k) {
          const uint64_t off = (k < 4 ? k * 2 : 1024 + (k - 4) * 2);
          mma_f16_ss(tm + t * 128, qa + off, kd + off, idqk, k > 0);
        }
        mma_commit(&bar[t]);
      }
      for (int t = 0; t < 2; ++t) {  // PV_t: 8 K=16 steps over keys
        for (int m = 0; m < 8; ++m)
          mma_f16_ts(tm + 256 + t * 128, tm + t * 128 + 8 * m, vd + (kVmn ? 128 : 2) * m, idpv, 1u);
        mma_commit(&bar[2 + t]);
      }
    }
    mma_commit(&bar[0]);
    tc_fence_before();
    // wait for everything: the last commit's phase parity is unknown here,
    // so drain through a fresh barrier
    mbar_init(&bar[1], 1);
    fence_barrier_init();
    mma_commit(&bar[1]);
    mbar_wait(&bar[1], 0);
    cycles[blockIdx.x] = clock64() - c0;
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc(tm, 512);
  }
}

template <bool kVmn>
void run_pattern(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  auto k = pattern_rate<kVmn>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<148, 128, 100 * 1024>>>(d);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(err));
    return;
  }
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += (double)h[i] / 148;
  printf("%-28s %7.1f cycles/MMA (32 per tile pair)\n", name, avg / (256.0 * 32));
  cudaFree(d);
}

// MMA issue under SMSP contention: warp 1 issues the prefill pattern's QK
// stream (8 K=16 steps per group, commit per group) while warps 5 and 9 --
// the same SM sub-partition -- run an FFMA/MUFU loop like the softmax warps.
// kStyle 0: each MMA asm inside `if (lane == 0)` (ptxas wraps every UTCHMMA
// in an ELECT loop); 1: the whole warp executes the asm, elect.sync inside.
__device__ __forceinline__ void mma8_lane0(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  for (int k = 0; k < 8; ++k) mma_f16_ss(d, a + 2 * k, b + 2 * k, idesc, 1u);
}
__device__ __forceinline__ void mma8_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b64 a1, b1;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 b1, %2, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
      "add.s64 a1, %1, 4;\n\tadd.s64 b1, %2, 4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
      "add.s64 a1, %1, 6;\n\tadd.s64 b1, %2, 6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
      "add.s64 a1, %1, 8;\n\tadd.s64 b1, %2, 8;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
      "add.s64 a1, %1, 10;\n\tadd.s64 b1, %2, 10;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
      "add.s64 a1, %1, 12;\n\tadd.s64 b1, %2, 12;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
      "add.s64 a1, %1, 14;\n\tadd.s64 b1, %2, 14;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc)
      : "memory");
}
template <int kStyle, bool kHog>
__global__ void __launch_bounds__(384, 1) hog_rate(long long* cycles, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int done;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 96 * 1024 / 4; i += 384) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    done = 0;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (warp == 1) {
    const uint32_t idqk = idesc_bf16_f32(128, 128, false, false);
    const uint64_t q0 = sw128_desc(smem_u32(smem), 16, 1024);
    const uint64_t kd = sw128_desc(smem_u32(smem + 65536), 16, 1024);
    const int groups = 1024;
    const long long c0 = clock64();
    for (int j = 0; j < groups; ++j) {
      if (kStyle == 0) {
        if (lane == 0) {
          mma8_lane0(tm + (j & 3) * 128, q0, kd, idqk);
          mma_commit(&bar);
        }
        __syncwarp();
      } else {
        mma8_elect(tm + (j & 3) * 128, q0, kd, idqk);
        if (lane == 0) mma_commit(&bar);
        __syncwarp();
      }
    }
    if (lane == 0) {
      tc_fence_before();
      uint64_t* b2 = &bar;
      (void)b2;
    }
    const long long c1 = clock64();
    if (lane == 0) cycles[blockIdx.x] = c1 - c0;
    if (lane == 0) done = 1;
  } else if (kHog && (warp == 5 || warp == 9)) {
    float x = tid * 1e-3f, y = 1.f, z = 0.5f;
    while (!done) {
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        float e;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x));
        y = fmaf(y, 0.999f, e);
        z = fmaf(z, 1.0001f, y);
        x = fmaf(x, 0.5f, -z * 1e-6f);
      }
    }
    if (x == 123.f) sink[tid] = y + z;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tm, 512);
  }
}

template <int kStyle, bool kHog>
void run_hog(const char* name) {
  long long* d;
  float* sk;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaMalloc(&sk, 384 * 4);
  auto k = hog_rate<kStyle, kHog>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<148, 384, 100 * 1024>>>(d, sk);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(err));
    return;
  }
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += (double)h[i] / 148;
  printf("%-34s %7.1f issue cycles/MMA\n", name, avg / (1024.0 * 8));
  cudaFree(d);
  cudaFree(sk);
}

template <int kMode, int N, bool kRand = false, int kBg = 0>
void run(const char* name, const uint8_t* gsrc) {
  long long* d;
  int* dk;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaMalloc(&dk, 4);
  auto k = mma_rate<kMode, N, kRand, kBg>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<148, 128, 100 * 1024>>>(d, gsrc);
  cudaEventRecord(e0);
  k<<<148, 128, 100 * 1024>>>(d, gsrc);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(err));
    return;
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += (double)h[i] / 148;
  const double cyc = avg / kIters;
  const double flop = 2.0 * 128 * N * 16;
  // FLOP/s from the event time (all 148 SMs, includes launch + warm-up)
  printf("%-28s %7.1f cycles/MMA  %7.0f FLOP/clk/SM  %7.1f TFLOP/s (event)\n", name, cyc,
         flop / cyc, 148.0 * (kIters + 64) * flop / (ms * 1e-3) / 1e12);
  cudaFree(d);
  cudaFree(dk);
}

int main() {
  uint8_t* g;
  cudaMalloc(&g, (size_t)8192 * 32768);  // 256 MiB: bulk copies come from HBM / L2
  cudaMemset(g, 0x3c, (size_t)8192 * 32768);
  run<0, 128>("SS M128 N128 K16 (QK)", g);
  run<1, 128>("TS M128 N128 K16 (P.V)", g);
  run<0, 256>("SS M128 N256 K16", g);
  run<0, 64>("SS M128 N64 K16", g);
  run<0, 16>("SS M128 N16 K16 (decode QK)", g);
  run<0, 128, true>("SS N128 random data", g);
  run<1, 128, true>("TS N128 random data", g);
  run<0, 128, true, 1>("SS N128 + TMEM ld", g);
  run<1, 128, true, 1>("TS N128 + TMEM ld", g);
  run<0, 128, true, 2>("SS N128 + TMEM st", g);
  run<1, 128, true, 2>("TS N128 + TMEM st", g);
  run<0, 128, true, 3>("SS N128 + bulk g->s copies", g);
  run<1, 128, true, 3>("TS N128 + bulk g->s copies", g);
  run_pattern<true>("prefill pattern, V MN-major");
  run_pattern<false>("prefill pattern, V K-major");
  run_hog<0, false>("issue lane0, no hog");
  run_hog<1, false>("issue elect-asm, no hog");
  run_hog<0, true>("issue lane0, 2 hog warps on SMSP");
  run_hog<1, true>("issue elect-asm, 2 hog warps");
  return 0;
}
