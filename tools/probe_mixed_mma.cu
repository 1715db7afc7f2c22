// Probe: does tcgen05.mma kind::f16 accept A = fp16 with B = bf16?
// D[128 x 16] = A[128 x 16] * B[16 x 16]^T (both K-major, SW128), fp32 acc.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe tools/probe_mixed_mma.cu
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>

#include "../paper_2412_18169_b200/csrc/kb_sm100.cuh"

using namespace kb::sm100;

__global__ void probe(const __half* A, const __nv_bfloat16* Bm, float* D, int a_f16) {
  __shared__ __align__(1024) uint8_t sA[128 * 128];
  __shared__ __align__(1024) uint8_t sB[16 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  // A: 128 rows x 16 k (32 B per row inside a 128 B swizzled row)
  for (int i = tid; i < 128 * 16; i += 128) {
    int r = i / 16, k = i % 16;
    uint16_t bits = a_f16 ? __half_as_ushort(A[i]) : __bfloat16_as_ushort(__float2bfloat16(__half2float(A[i])));
    *reinterpret_cast<uint16_t*>(sA + sw128_offset(r, k)) = bits;
  }
  for (int i = tid; i < 16 * 16; i += 128) {
    int r = i / 16, k = i % 16;
    *reinterpret_cast<__nv_bfloat16*>(sB + sw128_offset(r, k)) = Bm[i];
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(&tbase, 32);
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    uint32_t idesc = (1u << 4) | ((a_f16 ? 0u : 1u) << 7) | (1u << 10) | (2u << 17) | (8u << 24);
    mma_f16_ss(tbase, sw128_desc(smem_u32(sA), 16, 1024), sw128_desc(smem_u32(sB), 16, 1024),
               idesc, 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[8];
  tmem_ld_32x32b_x8(tbase + ((warp * 32) << 16), v);
  for (int c = 0; c < 8; ++c) D[tid * 16 + c] = v[c];
  tmem_ld_32x32b_x8(tbase + ((warp * 32) << 16) + 8, v);
  for (int c = 0; c < 8; ++c) D[tid * 16 + 8 + c] = v[c];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 32);
}

int main() {
  const int M = 128, N = 16, K = 16;
  __half* hA; __nv_bfloat16* hB; float* hD;
  cudaMallocManaged(&hA, M * K * 2);
  cudaMallocManaged(&hB, N * K * 2);
  cudaMallocManaged(&hD, M * N * 4);
  srand(1);
  for (int i = 0; i < M * K; ++i) hA[i] = __float2half((rand() % 2001 - 1000) / 997.0f);
  for (int i = 0; i < N * K; ++i) hB[i] = __float2bfloat16((rand() % 2001 - 1000) / 613.0f);
  for (int mode = 1; mode >= 0; --mode) {
    probe<<<1, 128>>>(hA, hB, hD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d: error %s\n", mode, cudaGetErrorString(e)); return 1; }
    double maxerr = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) {
          float a = mode ? __half2float(hA[m * K + k]) : __bfloat162float(__float2bfloat16(__half2float(hA[m * K + k])));
          ref += (double)a * __bfloat162float(hB[n * K + k]);
        }
        maxerr = fmax(maxerr, fabs(ref - hD[m * N + n]));
      }
    printf("mode %s: max abs err vs fp64 ref = %.3e\n", mode ? "A=f16,B=bf16" : "A=bf16,B=bf16", maxerr);
  }
  return 0;
}
