// Position-sensitive content hash of device byte segments (parity checks at
// production sizes: whole weight slabs, every KV page of every resident).
//
// H(seg) = fmix(S ^ nbytes),  S = sum_j fmix(w_j ^ (j * phi))  (mod 2^64)
// over the segment's little-endian uint64 words w_j, where fmix is the
// splitmix64 finalizer and phi = 0x9E3779B97F4A7C15.  The word index enters
// every term, so a permutation of words inside a segment (or a swapped
// 16-byte vector, or a page copied to the wrong offset) changes the hash;
// the sum makes the reduction order-free, so the grid can split a segment
// over many CTAs and atomically add partials.  oracle/kvpool.py
// `hash_bytes` restates it in numpy (tests pin one against the other).
#include "kb_common.cuh"

namespace kb {

constexpr uint64_t kPhi = 0x9E3779B97F4A7C15ull;
constexpr int kHashThreads = 256;
constexpr int64_t kHashChunk = 64 << 10;  // bytes of one segment per CTA pass

__device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(kHashThreads)
hash_segments_kernel(const uint8_t* __restrict__ base, int64_t seg_bytes,
                     const int64_t* __restrict__ seg_index, int nseg, int64_t chunks_per_seg,
                     unsigned long long* __restrict__ out) {
  __shared__ uint64_t warp_sum[kHashThreads / 32];
  const int64_t jobs = (int64_t)nseg * chunks_per_seg;
  for (int64_t job = blockIdx.x; job < jobs; job += gridDim.x) {
    const int seg = (int)(job / chunks_per_seg);
    const int64_t c = job % chunks_per_seg;
    const int64_t idx = seg_index ? seg_index[seg] : seg;
    const uint8_t* p = base + idx * seg_bytes;
    const int64_t w0 = c * (kHashChunk / 8);
    const int64_t w1 = min(seg_bytes / 8, w0 + kHashChunk / 8);
    uint64_t acc = 0;
    // two words per thread per step: 16-byte loads, coalesced
    for (int64_t w = w0 + 2 * (int64_t)threadIdx.x; w < w1; w += 2 * kHashThreads) {
      const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(p + w * 8);
      acc += fmix64(v.x ^ ((uint64_t)w * kPhi));
      if (w + 1 < w1) acc += fmix64(v.y ^ ((uint64_t)(w + 1) * kPhi));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t s = 0;
#pragma unroll
      for (int i = 0; i < kHashThreads / 32; ++i) s += warp_sum[i];
      atomicAdd(out + seg, (unsigned long long)s);
    }
    __syncthreads();
  }
}

__global__ void hash_finish_kernel(unsigned long long* __restrict__ out, int nseg, int64_t seg_bytes) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nseg; i += gridDim.x * blockDim.x)
    out[i] = fmix64((uint64_t)out[i] ^ (uint64_t)seg_bytes);
}

}  // namespace kb

using namespace kb;

extern "C" int kb_hash_segments(uint64_t base, int64_t seg_bytes, uint64_t seg_index, int32_t nseg,
                                uint64_t out, uintptr_t stream) {
  if (nseg <= 0) return KB_OK;
  if (!base || !out) return fail(KB_EINVAL, "null pointer");
  if (seg_bytes <= 0 || seg_bytes % 16 || (base & 15))
    return fail(KB_EINVAL, "segments must be 16-byte aligned multiples of 16 bytes");
  cudaStream_t st = (cudaStream_t)stream;
  KB_RT(cudaMemsetAsync(reinterpret_cast<void*>(out), 0, (size_t)nseg * 8, st));
  const int64_t chunks = ceil_div(seg_bytes, kHashChunk);
  hash_segments_kernel<<<grid_for((int64_t)nseg * chunks, 1, 148 * 8), kHashThreads, 0, st>>>(
      reinterpret_cast<const uint8_t*>(base), seg_bytes, reinterpret_cast<const int64_t*>(seg_index),
      nseg, chunks, reinterpret_cast<unsigned long long*>(out));
  KB_LAUNCH_CHECK();
  hash_finish_kernel<<<grid_for(nseg, 256, 1024), 256, 0, st>>>(
      reinterpret_cast<unsigned long long*>(out), nseg, seg_bytes);
  KB_LAUNCH_CHECK();
  return KB_OK;
}
