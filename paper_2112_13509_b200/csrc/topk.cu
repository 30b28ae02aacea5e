// topk.cu — K6: per-job top-k candidates (SURVEY §8(f) NEXT 4 "top-k output"; R#19) over the
// score matrix K2 writes, and K7: the merge of per-rank lists after the multi-GPU all-gather.
//
// A candidate's key is the arg-max key of K2 (ord32(s) << 32 | (2^32 - 1 - c), 0 for NaN), so the
// k largest keys are the k best candidates in descending score order with ties to the smaller c
// (R#11) — the top-1 key is exactly autobyte_argmax's. Keys are exact, so merging per-rank lists
// gives the same result for any number of ranks.
//
// K6: one CTA (8 warps) per job. Each warp keeps its current top-32 as one key per lane (lane i =
// rank i, descending) and consumes the row 32 keys at a time: a batch none of whose keys beats
// the warp's k-th key is skipped with one ballot (after warm-up almost every batch), otherwise
// it is bitonic-sorted across the lanes and merged (max of the list against the reversed batch,
// then a bitonic merge). The 8 warp lists are merged the same way by warp 0. The row is read
// once with coalesced float4 loads, up to 8 CTAs per SM: HBM-bound (4 B per (job, candidate);
// C5 = 4.3 GB in ~0.7 ms).
#include "internal.h"
#include "ptx.cuh"

namespace ab {

constexpr int kTopkThreads = 256;

__device__ __forceinline__ unsigned long long cand_key(float s, long long c) {
  const uint32_t o = ord32(s);
  return o ? ((static_cast<unsigned long long>(o) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(c))) : 0ull;
}

// Bitonic sort of 32 keys across the lanes of a warp, descending (lane 0 = largest).
__device__ __forceinline__ unsigned long long warp_sort_desc(unsigned long long v, int lane) {
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, stride);
      const bool desc = (lane & size) == 0;          // this size-block sorts descending
      const bool lower = (lane & stride) == 0;       // the lower lane of the pair
      const bool keep_max = (lower == desc);
      v = keep_max ? (o > v ? o : v) : (o < v ? o : v);
    }
  }
  return v;
}
// Bitonic merge of a bitonic 32-sequence into descending order.
__device__ __forceinline__ unsigned long long warp_merge_desc(unsigned long long v, int lane) {
#pragma unroll
  for (int stride = 16; stride > 0; stride >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, stride);
    const bool lower = (lane & stride) == 0;
    v = lower ? (o > v ? o : v) : (o < v ? o : v);
  }
  return v;
}
// top-32 of (list, batch), both descending across lanes -> descending.
__device__ __forceinline__ unsigned long long warp_merge_lists(unsigned long long list, unsigned long long batch_desc,
                                                               int lane) {
  const unsigned long long rev = __shfl_sync(0xffffffffu, batch_desc, 31 - lane);
  const unsigned long long m = list > rev ? list : rev;   // bitonic: top half of the union
  return warp_merge_desc(m, lane);
}

__global__ void __launch_bounds__(kTopkThreads) topk_kernel(int J, long long C, const float* __restrict__ scores,
                                                            long long c_begin, int k,
                                                            unsigned long long* __restrict__ out) {
  __shared__ unsigned long long lists[kTopkThreads / 32][32];
  const int j = blockIdx.x;
  if (j >= J) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* row = scores + (size_t)j * C;
  const bool vec = (C & 3) == 0;   // every row 16-byte aligned
  unsigned long long list = 0ull;
  unsigned long long thr = 0ull;   // the warp's current k-th key
  // each warp takes 128 consecutive candidates per step (one float4 per lane) = four 32-key batches
  for (long long base = (long long)warp * 128; base < C; base += (long long)kTopkThreads * 4) {
    const long long c0 = base + 4 * lane;
    float v[4];
    if (vec && c0 + 3 < C) {
      const float4 f = __ldg(reinterpret_cast<const float4*>(row + c0));
      v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = c0 + q < C ? __ldg(row + c0 + q) : __uint_as_float(0x7FC00000u);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const unsigned long long key = cand_key(v[q], c_begin + c0 + q);   // NaN (incl. padding) -> 0
      if (!__any_sync(0xffffffffu, key > thr)) continue;
      list = warp_merge_lists(list, warp_sort_desc(key, lane), lane);
      thr = __shfl_sync(0xffffffffu, list, k - 1);
    }
  }
  lists[warp][lane] = list;
  __syncthreads();
  if (warp == 0) {
    for (int w = 1; w < kTopkThreads / 32; ++w) list = warp_merge_lists(list, lists[w][lane], lane);
    if (lane < k) out[(size_t)j * k + lane] = list;
  }
}

// K7: merge G per-rank lists [G][J][k] (each descending) per job and decode: one warp per job.
__global__ void topk_merge_kernel(int J, int G, int k, const unsigned long long* __restrict__ lists,
                                  int32_t* __restrict__ idx, float* __restrict__ score) {
  const int lane = threadIdx.x & 31;
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (j >= J) return;
  unsigned long long list = lane < k ? lists[(size_t)j * k + lane] : 0ull;
  for (int g = 1; g < G; ++g) {
    const unsigned long long other = lane < k ? lists[((size_t)g * J + j) * k + lane] : 0ull;
    list = warp_merge_lists(list, other, lane);
  }
  if (lane < k) {
    idx[(size_t)j * k + lane] = list ? static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(list & 0xFFFFFFFFull)) : -1;
    score[(size_t)j * k + lane] = list ? unord32(static_cast<uint32_t>(list >> 32)) : __uint_as_float(0x7FC00000u);
  }
}

cudaError_t launch_topk(int J, long long C, const float* scores, long long c_begin, int k, unsigned long long* out,
                        cudaStream_t s) {
  topk_kernel<<<J, kTopkThreads, 0, s>>>(J, C, scores, c_begin, k, out);
  return cudaGetLastError();
}

cudaError_t launch_topk_merge(int J, int G, int k, const unsigned long long* lists, int32_t* idx, float* score,
                              cudaStream_t s) {
  const int warps_per_block = 8;
  topk_merge_kernel<<<(J + warps_per_block - 1) / warps_per_block, 32 * warps_per_block, 0, s>>>(J, G, k, lists, idx,
                                                                                                   score);
  return cudaGetLastError();
}

}  // namespace ab
