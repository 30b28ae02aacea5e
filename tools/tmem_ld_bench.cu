// tmem_ld_bench.cu — does a CTA pair's peer read TMEM slower than the leader while the leader
// issues cta_group::2 MMAs? Warps 1..4 of both CTAs loop tcgen05.ld 32x32b.x32 (+ wait::ld) on
// accumulator columns [128, 256) while warp 0 of the leader keeps M=256 N=128 MMAs (columns
// [0, 128)) in flight; prints mean cycles per load for leader and peer, with and without MMAs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tmem_ld_bench tools/tmem_ld_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2112_13509_b200/csrc/ptx.cuh"

using namespace ab;

template <bool MMA, bool SMEMST>
__global__ void __launch_bounds__(160, 1) ld_loop(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) { stop = 0; mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) { tmem_alloc2(&tmem_base, 512); tmem_relinquish2(); }
  fence_proxy_async_smem();
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t rank = cluster_ctarank();
  constexpr uint32_t idesc = umma_idesc_bf16(256, 128);
  unsigned long long cyc = 0;
  if (warp == 0) {
    if (MMA && rank == 0) {
      const uint64_t a0 = umma_desc_sw128(smem_u32(smem));
      const uint64_t b0 = umma_desc_sw128(smem_u32(smem + 131072));
      uint32_t ph = 0;
      for (int it = 0; it < iters; ++it) {
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 32; ++k)
            umma_ss2(tmem, a0 + (uint64_t)((k >> 2) * 1024 + 2 * (k & 3)), b0 + (uint64_t)(((k >> 3) & 3) * 1024 + 2 * (k & 3)),
                     idesc, k != 0);
          umma_commit2(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
  } else {
    const int quad = warp & 3;
    const uint32_t addr = tmem + (static_cast<uint32_t>(quad * 32) << 16) + 128;
    uint32_t acc = 0;
    const int nld = iters * 8;
    const long long t0 = clock64();
    for (int i = 0; i < nld; ++i) {
      uint32_t r[32];
      tmem_ld32(addr + (i & 3) * 32, r);
      tmem_ld_wait();
#pragma unroll
      for (int k = 0; k < 32; ++k) acc += r[k];
      if (SMEMST) st_shared_v4(smem_u32(smem + 196608 - 16384) + (threadIdx.x & 127) * 16 + (i & 7) * 2048, acc, acc, acc, acc);
    }
    cyc = (clock64() - t0) / nld;
    if (acc == 0xdeadbeef) out[1023] = acc;
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0) tmem_dealloc2(tmem, 512);
  if (warp == 1 && lane == 0) out[blockIdx.x] = cyc;
}

template <bool MMA, bool SMEMST>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 1024 * sizeof(unsigned long long));
  cudaMemset(d, 0, 1024 * sizeof(unsigned long long));
  auto k = ld_loop<MMA, SMEMST>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 1024);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(160);
  cfg.dynamicSmemBytes = 196608 + 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, 2000, d);
  cudaError_t err = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double lead = 0, peer = 0;
  for (int i = 0; i < 148; ++i) (i & 1 ? peer : lead) += h[i];
  printf("%-28s %s  cycles per 32-col tcgen05.ld: leader %.1f  peer %.1f\n", name, cudaGetErrorString(err), lead / 74,
         peer / 74);
  fflush(stdout);
  cudaFree(d);
}

int main() {
  run<false, false>("no MMA");
  run<true, false>("MMA running");
  run<true, true>("MMA running + smem stores");
  return 0;
}
