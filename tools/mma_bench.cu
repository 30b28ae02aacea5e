// mma_bench.cu — calibration micro-benchmark: cycles per tcgen05.mma (kind::f16, bf16 -> fp32)
// for the shapes K2 uses, issued back to back from one elected thread with operands resident in
// shared memory / TMEM (no TMA, no epilogue). Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -std=c++17 -o mma_bench tools/mma_bench.cu ; run on a B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2112_13509_b200/csrc/ptx.cuh"

using namespace ab;

// WALK: A and B descriptors walk over a 128 KB / 64 KB smem region like K2 (else one 4 KB atom)
// NOISE: warps 1..3 store 16 B/thread to a separate smem region in a loop (epilogue-like traffic)
// K2LIKE: per 4 MMAs a try_wait on an already-complete barrier + fence + commit (no completion wait)
// NOISE < 0: warp 1 streams 16 KB TMA bulk copies from global memory into its own smem region
template <int CG, int N, bool TS, int PER_COMMIT, bool WALK = false, int NOISE = 0, bool K2LIKE = false, bool TF32 = false>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, unsigned long long* out, const uint8_t* gsrc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ volatile int stop;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar, done_bar, tbar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (196608 + 16384) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) stop = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1); mbar_init(&done_bar, 1); mbar_init(&tbar, 1);
    fence_barrier_init();
    mbar_arrive(&done_bar);   // phase 0 of done_bar completes immediately: try_wait(0) always succeeds
  }
  if (warp == 0) {
    if (CG == 2) { tmem_alloc2(&tmem_base, 512); tmem_relinquish2(); }
    else { tmem_alloc(&tmem_base, 512); tmem_relinquish(); }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
  constexpr uint32_t idesc = TF32 ? umma_idesc_tf32(128 * CG, N) : umma_idesc_bf16(128 * CG, N);
  long long t0 = clock64(), t1 = t0;
  if (warp == 0 && rank == 0) {
    const uint64_t a0 = umma_desc_sw128(smem_u32(smem));
    const uint64_t b0 = umma_desc_sw128(smem_u32(smem + 131072));
    uint32_t ph = 0;
    t0 = clock64();
    if (K2LIKE) {
      for (int it = 0; it < iters; it += 4) {
        mbar_wait(&done_bar, 0);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int ks = (it + k) & 31;
            const uint64_t ad = a0 + (uint64_t)((ks >> 2) * 1024 + 2 * (ks & 3));
            const uint64_t bd = b0 + (uint64_t)(((((it + k) >> 2) & 3) * 1024 + 2 * (ks & 3)));
            if (CG == 2) umma_ss2(tmem, ad, bd, idesc, (it + k) != 0);
            else umma_ss(tmem, ad, bd, idesc, (it + k) != 0);
          }
          if (CG == 2) umma_commit2(&tbar); else umma_commit(&tbar);
        }
        __syncwarp();
      }
      if (elect_one()) { if (CG == 2) umma_commit2(&bar); else umma_commit(&bar); }
      __syncwarp();
      mbar_wait(&bar, 0);
    }
    for (int it = 0; it < (K2LIKE ? 0 : iters); it += PER_COMMIT) {
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < PER_COMMIT; ++k) {
          const uint32_t acc = (it + k) != 0;
          const int ks = WALK ? ((it + k) & 31) : (k & 3);            // K step inside a 512-wide row
          const uint64_t ad = a0 + (uint64_t)((ks >> 2) * 1024 + 2 * (ks & 3));
          const uint64_t bd = b0 + (uint64_t)(WALK ? ((((it + k) >> 2) & 3) * 1024 + 2 * (ks & 3)) : 2 * (k & 3));
          const uint32_t at = tmem + 256 + ks * 8;
          if (TF32) {
            umma_ss_tf32(tmem, ad, bd, idesc, acc);
          } else if (CG == 2) {
            if (TS) umma_ts2(tmem, at, bd, idesc, acc);
            else umma_ss2(tmem, ad, bd, idesc, acc);
          } else {
            if (TS) umma_ts(tmem, at, bd, idesc, acc);
            else umma_ss(tmem, ad, bd, idesc, acc);
          }
        }
        if (CG == 2) umma_commit2(&bar); else umma_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, ph);   // wait for this batch (worst case: no queue overlap across batches)
      ph ^= 1;
    }
    t1 = clock64();
    stop = 1;
  } else if (NOISE < 0 && warp == 1 && rank == 0) {
    uint32_t tph = 0;
    uint64_t* b2 = &tbar;
    __shared__ __align__(8) uint64_t lbar;
    if (elect_one()) mbar_init(&lbar, 1);
    __syncwarp();
    b2 = &lbar;
    for (int r = 0; !stop; ++r) {
      if (elect_one()) {
        mbar_arrive_expect_tx(b2, 16384);
        bulk_g2s(smem + 196608, gsrc + (size_t)((r + blockIdx.x) & 63) * 16384, 16384, b2, l2_policy_evict_last());
      }
      __syncwarp();
      mbar_wait(b2, tph);
      tph ^= 1;
    }
  } else if (NOISE > 0 && warp >= 1 && warp <= NOISE && rank == 0) {
    // epilogue-like smem store traffic into its own 16 KB region
    const uint32_t base = smem_u32(smem + 196608) + (threadIdx.x & 127) * 16;
    while (!stop) {
#pragma unroll
      for (int r = 0; r < 8; ++r) st_shared_v4(base + ((r * 2048) & 16383), r, r, r, r);
    }
  }
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 0) {
    if (CG == 2) tmem_dealloc2(tmem, 512); else tmem_dealloc(tmem, 512);
  }
  if (threadIdx.x == 0 && rank == 0) out[blockIdx.x] = t1 - t0;
}

static uint8_t* g_src = nullptr;
template <int CG, int N, bool TS, int PER_COMMIT, bool WALK = false, int NOISE = 0, bool K2LIKE = false,
          bool TF32 = false>
void run(const char* name, int iters) {
  if (!g_src) { cudaMalloc(&g_src, 64 * 16384); cudaMemset(g_src, 0, 64 * 16384); }
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  cudaMemset(d, 0, 148 * sizeof(unsigned long long));
  auto k = mma_loop<CG, N, TS, PER_COMMIT, WALK, NOISE, K2LIKE, TF32>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 16384 + 1024);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 196608 + 16384 + 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const uint8_t* src = g_src;
  cudaLaunchKernelEx(&cfg, k, iters, d, src);   // warm-up
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, iters, d, src);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = 0; int n = 0;
  for (int i = 0; i < 148; ++i) if (h[i]) { cyc += h[i]; ++n; }
  cyc /= n;
  const int kstep = TF32 ? 8 : 16;
  const double flop = 2.0 * 128 * CG * N * kstep * (double)iters * (148 / CG);
  printf("%-34s %s  cycles/MMA %7.1f  per-SM FLOP/cycle %7.0f  chip TFLOP/s %7.1f\n", name, cudaGetErrorString(err),
         cyc / iters, 2.0 * 128 * N * kstep / (cyc / iters), flop / (ms * 1e-3) / 1e12);
  fflush(stdout);
  cudaFree(d);
}

int main(int argc, char** argv) {
  const int it = 1 << 16;
  if (argc > 1) {   // tf32 shapes of the K4 tile (kind::tf32, K = 8 per instruction)
    run<1, 64, false, 12, true, 0, false, true>("cg1 tf32 M128 N64 (12/commit)", it);
    run<1, 128, false, 12, true, 0, false, true>("cg1 tf32 M128 N128 (12/commit)", it);
    run<1, 256, false, 12, true, 0, false, true>("cg1 tf32 M128 N256 (12/commit)", it);
    run<1, 64, false, 48, true, 0, false, true>("cg1 tf32 M128 N64 (48/commit)", it);
    run<1, 128, false, 32, true>("cg1 bf16 M128 N128 (32/commit)", it);
    return 0;
  }
  run<1, 128, false, 32>("cg1 M128 N128 SS (32/commit)", it);
  run<1, 128, false, 32, true, 0, true>("cg1 K2-like loop", it);
  run<1, 128, false, 32, true, -1, true>("cg1 K2-like loop + TMA stream", it);
  run<1, 128, false, 32, true, -1>("cg1 SS walk + TMA stream", it);
  run<2, 128, false, 32, true, 0, true>("cg2 K2-like loop", it);
  run<2, 128, false, 32, true, -1, true>("cg2 K2-like loop + TMA stream", it);
  return 0;
}
