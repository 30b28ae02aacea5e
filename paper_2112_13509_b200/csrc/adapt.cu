// adapt.cu — K4: fused online adaptation (forward with stash, backward, SGD) in ONE cooperative
// persistent kernel ("offline training, online adapting ... transfer learning";
// P:438 triggered when prediction error > 10%; R#12 objective, R#13 head-only plain SGD).
//
// Per step, phases separated by a grid-wide barrier:
//   F_k   H_k = ReLU(H_{k-1} W_k^T + b_k), k = 1..L (H_0 = Z = [x | u])      fp32 SIMT tiles
//   OUT   R = mask_b (H_L W_o^T + b_o - V_bar) / B                            (dV of the objective)
//   BO    dW_o = R^T H_L, db_o = colsum R, D_L = (R W_o) * [H_L > 0]
//   Bk    dW_k = D_k^T H_{k-1}, db_k = colsum D_k, D_{k-1} = (D_k W_k) * [H_{k-1} > 0]  (pre-update W_k)
//   SGD   theta -= lr * grad over all head parameters
// Every output element is produced by exactly one thread with a fixed summation order, so the
// update is deterministic and replicas on different GPUs stay bit-identical without traffic.
// The work is ~3x a B-row forward (5 GFLOP at B=1024, 4x512): latency-bound, << 1% of a C5 step;
// fp32 SIMT keeps the gradient well inside the parity tolerance (K4).
#include "internal.h"
#include "ptx.cuh"

namespace ab {

constexpr int kAdaptThreads = 256;
constexpr int kTM = 64, kTN = 64, kTK = 16;
constexpr int kSplitK = kAdaptSplitK;   // K = B splits of the weight-gradient GEMMs (partials in grads[kSplitK][total])

struct Gemm {
  int M, N, K;
  const float* A; long long lam, lak;    // A(m, k) = A[m*lam + k*lak]
  const float* Bm; long long lbk, lbn;   // B(k, n) = Bm[k*lbk + n*lbn]
  float* C; long long ldc;               // C[m*ldc + n]
  int mode;                              // 0: ReLU(acc + bias[n]); 1: acc * [mask(m,n) > 0]; 2: acc;
                                         // 3: (acc + bias[n] - vbar[m][n]) * [n < nvalid[m]] * scale
  const float* bias;
  const float* mask; long long ldmask;
  const float* vbar; const int32_t* nvalid; float scale;
  int ksplit;                            // split-K count (mode 2 only): partial s -> C + s*cpart
  long long cpart;
  __device__ int tiles() const { return ((M + kTM - 1) / kTM) * ((N + kTN - 1) / kTN) * (ksplit > 1 ? ksplit : 1); }
};

constexpr int kStages = 3;   // cp.async pipeline depth of the SIMT GEMM tiles

__device__ __forceinline__ void cp_async4(float* smem_dst, const float* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(smem_dst)), "l"(src),
               "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// One 64 x 64 output tile (or one K-slice of it for split-K). Each thread owns 4 x 4 outputs;
// 16-wide K slices of both operands stream through a 3-stage cp.async ring (zero-filled at the
// edges), so global-load latency overlaps the FMAs of the two slices ahead.
__device__ void gemm_tile(const Gemm& g, int work, float (*As)[kTK][kTM + 4], float (*Bs)[kTK][kTN + 4]) {
  const int tiles_n = (g.N + kTN - 1) / kTN;
  const int tiles_mn = ((g.M + kTM - 1) / kTM) * tiles_n;
  const int split = g.ksplit > 1 ? work / tiles_mn : 0;
  const int tile = work % tiles_mn;
  const int m0 = (tile / tiles_n) * kTM, n0 = (tile % tiles_n) * kTN;
  int kbeg = 0, kend = g.K;
  if (g.ksplit > 1) {
    const int chunk = ((g.K + g.ksplit - 1) / g.ksplit + kTK - 1) / kTK * kTK;
    kbeg = split * chunk;
    kend = min(g.K, kbeg + chunk);
  }
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  int aml[4], akl[4], bnl[4], bkl[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int e = tid + r * kAdaptThreads;
    if (g.lak == 1) { akl[r] = e % kTK; aml[r] = e / kTK; } else { aml[r] = e % kTM; akl[r] = e / kTM; }
    if (g.lbk == 1) { bkl[r] = e % kTK; bnl[r] = e / kTK; } else { bnl[r] = e % kTN; bkl[r] = e / kTN; }
  }
  const int nk = kend > kbeg ? (kend - kbeg + kTK - 1) / kTK : 0;
  auto issue = [&](int it) {
    if (it < nk) {
      const int k0 = kbeg + it * kTK, st = it % kStages;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int m = m0 + aml[r], k = k0 + akl[r];
        const bool va = m < g.M && k < kend;
        cp_async4(&As[st][akl[r]][aml[r]], va ? g.A + (m * g.lam + k * g.lak) : g.A, va);
        const int n = n0 + bnl[r], kk = k0 + bkl[r];
        const bool vb = n < g.N && kk < kend;
        cp_async4(&Bs[st][bkl[r]][bnl[r]], vb ? g.Bm + (kk * g.lbk + n * g.lbn) : g.Bm, vb);
      }
    }
    cp_async_commit();   // (empty groups keep the wait arithmetic uniform)
  };
  float acc[4][4] = {};
  __syncthreads();       // the ring may still be read by the previous tile
  issue(0);
  issue(1);
  for (int it = 0; it < nk; ++it) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    issue(it + 2);       // overwrites the stage read two slices ago (all threads are past it)
    const int st = it % kStages;
#pragma unroll
    for (int kk = 0; kk < kTK; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&As[st][kk][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[st][kk][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[i][jj] = fmaf(av[i], bv[jj], acc[i][jj]);
    }
  }
  cp_async_wait<0>();
  float* C = g.C + (g.ksplit > 1 ? split * g.cpart : 0);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= g.M) continue;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int n = n0 + tx * 4 + jj;
      if (n >= g.N) continue;
      float v = acc[i][jj];
      if (g.mode == 0) v = relu(v + g.bias[n]);
      else if (g.mode == 1) v = g.mask[m * g.ldmask + n] > 0.f ? v : 0.f;
      else if (g.mode == 3) v = (n < g.nvalid[m]) ? (v + g.bias[n] - g.vbar[m * 16 + n]) * g.scale : 0.f;
      C[m * g.ldc + n] = v;
    }
  }
}

#ifdef AB_STATS
__device__ unsigned long long g_adapt_phase[64];   // block 0: clock at entry of each grid barrier
__device__ int g_adapt_nphase;
#endif
__device__ __forceinline__ void grid_sync(unsigned int* bar, unsigned int& gen) {
#ifdef AB_STATS
  if (blockIdx.x == 0 && threadIdx.x == 0 && g_adapt_nphase < 64) g_adapt_phase[g_adapt_nphase++] = clock64();
#endif
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int g = gen;
    if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(&bar[1], 1u);
    } else {
      unsigned int cur;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
      } while (cur == g);
    }
    gen = g + 1;
    __threadfence();
  }
  __syncthreads();
}

// Column sums over the batch as kSplitK partials (like the split-K weight gradients, summed in fixed
// order by the SGD sweep): out[s * stride + n] = sum_{b in segment s} X[b][n]. One warp per
// (32-column group, segment); each lane walks its column down the segment (coalesced rows).
__device__ void colsum_split(const float* X, int B, int N, long long ld, float* out, long long stride) {
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  const int groups = (N + 31) / 32, seg = (B + kSplitK - 1) / kSplitK;
  for (int w = gwarp; w < groups * kSplitK; w += nwarps) {
    const int sgi = w / groups, n = (w % groups) * 32 + lane;
    const int b0 = sgi * seg, b1 = min(B, b0 + seg);
    if (n >= N) continue;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    int b = b0;
    for (; b + 3 < b1; b += 4) {
      a0 += X[(long long)b * ld + n];
      a1 += X[(long long)(b + 1) * ld + n];
      a2 += X[(long long)(b + 2) * ld + n];
      a3 += X[(long long)(b + 3) * ld + n];
    }
    for (; b < b1; ++b) a0 += X[(long long)b * ld + n];
    out[sgi * stride + n] = (a0 + a1) + (a2 + a3);
  }
}

__global__ void __launch_bounds__(kAdaptThreads) adapt_kernel(const __grid_constant__ AdaptParams p) {
  __shared__ __align__(16) float As[kStages][kTK][kTM + 4];
  __shared__ __align__(16) float Bs[kStages][kTK][kTN + 4];
  const int B = p.B, H = p.H, L = p.L;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gthreads = gridDim.x * blockDim.x;
  unsigned int gen = 0;
  if (threadIdx.x == 0) {
    unsigned int cur;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(p.barrier + 1) : "memory");
    gen = cur;
  }
  float* P = p.params;
  float* Gr = p.grads;
  // workspace carve-up
  float* Z = p.ws;                              // [B][84]
  float* Hs = Z + (size_t)B * kZDim;            // [L][B][H], H_k at Hs + (k-1)*B*H
  float* R = Hs + (size_t)L * B * H;            // [B][16]
  float* D[2] = {R + (size_t)B * 16, R + (size_t)B * 16 + (size_t)B * H};
  auto Hk = [&](int k) { return Hs + (size_t)(k - 1) * B * H; };

  // phase 0: Z = [x | u(S_p, S_c)] (R#8)
  for (int e = gtid; e < B * kZDim; e += gthreads) {
    const int b = e / kZDim, i = e % kZDim;
    float v;
    if (i < kXDim) v = p.x[(size_t)b * kXDim + i];
    else if (i == kXDim) v = static_cast<float>((log2(static_cast<double>(p.S_p[b])) - 21.0) / 8.0);
    else v = static_cast<float>((static_cast<double>(p.S_c[b]) - 8.5) / 8.0);
    Z[e] = v;
  }
  grid_sync(p.barrier, gen);

  const int nsteps = p.steps > 0 ? p.steps : 0;
  for (int step = 0; step <= nsteps; ++step) {
    const bool fwd_only = (step == nsteps);   // trailing forward only when loss is still needed
    if (fwd_only && !(nsteps == 0 && p.loss_before)) break;
    // ---------------- forward with stash
    for (int k = 1; k <= L; ++k) {
      const int Kin = k == 1 ? kZDim : H;
      const float* in = k == 1 ? Z : Hk(k - 1);
      Gemm g{B, H, Kin, in, Kin, 1, P + p.off.W[k], 1, Kin, Hk(k), H, 0, P + p.off.b[k],
             nullptr, 0, nullptr, nullptr, 0.f};
      for (int t = blockIdx.x; t < g.tiles(); t += gridDim.x) gemm_tile(g, t, As, Bs);
      grid_sync(p.barrier, gen);
    }
    {
      Gemm g{B, kNMax, H, Hk(L), H, 1, P + p.off.W_o, 1, H, R, kNMax, 3, P + p.off.b_o,
             nullptr, 0, p.v_obs, p.n, 1.0f / static_cast<float>(B)};
      for (int t = blockIdx.x; t < g.tiles(); t += gridDim.x) gemm_tile(g, t, As, Bs);
      grid_sync(p.barrier, gen);
    }
    if (step == 0 && p.loss_before && blockIdx.x == 0) {
      // mean over b of the Eq. 2 norm ||mask (V_hat - V_bar)||_2; R holds residual / B
      __shared__ float s_norm[kAdaptThreads];
      float acc = 0.f;
      for (int b = threadIdx.x; b < B; b += kAdaptThreads) {
        float ss = 0.f;
        for (int w = 0; w < kNMax; ++w) { const float r = R[b * kNMax + w] * B; ss = fmaf(r, r, ss); }
        acc += sqrtf(ss);
      }
      s_norm[threadIdx.x] = acc;
      __syncthreads();
      if (threadIdx.x == 0) {
        float tot = 0.f;
        for (int i = 0; i < kAdaptThreads; ++i) tot += s_norm[i];
        *p.loss_before = tot / static_cast<float>(B);
      }
    }
    if (fwd_only) break;
    // ---------------- backward: output layer
    {
      Gemm gw{kNMax, H, B, R, 1, kNMax, Hk(L), H, 1, Gr + p.off.W_o, H, 2, nullptr, nullptr, 0, nullptr, nullptr, 0.f,
              kSplitK, p.off.total};
      Gemm gd{B, H, kNMax, R, kNMax, 1, P + p.off.W_o, H, 1, D[L & 1], H, 1, nullptr, Hk(L), H, nullptr, nullptr, 0.f};
      const int t1 = gw.tiles(), t2 = gd.tiles();
      for (int t = blockIdx.x; t < t1 + t2; t += gridDim.x) {
        if (t < t1) gemm_tile(gw, t, As, Bs);
        else gemm_tile(gd, t - t1, As, Bs);
      }
      colsum_split(R, B, kNMax, kNMax, Gr + p.off.b_o, p.off.total);
      grid_sync(p.barrier, gen);
    }
    // ---------------- backward: hidden layers L..1
    for (int k = L; k >= 1; --k) {
      const int Kin = k == 1 ? kZDim : H;
      const float* in = k == 1 ? Z : Hk(k - 1);
      const float* Dk = D[k & 1];
      Gemm gw{H, Kin, B, Dk, 1, H, in, Kin, 1, Gr + p.off.W[k], Kin, 2, nullptr, nullptr, 0, nullptr, nullptr, 0.f,
              kSplitK, p.off.total};
      const int t1 = gw.tiles();
      int t2 = 0;
      Gemm gd{};
      if (k > 1) {
        gd = Gemm{B, H, H, Dk, H, 1, P + p.off.W[k], H, 1, D[(k - 1) & 1], H, 1, nullptr, Hk(k - 1), H,
                  nullptr, nullptr, 0.f};
        t2 = gd.tiles();
      }
      for (int t = blockIdx.x; t < t1 + t2; t += gridDim.x) {
        if (t < t1) gemm_tile(gw, t, As, Bs);
        else gemm_tile(gd, t - t1, As, Bs);
      }
      colsum_split(Dk, B, H, H, Gr + p.off.b[k], p.off.total);
      grid_sync(p.barrier, gen);
    }
    // ---------------- SGD on the head parameters (contiguous from W1 to b_o in the blob order)
    const float lr = p.lr;
    // (the weight gradients arrive as kSplitK partial sums over B; summed here in fixed order)
    for (long long i = p.off.W[1] + gtid; i < p.off.total; i += gthreads) {
      float gsum = Gr[i];
#pragma unroll
      for (int sk = 1; sk < kSplitK; ++sk) gsum += Gr[sk * p.off.total + i];
      P[i] = P[i] - lr * gsum;
    }
    grid_sync(p.barrier, gen);
  }
}

size_t adapt_ws_floats(int B, int H, int L) {
  return (size_t)B * kZDim + (size_t)L * B * H + (size_t)B * kNMax + 2 * (size_t)B * H;
}

cudaError_t launch_adapt(const AdaptParams& p, int num_sms, cudaStream_t s, int* grid_used) {
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, adapt_kernel, kAdaptThreads, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int grid = num_sms * (per_sm < 2 ? per_sm : 2);
  *grid_used = grid;
  void* args[] = {const_cast<AdaptParams*>(&p)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(adapt_kernel), dim3(grid), dim3(kAdaptThreads), args, 0, s);
}

}  // namespace ab

#ifdef AB_STATS
extern "C" int ab_debug_adapt_phases(unsigned long long* out) {
  cudaDeviceSynchronize();
  int n = 0;
  cudaMemcpyFromSymbol(&n, ab::g_adapt_nphase, sizeof(int));
  cudaMemcpyFromSymbol(out, ab::g_adapt_phase, sizeof(unsigned long long) * 64);
  int z = 0;
  cudaMemcpyToSymbol(ab::g_adapt_nphase, &z, sizeof(int));
  return n;
}
#endif
