// adapt_small.cu — K4s: online adaptation for small minibatches (B <= 16) at single-call latency
// ("adapt ... when the prediction error exceeds 10%", one job's observation at a time;
// P:404-408 Eq. 2, R#12, R#13; the same objective, head scope and optimisers as K4, adapt.cu).
//
// K4 runs every phase as tcgen05 GEMM tiles over the whole GPU with grid barriers; at B = 1 its
// phases hold one or a few tiles each and the 11 grid barriers dominate. K4s runs ONE cluster of 16
// CTAs: every barrier is a hardware cluster barrier, every cross-CTA vector exchange a distributed-
// shared-memory read, and every weight slice a phase needs arrives by TMA bulk copy into a
// double-buffered shared-memory ring, issued one phase ahead (the next slice streams in while the
// current phase computes, and the update reads the pre-update values from that copy):
//   forward layer k   CTA c owns rows [cR, cR + R) of W_k (R = H / 16): z = b + W_k h_{k-1} over
//                     the full h_{k-1} gathered from the CTAs' slices; lanes split K, butterfly sums
//   output            every CTA forms V = W_o h_L + b_o for all samples (16 x H, redundant), the
//                     masked residual r and the Eq. 2 norm; delta_L on its own rows
//   backward layer k  CTA c owns COLUMNS [cR, cR + R) of W_k (= its rows of layer k-1):
//                     delta_{k-1} = relu'(h_{k-1}) (W_k^T delta_k) over the gathered delta_k, then
//                     the update of that column slice and of its bf16 shadows (packed layout), and
//                     b_k on its rows of layer k
//   layer 1           W1 / b1 rows of the CTA (dW1 = delta_1 [x | u]^T), no input gradient
// W_o's update waits for the barrier after delta_L (every CTA read all of W_o for V). All sums run
// in a fixed order (lane-strided partials + xor butterflies; warps in index order; samples in index
// order): deterministic, replicas bit-identical; fp32 SIMT arithmetic throughout.
#include "internal.h"
#include "ptx.cuh"

namespace ab {

constexpr int kSmallThreads = 512;
constexpr int kSmallWarps = kSmallThreads / 32;
constexpr int kSmallCL = 16;   // CTAs per cluster (non-portable size; K4 runs where unavailable)

#ifdef AB_STATS
__device__ long long g_k4s_marks[64];   // CTA 0, thread 0: clock64 at each phase boundary (tools/k4s_phases.py)
#define K4S_MARK(i) do { if (threadIdx.x == 0 && cluster_ctarank() == 0 && (i) < 64) g_k4s_marks[i] = clock64(); } while (0)
#else
#define K4S_MARK(i) do { } while (0)
#endif

__device__ __forceinline__ float ld_dsmem_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// shared memory (floats), per-sample arrays sized for NB samples (rows B..NB-1 stay zero):
// sZin [NB][84] | sIn [NB][H] | sH [L][NB][R] | sD [2][NB][R] | sV [NB][16] | sRed [16][NB][32] |
// sNorm [16] | sW [2][H * max(R, 16)] | 2 mbarriers
size_t adapt_small_smem_floats(int B, int H, int L) {
  const int R = H / kSmallCL, slice = H * (R > kNMax ? R : kNMax);
  return (size_t)B * kZDim + (size_t)B * H + (size_t)L * B * R + 2 * (size_t)B * R + (size_t)B * kNMax +
         (size_t)kSmallWarps * B * 32 + 16 + 2 * (size_t)slice + 8 + 32;
}

// one optimiser update of parameter i whose current value is w (SGD, or Adam with bias correction)
__device__ __forceinline__ float opt_step(const AdaptParams& p, long long i, float w, float g, float step_size,
                                          float sqrt_bc2) {
  if (p.opt == AB_OPT_ADAM) {
    const float m = fmaf(p.beta1, p.m[i], (1.0f - p.beta1) * g);
    const float v = fmaf(p.beta2, p.v[i], (1.0f - p.beta2) * (g * g));
    p.m[i] = m;
    p.v[i] = v;
    w = w - step_size * (m / (sqrtf(v) / sqrt_bc2 + p.eps));
  } else {
    w = w - p.lr * g;
  }
  p.params[i] = w;
  return w;
}

// H (head width) and NB (samples, rounded up to a power of two; rows b >= B are masked) are
// compile-time so every per-sample loop and every index split is resolved by the compiler.
template <int H, int NB>
__global__ void __launch_bounds__(kSmallThreads, 1) adapt_small_kernel(const __grid_constant__ AdaptParams p) {
  extern __shared__ __align__(16) float sm[];
  const int B = p.B, L = p.L;
  const int rank = static_cast<int>(cluster_ctarank());
  constexpr int R = H / kSmallCL;
  const int row0 = rank * R;
  constexpr int slice = H * (R > kNMax ? R : kNMax);
  float* sZin = sm;                                   // [NB][84]
  float* sIn = sZin + NB * kZDim;                     // [NB][H]
  float* sH = sIn + NB * H;                           // [L][NB][R]
  float* sD = sH + L * NB * R;                        // [2][NB][R]
  float* sV = sD + 2 * NB * R;                        // [NB][16]
  float* sRed = sV + NB * kNMax;                      // [16][NB][32]
  float* sNorm = sRed + kSmallWarps * NB * 32;        // [16]
  // (tensor-TMA destinations need 128-byte alignment)
  float* sW = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(sNorm + 16) + 127) & ~uintptr_t(127));   // [2][slice]
  uint64_t* wbar = reinterpret_cast<uint64_t*>(sW + 2 * slice);                                             // [2]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* P = p.params;
  const float invB = 1.0f / static_cast<float>(B);
  auto hs = [&](int k) { return sH + (size_t)(k - 1) * NB * R; };   // own slice of h_k
  int mark = 0;
  K4S_MARK(mark++);

  // ---- weight slices, in the order the phases use them (per step):
  //   n = 0..L-1       rows [row0, row0 + R) of W_{n+1}      ([R][Kin], contiguous)
  //   n = L            W_o                                  ([16][H], contiguous)
  //   n = L+1..2L-1    columns [row0, row0 + R) of W_{2L+1-n} ([H][R], one 4R-byte copy per row)
  //   n = 2L           rows of W1 again (for its update)
  const int nslices = 2 * L + 1;
  auto issue = [&](int n) {   // warp 0 issues slice n (of the current step) into buffer n & 1
    if (warp != 0 || n >= nslices) return;
    float* dst = sW + (n & 1) * slice;
    uint64_t* bar = &wbar[n & 1];
    if (n < L || n == 2 * L) {
      const int k = n < L ? n + 1 : 1, Kin = k == 1 ? kZDim : H;
      const uint32_t bytes = static_cast<uint32_t>(R * Kin * 4);
      if (lane == 0) {
        mbar_arrive_expect_tx(bar, bytes);
        bulk_g2s(dst, P + p.off.W[k] + (size_t)row0 * Kin, bytes, bar, 0ull);
      }
    } else if (n == L) {
      const uint32_t bytes = static_cast<uint32_t>(kNMax * H * 4);
      if (lane == 0) {
        mbar_arrive_expect_tx(bar, bytes);
        bulk_g2s(dst, P + p.off.W_o, bytes, bar, 0ull);
      }
    } else {   // the column slice: 2-D tensor boxes of [<= 256 rows][R cols]
      const int k = 2 * L + 1 - n;
      constexpr int BOXR = H < 256 ? H : 256;
      if (lane == 0) {
        mbar_arrive_expect_tx(bar, static_cast<uint32_t>(H * R * 4));
#pragma unroll
        for (int y = 0; y < H; y += BOXR) tma_load_2d(dst + y * R, &p.wcol[k], row0, y, bar);
      }
    }
  };
  uint32_t wph[2] = {0u, 0u};
  auto wait_slice = [&](int n) {   // every thread: slice n has landed in buffer n & 1
    mbar_wait(&wbar[n & 1], wph[n & 1]);
    wph[n & 1] ^= 1u;
    return sW + (n & 1) * slice;
  };

  if (tid == 0) {
    mbar_init(&wbar[0], 1);
    mbar_init(&wbar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  issue(0);
  issue(1);

  // [x | u] of every sample (R#8); the padding rows of sZin / sIn are zero
  for (int e = tid; e < NB * H; e += kSmallThreads) sIn[e] = 0.f;
  for (int e = tid; e < NB * kZDim; e += kSmallThreads) {
    const int b = e / kZDim, i = e % kZDim;
    float v;
    if (b >= B) v = 0.f;
    else if (i < kXDim) v = p.x[(size_t)b * kXDim + i];
    else if (i == kXDim) v = static_cast<float>((log2(static_cast<double>(p.S_p[b])) - 21.0) / 8.0);
    else v = static_cast<float>((static_cast<double>(p.S_c[b]) - 8.5) / 8.0);
    sZin[e] = v;
  }
  __syncthreads();

  // gather a [B][H] vector whose rows [cR, cR + R) live in CTA c's slice `src` ([B][R]) into sIn
  auto gather = [&](float* src) {
    const uint32_t base = smem_u32(src);
    for (int e = tid; e < B * H; e += kSmallThreads) {
      const int b = e / H, i = e % H, c = i / R, r = i - c * R;
      sIn[e] = ld_dsmem_f32(mapa_shared(base + 4u * static_cast<uint32_t>(b * R + r), static_cast<uint32_t>(c)));
    }
    __syncthreads();
  };

  const int nsteps = p.steps > 0 ? p.steps : 0;
  for (int step = 0; step <= nsteps; ++step) {
    const bool fwd_only = (step == nsteps);
    if (fwd_only && !(nsteps == 0 && p.loss_before)) break;
    const double t_adam = static_cast<double>(p.t0 + step + 1);
    const float step_size = p.opt == AB_OPT_ADAM ? static_cast<float>(p.lr / (1.0 - pow((double)p.beta1, t_adam))) : 0.f;
    const float sqrt_bc2 = p.opt == AB_OPT_ADAM ? static_cast<float>(sqrt(1.0 - pow((double)p.beta2, t_adam))) : 1.f;
    if (step > 0) { issue(0); issue(1); }   // (the previous step's slices are all consumed)

    // ---------------- forward: own rows of every layer (slices 0..L-1)
    for (int k = 1; k <= L; ++k) {
      const int Kin = k == 1 ? kZDim : H;
      const float* in = k == 1 ? sZin : sIn;          // sIn holds the gathered h_{k-1}
      const float* Ws = wait_slice(k - 1);            // [R][Kin]
      const float* bk = P + p.off.b[k];
      for (int r = warp; r < R; r += kSmallWarps) {
        float acc[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) acc[b] = 0.f;
        for (int kk = lane; kk < Kin; kk += 32) {
          const float w = Ws[r * Kin + kk];
#pragma unroll
          for (int b = 0; b < NB; ++b) acc[b] = fmaf(w, in[b * Kin + kk], acc[b]);
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          float v = acc[b];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane == 0) hs(k)[b * R + r] = b < B ? relu(v + bk[row0 + r]) : 0.f;
        }
      }
      K4S_MARK(mark++);
      cluster_sync();      // own slice of h_k published; slice k-1 consumed by every thread
      issue(k + 1);        // prefetch the slice after next into the buffer slice k-1 used
      gather(hs(k));       // full h_k -> sIn (input of layer k + 1, or of the output layer)
      K4S_MARK(mark++);
    }
    // ---------------- output layer (every CTA, all samples): V = W_o h_L + b_o, residual, norm
    const float* Wos = wait_slice(L);                  // [16][H]
    {
      const float* bo = P + p.off.b_o;
      float acc[NB];   // warp w -> output w (16 outputs, 16 warps); lanes split H
#pragma unroll
      for (int b = 0; b < NB; ++b) acc[b] = 0.f;
      for (int kk = lane; kk < H; kk += 32) {
        const float w = Wos[warp * H + kk];
#pragma unroll
        for (int b = 0; b < NB; ++b) acc[b] = fmaf(w, sIn[b * H + kk], acc[b]);
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        float v = acc[b];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0)
          sV[b * kNMax + warp] = (b < B && warp < p.n[b]) ? (v + bo[warp] - p.v_obs[(size_t)b * kNMax + warp]) : 0.f;
      }
      __syncthreads();
      if (tid < B) {   // Eq. 2 norm of sample tid (fixed order over workers)
        float ss = 0.f;
        for (int w = 0; w < kNMax; ++w) ss = fmaf(sV[tid * kNMax + w], sV[tid * kNMax + w], ss);
        sNorm[tid] = sqrtf(ss);
      }
      __syncthreads();
      if (rank == 0 && tid == 0 && ((step == 0 && p.loss_before) || (p.losses && !fwd_only))) {
        float tot = 0.f;
        for (int b = 0; b < B; ++b) tot += sNorm[b];
        if (step == 0 && p.loss_before) *p.loss_before = tot * invB;
        if (p.losses && !fwd_only) p.losses[step] = tot * invB;
      }
    }
    if (fwd_only) break;
    // delta_L on own rows of layer L: relu'(z_L) (W_o^T r / B)
    int dpar = 0;
    for (int e = tid; e < NB * R; e += kSmallThreads) {
      const int b = e / R, r = e - b * R;
      float acc = 0.f;
#pragma unroll
      for (int w = 0; w < kNMax; ++w) acc = fmaf(Wos[w * H + row0 + r], sV[b * kNMax + w], acc);
      sD[e] = hs(L)[e] > 0.f ? acc * invB : 0.f;
    }
    K4S_MARK(mark++);
    cluster_sync();   // delta_L published; every CTA is done reading W_o (from its own copy)
    // W_o columns of this CTA's rows of layer L (old values from the copy), b_o by CTA 0
    for (int e = tid; e < kNMax * R; e += kSmallThreads) {
      const int w = e / R, r = e - w * R;
      float g = 0.f;
      for (int b = 0; b < NB; ++b) g = fmaf(sV[b * kNMax + w], hs(L)[b * R + r], g);
      opt_step(p, p.off.W_o + (long long)w * H + row0 + r, Wos[w * H + row0 + r], g * invB, step_size, sqrt_bc2);
    }
    if (rank == 0 && tid < kNMax) {
      float g = 0.f;
      for (int b = 0; b < B; ++b) g += sV[b * kNMax + tid];
      opt_step(p, p.off.b_o + tid, P[p.off.b_o + tid], g * invB, step_size, sqrt_bc2);
    }
    __syncthreads();   // the W_o copy is consumed
    issue(L + 2);
    // ---------------- backward, layers L..2: own columns of W_k (= own rows of layer k-1)
    const int nch = packed_weight_nch(H, p.planes);
    const size_t rep = packed_weight_elems(H, L, p.planes);
    for (int k = L; k >= 2; --k) {
      const int n = 2 * L + 1 - k;                   // its slice
      float* dk = sD + dpar * NB * R;                // own slice of delta_k
      float* dnext = sD + (dpar ^ 1) * NB * R;       // own slice of delta_{k-1}
      gather(dk);                                    // full delta_k -> sIn
      K4S_MARK(mark++);
      const float* Wc = wait_slice(n);               // [H][R]
      // delta_{k-1}[b][j] = relu'(h_{k-1}[b][j]) sum_i W_k[i][j] delta_k[b][i]: lanes = columns,
      // warps = row chunks, then the 16 warp partials in warp order
      for (int j0 = 0; j0 < R; j0 += 32) {
        const int jl = j0 + lane;
        float acc[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) acc[b] = 0.f;
        if (jl < R) {
          for (int i = warp; i < H; i += kSmallWarps) {
            const float w = Wc[i * R + jl];
#pragma unroll
            for (int b = 0; b < NB; ++b) acc[b] = fmaf(w, sIn[b * H + i], acc[b]);
          }
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) sRed[(warp * NB + b) * 32 + lane] = acc[b];
        __syncthreads();
        for (int e = tid; e < NB * 32; e += kSmallThreads) {
          const int b = e >> 5, l = e & 31, j = j0 + l;
          if (j < R) {
            float s = 0.f;
#pragma unroll
            for (int w = 0; w < kSmallWarps; ++w) s += sRed[(w * NB + b) * 32 + l];
            dnext[b * R + j] = hs(k - 1)[b * R + j] > 0.f ? s : 0.f;
          }
        }
        __syncthreads();
      }
      // update of the column slice from its pre-update copy: dW_k = delta_k h_{k-1}^T, and its bf16
      // shadow(s) for K2 written in place (the packed layout, every replica)
      for (int e = tid; e < H * R; e += kSmallThreads) {
        const int i = e / R, r = e - i * R;
        float g = 0.f;
#pragma unroll
        for (int b = 0; b < NB; ++b) g = fmaf(sIn[b * H + i], hs(k - 1)[b * R + r], g);
        const float w = opt_step(p, p.off.W[k] + (long long)i * H + row0 + r, Wc[e], g, step_size, sqrt_bc2);
        const __nv_bfloat16 hi = __float2bfloat16_rn(w);
        const size_t ph = packed_weight_index(H, p.planes, nch, k - 2, i, row0 + r, 0);
#pragma unroll 1
        for (int rp = 0; rp < kWeightReplicas; ++rp) p.wpack[ph + rp * rep] = hi;
        if (p.planes == 2) {
          const __nv_bfloat16 lo = __float2bfloat16_rn(w - __bfloat162float(hi));
          const size_t pl = packed_weight_index(H, p.planes, nch, k - 2, i, row0 + r, 1);
#pragma unroll 1
          for (int rp = 0; rp < kWeightReplicas; ++rp) p.wpack[pl + rp * rep] = lo;
        }
      }
      for (int r = tid; r < R; r += kSmallThreads) {   // b_k on own rows of layer k
        float g = 0.f;
        for (int b = 0; b < B; ++b) g += dk[b * R + r];
        opt_step(p, p.off.b[k] + row0 + r, P[p.off.b[k] + row0 + r], g, step_size, sqrt_bc2);
      }
      dpar ^= 1;
      K4S_MARK(mark++);
      cluster_sync();        // delta_{k-1} published; the gathers of delta_k and slice n are done
      issue(n + 2);
    }
    // ---------------- layer 1: own rows of W1 (old values from slice 2L), b1
    {
      const float* d1 = sD + dpar * NB * R;
      const float* W1s = wait_slice(2 * L);            // [R][84]
      for (int e = tid; e < R * kZDim; e += kSmallThreads) {
        const int r = e / kZDim, kk = e - r * kZDim;
        float g = 0.f;
#pragma unroll
        for (int b = 0; b < NB; ++b) g = fmaf(d1[b * R + r], sZin[b * kZDim + kk], g);
        opt_step(p, p.off.W[1] + (long long)(row0 + r) * kZDim + kk, W1s[e], g, step_size, sqrt_bc2);
      }
      for (int r = tid; r < R; r += kSmallThreads) {
        float g = 0.f;
        for (int b = 0; b < B; ++b) g += d1[b * R + r];
        opt_step(p, p.off.b[1] + row0 + r, P[p.off.b[1] + row0 + r], g, step_size, sqrt_bc2);
      }
    }
    // the next step's slices are read by TMA (async proxy) after these generic-proxy updates
    fence_proxy_async_global();
    K4S_MARK(mark++);
    cluster_sync();
  }
  cluster_sync();     // no CTA leaves while another may still read its shared memory
  K4S_MARK(mark++);
}

template <int H, int NB>
cudaError_t launch_small_hb(const AdaptParams& p, cudaStream_t s) {
  auto* kern = adapt_small_kernel<H, NB>;
  static unsigned long long attr_done = 0, usable = 0;   // per device
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const size_t bytes = adapt_small_smem_floats(NB, H, kMaxHidden) * sizeof(float) + 64;
  if (!(attr_done >> (dev & 63) & 1ull)) {
    bool ok = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)) ==
                  cudaSuccess &&
              cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
    if (ok) {
      cudaLaunchConfig_t q{};
      q.gridDim = dim3(kSmallCL);
      q.blockDim = dim3(kSmallThreads);
      q.dynamicSmemBytes = bytes;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = kSmallCL; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
      q.attrs = a;
      q.numAttrs = 1;
      int n = 0;
      ok = cudaOccupancyMaxActiveClusters(&n, kern, &q) == cudaSuccess && n >= 1;
    }
    cudaGetLastError();
    if (ok) usable |= 1ull << (dev & 63);
    attr_done |= 1ull << (dev & 63);
  }
  if (!(usable >> (dev & 63) & 1ull)) return cudaErrorNotSupported;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kSmallCL);
  cfg.blockDim = dim3(kSmallThreads);
  cfg.dynamicSmemBytes = adapt_small_smem_floats(NB, H, p.L) * sizeof(float) + 64;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kSmallCL; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

template <int H>
cudaError_t launch_small_h(const AdaptParams& p, cudaStream_t s) {
  if (p.B <= 1) return launch_small_hb<H, 1>(p, s);
  if (p.B <= 2) return launch_small_hb<H, 2>(p, s);
  if (p.B <= 4) return launch_small_hb<H, 4>(p, s);
  if (p.B <= 8) return launch_small_hb<H, 8>(p, s);
  return launch_small_hb<H, 16>(p, s);
}

// One cluster of 16 CTAs; cudaErrorNotSupported when the shape is outside K4s's range or the
// device cannot schedule a 16-CTA cluster (the caller then runs K4).
cudaError_t launch_adapt_small(const AdaptParams& p, cudaStream_t s) {
  if (p.B < 1 || p.B > kAdaptSmallMaxB || p.dz_out || p.idx) return cudaErrorNotSupported;
  switch (p.H) {
    case 64: return launch_small_h<64>(p, s);
    case 128: return launch_small_h<128>(p, s);
    case 256: return launch_small_h<256>(p, s);
    case 512: return launch_small_h<512>(p, s);
  }
  return cudaErrorNotSupported;
}

AB_STATUS_SETTER(set_status_adapt_small)   // device status word pointer of this unit (ptx.cuh)
}  // namespace ab

#ifdef AB_STATS
extern "C" int ab_debug_k4s_marks(long long* out) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, ab::g_k4s_marks, sizeof(long long) * 64) == cudaSuccess;
}
#endif
