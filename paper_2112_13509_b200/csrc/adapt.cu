// adapt.cu — K4: fused online adaptation (forward with stash, backward, SGD) in ONE cooperative
// persistent kernel ("offline training, online adapting ... transfer learning";
// P:438 triggered when prediction error > 10%; R#12 objective, R#13 head-only plain SGD).
//
// Per step, phases separated by a grid-wide barrier:
//   F_k   H_k = ReLU(H_{k-1} W_k^T + b_k), k = 1..L (H_0 = Z = [x | u])      3xTF32 tensor-core tiles
//   OUT   R = mask_b (H_L W_o^T + b_o - V_bar) / B        (dV of the objective; one warp per row)
//   BO    dW_o = R^T H_L, db_o = colsum R, D_L = (R W_o) * [H_L > 0]
//   Bk    dW_k = D_k^T H_{k-1}, db_k = colsum D_k, D_{k-1} = (D_k W_k) * [H_{k-1} > 0]  (pre-update W_k)
//         + SGD of the layer above (its gradient is complete and no later phase reads it)
//   SGD   W1, b1 (after B1)   (SGD or Adam, see update_range)
// Every output element is produced by exactly one thread with a fixed summation order, so the
// update is deterministic and replicas on different GPUs stay bit-identical without traffic.
// The work is ~3x a B-row forward (5 GFLOP at B=1024, 4x512): latency-bound, << 1% of a C5 step.
// Every GEMM runs on the legacy mma.sync tensor path with 3xTF32 split operands (big*big +
// big*small + small*big, ~fp32 accuracy), which keeps the gradient well inside the parity
// tolerance (K4) at a fraction of the SIMT instruction count.
#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

namespace ab {

constexpr int kAdaptThreads = 256;
constexpr int kTM = 64, kTN = 64, kTK = 32;
constexpr int kSplitK = kAdaptSplitK;   // K = B splits of the weight-gradient GEMMs (partials in grads[kSplitK][total])

struct Gemm {
  int M, N, K;
  const float* A; long long lam, lak;    // A(m, k) = A[m*lam + k*lak]; lak == 1 or lam == 1
  const float* Bm; long long lbk, lbn;   // B(k, n) = Bm[k*lbk + n*lbn]; lbk == 1 or lbn == 1
  float* C; long long ldc;               // C[m*ldc + n]
  int mode;                              // 0: ReLU(acc + bias[n]); 1: acc * [mask(m,n) > 0]; 2: acc
  const float* bias;
  const float* mask; long long ldmask;
  int ksplit;                            // split-K count (mode 2 only): partial s -> C + s*cpart
  long long cpart;
  __device__ int tiles() const { return ((M + kTM - 1) / kTM) * ((N + kTN - 1) / kTN) * (ksplit > 1 ? ksplit : 1); }
};

constexpr int kStages = 4;   // cp.async pipeline depth of the raw operand slices (prefetch distance kStages - 1)
// Raw operand slices land in shared memory in the orientation of their global layout so every
// 16-byte cp.async copies a contiguous vector: K-contiguous [64][kTK + 4] or MN-contiguous
// [kTK][64 + 8]. A conversion pass then splits every element once per CTA into tf32 big / small
// planes stored K-contiguous [64][kTK + 4] (transposing MN-contiguous slices), from which the
// warps read whole m16n8k8 fragments with ldmatrix (a tf32 element is a pair of b16 lanes).
// Row stride kTK + 4 = 36 floats puts the 8 rows of an ldmatrix in 8 distinct 16-byte bank groups.
constexpr int kSK = kTK + 4, kSM = kTM + 8;
constexpr int kSliceFloats = (kTM * kSK > kTK * kSM) ? kTM * kSK : kTK * kSM;
constexpr int kPlaneFloats = kTM * kSK;                  // one split plane [64][36]
constexpr size_t kAdaptSmemBytes = sizeof(float) * (kStages * 2 * kSliceFloats + 4 * kPlaneFloats);

__device__ __forceinline__ void cp_async16(float* smem_dst, const float* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem_dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// x = big + small with both parts tf32 (10-bit mantissa each): the 3xTF32 product
// big*big + big*small + small*big carries ~fp32 accuracy (the dropped small*small is ~2^-22 relative).
__device__ __forceinline__ void split_tf32(float x, float& big, float& small) {
  uint32_t b, sm;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(b) : "f"(x));
  const float r = x - __uint_as_float(b);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(sm) : "f"(r));
  big = __uint_as_float(b);
  small = __uint_as_float(sm);
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

// Stage one 64 x kTK slice of an operand: X(mn, k) = base[mn*lmn + k*lk] for mn in [mn0, mn0+64),
// k in [k0, k0+kTK), zero-filled outside [0, MN) x [k0, kend). 16-byte vectors, kTK/16 per thread.
__device__ __forceinline__ void stage_slice(float* dst, const float* base, long long lmn, long long lk, int MN,
                                            int mn0, int k0, int kend) {
#pragma unroll
  for (int r = 0; r < kTK / 16; ++r) {
    const int e = threadIdx.x + r * kAdaptThreads;
    if (lk == 1) {   // K-contiguous: vector (mn, 4 k)
      const int mn = e / (kTK / 4), kq = (e % (kTK / 4)) * 4;
      const bool v = mn0 + mn < MN && k0 + kq < kend;
      cp_async16(dst + mn * kSK + kq, v ? base + (long long)(mn0 + mn) * lmn + (k0 + kq) : base, v);
    } else {         // MN-contiguous: vector (k, 4 mn)
      const int k = e >> 4, mq = (e & 15) * 4;
      const bool v = k0 + k < kend && mn0 + mq < MN;
      cp_async16(dst + k * kSM + mq, v ? base + (long long)(k0 + k) * lk + (mn0 + mq) : base, v);
    }
  }
}

// Split one raw slice into K-contiguous big / small planes (8 elements per thread). K-contiguous
// raw: thread -> (mn, 8 consecutive k), LDS.128 / STS.128. MN-contiguous raw: warp w -> k in
// [4w, 4w+4), lane -> (k = 4w + lane/8, mn = lane%8 + 8j): conflict-free on both the raw read
// (stride 72) and the transposed plane write (stride 36).
__device__ __forceinline__ void split_slice(const float* raw, bool kcontig, float* big, float* small) {
  const int tid = threadIdx.x;
  if (kcontig) {
    const int mn = tid >> 2, k0 = (tid & 3) * 8;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float4 v = *reinterpret_cast<const float4*>(raw + mn * kSK + k0 + 4 * h);
      float4 b, sm;
      split_tf32(v.x, b.x, sm.x); split_tf32(v.y, b.y, sm.y);
      split_tf32(v.z, b.z, sm.z); split_tf32(v.w, b.w, sm.w);
      *reinterpret_cast<float4*>(big + mn * kSK + k0 + 4 * h) = b;
      *reinterpret_cast<float4*>(small + mn * kSK + k0 + 4 * h) = sm;
    }
  } else {
    const int lane = tid & 31, w = tid >> 5;
    const int k = 4 * w + (lane >> 3);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int mn = (lane & 7) + 8 * j;
      float b, sm;
      split_tf32(raw[k * kSM + mn], b, sm);
      big[mn * kSK + k] = b;
      small[mn * kSK + k] = sm;
    }
  }
}

// One 64 x 64 output tile (or one K-slice range of it for split-K) on the tensor cores, 3xTF32.
// 8 warps as 2 (M) x 4 (N), each a 32 x 16 warp tile = 2 x 2 m16n8 fragments; kTK-wide K slices
// of both operands stream through a kStages-deep cp.async ring and are split once per CTA. The
// accumulation order is fixed, so the result is deterministic (replicas stay bit-identical).
__device__ void gemm_tile(const Gemm& g, int work, float* ring) {
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
  const bool a_kc = g.lak == 1, b_kc = g.lbk == 1;
  const int nk = kend > kbeg ? (kend - kbeg + kTK - 1) / kTK : 0;
  auto As = [&](int st) { return ring + st * 2 * kSliceFloats; };
  auto Bs = [&](int st) { return ring + st * 2 * kSliceFloats + kSliceFloats; };
  float* planes = ring + kStages * 2 * kSliceFloats;   // A big, A small, B big, B small
  auto issue = [&](int it) {
    if (it < nk) {
      const int k0 = kbeg + it * kTK, st = it % kStages;
      stage_slice(As(st), g.A, g.lam, g.lak, g.M, m0, k0, kend);
      stage_slice(Bs(st), g.Bm, g.lbn, g.lbk, g.N, n0, k0, kend);
    }
    cp_async_commit();   // (empty groups keep the wait arithmetic uniform)
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp >> 2) * 32, wn = (warp & 3) * 16;
  const int gq = lane >> 2, tq = lane & 3;
  // ldmatrix lane addresses (bytes, relative to a plane): A matrices (rows 0-7 | 8-15) x (k 0-3 | 4-7),
  // B matrices (n 0-7, k 0-3 | 4-7) then (n 8-15, ...)
  const uint32_t pl = smem_u32(planes);
  const uint32_t a_off = static_cast<uint32_t>(((wm + (lane & 7) + 8 * ((lane >> 3) & 1)) * kSK + 4 * (lane >> 4)) * 4);
  const uint32_t b_off = static_cast<uint32_t>(((wn + (lane & 7) + 8 * (lane >> 4)) * kSK + 4 * ((lane >> 3) & 1)) * 4);
  constexpr uint32_t kPlaneBytes = kPlaneFloats * 4;
  float acc[2][2][4] = {};
  __syncthreads();       // the ring and planes may still be read by the previous tile
#pragma unroll
  for (int i = 0; i < kStages - 1; ++i) issue(i);
  for (int it = 0; it < nk; ++it) {
    cp_async_wait<kStages - 2>();
    __syncthreads();     // slice `it` landed for everyone; every warp is past the previous MMAs
    issue(it + kStages - 1);
    split_slice(As(it % kStages), a_kc, planes, planes + kPlaneFloats);
    split_slice(Bs(it % kStages), b_kc, planes + 2 * kPlaneFloats, planes + 3 * kPlaneFloats);
    __syncthreads();
    // per-slice partial sums start from zero and are added to acc with IEEE fp32 adds: the
    // tensor core's internal accumulation then only spans 12 products-of-8, not the whole K
    float part[2][2][4] = {};
#pragma unroll
    for (int kk = 0; kk < kTK; kk += 8) {
      uint32_t ab[2][4], as[2][4], bb[4], bs[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const uint32_t o = a_off + static_cast<uint32_t>((16 * i * kSK + kk) * 4);
        ldsm_x4(ab[i], pl + o);
        ldsm_x4(as[i], pl + kPlaneBytes + o);
      }
      const uint32_t ob = b_off + static_cast<uint32_t>(kk * 4);
      ldsm_x4(bb, pl + 2 * kPlaneBytes + ob);
      ldsm_x4(bs, pl + 3 * kPlaneBytes + ob);
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          mma_tf32(part[i][j], as[i], bb[2 * j], bb[2 * j + 1]);
          mma_tf32(part[i][j], ab[i], bs[2 * j], bs[2 * j + 1]);
          mma_tf32(part[i][j], ab[i], bb[2 * j], bb[2 * j + 1]);
        }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[i][j][r] += part[i][j][r];
  }
  cp_async_wait<0>();
  float* C = g.C + (g.ksplit > 1 ? split * g.cpart : 0);
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int m = m0 + wm + i * 16 + gq + (r >> 1) * 8;
        const int n = n0 + wn + j * 8 + 2 * tq + (r & 1);
        if (m >= g.M || n >= g.N) continue;
        float v = acc[i][j][r];
        if (g.mode == 0) v = relu(v + g.bias[n]);
        else if (g.mode == 1) v = g.mask[m * g.ldmask + n] > 0.f ? v : 0.f;
        C[m * g.ldc + n] = v;
      }
}

#ifdef AB_STATS
__device__ unsigned long long g_adapt_phase[64];   // block 0: clock at entry of each grid barrier
__device__ int g_adapt_nphase;
__device__ long long g_adapt_blk[1024][3];   // per block: smid, clock at F2 tile start, at F2 tile end
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
// order by the SGD sweep): out[s * stride + n] = sum_{b in segment s} X[b][n]. One CTA per
// (32-column group, segment), handed out from the highest block index down (those CTAs hold the
// fewest GEMM tiles); warp w sums rows w, w+8, ... of the segment (coalesced, 4 loads in flight)
// and warp 0 adds the 8 warp partials in fixed order.
__device__ void colsum_split(const float* X, int B, int N, long long ld, float* out, long long stride) {
  __shared__ float red[kAdaptThreads / 32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kAdaptThreads / 32;
  const int groups = (N + 31) / 32, seg = (B + kSplitK - 1) / kSplitK;
  for (int item = gridDim.x - 1 - blockIdx.x; item < groups * kSplitK; item += gridDim.x) {
    const int sgi = item / groups, n = (item % groups) * 32 + lane;
    const int b0 = sgi * seg, b1 = min(B, b0 + seg);
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    if (n < N) {
      int b = b0 + warp;
      for (; b + 3 * nw < b1; b += 4 * nw) {
        a0 += X[(long long)b * ld + n];
        a1 += X[(long long)(b + nw) * ld + n];
        a2 += X[(long long)(b + 2 * nw) * ld + n];
        a3 += X[(long long)(b + 3 * nw) * ld + n];
      }
      for (; b < b1; b += nw) a0 += X[(long long)b * ld + n];
    }
    red[warp][lane] = (a0 + a1) + (a2 + a3);
    __syncthreads();
    if (warp == 0 && n < N) {
      float t = red[0][lane];
      for (int w = 1; w < nw; ++w) t += red[w][lane];
      out[sgi * stride + n] = t;
    }
    __syncthreads();
  }
}

// Output layer residual, one warp per sample row (the N = 16 output is too narrow for a GEMM tile):
// R[b][w] = [w < n_b] (W_o h_L,b + b_o - V_bar_b)[w] * scale, scale = 1/B (dV of the objective, R#12).
// W_o is staged in shared memory once per CTA; lane l accumulates k = l, l+32, ... in fp32 FMA and
// the 16 sums are reduced with a fixed xor butterfly (deterministic).
__device__ void out_rows(const float* Hl, const float* Wo, const float* bo, const float* vbar, const int32_t* nvalid,
                         float scale, int B, int H, float* R, float* sW) {
  for (int e = threadIdx.x; e < kNMax * H; e += kAdaptThreads) sW[e] = Wo[e];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * kAdaptThreads + threadIdx.x) >> 5, nwarps = (gridDim.x * kAdaptThreads) >> 5;
  for (int b = gwarp; b < B; b += nwarps) {
    float acc[kNMax];
#pragma unroll
    for (int w = 0; w < kNMax; ++w) acc[w] = 0.f;
    for (int k = lane; k < H; k += 32) {
      const float h = Hl[(long long)b * H + k];
#pragma unroll
      for (int w = 0; w < kNMax; ++w) acc[w] = fmaf(h, sW[w * H + k], acc[w]);
    }
    float mine = 0.f;
#pragma unroll
    for (int w = 0; w < kNMax; ++w) {
      float v = acc[w];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == w) mine = v;
    }
    if (lane < kNMax)
      R[b * kNMax + lane] = lane < nvalid[b] ? (mine + bo[lane] - vbar[b * kNMax + lane]) * scale : 0.f;
  }
  __syncthreads();   // sW aliases the GEMM ring
}

// One optimiser update over parameters [begin, end); g = the kSplitK gradient partials summed in
// fixed order. SGD: theta -= lr g. Adam (R#18, torch semantics): m = b1 m + (1-b1) g,
// v = b2 v + (1-b2) g^2, theta -= (lr / (1 - b1^t)) m / (sqrt(v) / sqrt(1 - b2^t) + eps).
__device__ void update_range(const AdaptParams& p, long long begin, long long end, int step) {
  float* P = p.params;
  const float* Gr = p.grads;
  const long long total = p.off.total;
  const long long gtid = (long long)blockIdx.x * kAdaptThreads + threadIdx.x, gthreads = (long long)gridDim.x * kAdaptThreads;
  if (p.opt == AB_OPT_ADAM) {
    const double t = static_cast<double>(p.t0 + step + 1);
    const float step_size = static_cast<float>(p.lr / (1.0 - pow(static_cast<double>(p.beta1), t)));
    const float sqrt_bc2 = static_cast<float>(sqrt(1.0 - pow(static_cast<double>(p.beta2), t)));
    const float b1 = p.beta1, b2 = p.beta2, c1 = 1.0f - p.beta1, c2 = 1.0f - p.beta2;
    for (long long i = begin + gtid; i < end; i += gthreads) {
      float g = Gr[i];
#pragma unroll
      for (int sk = 1; sk < kSplitK; ++sk) g += Gr[sk * total + i];
      const float m = fmaf(b1, p.m[i], c1 * g);
      const float v = fmaf(b2, p.v[i], c2 * (g * g));
      p.m[i] = m;
      p.v[i] = v;
      P[i] = P[i] - step_size * (m / (sqrtf(v) / sqrt_bc2 + p.eps));
    }
  } else {
    for (long long i = begin + gtid; i < end; i += gthreads) {
      float g = Gr[i];
#pragma unroll
      for (int sk = 1; sk < kSplitK; ++sk) g += Gr[sk * total + i];
      P[i] = P[i] - p.lr * g;
    }
  }
}

__global__ void __launch_bounds__(kAdaptThreads, 2) adapt_kernel(const __grid_constant__ AdaptParams p) {
  extern __shared__ __align__(16) float ring[];   // kStages x {A, B} slices
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
      Gemm g{B, H, Kin, in, Kin, 1, P + p.off.W[k], 1, Kin, Hk(k), H, 0, P + p.off.b[k], nullptr, 0};
#ifdef AB_STATS
      const long long tw0 = clock64();
#endif
      for (int t = blockIdx.x; t < g.tiles(); t += gridDim.x) gemm_tile(g, t, ring);
#ifdef AB_STATS
      if (k == 2 && step == 0 && threadIdx.x == 0 && blockIdx.x < 1024) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_adapt_blk[blockIdx.x][0] = smid;
        g_adapt_blk[blockIdx.x][1] = tw0;
        g_adapt_blk[blockIdx.x][2] = clock64();
      }
#endif
      grid_sync(p.barrier, gen);
    }
    out_rows(Hk(L), P + p.off.W_o, P + p.off.b_o, p.v_obs, p.n, 1.0f / static_cast<float>(B), B, H, R, ring);
    grid_sync(p.barrier, gen);
    if (((step == 0 && p.loss_before) || (p.losses && !fwd_only)) && blockIdx.x == 0) {
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
        const float lb = tot / static_cast<float>(B);
        if (step == 0 && p.loss_before) *p.loss_before = lb;
        if (p.losses && !fwd_only) p.losses[step] = lb;
      }
    }
    if (fwd_only) break;
    // ---------------- backward: output layer
    {
      Gemm gw{kNMax, H, B, R, 1, kNMax, Hk(L), H, 1, Gr + p.off.W_o, H, 2, nullptr, nullptr, 0, kSplitK, p.off.total};
      Gemm gd{B, H, kNMax, R, kNMax, 1, P + p.off.W_o, H, 1, D[L & 1], H, 1, nullptr, Hk(L), H};
      const int t1 = gw.tiles(), t2 = gd.tiles();
      for (int t = blockIdx.x; t < t1 + t2; t += gridDim.x) {
        if (t < t1) gemm_tile(gw, t, ring);
        else gemm_tile(gd, t - t1, ring);
      }
      colsum_split(R, B, kNMax, kNMax, Gr + p.off.b_o, p.off.total);
      grid_sync(p.barrier, gen);
    }
    // ---------------- backward: hidden layers L..1
    for (int k = L; k >= 1; --k) {
      const int Kin = k == 1 ? kZDim : H;
      const float* in = k == 1 ? Z : Hk(k - 1);
      const float* Dk = D[k & 1];
      Gemm gw{H, Kin, B, Dk, 1, H, in, Kin, 1, Gr + p.off.W[k], Kin, 2, nullptr, nullptr, 0, kSplitK, p.off.total};
      const int t1 = gw.tiles();
      int t2 = 0;
      Gemm gd{};
      if (k > 1) {
        gd = Gemm{B, H, H, Dk, H, 1, P + p.off.W[k], H, 1, D[(k - 1) & 1], H, 1, nullptr, Hk(k - 1), H};
        t2 = gd.tiles();
      }
      for (int t = blockIdx.x; t < t1 + t2; t += gridDim.x) {
        if (t < t1) gemm_tile(gw, t, ring);
        else gemm_tile(gd, t - t1, ring);
      }
      colsum_split(Dk, B, H, H, Gr + p.off.b[k], p.off.total);
      // SGD of the layer above, whose gradient partials completed in the previous phase and whose
      // weights no phase reads any more this step (W_o after BO; W_{k+1} after B_{k+1})
      if (k == L) update_range(p, p.off.W_o, p.off.total, step);
      else update_range(p, p.off.W[k + 1], p.off.b[k + 1] + H, step);
      grid_sync(p.barrier, gen);
    }
    // ---------------- SGD of layer 1 (W1, b1); the kernel exit orders it after the last step
    update_range(p, p.off.W[1], p.off.b[1] + H, step);
    if (step + 1 < nsteps) grid_sync(p.barrier, gen);
  }
}

size_t adapt_ws_floats(int B, int H, int L) {
  return (size_t)B * kZDim + (size_t)L * B * H + (size_t)B * kNMax + 2 * (size_t)B * H;
}

cudaError_t launch_adapt(const AdaptParams& p, int num_sms, cudaStream_t s, int* grid_used) {
  int per_sm = 0;
  cudaError_t e = cudaFuncSetAttribute(adapt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kAdaptSmemBytes));
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, adapt_kernel, kAdaptThreads, kAdaptSmemBytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  // Small batches (online adaptation): one CTA per SM — phases have fewer tiles than CTAs and two
  // co-resident busy CTAs halve each other's speed (B = 1024, 4x512: 0.31 vs 0.35 ms). Large
  // batches (offline training): two CTAs per SM hide the mma.sync / ldmatrix latency of the other
  // (B = 32768: 28.1 vs 21.5 TFLOP/s). AUTOBYTE_ADAPT_PER_SM=1|2 overrides.
  int want = p.B >= 4096 ? 2 : 1;
  if (const char* env = std::getenv("AUTOBYTE_ADAPT_PER_SM")) want = std::atoi(env) == 2 ? 2 : 1;
  int grid = num_sms * (per_sm < want ? per_sm : want);
  *grid_used = grid;
  void* args[] = {const_cast<AdaptParams*>(&p)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(adapt_kernel), dim3(grid), dim3(kAdaptThreads), args,
                                     kAdaptSmemBytes, s);
}

}  // namespace ab

#ifdef AB_STATS
extern "C" int ab_debug_adapt_blocks(long long* out, int n) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, ab::g_adapt_blk, sizeof(long long) * 3 * (n < 1024 ? n : 1024)) == cudaSuccess;
}
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
