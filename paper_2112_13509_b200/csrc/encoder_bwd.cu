// encoder_bwd.cu — encoder fine-tuning (R#20): the gradient of the objective
// with respect to every encoder parameter, given dX = d obj / d x_b from K4 (the layer-1 input
// gradient, pre-update W1), by back-propagation through time of the two-layer LSTM of K1a (P:402,
// R#5), the per-layer embedding W_e, b_e (R#4) and the type tables E_m, E_arc (R#6).
//
// K8 `encoder_bwd_kernel<HJ>`: 2*HJ samples per 256-thread CTA, the mirror image of K1a. The
// forward states come from K1a's stash ([e | i f g o c h | i f g o c h] per sample and step).
// Per reverse step: the cell threads (sample, unit) turn (dh, dc) into the four gate
// pre-activation gradients dz; the gate-row threads (g, half) accumulate dWx[g][:], dWh[g][:],
// db[g] in registers over their samples and all steps (like K1a keeps W in registers); the
// input-gradient threads (sample, d) form Wx^T dz and Wh^T dz from the weights in shared memory.
// Every per-sample quantity is computed in a fixed order and the CTA's weight-gradient partials
// are written, not atomically added, so the result is deterministic.
// K9 `encoder_update_kernel`: sums the CTA partials in fixed order (plus the E_m / E_arc rows from
// dX), then applies the same SGD / Adam update as K4 to the encoder parameters.
#include "internal.h"
#include "ptx.cuh"

namespace ab {

constexpr int kBwdThreads = 256;
constexpr int kG = 4 * kLstm;     // gate rows per layer (i, f, g, o)
// shared-memory weights, row-major [gate][input]: Wx1 [128][16], Wh1, Wx2, Wh2 [128][32]
constexpr int kWx1 = 0, kWh1 = kWx1 + kG * kEmbed, kWx2 = kWh1 + kG * kLstm, kWh2 = kWx2 + kG * kLstm;
constexpr int kWTot = kWh2 + kG * kLstm;

template <int HJ>
struct BwdCfg {
  static constexpr int NJ = 2 * HJ;
  static constexpr int RC = (NJ * kLstm + kBwdThreads - 1) / kBwdThreads;   // cells per thread
  // per-sample staging: e (16) | h1 prev (32) | h1 (32) | h2 prev (32)
  static constexpr int IN = kEmbed + 3 * kLstm;
  static constexpr int W_OFF = 0;
  static constexpr int IN_OFF = W_OFF + kWTot;              // [NJ][IN]
  static constexpr int DZ1_OFF = IN_OFF + NJ * IN;          // [NJ][128]
  static constexpr int DZ2_OFF = DZ1_OFF + NJ * kG;         // [NJ][128]
  static constexpr int DH1_OFF = DZ2_OFF + NJ * kG;         // [2][NJ][32] carried dh of layer 1 (ping-pong)
  static constexpr int DH2_OFF = DH1_OFF + 2 * NJ * kLstm;  // [2][NJ][32]
  static constexpr int DX2_OFF = DH2_OFF + 2 * NJ * kLstm;  // [NJ][32]  Wx2^T dz2
  static constexpr int DE_OFF = DX2_OFF + NJ * kLstm;       // [NJ][16]  Wx1^T dz1
  static constexpr int TF_OFF = DE_OFF + NJ * kEmbed;       // [NJ][16]  t' of the step
  static constexpr int N_OFF = TF_OFF + NJ * kNMax;         // int sN[NJ], sL[NJ]
  static constexpr int FLOATS = N_OFF + 2 * NJ;
  static constexpr size_t BYTES = sizeof(float) * FLOATS;
};

template <int HJ>
__global__ void __launch_bounds__(kBwdThreads) encoder_bwd_kernel(const __grid_constant__ EncodeParams p,
                                                                   const float* __restrict__ dX, int ldx,
                                                                   float* __restrict__ partial) {
  using C = BwdCfg<HJ>;
  extern __shared__ __align__(16) float sm[];
  float* sW = sm + C::W_OFF;
  float (*sIn)[C::IN] = reinterpret_cast<float (*)[C::IN]>(sm + C::IN_OFF);
  float (*sDZ1)[kG] = reinterpret_cast<float (*)[kG]>(sm + C::DZ1_OFF);
  float (*sDZ2)[kG] = reinterpret_cast<float (*)[kG]>(sm + C::DZ2_OFF);
  float* sDH1 = sm + C::DH1_OFF;
  float* sDH2 = sm + C::DH2_OFF;
  float (*sDX2)[kLstm] = reinterpret_cast<float (*)[kLstm]>(sm + C::DX2_OFF);
  float (*sDE)[kEmbed] = reinterpret_cast<float (*)[kEmbed]>(sm + C::DE_OFF);
  float (*sTF)[kNMax] = reinterpret_cast<float (*)[kNMax]>(sm + C::TF_OFF);
  int* sN = reinterpret_cast<int*>(sm + C::N_OFF);
  int* sL = sN + C::NJ;
  const int tid = threadIdx.x;
  const int g = tid & (kG - 1), half = tid >> 7;
  const int j0 = p.j_begin + blockIdx.x * C::NJ;
  const int nj = min(C::NJ, p.j_end - j0);
  const float* P = p.params;
  for (int e = tid; e < kG * kEmbed; e += kBwdThreads) sW[kWx1 + e] = P[p.off.l1Wx + e];
  for (int e = tid; e < kG * kLstm; e += kBwdThreads) {
    sW[kWh1 + e] = P[p.off.l1Wh + e];
    sW[kWx2 + e] = P[p.off.l2Wx + e];
    sW[kWh2 + e] = P[p.off.l2Wh + e];
  }
  if (tid < C::NJ) {
    sN[tid] = tid < nj ? p.n[j0 + tid] : 1;
    sL[tid] = tid < nj ? p.l[j0 + tid] : 0;
  }
  // carried dh: layer 2 starts from dX[0:32] (the top layer's final h is x[0:32]), layer 1 from 0
  for (int e = tid; e < C::NJ * kLstm; e += kBwdThreads) {
    const int jj = e >> 5, u = e & (kLstm - 1);
    sDH2[e] = jj < nj ? dX[(size_t)(j0 + jj) * ldx + u] : 0.f;
    sDH1[e] = 0.f;
  }
  float dc1[C::RC], dc2[C::RC];
#pragma unroll
  for (int r = 0; r < C::RC; ++r) dc1[r] = dc2[r] = 0.f;
  // gate-row gradient accumulators of row g over this half's samples
  float gWx1[kEmbed], gWh1[kLstm], gWx2[kLstm], gWh2[kLstm];
#pragma unroll
  for (int d = 0; d < kEmbed; ++d) gWx1[d] = 0.f;
#pragma unroll
  for (int d = 0; d < kLstm; ++d) gWh1[d] = gWx2[d] = gWh2[d] = 0.f;
  float gb1 = 0.f, gb2 = 0.f;
  float gWe = 0.f, gbe = 0.f;   // thread (d' = tid / 16, w = tid % 16) of W_e; b_e on w == 0
  __syncthreads();
  int lmax = 0;
  for (int k = 0; k < C::NJ; ++k) lmax = max(lmax, sL[k]);
  int cur = 0;   // ping-pong index of the carried dh
  const size_t ls = (size_t)p.l_max * kEncStash;

  for (int step = lmax - 1; step >= 0; --step) {
    // ---- stage the step's inputs: e, h1(step-1), h1(step), h2(step-1), t'(step)
    for (int e = tid; e < C::NJ * C::IN; e += kBwdThreads) {
      const int jj = e / C::IN, q = e % C::IN;
      float v = 0.f;
      if (jj < nj && step < sL[jj]) {
        const float* st = p.stash + (size_t)(j0 + jj) * ls + (size_t)step * kEncStash;
        if (q < kEmbed) v = st[q];
        else if (q < kEmbed + kLstm) v = step > 0 ? st[-kEncStash + kEmbed + 5 * kLstm + (q - kEmbed)] : 0.f;
        else if (q < kEmbed + 2 * kLstm) v = st[kEmbed + 5 * kLstm + (q - kEmbed - kLstm)];
        else v = step > 0 ? st[-kEncStash + kEmbed + 11 * kLstm + (q - kEmbed - 2 * kLstm)] : 0.f;
      }
      sIn[jj][q] = v;
    }
    for (int e = tid; e < C::NJ * kNMax; e += kBwdThreads) {
      const int jj = e / kNMax, w = e % kNMax;
      float v = 0.f;
      if (jj < nj && step < sL[jj] && w < sN[jj]) v = log2f(1.0f + p.T[((size_t)(j0 + jj) * p.l_max + step) * kNMax + w]);
      sTF[jj][w] = v;
    }
    // ---- layer 2 cell backward: dz2 from (dh2, dc2) and the stashed gates
    const float* dh2 = sDH2 + cur * C::NJ * kLstm;
    const float* dh1 = sDH1 + cur * C::NJ * kLstm;
    float* dh2n = sDH2 + (cur ^ 1) * C::NJ * kLstm;
    float* dh1n = sDH1 + (cur ^ 1) * C::NJ * kLstm;
#pragma unroll
    for (int r = 0; r < C::RC; ++r) {
      const int e = tid + r * kBwdThreads;
      if (e < C::NJ * kLstm) {
        const int jj = e >> 5, u = e & (kLstm - 1);
        float z0 = 0.f, z1 = 0.f, z2 = 0.f, z3 = 0.f;
        if (jj < nj && step < sL[jj]) {
          const float* st = p.stash + (size_t)(j0 + jj) * ls + (size_t)step * kEncStash + kEmbed + 6 * kLstm;
          const float ig = st[u], fg = st[kLstm + u], gg = st[2 * kLstm + u], og = st[3 * kLstm + u];
          const float c = st[4 * kLstm + u];
          const float cp = step > 0 ? st[-kEncStash + 4 * kLstm + u] : 0.f;
          const float tc = tanhf(c);
          const float dh = dh2[e];
          const float dc = fmaf(dh * og, 1.0f - tc * tc, dc2[r]);
          z0 = dc * gg * ig * (1.0f - ig);
          z1 = dc * cp * fg * (1.0f - fg);
          z2 = dc * ig * (1.0f - gg * gg);
          z3 = dh * tc * og * (1.0f - og);
          dc2[r] = dc * fg;
        }
        sDZ2[jj][u] = z0; sDZ2[jj][kLstm + u] = z1; sDZ2[jj][2 * kLstm + u] = z2; sDZ2[jj][3 * kLstm + u] = z3;
      }
    }
    __syncthreads();
    // ---- layer 2 weight gradients (row g) and input gradients Wx2^T dz2, Wh2^T dz2
#pragma unroll
    for (int k = 0; k < HJ; ++k) {
      const int jj = half * HJ + k;
      const float dz = sDZ2[jj][g];
      const float* x2 = sIn[jj] + kEmbed + kLstm;         // h1(step)
      const float* h2p = sIn[jj] + kEmbed + 2 * kLstm;    // h2(step-1)
#pragma unroll
      for (int d = 0; d < kLstm; ++d) {
        gWx2[d] = fmaf(dz, x2[d], gWx2[d]);
        gWh2[d] = fmaf(dz, h2p[d], gWh2[d]);
      }
      gb2 += dz;
    }
    for (int e = tid; e < C::NJ * 2 * kLstm; e += kBwdThreads) {
      const int jj = e / (2 * kLstm), q = e % (2 * kLstm), d = q & (kLstm - 1);
      const float* Wm = sW + (q < kLstm ? kWx2 : kWh2);
      float a0 = 0.f, a1 = 0.f;
#pragma unroll 8
      for (int gg = 0; gg < kG; gg += 2) {
        a0 = fmaf(Wm[gg * kLstm + d], sDZ2[jj][gg], a0);
        a1 = fmaf(Wm[(gg + 1) * kLstm + d], sDZ2[jj][gg + 1], a1);
      }
      const bool act = jj < nj && step < sL[jj];
      if (q < kLstm) sDX2[jj][d] = act ? a0 + a1 : 0.f;
      else dh2n[jj * kLstm + d] = act ? a0 + a1 : dh2[jj * kLstm + d];   // inactive: carry
    }
    __syncthreads();
    // ---- layer 1 cell backward (dh1 = carried + Wx2^T dz2)
#pragma unroll
    for (int r = 0; r < C::RC; ++r) {
      const int e = tid + r * kBwdThreads;
      if (e < C::NJ * kLstm) {
        const int jj = e >> 5, u = e & (kLstm - 1);
        float z0 = 0.f, z1 = 0.f, z2 = 0.f, z3 = 0.f;
        if (jj < nj && step < sL[jj]) {
          const float* st = p.stash + (size_t)(j0 + jj) * ls + (size_t)step * kEncStash + kEmbed;
          const float ig = st[u], fg = st[kLstm + u], gg = st[2 * kLstm + u], og = st[3 * kLstm + u];
          const float c = st[4 * kLstm + u];
          const float cp = step > 0 ? st[-kEncStash + 4 * kLstm + u] : 0.f;
          const float tc = tanhf(c);
          const float dh = dh1[e] + sDX2[jj][u];
          const float dc = fmaf(dh * og, 1.0f - tc * tc, dc1[r]);
          z0 = dc * gg * ig * (1.0f - ig);
          z1 = dc * cp * fg * (1.0f - fg);
          z2 = dc * ig * (1.0f - gg * gg);
          z3 = dh * tc * og * (1.0f - og);
          dc1[r] = dc * fg;
        }
        sDZ1[jj][u] = z0; sDZ1[jj][kLstm + u] = z1; sDZ1[jj][2 * kLstm + u] = z2; sDZ1[jj][3 * kLstm + u] = z3;
      }
    }
    __syncthreads();
    // ---- layer 1 weight gradients and input gradients Wx1^T dz1 (-> e), Wh1^T dz1 (-> h1(step-1))
#pragma unroll
    for (int k = 0; k < HJ; ++k) {
      const int jj = half * HJ + k;
      const float dz = sDZ1[jj][g];
      const float* x1 = sIn[jj];                   // e(step)
      const float* h1p = sIn[jj] + kEmbed;         // h1(step-1)
#pragma unroll
      for (int d = 0; d < kEmbed; ++d) gWx1[d] = fmaf(dz, x1[d], gWx1[d]);
#pragma unroll
      for (int d = 0; d < kLstm; ++d) gWh1[d] = fmaf(dz, h1p[d], gWh1[d]);
      gb1 += dz;
    }
    for (int e = tid; e < C::NJ * (kEmbed + kLstm); e += kBwdThreads) {
      const int jj = e / (kEmbed + kLstm), q = e % (kEmbed + kLstm);
      const bool isx = q < kEmbed;
      const int d = isx ? q : q - kEmbed, ld = isx ? kEmbed : kLstm;
      const float* Wm = sW + (isx ? kWx1 : kWh1);
      float a0 = 0.f, a1 = 0.f;
#pragma unroll 8
      for (int gg = 0; gg < kG; gg += 2) {
        a0 = fmaf(Wm[gg * ld + d], sDZ1[jj][gg], a0);
        a1 = fmaf(Wm[(gg + 1) * ld + d], sDZ1[jj][gg + 1], a1);
      }
      const bool act = jj < nj && step < sL[jj];
      if (isx) sDE[jj][d] = act ? a0 + a1 : 0.f;
      else dh1n[jj * kLstm + d] = act ? a0 + a1 : dh1[jj * kLstm + d];
    }
    __syncthreads();
    // ---- embedding: dW_e[d'][w] += de[d'] t'[w], db_e += de
    {
      const int dp = tid >> 4, w = tid & 15;
      for (int jj = 0; jj < C::NJ; ++jj) {
        const float de = sDE[jj][dp];
        gWe = fmaf(de, sTF[jj][w], gWe);
        if (w == 0) gbe += de;
      }
    }
    cur ^= 1;
    __syncthreads();
  }
  // ---- per-CTA partials in the blob layout of the encoder parameters (E_m / E_arc rows: K9)
  float* out = partial + (size_t)blockIdx.x * p.off.W[1];
  // the two halves hold different samples of the same row: combine through shared memory in a
  // fixed order (half 0 + half 1)
  float* red = sm;   // reuse the weight area (no longer needed)
  __syncthreads();
  auto combine = [&](float v, int64_t dst) {   // called by all threads, same dst for (g, 0) and (g, 1)
    if (half == 1) red[g] = v;
    __syncthreads();
    if (half == 0) out[dst] = v + red[g];
    __syncthreads();
  };
#pragma unroll
  for (int d = 0; d < kEmbed; ++d) combine(gWx1[d], p.off.l1Wx + g * kEmbed + d);
#pragma unroll
  for (int d = 0; d < kLstm; ++d) {
    combine(gWh1[d], p.off.l1Wh + g * kLstm + d);
    combine(gWx2[d], p.off.l2Wx + g * kLstm + d);
    combine(gWh2[d], p.off.l2Wh + g * kLstm + d);
  }
  combine(gb1, p.off.l1b + g);
  combine(gb2, p.off.l2b + g);
  out[p.off.W_e + tid] = gWe;                         // W_e [16][16] row-major = tid
  if ((tid & 15) == 0) out[p.off.b_e + (tid >> 4)] = gbe;
}

// K9: g[i] = sum over CTAs of partial[cta][i] (fixed order) for i in the encoder range, with the
// E_m / E_arc rows summed from dX over the samples in order; then SGD or Adam (as K4).
__global__ void encoder_update_kernel(const EncodeParams p, const float* __restrict__ dX, int ldx, int B,
                                      const float* __restrict__ partial, int nparts, int opt, float lr, float beta1,
                                      float beta2, float eps, long long t, float* m, float* v) {
  const long long n_enc = p.off.W[1];
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_enc) return;
  float gsum = 0.f;
  if (i < p.off.W_e) {   // E_m [types][8] then E_arc [arch][8]
    const bool is_m = i < p.off.E_arc;
    const long long rel = is_m ? i - p.off.E_m : i - p.off.E_arc;
    const int row = static_cast<int>(rel / kTypeEmbed), col = static_cast<int>(rel % kTypeEmbed);
    const int xcol = kLstm + 2 * kNMax + 2 + (is_m ? 0 : kTypeEmbed) + col;
    const int32_t* sel = is_m ? p.m : p.arc;
    for (int b = 0; b < B; ++b)
      if (sel[b] == row) gsum += dX[(size_t)b * ldx + xcol];
  } else {
    for (int c = 0; c < nparts; ++c) gsum += partial[(size_t)c * n_enc + i];
  }
  float* P = const_cast<float*>(p.params);
  if (opt == AB_OPT_ADAM) {
    const float step_size = static_cast<float>(lr / (1.0 - pow(static_cast<double>(beta1), static_cast<double>(t))));
    const float sqrt_bc2 = static_cast<float>(sqrt(1.0 - pow(static_cast<double>(beta2), static_cast<double>(t))));
    const float mm = fmaf(beta1, m[i], (1.0f - beta1) * gsum);
    const float vv = fmaf(beta2, v[i], (1.0f - beta2) * (gsum * gsum));
    m[i] = mm;
    v[i] = vv;
    P[i] = P[i] - step_size * (mm / (sqrtf(vv) / sqrt_bc2 + eps));
  } else {
    P[i] = P[i] - lr * gsum;
  }
}

int encoder_bwd_jobs_per_half(int n, int num_sms) {
  const int hj = (n + 2 * num_sms - 1) / (2 * num_sms);
  return hj <= 1 ? 1 : hj <= 2 ? 2 : hj <= 4 ? 4 : 8;
}

template <int HJ>
cudaError_t launch_bwd_hj(const EncodeParams& p, const float* dX, int ldx, float* partial, int* nparts,
                          cudaStream_t s) {
  using C = BwdCfg<HJ>;
  static unsigned long long attr_done = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (!(attr_done >> (dev & 63) & 1ull)) {
    e = cudaFuncSetAttribute(encoder_bwd_kernel<HJ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(C::BYTES));
    if (e != cudaSuccess) return e;
    attr_done |= 1ull << (dev & 63);
  }
  const int grid = (p.j_end - p.j_begin + C::NJ - 1) / C::NJ;
  *nparts = grid;
  encoder_bwd_kernel<HJ><<<grid, kBwdThreads, C::BYTES, s>>>(p, dX, ldx, partial);
  return cudaGetLastError();
}

int encoder_bwd_parts(int B, int num_sms) {
  const int hj = encoder_bwd_jobs_per_half(B, num_sms);
  return (B + 2 * hj - 1) / (2 * hj);
}

cudaError_t launch_encoder_bwd(const EncodeParams& p, const float* dX, int ldx, float* partial, int num_sms,
                               int* nparts, cudaStream_t s) {
  switch (encoder_bwd_jobs_per_half(p.j_end - p.j_begin, num_sms)) {
    case 1: return launch_bwd_hj<1>(p, dX, ldx, partial, nparts, s);
    case 2: return launch_bwd_hj<2>(p, dX, ldx, partial, nparts, s);
    case 4: return launch_bwd_hj<4>(p, dX, ldx, partial, nparts, s);
    default: return launch_bwd_hj<8>(p, dX, ldx, partial, nparts, s);
  }
}

cudaError_t launch_encoder_update(const EncodeParams& p, const float* dX, int ldx, int B, const float* partial,
                                  int nparts, int opt, float lr, float beta1, float beta2, float eps, long long t,
                                  float* m, float* v, cudaStream_t s) {
  const long long n = p.off.W[1];
  encoder_update_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, s>>>(p, dX, ldx, B, partial, nparts, opt, lr,
                                                                          beta1, beta2, eps, t, m, v);
  return cudaGetLastError();
}

AB_STATUS_SETTER(set_status_encoder_bwd)   // device status word pointer of this unit (ptx.cuh)

}  // namespace ab
