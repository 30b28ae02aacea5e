// encode.cu — K1: per-job prologue of the scoring path.
//
// K1a, 2*HJ jobs per 256-thread CTA (HJ sized so the grid is about one wave):
//   t'_i[w] = log2(1 + T[i][w] / 1 ms) on valid workers (R#7, R#8); e_i = W_e t'_i + b_e (R#4)
//   two-layer LSTM over i = 0..l_j-1, gates i,f,g,o, h0 = c0 = 0 ("two-layer LSTM", R#5);
//     thread (g, half) owns gate row g of both layers, weights in registers, for HJ jobs
//   x_j = [h | log2 B_d | log2 B_u | n/16 | l/64 | E_m[m] | E_arc[arc]]   (Table 2)
//   K1a takes a job range, so at G > 1 each rank encodes 1/G of the jobs and the x rows are
//   all-gathered before K1b (autobyte.cu run_lstm: NCCL, or stored by K1a's epilogue into every
//   rank's peer window with AUTOBYTE_PEER_X=1). T chunks are prefetched with cp.async (from
//   device memory, or in place from page-locked host memory on the *_host path).
// K1b, 32 jobs per CTA, all jobs:
//   a_j = W1[:, :82] x_j + b1     (layer-1 projection of the job half of the concatenation)
//   w_j = (1/n) sum_{w<n} W_o[w]  (worker-mean fold of the output layer, R#3)
//   beta_j = (1/n) sum_{w<n} b_o[w], and resets the job's arg-max keys.
// This is SIMT work (~1.6 MFLOP per job, 0.03% of C4).
#include <cstdlib>
#include <cstring>

#include "internal.h"
#include "ptx.cuh"

namespace ab {

constexpr int kEncThreads = 256;   // 128 LSTM gate rows x 2 job halves

#ifdef AB_STATS
// K1a phase cycles of block 0 / thread 0, per launch size class: [prologue, chunk staging, gates,
// cells, epilogue] accumulated over launches (tools/enc_phases.py)
__device__ unsigned long long g_enc_phase[5];
#define ENC_T(v) const long long v = clock64()
#define ENC_ACC(i, v) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_enc_phase[i] += clock64() - (v); } while (0)
#else
#define ENC_T(v)
#define ENC_ACC(i, v)
#endif

// logistic and tanh from the ex2 unit: |error| ~ 1e-7 absolute, well inside the 1e-4 / 2e-5
// tolerance the encoder is held to against the float64 oracle (tests/test_gpu_parity.py)
__device__ __forceinline__ float sigmoidf_acc(float z) { return __fdividef(1.0f, 1.0f + __expf(-z)); }
__device__ __forceinline__ float tanh_acc(float z) { return fmaf(2.0f, sigmoidf_acc(2.0f * z), -1.0f); }

// K1a: 2*HJ jobs per 256-thread CTA (HJ = jobs per half, chosen per call so the grid is about one
// wave: HJ = ceil(J / (2 * SMs)), 1..16). Thread (g, half) owns LSTM gate row g of both layers
// (weights in registers) and evaluates it for the HJ jobs of its half, so each step is an FMA-rich
// [HJ jobs x 48|64] x [48|64] product per thread instead of a latency-bound matvec. Jobs with fewer
// layers freeze after their last step (h, c kept), so the final h is the state at step l_j - 1.
// Every job's arithmetic (operation order, explicit fmaf) is independent of HJ and of the CTA it
// lands in, so x is bit-identical however the jobs are split across CTAs or ranks.
template <int HJ>
struct EncCfg {
  static constexpr int NJ = 2 * HJ;                       // jobs per CTA
  static constexpr int CH = HJ <= 8 ? 16 : 8;             // layers staged per chunk
  static constexpr int RC = (2 * NJ * kLstm + kEncThreads - 1) / kEncThreads;   // cells per thread (both layers)
  static constexpr int XS = kXDim + 2;
  static constexpr int E_OFF = 0;                         // sE [NJ][CH][16]
  static constexpr int TL_OFF = E_OFF + NJ * CH * kEmbed;  // sTl [2][NJ][CH][16] (T chunk ring); sX [NJ][XS] aliases it
  static constexpr int H1_OFF = TL_OFF + 2 * NJ * CH * kNMax;  // sH1 [NJ][32]
  static constexpr int H2_OFF = H1_OFF + NJ * kLstm;       // sH2 [NJ][32]
  static constexpr int G_OFF = H2_OFF + NJ * kLstm;        // sG [NJ][128]: layer-1 gates
  static constexpr int G2_OFF = G_OFF + NJ * 4 * kLstm;    // sG2 [NJ][128]: layer-2 gates
  static constexpr int WE_OFF = G2_OFF + NJ * 4 * kLstm;   // sWe [16][16], sBe [16]
  static constexpr int N_OFF = WE_OFF + kEmbed * kNMax + kEmbed;   // int sN[NJ], sL[NJ]
  static constexpr int FLOATS = N_OFF + 2 * NJ;
  static constexpr size_t BYTES = sizeof(float) * FLOATS;
  static_assert(CH * kNMax >= XS, "sX must fit in the sTl chunk it aliases");
};

template <int HJ>
__global__ void __launch_bounds__(kEncThreads) encode_kernel(const __grid_constant__ EncodeParams p) {
  ENC_T(t_kernel);
  using C = EncCfg<HJ>;
  extern __shared__ __align__(16) float smem[];
  float (*sE)[C::CH][kEmbed] = reinterpret_cast<float (*)[C::CH][kEmbed]>(smem + C::E_OFF);
  float* sTring = smem + C::TL_OFF;   // two [NJ][CH][16] chunk buffers
  float* sWe = smem + C::WE_OFF;
  float* sBe = sWe + kEmbed * kNMax;
  float (*sX)[C::XS] = reinterpret_cast<float (*)[C::XS]>(smem + C::TL_OFF);   // after the LSTM
  float (*sH1)[kLstm] = reinterpret_cast<float (*)[kLstm]>(smem + C::H1_OFF);
  float (*sH2)[kLstm] = reinterpret_cast<float (*)[kLstm]>(smem + C::H2_OFF);
  float (*sG)[4 * kLstm] = reinterpret_cast<float (*)[4 * kLstm]>(smem + C::G_OFF);
  float (*sG2)[4 * kLstm] = reinterpret_cast<float (*)[4 * kLstm]>(smem + C::G2_OFF);
  int* sN = reinterpret_cast<int*>(smem + C::N_OFF);
  int* sL = sN + C::NJ;
  const int tid = threadIdx.x;
  const int g = tid & (4 * kLstm - 1), half = tid >> 7;
  const int j0 = p.j_begin + blockIdx.x * C::NJ;
  const int nj = min(C::NJ, p.j_end - j0);
  const float* P = p.params;
  if (tid < C::NJ) {
    sN[tid] = tid < nj ? p.n[j0 + tid] : 1;
    sL[tid] = tid < nj ? p.l[j0 + tid] : 0;
  }
  for (int e = tid; e < kEmbed * kNMax + kEmbed; e += kEncThreads)
    sWe[e] = e < kEmbed * kNMax ? P[p.off.W_e + e] : P[p.off.b_e + e - kEmbed * kNMax];
  for (int e = tid; e < C::NJ * kLstm; e += kEncThreads) {
    (&sH1[0][0])[e] = 0.f;
    (&sH2[0][0])[e] = 0.f;
  }
  float wx1[kEmbed], wh1[kLstm], wx2[kLstm], wh2[kLstm];
  // gate row g of the four matrices: 16-byte loads when the blob offsets allow (they do for the
  // standard layout; one branch for the whole grid). Scalar loads of a row are 64-128 bytes apart
  // across the warp, so each one touched 32 sectors and the 112 of them cost ~27k cycles per launch
  // (tools/enc_phases.py: half of K1a at J = 512)
  if (((p.off.l1Wx | p.off.l1Wh | p.off.l2Wx | p.off.l2Wh) & 3) == 0) {
    const float4* a = reinterpret_cast<const float4*>(P + p.off.l1Wx + g * kEmbed);
    const float4* b = reinterpret_cast<const float4*>(P + p.off.l1Wh + g * kLstm);
    const float4* c = reinterpret_cast<const float4*>(P + p.off.l2Wx + g * kLstm);
    const float4* d4 = reinterpret_cast<const float4*>(P + p.off.l2Wh + g * kLstm);
#pragma unroll
    for (int q = 0; q < kEmbed / 4; ++q) {
      const float4 v = __ldg(a + q);
      wx1[4 * q] = v.x; wx1[4 * q + 1] = v.y; wx1[4 * q + 2] = v.z; wx1[4 * q + 3] = v.w;
    }
#pragma unroll
    for (int q = 0; q < kLstm / 4; ++q) {
      const float4 u = __ldg(b + q), v = __ldg(c + q), w = __ldg(d4 + q);
      wh1[4 * q] = u.x; wh1[4 * q + 1] = u.y; wh1[4 * q + 2] = u.z; wh1[4 * q + 3] = u.w;
      wx2[4 * q] = v.x; wx2[4 * q + 1] = v.y; wx2[4 * q + 2] = v.z; wx2[4 * q + 3] = v.w;
      wh2[4 * q] = w.x; wh2[4 * q + 1] = w.y; wh2[4 * q + 2] = w.z; wh2[4 * q + 3] = w.w;
    }
  } else {
#pragma unroll
    for (int d = 0; d < kEmbed; ++d) wx1[d] = P[p.off.l1Wx + g * kEmbed + d];
#pragma unroll
    for (int d = 0; d < kLstm; ++d) {
      wh1[d] = P[p.off.l1Wh + g * kLstm + d];
      wx2[d] = P[p.off.l2Wx + g * kLstm + d];
      wh2[d] = P[p.off.l2Wh + g * kLstm + d];
    }
  }
  const float bg1 = P[p.off.l1b + g], bg2 = P[p.off.l2b + g];
  // cell states: thread owns cells e = tid + 256 r of the 2·NJ·32 cells, layer 1 first (job
  // (e mod NJ·32) / 32, unit e % 32), so the two layers' updates of a step run on different warps
  float cst[C::RC];
#pragma unroll
  for (int r = 0; r < C::RC; ++r) cst[r] = 0.f;
  __syncthreads();
  int lmax = 0;
  for (int k = 0; k < C::NJ; ++k) lmax = max(lmax, sL[k]);

  // Cell updates of one wavefront step: layer-1 cells of step t (gates sG, t < lmax) and layer-2
  // cells of step t-1 (gates sG2, t > 0); warp-uniform layer (NJ·32 is a multiple of 32).
  // (stash, for encoder fine-tuning: per job and step [e | i f g o c h of layer 1 | of layer 2])
  auto cell_phase = [&](int t) {
#pragma unroll
    for (int r = 0; r < C::RC; ++r) {
      const int e = tid + r * kEncThreads;
      if (e < 2 * C::NJ * kLstm) {
        const bool l2 = e >= C::NJ * kLstm;
        const int idx = l2 ? e - C::NJ * kLstm : e, step = l2 ? t - 1 : t;
        if (l2 ? t > 0 : t < lmax) {
          float (*sGin)[4 * kLstm] = l2 ? sG2 : sG;
          float (*sHout)[kLstm] = l2 ? sH2 : sH1;
          const int jj = idx >> 5, u = idx & (kLstm - 1);
          if (step < sL[jj]) {
            const float ig = sigmoidf_acc(sGin[jj][u]), fg = sigmoidf_acc(sGin[jj][kLstm + u]);
            const float gg = tanh_acc(sGin[jj][2 * kLstm + u]), og = sigmoidf_acc(sGin[jj][3 * kLstm + u]);
            cst[r] = fmaf(fg, cst[r], ig * gg);
            const float h = og * tanh_acc(cst[r]);
            sHout[jj][u] = h;
            if (p.stash) {
              float* st = p.stash + ((size_t)(j0 + jj) * p.l_max + step) * kEncStash + (l2 ? kEmbed + 6 * kLstm : kEmbed);
              st[u] = ig; st[kLstm + u] = fg; st[2 * kLstm + u] = gg; st[3 * kLstm + u] = og;
              st[4 * kLstm + u] = cst[r]; st[5 * kLstm + u] = h;
            }
          }
        }
      }
    }
  };

  // Raw T of one chunk (layers i0 .. i0+CH-1 of the CTA's jobs) -> ring buffer `buf` with 16-byte
  // cp.async; padding workers (w >= n), layers (>= l) and jobs are zero-filled, and log2(1 + 0) = 0
  // is exactly the padding value of t' (R#7), so the log pass needs no masks. The copy of chunk
  // c+1 is in flight while chunk c's LSTM steps run.
  auto prefetch_T = [&](int i0, int buf) {
    float* dst = sTring + buf * (C::NJ * C::CH * kNMax);
    for (int e = tid; e < C::NJ * C::CH * (kNMax / 4); e += kEncThreads) {
      const int jj = e / (C::CH * (kNMax / 4)), r = e % (C::CH * (kNMax / 4)), i = r / (kNMax / 4), w0 = 4 * (r % (kNMax / 4));
      int bytes = 0;
      const float* src = p.T;
      if (jj < nj && i0 + i < sL[jj]) {
        const int left = sN[jj] - w0;
        bytes = left >= 4 ? 16 : (left > 0 ? 4 * left : 0);
        src = p.T + ((size_t)(j0 + jj) * p.l_max + i0 + i) * kNMax + w0;
      }
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst + e * 4)), "l"(src), "r"(bytes)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  ENC_ACC(0, t_kernel);
  if (lmax > 0) prefetch_T(0, 0);   // (sN, sL, sWe were published by the barrier above)
  int ring = 0;

  // Layer wavefront: layer 1 of step t and layer 2 of step t-1 both need only h1(t-1), so their
  // gates are formed in one phase and their cells updated in the next (2 barriers per step
  // instead of 4); the loop runs one step past lmax for the last layer-2 step. Each value is
  // computed with the same operations as in the sequential order.
  for (int i0 = 0; i0 <= lmax && lmax > 0; i0 += C::CH) {
    const int len = min(C::CH, lmax - i0);   // 0 for a tail-only chunk
    const int iend = i0 + C::CH > lmax ? lmax - i0 + 1 : C::CH;
    ENC_T(t_chunk);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();   // chunk i0 landed; the previous chunk's steps are done with the other buffer
    float (*sTl)[C::CH][kNMax] = reinterpret_cast<float (*)[C::CH][kNMax]>(sTring + ring * (C::NJ * C::CH * kNMax));
    if (len > 0 && i0 + C::CH < lmax) prefetch_T(i0 + C::CH, ring ^ 1);
    // t'_i[w] = log2(1 + T[i][w] / 1 ms) on valid workers, 0 on padding (R#7, R#8)
    for (int e = tid; e < C::NJ * len * kNMax; e += kEncThreads) {
      const int jj = e / (len * kNMax), r = e % (len * kNMax), i = r / kNMax, w = r % kNMax;
      sTl[jj][i][w] = log2f(1.0f + sTl[jj][i][w]);
    }
    __syncthreads();
    // e_i = W_e t'_i + b_e (R#4)
    for (int e = tid; e < C::NJ * len * kEmbed; e += kEncThreads) {
      const int jj = e / (len * kEmbed), r = e % (len * kEmbed), i = r / kEmbed, d = r % kEmbed;
      float acc = sBe[d];
#pragma unroll
      for (int w = 0; w < kNMax; ++w) acc = fmaf(sWe[d * kNMax + w], sTl[jj][i][w], acc);
      sE[jj][i][d] = acc;
      if (p.stash && jj < nj && i0 + i < sL[jj]) p.stash[((size_t)(j0 + jj) * p.l_max + i0 + i) * kEncStash + d] = acc;
    }
    __syncthreads();
    ENC_ACC(1, t_chunk);
    for (int i = 0; i < iend; ++i) {
      const int t = i0 + i;
      ENC_T(t_gates);
      if (t > 0 && t < lmax) {
        // both layers (the common case): one pass per job reads h1(t-1) once for the layer-1
        // recurrent term and the layer-2 input, and runs 8 independent FMA chains; each gate's
        // operation order is the one of the single-layer loops below (bit-identical results)
        float z1[HJ], z2[HJ];
#pragma unroll
        for (int k = 0; k < HJ; ++k) {
          const int jj = half * HJ + k;
          const float4* e4 = reinterpret_cast<const float4*>(sE[jj][i]);
          const float4* h14 = reinterpret_cast<const float4*>(sH1[jj]);
          const float4* h24 = reinterpret_cast<const float4*>(sH2[jj]);
          float a0 = bg1, a1 = 0.f, a2 = 0.f, a3 = 0.f;
          float b0 = bg2, b1 = 0.f, b2 = 0.f, b3 = 0.f;
#pragma unroll
          for (int q = 0; q < kEmbed / 4; ++q) {
            const float4 v = e4[q];
            a0 = fmaf(wx1[4 * q], v.x, a0); a1 = fmaf(wx1[4 * q + 1], v.y, a1);
            a2 = fmaf(wx1[4 * q + 2], v.z, a2); a3 = fmaf(wx1[4 * q + 3], v.w, a3);
          }
#pragma unroll
          for (int q = 0; q < kLstm / 4; ++q) {
            const float4 v = h14[q], w = h24[q];
            a0 = fmaf(wh1[4 * q], v.x, a0); a1 = fmaf(wh1[4 * q + 1], v.y, a1);
            a2 = fmaf(wh1[4 * q + 2], v.z, a2); a3 = fmaf(wh1[4 * q + 3], v.w, a3);
            b0 = fmaf(wx2[4 * q], v.x, b0); b1 = fmaf(wx2[4 * q + 1], v.y, b1);
            b2 = fmaf(wx2[4 * q + 2], v.z, b2); b3 = fmaf(wx2[4 * q + 3], v.w, b3);
            b0 = fmaf(wh2[4 * q], w.x, b0); b1 = fmaf(wh2[4 * q + 1], w.y, b1);
            b2 = fmaf(wh2[4 * q + 2], w.z, b2); b3 = fmaf(wh2[4 * q + 3], w.w, b3);
          }
          z1[k] = (a0 + a1) + (a2 + a3);
          z2[k] = (b0 + b1) + (b2 + b3);
        }
#pragma unroll
        for (int k = 0; k < HJ; ++k) {
          sG[half * HJ + k][g] = z1[k];
          sG2[half * HJ + k][g] = z2[k];
        }
      } else if (t < lmax) {   // ---- layer-1 gates of step t (input e_t, h1(t-1)) -> sG
        float z[HJ];
#pragma unroll
        for (int k = 0; k < HJ; ++k) {
          const int jj = half * HJ + k;
          const float4* e4 = reinterpret_cast<const float4*>(sE[jj][i]);
          const float4* h4 = reinterpret_cast<const float4*>(sH1[jj]);
          float a0 = bg1, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
          for (int q = 0; q < kEmbed / 4; ++q) {
            const float4 v = e4[q];
            a0 = fmaf(wx1[4 * q], v.x, a0); a1 = fmaf(wx1[4 * q + 1], v.y, a1);
            a2 = fmaf(wx1[4 * q + 2], v.z, a2); a3 = fmaf(wx1[4 * q + 3], v.w, a3);
          }
#pragma unroll
          for (int q = 0; q < kLstm / 4; ++q) {
            const float4 v = h4[q];
            a0 = fmaf(wh1[4 * q], v.x, a0); a1 = fmaf(wh1[4 * q + 1], v.y, a1);
            a2 = fmaf(wh1[4 * q + 2], v.z, a2); a3 = fmaf(wh1[4 * q + 3], v.w, a3);
          }
          z[k] = (a0 + a1) + (a2 + a3);
        }
#pragma unroll
        for (int k = 0; k < HJ; ++k) sG[half * HJ + k][g] = z[k];
      } else if (t > 0) {      // ---- layer-2 gates of step t-1 (input h1(t-1), h2(t-2)) -> sG2
        float z[HJ];
#pragma unroll
        for (int k = 0; k < HJ; ++k) {
          const int jj = half * HJ + k;
          const float4* x4 = reinterpret_cast<const float4*>(sH1[jj]);
          const float4* h4 = reinterpret_cast<const float4*>(sH2[jj]);
          float a0 = bg2, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
          for (int q = 0; q < kLstm / 4; ++q) {
            const float4 v = x4[q], w = h4[q];
            a0 = fmaf(wx2[4 * q], v.x, a0); a1 = fmaf(wx2[4 * q + 1], v.y, a1);
            a2 = fmaf(wx2[4 * q + 2], v.z, a2); a3 = fmaf(wx2[4 * q + 3], v.w, a3);
            a0 = fmaf(wh2[4 * q], w.x, a0); a1 = fmaf(wh2[4 * q + 1], w.y, a1);
            a2 = fmaf(wh2[4 * q + 2], w.z, a2); a3 = fmaf(wh2[4 * q + 3], w.w, a3);
          }
          z[k] = (a0 + a1) + (a2 + a3);
        }
#pragma unroll
        for (int k = 0; k < HJ; ++k) sG2[half * HJ + k][g] = z[k];
      }
      __syncthreads();
      ENC_ACC(2, t_gates);
      ENC_T(t_cells);
      cell_phase(t);
      __syncthreads();
      ENC_ACC(3, t_cells);
    }
    ring ^= 1;
  }
  ENC_T(t_epi);
  // ---- feature vectors x_j (Table 2; R#6-R#8)
  for (int e = tid; e < nj * kXDim; e += kEncThreads) {
    const int jj = e / kXDim, i = e % kXDim, j = j0 + jj, n = sN[jj];
    float v;
    if (i < kLstm) v = sH2[jj][i];
    else if (i < kLstm + kNMax) v = (i - kLstm) < n ? log2f(p.B_d[(size_t)j * kNMax + i - kLstm]) : 0.f;
    else if (i < kLstm + 2 * kNMax) v = (i - kLstm - kNMax) < n ? log2f(p.B_u[(size_t)j * kNMax + i - kLstm - kNMax]) : 0.f;
    else if (i == kLstm + 2 * kNMax) v = static_cast<float>(n) / 16.0f;
    else if (i == kLstm + 2 * kNMax + 1) v = static_cast<float>(sL[jj]) / 64.0f;
    else if (i < kLstm + 2 * kNMax + 2 + kTypeEmbed) v = P[p.off.E_m + p.m[j] * kTypeEmbed + (i - kLstm - 2 * kNMax - 2)];
    else v = P[p.off.E_arc + p.arc[j] * kTypeEmbed + (i - kLstm - 2 * kNMax - 2 - kTypeEmbed)];
    sX[jj][i] = v;
  }
  __syncthreads();
  if (p.xG <= 1) {
    for (int e = tid; e < nj * kXDim; e += kEncThreads)
      p.x_out[(size_t)(j0 + e / kXDim) * kXDim + e % kXDim] = sX[e / kXDim][e % kXDim];
  } else {
    // x all-gather fused into the epilogue: the rows go straight into every rank's window over
    // NVLink (own window included); the last CTA of this rank raises its flag in every window
    for (int e = tid; e < nj * kXDim; e += kEncThreads) {
      const float v = sX[e / kXDim][e % kXDim];
      const size_t o = (size_t)(j0 + e / kXDim) * kXDim + e % kXDim;
#pragma unroll 1
      for (int r = 0; r < p.xG; ++r) p.xg[r][o] = v;
    }
    __threadfence_system();
    __syncthreads();
    if (tid == 0 && atomicAdd(p.xcounter, 1u) == gridDim.x - 1) {
      *p.xcounter = 0u;
      __threadfence_system();
#pragma unroll 1
      for (int r = 0; r < p.xG; ++r)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p.xflag[r] + p.xrank), "l"(p.xepoch) : "memory");
    }
  }
  ENC_ACC(4, t_epi);
}

// K1b: per-job projections for K2, 32 jobs per CTA, one output column per thread per pass:
//   a[j][c]    = b1[c] + sum_i W1[c][i] x[j][i]            (job half of layer 1)
//   what[j][c] = sum_{w < n_j} W_o[w][c] / n_j             (worker-mean fold of the output layer)
//   beta[j]    = sum_{w < n_j} b_o[w] / n_j, and the job's arg-max keys reset to 0.
// Thread c holds row c of W1's job columns in registers (16-byte loads) and W_o's column c; each
// x_j is a broadcast LDS.128 of the transposed job block.
constexpr int kProjJobs = 32;
constexpr int kProjThreads = 256;

// Candidate-grid axes (a-1; R#8): u_p[p] = (log2 S_p - 21) / 8 and
// u_c[q] = (S_c - 8.5) / 8 in double, rounded once to fp32; K2 reads u_c = (up[c / Q], uc[c % Q]).
__device__ void grid_axes(const EncodeParams& p, long long first, long long stride) {
  for (long long i = first; i < (long long)p.P + p.Q; i += stride) {
    if (i < p.P) p.up_out[i] = static_cast<float>((log2(static_cast<double>(p.S_p[i])) - 21.0) / 8.0);
    else p.uc_out[i - p.P] = static_cast<float>((static_cast<double>(p.S_c[i - p.P]) - 8.5) / 8.0);
  }
}

// K1b's per-job outputs for ONE job j whose x row is xs (shared memory), by `nthreads` threads:
// the operations of project_kernel for that job in the same order (bit-identical): a[c] = (sum_k
// fma(W1[c][k], x[k]) from 0) + b1[c]; w[c] = sum_w fma(W_o[w][c], m[w]) from 0, m = 1/n on valid
// workers; beta = (sum_{w<n} b_o[w]) / n; keys reset.
__device__ void project_one(const EncodeParams& p, int j, const float* xs, int tid, int nthreads) {
  const float* P = p.params;
  const int H = p.H, n = p.n[j];
  if (tid == 0) {
    if (p.beta_out) {
      float acc = 0.f;
      for (int w = 0; w < n; ++w) acc += P[p.off.b_o + w];
      p.beta_out[(size_t)j * p.jv] = acc / static_cast<float>(n);
    }
    if (p.keys) p.keys[j] = 0ull;
    if (p.cur_keys) p.cur_keys[j] = 0ull;
  }
  const float inv_n = 1.0f / static_cast<float>(n);
  const bool vec = (p.off.W[1] & 3) == 0;
  for (int col = tid; col < H; col += nthreads) {
    // the row of W1 and the column of W_o into registers first (all loads in flight together)
    const float* wr = P + p.off.W[1] + (size_t)col * kZDim;
    float w[kZDim], wo[kNMax];
    if (vec) {
#pragma unroll
      for (int q = 0; q < kZDim / 4; ++q) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(wr) + q);
        w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < kZDim; ++k) w[k] = wr[k];
    }
#pragma unroll
    for (int ww = 0; ww < kNMax; ++ww) wo[ww] = P[p.off.W_o + (size_t)ww * H + col];
    const float b1 = P[p.off.b[1] + col];
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < kXDim; ++k) acc = fmaf(w[k], xs[k], acc);
    p.a_out[(size_t)j * p.jv + col] = acc + b1;
    float aw = 0.f;
#pragma unroll
    for (int ww = 0; ww < kNMax; ++ww) aw = fmaf(wo[ww], ww < n ? inv_n : 0.f, aw);
    p.what_out[(size_t)j * p.jv + col] = aw;
  }
}

__global__ void __launch_bounds__(kProjThreads) project_kernel(const __grid_constant__ EncodeParams p) {
  __shared__ __align__(16) float sXt[kXDim][kProjJobs];    // transposed: 4 jobs per LDS.128
  __shared__ __align__(16) float sM[kNMax][kProjJobs];     // mask / n
  const int j0 = blockIdx.x * kProjJobs, tid = threadIdx.x;
  const float* P = p.params;
  const int jn = min(kProjJobs, p.J - j0);
  for (int e = tid; e < kXDim * kProjJobs; e += kProjThreads) {
    const int jj = e / kXDim, i = e % kXDim;
    sXt[i][jj] = (jj < jn) ? p.x_out[(size_t)(j0 + jj) * kXDim + i] : 0.f;
  }
  for (int e = tid; e < kNMax * kProjJobs; e += kProjThreads) {
    const int w = e / kProjJobs, jj = e % kProjJobs;
    const int nj = (jj < jn) ? p.n[j0 + jj] : 1;
    sM[w][jj] = w < nj ? 1.0f / static_cast<float>(nj) : 0.f;
  }
  if (p.up_out && (long long)p.P + p.Q <= kFusedAxes) grid_axes(p, (long long)blockIdx.x * kProjThreads + tid,
                                                                   (long long)gridDim.x * kProjThreads);
  if (tid < jn) {
    const int j = j0 + tid, n = p.n[j];
    if (p.beta_out) {
      float acc = 0.f;
      for (int w = 0; w < n; ++w) acc += P[p.off.b_o + w];
      p.beta_out[(size_t)j * p.jv] = acc / static_cast<float>(n);
    }
    if (p.keys) p.keys[j] = 0ull;
    if (p.cur_keys) p.cur_keys[j] = 0ull;
  }
  const int H = p.H;
  __syncthreads();   // sXt / sM staged
  const bool vec = (p.off.W[1] & 3) == 0;   // rows of W1 (84 floats) are 16-byte aligned
  for (int cb = 0; cb < H; cb += kProjThreads) {
    const int col = cb + tid;
    if (col >= H) continue;
    // row `col` of W1 (its 82 job columns; the last two are the candidate columns, used by K2)
    // straight into registers with 16-byte loads: all 21 are in flight at once, no per-slice
    // barriers (the shared-memory slice staging waited out ~12 L2 round trips per pass)
    float w[kZDim];
    const float* wr = P + p.off.W[1] + (size_t)col * kZDim;
    if (vec) {
#pragma unroll
      for (int q = 0; q < kZDim / 4; ++q) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(wr) + q);
        w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < kZDim; ++k) w[k] = wr[k];
    }
    float wo[kNMax];
#pragma unroll
    for (int ww = 0; ww < kNMax; ++ww) wo[ww] = P[p.off.W_o + (size_t)ww * H + col];
    const float b1 = P[p.off.b[1] + col];
    float acc[kProjJobs];
#pragma unroll
    for (int jj = 0; jj < kProjJobs; ++jj) acc[jj] = 0.f;
#pragma unroll
    for (int k = 0; k < kXDim; ++k) {   // same k order as a plain dot product
      const float4* xv = reinterpret_cast<const float4*>(sXt[k]);
#pragma unroll
      for (int q = 0; q < kProjJobs / 4; ++q) {
        const float4 v = xv[q];
        acc[4 * q] = fmaf(w[k], v.x, acc[4 * q]); acc[4 * q + 1] = fmaf(w[k], v.y, acc[4 * q + 1]);
        acc[4 * q + 2] = fmaf(w[k], v.z, acc[4 * q + 2]); acc[4 * q + 3] = fmaf(w[k], v.w, acc[4 * q + 3]);
      }
    }
#pragma unroll
    for (int jj = 0; jj < kProjJobs; ++jj)
      if (jj < jn) p.a_out[(size_t)(j0 + jj) * p.jv + col] = acc[jj] + b1;
#pragma unroll
    for (int jj = 0; jj < kProjJobs; ++jj) acc[jj] = 0.f;
#pragma unroll
    for (int ww = 0; ww < kNMax; ++ww) {
      const float4* mv = reinterpret_cast<const float4*>(sM[ww]);
#pragma unroll
      for (int q = 0; q < kProjJobs / 4; ++q) {
        const float4 v = mv[q];
        acc[4 * q] = fmaf(wo[ww], v.x, acc[4 * q]); acc[4 * q + 1] = fmaf(wo[ww], v.y, acc[4 * q + 1]);
        acc[4 * q + 2] = fmaf(wo[ww], v.z, acc[4 * q + 2]); acc[4 * q + 3] = fmaf(wo[ww], v.w, acc[4 * q + 3]);
      }
    }
#pragma unroll
    for (int jj = 0; jj < kProjJobs; ++jj)
      if (jj < jn) p.what_out[(size_t)(j0 + jj) * p.jv + col] = acc[jj];
  }
}

template <int HJ>
cudaError_t launch_lstm_hj(const EncodeParams& p, cudaStream_t s) {
  using C = EncCfg<HJ>;
  static unsigned long long attr_done = 0;   // per device: opt in to > 48 KB dynamic shared memory
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (!(attr_done >> (dev & 63) & 1ull)) {
    e = cudaFuncSetAttribute(encode_kernel<HJ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(C::BYTES));
    if (e != cudaSuccess) return e;
    attr_done |= 1ull << (dev & 63);
  }
  const int n = p.j_end - p.j_begin;
  const int blocks = n > 0 ? (n + C::NJ - 1) / C::NJ : 1;
  encode_kernel<HJ><<<blocks, kEncThreads, C::BYTES, s>>>(p);
  return cudaGetLastError();
}

int encode_jobs_per_half(int n, int num_sms) {
  const int hj = (n + 2 * num_sms - 1) / (2 * num_sms);
  return hj < 1 ? 1 : (hj > 16 ? 16 : hj);
}

// ---------------------------------------------------------------- K1s: latency encoder
// One job per 256-thread CTA, for calls with few jobs (the paper's per-job use, PAPER.md:342,
// :539-540: one job scored at a time). Warps 0-3 hold layer 1, warps 4-7 layer 2; lane 4k + gate of
// a warp owns gate row `gate` of unit 8*(warp % 4) + k, weights in registers, so the four gates of a
// cell sit in four adjacent lanes: a step is one gate row per thread (K1a's four accumulation
// chains, bias on chain 0, then (a0 + a1) + (a2 + a3)), three shuffles, K1a's cell update on the
// gate-0 lane, and ONE __syncthreads (h1 / h2 double-buffered by step parity) instead of K1a's two.
// Same operations in the same order as K1a, so x is bit-identical (tested): the kernel choice never
// changes a result. Embeddings e_i are formed 64 layers at a time.
constexpr int kLatThreads = 256;
constexpr int kLatChunk = 64;   // layers of T staged per chunk

__global__ void __launch_bounds__(kLatThreads, 1) encode_latency_kernel(const __grid_constant__ EncodeParams p) {
  __shared__ __align__(16) float sT[kLatChunk][kNMax];      // t' of the chunk
  __shared__ __align__(16) float sE[kLatChunk][kEmbed];     // e_i of the chunk
  __shared__ __align__(16) float sH1[2][kLstm];             // h1 by step parity
  __shared__ __align__(16) float sH2[2][kLstm];             // h2 by step parity
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int j = p.j_begin + blockIdx.x;
  const float* P = p.params;
  const int n = p.n[j], l = p.l[j];
  const bool l2 = warp >= 4;
  const int u = (warp & 3) * 8 + (lane >> 2), gate = lane & 3;
  const int g = gate * kLstm + u;                   // gate row of this thread's layer
  float wx[kLstm], wh[kLstm];                       // layer 1: wx[0..15] = W_x row (over e)
  {
    const float4* a = reinterpret_cast<const float4*>(P + (l2 ? p.off.l2Wx + g * kLstm : p.off.l1Wx + g * kEmbed));
    const float4* b = reinterpret_cast<const float4*>(P + (l2 ? p.off.l2Wh : p.off.l1Wh) + g * kLstm);
    const bool al = ((p.off.l1Wx | p.off.l1Wh | p.off.l2Wx | p.off.l2Wh) & 3) == 0;
#pragma unroll
    for (int q = 0; q < kLstm / 4; ++q) {
      if (q < kEmbed / 4 || l2) {
        const float4 v = al ? __ldg(a + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        wx[4 * q] = v.x; wx[4 * q + 1] = v.y; wx[4 * q + 2] = v.z; wx[4 * q + 3] = v.w;
      } else {
        wx[4 * q] = wx[4 * q + 1] = wx[4 * q + 2] = wx[4 * q + 3] = 0.f;
      }
      const float4 w = al ? __ldg(b + q) : make_float4(0.f, 0.f, 0.f, 0.f);
      wh[4 * q] = w.x; wh[4 * q + 1] = w.y; wh[4 * q + 2] = w.z; wh[4 * q + 3] = w.w;
    }
    if (!al) {   // (unaligned blob offsets: scalar loads)
#pragma unroll
      for (int d = 0; d < kLstm; ++d) {
        wx[d] = l2 ? P[p.off.l2Wx + g * kLstm + d] : (d < kEmbed ? P[p.off.l1Wx + g * kEmbed + d] : 0.f);
        wh[d] = P[(l2 ? p.off.l2Wh : p.off.l1Wh) + g * kLstm + d];
      }
    }
  }
  const float bias = P[(l2 ? p.off.l2b : p.off.l1b) + g];
  // embedding outputs e[i][ed] for i = ei + 16 r (r < 4) of each chunk, W_e row ed in registers
  const int ed = tid & (kEmbed - 1), ei = tid >> 4;
  float we[kNMax];
#pragma unroll
  for (int w = 0; w < kNMax; ++w) we[w] = P[p.off.W_e + ed * kNMax + w];
  const float be = P[p.off.b_e + ed];
  if (tid < 2 * kLstm) {
    (&sH1[0][0])[tid] = 0.f;
    (&sH2[0][0])[tid] = 0.f;
  }
  float cst = 0.f;
  for (int i0 = 0; i0 <= l; i0 += kLatChunk) {
    const int len = min(kLatChunk, l - i0);
    // t'_i[w] = log2(1 + T[i][w] / 1 ms) on valid workers, 0 on padding (R#7, R#8)
#pragma unroll
    for (int r = 0; r < kLatChunk * kNMax / kLatThreads; ++r) {
      const int e = tid + r * kLatThreads, i = e >> 4, w = e & 15;
      float v = 0.f;
      if (i < len && w < n) v = log2f(1.0f + p.T[((size_t)j * p.l_max + i0 + i) * kNMax + w]);
      sT[i][w] = v;
    }
    __syncthreads();
    // e_i = W_e t'_i + b_e (R#4), the accumulation order of K1a
#pragma unroll
    for (int r = 0; r < kLatChunk * kEmbed / kLatThreads; ++r) {
      const int i = ei + 16 * r;
      if (i < len) {
        float acc = be;
#pragma unroll
        for (int w = 0; w < kNMax; ++w) acc = fmaf(we[w], sT[i][w], acc);
        sE[i][ed] = acc;
      }
    }
    __syncthreads();
    // wavefront: layer 1 at step t, layer 2 at step t - 1 (one past the last step for layer 2)
    const int iend = i0 + kLatChunk > l ? l - i0 + 1 : kLatChunk;
    for (int i = 0; i < iend; ++i) {
      const int t = i0 + i;
      const int step = l2 ? t - 1 : t;
      const bool active = step >= 0 && step < l;
      const int rd = (t & 1) ^ 1, wr = t & 1;       // h(t-1) / h(t-2) read, h written
      float a0 = bias, a1 = 0.f, a2 = 0.f, a3 = 0.f;
      if (active) {
        if (!l2) {
          const float4* e4 = reinterpret_cast<const float4*>(sE[i]);
          const float4* h4 = reinterpret_cast<const float4*>(sH1[rd]);
#pragma unroll
          for (int q = 0; q < kEmbed / 4; ++q) {
            const float4 v = e4[q];
            a0 = fmaf(wx[4 * q], v.x, a0); a1 = fmaf(wx[4 * q + 1], v.y, a1);
            a2 = fmaf(wx[4 * q + 2], v.z, a2); a3 = fmaf(wx[4 * q + 3], v.w, a3);
          }
#pragma unroll
          for (int q = 0; q < kLstm / 4; ++q) {
            const float4 v = h4[q];
            a0 = fmaf(wh[4 * q], v.x, a0); a1 = fmaf(wh[4 * q + 1], v.y, a1);
            a2 = fmaf(wh[4 * q + 2], v.z, a2); a3 = fmaf(wh[4 * q + 3], v.w, a3);
          }
        } else {
          const float4* x4 = reinterpret_cast<const float4*>(sH1[rd]);
          const float4* h4 = reinterpret_cast<const float4*>(sH2[rd]);
#pragma unroll
          for (int q = 0; q < kLstm / 4; ++q) {
            const float4 v = x4[q], w = h4[q];
            a0 = fmaf(wx[4 * q], v.x, a0); a1 = fmaf(wx[4 * q + 1], v.y, a1);
            a2 = fmaf(wx[4 * q + 2], v.z, a2); a3 = fmaf(wx[4 * q + 3], v.w, a3);
            a0 = fmaf(wh[4 * q], w.x, a0); a1 = fmaf(wh[4 * q + 1], w.y, a1);
            a2 = fmaf(wh[4 * q + 2], w.z, a2); a3 = fmaf(wh[4 * q + 3], w.w, a3);
          }
        }
      }
      const float z = (a0 + a1) + (a2 + a3);
      const int base = lane & ~3;
      const float zf = __shfl_sync(0xffffffffu, z, base + 1);
      const float zg = __shfl_sync(0xffffffffu, z, base + 2);
      const float zo = __shfl_sync(0xffffffffu, z, base + 3);
      if (gate == 0) {
        if (active) {
          const float ig = sigmoidf_acc(z), fg = sigmoidf_acc(zf), gg = tanh_acc(zg), og = sigmoidf_acc(zo);
          cst = fmaf(fg, cst, ig * gg);
          (l2 ? sH2 : sH1)[wr][u] = og * tanh_acc(cst);
        } else if (step >= l) {
          (l2 ? sH2 : sH1)[wr][u] = (l2 ? sH2 : sH1)[rd][u];   // frozen after the job's last layer
        }
      }
      __syncthreads();
    }
  }
  // ---- feature vector x_j (Table 2; R#6-R#8): the top layer's h after its last step
  __shared__ __align__(16) float sX[kXDim + 2];
  const int hfin = l & 1;   // layer 2's step l - 1 ran at t = l, written to parity l & 1
  if (tid < kXDim) {
    const int i = tid;
    float v;
    if (i < kLstm) v = sH2[hfin][i];
    else if (i < kLstm + kNMax) v = (i - kLstm) < n ? log2f(p.B_d[(size_t)j * kNMax + i - kLstm]) : 0.f;
    else if (i < kLstm + 2 * kNMax) v = (i - kLstm - kNMax) < n ? log2f(p.B_u[(size_t)j * kNMax + i - kLstm - kNMax]) : 0.f;
    else if (i == kLstm + 2 * kNMax) v = static_cast<float>(n) / 16.0f;
    else if (i == kLstm + 2 * kNMax + 1) v = static_cast<float>(l) / 64.0f;
    else if (i < kLstm + 2 * kNMax + 2 + kTypeEmbed) v = P[p.off.E_m + p.m[j] * kTypeEmbed + (i - kLstm - 2 * kNMax - 2)];
    else v = P[p.off.E_arc + p.arc[j] * kTypeEmbed + (i - kLstm - 2 * kNMax - 2 - kTypeEmbed)];
    p.x_out[(size_t)j * kXDim + i] = v;
    sX[i] = v;
  }
  if (p.fuse_project) {   // K1b's work for this job (and the grid axes once), no extra launch
    __syncthreads();
    project_one(p, j, sX, tid, kLatThreads);
    if (p.up_out && blockIdx.x == 0 && (long long)p.P + p.Q <= kFusedAxes) grid_axes(p, tid, kLatThreads);
  }
}

// AUTOBYTE_ENCODER=batched|latency forces K1a / K1s (tests); default: K1s when the call has at most
// one job per SM (and no stash / fused gather, which only K1a implements).
int encoder_choice() {
  const char* e = std::getenv("AUTOBYTE_ENCODER");
  return (e && std::strcmp(e, "batched") == 0) ? 1 : (e && std::strcmp(e, "latency") == 0) ? 2 : 0;
}

// K1a over jobs [p.j_begin, p.j_end): writes rows of p.x_out (global job index).
cudaError_t launch_encode_lstm(const EncodeParams& p, int num_sms, cudaStream_t s, bool* projected) {
  if (projected) *projected = false;
  // (an empty range still launches one CTA when its flag must be raised for the x all-gather)
  if (p.j_end <= p.j_begin && p.xG <= 1) return cudaSuccess;
  const int nj = p.j_end - p.j_begin;
  const int ch = encoder_choice();
  if (p.stash == nullptr && p.xG <= 1 && ch != 1 && (ch == 2 || nj <= num_sms)) {
    encode_latency_kernel<<<nj, kLatThreads, 0, s>>>(p);
    if (projected) *projected = p.fuse_project != 0;
    return cudaGetLastError();
  }
  if (p.fuse_project) {   // K1a does not project: the caller runs K1b
    EncodeParams q = p;
    q.fuse_project = 0;
    return launch_encode_lstm(q, num_sms, s, projected);
  }
  switch (encode_jobs_per_half(p.j_end - p.j_begin, num_sms)) {
    case 1: return launch_lstm_hj<1>(p, s);
    case 2: return launch_lstm_hj<2>(p, s);
    case 3: return launch_lstm_hj<3>(p, s);
    case 4: return launch_lstm_hj<4>(p, s);
    case 5: return launch_lstm_hj<5>(p, s);
    case 6: return launch_lstm_hj<6>(p, s);
    case 7: return launch_lstm_hj<7>(p, s);
    case 8: return launch_lstm_hj<8>(p, s);
    case 9: return launch_lstm_hj<9>(p, s);
    case 10: return launch_lstm_hj<10>(p, s);
    case 11: return launch_lstm_hj<11>(p, s);
    case 12: return launch_lstm_hj<12>(p, s);
    case 13: return launch_lstm_hj<13>(p, s);
    case 14: return launch_lstm_hj<14>(p, s);
    case 15: return launch_lstm_hj<15>(p, s);
    default: return launch_lstm_hj<16>(p, s);
  }
}

// K1b over all p.J jobs (reads p.x_out rows 0..J-1).
cudaError_t launch_project(const EncodeParams& p, cudaStream_t s) {
  if (p.J <= 0) return cudaSuccess;
  project_kernel<<<(p.J + kProjJobs - 1) / kProjJobs, kProjThreads, 0, s>>>(p);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- K0: candidate-grid axes
// Only for grids with P + Q > kFusedAxes (otherwise K1b / K1s form the axes in their epilogue).
__global__ void grid_axes_kernel(const __grid_constant__ EncodeParams p) {
  grid_axes(p, blockIdx.x * (long long)blockDim.x + threadIdx.x, (long long)gridDim.x * blockDim.x);
}

cudaError_t launch_grid_axes(const EncodeParams& p, cudaStream_t s) {
  const long long n = (long long)p.P + p.Q;
  const long long blocks = (n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096;
  grid_axes_kernel<<<static_cast<int>(blocks), 256, 0, s>>>(p);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- AUTOBYTE_CHECK=1 validation
__global__ void check_jobs_kernel(int J, int l_max, const float* T, const float* B_d, const float* B_u,
                                  const int32_t* n, const int32_t* l, const int32_t* m, const int32_t* arc,
                                  int n_model, int n_arch, int* flag) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  const int nj = n[j], lj = l[j];
  bool bad = nj < 1 || nj > kNMax || lj < 1 || lj > l_max || m[j] < 0 || m[j] >= n_model || arc[j] < 0 ||
             arc[j] >= n_arch;
  if (!bad) {
    for (int w = 0; w < nj; ++w)
      bad |= !(B_d[(size_t)j * kNMax + w] > 0.f) || !(B_u[(size_t)j * kNMax + w] > 0.f);
    for (int i = 0; i < lj && !bad; ++i)
      for (int w = 0; w < nj; ++w) bad |= !(T[((size_t)j * l_max + i) * kNMax + w] >= 0.f);
  }
  if (bad) atomicOr(flag, 1);
}

cudaError_t launch_check(const autobyte_job_stats& jb, int n_max, int n_model, int n_arch, int* flag,
                         cudaStream_t s) {
  (void)n_max;
  check_jobs_kernel<<<(jb.J + 127) / 128, 128, 0, s>>>(jb.J, jb.l_max, jb.T, jb.B_down, jb.B_up, jb.n_workers,
                                                       jb.n_layers, jb.model_type, jb.arch_type, n_model, n_arch,
                                                       flag);
  return cudaGetLastError();
}

__global__ void check_grid_kernel(int P, int Q, const int64_t* sp, const float* sc, int* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool bad = false;
  if (i < P) bad |= sp[i] < 4096 || (i > 0 && !(sp[i] > sp[i - 1]));
  if (i < Q) bad |= !(sc[i] >= 1.0f) || (i > 0 && !(sc[i] > sc[i - 1]));
  if (bad) atomicOr(flag, 2);
}

cudaError_t launch_check_grid(const autobyte_grid& g, int* flag, cudaStream_t s) {
  const int n = g.P > g.Q ? g.P : g.Q;
  check_grid_kernel<<<(n + 127) / 128, 128, 0, s>>>(g.P, g.Q, g.partition_bytes, g.credit_mult, flag);
  return cudaGetLastError();
}

AB_STATUS_SETTER(set_status_encode)   // device status word pointer of this unit (ptx.cuh)

}  // namespace ab

#ifdef AB_STATS
extern "C" int ab_debug_enc_phases(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, ab::g_enc_phase, sizeof(unsigned long long) * 5) != cudaSuccess) return -1;
  if (reset) {
    unsigned long long z[5] = {};
    cudaMemcpyToSymbol(ab::g_enc_phase, z, sizeof(z));
  }
  return 0;
}
#endif
