// encode.cu — K1: per-job prologue of the scoring path.
//
// K1a, 16 jobs per 256-thread CTA:
//   t'_i[w] = log2(1 + T[i][w] / 1 ms) on valid workers (R#7, R#8); e_i = W_e t'_i + b_e (R#4)
//   two-layer LSTM over i = 0..l_j-1, gates i,f,g,o, h0 = c0 = 0 ("two-layer LSTM", R#5);
//     thread (g, half) owns gate row g of both layers, weights in registers, for 8 jobs
//   x_j = [h | log2 B_d | log2 B_u | n/16 | l/64 | E_m[m] | E_arc[arc]]   (Table 2)
//   beta_j = (1/n) sum_{w<n} b_o[w], and resets the job's arg-max keys.
// K1b, 32 jobs per CTA:
//   a_j = W1[:, :82] x_j + b1     (layer-1 projection of the job half of the concatenation)
//   w_j = (1/n) sum_{w<n} W_o[w]  (worker-mean fold of the output layer, R#3)
// This is SIMT work (~1.6 MFLOP per job, 0.03% of C4).
#include "internal.h"
#include "ptx.cuh"

namespace ab {

constexpr int kEncThreads = 256;   // 128 LSTM gate rows x 2 job halves
constexpr int kEncJobs = 16;       // jobs per CTA (8 per half)
constexpr int kHalfJobs = kEncJobs / 2;
constexpr int kChunk = 16;         // layers whose embeddings are staged in shared memory at a time

// logistic and tanh from the ex2 unit: |error| ~ 1e-7 absolute, well inside the 1e-4 / 2e-5
// tolerance the encoder is held to against the float64 oracle (tests/test_gpu_parity.py)
__device__ __forceinline__ float sigmoidf_acc(float z) { return __fdividef(1.0f, 1.0f + __expf(-z)); }
__device__ __forceinline__ float tanh_acc(float z) { return 2.0f * sigmoidf_acc(2.0f * z) - 1.0f; }

// K1a: 16 jobs per CTA. Thread (g, half) owns LSTM gate row g of both layers (weights in
// registers) and evaluates it for the 8 jobs of its half, so each step is an FMA-rich
// [8 jobs x 48|64] x [48|64] product per thread instead of a latency-bound matvec. Jobs with fewer
// layers freeze after their last step (h, c kept), so the final h is the state at step l_j - 1.
__global__ void __launch_bounds__(kEncThreads) encode_kernel(const __grid_constant__ EncodeParams p) {
  __shared__ __align__(16) float sE[kEncJobs][kChunk][kEmbed];   // layer embeddings e_i of the chunk
  __shared__ float sTl[kEncJobs][kChunk][kNMax];                  // log2(1 + T) of the chunk
  __shared__ __align__(16) float sH1[kEncJobs][kLstm], sH2[kEncJobs][kLstm];
  __shared__ float sG[kEncJobs][4 * kLstm];
  float (*sX)[kXDim + 2] = reinterpret_cast<float (*)[kXDim + 2]>(&sTl[0][0][0]);   // reused after the LSTM
  __shared__ int sN[kEncJobs], sL[kEncJobs];
  const int tid = threadIdx.x;
  const int g = tid & (4 * kLstm - 1), half = tid >> 7;
  const int j0 = blockIdx.x * kEncJobs;
  const int nj = min(kEncJobs, p.J - j0);
  const float* P = p.params;
  if (tid < kEncJobs) {
    sN[tid] = tid < nj ? p.n[j0 + tid] : 1;
    sL[tid] = tid < nj ? p.l[j0 + tid] : 0;
  }
  for (int e = tid; e < kEncJobs * kLstm; e += kEncThreads) {
    (&sH1[0][0])[e] = 0.f;
    (&sH2[0][0])[e] = 0.f;
  }
  float wx1[kEmbed], wh1[kLstm], wx2[kLstm], wh2[kLstm];
#pragma unroll
  for (int d = 0; d < kEmbed; ++d) wx1[d] = P[p.off.l1Wx + g * kEmbed + d];
#pragma unroll
  for (int d = 0; d < kLstm; ++d) {
    wh1[d] = P[p.off.l1Wh + g * kLstm + d];
    wx2[d] = P[p.off.l2Wx + g * kLstm + d];
    wh2[d] = P[p.off.l2Wh + g * kLstm + d];
  }
  const float bg1 = P[p.off.l1b + g], bg2 = P[p.off.l2b + g];
  // cell states: thread owns (job = tid / 16, cells 2*(tid % 16), +1) of each layer
  const int cj = tid >> 4, cc = (tid & 15) * 2;
  float c1[2] = {0.f, 0.f}, c2[2] = {0.f, 0.f};
  __syncthreads();
  int lmax = 0;
  for (int k = 0; k < kEncJobs; ++k) lmax = max(lmax, sL[k]);

  for (int i0 = 0; i0 < lmax; i0 += kChunk) {
    const int len = min(kChunk, lmax - i0);
    __syncthreads();
    // t'_i[w] = log2(1 + T[i][w] / 1 ms) on valid workers, 0 on padding (R#7, R#8)
    for (int e = tid; e < kEncJobs * len * kNMax; e += kEncThreads) {
      const int jj = e / (len * kNMax), r = e % (len * kNMax), i = r / kNMax, w = r % kNMax;
      float v = 0.f;
      if (jj < nj && i0 + i < sL[jj] && w < sN[jj]) v = log2f(1.0f + p.T[((size_t)(j0 + jj) * p.l_max + i0 + i) * kNMax + w]);
      sTl[jj][i][w] = v;
    }
    __syncthreads();
    // e_i = W_e t'_i + b_e (R#4)
    for (int e = tid; e < kEncJobs * len * kEmbed; e += kEncThreads) {
      const int jj = e / (len * kEmbed), r = e % (len * kEmbed), i = r / kEmbed, d = r % kEmbed;
      float acc = P[p.off.b_e + d];
#pragma unroll
      for (int w = 0; w < kNMax; ++w) acc = fmaf(P[p.off.W_e + d * kNMax + w], sTl[jj][i][w], acc);
      sE[jj][i][d] = acc;
    }
    __syncthreads();
    for (int i = 0; i < len; ++i) {
      // ---- layer 1 gates for the 8 jobs of this half
      float z[kHalfJobs];
#pragma unroll
      for (int k = 0; k < kHalfJobs; ++k) {
        const int jj = half * kHalfJobs + k;
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
      for (int k = 0; k < kHalfJobs; ++k) sG[half * kHalfJobs + k][g] = z[k];
      __syncthreads();
      if (i0 + i < sL[cj]) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int c = cc + u;
          const float ig = sigmoidf_acc(sG[cj][c]), fg = sigmoidf_acc(sG[cj][kLstm + c]);
          const float gg = tanh_acc(sG[cj][2 * kLstm + c]), og = sigmoidf_acc(sG[cj][3 * kLstm + c]);
          c1[u] = fg * c1[u] + ig * gg;
          sH1[cj][c] = og * tanh_acc(c1[u]);
        }
      }
      __syncthreads();
      // ---- layer 2 gates
#pragma unroll
      for (int k = 0; k < kHalfJobs; ++k) {
        const int jj = half * kHalfJobs + k;
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
      for (int k = 0; k < kHalfJobs; ++k) sG[half * kHalfJobs + k][g] = z[k];
      __syncthreads();
      if (i0 + i < sL[cj]) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int c = cc + u;
          const float ig = sigmoidf_acc(sG[cj][c]), fg = sigmoidf_acc(sG[cj][kLstm + c]);
          const float gg = tanh_acc(sG[cj][2 * kLstm + c]), og = sigmoidf_acc(sG[cj][3 * kLstm + c]);
          c2[u] = fg * c2[u] + ig * gg;
          sH2[cj][c] = og * tanh_acc(c2[u]);
        }
      }
      __syncthreads();
    }
  }
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
  if (p.x_out)
    for (int e = tid; e < nj * kXDim; e += kEncThreads)
      p.x_out[(size_t)(j0 + e / kXDim) * kXDim + e % kXDim] = sX[e / kXDim][e % kXDim];
  if (tid < nj) {
    const int j = j0 + tid, n = sN[tid];
    if (p.beta_out) {
      float acc = 0.f;
      for (int w = 0; w < n; ++w) acc += P[p.off.b_o + w];
      p.beta_out[(size_t)j * p.jv] = acc / static_cast<float>(n);
    }
    if (p.keys) p.keys[j] = 0ull;
    if (p.cur_keys) p.cur_keys[j] = 0ull;
  }
}

// K1b: per-job projections for K2, 32 jobs per CTA, one output column per thread per pass:
//   a[j][c]    = b1[c] + sum_i W1[c][i] x[j][i]            (job half of layer 1)
//   what[j][c] = sum_{w < n_j} W_o[w][c] / n_j             (worker-mean fold of the output layer)
constexpr int kProjJobs = 32;
constexpr int kProjThreads = 256;

__global__ void __launch_bounds__(kProjThreads) project_kernel(const __grid_constant__ EncodeParams p) {
  __shared__ __align__(16) float sXt[kXDim][kProjJobs];    // transposed: 4 jobs per LDS.128
  __shared__ __align__(16) float sM[kNMax][kProjJobs];     // mask / n
  const int j0 = blockIdx.x * kProjJobs, tid = threadIdx.x;
  const float* P = p.params;
  for (int e = tid; e < kXDim * kProjJobs; e += kProjThreads) {
    const int jj = e / kXDim, i = e % kXDim;
    sXt[i][jj] = (j0 + jj < p.J) ? p.x_out[(size_t)(j0 + jj) * kXDim + i] : 0.f;
  }
  for (int e = tid; e < kNMax * kProjJobs; e += kProjThreads) {
    const int w = e / kProjJobs, jj = e % kProjJobs;
    const int nj = (j0 + jj < p.J) ? p.n[j0 + jj] : 1;
    sM[w][jj] = w < nj ? 1.0f / static_cast<float>(nj) : 0.f;
  }
  __syncthreads();
  const int H = p.H;
  const int jn = min(kProjJobs, p.J - j0);
  for (int col = tid; col < H; col += kProjThreads) {
    float acc[kProjJobs];
#pragma unroll
    for (int jj = 0; jj < kProjJobs; ++jj) acc[jj] = 0.f;
    const float* wrow = P + p.off.W[1] + (size_t)col * kZDim;
    for (int i = 0; i < kXDim; ++i) {
      const float w = wrow[i];
      const float4* xv = reinterpret_cast<const float4*>(sXt[i]);
#pragma unroll
      for (int q = 0; q < kProjJobs / 4; ++q) {
        const float4 v = xv[q];
        acc[4 * q] = fmaf(w, v.x, acc[4 * q]); acc[4 * q + 1] = fmaf(w, v.y, acc[4 * q + 1]);
        acc[4 * q + 2] = fmaf(w, v.z, acc[4 * q + 2]); acc[4 * q + 3] = fmaf(w, v.w, acc[4 * q + 3]);
      }
    }
    const float b1 = P[p.off.b[1] + col];
#pragma unroll
    for (int jj = 0; jj < kProjJobs; ++jj)
      if (jj < jn) p.a_out[(size_t)(j0 + jj) * p.jv + col] = acc[jj] + b1;
#pragma unroll
    for (int jj = 0; jj < kProjJobs; ++jj) acc[jj] = 0.f;
    for (int w = 0; w < kNMax; ++w) {
      const float wo = P[p.off.W_o + (size_t)w * H + col];
      const float4* mv = reinterpret_cast<const float4*>(sM[w]);
#pragma unroll
      for (int q = 0; q < kProjJobs / 4; ++q) {
        const float4 v = mv[q];
        acc[4 * q] = fmaf(wo, v.x, acc[4 * q]); acc[4 * q + 1] = fmaf(wo, v.y, acc[4 * q + 1]);
        acc[4 * q + 2] = fmaf(wo, v.z, acc[4 * q + 2]); acc[4 * q + 3] = fmaf(wo, v.w, acc[4 * q + 3]);
      }
    }
#pragma unroll
    for (int jj = 0; jj < kProjJobs; ++jj)
      if (jj < jn) p.what_out[(size_t)(j0 + jj) * p.jv + col] = acc[jj];
  }
}

// K1 = K1a (+ K1b when the projections are requested; they need x, so x_out must be set).
cudaError_t launch_encode(const EncodeParams& p, cudaStream_t s) {
  if (p.J <= 0) return cudaSuccess;
  encode_kernel<<<(p.J + kEncJobs - 1) / kEncJobs, kEncThreads, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !p.a_out) return e;
  project_kernel<<<(p.J + kProjJobs - 1) / kProjJobs, kProjThreads, 0, s>>>(p);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- K0: candidate encodings
// u_c = ((log2 S_p - 21) / 8, (S_c - 8.5) / 8) for c = p*Q + q in [shard_begin, shard_end)
// (R#8), computed in double and rounded once to fp32.
__global__ void encode_grid_kernel(int Q, long long c0, long long n, const long long* __restrict__ S_p,
                                   const float* __restrict__ S_c, float2* __restrict__ u) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long c = c0 + i;
    const long long pi = c / Q, qi = c % Q;
    u[i] = make_float2(static_cast<float>((log2(static_cast<double>(S_p[pi])) - 21.0) / 8.0),
                       static_cast<float>((static_cast<double>(S_c[qi]) - 8.5) / 8.0));
  }
}

cudaError_t launch_encode_grid(const autobyte_grid& g, float2* u, cudaStream_t s) {
  const long long n = g.shard_end - g.shard_begin;
  const long long blocks = (n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096;
  encode_grid_kernel<<<static_cast<int>(blocks), 256, 0, s>>>(
      g.Q, g.shard_begin, n, reinterpret_cast<const long long*>(g.partition_bytes), g.credit_mult, u);
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

}  // namespace ab
