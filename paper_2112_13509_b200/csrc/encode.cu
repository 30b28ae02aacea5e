// encode.cu — K1: per-job prologue of the scoring path.
//
// K1a, one 256-thread CTA per job:
//   t'_i[w] = log2(1 + T[i][w] / 1 ms) on valid workers (R#7, R#8); e_i = W_e t'_i + b_e (R#4)
//   two-layer LSTM over i = 0..l_j-1, gates i,f,g,o, h0 = c0 = 0 ("two-layer LSTM", R#5);
//     thread g owns gate row g of one layer with its weights held in registers
//   x_j = [h | log2 B_d | log2 B_u | n/16 | l/64 | E_m[m] | E_arc[arc]]   (Table 2)
//   beta_j = (1/n) sum_{w<n} b_o[w], and resets the job's arg-max keys.
// K1b, 32 jobs per CTA:
//   a_j = W1[:, :82] x_j + b1     (layer-1 projection of the job half of the concatenation)
//   w_j = (1/n) sum_{w<n} W_o[w]  (worker-mean fold of the output layer, R#3) This is SIMT work (~1.6 MFLOP per job, 0.03% of C4).
#include "internal.h"
#include "ptx.cuh"

namespace ab {

constexpr int kEncThreads = 256;   // threads 0..127: LSTM layer 1 gate rows; 128..255: layer 2
constexpr int kChunk = 64;         // layers whose embeddings are staged in shared memory at a time

__device__ __forceinline__ float sigmoidf_acc(float z) { return 1.0f / (1.0f + expf(-z)); }

// dot of a register-resident weight row with a shared-memory vector, 4 independent partial sums
template <int N>
__device__ __forceinline__ float dot_row(const float (&w)[N], const float* v) {
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
  for (int d = 0; d < N; d += 4) {
    a0 = fmaf(w[d], v[d], a0);
    a1 = fmaf(w[d + 1], v[d + 1], a1);
    a2 = fmaf(w[d + 2], v[d + 2], a2);
    a3 = fmaf(w[d + 3], v[d + 3], a3);
  }
  return (a0 + a1) + (a2 + a3);
}

// K1a: one CTA per job. The two LSTM layers run as a wavefront: in iteration i layer 1 takes
// step i while layer 2 takes step i-1 (both read h1 of step i-1 before it is overwritten).
__global__ void __launch_bounds__(kEncThreads) encode_kernel(const __grid_constant__ EncodeParams p) {
  __shared__ float sT[kChunk][kNMax];
  __shared__ float sE[kChunk][kEmbed];
  __shared__ float sG1[4 * kLstm], sG2[4 * kLstm];
  __shared__ float sH1[kLstm], sH2[kLstm];
  __shared__ float sX[kXDim + 2];
  const int j = blockIdx.x, tid = threadIdx.x;
  const int n = p.n[j], l = p.l[j], m = p.m[j], arc = p.arc[j];
  const float* P = p.params;
  const bool layer1 = tid < 4 * kLstm;
  const int row = layer1 ? tid : tid - 4 * kLstm;

  float wx[kLstm], wh[kLstm];   // layer 1 uses wx[0..15] only
  if (layer1) {
#pragma unroll
    for (int d = 0; d < kEmbed; ++d) wx[d] = P[p.off.l1Wx + row * kEmbed + d];
#pragma unroll
    for (int d = kEmbed; d < kLstm; ++d) wx[d] = 0.f;
#pragma unroll
    for (int d = 0; d < kLstm; ++d) wh[d] = P[p.off.l1Wh + row * kLstm + d];
  } else {
#pragma unroll
    for (int d = 0; d < kLstm; ++d) {
      wx[d] = P[p.off.l2Wx + row * kLstm + d];
      wh[d] = P[p.off.l2Wh + row * kLstm + d];
    }
  }
  const float bias = layer1 ? P[p.off.l1b + row] : P[p.off.l2b + row];
  float c = 0.f;  // cell state: threads 0..31 (layer 1) and 128..159 (layer 2)
  if (tid < kLstm) { sH1[tid] = 0.f; sH2[tid] = 0.f; }

  const float* T = p.T + (size_t)j * p.l_max * kNMax;
  for (int i0 = 0; i0 <= l; i0 += kChunk) {
    const int len = min(kChunk, l - i0);
    __syncthreads();
    for (int e = tid; e < len * kNMax; e += kEncThreads) {
      const int i = e / kNMax, w = e % kNMax;
      sT[i][w] = (w < n) ? log2f(1.0f + T[(size_t)(i0 + i) * kNMax + w]) : 0.f;
    }
    __syncthreads();
    for (int e = tid; e < len * kEmbed; e += kEncThreads) {
      const int i = e / kEmbed, d = e % kEmbed;
      float acc = P[p.off.b_e + d];
#pragma unroll
      for (int w = 0; w < kNMax; ++w) acc = fmaf(P[p.off.W_e + d * kNMax + w], sT[i][w], acc);
      sE[i][d] = acc;
    }
    __syncthreads();
    const int iend = min(i0 + kChunk, l + 1);   // the wavefront runs one extra iteration
    for (int i = i0; i < iend; ++i) {
      if (layer1) {
        if (i < l) {
          float z = bias;
          float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
          const float* e = sE[i - i0];
#pragma unroll
          for (int d = 0; d < kEmbed; d += 4) {
            a0 = fmaf(wx[d], e[d], a0); a1 = fmaf(wx[d + 1], e[d + 1], a1);
            a2 = fmaf(wx[d + 2], e[d + 2], a2); a3 = fmaf(wx[d + 3], e[d + 3], a3);
          }
          z += ((a0 + a1) + (a2 + a3)) + dot_row<kLstm>(wh, sH1);
          sG1[row] = z;
        }
      } else if (i >= 1) {
        sG2[row] = bias + dot_row<kLstm>(wx, sH1) + dot_row<kLstm>(wh, sH2);
      }
      __syncthreads();
      if (tid < kLstm && i < l) {
        const float ig = sigmoidf_acc(sG1[tid]), fg = sigmoidf_acc(sG1[kLstm + tid]);
        const float gg = tanhf(sG1[2 * kLstm + tid]), og = sigmoidf_acc(sG1[3 * kLstm + tid]);
        c = fg * c + ig * gg;
        sH1[tid] = og * tanhf(c);
      } else if (tid >= 4 * kLstm && tid < 5 * kLstm && i >= 1) {
        const int t = tid - 4 * kLstm;
        const float ig = sigmoidf_acc(sG2[t]), fg = sigmoidf_acc(sG2[kLstm + t]);
        const float gg = tanhf(sG2[2 * kLstm + t]), og = sigmoidf_acc(sG2[3 * kLstm + t]);
        c = fg * c + ig * gg;
        sH2[t] = og * tanhf(c);
      }
      __syncthreads();
    }
  }
  // feature vector x_j
  if (tid < kLstm) sX[tid] = sH2[tid];
  if (tid < kNMax) {
    sX[kLstm + tid] = tid < n ? log2f(p.B_d[(size_t)j * kNMax + tid]) : 0.f;
    sX[kLstm + kNMax + tid] = tid < n ? log2f(p.B_u[(size_t)j * kNMax + tid]) : 0.f;
  }
  if (tid == 0) {
    sX[kLstm + 2 * kNMax] = static_cast<float>(n) / 16.0f;
    sX[kLstm + 2 * kNMax + 1] = static_cast<float>(l) / 64.0f;
  }
  if (tid < kTypeEmbed) {
    sX[kLstm + 2 * kNMax + 2 + tid] = P[p.off.E_m + m * kTypeEmbed + tid];
    sX[kLstm + 2 * kNMax + 2 + kTypeEmbed + tid] = P[p.off.E_arc + arc * kTypeEmbed + tid];
  }
  __syncthreads();
  if (p.x_out)
    for (int i = tid; i < kXDim; i += kEncThreads) p.x_out[(size_t)j * kXDim + i] = sX[i];
  if (tid == 0) {
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
  encode_kernel<<<p.J, kEncThreads, 0, s>>>(p);
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
