// encode.cu — K1: per-job prologue of the scoring path.
//
// For every job j (one 128-thread CTA per job):
//   t'_i[w] = log2(1 + T[i][w] / 1 ms) on valid workers (R#7, R#8); e_i = W_e t'_i + b_e (R#4)
//   two-layer LSTM over i = 0..l_j-1, gates i,f,g,o, h0 = c0 = 0 ("two-layer LSTM", R#5);
//     thread g owns gate row g of both layers with its weights held in registers
//   x_j = [h | log2 B_d | log2 B_u | n/16 | l/64 | E_m[m] | E_arc[arc]]   (Table 2)
//   a_j = W1[:, :82] x_j + b1     (layer-1 projection of the job half of the concatenation)
//   w_j = (1/n) sum_{w<n} W_o[w],  beta_j = (1/n) sum_{w<n} b_o[w]   (worker-mean fold, R#3)
// and resets the job's arg-max keys. This is SIMT work (~1.6 MFLOP per job, 0.03% of C4).
#include "internal.h"
#include "ptx.cuh"

namespace ab {

constexpr int kEncThreads = 128;
constexpr int kChunk = 64;   // layers whose embeddings are staged in shared memory at a time

__device__ __forceinline__ float sigmoidf_acc(float z) { return 1.0f / (1.0f + expf(-z)); }

__global__ void __launch_bounds__(kEncThreads) encode_kernel(const __grid_constant__ EncodeParams p) {
  __shared__ float sT[kChunk][kNMax];
  __shared__ float sE[kChunk][kEmbed];
  __shared__ float sGate[4 * kLstm];
  __shared__ float sH1[kLstm], sH2[kLstm];
  __shared__ float sX[kXDim + 2];
  const int j = blockIdx.x, tid = threadIdx.x;
  const int n = p.n[j], l = p.l[j], m = p.m[j], arc = p.arc[j];
  const float* P = p.params;

  // gate row `tid` of both LSTM layers, in registers
  float wx1[kEmbed], wh1[kLstm], wx2[kLstm], wh2[kLstm];
#pragma unroll
  for (int d = 0; d < kEmbed; ++d) wx1[d] = P[p.off.l1Wx + tid * kEmbed + d];
#pragma unroll
  for (int d = 0; d < kLstm; ++d) {
    wh1[d] = P[p.off.l1Wh + tid * kLstm + d];
    wx2[d] = P[p.off.l2Wx + tid * kLstm + d];
    wh2[d] = P[p.off.l2Wh + tid * kLstm + d];
  }
  const float bb1 = P[p.off.l1b + tid], bb2 = P[p.off.l2b + tid];
  float c1 = 0.f, c2 = 0.f;  // cell state, owned by threads 0..31
  if (tid < kLstm) { sH1[tid] = 0.f; sH2[tid] = 0.f; }

  const float* T = p.T + (size_t)j * p.l_max * kNMax;
  for (int i0 = 0; i0 < l; i0 += kChunk) {
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
    for (int i = 0; i < len; ++i) {
      // layer 1
      float z = bb1;
#pragma unroll
      for (int d = 0; d < kEmbed; ++d) z = fmaf(wx1[d], sE[i][d], z);
#pragma unroll
      for (int d = 0; d < kLstm; ++d) z = fmaf(wh1[d], sH1[d], z);
      sGate[tid] = z;
      __syncthreads();
      if (tid < kLstm) {
        const float ig = sigmoidf_acc(sGate[tid]), fg = sigmoidf_acc(sGate[kLstm + tid]);
        const float gg = tanhf(sGate[2 * kLstm + tid]), og = sigmoidf_acc(sGate[3 * kLstm + tid]);
        c1 = fg * c1 + ig * gg;
        sH1[tid] = og * tanhf(c1);
      }
      __syncthreads();
      // layer 2
      z = bb2;
#pragma unroll
      for (int d = 0; d < kLstm; ++d) z = fmaf(wx2[d], sH1[d], z);
#pragma unroll
      for (int d = 0; d < kLstm; ++d) z = fmaf(wh2[d], sH2[d], z);
      sGate[tid] = z;
      __syncthreads();
      if (tid < kLstm) {
        const float ig = sigmoidf_acc(sGate[tid]), fg = sigmoidf_acc(sGate[kLstm + tid]);
        const float gg = tanhf(sGate[2 * kLstm + tid]), og = sigmoidf_acc(sGate[3 * kLstm + tid]);
        c2 = fg * c2 + ig * gg;
        sH2[tid] = og * tanhf(c2);
      }
      __syncthreads();
    }
  }
  __syncthreads();
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

  const int H = p.H;
  if (p.a_out) {
    // a_j[k] = b1[k] + sum_i W1[k][i] x[i]: one warp per row, lanes over i (coalesced rows)
    const int warp = tid >> 5, lane = tid & 31;
    const float* W1 = P + p.off.W[1];
    for (int k = warp; k < H; k += kEncThreads / 32) {
      float acc = 0.f;
      for (int i = lane; i < kXDim; i += 32) acc = fmaf(W1[(size_t)k * kZDim + i], sX[i], acc);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) p.a_out[(size_t)j * H + k] = acc + P[p.off.b[1] + k];
    }
  }
  if (p.what_out) {
    const float inv_n = 1.0f / static_cast<float>(n);
    for (int k = tid; k < H; k += kEncThreads) {
      float acc = 0.f;
      for (int w = 0; w < n; ++w) acc += P[p.off.W_o + (size_t)w * H + k];
      p.what_out[(size_t)j * H + k] = acc * inv_n;
    }
  }
  if (tid == 0) {
    if (p.beta_out) {
      float acc = 0.f;
      for (int w = 0; w < n; ++w) acc += P[p.off.b_o + w];
      p.beta_out[j] = acc / static_cast<float>(n);
    }
    if (p.keys) p.keys[j] = 0ull;
    if (p.cur_keys) p.cur_keys[j] = 0ull;
  }
}

cudaError_t launch_encode(const EncodeParams& p, cudaStream_t s) {
  if (p.J <= 0) return cudaSuccess;
  encode_kernel<<<p.J, kEncThreads, 0, s>>>(p);
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
