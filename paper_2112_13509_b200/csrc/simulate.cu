// simulate.cu — K10: GPU-batched ByteScheduler iteration evaluator: the time of
// one training iteration of job j under candidate <S_p, S_c>, for every (job, candidate) pair of a
// grid shard, one thread each — the "ground truth" a grid search over the candidates would measure
// (PAPER.md:534), under the mechanism of PAPER.md:213-255 and the readings R#24-R#26:
//   backward back-to-front (layer i ready at sum_{j >= i} Tb[j]); tensors cut into ceil(size / S_p)
//   chunks; the sender commits the next chunk of the front-most ready layer (priority) while
//   committed-but-unacknowledged bytes stay within S_c * S_p (credit) and at most 64 chunks;
//   the link sends committed chunks in commit order, s * factor / bw + delta each, acknowledged alpha
//   later; the next forward runs front-to-back, layer i once its tensor is acknowledged.
// The per-thread event loop is the oracle's (oracle/bytescheduler.py) with two equivalent
// reorganisations: the next layer to send is tracked with a pointer instead of a scan (a newly ready
// layer is always the front-most one, so it preempts; after a layer completes, every ready layer in
// front of it is complete, so the next one is found by scanning backwards from it), and the forward
// pass is the max-plus form max_i(delivered_i + sum_{k >= i} Tf_k) accumulated as layers complete
// (equal to the sequential recurrence up to rounding order). Double precision throughout; explicit
// __d*_rn intrinsics keep the compiler from contracting into FMAs (the oracle rounds every op).
// Block = 64 candidates of one job; per-thread chunk counters and the in-flight FIFO live in
// shared memory (column per thread).
#include "internal.h"
#include "ptx.cuh"

namespace ab {

constexpr int kSimThreads = 64;
constexpr int kSimMaxInflight = 64;   // R#24 (oracle MAX_INFLIGHT)

struct SimKernelParams {
  int J, l_max, P, Q;
  long long c_begin, c_end;
  const float* T; const float* B_d; const float* B_u;
  const int32_t* n; const int32_t* l; const int32_t* arc;
  const float* layer_bytes;   // [J][l_max]
  const float* fwd_ms;        // [J][l_max] or null (then Tb / 2)
  const long long* S_p; const float* S_c;
  double alpha_s, delta_s;
  double* iter_ms;            // [J][c_end - c_begin]
};

__global__ void __launch_bounds__(kSimThreads) simulate_kernel(const __grid_constant__ SimKernelParams p) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int j = blockIdx.y, tid = threadIdx.x;
  const int L = p.l[j], nw = p.n[j], arc = p.arc[j];
  double* sReady = reinterpret_cast<double*>(smraw);       // [L] ready time of layer i (s)
  double* sSufTf = sReady + p.l_max;                        // [L] sum_{k >= i} Tf[k] (s)
  double* sSize = sSufTf + p.l_max;                         // [L] bytes
  double* sDone = sSize + p.l_max;                          // [kSimMaxInflight][threads] in-flight ack times
  double* sBytes = sDone + kSimMaxInflight * kSimThreads;   // [kSimMaxInflight][threads] in-flight bytes
  int* sSent = reinterpret_cast<int*>(sBytes + kSimMaxInflight * kSimThreads);       // [l_max][threads] chunks sent
  __shared__ double sBw, sFactor;
  // ---- per-job inputs (R#26): slowest worker's backward time, forward time, bottleneck bandwidth
  if (tid == 0) {
    double bw = 0.0;
    for (int w = 0; w < nw; ++w) {
      const double bd = p.B_d[(size_t)j * kNMax + w], bu = p.B_u[(size_t)j * kNMax + w];
      const double m = bd < bu ? bd : bu;
      bw = (w == 0 || m < bw) ? m : bw;
    }
    sBw = __dmul_rn(bw, 1e9) / 8.0;
    sFactor = arc == 0 ? 2.0 : __ddiv_rn(__dmul_rn(2.0, static_cast<double>(nw - 1)), static_cast<double>(nw));
    // readiness back to front and the forward suffix sums, in the oracle's order
    double acc = 0.0, suf = 0.0;
    for (int i = L - 1; i >= 0; --i) {
      double tb = 0.0;
      for (int w = 0; w < nw; ++w) {
        const double v = p.T[((size_t)j * p.l_max + i) * kNMax + w];
        tb = (w == 0 || v > tb) ? v : tb;
      }
      const double tf = p.fwd_ms ? static_cast<double>(p.fwd_ms[(size_t)j * p.l_max + i]) : __dmul_rn(0.5, tb);
      acc = __dadd_rn(acc, __ddiv_rn(tb, 1e3));
      sReady[i] = acc;
      suf = __dadd_rn(suf, __ddiv_rn(tf, 1e3));
      sSufTf[i] = suf;
      sSize[i] = static_cast<double>(p.layer_bytes[(size_t)j * p.l_max + i]);
    }
  }
  __syncthreads();
  const long long c = p.c_begin + (long long)blockIdx.x * kSimThreads + tid;
  if (c >= p.c_end) return;
  const double Sp = static_cast<double>(p.S_p[c / p.Q]);
  const double Sc = static_cast<double>(p.S_c[c % p.Q]);
  const double credit = __dmul_rn(Sc, Sp), bw = sBw, factor = sFactor;
  const double alpha = p.alpha_s, delta = p.delta_s;
  for (int i = 0; i < L; ++i) sSent[i * kSimThreads + tid] = 0;
  auto nch = [&](int i) -> int { return sSize[i] > 0.0 ? static_cast<int>(ceil(__ddiv_rn(sSize[i], Sp))) : 0; };
  double t = 0.0, link_free = 0.0, inflight = 0.0, M = 0.0;
  int head = 0, count = 0;
  int lo = L;      // ready layers are [lo, L)
  int cur = -1;    // front-most ready layer with chunks left (-1: none)
  int cur_n = 0;
  while (true) {
    // admit layers that became ready by t (each new one is the front-most: it preempts)
    while (lo > 0 && sReady[lo - 1] <= t) {
      --lo;
      const int k = nch(lo);
      if (k == 0) {
        const double v = __dadd_rn(sReady[lo], sSufTf[lo]);   // no bytes: delivered when ready
        M = v > M ? v : M;
      } else {
        cur = lo;
        cur_n = k;
      }
    }
    if (cur < 0) {
      if (lo == 0) break;       // every layer delivered
      t = sReady[lo - 1];       // nothing to send until the next layer is ready
      continue;
    }
    const int sent = sSent[cur * kSimThreads + tid];
    const double rem = __dsub_rn(sSize[cur], __dmul_rn(static_cast<double>(sent), Sp));
    const double s = Sp < rem ? Sp : rem;
    if (count > 0 && (__dadd_rn(inflight, s) > credit || count == kSimMaxInflight)) {   // credit: wait for the oldest ack
      const double d = sDone[head * kSimThreads + tid];
      t = t > d ? t : d;
      inflight = __dsub_rn(inflight, sBytes[head * kSimThreads + tid]);
      head = head + 1 == kSimMaxInflight ? 0 : head + 1;
      --count;
      continue;
    }
    // commit at t; FIFO link
    const double start = t > link_free ? t : link_free;
    link_free = __dadd_rn(__dadd_rn(start, __ddiv_rn(__dmul_rn(s, factor), bw)), delta);
    const double done = __dadd_rn(link_free, alpha);
    const int slot = (head + count) % kSimMaxInflight;
    sDone[slot * kSimThreads + tid] = done;
    sBytes[slot * kSimThreads + tid] = s;
    ++count;
    inflight = __dadd_rn(inflight, s);
    sSent[cur * kSimThreads + tid] = sent + 1;
    if (sent + 1 == cur_n) {
      const double v = __dadd_rn(done, sSufTf[cur]);   // the layer is delivered
      M = v > M ? v : M;
      // every ready layer in front of cur is complete: the next one is behind it
      int nx = -1, nn = 0;
      for (int i = cur + 1; i < L; ++i) {
        const int k = nch(i);
        if (k > 0 && sSent[i * kSimThreads + tid] < k) { nx = i; nn = k; break; }
      }
      cur = nx;
      cur_n = nn;
    }
  }
  p.iter_ms[(size_t)j * (p.c_end - p.c_begin) + (c - p.c_begin)] = __dmul_rn(M, 1e3);
}

size_t simulate_smem_bytes(int l_max) {
  return (size_t)3 * l_max * sizeof(double) + (size_t)kSimMaxInflight * kSimThreads * 2 * sizeof(double) +
         (size_t)l_max * kSimThreads * sizeof(int);
}

cudaError_t launch_simulate(const autobyte_job_stats& jobs, const float* layer_bytes, const float* fwd_ms,
                            const autobyte_grid& g, double alpha_ms, double delta_ms, double* iter_ms, cudaStream_t s) {
  SimKernelParams p{};
  p.J = jobs.J; p.l_max = jobs.l_max; p.P = g.P; p.Q = g.Q;
  p.c_begin = g.shard_begin; p.c_end = g.shard_end;
  p.T = jobs.T; p.B_d = jobs.B_down; p.B_u = jobs.B_up;
  p.n = jobs.n_workers; p.l = jobs.n_layers; p.arc = jobs.arch_type;
  p.layer_bytes = layer_bytes; p.fwd_ms = fwd_ms;
  p.S_p = reinterpret_cast<const long long*>(g.partition_bytes); p.S_c = g.credit_mult;
  p.alpha_s = alpha_ms / 1e3; p.delta_s = delta_ms / 1e3;
  p.iter_ms = iter_ms;
  const size_t smem = simulate_smem_bytes(jobs.l_max);
  cudaError_t e = cudaFuncSetAttribute(simulate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const long long cs = g.shard_end - g.shard_begin;
  dim3 grid(static_cast<unsigned>((cs + kSimThreads - 1) / kSimThreads), static_cast<unsigned>(jobs.J));
  simulate_kernel<<<grid, kSimThreads, smem, s>>>(p);
  return cudaGetLastError();
}

AB_STATUS_SETTER(set_status_simulate)   // device status word pointer of this unit (ptx.cuh)

}  // namespace ab
