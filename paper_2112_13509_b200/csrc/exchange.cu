// exchange.cu — K3+K5 fused: the cross-GPU arg-max exchange over NVLink peer memory (§8(a) a-7,
// §8(e)), one kernel per call instead of an NCCL all-gather followed by K5.
//
// Every rank owns a "window" in device memory that all ranks of the communicator map through CUDA
// IPC (autobyte.cu setup_peer_window):
//   flags [64] u64              flags[r] = last epoch whose keys rank r has finished storing here
//   data  [2][G][2*cap] u64     parity p = epoch & 1, slot r = rank r's 2J keys (best, then current)
// One call (epoch e, parity p):
//   1. push: every block stores its share of this rank's 2J keys into slot [p][rank] of EVERY
//      rank's window (NVLink P2P stores; the own window included), then __threadfence_system;
//   2. signal: the last block to finish pushing (a per-rank counter) releases flags[rank] = e in
//      every window (st.release.sys);
//   3. wait: thread 0 of each block spins (ld.acquire.sys, watchdog) until flags[r] >= e for all r;
//   4. reduce: per job, the max over the G slots -> best index / score / current score (as K5).
// Epochs only grow, so flags never need resetting. Two parities suffice: a rank can only store
// epoch e+2 into parity p after passing the epoch e+1 wait, which needs this rank's epoch e+1
// flag, which this rank raises only after its epoch e kernel (and its reads of parity p) ended.
// Max is order-free, so the result is the same bits as the all-gather path and as one GPU.
// All blocks must be resident at once (they wait on each other): the grid is capped at the SM count.
#include "internal.h"
#include "ptx.cuh"

namespace ab {

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(256) peer_exchange_kernel(const __grid_constant__ PeerExchangeParams p) {
  const int tid = threadIdx.x;
  const long long n2 = 2LL * p.J;
  const int par = static_cast<int>(p.epoch & 1ull);
  // 1. push this rank's keys into slot [par][rank] of every window
  for (long long e = blockIdx.x * (long long)blockDim.x + tid; e < n2; e += (long long)gridDim.x * blockDim.x) {
    const unsigned long long v = p.keys[e];
#pragma unroll 1
    for (int r = 0; r < p.G; ++r) p.win[r][kPeerFlagWords + ((long long)par * p.G + p.rank) * p.cap2 + e] = v;
  }
  __threadfence_system();
  __syncthreads();
  // 2. the last block to finish pushing raises this rank's flag in every window
  if (tid == 0) {
    const unsigned int done = atomicAdd(p.counter, 1u);
    if (done == gridDim.x - 1) {
      *p.counter = 0u;   // next call (stream-ordered after this kernel) counts from zero again
      __threadfence_system();
#pragma unroll 1
      for (int r = 0; r < p.G; ++r) st_release_sys(p.win[r] + p.rank, p.epoch);
    }
    // 3. wait for every rank's keys of this epoch in the own window
    const unsigned long long* flags = p.win[p.rank];
    const long long t0 = clock64();
#pragma unroll 1
    for (int r = 0; r < p.G; ++r) {
      while (ld_acquire_sys(flags + r) < p.epoch) {
        if (clock64() - t0 > (1ll << 34)) {   // ~9 s: a peer never arrived
          printf("autobyte: peer exchange watchdog (rank %d waiting for rank %d, epoch %llu)\n", p.rank, r,
                 p.epoch);
          __trap();
        }
      }
    }
    __threadfence();
  }
  __syncthreads();
  // 4. per-job max over the G slots (max is order-free: identical to one GPU and to the all-gather)
  const unsigned long long* data = p.win[p.rank] + kPeerFlagWords + (long long)par * p.G * p.cap2;
  for (int j = blockIdx.x * blockDim.x + tid; j < p.J; j += gridDim.x * blockDim.x) {
    unsigned long long k = 0ull, ck = 0ull;
#pragma unroll 1
    for (int r = 0; r < p.G; ++r) {
      k = max(k, data[(long long)r * p.cap2 + j]);
      ck = max(ck, data[(long long)r * p.cap2 + p.J + j]);
    }
    if (k == 0ull) {
      p.best_idx[j] = -1;
      p.best_score[j] = __uint_as_float(0x7FC00000u);
    } else {
      p.best_idx[j] = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(k & 0xFFFFFFFFull));
      p.best_score[j] = unord32(static_cast<uint32_t>(k >> 32));
    }
    if (p.cur_score) p.cur_score[j] = ck ? unord32(static_cast<uint32_t>(ck >> 32)) : __uint_as_float(0x7FC00000u);
  }
}

// Consumers of the x all-gather (K1b, K4) run after this on the stream: the fused K1a epilogue
// (encode.cu) stores every rank's rows into this rank's window before raising its flag.
__global__ void peer_wait_kernel(const unsigned long long* flags, int G, unsigned long long epoch, int rank) {
  if (threadIdx.x >= G) return;
  const long long t0 = clock64();
  while (ld_acquire_sys(flags + threadIdx.x) < epoch) {
    if (clock64() - t0 > (1ll << 34)) {
      printf("autobyte: x all-gather watchdog (rank %d waiting for rank %d, epoch %llu)\n", rank, threadIdx.x, epoch);
      __trap();
    }
  }
  __threadfence();
}

cudaError_t launch_peer_wait(const unsigned long long* flags, int G, unsigned long long epoch, int rank,
                             cudaStream_t s) {
  peer_wait_kernel<<<1, 32, 0, s>>>(flags, G, epoch, rank);
  return cudaGetLastError();
}

cudaError_t launch_peer_exchange(const PeerExchangeParams& p, int num_sms, cudaStream_t s) {
  const long long n2 = 2LL * p.J;
  long long nb = (n2 + 255) / 256;
  if (nb > num_sms) nb = num_sms;   // every block waits for the others: all must be resident
  if (nb < 1) nb = 1;
  peer_exchange_kernel<<<static_cast<int>(nb), 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace ab
