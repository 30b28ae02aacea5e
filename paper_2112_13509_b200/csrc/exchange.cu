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
//   3. wait: thread 0 of each block spins (ld.acquire.sys) until flags[r] >= e for all r; a wait
//      longer than AUTOBYTE_PEER_TIMEOUT_S records an error in the status word (no trap, ptx.cuh);
//   4. reduce: per job, the max over the G slots -> best index / score / current score (as K5).
// The epoch is a device counter advanced by the kernel itself (so CUDA-graph replays stay correct);
// windows, flags and counters are zeroed whenever a window is set up, so all ranks start at 0.
// Epochs only grow, so flags never need resetting. Two parities suffice: a rank can only store
// epoch e+2 into parity p after passing the epoch e+1 wait, which needs this rank's epoch e+1
// flag, which this rank raises only after its epoch e kernel (and its reads of parity p) ended.
// Max is order-free, so the result is the same bits as the all-gather path and as one GPU.
// All blocks must be resident at once (they wait on each other): cooperative launch.
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

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spin until *flag >= epoch. Returns false (after recording `code` in the status word, ptx.cuh) when
// timeout_ns > 0 elapses first, or at once when another wait already gave up: a dead or stalled peer
// becomes an AB_E_NCCL return on the host instead of a trapped (unusable) CUDA context.
__device__ bool wait_flag(const unsigned long long* flag, unsigned long long epoch, unsigned long long timeout_ns,
                          int code, int peer) {
  const unsigned long long t0 = global_ns();
#pragma unroll 1
  for (uint32_t i = 1; ld_acquire_sys(flag) < epoch; ++i) {
    if ((i & 255u) != 0) continue;
    const unsigned long long dt = global_ns() - t0;
    if (dt > 10000000ull && ab_aborted()) return false;   // status word only after 10 ms of waiting
    if (timeout_ns != 0 && dt > timeout_ns) {
      ab_raise(code, peer);
      return false;
    }
  }
  return true;
}

__global__ void __launch_bounds__(256) peer_exchange_kernel(const __grid_constant__ PeerExchangeParams p) {
  const int tid = threadIdx.x;
  __shared__ int s_ok;
  const long long n2 = 2LL * p.J;
  // the call's epoch lives in device memory and advances here, so a captured-and-replayed call (CUDA
  // graph) still gets a fresh epoch every time. Every block reads it before it counts itself done
  // below, and only the last block to do so writes the new value.
  const unsigned long long epoch = *reinterpret_cast<const volatile unsigned long long*>(p.epoch) + 1ull;
  const int par = static_cast<int>(epoch & 1ull);
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
      *p.epoch = epoch;  // every block has read the old value (it counted itself in after that)
      __threadfence_system();
#pragma unroll 1
      for (int r = 0; r < p.G; ++r) st_release_sys(p.win[r] + p.rank, epoch);
    }
    // 3. wait for every rank's keys of this epoch in the own window
    const unsigned long long* flags = p.win[p.rank];
    int ok = 1;
#pragma unroll 1
    for (int r = 0; r < p.G && ok; ++r) ok = wait_flag(flags + r, epoch, p.timeout_ns, kStatusPeerKeys, r);
    __threadfence();
    s_ok = ok;
  }
  __syncthreads();
  const bool ok = s_ok != 0;
  // 4. per-job max over the G slots (max is order-free: identical to one GPU and to the all-gather);
  // after a timeout the outputs are marked invalid (-1 / NaN) and the host reports AB_E_NCCL
  const unsigned long long* data = p.win[p.rank] + kPeerFlagWords + (long long)par * p.G * p.cap2;
  for (int j = blockIdx.x * blockDim.x + tid; j < p.J; j += gridDim.x * blockDim.x) {
    unsigned long long k = 0ull, ck = 0ull;
#pragma unroll 1
    for (int r = 0; r < p.G && ok; ++r) {
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
__global__ void peer_wait_kernel(const unsigned long long* flags, int G, unsigned long long epoch,
                                 unsigned long long timeout_ns) {
  if (threadIdx.x >= G) return;
  wait_flag(flags + threadIdx.x, epoch, timeout_ns, kStatusPeerX, threadIdx.x);
  __threadfence();
}

cudaError_t launch_peer_wait(const unsigned long long* flags, int G, unsigned long long epoch,
                             unsigned long long timeout_ns, cudaStream_t s) {
  peer_wait_kernel<<<1, 32, 0, s>>>(flags, G, epoch, timeout_ns);
  return cudaGetLastError();
}

// Every block waits for the others' pushes, so all blocks must be resident at once: a cooperative
// launch guarantees that (it is scheduled only when the whole grid fits, even next to other work on
// the GPU), and the grid is capped at the occupancy-derived co-resident maximum.
cudaError_t launch_peer_exchange(const PeerExchangeParams& p, int num_sms, cudaStream_t s, bool cooperative) {
  if (!cooperative) {   // test loopback (several virtual ranks on one device): one block per rank
    peer_exchange_kernel<<<1, 256, 0, s>>>(p);
    return cudaGetLastError();
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, peer_exchange_kernel, 256, 0);
  if (e != cudaSuccess) return e;
  const long long n2 = 2LL * p.J;
  long long nb = (n2 + 255) / 256;
  const long long cap = (long long)num_sms * (per_sm > 0 ? per_sm : 1);
  if (nb > cap) nb = cap;
  if (nb > num_sms) nb = num_sms;
  if (nb < 1) nb = 1;
  void* args[] = {const_cast<PeerExchangeParams*>(&p)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(peer_exchange_kernel), dim3(static_cast<unsigned>(nb)),
                                     dim3(256), args, 0, s);
}

AB_STATUS_SETTER(set_status_exchange)   // device status word pointer of this unit (ptx.cuh)

}  // namespace ab
