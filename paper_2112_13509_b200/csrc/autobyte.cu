// autobyte.cu — the C ABI (include/autobyte.h): argument checks, weight blob, device memory,
// stream ordering of the kernels K1 (encode), K2 (score/arg-max), K3 (NCCL exchange),
// K4 (adapt), K5 (finalize), and profiling.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/autobyte_testing.h"
#include "internal.h"

using namespace ab;

namespace {

constexpr uint32_t kBlobHeader = 48;

enum Kind { K_ENCODE = 0, K_SCORE, K_FINALIZE, K_EXCHANGE, K_ADAPT, K_PACK, K_OTHER, K_N };

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Memory debugging (AUTOBYTE_DEBUG_MEM=1 at create; the pool's compute-sanitizer is unavailable):
// every library allocation is poisoned with 0xFF bytes (NaN as fp32, ~0 as integers), so a kernel
// that reads workspace it never wrote produces NaN / garbage that the parity tests catch, and the
// 256-byte slack after the requested size holds a 0xA5 canary that autobyte_debug_mem_check reads
// back, so a write past the end of any workspace is counted.
bool g_debug_mem = false;
std::mutex g_canary_mu;
std::vector<std::pair<uint8_t*, size_t>> g_canaries;   // (tail address, owner device)
constexpr size_t kCanaryBytes = 256;

template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t want) {
    if (want <= n && ptr) return cudaSuccess;
    release();
    cudaError_t e = cudaMalloc(&ptr, want * sizeof(T) + kCanaryBytes);
    if (e != cudaSuccess) { ptr = nullptr; return e; }
    n = want;
    if (g_debug_mem) {
      uint8_t* tail = reinterpret_cast<uint8_t*>(ptr) + want * sizeof(T);
      if ((e = cudaMemset(ptr, 0xFF, want * sizeof(T))) != cudaSuccess) return e;
      if ((e = cudaMemset(tail, 0xA5, kCanaryBytes)) != cudaSuccess) return e;
      if ((e = cudaDeviceSynchronize()) != cudaSuccess) return e;   // before any stream uses it
      int dev = 0;
      cudaGetDevice(&dev);
      std::lock_guard<std::mutex> lock(g_canary_mu);
      g_canaries.push_back({tail, static_cast<size_t>(dev)});
    }
    return cudaSuccess;
  }
  void release() {
    if (ptr && g_debug_mem) {
      uint8_t* tail = reinterpret_cast<uint8_t*>(ptr) + n * sizeof(T);
      std::lock_guard<std::mutex> lock(g_canary_mu);
      for (auto it = g_canaries.begin(); it != g_canaries.end(); ++it)
        if (it->first == tail) { g_canaries.erase(it); break; }
    }
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    n = 0;
  }
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
};

}  // namespace

struct autobyte_ctx {
  autobyte_net_desc desc{};
  ParamOffsets off{};
  autobyte_precision precision = AB_PREC_BF16;
  int device = 0;
  int num_sms = 148;
  int cta_group = 2;             // K2 variant: CTA pairs or single CTAs (AUTOBYTE_CTA_GROUP=1|2)
  int planes = 1;                // 2 for the fp32-accuracy path (bf16 hi + lo weight planes)
  CUtensorMap wmap{};            // tensor map over wpack for the CTA-pair TMA
  CUtensorMap wcol[kMaxHidden + 1] = {};   // K4s column-slice maps over the fp32 masters
  cudaStream_t stream = nullptr;
  bool check = false;
  bool shard_encode = true;      // G > 1: K1a on 1/G of the jobs + all-gather of x (AUTOBYTE_SHARD_ENCODE=0 off)
  std::string last_error;

  DevBuf<float> params;          // fp32 masters (blob payload order)
  DevBuf<float> grads;           // same layout, head part used by adapt
  DevBuf<__nv_bfloat16> wpack;   // packed bf16 W_2..W_L for K2
  DevBuf<uint32_t> spill;        // K2 activation scratch of the fp32 path at H = 512
  DevBuf<unsigned int> barrier;  // grid barrier of K4 (2 words)
  DevBuf<int> flag;              // AUTOBYTE_CHECK device flag
  // per-call workspace
  DevBuf<float> jobvec, x, adapt_ws, loss_tmp;
  DevBuf<float> opt_m, opt_v;        // Adam moments (autobyte_train), blob layout
  DevBuf<float> topk_scores;         // [J][shard] score matrix of autobyte_topk
  DevBuf<float> enc_stash, enc_dz, enc_part;   // encoder fine-tuning: K1a stash, dX [B][84], K8 partials
  DevBuf<unsigned long long> topk_keys;   // [G][J][k] per-rank top-k keys
  long long opt_t = 0;               // Adam step count
  DevBuf<float> u;                   // [P + Q] candidate-grid axes u_p | u_c (K1b / K1s / K0)
  DevBuf<unsigned int> done;         // K2's CTA completion counter (K5 folded into K2 at G = 1)
  DevBuf<unsigned long long> keys;   // [2J]: best keys then current-config keys
  DevBuf<unsigned long long> keys_all;   // [G][2J]: every rank's keys (all-gather exchange)
  bool exchange_allreduce = false;   // AUTOBYTE_EXCHANGE=allreduce: ncclAllReduce(max) instead
  bool exchange_nccl = false;        // AUTOBYTE_EXCHANGE=nccl|allreduce: no peer-memory window
  // peer-memory exchange (exchange.cu): own window + IPC mappings of the other ranks' windows
  bool peer = false;
  DevBuf<unsigned long long> win;
  DevBuf<unsigned int> win_counter;
  DevBuf<unsigned long long> win_epoch;   // device counter of completed key exchanges (exchange.cu advances it)
  unsigned long long* peer_win[kMaxPeers] = {};
  long long win_cap2 = 0;            // slot stride in u64 (2 x job capacity)
  unsigned long long peer_timeout_ns = 0;   // AUTOBYTE_PEER_TIMEOUT_S (default 120 s; 0 = wait forever)
  // x all-gather through the same windows (K1a epilogue stores, encode.cu): [2 parities][xcap][82] fp32
  DevBuf<unsigned int> win_xcounter;
  long long win_xcap = 0;
  size_t win_xoff = 0;               // u64 word offset of the x region in a window
  unsigned long long xepoch = 0;
  bool peer_x = false;               // AUTOBYTE_PEER_X=1: x all-gather through the windows (opt-in)
  bool zero_copy = true;             // *_host: K1a reads page-locked T over PCIe (AUTOBYTE_ZERO_COPY=0 off)
  volatile int* status = nullptr;    // device status word of this device (ptx.cuh), mapped host memory
  // staging for the *_host entry points
  DevBuf<float> sT, sBd, sBu, sSc, sV, rScore, rCur;
  DevBuf<int32_t> sN, sL, sM, sArc, sCur, rIdx;
  DevBuf<long long> sSp;
  // multi-GPU
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  // profiling
  bool profiling = false;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  double ms[K_N] = {};
  long long launches[K_N] = {};
  double score_pairs = 0.0;
};

namespace {

autobyte_status fail(autobyte_ctx* c, autobyte_status s, const std::string& msg) {
  if (c) c->last_error = msg;
  return s;
}
autobyte_status cuda_fail(autobyte_ctx* c, cudaError_t e, const char* what) {
  return fail(c, AB_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// One status word per device (ptx.cuh "device status word"): [0] = code, [1] = detail (block or peer
// rank). Page-locked and mapped, so the host reads it without synchronising; every translation unit
// gets the device address once per device.
std::mutex g_status_mu;
int* g_status_host[64] = {};

cudaError_t device_status_word(int device, volatile int** out) {
  std::lock_guard<std::mutex> lock(g_status_mu);
  if (device < 0 || device >= 64) return cudaErrorInvalidDevice;
  if (!g_status_host[device]) {
    int* h = nullptr;
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&h), 64, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) return e;
    h[0] = h[1] = 0;
    int* d = nullptr;
    if ((e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&d), h, 0)) != cudaSuccess) return e;
    for (auto set : {set_status_adapt, set_status_encode, set_status_encoder_bwd, set_status_exchange,
                     set_status_score, set_status_topk, set_status_adapt_small, set_status_simulate})
      if ((e = set(d)) != cudaSuccess) return e;
    g_status_host[device] = h;
  }
  *out = g_status_host[device];
  return cudaSuccess;
}

// A watchdog fired in an earlier kernel of this device: report it once (and clear it). Results of
// the call whose kernel recorded it are invalid; the context and the CUDA context stay usable.
autobyte_status take_status(autobyte_ctx* c) {
  if (!c->status) return AB_OK;
  const int code = c->status[0];
  if (code == 0) return AB_OK;
  const int detail = c->status[1];
  c->status[1] = 0;
  c->status[0] = 0;
  if (code == kStatusPeerKeys || code == kStatusPeerX)
    return fail(c, AB_E_NCCL, std::string(code == kStatusPeerKeys ? "peer key exchange" : "peer x all-gather") +
                                  " timed out waiting for rank " + std::to_string(detail) +
                                  " (AUTOBYTE_PEER_TIMEOUT_S); the results of that call are invalid");
  // an aborted K4 may leave its grid-barrier counter off a multiple of its grid: zero it, stream-
  // ordered after the aborted launch and before any later one
  if (c->barrier.ptr) cudaMemsetAsync(c->barrier.ptr, 0, 2 * sizeof(unsigned int), c->stream);
  return fail(c, AB_E_CUDA, "kernel pipeline watchdog fired in block " + std::to_string(detail) +
                                " (an internal wait exceeded ~2^36 cycles); the results of that call are invalid");
}

#define AB_CUDA(ctx, expr)                                            \
  do {                                                                \
    cudaError_t _e = (expr);                                          \
    if (_e != cudaSuccess) return cuda_fail((ctx), _e, #expr);        \
  } while (0)

// NVTX ranges (header-only NVTX3; near free without a tool attached): one per entry point and one
// per kernel launch, named by kernel role, so an nsys / ncu timeline reads as the method's steps.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
const char* const kKindName[K_N] = {"K1 encode", "K2 score", "K5 finalize", "K3 exchange", "K4 adapt", "pack",
                                    "other"};

// Bracket one launch with profiling events (when enabled) and count it.
template <typename F>
cudaError_t timed(autobyte_ctx* c, int kind, F&& launch) {
  NvtxRange range(kKindName[kind]);
  cudaEvent_t a = nullptr, b = nullptr;
  if (c->profiling) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, c->stream);
  }
  cudaError_t e = launch();
  if (c->profiling) {
    cudaEventRecord(b, c->stream);
    c->pending.push_back({kind, {a, b}});
  }
  if (e == cudaSuccess) c->launches[kind] += 1;
  return e;
}

autobyte_status check_jobs_host(autobyte_ctx* c, const autobyte_job_stats* j) {
  if (!j) return fail(c, AB_E_INVALID, "job stats pointer is NULL");
  if (j->J < 1) return fail(c, AB_E_SHAPE, "J must be >= 1");
  if (j->l_max < 1) return fail(c, AB_E_SHAPE, "l_max must be >= 1");
  if (!j->T || !j->B_down || !j->B_up || !j->n_workers || !j->n_layers || !j->model_type || !j->arch_type)
    return fail(c, AB_E_INVALID, "job stats array pointer is NULL");
  if (reinterpret_cast<uintptr_t>(j->T) & 15u)   // K1a stages T rows with 16-byte cp.async
    return fail(c, AB_E_INVALID, "T must be 16-byte aligned");
  return AB_OK;
}

autobyte_status check_grid_host(autobyte_ctx* c, const autobyte_grid* g) {
  if (!g) return fail(c, AB_E_INVALID, "grid pointer is NULL");
  if (g->P < 1 || g->Q < 1) return fail(c, AB_E_SHAPE, "grid P and Q must be >= 1");
  const long long C = (long long)g->P * g->Q;
  // (K2 forms candidate indices of a whole 128-row tile past the shard end in 32 bits)
  if (C > 0x7FFFFFFFLL - kTileM) return fail(c, AB_E_SHAPE, "grid has more than 2^31-129 candidates");
  // with a communicator attached an empty shard is a valid part of a partition of [0, C) (C < world
  // gives some ranks nothing to score): that rank skips K0/K2 but still joins the collectives
  const bool multi = c && c->comm && c->world > 1;
  if (g->shard_begin < 0 || g->shard_end > C || g->shard_begin > g->shard_end ||
      (g->shard_begin == g->shard_end && !multi))
    return fail(c, AB_E_SHAPE, multi ? "shard must satisfy 0 <= begin <= end <= P*Q"
                                     : "shard must satisfy 0 <= begin < end <= P*Q");
  if (!g->partition_bytes || !g->credit_mult) return fail(c, AB_E_INVALID, "grid array pointer is NULL");
  return AB_OK;
}

autobyte_status device_checks(autobyte_ctx* c, const autobyte_job_stats* jobs, const autobyte_grid* grid) {
  if (!c->check) return AB_OK;
  AB_CUDA(c, c->flag.ensure(1));
  AB_CUDA(c, cudaMemsetAsync(c->flag.ptr, 0, sizeof(int), c->stream));
  if (jobs) AB_CUDA(c, timed(c, K_OTHER, [&] {
                      return launch_check(*jobs, c->desc.n_max, c->desc.n_model_types, c->desc.n_arch_types,
                                          c->flag.ptr, c->stream);
                    }));
  if (grid) AB_CUDA(c, timed(c, K_OTHER, [&] { return launch_check_grid(*grid, c->flag.ptr, c->stream); }));
  int h = 0;
  AB_CUDA(c, cudaMemcpyAsync(&h, c->flag.ptr, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  AB_CUDA(c, cudaStreamSynchronize(c->stream));
  if (h) return fail(c, AB_E_INVALID, h & 1 ? "job statistics out of range (AUTOBYTE_CHECK)" : "grid out of range (AUTOBYTE_CHECK)");
  return AB_OK;
}

autobyte_status ensure_job_ws(autobyte_ctx* c, int J) {
  const int H = c->desc.hidden_width;
  AB_CUDA(c, c->jobvec.ensure((size_t)J * (2 * H + 4)));
  AB_CUDA(c, c->keys.ensure((size_t)2 * J));
  return AB_OK;
}

EncodeParams encode_params(autobyte_ctx* c, const autobyte_job_stats* j) {
  EncodeParams p{};
  p.J = j->J; p.l_max = j->l_max; p.H = c->desc.hidden_width;
  p.T = j->T; p.B_d = j->B_down; p.B_u = j->B_up;
  p.n = j->n_workers; p.l = j->n_layers; p.m = j->model_type; p.arc = j->arch_type;
  p.params = c->params.ptr; p.off = c->off;
  return p;
}

// K1a into c->x for all jobs (returns the params K1b continues from). At G > 1 each rank encodes
// its 1/G slice of the jobs and the x rows are all-gathered in place over NCCL: K1a's per-job
// arithmetic does not depend on how jobs are grouped, so x (and every key after it) is
// bit-identical to the single-rank result.
// The jobs [*jb, *je) whose statistics this rank's K1a reads (all of them at G = 1).
bool encode_range(const autobyte_ctx* c, int J, int* jb, int* je) {
  const bool shard = c->shard_encode && c->comm && c->world > 1;
  const int G = shard ? c->world : 1;
  const int Jp = (J + G - 1) / G;
  *jb = shard ? std::min(J, c->rank * Jp) : 0;
  *je = shard ? std::min(J, (c->rank + 1) * Jp) : J;
  return shard;
}

// proj (nullable): K1b's outputs; when the unsharded call runs K1s, K1s computes them too and
// *projected is set (the caller then skips K1b).
autobyte_status run_lstm(autobyte_ctx* c, const autobyte_job_stats* jobs, EncodeParams* out,
                         const EncodeParams* proj = nullptr, bool* projected = nullptr) {
  if (projected) *projected = false;
  const int J = jobs->J;
  int jb = 0, je = J;
  const bool shard = encode_range(c, J, &jb, &je);
  const int G = shard ? c->world : 1;
  const int Jp = (J + G - 1) / G;
  AB_CUDA(c, c->x.ensure((size_t)Jp * G * kXDim));
  EncodeParams ep = encode_params(c, jobs);
  ep.x_out = c->x.ptr;
  ep.j_begin = jb;
  ep.j_end = je;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(c->stream, &cap) != cudaSuccess) { cudaGetLastError(); cap = cudaStreamCaptureStatusNone; }
  // the fused x gather takes its epoch from the host, so a captured call would replay a stale one:
  // while the stream is being captured the NCCL all-gather (graph-capturable) is used instead
  if (shard && c->peer && c->peer_x && J <= c->win_xcap && cap == cudaStreamCaptureStatusNone) {
    // x all-gather fused into K1a (opt-in, AUTOBYTE_PEER_X=1): its epilogue stores the rank's rows
    // into every window and raises an epoch flag; one warp then waits for all ranks' flags before
    // K1b / K4 read the own window. Measured at G = 4 it is ~1 % slower per step than the NCCL
    // all-gather (4.89 vs 4.84 ms: the system-scope fence after the remote stores sits at the end
    // of every K1a CTA, plus one more launch), so the NCCL path stays the default.
    const unsigned long long e = c->xepoch + 1;   // committed only once both launches succeeded
    for (int r = 0; r < G; ++r) {
      ep.xg[r] = reinterpret_cast<float*>(c->peer_win[r] + c->win_xoff) + (size_t)(e & 1ull) * c->win_xcap * kXDim;
      ep.xflag[r] = c->peer_win[r] + kPeerXFlags;
    }
    ep.xG = G; ep.xrank = c->rank; ep.xcounter = c->win_xcounter.ptr; ep.xepoch = e;
    ep.x_out = ep.xg[c->rank];
    AB_CUDA(c, timed(c, K_ENCODE, [&] { return launch_encode_lstm(ep, c->num_sms, c->stream); }));
    AB_CUDA(c, timed(c, K_OTHER, [&] {
              return launch_peer_wait(c->win.ptr + kPeerXFlags, G, e, c->peer_timeout_ns, c->stream);
            }));
    c->xepoch = e;
    ep.xG = 0;   // K1b and later launches with these params are not part of the gather
    *out = ep;
    return AB_OK;
  }
  if (ep.j_end > ep.j_begin) {
    EncodeParams lp = ep;
    if (proj && !shard) {   // one kernel for the whole job prologue when K1s runs (few jobs, one rank)
      lp.jv = proj->jv; lp.a_out = proj->a_out; lp.what_out = proj->what_out; lp.beta_out = proj->beta_out;
      lp.keys = proj->keys; lp.cur_keys = proj->cur_keys;
      lp.P = proj->P; lp.Q = proj->Q; lp.S_p = proj->S_p; lp.S_c = proj->S_c;
      lp.up_out = proj->up_out; lp.uc_out = proj->uc_out;
      lp.fuse_project = 1;
    }
    AB_CUDA(c, timed(c, K_ENCODE, [&] { return launch_encode_lstm(lp, c->num_sms, c->stream, projected); }));
  }
  if (shard) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (c->profiling) { cudaEventCreate(&a); cudaEventCreate(&b); cudaEventRecord(a, c->stream); }
    ncclResult_t r = ncclAllGather(c->x.ptr + (size_t)c->rank * Jp * kXDim, c->x.ptr, (size_t)Jp * kXDim, ncclFloat,
                                   c->comm, c->stream);
    if (c->profiling) { cudaEventRecord(b, c->stream); c->pending.push_back({K_EXCHANGE, {a, b}}); }
    if (r != ncclSuccess) return fail(c, AB_E_NCCL, std::string("ncclAllGather: ") + ncclGetErrorString(r));
    c->launches[K_EXCHANGE] += 1;
  }
  *out = ep;
  return AB_OK;
}

// Peer-memory window for the fused exchange (exchange.cu). Every rank allocates a window, its CUDA
// IPC handle is all-gathered over NCCL and the other ranks' windows are mapped; the ranks then agree
// (NCCL min) that every mapping succeeded, else all of them keep the NCCL all-gather path.
void close_peer_window(autobyte_ctx* c) {
  for (int r = 0; r < kMaxPeers; ++r) {
    if (c->peer_win[r] && r != c->rank) cudaIpcCloseMemHandle(c->peer_win[r]);
    c->peer_win[r] = nullptr;
  }
  c->win.release();
  c->win_counter.release();
  c->win_epoch.release();
  c->win_xcounter.release();
  c->peer = false;
  c->win_cap2 = 0;
  c->win_xcap = 0;
}

bool setup_peer_window(autobyte_ctx* c) {
  const int G = c->world;
  if (G < 2 || G > kMaxPeers || c->exchange_nccl) return false;
  const char* capenv = std::getenv("AUTOBYTE_PEER_JOBS");
  const long long cap_jobs = capenv ? std::atoll(capenv) : 65536;
  c->win_cap2 = 2 * (cap_jobs > 0 ? cap_jobs : 65536);
  c->win_xcap = c->win_cap2 / 2;
  c->win_xoff = kPeerFlagWords + 2 * (size_t)G * c->win_cap2;
  const size_t words = c->win_xoff + (size_t)c->win_xcap * kXDim;   // 2 parities x 82 fp32 = 82 words per job
  // every rank starts from zeroed flags, counters and epochs (a re-attached ctx included), so the
  // ranks' epoch sequences agree from the first exchange on
  c->xepoch = 0;
  int ok = c->win.ensure(words) == cudaSuccess && c->win_counter.ensure(1) == cudaSuccess &&
           c->win_xcounter.ensure(1) == cudaSuccess && c->win_epoch.ensure(1) == cudaSuccess &&
           cudaMemsetAsync(c->win.ptr, 0, words * 8, c->stream) == cudaSuccess &&
           cudaMemsetAsync(c->win_counter.ptr, 0, sizeof(unsigned int), c->stream) == cudaSuccess &&
           cudaMemsetAsync(c->win_epoch.ptr, 0, sizeof(unsigned long long), c->stream) == cudaSuccess &&
           cudaMemsetAsync(c->win_xcounter.ptr, 0, sizeof(unsigned int), c->stream) == cudaSuccess;
  cudaIpcMemHandle_t mine{};
  if (ok) ok = cudaIpcGetMemHandle(&mine, c->win.ptr) == cudaSuccess;
  DevBuf<uint8_t> hbuf;
  DevBuf<int> okbuf;
  std::vector<cudaIpcMemHandle_t> all(G);
  if (hbuf.ensure(sizeof(cudaIpcMemHandle_t) * G) != cudaSuccess || okbuf.ensure(1) != cudaSuccess) return false;
  cudaMemcpyAsync(hbuf.ptr + sizeof(cudaIpcMemHandle_t) * c->rank, &mine, sizeof(mine), cudaMemcpyHostToDevice, c->stream);
  if (ncclAllGather(hbuf.ptr + sizeof(cudaIpcMemHandle_t) * c->rank, hbuf.ptr, sizeof(cudaIpcMemHandle_t), ncclChar,
                    c->comm, c->stream) != ncclSuccess)
    return false;
  cudaMemcpyAsync(all.data(), hbuf.ptr, sizeof(cudaIpcMemHandle_t) * G, cudaMemcpyDeviceToHost, c->stream);
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return false;
  for (int r = 0; r < G && ok; ++r) {
    if (r == c->rank) { c->peer_win[r] = c->win.ptr; continue; }
    void* ptr = nullptr;
    ok = cudaIpcOpenMemHandle(&ptr, all[r], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
    c->peer_win[r] = static_cast<unsigned long long*>(ptr);
  }
  if (!ok) cudaGetLastError();   // clear a failed mapping's error before agreeing
  cudaMemcpyAsync(okbuf.ptr, &ok, sizeof(int), cudaMemcpyHostToDevice, c->stream);
  if (ncclAllReduce(okbuf.ptr, okbuf.ptr, 1, ncclInt, ncclMin, c->comm, c->stream) != ncclSuccess) return false;
  int all_ok = 0;
  cudaMemcpyAsync(&all_ok, okbuf.ptr, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return false;
  return all_ok == 1;
}

// Host staging of job statistics for the *_host entry points. Only this rank's K1a job range
// reads T, B_d, B_u, l, m and arc (every rank encodes 1/G of the jobs and all-gathers x), so only
// that slice crosses PCIe, copied to its global offset; n is read for every job (K1b's worker
// mean, K4's mask). With AUTOBYTE_CHECK=1 everything is copied (the range checks read all jobs).
// Arrays read by K1a alone (T -- three quarters of the bytes --, B_down, B_up, n_layers, model_type,
// arch_type) are not staged when they live in page-locked host memory: K1a reads its shard of them
// over PCIe itself (its cp.async chunk prefetch streams T from the mapped host buffer), so the
// transfer overlaps the LSTM steps and no copy is issued. n_workers (also read by K1b and K4) is
// always copied. *dj receives the pointers the kernels read. AUTOBYTE_ZERO_COPY=0 always stages.
// Device address of a page-locked host buffer (zero-copy), or nullptr (pageable: must be copied).
const void* host_in_place(const autobyte_ctx* c, const void* h) {
  cudaPointerAttributes pa{};
  if (c->zero_copy && !c->check && cudaPointerGetAttributes(&pa, h) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
      pa.devicePointer)
    return pa.devicePointer;
  cudaGetLastError();   // (pageable memory: clear the query's error)
  return nullptr;
}

cudaError_t stage_jobs_host(autobyte_ctx* c, const autobyte_job_stats* jobs, autobyte_job_stats* dj) {
  const int J = jobs->J;
  int jb = 0, je = J;
  encode_range(c, J, &jb, &je);
  if (c->check) { jb = 0; je = J; }
  const size_t nj = (size_t)(je - jb), lt = (size_t)jobs->l_max * kNMax;
  cudaError_t e = cudaSuccess;
  // in place if page-locked, else copy the rank's slice [jb, je) (row width w elements of size es)
  auto place = [&](const void* h, void* staging, size_t w, size_t es) -> const void* {
    if (const void* d = host_in_place(c, h)) return d;
    const size_t off = (size_t)jb * w * es, bytes = nj * w * es;
    if (bytes && e == cudaSuccess)
      e = cudaMemcpyAsync(static_cast<uint8_t*>(staging) + off, static_cast<const uint8_t*>(h) + off, bytes,
                          cudaMemcpyHostToDevice, c->stream);
    return staging;
  };
  *dj = *jobs;
  dj->T = static_cast<const float*>(place(jobs->T, c->sT.ptr, lt, 4));
  dj->B_down = static_cast<const float*>(place(jobs->B_down, c->sBd.ptr, kNMax, 4));
  dj->B_up = static_cast<const float*>(place(jobs->B_up, c->sBu.ptr, kNMax, 4));
  dj->n_layers = static_cast<const int32_t*>(place(jobs->n_layers, c->sL.ptr, 1, 4));
  dj->model_type = static_cast<const int32_t*>(place(jobs->model_type, c->sM.ptr, 1, 4));
  dj->arch_type = static_cast<const int32_t*>(place(jobs->arch_type, c->sArc.ptr, 1, 4));
  if (e != cudaSuccess) return e;
  dj->n_workers = c->sN.ptr;
  return cudaMemcpyAsync(c->sN.ptr, jobs->n_workers, (size_t)J * 4, cudaMemcpyHostToDevice, c->stream);
}

// Bytes the *_host staging above moves for J jobs on this rank (for the e2e accounting).
size_t staged_job_bytes(const autobyte_ctx* c, int J, int l_max) {
  int jb = 0, je = J;
  encode_range(c, J, &jb, &je);
  if (c->check) { jb = 0; je = J; }
  const size_t nj = (size_t)(je - jb);
  return nj * ((size_t)l_max * kNMax * 4 + 2 * kNMax * 4 + 3 * 4) + (size_t)J * 4;
}

autobyte_status run_encode_and_score(autobyte_ctx* c, const autobyte_job_stats* jobs, const autobyte_grid* grid,
                                     const int32_t* cur_idx, float* scores, int32_t* best_idx = nullptr,
                                     float* best_score = nullptr, float* cur_score = nullptr,
                                     bool* finalized = nullptr) {
  if (finalized) *finalized = false;
  const int J = jobs->J;
  autobyte_status st = ensure_job_ws(c, J);
  if (st != AB_OK) return st;
  const int H = c->desc.hidden_width;
  const long long cs = grid->shard_end - grid->shard_begin;
  // K1b's outputs and the grid axes (a-1): up[P] | uc[Q]
  EncodeParams proj{};
  proj.jv = 2 * H + 4;
  proj.a_out = c->jobvec.ptr; proj.what_out = c->jobvec.ptr + H; proj.beta_out = c->jobvec.ptr + 2 * H;
  proj.keys = c->keys.ptr; proj.cur_keys = c->keys.ptr + J;
  proj.P = grid->P; proj.Q = grid->Q;
  proj.S_p = reinterpret_cast<const long long*>(grid->partition_bytes); proj.S_c = grid->credit_mult;
  if (cs > 0) {
    AB_CUDA(c, c->u.ensure((size_t)grid->P + grid->Q));
    proj.up_out = c->u.ptr; proj.uc_out = c->u.ptr + grid->P;
  }
  EncodeParams ep{};
  bool projected = false;
  if ((st = run_lstm(c, jobs, &ep, &proj, &projected)) != AB_OK) return st;
  if (!projected) {
    ep.jv = proj.jv; ep.a_out = proj.a_out; ep.what_out = proj.what_out; ep.beta_out = proj.beta_out;
    ep.keys = proj.keys; ep.cur_keys = proj.cur_keys;
    ep.P = proj.P; ep.Q = proj.Q; ep.S_p = proj.S_p; ep.S_c = proj.S_c;
    ep.up_out = proj.up_out; ep.uc_out = proj.uc_out;
    AB_CUDA(c, timed(c, K_ENCODE, [&] { return launch_project(ep, c->stream); }));
  }
  if (cs == 0) return AB_OK;   // empty shard of a multi-rank partition: the keys stay 0 (K1b reset them)
  if ((long long)grid->P + grid->Q > kFusedAxes) {   // K0: large axes get their own launch
    EncodeParams ap = proj;
    AB_CUDA(c, timed(c, K_ENCODE, [&] { return launch_grid_axes(ap, c->stream); }));
  }

  ScoreParams sp{};
  sp.J = J; sp.H = c->desc.hidden_width; sp.G = c->desc.hidden_layers - 1;
  sp.P = grid->P; sp.Q = grid->Q;
  sp.c_begin = grid->shard_begin; sp.c_end = grid->shard_end;
  sp.tiles_per_job = static_cast<int>((cs + kTileM - 1) / kTileM);
  sp.n_tiles = (long long)sp.tiles_per_job * J;
  if (sp.n_tiles >= (1ll << 31))   // K2 indexes tiles in 32 bits
    return fail(c, AB_E_SHAPE, "J * ceil(shard / 128) must stay below 2^31 per call");
  make_fastdiv(static_cast<uint32_t>(sp.tiles_per_job), &sp.tpj_mul, &sp.tpj_shr);
  make_fastdiv(static_cast<uint32_t>(grid->Q), &sp.q_mul, &sp.q_shr);
  sp.S_p = reinterpret_cast<const long long*>(grid->partition_bytes); sp.S_c = grid->credit_mult;
  sp.params = c->params.ptr; sp.off = c->off;
  sp.jobvec = c->jobvec.ptr;
  sp.up = c->u.ptr; sp.uc = c->u.ptr + grid->P;
  sp.wpack = c->wpack.ptr;
  sp.wmap = c->wmap;
  sp.cta_group = c->planes == 2 ? (c->desc.hidden_width == 512 ? 2 : 1) : c->cta_group;
  sp.spill = c->spill.ptr;
  sp.precision3 = c->planes == 2 ? 1 : 0;
  sp.keys = c->keys.ptr; sp.cur_keys = c->keys.ptr + J;
  sp.cur_idx = cur_idx; sp.scores = scores;
  sp.done = c->done.ptr;   // CTA exit counter; the last CTA zeroes it
  if (best_idx && !(c->comm && c->world > 1)) {   // single rank: K2's last CTA decodes the keys
    sp.finalize = 1;
    sp.best_idx = best_idx; sp.best_score = best_score; sp.cur_score = cur_score;
    if (finalized) *finalized = true;
  }
  AB_CUDA(c, timed(c, K_SCORE, [&] { return launch_score(sp, c->num_sms, c->stream); }));
  c->score_pairs += (double)J * (double)cs;
  return AB_OK;
}

}  // namespace

// =====================================================================================
extern "C" {

int32_t autobyte_abi_version(void) { return AUTOBYTE_ABI_VERSION; }

const char* autobyte_status_string(autobyte_status s) {
  switch (s) {
    case AB_OK: return "ok";
    case AB_E_INVALID: return "invalid argument";
    case AB_E_SHAPE: return "shape mismatch";
    case AB_E_CUDA: return "CUDA error";
    case AB_E_NCCL: return "NCCL error";
    case AB_E_NONFINITE: return "non-finite weights";
    case AB_E_UNSUPPORTED: return "unsupported";
    case AB_E_NOMEM: return "out of memory";
  }
  return "unknown status";
}

autobyte_status autobyte_validate_desc(const autobyte_net_desc* d) {
  if (!d) return AB_E_INVALID;
  if (d->hidden_layers < 1 || d->hidden_layers > kMaxHidden) return AB_E_INVALID;
  const int H = d->hidden_width;
  if (H != 64 && H != 128 && H != 256 && H != 512) return AB_E_INVALID;
  if (d->n_max != kNMax || d->embed_dim != kEmbed || d->lstm_hidden != kLstm || d->type_embed_dim != kTypeEmbed)
    return AB_E_INVALID;
  if (d->n_model_types < 1 || d->n_model_types > 64 || d->n_arch_types < 1 || d->n_arch_types > 16)
    return AB_E_INVALID;
  return AB_OK;
}

autobyte_status autobyte_blob_bytes(const autobyte_net_desc* d, size_t* out) {
  if (!out) return AB_E_INVALID;
  autobyte_status s = autobyte_validate_desc(d);
  if (s != AB_OK) return s;
  *out = kBlobHeader + (size_t)make_offsets(*d).total * sizeof(float);
  return AB_OK;
}

autobyte_status autobyte_validate_blob(const autobyte_net_desc* d, const void* blob, size_t bytes) {
  if (!blob) return AB_E_INVALID;
  size_t want = 0;
  autobyte_status s = autobyte_blob_bytes(d, &want);
  if (s != AB_OK) return s;
  if (bytes != want) return AB_E_SHAPE;
  const uint8_t* b = static_cast<const uint8_t*>(blob);
  if (std::memcmp(b, AUTOBYTE_BLOB_MAGIC, 4) != 0) return AB_E_INVALID;
  uint32_t ver;
  std::memcpy(&ver, b + 4, 4);
  if (ver != AUTOBYTE_BLOB_VERSION) return AB_E_INVALID;
  autobyte_net_desc bd;
  std::memcpy(&bd, b + 8, sizeof(bd));
  if (std::memcmp(&bd, d, sizeof(bd)) != 0) return AB_E_SHAPE;
  uint32_t n_arrays;
  std::memcpy(&n_arrays, b + 40, 4);
  if (n_arrays != static_cast<uint32_t>(12 + 2 * (d->hidden_layers - 1) + 2)) return AB_E_SHAPE;
  const size_t nf = (bytes - kBlobHeader) / sizeof(float);
  const float* f = reinterpret_cast<const float*>(b + kBlobHeader);
  for (size_t i = 0; i < nf; ++i) {
    float v;
    std::memcpy(&v, f + i, 4);
    if (!std::isfinite(v)) return AB_E_NONFINITE;
  }
  return AB_OK;
}

autobyte_status autobyte_create(const autobyte_net_desc* desc, const void* blob, size_t blob_bytes, int device,
                                void* cuda_stream, autobyte_precision precision, autobyte_ctx** out) {
  NvtxRange nvtx_range("autobyte_create");
  if (!out) return AB_E_INVALID;
  *out = nullptr;
  autobyte_status s = autobyte_validate_desc(desc);
  if (s != AB_OK) return s;
  s = autobyte_validate_blob(desc, blob, blob_bytes);
  if (s != AB_OK) return s;
  if (precision != AB_PREC_BF16 && precision != AB_PREC_FP32) return AB_E_INVALID;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return AB_E_CUDA;
  }
  if (device < 0 || device >= ndev) return AB_E_INVALID;
  DeviceGuard guard(device);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return AB_E_CUDA;
  if (prop.major != 10 || prop.minor != 0) return AB_E_UNSUPPORTED;  // sm_100a code only

  autobyte_ctx* c = new autobyte_ctx();
  c->desc = *desc;
  c->off = make_offsets(*desc);
  c->precision = precision;
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  c->stream = static_cast<cudaStream_t>(cuda_stream);
  const char* se = std::getenv("AUTOBYTE_SHARD_ENCODE");
  c->shard_encode = !(se && se[0] == '0');
  const char* ex = std::getenv("AUTOBYTE_EXCHANGE");
  c->exchange_allreduce = ex && std::strcmp(ex, "allreduce") == 0;
  c->exchange_nccl = ex && (std::strcmp(ex, "nccl") == 0 || c->exchange_allreduce);
  const char* zc = std::getenv("AUTOBYTE_ZERO_COPY");
  c->zero_copy = !(zc && zc[0] == '0');
  const char* px = std::getenv("AUTOBYTE_PEER_X");
  c->peer_x = px && px[0] == '1';
  const char* chk = std::getenv("AUTOBYTE_CHECK");
  c->check = chk && chk[0] == '1';
  const char* dm = std::getenv("AUTOBYTE_DEBUG_MEM");
  if (dm && dm[0] == '1') g_debug_mem = true;   // process-wide from the first such create on
  const char* pt = std::getenv("AUTOBYTE_PEER_TIMEOUT_S");
  const double pts = pt ? std::atof(pt) : 120.0;
  c->peer_timeout_ns = pts > 0 ? static_cast<unsigned long long>(pts * 1e9) : 0ull;
  auto bail = [&](cudaError_t e, const char* what) {
    std::fprintf(stderr, "autobyte_create: %s: %s\n", what, cudaGetErrorString(e));
    autobyte_destroy(c);
    return AB_E_CUDA;
  };
  cudaError_t e;
  if ((e = device_status_word(device, &c->status)) != cudaSuccess) return bail(e, "device status word");
  if ((e = c->params.ensure(c->off.total)) != cudaSuccess) return bail(e, "alloc params");
  if ((e = c->grads.ensure(c->off.total * kAdaptSplitK)) != cudaSuccess) return bail(e, "alloc grads");
  if ((e = cudaMemsetAsync(c->grads.ptr, 0, c->off.total * kAdaptSplitK * sizeof(float), c->stream)) != cudaSuccess)
    return bail(e, "memset grads");
  if ((e = cudaMemcpyAsync(c->params.ptr, static_cast<const uint8_t*>(blob) + kBlobHeader,
                           c->off.total * sizeof(float), cudaMemcpyHostToDevice, c->stream)) != cudaSuccess)
    return bail(e, "copy blob");
  c->planes = precision == AB_PREC_FP32 ? 2 : 1;
  const size_t wp = packed_weight_elems(desc->hidden_width, desc->hidden_layers, c->planes);
  if ((e = c->wpack.ensure(wp ? wp * kWeightReplicas : 1)) != cudaSuccess) return bail(e, "alloc wpack");
  if ((e = c->barrier.ensure(2)) != cudaSuccess) return bail(e, "alloc barrier");
  if ((e = c->done.ensure(1)) != cudaSuccess) return bail(e, "alloc done counter");
  if ((e = cudaMemsetAsync(c->done.ptr, 0, sizeof(unsigned int), c->stream)) != cudaSuccess) return bail(e, "memset done");
  // K2 variant: CTA pairs win when the head is deep and wide (4x512: 1158 vs 1133 TFLOP/s),
  // CTA pairs win from H = 256 up (C4 4x512: 1416 vs 1119 TFLOP/s; 3x256: 808 vs 757); single
  // CTAs on the narrow heads (3x128: 320 vs 314). AUTOBYTE_CTA_GROUP=1|2 overrides.
  const char* cg = std::getenv("AUTOBYTE_CTA_GROUP");
  c->cta_group = desc->hidden_width >= 256 ? 2 : 1;
  if (cg && (cg[0] == '1' || cg[0] == '2')) c->cta_group = cg[0] - '0';
  if (precision == AB_PREC_FP32 && desc->hidden_width == 512 && desc->hidden_layers > 1) {
    // K2's activation scratch of the fp32 path at H = 512 (score.cu SPILL): per CTA 128 rows x the
    // hi and lo bf16 of one layer (256 KB), one CTA per SM; it stays L2-resident
    if ((e = c->spill.ensure((size_t)c->num_sms * kTileM * desc->hidden_width)) != cudaSuccess)
      return bail(e, "alloc fp32 scratch");
  }
  if (!make_column_tmaps(c->wcol, c->params.ptr, c->off, desc->hidden_width, desc->hidden_layers)) {
    autobyte_destroy(c);
    return AB_E_CUDA;
  }
  if (!make_weight_tmap(&c->wmap, c->wpack.ptr, desc->hidden_width, desc->hidden_layers, c->planes)) {
    autobyte_destroy(c);
    return AB_E_CUDA;
  }
  if ((e = cudaMemsetAsync(c->barrier.ptr, 0, 2 * sizeof(unsigned int), c->stream)) != cudaSuccess)
    return bail(e, "memset barrier");
  if ((e = timed(c, K_PACK, [&] {
         return launch_pack(c->params.ptr, c->off, desc->hidden_width, desc->hidden_layers, c->planes, c->wpack.ptr,
                            c->stream);
       })) != cudaSuccess)
    return bail(e, "pack weights");
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return bail(e, "synchronize");
  *out = c;
  return AB_OK;
}

void autobyte_destroy(autobyte_ctx* c) {
  if (!c) return;
  DeviceGuard guard(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& p : c->pending) {
    cudaEventDestroy(p.second.first);
    cudaEventDestroy(p.second.second);
  }
  close_peer_window(c);
  if (c->comm) ncclCommDestroy(c->comm);
  c->params.release(); c->grads.release(); c->wpack.release(); c->spill.release(); c->barrier.release(); c->flag.release();
  c->jobvec.release(); c->u.release(); c->done.release(); c->x.release(); c->adapt_ws.release();
  c->opt_m.release(); c->opt_v.release(); c->topk_scores.release(); c->topk_keys.release();
  c->enc_stash.release(); c->enc_dz.release(); c->enc_part.release();
  c->loss_tmp.release(); c->keys.release();
  c->sT.release(); c->sBd.release(); c->sBu.release(); c->sSc.release(); c->sV.release();
  c->rScore.release(); c->rCur.release();
  c->sN.release(); c->sL.release(); c->sM.release(); c->sArc.release(); c->sCur.release(); c->rIdx.release();
  c->sSp.release();
  delete c;
}

const char* autobyte_last_error(const autobyte_ctx* c) { return c ? c->last_error.c_str() : "NULL ctx"; }

autobyte_status autobyte_synchronize(autobyte_ctx* c) {
  if (!c) return AB_E_INVALID;
  DeviceGuard guard(c->device);
  AB_CUDA(c, cudaStreamSynchronize(c->stream));
  return take_status(c);
}

autobyte_status autobyte_get_unique_id(void* out) {
  if (!out) return AB_E_INVALID;
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return AB_E_NCCL;
  std::memcpy(out, &id, sizeof(id));
  return AB_OK;
}

autobyte_status autobyte_attach_comm(autobyte_ctx* c, const void* uid, int rank, int world) {
  NvtxRange nvtx_range("autobyte_attach_comm");
  if (!c) return AB_E_INVALID;
  if (world < 1 || rank < 0 || rank >= world) return fail(c, AB_E_INVALID, "bad rank/world");
  DeviceGuard guard(c->device);
  if (c->comm) {
    close_peer_window(c);
    ncclCommDestroy(c->comm);
    c->comm = nullptr;
  }
  c->rank = rank;
  c->world = world;
  if (world == 1) return AB_OK;
  if (!uid) return fail(c, AB_E_INVALID, "unique id is NULL");
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
  if (r != ncclSuccess) {
    c->comm = nullptr;
    return fail(c, AB_E_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  c->peer = setup_peer_window(c);
  if (!c->peer) close_peer_window(c);
  return AB_OK;
}

int32_t autobyte_peer_exchange(const autobyte_ctx* c) { return c && c->peer ? 1 : 0; }

autobyte_status autobyte_encode(autobyte_ctx* c, const autobyte_job_stats* jobs, float* x_out) {
  NvtxRange nvtx_range("autobyte_encode");
  if (!c) return AB_E_INVALID;
  if (autobyte_status ws = take_status(c)) return ws;
  autobyte_status s = check_jobs_host(c, jobs);
  if (s != AB_OK) return s;
  if (!x_out) return fail(c, AB_E_INVALID, "x_out is NULL");
  DeviceGuard guard(c->device);
  if ((s = device_checks(c, jobs, nullptr)) != AB_OK) return s;
  EncodeParams ep = encode_params(c, jobs);
  ep.x_out = x_out;
  ep.j_begin = 0; ep.j_end = jobs->J;
  AB_CUDA(c, timed(c, K_ENCODE, [&] { return launch_encode_lstm(ep, c->num_sms, c->stream); }));
  return AB_OK;
}

autobyte_status autobyte_score(autobyte_ctx* c, const autobyte_job_stats* jobs, const autobyte_grid* grid,
                               float* scores) {
  NvtxRange nvtx_range("autobyte_score");
  if (!c) return AB_E_INVALID;
  if (autobyte_status ws = take_status(c)) return ws;
  autobyte_status s = check_jobs_host(c, jobs);
  if (s != AB_OK) return s;
  if ((s = check_grid_host(c, grid)) != AB_OK) return s;
  if (!scores && grid->shard_end > grid->shard_begin) return fail(c, AB_E_INVALID, "scores is NULL");
  DeviceGuard guard(c->device);
  if ((s = device_checks(c, jobs, grid)) != AB_OK) return s;
  return run_encode_and_score(c, jobs, grid, nullptr, scores);
}

autobyte_status autobyte_argmax(autobyte_ctx* c, const autobyte_job_stats* jobs, const autobyte_grid* grid,
                                const int32_t* cur_idx, int32_t* best_idx, float* best_score, float* cur_score) {
  NvtxRange nvtx_range("autobyte_argmax");
  if (!c) return AB_E_INVALID;
  if (autobyte_status ws = take_status(c)) return ws;
  autobyte_status s = check_jobs_host(c, jobs);
  if (s != AB_OK) return s;
  if ((s = check_grid_host(c, grid)) != AB_OK) return s;
  if (!best_idx || !best_score) return fail(c, AB_E_INVALID, "best_idx / best_score is NULL");
  DeviceGuard guard(c->device);
  if ((s = device_checks(c, jobs, grid)) != AB_OK) return s;
  bool finalized = false;
  if ((s = run_encode_and_score(c, jobs, grid, cur_idx, nullptr, best_idx, best_score, cur_score, &finalized)) != AB_OK)
    return s;
  const int J = jobs->J;
  if (finalized) return AB_OK;   // one rank: K2's last CTA already decoded the keys (K5 folded in)
  // K3 (§8(a) a-7): the per-rank (score, index) keys are all-gathered over NVLink (one pass; the
  // per-job max is folded into K5), or with AUTOBYTE_EXCHANGE=allreduce reduced by ncclAllReduce(max)
  const unsigned long long* kin = c->keys.ptr;
  int G = 1;
  if (c->comm && c->world > 1 && c->peer && 2LL * J <= c->win_cap2) {
    // fused K3 + K5 over NVLink peer memory (exchange.cu)
    PeerExchangeParams xp{};
    for (int r = 0; r < c->world; ++r) xp.win[r] = c->peer_win[r];
    xp.keys = c->keys.ptr; xp.counter = c->win_counter.ptr;
    xp.best_idx = best_idx; xp.best_score = best_score; xp.cur_score = cur_score;
    xp.epoch = c->win_epoch.ptr; xp.timeout_ns = c->peer_timeout_ns;
    xp.cap2 = c->win_cap2; xp.J = J; xp.G = c->world; xp.rank = c->rank;
    // (profiled as K5, whose work it includes: finalize_ms then also holds the wait for the
    // slowest rank, exchange_ms only the NCCL x all-gathers)
    AB_CUDA(c, timed(c, K_FINALIZE, [&] { return launch_peer_exchange(xp, c->num_sms, c->stream); }));
    return AB_OK;
  }
  if (c->comm && c->world > 1) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (c->profiling) { cudaEventCreate(&a); cudaEventCreate(&b); cudaEventRecord(a, c->stream); }
    ncclResult_t r;
    if (c->exchange_allreduce) {
      r = ncclAllReduce(c->keys.ptr, c->keys.ptr, (size_t)2 * J, ncclUint64, ncclMax, c->comm, c->stream);
    } else {
      AB_CUDA(c, c->keys_all.ensure((size_t)2 * J * c->world));
      r = ncclAllGather(c->keys.ptr, c->keys_all.ptr, (size_t)2 * J, ncclUint64, c->comm, c->stream);
      kin = c->keys_all.ptr;
      G = c->world;
    }
    if (c->profiling) { cudaEventRecord(b, c->stream); c->pending.push_back({K_EXCHANGE, {a, b}}); }
    if (r != ncclSuccess) return fail(c, AB_E_NCCL, std::string("nccl key exchange: ") + ncclGetErrorString(r));
    c->launches[K_EXCHANGE] += 1;
  }
  AB_CUDA(c, timed(c, K_FINALIZE, [&] {
            return launch_finalize(J, G, 2LL * J, kin, kin + J, best_idx, best_score, cur_score, c->stream);
          }));
  return AB_OK;
}

autobyte_status autobyte_argmax_keys(autobyte_ctx* c, const autobyte_job_stats* jobs, const autobyte_grid* grid,
                                     const int32_t* cur_idx, uint64_t* keys_out) {
  NvtxRange nvtx_range("autobyte_argmax_keys");
  if (!c) return AB_E_INVALID;
  if (autobyte_status ws = take_status(c)) return ws;
  autobyte_status s = check_jobs_host(c, jobs);
  if (s != AB_OK) return s;
  if ((s = check_grid_host(c, grid)) != AB_OK) return s;
  if (!keys_out) return fail(c, AB_E_INVALID, "keys_out is NULL");
  DeviceGuard guard(c->device);
  if ((s = device_checks(c, jobs, grid)) != AB_OK) return s;
  if ((s = run_encode_and_score(c, jobs, grid, cur_idx, nullptr)) != AB_OK) return s;
  AB_CUDA(c, cudaMemcpyAsync(keys_out, c->keys.ptr, (size_t)2 * jobs->J * sizeof(uint64_t), cudaMemcpyDeviceToDevice,
                             c->stream));
  return AB_OK;
}

autobyte_status autobyte_reduce_keys(autobyte_ctx* c, int32_t J, int32_t G, const uint64_t* keys, int32_t* best_idx,
                                     float* best_score, float* cur_score) {
  NvtxRange nvtx_range("autobyte_reduce_keys");
  if (!c) return AB_E_INVALID;
  if (autobyte_status ws = take_status(c)) return ws;
  if (J < 1 || G < 1) return fail(c, AB_E_SHAPE, "J and G must be >= 1");
  if (!keys || !best_idx || !best_score) return fail(c, AB_E_INVALID, "keys / best_idx / best_score is NULL");
  DeviceGuard guard(c->device);
  const unsigned long long* k = reinterpret_cast<const unsigned long long*>(keys);
  AB_CUDA(c, timed(c, K_FINALIZE, [&] {
            return launch_finalize(J, G, 2LL * J, k, k + J, best_idx, best_score, cur_score, c->stream);
          }));
  return AB_OK;
}

autobyte_status autobyte_debug_fastdiv(uint32_t d, const uint32_t* n, int32_t count, uint32_t* out) {
  if (d < 1 || count < 0 || (count > 0 && (!n || !out))) return AB_E_SHAPE;
  uint32_t mul = 0, shr = 0;
  make_fastdiv(d, &mul, &shr);
  for (int32_t i = 0; i < count; ++i) {
    if (n[i] >= 0x80000000u) return AB_E_SHAPE;
    // fdiv() of internal.h on the host: __umulhi(n, mul) >> shr
    out[i] = d == 1 ? n[i] : static_cast<uint32_t>((static_cast<uint64_t>(n[i]) * mul) >> 32) >> shr;
  }
  return AB_OK;
}

int32_t autobyte_debug_mem_check(autobyte_ctx* c) {
  if (!c) return -1;
  DeviceGuard guard(c->device);
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  std::lock_guard<std::mutex> lock(g_canary_mu);
  int32_t bad = 0;
  std::vector<uint8_t> h(kCanaryBytes);
  for (auto& t : g_canaries) {
    if (static_cast<int>(t.second) != c->device) continue;
    if (cudaMemcpy(h.data(), t.first, kCanaryBytes, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    for (uint8_t b : h)
      if (b != 0xA5) { ++bad; break; }
  }
  return bad;
}

autobyte_status autobyte_debug_peer_loopback(autobyte_ctx* c, int32_t G, int32_t J, int32_t calls, int32_t absent_rank,
                                             int32_t timeout_ms, const uint64_t* keys, int32_t* best_idx,
                                             float* best_score, float* cur_score) {
  if (!c) return AB_E_INVALID;
  if (autobyte_status ws = take_status(c)) return ws;
  if (G < 1 || G > kMaxPeers || J < 1 || calls < 1 || timeout_ms < 1)
    return fail(c, AB_E_SHAPE, "need 1 <= G <= 8, J >= 1, calls >= 1, timeout_ms >= 1");
  if (!keys || !best_idx || !best_score || !cur_score) return fail(c, AB_E_INVALID, "NULL pointer");
  DeviceGuard guard(c->device);
  AB_CUDA(c, cudaStreamSynchronize(c->stream));
  // G windows on this device, laid out exactly as setup_peer_window lays out the IPC-shared ones
  const long long cap2 = 2LL * J;
  const size_t words = kPeerFlagWords + 2 * (size_t)G * cap2;
  DevBuf<unsigned long long> win, epochs;
  DevBuf<unsigned int> counters;
  AB_CUDA(c, win.ensure(words * G));
  AB_CUDA(c, epochs.ensure(G));
  AB_CUDA(c, counters.ensure(G));
  AB_CUDA(c, cudaMemset(win.ptr, 0, words * G * 8));
  AB_CUDA(c, cudaMemset(epochs.ptr, 0, G * 8));
  AB_CUDA(c, cudaMemset(counters.ptr, 0, G * 4));
  std::vector<cudaStream_t> st(G, nullptr);
  for (auto& x : st) AB_CUDA(c, cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
  cudaError_t e = cudaSuccess;
  for (int call = 0; call < calls && e == cudaSuccess; ++call) {
    for (int r = 0; r < G && e == cudaSuccess; ++r) {   // virtual rank r on its own stream
      if (r == absent_rank) continue;
      PeerExchangeParams xp{};
      for (int q = 0; q < G; ++q) xp.win[q] = win.ptr + (size_t)q * words;
      xp.keys = reinterpret_cast<const unsigned long long*>(keys) + (size_t)r * cap2;
      xp.counter = counters.ptr + r;
      xp.best_idx = best_idx + (size_t)r * J; xp.best_score = best_score + (size_t)r * J;
      xp.cur_score = cur_score + (size_t)r * J;
      xp.epoch = epochs.ptr + r; xp.timeout_ns = 1000000ull * static_cast<unsigned long long>(timeout_ms);
      xp.cap2 = cap2; xp.J = J; xp.G = G; xp.rank = r;
      e = launch_peer_exchange(xp, c->num_sms, st[r], false);
    }
    for (auto& x : st)
      if (e == cudaSuccess) e = cudaStreamSynchronize(x);
  }
  for (auto& x : st) cudaStreamDestroy(x);
  if (e != cudaSuccess) return cuda_fail(c, e, "peer loopback");
  return take_status(c);
}

}  // extern "C"

namespace {
// K1a on the samples (sharded across ranks) + K4 + re-pack: the body of adapt and train.
autobyte_status run_head_update(autobyte_ctx* c, const autobyte_job_stats* samples, const int64_t* sp_bytes,
                                const float* sc_mult, const float* v_obs, int opt, float lr, float beta1,
                                float beta2, float eps, int32_t steps, float* loss_before, float* losses,
                                const int32_t* idx = nullptr, int batch = 0) {
  // idx != nullptr (train_epoch): samples is the whole dataset (encoded once, encoder frozen) and
  // step s trains on the `batch` rows idx[s][0..batch) of it, gathered inside K4
  const int B = idx ? batch : samples->J, H = c->desc.hidden_width, L = c->desc.hidden_layers;
  AB_CUDA(c, c->adapt_ws.ensure(adapt_ws_floats(B, H, L)));
  EncodeParams ep{};
  autobyte_status s = run_lstm(c, samples, &ep);
  if (s != AB_OK) return s;
  AdaptParams ap{};
  ap.B = B; ap.H = H; ap.L = L; ap.steps = steps; ap.lr = lr;
  ap.x = ep.x_out;   // the peer window's x region when the gather ran through it
  ap.S_p = reinterpret_cast<const long long*>(sp_bytes); ap.S_c = sc_mult; ap.v_obs = v_obs;
  ap.n = samples->n_workers;
  ap.params = c->params.ptr; ap.off = c->off; ap.ws = c->adapt_ws.ptr; ap.grads = c->grads.ptr;
  ap.loss_before = loss_before; ap.losses = losses; ap.barrier = c->barrier.ptr;
  ap.opt = opt; ap.beta1 = beta1; ap.beta2 = beta2; ap.eps = eps;
  ap.idx = idx;
  ap.wpack = c->wpack.ptr; ap.planes = c->planes;
  for (int k = 0; k <= kMaxHidden; ++k) ap.wcol[k] = c->wcol[k];
  if (opt == AB_OPT_ADAM) {
    if (!c->opt_m.ptr) {   // moments start at zero (blob layout; only the head part is used)
      AB_CUDA(c, c->opt_m.ensure(c->off.total));
      AB_CUDA(c, c->opt_v.ensure(c->off.total));
      AB_CUDA(c, cudaMemsetAsync(c->opt_m.ptr, 0, c->off.total * sizeof(float), c->stream));
      AB_CUDA(c, cudaMemsetAsync(c->opt_v.ptr, 0, c->off.total * sizeof(float), c->stream));
    }
    ap.m = c->opt_m.ptr; ap.v = c->opt_v.ptr; ap.t0 = c->opt_t;
  }
  int grid_used = 0;
  // small minibatches (the per-job online adaptation): one thread-block cluster (K4s,
  // adapt_small.cu) instead of the grid-wide tcgen05 kernel; the choice depends on B only, so every
  // replica and every entry point (adapt, train) runs the same kernel for the same minibatch
  bool small_done = false;
  AB_CUDA(c, timed(c, K_ADAPT, [&] {
            cudaError_t e = launch_adapt_small(ap, c->stream);
            if (e != cudaErrorNotSupported) { small_done = true; return e; }
            cudaGetLastError();
            return launch_adapt(ap, c->num_sms, c->stream, &grid_used);
          }));
  if (opt == AB_OPT_ADAM) c->opt_t += steps;
  if (steps > 0 && !small_done)   // (K4s refreshed the shadows of what it updated in place)
    AB_CUDA(c, timed(c, K_PACK, [&] {
              return launch_pack(c->params.ptr, c->off, H, L, c->planes, c->wpack.ptr, c->stream);
            }));
  return AB_OK;
}
}  // namespace

extern "C" {

autobyte_status autobyte_topk(autobyte_ctx* c, const autobyte_job_stats* jobs, const autobyte_grid* grid, int32_t k,
                              int32_t* idx, float* score) {
  NvtxRange nvtx_range("autobyte_topk");
  if (!c) return AB_E_INVALID;
  if (autobyte_status ws = take_status(c)) return ws;
  autobyte_status s = check_jobs_host(c, jobs);
  if (s != AB_OK) return s;
  if ((s = check_grid_host(c, grid)) != AB_OK) return s;
  if (k < 1 || k > 32) return fail(c, AB_E_INVALID, "k must be in [1, 32]");
  if (!idx || !score) return fail(c, AB_E_INVALID, "idx / score is NULL");
  DeviceGuard guard(c->device);
  if ((s = device_checks(c, jobs, grid)) != AB_OK) return s;
  const int J = jobs->J;
  const long long cs = grid->shard_end - grid->shard_begin;
  const int G = (c->comm && c->world > 1) ? c->world : 1;
  AB_CUDA(c, c->topk_scores.ensure(cs > 0 ? (size_t)J * cs : 1));
  AB_CUDA(c, c->topk_keys.ensure((size_t)G * J * k));
  if ((s = run_encode_and_score(c, jobs, grid, nullptr, c->topk_scores.ptr)) != AB_OK) return s;
  unsigned long long* mine = c->topk_keys.ptr + (G > 1 ? (size_t)c->rank * J * k : 0);
  if (cs == 0)   // empty shard of a multi-rank partition: an all-empty list (key 0 = no candidate)
    AB_CUDA(c, cudaMemsetAsync(mine, 0, (size_t)J * k * sizeof(unsigned long long), c->stream));
  else
    AB_CUDA(c, timed(c, K_FINALIZE, [&] {
              return launch_topk(J, cs, c->topk_scores.ptr, grid->shard_begin, k, mine, c->stream);
            }));
  if (G > 1) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (c->profiling) { cudaEventCreate(&a); cudaEventCreate(&b); cudaEventRecord(a, c->stream); }
    ncclResult_t r = ncclAllGather(mine, c->topk_keys.ptr, (size_t)J * k, ncclUint64, c->comm, c->stream);
    if (c->profiling) { cudaEventRecord(b, c->stream); c->pending.push_back({K_EXCHANGE, {a, b}}); }
    if (r != ncclSuccess) return fail(c, AB_E_NCCL, std::string("ncclAllGather: ") + ncclGetErrorString(r));
    c->launches[K_EXCHANGE] += 1;
  }
  AB_CUDA(c, timed(c, K_FINALIZE, [&] {
            return launch_topk_merge(J, G, k, c->topk_keys.ptr, idx, score, c->stream);
          }));
  return AB_OK;
}

autobyte_status autobyte_adapt(autobyte_ctx* c, const autobyte_job_stats* samples, const int64_t* sp_bytes,
                               const float* sc_mult, const float* v_obs, float lr, int32_t steps,
                               float* loss_before) {
  NvtxRange nvtx_range("autobyte_adapt");
  if (!c) return AB_E_INVALID;
  if (autobyte_status ws = take_status(c)) return ws;
  autobyte_status s = check_jobs_host(c, samples);
  if (s != AB_OK) return s;
  if (!sp_bytes || !sc_mult || !v_obs) return fail(c, AB_E_INVALID, "adapt input pointer is NULL");
  if (steps < 0) return fail(c, AB_E_INVALID, "steps must be >= 0");
  if (!std::isfinite(lr)) return fail(c, AB_E_INVALID, "lr must be finite");
  DeviceGuard guard(c->device);
  if ((s = device_checks(c, samples, nullptr)) != AB_OK) return s;
  if (steps == 0 && !loss_before) return AB_OK;
  return run_head_update(c, samples, sp_bytes, sc_mult, v_obs, AB_OPT_SGD, lr, 0.f, 0.f, 0.f, steps, loss_before,
                         nullptr);
}

autobyte_status autobyte_train(autobyte_ctx* c, const autobyte_job_stats* samples, const int64_t* sp_bytes,
                               const float* sc_mult, const float* v_obs, const autobyte_optimizer* opt,
                               int32_t steps, float* losses) {
  NvtxRange nvtx_range("autobyte_train");
  if (!c) return AB_E_INVALID;
  if (autobyte_status ws = take_status(c)) return ws;
  autobyte_status s = check_jobs_host(c, samples);
  if (s != AB_OK) return s;
  if (!sp_bytes || !sc_mult || !v_obs) return fail(c, AB_E_INVALID, "train input pointer is NULL");
  if (!opt) return fail(c, AB_E_INVALID, "optimizer is NULL");
  if (opt->kind != AB_OPT_SGD && opt->kind != AB_OPT_ADAM) return fail(c, AB_E_INVALID, "unknown optimizer kind");
  if (steps < 0) return fail(c, AB_E_INVALID, "steps must be >= 0");
  if (!std::isfinite(opt->lr)) return fail(c, AB_E_INVALID, "lr must be finite");
  if (opt->kind == AB_OPT_ADAM && !(opt->beta1 >= 0.f && opt->beta1 < 1.f && opt->beta2 >= 0.f && opt->beta2 < 1.f &&
                                    opt->eps > 0.f && std::isfinite(opt->eps)))
    return fail(c, AB_E_INVALID, "Adam needs 0 <= beta1, beta2 < 1 and eps > 0");
  if (opt->scope != AB_SCOPE_HEAD && opt->scope != AB_SCOPE_ALL) return fail(c, AB_E_INVALID, "unknown train scope");
  DeviceGuard guard(c->device);
  if ((s = device_checks(c, samples, nullptr)) != AB_OK) return s;
  if (steps == 0) return AB_OK;
  if (opt->scope == AB_SCOPE_HEAD)
    return run_head_update(c, samples, sp_bytes, sc_mult, v_obs, opt->kind, opt->lr, opt->beta1, opt->beta2,
                           opt->eps, steps, nullptr, losses);
  // AB_SCOPE_ALL (R#20): per step K1a with stash -> K4 (1 step, dX out, head update) -> K8 BPTT
  // partials -> K9 encoder update; the samples are re-encoded with the updated encoder each step
  const int B = samples->J, H = c->desc.hidden_width, L = c->desc.hidden_layers;
  AB_CUDA(c, c->adapt_ws.ensure(adapt_ws_floats(B, H, L)));
  AB_CUDA(c, c->x.ensure((size_t)B * kXDim));
  AB_CUDA(c, c->enc_stash.ensure((size_t)B * samples->l_max * kEncStash));
  AB_CUDA(c, c->enc_dz.ensure((size_t)B * kZDim));
  AB_CUDA(c, c->enc_part.ensure((size_t)encoder_bwd_parts(B, c->num_sms) * c->off.W[1]));
  if (opt->kind == AB_OPT_ADAM && !c->opt_m.ptr) {
    AB_CUDA(c, c->opt_m.ensure(c->off.total));
    AB_CUDA(c, c->opt_v.ensure(c->off.total));
    AB_CUDA(c, cudaMemsetAsync(c->opt_m.ptr, 0, c->off.total * sizeof(float), c->stream));
    AB_CUDA(c, cudaMemsetAsync(c->opt_v.ptr, 0, c->off.total * sizeof(float), c->stream));
  }
  for (int32_t st = 0; st < steps; ++st) {
    EncodeParams ep = encode_params(c, samples);
    ep.x_out = c->x.ptr;
    ep.j_begin = 0; ep.j_end = B;
    ep.stash = c->enc_stash.ptr;
    AB_CUDA(c, timed(c, K_ENCODE, [&] { return launch_encode_lstm(ep, c->num_sms, c->stream); }));
    AdaptParams ap{};
    ap.B = B; ap.H = H; ap.L = L; ap.steps = 1; ap.lr = opt->lr;
    ap.x = c->x.ptr; ap.S_p = reinterpret_cast<const long long*>(sp_bytes); ap.S_c = sc_mult; ap.v_obs = v_obs;
    ap.n = samples->n_workers;
    ap.params = c->params.ptr; ap.off = c->off; ap.ws = c->adapt_ws.ptr; ap.grads = c->grads.ptr;
    ap.losses = losses ? losses + st : nullptr; ap.barrier = c->barrier.ptr;
    ap.opt = opt->kind; ap.beta1 = opt->beta1; ap.beta2 = opt->beta2; ap.eps = opt->eps;
    ap.m = c->opt_m.ptr; ap.v = c->opt_v.ptr; ap.t0 = c->opt_t;
    ap.dz_out = c->enc_dz.ptr;
    int grid_used = 0;
    AB_CUDA(c, timed(c, K_ADAPT, [&] { return launch_adapt(ap, c->num_sms, c->stream, &grid_used); }));
    int nparts = 0;
    AB_CUDA(c, timed(c, K_ADAPT, [&] {
              return launch_encoder_bwd(ep, c->enc_dz.ptr, kZDim, c->enc_part.ptr, c->num_sms, &nparts, c->stream);
            }));
    AB_CUDA(c, timed(c, K_ADAPT, [&] {
              return launch_encoder_update(ep, c->enc_dz.ptr, kZDim, B, c->enc_part.ptr, nparts, opt->kind, opt->lr,
                                           opt->beta1, opt->beta2, opt->eps, c->opt_t + 1, c->opt_m.ptr,
                                           c->opt_v.ptr, c->stream);
            }));
    if (opt->kind == AB_OPT_ADAM) c->opt_t += 1;
  }
  AB_CUDA(c, timed(c, K_PACK, [&] {
            return launch_pack(c->params.ptr, c->off, H, L, c->planes, c->wpack.ptr, c->stream);
          }));
  return AB_OK;
}

autobyte_status autobyte_train_epoch(autobyte_ctx* c, const autobyte_job_stats* dataset, const int64_t* sp_bytes,
                                     const float* sc_mult, const float* v_obs, const int32_t* order, int32_t batch,
                                     int32_t steps, const autobyte_optimizer* opt, float* losses) {
  NvtxRange nvtx_range("autobyte_train_epoch");
  if (!c) return AB_E_INVALID;
  if (autobyte_status ws = take_status(c)) return ws;
  autobyte_status s = check_jobs_host(c, dataset);
  if (s != AB_OK) return s;
  if (!sp_bytes || !sc_mult || !v_obs || !order) return fail(c, AB_E_INVALID, "train_epoch input pointer is NULL");
  if (!opt) return fail(c, AB_E_INVALID, "optimizer is NULL");
  if (opt->kind != AB_OPT_SGD && opt->kind != AB_OPT_ADAM) return fail(c, AB_E_INVALID, "unknown optimizer kind");
  if (batch < 1 || steps < 0) return fail(c, AB_E_SHAPE, "need batch >= 1 and steps >= 0");
  if (!std::isfinite(opt->lr)) return fail(c, AB_E_INVALID, "lr must be finite");
  if (opt->kind == AB_OPT_ADAM && !(opt->beta1 >= 0.f && opt->beta1 < 1.f && opt->beta2 >= 0.f && opt->beta2 < 1.f &&
                                    opt->eps > 0.f && std::isfinite(opt->eps)))
    return fail(c, AB_E_INVALID, "Adam needs 0 <= beta1, beta2 < 1 and eps > 0");
  if (opt->scope != AB_SCOPE_HEAD)
    return fail(c, AB_E_UNSUPPORTED, "train_epoch trains the head (the encoder is encoded once per call)");
  DeviceGuard guard(c->device);
  if ((s = device_checks(c, dataset, nullptr)) != AB_OK) return s;
  if (steps == 0) return AB_OK;
  return run_head_update(c, dataset, sp_bytes, sc_mult, v_obs, opt->kind, opt->lr, opt->beta1, opt->beta2, opt->eps,
                         steps, nullptr, losses, order, batch);
}

autobyte_status autobyte_simulate(autobyte_ctx* c, const autobyte_job_stats* jobs, const float* layer_bytes,
                                  const float* fwd_ms, const autobyte_grid* grid, const autobyte_sim_params* sp,
                                  double* iter_ms) {
  NvtxRange nvtx_range("autobyte_simulate");
  if (!c) return AB_E_INVALID;
  if (autobyte_status ws = take_status(c)) return ws;
  autobyte_status s = check_jobs_host(c, jobs);
  if (s != AB_OK) return s;
  if ((s = check_grid_host(c, grid)) != AB_OK) return s;
  if (!layer_bytes || !sp || !iter_ms) return fail(c, AB_E_INVALID, "layer_bytes / params / iter_ms is NULL");
  if (!(sp->alpha_ms >= 0.0) || !(sp->delta_ms >= 0.0) || !std::isfinite(sp->alpha_ms) || !std::isfinite(sp->delta_ms))
    return fail(c, AB_E_INVALID, "alpha_ms and delta_ms must be finite and >= 0");
  if (simulate_smem_bytes(jobs->l_max) > 227 * 1024)
    return fail(c, AB_E_SHAPE, "l_max too large for the simulator's per-thread state (at most ~590 layers)");
  DeviceGuard guard(c->device);
  if ((s = device_checks(c, jobs, grid)) != AB_OK) return s;
  if (grid->shard_end == grid->shard_begin) return AB_OK;
  AB_CUDA(c, timed(c, K_OTHER, [&] {
            return launch_simulate(*jobs, layer_bytes, fwd_ms, *grid, sp->alpha_ms, sp->delta_ms, iter_ms, c->stream);
          }));
  return AB_OK;
}

autobyte_status autobyte_reset_optimizer(autobyte_ctx* c) {
  if (!c) return AB_E_INVALID;
  DeviceGuard guard(c->device);
  if (c->opt_m.ptr) {
    AB_CUDA(c, cudaMemsetAsync(c->opt_m.ptr, 0, c->off.total * sizeof(float), c->stream));
    AB_CUDA(c, cudaMemsetAsync(c->opt_v.ptr, 0, c->off.total * sizeof(float), c->stream));
  }
  c->opt_t = 0;
  return AB_OK;
}

int64_t autobyte_optimizer_step(const autobyte_ctx* c) { return c ? c->opt_t : -1; }

autobyte_status autobyte_trigger(autobyte_ctx* c, int32_t J, const int32_t* best_idx, const float* best_score,
                                 const int32_t* cur_idx, const float* cur_score, const float* v_observed,
                                 float gain, float drift, int32_t* action) {
  NvtxRange nvtx_range("autobyte_trigger");
  if (!c) return AB_E_INVALID;
  if (autobyte_status ws = take_status(c)) return ws;
  if (J < 1) return fail(c, AB_E_SHAPE, "J must be >= 1");
  if (!best_idx || !best_score || !cur_idx || !cur_score || !action)
    return fail(c, AB_E_INVALID, "trigger array pointer is NULL");
  if (!(gain >= 0.f) || !(drift >= 0.f)) return fail(c, AB_E_INVALID, "thresholds must be >= 0");
  DeviceGuard guard(c->device);
  AB_CUDA(c, timed(c, K_OTHER, [&] {
            return launch_trigger(J, best_idx, best_score, cur_idx, cur_score, v_observed, gain, drift, action,
                                  c->stream);
          }));
  return AB_OK;
}

size_t autobyte_staged_job_bytes(const autobyte_ctx* c, int32_t J, int32_t l_max) {
  return c && J > 0 && l_max > 0 ? staged_job_bytes(c, J, l_max) : 0;
}

autobyte_status autobyte_argmax_host(autobyte_ctx* c, const autobyte_job_stats* jobs, const autobyte_grid* grid,
                                     const int32_t* cur_idx, int32_t* best_idx, float* best_score,
                                     float* cur_score) {
  NvtxRange nvtx_range("autobyte_argmax_host");
  if (!c) return AB_E_INVALID;
  if (autobyte_status ws = take_status(c)) return ws;
  autobyte_status s = check_jobs_host(c, jobs);
  if (s != AB_OK) return s;
  if ((s = check_grid_host(c, grid)) != AB_OK) return s;
  if (!best_idx || !best_score) return fail(c, AB_E_INVALID, "best_idx / best_score is NULL");
  DeviceGuard guard(c->device);
  const int J = jobs->J;
  const size_t nT = (size_t)J * jobs->l_max * kNMax;
  AB_CUDA(c, c->sT.ensure(nT)); AB_CUDA(c, c->sBd.ensure((size_t)J * kNMax)); AB_CUDA(c, c->sBu.ensure((size_t)J * kNMax));
  AB_CUDA(c, c->sN.ensure(J)); AB_CUDA(c, c->sL.ensure(J)); AB_CUDA(c, c->sM.ensure(J)); AB_CUDA(c, c->sArc.ensure(J));
  AB_CUDA(c, c->sSp.ensure(grid->P)); AB_CUDA(c, c->sSc.ensure(grid->Q));
  AB_CUDA(c, c->rIdx.ensure(J)); AB_CUDA(c, c->rScore.ensure(J)); AB_CUDA(c, c->rCur.ensure(J));
  if (cur_idx) AB_CUDA(c, c->sCur.ensure(J));
  auto h2d = [&](void* d, const void* h, size_t bytes) { return cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, c->stream); };
  autobyte_job_stats dj{};
  AB_CUDA(c, stage_jobs_host(c, jobs, &dj));
  // the grid is read once (K0): in place when page-locked; current configs (read per tile by K2) are copied
  const void* sp_h = host_in_place(c, grid->partition_bytes);
  const void* sc_h = host_in_place(c, grid->credit_mult);
  if (!sp_h) AB_CUDA(c, h2d(c->sSp.ptr, grid->partition_bytes, (size_t)grid->P * 8));
  if (!sc_h) AB_CUDA(c, h2d(c->sSc.ptr, grid->credit_mult, (size_t)grid->Q * 4));
  if (cur_idx) AB_CUDA(c, h2d(c->sCur.ptr, cur_idx, (size_t)J * 4));
  autobyte_grid dg = *grid;
  dg.partition_bytes = sp_h ? static_cast<const int64_t*>(sp_h) : reinterpret_cast<const int64_t*>(c->sSp.ptr);
  dg.credit_mult = sc_h ? static_cast<const float*>(sc_h) : c->sSc.ptr;
  s = autobyte_argmax(c, &dj, &dg, cur_idx ? c->sCur.ptr : nullptr, c->rIdx.ptr, c->rScore.ptr,
                      cur_score ? c->rCur.ptr : nullptr);
  if (s != AB_OK) return s;
  auto d2h = [&](void* h, const void* d, size_t bytes) { return cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, c->stream); };
  AB_CUDA(c, d2h(best_idx, c->rIdx.ptr, (size_t)J * 4));
  AB_CUDA(c, d2h(best_score, c->rScore.ptr, (size_t)J * 4));
  if (cur_score) AB_CUDA(c, d2h(cur_score, c->rCur.ptr, (size_t)J * 4));
  AB_CUDA(c, cudaStreamSynchronize(c->stream));
  return take_status(c);
}

autobyte_status autobyte_adapt_host(autobyte_ctx* c, const autobyte_job_stats* samples, const int64_t* sp_bytes,
                                    const float* sc_mult, const float* v_obs, float lr, int32_t steps,
                                    float* loss_before) {
  NvtxRange nvtx_range("autobyte_adapt_host");
  if (!c) return AB_E_INVALID;
  if (autobyte_status ws = take_status(c)) return ws;
  autobyte_status s = check_jobs_host(c, samples);
  if (s != AB_OK) return s;
  if (!sp_bytes || !sc_mult || !v_obs) return fail(c, AB_E_INVALID, "adapt input pointer is NULL");
  DeviceGuard guard(c->device);
  const int B = samples->J;
  const size_t nT = (size_t)B * samples->l_max * kNMax;
  AB_CUDA(c, c->sT.ensure(nT)); AB_CUDA(c, c->sBd.ensure((size_t)B * kNMax)); AB_CUDA(c, c->sBu.ensure((size_t)B * kNMax));
  AB_CUDA(c, c->sN.ensure(B)); AB_CUDA(c, c->sL.ensure(B)); AB_CUDA(c, c->sM.ensure(B)); AB_CUDA(c, c->sArc.ensure(B));
  AB_CUDA(c, c->sSp.ensure(B)); AB_CUDA(c, c->sSc.ensure(B)); AB_CUDA(c, c->sV.ensure((size_t)B * kNMax));
  AB_CUDA(c, c->loss_tmp.ensure(1));
  auto h2d = [&](void* d, const void* h, size_t bytes) { return cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, c->stream); };
  autobyte_job_stats dj{};
  AB_CUDA(c, stage_jobs_host(c, samples, &dj));
  // observed configurations and speeds are read by K4 once per step: in place when page-locked
  const void* sp_h = host_in_place(c, sp_bytes);
  const void* sc_h = host_in_place(c, sc_mult);
  const void* v_h = host_in_place(c, v_obs);
  if (!sp_h) AB_CUDA(c, h2d(c->sSp.ptr, sp_bytes, (size_t)B * 8));
  if (!sc_h) AB_CUDA(c, h2d(c->sSc.ptr, sc_mult, (size_t)B * 4));
  if (!v_h) AB_CUDA(c, h2d(c->sV.ptr, v_obs, (size_t)B * kNMax * 4));
  s = autobyte_adapt(c, &dj, sp_h ? static_cast<const int64_t*>(sp_h) : reinterpret_cast<const int64_t*>(c->sSp.ptr),
                     sc_h ? static_cast<const float*>(sc_h) : c->sSc.ptr,
                     v_h ? static_cast<const float*>(v_h) : c->sV.ptr, lr, steps,
                     loss_before ? c->loss_tmp.ptr : nullptr);
  if (s != AB_OK) return s;
  if (loss_before)
    AB_CUDA(c, cudaMemcpyAsync(loss_before, c->loss_tmp.ptr, 4, cudaMemcpyDeviceToHost, c->stream));
  AB_CUDA(c, cudaStreamSynchronize(c->stream));
  return take_status(c);
}

autobyte_status autobyte_get_weights(autobyte_ctx* c, void* host_blob, size_t bytes) {
  if (!c || !host_blob) return AB_E_INVALID;
  size_t want = 0;
  autobyte_blob_bytes(&c->desc, &want);
  if (bytes != want) return fail(c, AB_E_SHAPE, "blob size mismatch");
  DeviceGuard guard(c->device);
  uint8_t* b = static_cast<uint8_t*>(host_blob);
  std::memcpy(b, AUTOBYTE_BLOB_MAGIC, 4);
  const uint32_t ver = AUTOBYTE_BLOB_VERSION;
  std::memcpy(b + 4, &ver, 4);
  std::memcpy(b + 8, &c->desc, sizeof(c->desc));
  const uint32_t n_arrays = 12 + 2 * (c->desc.hidden_layers - 1) + 2, zero = 0;
  std::memcpy(b + 40, &n_arrays, 4);
  std::memcpy(b + 44, &zero, 4);
  AB_CUDA(c, cudaMemcpyAsync(b + kBlobHeader, c->params.ptr, c->off.total * sizeof(float), cudaMemcpyDeviceToHost,
                             c->stream));
  AB_CUDA(c, cudaStreamSynchronize(c->stream));
  return take_status(c);
}

autobyte_status autobyte_set_profiling(autobyte_ctx* c, int enable) {
  if (!c) return AB_E_INVALID;
  c->profiling = enable != 0;
  return AB_OK;
}

autobyte_status autobyte_get_profile(autobyte_ctx* c, autobyte_profile* out) {
  if (!c || !out) return AB_E_INVALID;
  DeviceGuard guard(c->device);
  AB_CUDA(c, cudaStreamSynchronize(c->stream));
  for (auto& p : c->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.second.first, p.second.second) == cudaSuccess) c->ms[p.first] += ms;
    cudaEventDestroy(p.second.first);
    cudaEventDestroy(p.second.second);
  }
  c->pending.clear();
  out->encode_ms = c->ms[K_ENCODE]; out->encode_launches = c->launches[K_ENCODE];
  out->score_ms = c->ms[K_SCORE]; out->score_launches = c->launches[K_SCORE];
  out->finalize_ms = c->ms[K_FINALIZE]; out->finalize_launches = c->launches[K_FINALIZE];
  out->exchange_ms = c->ms[K_EXCHANGE]; out->exchange_calls = c->launches[K_EXCHANGE];
  out->adapt_ms = c->ms[K_ADAPT]; out->adapt_launches = c->launches[K_ADAPT];
  out->pack_ms = c->ms[K_PACK]; out->pack_launches = c->launches[K_PACK];
  out->other_launches = c->launches[K_OTHER];
  out->score_pairs = c->score_pairs;
  return AB_OK;
}

autobyte_status autobyte_reset_profile(autobyte_ctx* c) {
  if (!c) return AB_E_INVALID;
  autobyte_profile tmp;
  autobyte_status s = autobyte_get_profile(c, &tmp);   // drains pending events
  if (s != AB_OK) return s;
  for (int k = 0; k < K_N; ++k) { c->ms[k] = 0.0; c->launches[k] = 0; }
  c->score_pairs = 0.0;
  return AB_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------------------------
namespace ab {
ParamOffsets make_offsets(const autobyte_net_desc& d) {
  ParamOffsets o{};
  int64_t p = 0;
  auto take = [&](int64_t n) { int64_t r = p; p += n; return r; };
  const int64_t te = d.type_embed_dim, de = d.embed_dim, h = d.lstm_hidden, H = d.hidden_width, nm = d.n_max;
  o.E_m = take((int64_t)d.n_model_types * te);
  o.E_arc = take((int64_t)d.n_arch_types * te);
  o.W_e = take(de * nm);
  o.b_e = take(de);
  o.l1Wx = take(4 * h * de);
  o.l1Wh = take(4 * h * h);
  o.l1b = take(4 * h);
  o.l2Wx = take(4 * h * h);
  o.l2Wh = take(4 * h * h);
  o.l2b = take(4 * h);
  o.W[1] = take(H * kZDim);
  o.b[1] = take(H);
  for (int k = 2; k <= d.hidden_layers; ++k) {
    o.W[k] = take(H * H);
    o.b[k] = take(H);
  }
  o.W_o = take(nm * H);
  o.b_o = take(nm);
  o.total = p;
  return o;
}
}  // namespace ab
