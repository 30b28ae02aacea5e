// internal.h — library-private declarations shared by the .cu files of libautobyte.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/autobyte.h"

namespace ab {

constexpr int kNMax = 16;
constexpr int kEmbed = 16;
constexpr int kLstm = 32;
constexpr int kTypeEmbed = 8;
constexpr int kXDim = AUTOBYTE_X_DIM;          // 82
constexpr int kZDim = AUTOBYTE_X_DIM + 2;      // 84 = [x | u]
constexpr int kMaxHidden = 8;
constexpr int kTileM = 128;                    // candidates per tcgen05 tile (TMEM lanes)
constexpr int kEncStash = kEmbed + 12 * kLstm; // floats stashed per job and layer step (e, 2 x [i f g o c h])

// Offsets (in floats) of every parameter inside the fp32 master buffer (= blob payload order).
// n / d for 0 <= n < 2^31 as a multiply-shift (Granlund-Montgomery with p = 31 + ceil(log2 d),
// mul = ceil(2^p / d); exact for every n < 2^31, checked exhaustively at the edges in
// tests/test_boundary.py::test_fastdiv_reference): the kernels' per-tile index splits.
struct FastDiv {
  uint32_t d, mul, shr;
};
inline void make_fastdiv(uint32_t d, uint32_t* mul, uint32_t* shr) {
  if (d <= 1) { *mul = 0; *shr = 0; return; }
  int l = 0;
  while ((1ull << l) < d) ++l;   // ceil(log2 d)
  const int p = 31 + l;
  *mul = static_cast<uint32_t>(((1ull << p) + d - 1) / d);
  *shr = static_cast<uint32_t>(p - 32);
}
#ifdef __CUDACC__
__device__ __forceinline__ int fdiv(int n, const FastDiv& f) {
  return f.d == 1 ? n : static_cast<int>(__umulhi(static_cast<uint32_t>(n), f.mul) >> f.shr);
}
#endif

struct ParamOffsets {
  int64_t E_m, E_arc, W_e, b_e;
  int64_t l1Wx, l1Wh, l1b, l2Wx, l2Wh, l2b;
  int64_t W[kMaxHidden + 1];   // W[1] = W1 [H][84]; W[k] = W_k [H][H], k = 2..L
  int64_t b[kMaxHidden + 1];
  int64_t W_o, b_o;
  int64_t total;
};
ParamOffsets make_offsets(const autobyte_net_desc& d);

// Device status word codes (ptx.cuh): what a watchdog records instead of trapping.
enum : int {
  kStatusPipeline = 1,   // an mbarrier / grid-barrier wait inside one kernel exceeded ~2^36 cycles
  kStatusPeerKeys = 2,   // the NVLink key exchange waited longer than AUTOBYTE_PEER_TIMEOUT_S for a peer
  kStatusPeerX = 3,      // the NVLink x all-gather waited longer than AUTOBYTE_PEER_TIMEOUT_S for a peer
};

// ---------------------------------------------------------------- kernel parameter blocks
struct EncodeParams {
  int J, l_max, H;
  int j_begin, j_end;  // K1a job range (K1b always covers [0, J))
  const float* T; const float* B_d; const float* B_u;
  const int32_t* n; const int32_t* l; const int32_t* m; const int32_t* arc;
  const float* params; ParamOffsets off;
  float* x_out;        // [J][82] (K1a writes rows of its range, K1b reads all rows)
  // per-job vectors, row stride jv floats (K2 reads one contiguous block [a | w | beta] per job)
  long long jv;
  float* a_out;        // [J][jv]: W1x x + b1 in [0, H), or null
  float* what_out;     // [J][jv]: mean of the first n rows of W_o, or null
  float* beta_out;     // [J][jv]: mean of the first n entries of b_o, or null
  unsigned long long* keys;      // [J] reset to 0, or null
  unsigned long long* cur_keys;  // [J] reset to 0, or null
  float* stash;        // [J][l_max][kEncStash] forward states for encoder fine-tuning, or null
  // candidate-grid axes (a-1, R#8), formed by K1b (or K1s when it projects) when up_out != null:
  // up_out[p] = (log2 S_p[p] - 21) / 8, uc_out[q] = (S_c[q] - 8.5) / 8, in double, rounded once
  int P, Q;
  const long long* S_p; const float* S_c;
  float* up_out; float* uc_out;
  int fuse_project;    // K1s: also K1b's per-job projections (a, w, beta, key reset) for its jobs
  // G > 1 with the peer-memory window: K1a also stores its x rows into every rank's window
  // (xg[r], row j at xg[r] + j*82; xg[rank] == x_out) and its last CTA raises xflag[r][rank] = epoch
  int xG, xrank;
  float* xg[8];
  unsigned long long* xflag[8];
  unsigned int* xcounter;
  unsigned long long xepoch;
};

struct alignas(64) ScoreParams {
  CUtensorMap wmap;             // 2-D view of wpack (rows of 128 B) for the CTA-pair TMA loads
  int cta_group;                // 1: one CTA per tile (M = 128); 2: CTA pairs (M = 256)
  int precision3;               // 1: fp32-accuracy path (bf16 hi/lo split, 3 products per K step)
  int J, H, G;                  // G = L - 1 tensor-core layers
  int P, Q;
  long long c_begin, c_end;     // shard [begin, end)
  int tiles_per_job;
  long long n_tiles;            // < 2^31 (like c_end): the kernel indexes tiles in 32 bits
  uint32_t tpj_mul, tpj_shr;    // FastDiv of tiles_per_job and of Q (make_fastdiv)
  uint32_t q_mul, q_shr;
  const long long* S_p;         // [P]
  const float* S_c;             // [Q]
  const float* params;          // fp32 masters (W1's u-columns, biases)
  ParamOffsets off;
  const float* jobvec;          // [J][2H+4]: a_j | w_j | beta_j, 0, 0, 0  (K1)
  const float* up;              // [P] partition-size encodings (R#8; K1b / K1s)
  const float* uc;              // [Q] credit-size encodings
  const __nv_bfloat16* wpack;   // packed bf16 W_2..W_L (see pack_weights)
  unsigned long long* keys;     // [J]
  unsigned long long* cur_keys; // [J]
  const int32_t* cur_idx;       // [J] or null
  float* scores;                // [J][c_end - c_begin] or null
  uint32_t* spill;              // fp32 path at H = 512: [grid][128][spill_u32] activation scratch
  // single-rank argmax: the last CTA to finish decodes the keys (K5 folded into K2)
  int finalize;
  unsigned int* done;           // CTA completion counter (zero between calls)
  int32_t* best_idx; float* best_score; float* cur_score;
};

struct alignas(64) AdaptParams {
  // K4s: tensor maps of W_k (k = 2..L) as fp32 [H rows][H cols], box = [min(H, 256) rows][H/16 cols]
  // (one CTA's column slice per 256 rows; adapt_small.cu)
  CUtensorMap wcol[kMaxHidden + 1];
  int B, H, L, steps;
  float lr;
  const float* x;          // [B][82] frozen encoder output
  const long long* S_p;    // [B]
  const float* S_c;        // [B]
  const float* v_obs;      // [B][16]
  const int32_t* n;        // [B]
  float* params;           // fp32 masters (updated in place)
  ParamOffsets off;
  float* ws;               // workspace (see adapt.cu)
  float* grads;            // [head params] gradient buffer
  float* loss_before;      // [1] or null
  float* losses;           // [steps] or null: mean Eq. 2 norm before each step
  unsigned int* barrier;   // grid barrier: one 64-bit arrival counter (2 words, never reset)
  // optimiser (autobyte_train; autobyte_adapt = SGD with no state)
  int opt;                 // AB_OPT_SGD / AB_OPT_ADAM
  float beta1, beta2, eps;
  long long t0;            // Adam steps taken before this launch
  float* m;                // Adam first moments (blob layout, head part used) or null
  float* v;                // Adam second moments
  float* dz_out;           // [B][84] d objective / d [x | u] (encoder fine-tuning) or null
  const int32_t* idx;      // [steps][B] dataset rows of each step's minibatch (train_epoch) or null:
                           // then x / S_p / S_c / v_obs / n are the whole dataset's arrays
  // K4s refreshes the bf16 shadows of W_2..W_L as it updates them (no separate pack launch)
  __nv_bfloat16* wpack;    // packed shadows (kWeightReplicas copies of packed_weight_elems)
  int planes;              // 1 = bf16, 2 = hi/lo (fp32 path)
};

// ---------------------------------------------------------------- launches (return cudaError_t)
// K1a / K1s; *projected = true when K1s also did K1b's work (p.fuse_project and the latency kernel ran)
cudaError_t launch_encode_lstm(const EncodeParams& p, int num_sms, cudaStream_t s, bool* projected = nullptr);
cudaError_t launch_project(const EncodeParams& p, cudaStream_t s);                    // K1b
cudaError_t launch_score(const ScoreParams& p, int num_sms, cudaStream_t s);
cudaError_t launch_grid_axes(const EncodeParams& p, cudaStream_t s);   // K0: only when P + Q is large
constexpr int kFusedAxes = 8192;   // P + Q up to this: the axes are formed inside K1b / K1s
cudaError_t launch_trigger(int J, const int32_t* best_idx, const float* best_score, const int32_t* cur_idx,
                           const float* cur_score, const float* v_obs, float gain, float drift, int32_t* action,
                           cudaStream_t s);
cudaError_t launch_finalize(int J, int G, long long stride, const unsigned long long* keys,
                            const unsigned long long* cur_keys, int32_t* best_idx, float* best_score,
                            float* cur_score, cudaStream_t s);
// K3+K5 over NVLink peer memory (exchange.cu): windows are [kPeerFlagWords flags | 2][G][cap2] u64
constexpr int kPeerFlagWords = 64;   // [0, 32): key-exchange flags, [32, 64): x all-gather flags
constexpr int kPeerXFlags = 32;
constexpr int kMaxPeers = 8;
struct PeerExchangeParams {
  unsigned long long* win[kMaxPeers];   // every rank's window (IPC-mapped; win[rank] is the own one)
  const unsigned long long* keys;       // [2J] this rank's keys (K2)
  unsigned int* counter;                // per-rank block counter (zero between calls)
  int32_t* best_idx; float* best_score; float* cur_score;
  unsigned long long* epoch;            // device counter: last completed epoch (the kernel advances it)
  unsigned long long timeout_ns;        // peer wait limit (0 = wait forever)
  long long cap2;                       // slot stride (u64), >= 2J
  int J, G, rank;
};
cudaError_t launch_peer_exchange(const PeerExchangeParams& p, int num_sms, cudaStream_t s, bool cooperative = true);
// one warp waits until flags[r] >= epoch for r < G (stream order then holds the consumers back)
cudaError_t launch_peer_wait(const unsigned long long* flags, int G, unsigned long long epoch,
                             unsigned long long timeout_ns, cudaStream_t s);
cudaError_t launch_pack(const float* params, const ParamOffsets& off, int H, int L, int planes,
                        __nv_bfloat16* wpack, cudaStream_t s);
// elements of one replica of the packed bf16 shadows of W_2..W_L
__host__ __device__ inline size_t packed_weight_elems(int H, int L, int planes) {
  return (size_t)(L > 1 ? L - 1 : 0) * H * H * planes;
}
// rows per packed tile = N of K2's accumulator chunks (ScoreCfg::NCH)
__host__ __device__ inline int packed_weight_nch(int H, int planes) {
  return planes == 2 ? (H == 512 ? 128 : 64) : (H >= 128 ? 128 : H);
}
// Element index in the packed bf16 shadow (one replica) of W_{g+2}[n][k], plane 0 = hi, 1 = lo:
// tile ((g*NQ + n/NCH)*NKB + k/64)*planes + plane of NCH rows x 64 (UMMA SW128 K-major: 16-byte
// chunk j of row r stored at chunk j ^ (r % 8)) — the inverse of pack_kernel's walk (score.cu).
__host__ __device__ inline size_t packed_weight_index(int H, int planes, int nch, int g, int n, int k, int plane) {
  const int nq = H / nch, nkb = H / 64;
  const int q = n / nch, nl = n - q * nch, b = k >> 6, kl = k & 63;
  const int slot = ((((kl >> 3) ^ (nl & 7)) << 3) | (kl & 7));
  const size_t tile = (((size_t)g * nq + q) * nkb + b) * planes + plane;
  return tile * (size_t)nch * 64 + (size_t)nl * 64 + slot;
}
#ifndef AB_WREP
#define AB_WREP 1   // L2 replicas of the packed bf16 weights (CTA pair i streams replica i % AB_WREP)
#endif
constexpr int kWeightReplicas = AB_WREP;
cudaError_t launch_adapt(const AdaptParams& p, int num_sms, cudaStream_t s, int* grid_used);
// K4s (adapt_small.cu): one thread-block cluster, for minibatches of at most kAdaptSmallMaxB samples
// (no encoder gradient, no dataset index); cudaErrorNotSupported otherwise (run K4)
constexpr int kAdaptSmallMaxB = 16;
cudaError_t launch_adapt_small(const AdaptParams& p, cudaStream_t s);
cudaError_t launch_encoder_bwd(const EncodeParams& p, const float* dX, int ldx, float* partial, int num_sms,
                               int* nparts, cudaStream_t s);                                   // K8
cudaError_t launch_encoder_update(const EncodeParams& p, const float* dX, int ldx, int B, const float* partial,
                                  int nparts, int opt, float lr, float beta1, float beta2, float eps, long long t,
                                  float* m, float* v, cudaStream_t s);                          // K9
int encoder_bwd_parts(int B, int num_sms);
cudaError_t launch_topk(int J, long long C, const float* scores, long long c_begin, int k, unsigned long long* out,
                        cudaStream_t s);                                                       // K6
cudaError_t launch_topk_merge(int J, int G, int k, const unsigned long long* lists, int32_t* idx, float* score,
                              cudaStream_t s);                                                 // K7
size_t adapt_ws_floats(int B, int H, int L);
constexpr int kAdaptSplitK = 4;   // must match adapt.cu kSplitK (gradient partial buffers)
cudaError_t launch_check(const autobyte_job_stats& jobs, int n_max, int n_model, int n_arch,
                         int* flag, cudaStream_t s);
cudaError_t launch_check_grid(const autobyte_grid& g, int* flag, cudaStream_t s);
bool make_weight_tmap(CUtensorMap* map, const __nv_bfloat16* wpack, int H, int L, int planes);
// K4s column-slice maps over the fp32 masters (score.cu, next to the other tensor-map encoder)
bool make_column_tmaps(CUtensorMap* maps, const float* params, const ParamOffsets& off, int H, int L);
// device status word (ptx.cuh): each translation unit's copy of the pointer, set per device
cudaError_t set_status_adapt(int* p);
cudaError_t set_status_encode(int* p);
cudaError_t set_status_encoder_bwd(int* p);
cudaError_t set_status_exchange(int* p);
cudaError_t set_status_score(int* p);
cudaError_t set_status_topk(int* p);
cudaError_t set_status_adapt_small(int* p);
cudaError_t set_status_simulate(int* p);
// K10 (simulate.cu): one ByteScheduler iteration per (job, candidate) of the shard (NEXT 3)
cudaError_t launch_simulate(const autobyte_job_stats& jobs, const float* layer_bytes, const float* fwd_ms,
                            const autobyte_grid& g, double alpha_ms, double delta_ms, double* iter_ms, cudaStream_t s);
size_t simulate_smem_bytes(int l_max);

}  // namespace ab
