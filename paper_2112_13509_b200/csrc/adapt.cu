// adapt.cu — K4: fused online adaptation (forward with stash, backward, SGD) in ONE cooperative
// persistent kernel ("offline training, online adapting ... transfer learning";
// P:438 triggered when prediction error > 10%; R#12 objective, R#13 head-only plain SGD).
//
// Per step, phases separated by a grid-wide barrier:
//   F_k   H_k = ReLU(H_{k-1} W_k^T + b_k), k = 1..L (H_0 = Z = [x | u])      3xTF32 tensor-core tiles
//   OUT   R = mask_b (H_L W_o^T + b_o - V_bar) / B        (dV of the objective; one warp per row)
//   BO    dW_o = R^T H_L, db_o = colsum R, D_L = (R W_o) * [H_L > 0]
//   Bk    dW_k = D_k^T H_{k-1}, db_k = colsum D_k, D_{k-1} = (D_k W_k) * [H_{k-1} > 0]  (pre-update W_k)
//         + SGD of the layer above (its gradient is complete and no later phase reads it)
//   SGD   W1, b1 (after B1)   (SGD or Adam, see update_range)
// Every output element is produced by exactly one thread with a fixed summation order, so the
// update is deterministic and replicas on different GPUs stay bit-identical without traffic.
// The work is ~3x a B-row forward (5 GFLOP at B=1024, 4x512): latency-bound, << 1% of a C5 step.
// Every GEMM runs on tcgen05 (kind::tf32, accumulators in TMEM) with 3xTF32 split operands
// (big*big + big*small + small*big, ~2^-20 relative), which keeps the gradient well inside the
// parity tolerance (K4): a dedicated issuer warp, 8 worker warps that stage, split
// and run the epilogue (gemm_tile).
#include <climits>
#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

namespace ab {

#ifdef AB_STATS
__device__ long long g_adapt_trace[2][64][4];   // [worker t0 | issuer][slice][stamp] of one traced tile
__device__ int g_adapt_trace_on;
#define AB_TR(who, it, i) do { if (trace && (it) < 64) g_adapt_trace[who][it][i] = clock64(); } while (0)
#else
#define AB_TR(who, it, i) do { } while (0)
#endif
constexpr int kWorkThreads = 256;                 // warps 0-7: staging, operand split, epilogue, SIMT phases
constexpr int kIssuerWarp = kWorkThreads / 32;    // warp 8: tcgen05.mma issuer
constexpr int kAdaptThreads = kWorkThreads + 32;
constexpr uint32_t kWorkBar = 1;                  // named barrier of the 256 worker threads
constexpr int kTM = 128, kTK = 32;   // tcgen05 tile: M = 128 TMEM lanes x N (TileCfg), K slices of 32 tf32
constexpr int kSplitK = kAdaptSplitK;   // K = B splits of the weight-gradient GEMMs (partials in grads[kSplitK][total])
constexpr int kNAcc = 4;                // TMEM accumulators per tile (K slices round-robin, summed in fp32)

struct Gemm {
  int M, N, K;
  const float* A; long long lam, lak;    // A(m, k) = A[m*lam + k*lak]; lak == 1 or lam == 1
  const float* Bm; long long lbk, lbn;   // B(k, n) = Bm[k*lbk + n*lbn]; lbk == 1 or lbn == 1
  float* C; long long ldc;               // C[m*ldc + n]
  int mode;                              // 0: ReLU(acc + bias[n]); 1: acc * [mask(m,n) > 0]; 2: acc
  const float* bias;
  const float* mask; long long ldmask;
  int ksplit;                            // split-K count (mode 2 only): partial s -> C + s*cpart
  long long cpart;
  template <int TN>
  __device__ int tiles() const { return ((M + kTM - 1) / kTM) * ((N + TN - 1) / TN) * (ksplit > 1 ? ksplit : 1); }
};

// Shared memory (dynamic, 1 KB aligned):
//   planes  kBufs buffers x {A big, A small [128][32] tf32, B big, B small [TN][32] tf32}, UMMA
//           SW128 K-major (row r of an 8-row 1 KB atom at 128 r bytes, 16-byte chunk j at j ^ (r % 8))
//   raw     kStages x {A, B} fp32 slices as copied from global in their own orientation:
//           K-contiguous [rows][kTK + 4] or MN-contiguous [kTK][rows + 8]
// Two tile widths: N = 64 with 3 plane buffers and a 2-deep raw ring for small batches (online
// adaptation: more tiles per phase), N = 128 with 2 buffers and a 2-deep ring for large batches
// (offline training: half the MMAs per FLOP, 8.2 vs 7.2 M samples/s at B = 32768).
template <int TN>
struct TileCfg {
#ifndef AB_ADAPT_STAGES64
#define AB_ADAPT_STAGES64 2
#endif
  // cp.async depth of the raw slices. Depth 3 vs 4 measured the same (a slice's data lands long
  // before it is split, K-slice trace), so N = 64 tiles spend the shared memory on a third plane
  // buffer instead and keep a 2-deep ring (prefetch distance one slice, ~1.5k cycles)
  static constexpr int kStages = TN == 64 ? AB_ADAPT_STAGES64 : 2;
  static constexpr int kRawA = (kTM * (kTK + 4) > kTK * (kTM + 8)) ? kTM * (kTK + 4) : kTK * (kTM + 8);   // floats
  static constexpr int kRawB = (TN * (kTK + 4) > kTK * (TN + 8)) ? TN * (kTK + 4) : kTK * (TN + 8);
  static constexpr int kPlaneA = kTM * kTK * 4, kPlaneB = TN * kTK * 4;               // bytes
  static constexpr int kPlaneBuf = 2 * kPlaneA + 2 * kPlaneB;                          // one buffer
#ifndef AB_ADAPT_BUFS64
#define AB_ADAPT_BUFS64 3
#endif
  // plane buffers: with two, splitting slice i+1 waited for the MMAs of slice i-1 to COMPLETE and
  // the split and the MMA chain ran back to back (~1.6k cycles per slice); a third buffer lets the
  // split run one slice further ahead (N = 64 only: three N = 128 buffers do not fit)
  static constexpr int kBufs = TN == 64 ? AB_ADAPT_BUFS64 : 2;
  static constexpr size_t kRawOff = kBufs * (size_t)kPlaneBuf;
  static constexpr size_t kSmem = kRawOff + sizeof(float) * kStages * (kRawA + kRawB);
  static constexpr uint32_t kIdesc = umma_idesc_tf32(kTM, TN);
};
constexpr int kSK = kTK + 4;
constexpr size_t kAdaptSmemBytes =
    1024 + (TileCfg<64>::kSmem > TileCfg<128>::kSmem ? TileCfg<64>::kSmem : TileCfg<128>::kSmem);
static_assert(kAdaptSmemBytes + 4096 <= 232448, "dynamic + static shared memory of K4 exceeds 227 KB");
constexpr uint32_t kTmemCols = kNAcc * 128;   // 512: four accumulators of the widest tile
constexpr int kBigBatch = 4096;               // B >= this: N = 128 tiles

__device__ __forceinline__ void cp_async16(float* smem_dst, const float* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem_dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// x ~ big + small with both parts exact tf32 values (10 explicit mantissa bits): big = x with its
// low 13 mantissa bits cleared (truncation), small = the exact fp32 remainder x - big, truncated the
// same way. The 3xTF32 product big*big + big*small + small*big then carries ~2^-20 relative error
// (|small| < 2^-10 |x|, small's own truncation < 2^-10 |small|; small*small is dropped). Two LOP3 and
// one FADD per element: cvt.rna.tf32 runs at a fraction of the ALU rate, and with it the split was
// ~60 % of every K slice (tools/adapt_phases.py slice trace: ~900 of ~1600 cycles).
#ifndef AB_TF32_CVT
__device__ __forceinline__ void split_tf32(float x, float& big, float& small) {
  const float b = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  big = b;
  small = __uint_as_float(__float_as_uint(x - b) & 0xFFFFE000u);
}
#else   // the round-to-nearest split (timing comparison)
__device__ __forceinline__ void split_tf32(float x, float& big, float& small) {
  uint32_t b, sm;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(b) : "f"(x));
  const float r = x - __uint_as_float(b);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(sm) : "f"(r));
  big = __uint_as_float(b);
  small = __uint_as_float(sm);
}
#endif

// Stage one ROWS x kTK slice of an operand: X(mn, k) = base[mn*lmn + k*lk] for mn in [mn0, mn0+ROWS),
// k in [k0, k0+kTK), zero-filled outside [0, MN) x [k0, kend). 16-byte vectors.
template <int ROWS>
__device__ __forceinline__ void stage_slice(float* dst, const float* base, long long lmn, long long lk, int MN,
                                            int mn0, int k0, int kend) {
  constexpr int kVec = ROWS * kTK / 4 / kWorkThreads;   // vectors per thread
#pragma unroll
  for (int r = 0; r < kVec; ++r) {
    const int e = threadIdx.x + r * kWorkThreads;
    if (lk == 1) {   // K-contiguous: vector (mn, 4 k)
      const int mn = e / (kTK / 4), kq = (e % (kTK / 4)) * 4;
      const bool v = mn0 + mn < MN && k0 + kq < kend;
      cp_async16(dst + mn * kSK + kq, v ? base + (long long)(mn0 + mn) * lmn + (k0 + kq) : base, v);
    } else {         // MN-contiguous: vector (k, 4 mn)
      const int k = e / (ROWS / 4), mq = (e % (ROWS / 4)) * 4;
      const bool v = k0 + k < kend && mn0 + mq < MN;
      cp_async16(dst + k * (ROWS + 8) + mq, v ? base + (long long)(k0 + k) * lk + (mn0 + mq) : base, v);
    }
  }
}

// Split a raw slice into SW128 K-major big / small planes, one 16-byte chunk (4 k) at a time.
// K-contiguous raw: thread -> (row, chunk) with the 8 threads of a row covering its 8 chunks.
// MN-contiguous raw: warp w -> chunk w, lanes -> rows (4 strided LDS per chunk, conflict-free).
template <int ROWS>
__device__ __forceinline__ void split_slice(const float* raw, bool kcontig, uint8_t* big, uint8_t* small) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // plain C++ shared-memory accesses (no asm memory clobbers), so the compiler can hoist every
  // raw load of the slice ahead of the plane stores; ordering against the tensor core comes from
  // the fence.proxy.async + mbarrier arrive that follow
  auto store = [&](int r, int j, const float4& v) {
    float4 b, sm;
    split_tf32(v.x, b.x, sm.x); split_tf32(v.y, b.y, sm.y);
    split_tf32(v.z, b.z, sm.z); split_tf32(v.w, b.w, sm.w);
    const int off = (r >> 3) * 1024 + (r & 7) * 128 + ((j ^ (r & 7)) << 4);
    *reinterpret_cast<float4*>(big + off) = b;
    *reinterpret_cast<float4*>(small + off) = sm;
  };
  if (kcontig) {
    constexpr int kN = ROWS * 8 / kWorkThreads;
    float4 v[kN];
#pragma unroll
    for (int i = 0; i < kN; ++i) {
      const int e = tid + i * kWorkThreads, r = e >> 3, j = e & 7;
      v[i] = *reinterpret_cast<const float4*>(raw + r * kSK + 4 * j);
    }
#pragma unroll
    for (int i = 0; i < kN; ++i) {
      const int e = tid + i * kWorkThreads;
      store(e >> 3, e & 7, v[i]);
    }
  } else {
    constexpr int kN = ROWS / 32;
    float4 v[kN];
#pragma unroll
    for (int i = 0; i < kN; ++i) {
      const int r = lane + 32 * i, j = w;
      v[i].x = raw[(4 * j) * (ROWS + 8) + r];
      v[i].y = raw[(4 * j + 1) * (ROWS + 8) + r];
      v[i].z = raw[(4 * j + 2) * (ROWS + 8) + r];
      v[i].w = raw[(4 * j + 3) * (ROWS + 8) + r];
    }
#pragma unroll
    for (int i = 0; i < kN; ++i) store(lane + 32 * i, w, v[i]);
  }
}

// Per-CTA tensor-core state that persists across tiles and phases (each thread keeps the counters
// of its own role; mbarrier parities are derived from them).
struct TcState {
  uint32_t tmem;         // kTmemCols fp32 accumulator columns
  uint64_t* full;        // [kMaxBufs]: the 8 worker warps have written plane buffer b
  uint64_t* empty;       // [kMaxBufs]: the MMAs that read plane buffer b have completed (tcgen05.commit)
  uint64_t* acc_free;    // the epilogue has read the accumulators of the last MMA tile
  // plane buffers are used round-robin over all tiles of the launch: slice n (counted from the
  // launch start) goes to buffer n % kBufs as its (n / kBufs)-th fill, so the phase bookkeeping is
  // one counter per role (per-buffer counters indexed by a rotating b lived in local memory: a
  // load and a store per K slice on both the workers' and the issuer's critical path)
  uint32_t wsl;          // workers: slices filled
  uint32_t isl;          // issuer: slices consumed
  uint32_t tiles;        // issuer: MMA tiles issued
};

// One 128 x 128 output tile (or one K range of it for split-K) on tcgen05, 3xTF32. Per K slice of
// 32: the CTA stages the raw fp32 operands (cp.async, kStages deep), splits them once into tf32
// big/small SW128 planes (double-buffered, so the split of slice i+1 overlaps the MMAs of slice i),
// and one elected thread issues 4 K-steps x 3 products of M128 N128 K8 into TMEM accumulator
// (slice % 4); tcgen05.commit frees the plane buffer. The epilogue sums the 4 accumulators in
// fixed order with IEEE adds (long accumulations inside the tensor core lose ~1e-3 on the
// gradients) and applies the mode. Deterministic: fixed issue and summation order.
template <int TN>
__device__ void gemm_tile(const Gemm& g, int work, uint8_t* smem, TcState& ts) {
  using T = TileCfg<TN>;
  constexpr int kStages = T::kStages, kRawA = T::kRawA, kRawB = T::kRawB;
  constexpr int kPlaneA = T::kPlaneA, kPlaneB = T::kPlaneB, kPlaneBuf = T::kPlaneBuf, kBufs = T::kBufs;
  constexpr uint32_t kIdesc = T::kIdesc;
  const int tiles_n = (g.N + TN - 1) / TN;
  const int tiles_mn = ((g.M + kTM - 1) / kTM) * tiles_n;
  const int split = g.ksplit > 1 ? work / tiles_mn : 0;
  const int tile = work % tiles_mn;
  const int m0 = (tile / tiles_n) * kTM, n0 = (tile % tiles_n) * TN;
  int kbeg = 0, kend = g.K;
  if (g.ksplit > 1) {
    const int chunk = ((g.K + g.ksplit - 1) / g.ksplit + kTK - 1) / kTK * kTK;
    kbeg = split * chunk;
    kend = min(g.K, kbeg + chunk);
  }
  const int nk = kend > kbeg ? (kend - kbeg + kTK - 1) / kTK : 0;
  const uint32_t pbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef AB_STATS
  // armed with (mode + 1) | (block << 8): the first tile of that mode with >= 8 slices on that block
  const int arm = g_adapt_trace_on;
  const bool trace_tile = arm && blockIdx.x == (arm >> 8) && nk >= 8 && g.mode == (arm & 255) - 1;
  __syncthreads();   // every thread has read the arm word before thread 0 clears it
  if (trace_tile && threadIdx.x == 0) g_adapt_trace_on = 0;
  const bool trace = trace_tile && (threadIdx.x == 0 || (warp == kIssuerWarp && lane == 0));
#endif
  if (warp == kIssuerWarp) {
    // ---------------- MMA issuer: per slice, wait for the split planes, issue 4 K-steps x 3
    // products into accumulator (slice % 4), commit -> empty[b] frees the buffer
    if (nk == 0) return;
    if (ts.tiles > 0) mbar_wait(ts.acc_free, (ts.tiles - 1) & 1);   // previous tile's epilogue has read TMEM
    for (int it = 0; it < nk; ++it) {
      const uint32_t n = ts.isl + it;
      const int b = static_cast<int>(n % kBufs);
      AB_TR(1, it, 0);
      mbar_wait(&ts.full[b], (n / kBufs) & 1u);
      AB_TR(1, it, 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t buf = pbase + b * kPlaneBuf;
        const uint64_t ab = umma_desc_sw128(buf), as = umma_desc_sw128(buf + kPlaneA);
        const uint64_t bb = umma_desc_sw128(buf + 2 * kPlaneA), bs = umma_desc_sw128(buf + 2 * kPlaneA + kPlaneB);
        const uint32_t d = ts.tmem + static_cast<uint32_t>((it % kNAcc) * TN);
        const uint32_t first = it < kNAcc ? 1u : 0u;   // first slice of this accumulator in the tile
#pragma unroll
        for (int ks = 0; ks < kTK / 8; ++ks) {          // K = 8 tf32 = 32 bytes per step
          const uint64_t o = static_cast<uint64_t>(2 * ks);
          umma_ss_tf32(d, as + o, bb + o, kIdesc, (first && ks == 0) ? 0u : 1u);   // small terms first
          umma_ss_tf32(d, ab + o, bs + o, kIdesc, 1u);
          umma_ss_tf32(d, ab + o, bb + o, kIdesc, 1u);
        }
        umma_commit(&ts.empty[b]);
      }
      __syncwarp();
      AB_TR(1, it, 2);
    }
    ts.isl += nk;
    ++ts.tiles;
    return;
  }
  // ---------------- workers (warps 0-7): stage raw slices, split into planes, epilogue
  const bool a_kc = g.lak == 1, b_kc = g.lbk == 1;
  float* raw = reinterpret_cast<float*>(smem + T::kRawOff);
  auto rawA = [&](int st) { return raw + st * (kRawA + kRawB); };
  auto rawB = [&](int st) { return raw + st * (kRawA + kRawB) + kRawA; };
  auto issue = [&](int it) {
    if (it < nk) {
      const int k0 = kbeg + it * kTK, st = it % kStages;
      stage_slice<kTM>(rawA(st), g.A, g.lam, g.lak, g.M, m0, k0, kend);
      stage_slice<TN>(rawB(st), g.Bm, g.lbn, g.lbk, g.N, n0, k0, kend);
    }
    cp_async_commit();   // (empty groups keep the wait arithmetic uniform)
  };
  named_bar_sync(kWorkBar, kWorkThreads);   // the raw ring may still be read by the previous tile's split
#pragma unroll
  for (int i = 0; i < kStages - 1; ++i) issue(i);
  for (int it = 0; it < nk; ++it) {
    const uint32_t n = ts.wsl + it;
    const int b = static_cast<int>(n % kBufs);
    AB_TR(0, it, 0);
    cp_async_wait<kStages - 2>();
    AB_TR(0, it, 1);
    named_bar_sync(kWorkBar, kWorkThreads);   // slice `it` landed for every worker
    AB_TR(0, it, 2);
    issue(it + kStages - 1);
    if (n >= kBufs) mbar_wait(&ts.empty[b], (n / kBufs - 1) & 1u);   // MMAs on buffer b's last fill done
    AB_TR(0, it, 3);
    uint8_t* buf = smem + b * kPlaneBuf;
    split_slice<kTM>(rawA(it % kStages), a_kc, buf, buf + kPlaneA);
    split_slice<TN>(rawB(it % kStages), b_kc, buf + 2 * kPlaneA, buf + 2 * kPlaneA + kPlaneB);
    fence_proxy_async_smem();   // generic-proxy plane writes -> visible to the tensor core
    __syncwarp();
    if (lane == 0) mbar_arrive(&ts.full[b]);
  }
  ts.wsl += nk;
  cp_async_wait<0>();
  if (nk > 0) {   // the last commit completes after every MMA of the tile
    const uint32_t nl = ts.wsl - 1;
    mbar_wait(&ts.empty[nl % kBufs], (nl / kBufs) & 1u);
  }
  tc_fence_after();
  // epilogue: warp w reads TMEM lane quadrant w % 4 (rows) and column groups w / 4, w / 4 + 2 (32
  // columns each) of every accumulator, sums the accumulators in fixed order, and writes through
  // a shared-memory transpose (the raw ring is idle now) so that lanes run along n: bias, mask and
  // C accesses become one coalesced 128-byte row per instruction
  const int quad = warp & 3;
  const int nacc = nk < kNAcc ? nk : kNAcc;
  float* tr = raw + warp * (32 * 33);
  float* C = g.C + (g.ksplit > 1 ? split * g.cpart : 0);
  const int mrow0 = m0 + quad * 32;
#pragma unroll 1
  for (int t = 0; t < TN / 64; ++t) {
    const int cg = (warp >> 2) + 2 * t;
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0.f;
    for (int a = 0; a < nacc; ++a) {
      uint32_t r[32];
      tmem_ld32(ts.tmem + (static_cast<uint32_t>(quad * 32) << 16) + static_cast<uint32_t>(a * TN + cg * 32), r);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += __uint_as_float(r[i]);
    }
    if (nk > 0 && t == TN / 64 - 1) {   // accumulators read: the issuer may start the next tile
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ts.acc_free);
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) tr[lane * 33 + i] = v[i];
    __syncwarp();
    const int n = n0 + cg * 32 + lane;
    const float bn = (g.mode == 0 && n < g.N) ? g.bias[n] : 0.f;
    for (int rr = 0; rr < 32; ++rr) {
      const int mr = mrow0 + rr;
      if (mr >= g.M) break;
      if (n < g.N) {
        float x = tr[rr * 33 + lane];
        if (g.mode == 0) x = relu(x + bn);
        else if (g.mode == 1) x = g.mask[(long long)mr * g.ldmask + n] > 0.f ? x : 0.f;
        C[(long long)mr * g.ldc + n] = x;
      }
    }
    __syncwarp();
  }
}

#ifdef AB_STATS
__device__ unsigned long long g_adapt_phase[64];   // block 0: clock at entry of each grid barrier
__device__ int g_adapt_nphase;
__device__ long long g_adapt_blk[1024][3];   // per block: smid, clock at F2 tile start, at F2 tile end
__device__ long long g_adapt_sub[1024][5];   // per block, phase B_{L-1}: start, GEMMs, colsum, update, after sync
#define AB_SUB(i) do { if (k == L - 1 && step == 0 && threadIdx.x == 0 && blockIdx.x < 1024) g_adapt_sub[blockIdx.x][i] = clock64(); } while (0)
#else
#define AB_SUB(i) do { } while (0)
#endif
// Grid barrier on a 64-bit arrival counter that only ever grows (never reset, so no "last arriver"
// step): barrier k of a launch completes when the counter reaches base + k * gridDim. One release
// atomic per CTA, then acquire polls; `target` is the next barrier's completion value.
__device__ __forceinline__ void grid_sync(unsigned long long* bar, unsigned long long& target) {
#ifdef AB_STATS
  if (blockIdx.x == 0 && threadIdx.x == 0 && g_adapt_nphase < 64) g_adapt_phase[g_adapt_nphase++] = clock64();
#endif
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned long long old;
    asm volatile("atom.add.release.gpu.u64 %0, [%1], 1;" : "=l"(old) : "l"(bar) : "memory");
    if (old + 1 < target) {
      unsigned long long cur;
      const long long t0 = clock64();
#pragma unroll 1
      for (uint32_t i = 1;; ++i) {
        asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(cur) : "l"(bar) : "memory");
        if (cur >= target) break;
        if ((i & 1023u) == 0) {   // watchdog (ptx.cuh): record, then run to the end instead of trapping
          const long long dt = clock64() - t0;
          if (dt >= (1ll << 26) && ab_aborted()) break;   // (status word only once the wait is stuck)
          if (dt > (1ll << 36)) { ab_raise(kStatusPipeline, blockIdx.x); break; }
        }
      }
    }
    target += gridDim.x;
  }
  __syncthreads();
}

// Column sums over the batch as kSplitK partials (like the split-K weight gradients, summed in fixed
// order by the SGD sweep): out[s * stride + n] = sum_{b in segment s} X[b][n]. One CTA per
// (32-column group, segment), handed out from the highest block index down (those CTAs hold the
// fewest GEMM tiles); warp w sums rows w, w+8, ... of the segment (coalesced, 4 loads in flight)
// and warp 0 adds the 8 warp partials in fixed order.
__device__ void colsum_split(const float* X, int B, int N, long long ld, float* out, long long stride) {
  __shared__ float red[kWorkThreads / 32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kWorkThreads / 32;
  const bool worker = threadIdx.x < kWorkThreads;   // the issuer warp only joins the barriers
  const int groups = (N + 31) / 32, seg = (B + kSplitK - 1) / kSplitK;
  for (int item = gridDim.x - 1 - blockIdx.x; item < groups * kSplitK; item += gridDim.x) {
    const int sgi = item / groups, n = (item % groups) * 32 + lane;
    const int b0 = sgi * seg, b1 = min(B, b0 + seg);
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    if (worker && n < N) {
      int b = b0 + warp;
      for (; b + 3 * nw < b1; b += 4 * nw) {
        a0 += X[(long long)b * ld + n];
        a1 += X[(long long)(b + nw) * ld + n];
        a2 += X[(long long)(b + 2 * nw) * ld + n];
        a3 += X[(long long)(b + 3 * nw) * ld + n];
      }
      for (; b < b1; b += nw) a0 += X[(long long)b * ld + n];
    }
    if (worker) red[warp][lane] = (a0 + a1) + (a2 + a3);
    __syncthreads();
    if (warp == 0 && n < N) {
      float t = red[0][lane];
      for (int w = 1; w < nw; ++w) t += red[w][lane];
      out[sgi * stride + n] = t;
    }
    __syncthreads();
  }
}

// Output layer residual, one warp per sample row (the N = 16 output is too narrow for a GEMM tile):
// R[b][w] = [w < n_b] (W_o h_L,b + b_o - V_bar_b)[w] * scale, scale = 1/B (dV of the objective, R#12).
// W_o is staged in shared memory once per CTA; lane l accumulates k = l, l+32, ... in fp32 FMA and
// the 16 sums are reduced with a fixed xor butterfly (deterministic).
__device__ void out_rows(const float* Hl, const float* Wo, const float* bo, const float* vbar, const int32_t* nvalid,
                         const int32_t* idx, float scale, int B, int H, float* R, float* sW) {
  {   // W_o -> shared memory with 8 independent 16-byte loads in flight per thread (H % 4 == 0)
    const float4* src = reinterpret_cast<const float4*>(Wo);
    float4* dst = reinterpret_cast<float4*>(sW);
    const int n4 = kNMax * H / 4;
    for (int e0 = threadIdx.x; e0 < n4; e0 += 8 * kAdaptThreads) {
      float4 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = e0 + i * kAdaptThreads;
        if (e < n4) v[i] = src[e];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = e0 + i * kAdaptThreads;
        if (e < n4) dst[e] = v[i];
      }
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * kAdaptThreads + threadIdx.x) >> 5, nwarps = (gridDim.x * kAdaptThreads) >> 5;
  for (int b = gwarp; b < B; b += nwarps) {   // (every warp of the CTA, issuer included)
    float acc[kNMax];
#pragma unroll
    for (int w = 0; w < kNMax; ++w) acc[w] = 0.f;
    for (int k0 = lane; k0 < H; k0 += 32 * 8) {   // the row's loads issued 8 at a time
      float h[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) h[i] = k0 + 32 * i < H ? Hl[(long long)b * H + k0 + 32 * i] : 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (k0 + 32 * i < H) {
#pragma unroll
          for (int w = 0; w < kNMax; ++w) acc[w] = fmaf(h[i], sW[w * H + k0 + 32 * i], acc[w]);
        }
      }
    }
    float mine = 0.f;
#pragma unroll
    for (int w = 0; w < kNMax; ++w) {
      float v = acc[w];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == w) mine = v;
    }
    const long long s = idx ? idx[b] : b;   // dataset row of minibatch row b (autobyte_train_epoch)
    if (lane < kNMax)
      R[b * kNMax + lane] = lane < nvalid[s] ? (mine + bo[lane] - vbar[s * kNMax + lane]) * scale : 0.f;
  }
  __syncthreads();   // sW aliases the GEMM ring
}

// One optimiser update over parameters [begin, end); g = the kSplitK gradient partials summed in
// fixed order. SGD: theta -= lr g. Adam (R#18, torch semantics): m = b1 m + (1-b1) g,
// v = b2 v + (1-b2) g^2, theta -= (lr / (1 - b1^t)) m / (sqrt(v) / sqrt(1 - b2^t) + eps).
__device__ void update_range(const AdaptParams& p, long long begin, long long end, int step) {
  float* P = p.params;
  const float* Gr = p.grads;
  const long long total = p.off.total;
  const long long gtid = (long long)blockIdx.x * kAdaptThreads + threadIdx.x, gthreads = (long long)gridDim.x * kAdaptThreads;
  // (all kAdaptThreads threads of every CTA take part: gtid covers [0, gthreads) exactly once)
  if (p.opt == AB_OPT_ADAM) {
    const double t = static_cast<double>(p.t0 + step + 1);
    const float step_size = static_cast<float>(p.lr / (1.0 - pow(static_cast<double>(p.beta1), t)));
    const float sqrt_bc2 = static_cast<float>(sqrt(1.0 - pow(static_cast<double>(p.beta2), t)));
    const float b1 = p.beta1, b2 = p.beta2, c1 = 1.0f - p.beta1, c2 = 1.0f - p.beta2;
    for (long long i = begin + gtid; i < end; i += gthreads) {
      float g = Gr[i];
#pragma unroll
      for (int sk = 1; sk < kSplitK; ++sk) g += Gr[sk * total + i];
      const float m = fmaf(b1, p.m[i], c1 * g);
      const float v = fmaf(b2, p.v[i], c2 * (g * g));
      p.m[i] = m;
      p.v[i] = v;
      P[i] = P[i] - step_size * (m / (sqrtf(v) / sqrt_bc2 + p.eps));
    }
  } else {
    for (long long i = begin + gtid; i < end; i += gthreads) {
      float g = Gr[i];
#pragma unroll
      for (int sk = 1; sk < kSplitK; ++sk) g += Gr[sk * total + i];
      P[i] = P[i] - p.lr * g;
    }
  }
}

__global__ void __launch_bounds__(kAdaptThreads, 1) adapt_kernel(const __grid_constant__ AdaptParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // SW128 atoms: 1 KB aligned
  float* ring = reinterpret_cast<float*>(smem);   // out_rows stages W_o here between GEMM phases
  __shared__ __align__(8) uint64_t s_bar[7];   // full[3], empty[3], acc_free
  __shared__ uint32_t s_tmem;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 3; ++b) {
      mbar_init(&s_bar[b], kWorkThreads / 32);   // full: one arrive per worker warp
      mbar_init(&s_bar[3 + b], 1);               // empty: tcgen05.commit
    }
    mbar_init(&s_bar[6], kWorkThreads / 32);     // acc_free: one arrive per worker warp
    fence_barrier_init();
  }
  if (threadIdx.x < 32) { tmem_alloc(&s_tmem, kTmemCols); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  TcState ts{s_tmem, &s_bar[0], &s_bar[3], &s_bar[6], 0u, 0u, 0u};
  const bool big = p.B >= kBigBatch;   // uniform: every CTA takes the same tile width
  auto tiles = [&](const Gemm& g) { return big ? g.tiles<128>() : g.tiles<64>(); };
  auto gemm = [&](const Gemm& g, int t) {
    if (big) gemm_tile<128>(g, t, smem, ts);
    else gemm_tile<64>(g, t, smem, ts);
  };
  // Two independent GEMMs in one phase (t1 tiles of g1, t2 of g2; every thread takes the same
  // decision). Round-robin over the concatenated tile list can stack a long tile and a short one
  // on the same CTA (backward at B = 1024: 64 K = 512 input-gradient tiles + 128 K = 256 split-K
  // weight-gradient tiles on 148 CTAs); when it is shorter, the g2 tiles get dedicated CTAs
  // [0, t2) and the g1 tiles are dealt round-robin over the rest. Costs are K slices per tile.
  // Tile arithmetic does not depend on the CTA that runs it, so results are unchanged.
  auto gemm_pair = [&](const Gemm& g1, const Gemm& g2) {
    const int t1 = tiles(g1), t2 = tiles(g2), G = gridDim.x;
    auto slices = [&](const Gemm& g) {
      const int kk = g.ksplit > 1 ? (g.K + g.ksplit - 1) / g.ksplit : g.K;
      return (kk + kTK - 1) / kTK;
    };
    const int c1 = slices(g1), c2 = slices(g2), n = t1 + t2, lim = min(G, n);
    // round-robin makespan (in slices): CTA b holds ceil((n-b)/G) tiles, ceil((t1-b)/G) of them
    // from g1; both counts step down once in [0, G) (at t1 % G and n % G), so the maximum over b
    // is attained at b = 0, t1 % G or n % G (closed form: the per-CTA loop cost ~7 % of K4)
    auto rr_cost = [&](int b) {
      const int n1 = b < t1 ? (t1 - b + G - 1) / G : 0, k = (n - b + G - 1) / G;
      return c1 * n1 + c2 * (k - n1);
    };
    int rr = lim > 0 ? rr_cost(0) : 0;
    if (t1 % G < lim) rr = max(rr, rr_cost(t1 % G));
    if (n % G < lim) rr = max(rr, rr_cost(n % G));
    const int rest = G - t2;
    const int ded = (t2 > 0 && rest > 0) ? max(c2, ((t1 + rest - 1) / rest) * c1) : INT_MAX;
    if (ded < rr) {
      if (blockIdx.x < t2) gemm(g2, blockIdx.x);
      else for (int t = blockIdx.x - t2; t < t1; t += rest) gemm(g1, t);
    } else {
      for (int t = blockIdx.x; t < t1 + t2; t += G) {
        if (t < t1) gemm(g1, t);
        else gemm(g2, t - t1);
      }
    }
  };
  const int B = p.B, H = p.H, L = p.L;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gthreads = gridDim.x * blockDim.x;
  // grid barrier: every launch on this ctx has the same grid, so the counter is a multiple of it
  // between launches, and a CTA reading it before its own first arrival sees base .. base + grid - 1
  // (the first barrier cannot complete without it)
  unsigned long long* const gbar = reinterpret_cast<unsigned long long*>(p.barrier);
  unsigned long long gen = 0;
  if (threadIdx.x == 0) {
    unsigned long long cur;
    asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(cur) : "l"(gbar) : "memory");
    gen = cur - cur % gridDim.x + gridDim.x;
  }
  float* P = p.params;
  float* Gr = p.grads;
  // workspace carve-up
  float* Z = p.ws;                              // [B][84]
  float* Hs = Z + (size_t)B * kZDim;            // [L][B][H], H_k at Hs + (k-1)*B*H
  float* R = Hs + (size_t)L * B * H;            // [B][16]
  float* D[2] = {R + (size_t)B * 16, R + (size_t)B * 16 + (size_t)B * H};
  auto Hk = [&](int k) { return Hs + (size_t)(k - 1) * B * H; };

  // phase 0: Z = [x | u(S_p, S_c)] (R#8) of the minibatch; with p.idx (autobyte_train_epoch) row b
  // of step `step` is dataset row idx[step][b], gathered here, and Z is rebuilt every step
  auto build_Z = [&](int step) {
    const int32_t* ix = p.idx ? p.idx + (size_t)step * B : nullptr;
    for (int e = gtid; e < B * kZDim; e += gthreads) {
      const int b = e / kZDim, i = e % kZDim;
      const long long r = ix ? ix[b] : b;
      float v;
      if (i < kXDim) v = p.x[(size_t)r * kXDim + i];
      else if (i == kXDim) v = static_cast<float>((log2(static_cast<double>(p.S_p[r])) - 21.0) / 8.0);
      else v = static_cast<float>((static_cast<double>(p.S_c[r]) - 8.5) / 8.0);
      Z[e] = v;
    }
  };
  build_Z(0);
  grid_sync(gbar, gen);

  const int nsteps = p.steps > 0 ? p.steps : 0;
  for (int step = 0; step <= nsteps; ++step) {
    const bool fwd_only = (step == nsteps);   // trailing forward only when loss is still needed
    if (fwd_only && !(nsteps == 0 && p.loss_before)) break;
    if (p.idx && step > 0) {   // the previous step's last update (W1, b1) ran before this barrier
      build_Z(step);
      grid_sync(gbar, gen);
    }
    // ---------------- forward with stash
    for (int k = 1; k <= L; ++k) {
      const int Kin = k == 1 ? kZDim : H;
      const float* in = k == 1 ? Z : Hk(k - 1);
      Gemm g{B, H, Kin, in, Kin, 1, P + p.off.W[k], 1, Kin, Hk(k), H, 0, P + p.off.b[k], nullptr, 0};
#ifdef AB_STATS
      const long long tw0 = clock64();
#endif
      for (int t = blockIdx.x; t < tiles(g); t += gridDim.x) gemm(g, t);
#ifdef AB_STATS
      if (k == 2 && step == 0 && threadIdx.x == 0 && blockIdx.x < 1024) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_adapt_blk[blockIdx.x][0] = smid;
        g_adapt_blk[blockIdx.x][1] = tw0;
        g_adapt_blk[blockIdx.x][2] = clock64();
      }
#endif
      grid_sync(gbar, gen);
    }
    out_rows(Hk(L), P + p.off.W_o, P + p.off.b_o, p.v_obs, p.n, p.idx ? p.idx + (size_t)step * B : nullptr,
             1.0f / static_cast<float>(B), B, H, R, ring);
    grid_sync(gbar, gen);
    if (((step == 0 && p.loss_before) || (p.losses && !fwd_only)) && blockIdx.x == 0) {
      // mean over b of the Eq. 2 norm ||mask (V_hat - V_bar)||_2; R holds residual / B
      __shared__ float s_norm[kAdaptThreads];
      float acc = 0.f;
      for (int b = threadIdx.x; b < B; b += kAdaptThreads) {
        float ss = 0.f;
        for (int w = 0; w < kNMax; ++w) { const float r = R[b * kNMax + w] * B; ss = fmaf(r, r, ss); }
        acc += sqrtf(ss);
      }
      s_norm[threadIdx.x] = acc;
      __syncthreads();
      if (threadIdx.x == 0) {
        float tot = 0.f;
        for (int i = 0; i < kAdaptThreads; ++i) tot += s_norm[i];
        const float lb = tot / static_cast<float>(B);
        if (step == 0 && p.loss_before) *p.loss_before = lb;
        if (p.losses && !fwd_only) p.losses[step] = lb;
      }
    }
    if (fwd_only) break;
    // ---------------- backward: output layer
    {
      Gemm gw{kNMax, H, B, R, 1, kNMax, Hk(L), H, 1, Gr + p.off.W_o, H, 2, nullptr, nullptr, 0, kSplitK, p.off.total};
      Gemm gd{B, H, kNMax, R, kNMax, 1, P + p.off.W_o, H, 1, D[L & 1], H, 1, nullptr, Hk(L), H};
      gemm_pair(gw, gd);
      colsum_split(R, B, kNMax, kNMax, Gr + p.off.b_o, p.off.total);
      grid_sync(gbar, gen);
    }
    // ---------------- backward: hidden layers L..1
    for (int k = L; k >= 1; --k) {
      const int Kin = k == 1 ? kZDim : H;
      const float* in = k == 1 ? Z : Hk(k - 1);
      const float* Dk = D[k & 1];
      Gemm gw{H, Kin, B, Dk, 1, H, in, Kin, 1, Gr + p.off.W[k], Kin, 2, nullptr, nullptr, 0, kSplitK, p.off.total};
      Gemm gd{};   // M = 0: no tiles
      if (k > 1) {
        gd = Gemm{B, H, H, Dk, H, 1, P + p.off.W[k], H, 1, D[(k - 1) & 1], H, 1, nullptr, Hk(k - 1), H};
      } else if (p.dz_out) {   // encoder fine-tuning: d obj / d [x | u] = D_1 W1 (pre-update W1)
        gd = Gemm{B, kZDim, H, Dk, H, 1, P + p.off.W[1], kZDim, 1, p.dz_out, kZDim, 2, nullptr, nullptr, 0, 1, 0};
      }
      AB_SUB(0);
      gemm_pair(gw, gd);
      AB_SUB(1);
      colsum_split(Dk, B, H, H, Gr + p.off.b[k], p.off.total);
      AB_SUB(2);
      // SGD of the layer above, whose gradient partials completed in the previous phase and whose
      // weights no phase reads any more this step (W_o after BO; W_{k+1} after B_{k+1})
      if (k == L) update_range(p, p.off.W_o, p.off.total, step);
      else update_range(p, p.off.W[k + 1], p.off.b[k + 1] + H, step);
      AB_SUB(3);
      grid_sync(gbar, gen);
      AB_SUB(4);
    }
    // ---------------- SGD of layer 1 (W1, b1); the kernel exit orders it after the last step
    update_range(p, p.off.W[1], p.off.b[1] + H, step);
    if (step + 1 < nsteps) grid_sync(gbar, gen);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(ts.tmem, kTmemCols);
}

size_t adapt_ws_floats(int B, int H, int L) {
  return (size_t)B * kZDim + (size_t)L * B * H + (size_t)B * kNMax + 2 * (size_t)B * H;
}

cudaError_t launch_adapt(const AdaptParams& p, int num_sms, cudaStream_t s, int* grid_used) {
  int per_sm = 0;
  cudaError_t e = cudaFuncSetAttribute(adapt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kAdaptSmemBytes));
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, adapt_kernel, kAdaptThreads, kAdaptSmemBytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  // one CTA per SM (the tensor-core tile needs ~180 KB of shared memory)
  const int want = 1;
  int grid = num_sms * (per_sm < want ? per_sm : want);
  *grid_used = grid;
  void* args[] = {const_cast<AdaptParams*>(&p)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(adapt_kernel), dim3(grid), dim3(kAdaptThreads), args,
                                     kAdaptSmemBytes, s);
}

AB_STATUS_SETTER(set_status_adapt)   // device status word pointer of this unit (ptx.cuh)

}  // namespace ab

#ifdef AB_STATS
extern "C" int ab_debug_adapt_blocks(long long* out, int n) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, ab::g_adapt_blk, sizeof(long long) * 3 * (n < 1024 ? n : 1024)) == cudaSuccess;
}
extern "C" int ab_debug_adapt_trace(long long* out, int arm) {
  cudaDeviceSynchronize();
  if (arm) {
    return cudaMemcpyToSymbol(ab::g_adapt_trace_on, &arm, sizeof(int)) == cudaSuccess;
  }
  return cudaMemcpyFromSymbol(out, ab::g_adapt_trace, sizeof(long long) * 2 * 64 * 4) == cudaSuccess;
}
extern "C" int ab_debug_adapt_sub(long long* out, int n) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, ab::g_adapt_sub, sizeof(long long) * 5 * (n < 1024 ? n : 1024)) == cudaSuccess;
}
extern "C" int ab_debug_adapt_phases(unsigned long long* out) {
  cudaDeviceSynchronize();
  int n = 0;
  cudaMemcpyFromSymbol(&n, ab::g_adapt_nphase, sizeof(int));
  cudaMemcpyFromSymbol(out, ab::g_adapt_phase, sizeof(unsigned long long) * 64);
  int z = 0;
  cudaMemcpyToSymbol(ab::g_adapt_nphase, &z, sizeof(int));
  return n;
}
#endif
