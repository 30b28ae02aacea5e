// score.cu — K2: fused meta-network head + per-job arg-max on sm_100a tensor cores.
//
// For one job j and 128 candidates c (one TMEM lane / epilogue thread per candidate) the
// kernel computes, without touching HBM for activations:
//   h1 = ReLU(a_j + W1c u_c)                    (layer 1, split algebraically: a_j = W1x x_j + b1
//                                                comes from K1; "concatenate ... dense")
//   h_k = ReLU(W_k h_{k-1} + b_k), k = 2..L     (tcgen05.mma kind::f16, bf16 operands, fp32 TMEM
//                                                accumulators; P:402 dense layers, R#1, R#2, R#16)
//   s = w_j . h_L + beta_j                      (mean over the n_j valid workers of W_o h_L + b_o,
//                                                folded into w_j / beta_j by K1, R#3)
//   key = ord32(s) << 32 | ~c  -> atomicMax per job   (P:342 arg-max, ties to smallest c, R#11)
//
// Structure: persistent CTAs (one per SM; CTA pairs by default for H >= 256), 18 warps.
//   warp 0      TMA producer: streams 64-wide K blocks of the packed bf16 weights into an
//               NS-stage shared-memory ring (cp.async.bulk, or 2-D tensor-map copies with
//               .cta_group::2 for CTA pairs; L2 evict_last: every CTA re-reads the same 1.5 MB
//               at 4x512, so they stay L2-resident). When one unit's stages fit the ring (small
//               heads, kernel variant RS) it loads them once and the weights stay resident.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer.
//   warps 2..17 epilogue: 4 warps per TMEM lane quadrant, each owning a quarter of the columns.
// Activations ping-pong between buffer X (shared memory, UMMA SW128 K-major layout, used as
// the A operand of SS-MMAs) and buffer Y (TMEM columns 256.., packed bf16 pairs, A operand
// of TS-MMAs); accumulators are two 128-column TMEM chunks so the epilogue of chunk q
// overlaps the MMAs of chunk q+1. The next tile's h1 is built during the last layer.
// Kernel variants: <H, CG, P3 (fp32 path), BS (every bias in shared memory), RS (resident
// weights)>. Tile / unit / candidate indices are 32-bit with multiply-shift divisions (FastDiv).
#include <cudaTypedefs.h>

#include <cstring>

#include "internal.h"
#include "ptx.cuh"

namespace ab {

#ifndef AB_KBS
#define AB_KBS 2   // 64-wide K blocks per weight stage for CTA pairs
#endif
#ifndef AB_NT
#define AB_NT 1    // tiles in flight per CTA on narrow bf16 heads (H <= 256); 2 measured slower (epilogue-bound)
#endif
#ifndef AB_NACC
#define AB_NACC 2  // TMEM accumulators; 3 fit beside buffer Y at bf16 H = 128 / 256 (NT = 1) but measured slower
#endif

// Optional cycle accounting (build with -DAB_STATS): where each warp role spends its time.
#ifdef AB_STATS
__device__ unsigned long long g_ab_stats[20];
// per-CTA timeline (%globaltimer, ns): entry, prologue done, first MMA issued, first h1 published,
// last MMA issued, epilogue done, exit (after the folded K5)
__device__ unsigned long long g_ab_tl[256][8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define AB_TL(i) do { if (blockIdx.x < 256) g_ab_tl[blockIdx.x][i] = gtimer(); } while (0)
#define AB_T0(v) const long long v = clock64()
#define AB_ACC(st, i, v) (st)[i] += clock64() - (v)
__device__ unsigned long long g_ab_trace[8 * 1024 * 2];   // [cta 0/1][role 0..3][1024 events][code, clock]
// timeline of CTAs 0/1 for their third work unit, plain stores into per-role regions (no atomics)
#define AB_TRACE(on, ev, g, q)                                                                   \
  do {                                                                                           \
    if ((on) && blockIdx.x < 2) {                                                                \
      const int _role = warp == 0 ? 0 : warp == 1 ? 1 : warp == 2 ? 2 : 3;                       \
      unsigned long long* _r = g_ab_trace + ((size_t)(blockIdx.x * 4 + _role) * 1024) * 2;       \
      if (trace_n < 1023) {                                                                      \
        _r[2 * trace_n] = ((unsigned long long)blockIdx.x << 32) | ((ev) << 16) | ((g) << 8) | (q); \
        _r[2 * trace_n + 1] = clock64();                                                         \
        ++trace_n;                                                                               \
      }                                                                                          \
    }                                                                                            \
  } while (0)
#else
#define AB_TRACE(on, ev, g, q)
#define AB_T0(v)
#define AB_ACC(st, i, v)
#define AB_TL(i)
#endif

// P3 = 1 is the fp32-accuracy path (AB_PREC_FP32): every operand x is split into bf16 hi = rn(x) and
// lo = rn(x - hi), and each product is hi*hi + hi*lo + lo*hi (the lo*lo term, ~2^-16 relative, is
// dropped), so activations and weights take twice the storage and three MMAs per K step.
// At H <= 256 both planes of both activation buffers fit on chip (X hi+lo in shared memory, Y hi+lo
// in TMEM). At H = 512 (SPILL) they do not: a layer's input lives as hi plane in X (128 KB of shared
// memory) + lo plane in TMEM (256 columns), next to two 128-column accumulators, and there is no
// second buffer. Each epilogue thread therefore parks its share of the layer's output (hi and lo
// bf16 of its row and column group, 128 B per chunk) in a per-CTA global scratch that stays in L2,
// and once the layer's last chunk shows all of its MMAs done, reads its own share back into X / TMEM
// piece by piece (afull per piece), so the next layer starts on piece 0 while later pieces load.
template <int H, int CG, int P3 = 0>
struct ScoreCfg {
  static constexpr bool SPILL = P3 && H == 512;
  // NT tiles in flight per CTA (narrow bf16 heads): the issuer interleaves their chunks (layer g,
  // chunk q, tile t), so one tile's layer-boundary epilogue latency hides behind the other tile's
  // MMAs. Each tile has its own X (shared memory) and Y (TMEM, YS columns) buffers; at H <= 256 TMEM
  // holds the two 128-column accumulators plus NT Y buffers.
  static constexpr int NT = (!P3 && H <= 256) ? AB_NT : 1;
  static constexpr int NCH = P3 ? (SPILL ? 128 : 64) : (H >= 128 ? 128 : H);  // N of one MMA / accumulator chunk
  static constexpr int NP = P3 ? 2 : 1;           // operand planes (hi, lo)
  static constexpr int NQ = H / NCH;              // chunks per layer
  static constexpr int NKB = H / 64;              // 64-element K blocks per layer
  static constexpr int KB_PER_Q = NCH / 64;       // K blocks of the next layer produced by one chunk
  static constexpr int TILE_BYTES = NCH * 128;    // one (chunk, K block) weight tile of one plane
  static constexpr int STAGE_BYTES = TILE_BYTES * NP;   // ... of all planes
  static constexpr int KBS = (CG == 2 && NKB >= 2 && !P3) ? AB_KBS : 1;  // K blocks per pipeline stage
  static constexpr int ATOM_BYTES = STAGE_BYTES / CG;        // this CTA's part of one K block (N-half for CG=2)
  static constexpr int CTA_STAGE_BYTES = ATOM_BYTES * KBS;   // this CTA's bytes per stage
  static constexpr int STAGE_TX = STAGE_BYTES * KBS;         // bytes per stage over the pair
  static constexpr int A_PLANE = kTileM * H * 2;  // bf16 activation tile (one plane), buffer X
  static constexpr int A_BYTES = A_PLANE * (SPILL ? 1 : NP);   // SPILL: only the hi plane in smem
  static constexpr int NSPLIT = 4;                // epilogue warps per TMEM lane quadrant
  static constexpr int QC = NCH / NSPLIT;         // columns per epilogue warp per chunk
  static constexpr int G_CAP = SPILL ? 0 : (H == 512 ? 3 : 7);  // hidden-layer biases kept in shared memory
                                                  // (SPILL: none; the space deepens the weight ring)
  static constexpr uint32_t Y_LO = SPILL ? 0 : H / 2;   // TMEM column offset of the lo plane of buffer Y
  static constexpr uint32_t YS = H / 2;           // TMEM columns between the Y buffers of the NT tiles
  static constexpr int AW_BYTES = (NT + 2) * H * 4;   // a_j of each tile, W1[:,82], W1[:,83] (SoA)
  static constexpr int WV = H + 4;                // w_j | beta_j, 0, 0, 0 (one tile slot)
  static constexpr int WHAT_BYTES = 2 * NT * WV * 4;   // (current, next) x NT tiles
  static constexpr int BIAS_BYTES = G_CAP * H * 4;
  static constexpr int PART_BYTES = NSPLIT * kTileM * 4;
  static constexpr int MISC_BYTES = 512;
  static constexpr int FIXED = NT * A_BYTES + AW_BYTES + WHAT_BYTES + BIAS_BYTES + PART_BYTES + MISC_BYTES;
  static constexpr int BUDGET = 232448 - 1024;    // opt-in maximum minus the 1 KB alignment slack
  static constexpr int NS_FIT = (BUDGET - FIXED) / CTA_STAGE_BYTES;
#ifdef AB_NS_MAX
  static constexpr int NS = NS_FIT > AB_NS_MAX ? AB_NS_MAX : NS_FIT;   // pipeline-depth experiments
#else
  static constexpr int NS = NS_FIT > 12 ? 12 : NS_FIT;
#endif
  static constexpr int SMEM = 1024 + FIXED + NS * CTA_STAGE_BYTES;
  static constexpr uint32_t IDESC = umma_idesc_bf16(128 * CG, NCH);
  static constexpr uint32_t TMEM_COLS = 512;
  // NACC 128-column accumulators rotate over the chunks (commit order = epilogue order). A third
  // one fits beside Y at H = 128 / 256 (bf16, NT = 1) so the issuer never waits for the epilogue
  // to read the accumulator it overwrites; measured 945 vs 971 TFLOP/s at 3x256 (the epilogue, not
  // the issuer, is the bottleneck), hence off by default.
  static constexpr int NACC = (!P3 && NT == 1 && H >= 128 && H <= 256) ? AB_NACC : 2;
  static constexpr uint32_t Y_COL = NACC * NCH;   // TMEM column of activation buffer Y
  static constexpr int EPI_ARRIVALS = CG == 2 ? 32 : 16;   // 16 epilogue warps per CTA of the pair
  static constexpr int SPILL_U32 = SPILL ? NQ * NSPLIT * (QC / 2) * NP : 0;   // scratch u32 per row (per CTA)
  static_assert(NS >= 4, "not enough shared memory for the weight pipeline");
  static_assert(SMEM <= 232448, "shared memory budget");
  static_assert(NT == 1 || Y_COL + NT * YS <= TMEM_COLS, "TMEM budget of the NT Y buffers");
  static_assert(CTA_STAGE_BYTES % 1024 == 0 && A_BYTES % 1024 == 0, "SW128 atoms need 1 KB alignment");
};

constexpr int kEpiWarps = 16;
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kScoreThreads = 64 + kEpiThreads;
constexpr uint32_t kEpiBar = 1;

// One output chunk of one layer: NKB weight stages x 4 MMAs (K = 16 each) into accumulator d_t.
// A comes from buffer X (SS: smem descriptor) or buffer Y (TS: TMEM address). For the first
// chunk of a layer, K block b is only consumed once the epilogues have published the matching
// 128-column piece of A (afull[b / KB_PER_Q]), so a layer starts before its input is complete.
template <typename C, int CG, bool TS, bool RES = false>
__device__ __forceinline__ void mma_chunk(uint32_t d_t, uint64_t a_desc0, uint32_t a_tmem0, uint64_t b_desc0,
                                          uint64_t* full, uint64_t* empty, uint64_t* afull, uint32_t aph,
                                          int& s, uint32_t& ph, long long* st, bool trace_on, int g, int q,
                                          int& trace_n, int spu = C::NS) {
  const int warp = 1;
  (void)warp;
#pragma unroll 1
  for (int b = 0; b < C::NKB; b += C::KBS) {
    if (afull != nullptr && (b % C::KB_PER_Q) == 0) {
      AB_T0(ta);
      if (CG == 2) mbar_wait_cluster(&afull[b / C::KB_PER_Q], aph);
      else mbar_wait(&afull[b / C::KB_PER_Q], aph);
      AB_ACC(st, 2, ta);
      tc_fence_after();
    }
    AB_T0(tf);
    mbar_wait(&full[s], ph);
    AB_ACC(st, 1, tf);
    AB_TRACE(trace_on && (threadIdx.x & 31) == 0, 42, g, q * 16 + b);
    tc_fence_after();
    if (elect_one()) {
      const uint64_t bst = b_desc0 + static_cast<uint64_t>(s * (C::CTA_STAGE_BYTES >> 4));
#pragma unroll
      for (int a = 0; a < C::KBS; ++a) {
        const uint64_t bd = bst + static_cast<uint64_t>(a * (C::ATOM_BYTES >> 4));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t acc = ((b + a) | kk) != 0;
          const uint64_t ad = a_desc0 + static_cast<uint64_t>((b + a) * 1024 + 2 * kk);
          const uint32_t at = a_tmem0 + ((b + a) * 4 + kk) * 8;
          if (CG == 2) {
            if (TS) umma_ts2(d_t, at, bd + 2 * kk, C::IDESC, acc);
            else umma_ss2(d_t, ad, bd + 2 * kk, C::IDESC, acc);
            if (C::NP == 2) {   // SPILL: + A_hi (X) * W_lo + A_lo (TMEM, a_tmem0) * W_hi
              umma_ss2(d_t, ad, bd + 2 * kk + ((C::TILE_BYTES / CG) >> 4), C::IDESC, 1u);
              umma_ts2(d_t, at, bd + 2 * kk, C::IDESC, 1u);
            }
          } else {
            if (TS) umma_ts(d_t, at, bd + 2 * kk, C::IDESC, acc);
            else umma_ss(d_t, ad, bd + 2 * kk, C::IDESC, acc);
            if (C::NP == 2) {   // + A_hi * W_lo + A_lo * W_hi
              const uint64_t bl = bd + 2 * kk + (C::TILE_BYTES >> 4);
              if (TS) {
                umma_ts(d_t, at, bl, C::IDESC, 1u);
                umma_ts(d_t, at + C::Y_LO, bd + 2 * kk, C::IDESC, 1u);
              } else {
                umma_ss(d_t, ad, bl, C::IDESC, 1u);
                umma_ss(d_t, ad + (C::A_PLANE >> 4), bd + 2 * kk, C::IDESC, 1u);
              }
            }
          }
        }
      }
      if (CG == 2) umma_commit2(&empty[s]);
      else umma_commit(&empty[s]);
    }
    __syncwarp();
    if constexpr (RES) {   // resident weights: the unit's spu stages, loaded once (full stays complete)
      if (++s == spu) s = 0;
    } else {
      if (++s == C::NS) { s = 0; ph ^= 1; }
    }
  }
}

// CG = 1: one CTA per SM computes 128-candidate tiles (M = 128 MMAs).
// CG = 2: a cluster of two CTAs on a TPC forms a CTA pair; each CTA owns one 128-candidate tile
// (its A rows, its TMEM accumulators, its epilogue) and half of every weight stage (64 of the 128
// output rows), and the leader issues M = 256 tcgen05.mma.cta_group::2 for both. Weight bytes
// streamed from L2 per candidate are halved.
// BS: every hidden-layer bias fits the shared-memory copy (G <= G_CAP), so the global-load path of
// the chunk epilogue is compiled out (as a run-time branch both paths were if-converted and issued:
// the predicated-off global loads were 12 % of K2's instructions under ncu).
// RS: resident weights (one unit's weight stages fit the ring; see `spu` below), chosen on the host.
template <int H, int CG, int P3, bool BS, bool RS>
__global__ void __launch_bounds__(kScoreThreads, 1) score_kernel(const __grid_constant__ ScoreParams p) {
  using C = ScoreCfg<H, CG, P3>;
  extern __shared__ uint8_t smem_raw[];
  // 1 KB-aligned base derived by pointer arithmetic on the __shared__ array (no integer round trip),
  // so the compiler keeps every derived pointer in the shared window and emits LDS/STS, not generic loads
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = base;                                                           // [NT][A_BYTES]: X per tile
  uint8_t* sStage = sA + C::NT * C::A_BYTES;
  float* sAw = reinterpret_cast<float*>(sStage + C::NS * C::CTA_STAGE_BYTES);   // [NT+2][H]: a_j.. | W1c0 | W1c1
  float* sWhat = sAw + (C::NT + 2) * H;                                         // [2][NT][WV]
  float* sBias = sWhat + 2 * C::NT * C::WV;                                     // [G_CAP][H]
  float* sPart = sBias + C::G_CAP * H;                                          // [NSPLIT][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sPart + C::NSPLIT * kTileM);
  uint64_t* full = bars;
  uint64_t* empty = full + C::NS;
  uint64_t* dfull = empty + C::NS;
  uint64_t* dempty = dfull + C::NACC;
  uint64_t* afull = dempty + C::NACC;                                           // [NT][NQ]
  uint64_t* vfull = afull + C::NT * C::NQ;                                      // next unit's job vectors
  uint32_t* sTmem = reinterpret_cast<uint32_t*>(vfull + 1);
  unsigned long long* sWkey = reinterpret_cast<unsigned long long*>(sTmem + 2);
  static_assert((2 * C::NS + 2 * C::NACC + C::NT * C::NQ + 1) * 8 + 8 + 32 <= C::MISC_BYTES, "barrier / scalar region");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = p.G;
  const int tpj = p.tiles_per_job;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  long long st[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int trace_n = 0;
  (void)trace_n;
  AB_T0(t_start);
  if (threadIdx.x == 0) AB_TL(0);
#ifdef AB_STATS
  if (threadIdx.x == 0 && blockIdx.x < 256) {   // the CTA's SM (tools/ktimeline.py)
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_ab_tl[blockIdx.x][7] = smid;
  }
#endif

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int i = 0; i < C::NACC; ++i) { mbar_init(&dfull[i], 1); mbar_init(&dempty[i], C::EPI_ARRIVALS); }
    for (int q = 0; q < C::NT * C::NQ; ++q) mbar_init(&afull[q], C::EPI_ARRIVALS);
    mbar_init(vfull, 1);
    fence_barrier_init();
  }
  if (warp == 0 && CG == 2) prefetch_tmap(&p.wmap);
  if (warp == 1) {
    if (CG == 2) { tmem_alloc2(sTmem, C::TMEM_COLS); tmem_relinquish2(); }
    else { tmem_alloc(sTmem, C::TMEM_COLS); tmem_relinquish(); }
  }
  if (warp >= 2) {
    const float* W1 = p.params + p.off.W[1];
    for (int k = threadIdx.x - 64; k < H; k += kEpiThreads) {
      sAw[C::NT * H + k] = W1[(size_t)k * kZDim + kXDim];
      sAw[(C::NT + 1) * H + k] = W1[(size_t)k * kZDim + kXDim + 1];
    }
    const int gs = G < C::G_CAP ? G : C::G_CAP;
    for (int e = threadIdx.x - 64; e < gs * H; e += kEpiThreads) sBias[e] = p.params[p.off.b[e / H + 2] + e % H];
  }
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) AB_TL(1);
  const uint32_t tmem = *sTmem;
  // work unit u = NT tiles per CTA (of a pair): this CTA's tile t of unit u is (u*NT + t)*CG + rank;
  // units are handed out round-robin: first + i*stride
  // tile, unit and candidate indices are 32-bit (the host guarantees n_tiles, c_end < 2^31); the
  // divisions by tiles_per_job and Q are multiply-shifts (FastDiv): a 64-bit division is a ~30-
  // instruction sequence that every epilogue thread ran per tile (ncu: 7.6 % of K2's instructions)
  const int n_tiles = static_cast<int>(p.n_tiles);
  const int n_units = (n_tiles + CG * C::NT - 1) / (CG * C::NT);
  const int first = CG == 2 ? (blockIdx.x >> 1) : blockIdx.x;
  const int stride = CG == 2 ? (gridDim.x >> 1) : gridDim.x;
  // Resident weights: when one unit's weight stages (G layers x NQ chunks x NKB / KBS) fit the ring
  // (3x256 / 2x256 with CTA pairs: 8 / 4 of 9 stages; 3x128: 4 of 11), the producer loads them once
  // into slots 0..spu-1 and stops, and the issuer cycles over those slots for every unit without
  // waiting (their full barriers stay complete) — the weights stay in shared memory for the whole
  // launch instead of being re-streamed from L2 every unit (P:402 dense layers; north star: "weights
  // resident in shared memory").
  const int spu = G * C::NQ * C::NT * (C::NKB / C::KBS);
  constexpr bool resident = RS;   // (the host launches RS = true exactly when spu <= NS)

  if (warp == 0) {
    // ================================================================ TMA producer (both CTAs)
    if (G > 0) {
      const uint64_t pol = l2_policy_evict_last();
      int s = 0;
      uint32_t ph = 0;
      // this pair's (CTA's) replica of the packed weights (same bytes, different L2 lines)
      const int rep = static_cast<int>((CG == 2 ? (blockIdx.x >> 1) : blockIdx.x) % kWeightReplicas);
      const int rep_rows = G * C::NQ * C::NKB * C::NCH * C::NP;   // 64-element rows per replica
      const int u_end = resident ? first + 1 : n_units;   // (first < n_units)
      for (int u = first, k = 0; u < u_end; u += stride, ++k)
        for (int g = 0; g < G; ++g)
          for (int q = 0; q < C::NQ; ++q)
            for (int t = 0; t < C::NT; ++t)   // every tile of the unit streams the same chunk weights
            for (int b = 0; b < C::NKB; b += C::KBS) {
              AB_T0(te);
              mbar_wait(&empty[s], ph ^ 1);
              AB_ACC(st, 0, te);
              AB_TRACE(k == 2 && lane == 0, 40, g, q * 16 + b);
              if (elect_one()) {
                const int ti = (g * C::NQ + q) * C::NKB + b;
#if defined(AB_EXP) && (AB_EXP & 2)
                (void)ti;
                if (leader || CG == 1) mbar_arrive(&full[s]);   // timing experiment: no weight traffic
                if (false)
#endif
                if (CG == 2) {
                  if (leader) mbar_arrive_expect_tx(&full[s], C::STAGE_TX);   // both halves of KBS blocks
#pragma unroll
                  for (int a = 0; a < C::KBS; ++a)
#pragma unroll
                    for (int pl = 0; pl < C::NP; ++pl)   // this CTA's half of the hi (then lo) tile
                      tma_load_2d_pair(sStage + s * C::CTA_STAGE_BYTES + a * C::ATOM_BYTES + pl * (C::TILE_BYTES / 2),
                                       &p.wmap, 0,
                                       rep * rep_rows + ((ti + a) * C::NP + pl) * C::NCH +
                                           static_cast<int>(rank) * (C::NCH / 2),
                                       &full[s], pol);
                } else {
                  mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
                  bulk_g2s(sStage + s * C::STAGE_BYTES, p.wpack + (size_t)rep * rep_rows * 64 + (size_t)ti * (C::NCH * 64 * C::NP),
                           C::STAGE_BYTES, &full[s], pol);
                }
              }
              __syncwarp();
              if (++s == C::NS) { s = 0; ph ^= 1; }
            }
    }
  } else if (warp == 1) {
    // ================================================================ MMA issuer (leader only;
    // warp-converged, one elected lane issues, operands are warp-uniform)
    if (G > 0 && leader) {
      int s = 0;
      uint32_t ph = 0, aph = 0, dbits = 0;
      int dq = 0, b0 = 0;
      const uint64_t b_desc0 = umma_desc_sw128(smem_u32(sStage));
      for (int u = first, k = 0; u < n_units; u += stride, ++k) {
        for (int g = 0; g < G; ++g) {
          const int src = (b0 + g) & 1;
          for (int q = 0; q < C::NQ; ++q)
          for (int t = 0; t < C::NT; ++t) {   // chunks of the unit's tiles interleaved
            const uint64_t a_desc0 = umma_desc_sw128(smem_u32(sA + t * C::A_BYTES));
            const uint32_t y_t = tmem + C::Y_COL + t * C::YS;
            AB_T0(td);
            if (CG == 2) mbar_wait_cluster(&dempty[dq], ((dbits >> dq) & 1u) ^ 1u);
            else mbar_wait(&dempty[dq], ((dbits >> dq) & 1u) ^ 1u);
            AB_ACC(st, 0, td);
            AB_TRACE(k == 2, 10, g, q);
            dbits ^= 1u << dq;
            tc_fence_after();
            const uint32_t d_t = tmem + dq * C::NCH;
            uint64_t* aw = q == 0 ? afull + t * C::NQ : nullptr;
            // (SPILL: every layer reads A hi from X and A lo from TMEM column Y_COL)
            if (C::SPILL || src == 0)
              mma_chunk<C, CG, false, RS>(d_t, a_desc0, C::SPILL ? y_t : 0u, b_desc0, full, empty, aw, aph, s,
                                          ph, st, k == 2, g, q, trace_n, spu);
            else
              mma_chunk<C, CG, true, RS>(d_t, 0ull, y_t, b_desc0, full, empty, aw, aph, s, ph, st, k == 2, g, q,
                                         trace_n, spu);
            if (elect_one()) {
              if (CG == 2) umma_commit2(&dfull[dq]);
              else umma_commit(&dfull[dq]);
            }
            if (u == first && g == 0 && q == 0 && t == 0 && lane == 0) AB_TL(2);
            AB_TRACE(k == 2 && lane == 0, 12, g, q);
            __syncwarp();
            dq = dq + 1 == C::NACC ? 0 : dq + 1;
          }
          aph ^= 1;
        }
        b0 = ((b0 + G - 1) & 1) ^ 1;
      }
      if (lane == 0) AB_TL(4);
    }
  } else {
    // ================================================================ epilogue (256 threads)
    const int etid = threadIdx.x - 64;
    const int ew = warp - 2, quad = warp & 3, grp = ew >> 2;   // grp: column group of a chunk
    const int row = quad * 32 + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    const int c_begin = static_cast<int>(p.c_begin), c_end = static_cast<int>(p.c_end);
    const int cshard = c_end - c_begin;
    const FastDiv tpj_div{static_cast<uint32_t>(tpj), p.tpj_mul, p.tpj_shr};
    const FastDiv q_div{static_cast<uint32_t>(p.Q), p.q_mul, p.q_shr};
    const float* w0s = sAw + C::NT * H;
    const float* w1s = sAw + (C::NT + 1) * H;
    // the MMA issuer's barriers live in the leader CTA: every epilogue warp of the pair counts in
    // on its own (the leader's locally, the peer's with a remote arrive), so no warp waits for the
    // other warps of its CTA
    uint32_t dempty_c[C::NACC];
#pragma unroll
    for (int i = 0; i < C::NACC; ++i) dempty_c[i] = mapa_shared(smem_u32(&dempty[i]), 0);
    auto my_tile = [&](int u, int t) { return (u * C::NT + t) * CG + static_cast<int>(rank); };
    auto signal = [&](uint64_t* bar, uint32_t cluster_addr) {   // called by the whole warp after __syncwarp
      if (lane == 0) {
        if (CG == 2 && !leader) mbar_arrive_remote(cluster_addr);
        else mbar_arrive(bar);
      }
    };

    const int jv = 2 * H + 4;
    auto job_of = [&](int tile) {
      const int tt = tile < n_tiles ? tile : n_tiles - 1;   // ghost tile of an odd pair
      return fdiv(tt, tpj_div);
    };
    // job vectors of unit u's tiles -> their a slots and w|beta slots `slot`, synchronously
    auto load_vecs = [&](int slot, int u) {
      for (int t = 0; t < C::NT; ++t) {
        const float* v = p.jobvec + (size_t)job_of(my_tile(u, t)) * jv;
        for (int k = etid; k < H; k += kEpiThreads) sAw[t * H + k] = v[k];
        for (int k = etid; k < C::WV; k += kEpiThreads) sWhat[(slot * C::NT + t) * C::WV + k] = v[H + k];
      }
    };
    // the same, as TMA bulk copies completing on vfull (issued by one thread)
    auto prefetch_vecs = [&](int slot, int u) {
      if (etid == 0) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(vfull, C::NT * (H + C::WV) * 4);
        for (int t = 0; t < C::NT; ++t) {
          const float* v = p.jobvec + (size_t)job_of(my_tile(u, t)) * jv;
          bulk_g2s(sAw + t * H, v, H * 4, vfull, 0ull);
          bulk_g2s(sWhat + (slot * C::NT + t) * C::WV, v + H, C::WV * 4, vfull, 0ull);
        }
      }
    };
    // candidate index and encoding (K0) of this thread's row of `tile`
    auto row_u = [&](int tile, float& up, float& uc, int& c) {
      const int tt = tile < n_tiles ? tile : n_tiles - 1;
      const int ct = tt - fdiv(tt, tpj_div) * tpj;
      c = c_begin + ct * kTileM + row;
      const int cc = c < c_end ? c : c_end - 1;
      // u_c = (u_p[c / Q], u_c[c % Q]) (a-1, R#8; axes from K1b / K1s)
      const int pi = fdiv(cc, q_div);
      up = p.up[pi];
      uc = p.uc[cc - pi * p.Q];
    };
    // QC bf16 activations of this thread's row starting at column c0 -> buffer X (smem) or Y (TMEM)
    auto store_plane = [&](int t, int dst, int c0, const uint32_t (&pk)[C::QC / 2], int plane) {
#if defined(AB_EXP) && (AB_EXP & 4)
      if (dst == 0) return;   // timing experiment: no shared-memory activation stores
#endif
      if (dst == 0) {  // buffer X: SW128 K-major, 16-byte chunk j of row r stored at chunk j ^ (r % 8)
        const uint32_t rowbase = smem_u32(sA + t * C::A_BYTES) + plane * C::A_PLANE + (c0 >> 6) * 16384 + row * 128;
        const int j0 = (c0 & 63) >> 3;
#pragma unroll
        for (int u = 0; u < C::QC / 8; ++u)
          st_shared_v4(rowbase + (((j0 + u) ^ (row & 7)) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
      } else {         // buffer Y: TMEM, column = element pair index
        tmem_st_cols<C::QC / 2>(lane_base + C::Y_COL + t * C::YS + plane * C::Y_LO + (c0 >> 1), pk);
      }
    };
    // QC post-activation values v (fp32) of this thread's row -> the A operand of the next layer:
    // bf16 (P3 = 0, values already ReLU'd) or hi/lo bf16 planes (P3 = 1)
    auto store_vals = [&](int t, int dst, int c0, const float (&v)[C::QC]) {
      uint32_t hi[C::QC / 2];
#pragma unroll
      for (int i = 0; i < C::QC / 2; ++i) hi[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
      store_plane(t, dst, c0, hi, 0);
      if (C::NP == 2) {
        uint32_t lo[C::QC / 2];
#pragma unroll
        for (int i = 0; i < C::QC / 2; ++i)
          lo[i] = pack_bf16x2(v[2 * i] - __uint_as_float(hi[i] << 16), v[2 * i + 1] - __uint_as_float(hi[i] & 0xFFFF0000u));
        store_plane(t, dst, c0, lo, 1);
      }
    };
    // make this warp's part of A-chunk q of tile slot t visible to the tensor core and count the warp in
    auto publish = [&](int t, int dst, int q) {
      if (dst == 0) fence_proxy_async_smem();
      else { tmem_st_wait(); tc_fence_before(); }
      __syncwarp();
      uint64_t* bar = &afull[t * C::NQ + q];
      signal(bar, CG == 2 ? mapa_shared(smem_u32(bar), 0) : 0u);
    };
    // SPILL: a layer input's piece q is complete in X (hi) and TMEM (lo) for this warp
    auto publish_both = [&](int q) {
      fence_proxy_async_smem();
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      signal(&afull[q], CG == 2 ? mapa_shared(smem_u32(&afull[q]), 0) : 0u);
    };
    // SPILL: QC values -> hi plane into X, lo plane into TMEM (Y_COL), both at column c0
    auto store_split = [&](int c0, const float (&v)[C::QC]) {
      uint32_t hi[C::QC / 2], lo[C::QC / 2];
#pragma unroll
      for (int i = 0; i < C::QC / 2; ++i) {
        hi[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
        lo[i] = pack_bf16x2(v[2 * i] - __uint_as_float(hi[i] << 16), v[2 * i + 1] - __uint_as_float(hi[i] & 0xFFFF0000u));
      }
      store_plane(0, 0, c0, hi, 0);
      store_plane(0, 1, c0, lo, 1);
    };
    // SPILL scratch: this thread's (row, column group) share of chunk q, hi then lo, as 2*QC/8 16-byte
    // words; word i of the warp's 32 rows is 512 contiguous bytes (one coalesced access per warp
    // instruction). Only this thread writes and reads its words back (program order): no fence.
    // Layout per CTA: [chunk q][group grp][quadrant][word i][lane] x 16 B.
    uint4* const spill_warp = C::SPILL ? reinterpret_cast<uint4*>(p.spill + (size_t)blockIdx.x * kTileM * C::SPILL_U32) +
                                             (size_t)quad * (C::QC / 4) * 32 + lane
                                       : nullptr;
    auto spill_at = [&](int q) { return spill_warp + (size_t)(q * C::NSPLIT + grp) * 4 * (C::QC / 4) * 32; };
    auto spill_store = [&](int q, const float (&v)[C::QC]) {
      uint4* d = spill_at(q);
      uint32_t hi[C::QC / 2], lo[C::QC / 2];
#pragma unroll
      for (int i = 0; i < C::QC / 2; ++i) {
        hi[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
        lo[i] = pack_bf16x2(v[2 * i] - __uint_as_float(hi[i] << 16), v[2 * i + 1] - __uint_as_float(hi[i] & 0xFFFF0000u));
      }
#pragma unroll
      for (int i = 0; i < C::QC / 8; ++i) {
        d[32 * i] = make_uint4(hi[4 * i], hi[4 * i + 1], hi[4 * i + 2], hi[4 * i + 3]);
        d[32 * (C::QC / 8 + i)] = make_uint4(lo[4 * i], lo[4 * i + 1], lo[4 * i + 2], lo[4 * i + 3]);
      }
    };
    auto spill_reload = [&](int q) {   // chunk q's share back into X / TMEM
      const uint4* d = spill_at(q);
      uint32_t hi[C::QC / 2], lo[C::QC / 2];
#pragma unroll
      for (int i = 0; i < C::QC / 8; ++i) {
        const uint4 a = d[32 * i], b = d[32 * (C::QC / 8 + i)];
        hi[4 * i] = a.x; hi[4 * i + 1] = a.y; hi[4 * i + 2] = a.z; hi[4 * i + 3] = a.w;
        lo[4 * i] = b.x; lo[4 * i + 1] = b.y; lo[4 * i + 2] = b.z; lo[4 * i + 3] = b.w;
      }
      const int c0 = q * C::NCH + grp * C::QC;
      store_plane(0, 0, c0, hi, 0);
      store_plane(0, 1, c0, lo, 1);
    };
    // layer-1 activations h1 = ReLU(a_j + W1c u_c) of tile slot t for the 128-column piece q (this
    // warp's columns)
    auto build_piece = [&](int t, int q, float up, float uc, int dst) {
      const int c0 = q * C::NCH + grp * C::QC;
      const float* aj = sAw + t * H;
#if defined(AB_EXP) && (AB_EXP & 17)
      if (true) { publish(t, dst, q); return; }   // timing experiment: no h1 build
#endif
      if (C::NP == 1) {
        uint32_t pk[C::QC / 2];
#pragma unroll
        for (int i = 0; i < C::QC / 4; ++i) {
          const float4 a4 = *reinterpret_cast<const float4*>(aj + c0 + 4 * i);
          const float4 u4 = *reinterpret_cast<const float4*>(w0s + c0 + 4 * i);
          const float4 v4 = *reinterpret_cast<const float4*>(w1s + c0 + 4 * i);
          // fma(w1, uc, fma(w0, up, a)) per element, two elements per FFMA2 (bit-identical)
          const float2 h01 = ffma2(make_float2(v4.x, v4.y), make_float2(uc, uc),
                                   ffma2(make_float2(u4.x, u4.y), make_float2(up, up), make_float2(a4.x, a4.y)));
          const float2 h23 = ffma2(make_float2(v4.z, v4.w), make_float2(uc, uc),
                                   ffma2(make_float2(u4.z, u4.w), make_float2(up, up), make_float2(a4.z, a4.w)));
          pk[2 * i] = pack_relu_bf16x2(h01.x, h01.y);
          pk[2 * i + 1] = pack_relu_bf16x2(h23.x, h23.y);
        }
        store_plane(t, dst, c0, pk, 0);
      } else {
        float v[C::QC];
#pragma unroll
        for (int i = 0; i < C::QC / 4; ++i) {
          const float4 a4 = *reinterpret_cast<const float4*>(aj + c0 + 4 * i);
          const float4 u4 = *reinterpret_cast<const float4*>(w0s + c0 + 4 * i);
          const float4 v4 = *reinterpret_cast<const float4*>(w1s + c0 + 4 * i);
          v[4 * i] = relu(fmaf(v4.x, uc, fmaf(u4.x, up, a4.x)));
          v[4 * i + 1] = relu(fmaf(v4.y, uc, fmaf(u4.y, up, a4.y)));
          v[4 * i + 2] = relu(fmaf(v4.z, uc, fmaf(u4.z, up, a4.z)));
          v[4 * i + 3] = relu(fmaf(v4.w, uc, fmaf(u4.w, up, a4.w)));
        }
        if constexpr (C::SPILL) {
          store_split(c0, v);
          publish_both(q);
          return;
        } else {
          store_vals(t, dst, c0, v);
        }
      }
      publish(t, dst, q);
    };

    // score, arg-max key and per-job reduction of a tile (all epilogue threads; a quadrant-local
    // variant without the CTA-wide barriers measured 6 % slower at 3x256: the issuer waited longer
    // for accumulators once the quadrants drifted apart)
    auto reduce_tile = [&](float dot, int wslot, bool real, int j, int c) {
      AB_T0(tr);
      sPart[grp * kTileM + row] = dot;
      named_bar_sync(kEpiBar, kEpiThreads);
      if (grp == 0) {
        float score = sPart[row];
#pragma unroll
        for (int i = 1; i < C::NSPLIT; ++i) score += sPart[i * kTileM + row];
        score += sWhat[wslot * C::WV + H];
        const bool valid = real && c < c_end;
        if (valid && p.scores) p.scores[(size_t)j * cshard + (c - c_begin)] = score;
        const uint32_t o = ord32(score);
        unsigned long long key = (valid && o) ? ((static_cast<unsigned long long>(o) << 32) |
                                                 (0xFFFFFFFFu - static_cast<uint32_t>(c)))
                                              : 0ull;
        if (valid && o && p.cur_idx && c == p.cur_idx[j])
          atomicMax(p.cur_keys + j, (static_cast<unsigned long long>(o) << 32) | 1ull);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, off);
          key = other > key ? other : key;
        }
        if (lane == 0) sWkey[quad] = key;
      }
      named_bar_sync(kEpiBar, kEpiThreads);
      if (etid == 0 && real) {
        unsigned long long k = sWkey[0];
        for (int i = 1; i < 4; ++i) k = sWkey[i] > k ? sWkey[i] : k;
        if (k) atomicMax(p.keys + j, k);
      }
      AB_ACC(st, 4, tr);
    };

    int dq = 0, b0 = 0, it = 0;
    uint32_t dbits = 0, vph = 0;
    int u = first;
    load_vecs(0, u);
    named_bar_sync(kEpiBar, kEpiThreads);
    if (G > 0) {
      for (int t = 0; t < C::NT; ++t) {
        float up, uc;
        int c;
        row_u(my_tile(u, t), up, uc, c);
#pragma unroll 1
        for (int q = 0; q < C::NQ; ++q) build_piece(t, q, up, uc, 0);
      }
    }
    if (etid == 0) AB_TL(3);
    named_bar_sync(kEpiBar, kEpiThreads);   // every thread is done with the a-slots before they are refilled
    for (; u < n_units; u += stride, ++it) {
      const int slot = it & 1;
      const int u_next = u + stride;
      const bool has_next = u_next < n_units;
      float up[C::NT], uc[C::NT], up2[C::NT], uc2[C::NT], dot[C::NT];
      int c[C::NT];
      bool real[C::NT];
      int j[C::NT];
#pragma unroll
      for (int t = 0; t < C::NT; ++t) {
        const int tl = my_tile(u, t);
        real[t] = tl < n_tiles;
        const int tt = real[t] ? tl : n_tiles - 1;
        j[t] = fdiv(tt, tpj_div);
        // this tile's candidate index (its h1 was built earlier; only the G = 0 path reads u here)
        c[t] = c_begin + (tt - j[t] * tpj) * kTileM + row;
        up[t] = uc[t] = 0.f;
        if (G == 0) row_u(tl, up[t], uc[t], c[t]);
        up2[t] = uc2[t] = dot[t] = 0.f;
      }
      if (G > 0 && has_next) {
        // h1 of this unit's tiles is complete, so the a-slots are free: fetch the next unit's job vectors
        prefetch_vecs(slot ^ 1, u_next);
#pragma unroll
        for (int t = 0; t < C::NT; ++t) {
          int c2;
          row_u(my_tile(u_next, t), up2[t], uc2[t], c2);
        }
      }
      if (G == 0) {
        if (it > 0) { load_vecs(slot, u); named_bar_sync(kEpiBar, kEpiThreads); }
#pragma unroll 1
        for (int t = 0; t < C::NT; ++t) {
          const float* wv = sWhat + (slot * C::NT + t) * C::WV;
          const float* aj = sAw + t * H;
          float d = 0.f;
          for (int k = grp * (H / C::NSPLIT); k < (grp + 1) * (H / C::NSPLIT); ++k)
            d = fmaf(relu(fmaf(w1s[k], uc[t], fmaf(w0s[k], up[t], aj[k]))), wv[k], d);
          reduce_tile(d, slot * C::NT + t, real[t], j[t], c[t]);
        }
      }
      for (int g = 0; g < G; ++g) {
        const int src = (b0 + g) & 1, dst = src ^ 1;
        const bool last = (g == G - 1);
        const float* gbias = p.params + p.off.b[g + 2];   // beyond G_CAP layers: read through L1
        if (last && has_next) {
          // the next unit's h1 is built into the buffer this layer does not read (free once chunk
          // 0's MMAs, so every earlier MMA of the tile, are done)
          AB_T0(th);
          mbar_wait(vfull, vph);
          vph ^= 1;
          AB_ACC(st, 5, th);
        }
        for (int q = 0; q < C::NQ; ++q) {
          // this warp's QC biases of chunk q, loaded before the accumulator wait so their latency
          // hides behind it (they sat on the critical path of every chunk epilogue)
          const int n0 = q * C::NCH + grp * C::QC;
          float bq[C::QC];
          if (BS || g < C::G_CAP) {
            const float4* s4 = reinterpret_cast<const float4*>(sBias + g * H + n0);
#pragma unroll
            for (int i = 0; i < C::QC / 4; ++i) {
              const float4 v = s4[i];
              bq[4 * i] = v.x; bq[4 * i + 1] = v.y; bq[4 * i + 2] = v.z; bq[4 * i + 3] = v.w;
            }
          } else {
            const float4* g4 = reinterpret_cast<const float4*>(gbias + n0);
#pragma unroll
            for (int i = 0; i < C::QC / 4; ++i) {
              const float4 v = __ldg(g4 + i);
              bq[4 * i] = v.x; bq[4 * i + 1] = v.y; bq[4 * i + 2] = v.z; bq[4 * i + 3] = v.w;
            }
          }
#pragma unroll 1
          for (int t = 0; t < C::NT; ++t) {   // the issuer's order: chunk q of every tile of the unit
            AB_T0(tw);
            mbar_wait(&dfull[dq], (dbits >> dq) & 1u);
            AB_ACC(st, 0, tw);
            AB_TRACE(it == 2 && lane == 0 && (warp == 2 || warp == 17), 20 + (warp == 17) * 10, g, q);
            AB_T0(tl);
            dbits ^= 1u << dq;
            tc_fence_after();
            uint32_t acc[C::QC];
            tmem_ld_cols<C::QC>(lane_base + dq * C::NCH + grp * C::QC, acc);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            signal(&dempty[dq], dempty_c[dq]);
            AB_ACC(st, 1, tl);
            AB_TRACE(it == 2 && lane == 0 && (warp == 2 || warp == 17), 21 + (warp == 17) * 10, g, q);
            AB_T0(tc);
            dq = dq + 1 == C::NACC ? 0 : dq + 1;
#if defined(AB_EXP) && (AB_EXP & 1)
            if (false)   // timing experiment: no epilogue math or activation stores
#endif
            {
              if (!last && C::SPILL) {   // bias + ReLU in fp32 -> scratch; the last chunk refills X / TMEM
                float v[C::QC];
#pragma unroll
                for (int i = 0; i < C::QC; ++i) v[i] = relu(__uint_as_float(acc[i]) + bq[i]);
                if (q < C::NQ - 1) {
                  spill_store(q, v);
                } else {
                  // this chunk's accumulator is ready, so every MMA of the layer (all readers of X and
                  // of the TMEM lo plane) has completed: this chunk's piece goes straight in (freeing
                  // its registers), then the parked pieces come back in the order the next layer reads them
                  store_split(n0, v);
                  publish_both(q);
#pragma unroll 1
                  for (int pq = 0; pq < C::NQ - 1; ++pq) {
                    spill_reload(pq);
                    publish_both(pq);
                  }
                }
              } else if (!last && C::NP == 2) {   // bias + ReLU in fp32, then hi/lo split
                float v[C::QC];
#pragma unroll
                for (int i = 0; i < C::QC; ++i) v[i] = relu(__uint_as_float(acc[i]) + bq[i]);
                store_vals(t, dst, n0, v);
              } else if (!last) {   // bias + ReLU + round to bf16 (cvt.rn.relu) -> next layer's A operand
                uint32_t pk[C::QC / 2];
#pragma unroll
                for (int i = 0; i < C::QC / 2; ++i) {
                  const float2 z = fadd2(make_float2(__uint_as_float(acc[2 * i]), __uint_as_float(acc[2 * i + 1])),
                                         make_float2(bq[2 * i], bq[2 * i + 1]));
                  pk[i] = pack_relu_bf16x2(z.x, z.y);
                }
                store_plane(t, dst, n0, pk, 0);
              } else {       // last hidden layer stays fp32: dot with the folded output row w_j (R#16)
                const float4* w4 = reinterpret_cast<const float4*>(sWhat + (slot * C::NT + t) * C::WV + n0);
                // four independent FMA chains (element 4i+k into chain k), two per FFMA2
                float2 d01 = make_float2(0.f, 0.f), d23 = make_float2(0.f, 0.f);
#if defined(AB_EXP) && (AB_EXP & 32)
                if (false)   // timing experiment: no last-layer dot
#endif
#pragma unroll
                for (int i = 0; i < C::QC / 4; ++i) {
                  const float4 ww = w4[i];
                  float2 z01 = fadd2(make_float2(__uint_as_float(acc[4 * i]), __uint_as_float(acc[4 * i + 1])),
                                     make_float2(bq[4 * i], bq[4 * i + 1]));
                  float2 z23 = fadd2(make_float2(__uint_as_float(acc[4 * i + 2]), __uint_as_float(acc[4 * i + 3])),
                                     make_float2(bq[4 * i + 2], bq[4 * i + 3]));
                  z01.x = relu(z01.x); z01.y = relu(z01.y); z23.x = relu(z23.x); z23.y = relu(z23.y);
                  d01 = ffma2(z01, make_float2(ww.x, ww.y), d01);
                  d23 = ffma2(z23, make_float2(ww.z, ww.w), d23);
                }
                dot[t] += (d01.x + d01.y) + (d23.x + d23.y);
              }
            }
            if (!last && !C::SPILL) publish(t, dst, q);
            AB_ACC(st, 2, tc);
            AB_TRACE(it == 2 && lane == 0 && (warp == 2 || warp == 17), 22 + (warp == 17) * 10, g, q);
            // (SPILL: only once the last chunk shows the layer's MMAs done, X and TMEM are free)
            if (last && has_next && q == (C::SPILL ? C::NQ - 1 : 0)) {
              // the next unit's h1 of this tile slot, all pieces at once: once this warp has seen
              // chunk 0 of the slot's last layer, the issuer has consumed every afull phase of the
              // slot, so publishing the next unit's phase cannot alias; building early takes h1 off
              // the tile boundary
              AB_T0(th);
#pragma unroll 1
              for (int pq = 0; pq < C::NQ; ++pq) build_piece(t, pq, up2[t], uc2[t], src ^ 1);
              AB_ACC(st, 3, th);
              AB_TRACE(it == 2 && lane == 0 && (warp == 2 || warp == 17), 23 + (warp == 17) * 10, g, q);
            }
            if (last && q == C::NQ - 1) reduce_tile(dot[t], slot * C::NT + t, real[t], j[t], c[t]);
          }
        }
      }
      if (G > 0) b0 = ((b0 + G - 1) & 1) ^ 1;
    }
    if (etid == 0) AB_TL(5);
  }
#ifdef AB_STATS
  // slots: 0-3 producer/MMA/epilogue waits, see tools/kstats.py
  if (lane == 0 && rank == 1 && warp >= 2)   // the peer's epilogue: dfull wait, ld, compute+store, h1
    for (int i = 0; i < 4; ++i) atomicAdd(&g_ab_stats[12 + i], st[i]);
  if (lane == 0 && rank == 0) {
    const long long total = clock64() - t_start;
    if (warp == 0) { atomicAdd(&g_ab_stats[0], st[0]); atomicAdd(&g_ab_stats[1], total); }
    if (warp == 1) {
      atomicAdd(&g_ab_stats[2], st[0]); atomicAdd(&g_ab_stats[3], st[1]);
      atomicAdd(&g_ab_stats[4], st[2]); atomicAdd(&g_ab_stats[5], total);
    }
    if (warp >= 2) {
      for (int i = 0; i < 5; ++i) atomicAdd(&g_ab_stats[6 + i], st[i]);
      atomicAdd(&g_ab_stats[11], total);
      atomicAdd(&g_ab_stats[16], st[5]);
    }
  }
#endif
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    if (CG == 2) tmem_dealloc2(tmem, C::TMEM_COLS);
    else tmem_dealloc(tmem, C::TMEM_COLS);
  }
  {
    // The last CTA to finish zeroes the exit counter for the next (stream-ordered) launch and,
    // single rank, decodes every job's keys (K5 folded in). Each CTA's atomicMax updates happen
    // before its fence + count; the last CTA reads the keys past L1.
    __shared__ int s_last;
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(p.done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && p.finalize) {
      __threadfence();
      for (int j = threadIdx.x; j < p.J; j += blockDim.x) {
        const unsigned long long k = __ldcg(p.keys + j);
        if (k == 0ull) {
          p.best_idx[j] = -1;
          p.best_score[j] = __uint_as_float(0x7FC00000u);
        } else {
          p.best_idx[j] = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(k & 0xFFFFFFFFull));
          p.best_score[j] = unord32(static_cast<uint32_t>(k >> 32));
        }
        if (p.cur_score) {
          const unsigned long long ck = __ldcg(p.cur_keys + j);
          p.cur_score[j] = ck ? unord32(static_cast<uint32_t>(ck >> 32)) : __uint_as_float(0x7FC00000u);
        }
      }
    }
    if (s_last && threadIdx.x == 0) p.done[0] = 0u;
  }
  if (threadIdx.x == 0) AB_TL(6);
}

template <int H, int CG, int P3, bool BS, bool RS>
static cudaError_t launch_score_hcb(const ScoreParams& p, int num_sms, cudaStream_t s) {
  using C = ScoreCfg<H, CG, P3>;
  static unsigned long long attr_done = 0;   // per device: the > 48 KB opt-in is a per-device attribute
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (!(attr_done >> (dev & 63) & 1ull)) {
    e = cudaFuncSetAttribute(score_kernel<H, CG, P3, BS, RS>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_done |= 1ull << (dev & 63);
  }
  const long long units = (p.n_tiles + CG * C::NT - 1) / (CG * C::NT);   // as score_kernel's n_units
  const long long max_units = num_sms / CG;
  const long long grid = (units < max_units ? units : max_units) * CG;
  if (grid < 1) return cudaSuccess;   // (the caller only sets finalize when there is a tile)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kScoreThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, score_kernel<H, CG, P3, BS, RS>, p);
}

template <int H, int CG, int P3, bool BS>
static cudaError_t launch_score_hcbr(const ScoreParams& p, int num_sms, cudaStream_t s) {
  using C = ScoreCfg<H, CG, P3>;
  // resident weights need spu = G * NQ * NT * NKB / KBS <= NS (possible only on small heads)
  if constexpr (!P3 && H <= 256) {
    if (p.G * C::NQ * C::NT * (C::NKB / C::KBS) <= C::NS) return launch_score_hcb<H, CG, P3, BS, true>(p, num_sms, s);
  }
  return launch_score_hcb<H, CG, P3, BS, false>(p, num_sms, s);
}

template <int H, int CG, int P3>
static cudaError_t launch_score_hc(const ScoreParams& p, int num_sms, cudaStream_t s) {
  using C = ScoreCfg<H, CG, P3>;
  if constexpr (C::G_CAP >= kMaxHidden - 1) {   // every head this library accepts (H <= 256)
    return launch_score_hcbr<H, CG, P3, true>(p, num_sms, s);
  } else {
    if (p.G <= C::G_CAP) return launch_score_hcbr<H, CG, P3, true>(p, num_sms, s);
    return launch_score_hcbr<H, CG, P3, false>(p, num_sms, s);
  }
}

template <int H>
static cudaError_t launch_score_h(const ScoreParams& p, int num_sms, cudaStream_t s) {
  if constexpr (H <= 256) {
    if (p.precision3) return launch_score_hc<H, 1, 1>(p, num_sms, s);
  } else {
    if (p.precision3) return launch_score_hc<H, 2, 1>(p, num_sms, s);   // SPILL variant (CTA pairs)
  }
  if (p.cta_group == 2) return launch_score_hc<H, 2, 0>(p, num_sms, s);
  return launch_score_hc<H, 1, 0>(p, num_sms, s);
}

cudaError_t launch_score(const ScoreParams& p, int num_sms, cudaStream_t s) {
  switch (p.H) {
    case 64: return launch_score_h<64>(p, num_sms, s);
    case 128: return launch_score_h<128>(p, num_sms, s);
    case 256: return launch_score_h<256>(p, num_sms, s);
    case 512: return launch_score_h<512>(p, num_sms, s);
  }
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------- K5: decode per-job keys
// K5: keys -> (best index, best score, current score). G > 1 with the all-gather exchange: the
// keys arrive as G rank blocks of [2J] (best keys, then current-config keys) and the per-job max
// is taken here (max is order-free, so the result is the same for any G and shard layout).
__global__ void finalize_kernel(int J, int G, long long stride, const unsigned long long* __restrict__ keys,
                                const unsigned long long* __restrict__ cur_keys, int32_t* best_idx,
                                float* best_score, float* cur_score) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  unsigned long long k = keys[j];
  for (int g = 1; g < G; ++g) k = max(k, keys[g * stride + j]);
  if (k == 0ull) {
    best_idx[j] = -1;
    best_score[j] = __uint_as_float(0x7FC00000u);
  } else {
    best_idx[j] = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(k & 0xFFFFFFFFull));
    best_score[j] = unord32(static_cast<uint32_t>(k >> 32));
  }
  if (cur_score) {
    unsigned long long ck = cur_keys[j];
    for (int g = 1; g < G; ++g) ck = max(ck, cur_keys[g * stride + j]);
    cur_score[j] = ck ? unord32(static_cast<uint32_t>(ck >> 32)) : __uint_as_float(0x7FC00000u);
  }
}

cudaError_t launch_finalize(int J, int G, long long stride, const unsigned long long* keys,
                            const unsigned long long* cur_keys, int32_t* best_idx, float* best_score,
                            float* cur_score, cudaStream_t s) {
  finalize_kernel<<<(J + 255) / 256, 256, 0, s>>>(J, G, stride, keys, cur_keys, best_idx, best_score, cur_score);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- Optimization Trigger (NEXT 1)
// P:435 (5% gain hysteresis) and P:438 (10% drift -> online adaptation), drift checked first.
__global__ void trigger_kernel(int J, const int32_t* __restrict__ best_idx, const float* __restrict__ best_score,
                               const int32_t* __restrict__ cur_idx, const float* __restrict__ cur_score,
                               const float* __restrict__ v_obs, float gain, float drift, int32_t* action) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  const float sc = cur_score[j], sb = best_score[j];
  const int b = best_idx[j], c = cur_idx[j];
  int a = 0;
  if (v_obs) {
    const float v = v_obs[j];
    if (v > 0.f && fabsf(sc - v) / v > drift) a = 2;
  }
  if (a == 0 && b >= 0 && b != c && sb - sc > gain * fabsf(sc)) a = 1;   // NaN compares false
  action[j] = a;
}

cudaError_t launch_trigger(int J, const int32_t* best_idx, const float* best_score, const int32_t* cur_idx,
                           const float* cur_score, const float* v_obs, float gain, float drift, int32_t* action,
                           cudaStream_t s) {
  trigger_kernel<<<(J + 255) / 256, 256, 0, s>>>(J, best_idx, best_score, cur_idx, cur_score, v_obs, gain, drift,
                                                 action);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- weight packing (bf16 shadows)
// wpack layout: for GEMM layer g (W_{g+2}), chunk q of NCH output rows, K block b of 64 inputs:
// NP contiguous NCH x 128-byte tiles (hi, then lo for the fp32 path) in UMMA SW128 K-major order
// (row n at n*128 bytes, 16-byte chunk j stored at chunk j ^ (n % 8)) — exactly what one
// cp.async.bulk drops into a pipeline stage.


__global__ void pack_kernel(const float* __restrict__ params, ParamOffsets off, int H, int L, int planes,
                            __nv_bfloat16* __restrict__ wpack) {
  const int NCH = packed_weight_nch(H, planes), NQ = H / NCH, NKB = H / 64;
  const size_t total = packed_weight_elems(H, L, planes);
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const size_t tile_elems = (size_t)NCH * 64;
    const size_t tile = e / tile_elems;                        // (g, q, b, plane)
    const int plane = static_cast<int>(tile % planes);
    const size_t tq = tile / planes;
    const int within = static_cast<int>(e % tile_elems);
    const int nl = within / 64, slot = within % 64;         // slot = position inside the 128-byte row
    const int kl = (((slot >> 3) ^ (nl & 7)) << 3) | (slot & 7);   // logical k of that position
    const int b = static_cast<int>(tq % NKB);
    const int q = static_cast<int>((tq / NKB) % NQ);
    const int g = static_cast<int>(tq / ((size_t)NKB * NQ));
    const int n = q * NCH + nl, k = b * 64 + kl;
    const float w = params[off.W[g + 2] + (size_t)n * H + k];
    const __nv_bfloat16 hi = __float2bfloat16_rn(w);
    const __nv_bfloat16 v = plane == 0 ? hi : __float2bfloat16_rn(w - __bfloat162float(hi));
#pragma unroll
    for (int r = 0; r < kWeightReplicas; ++r) wpack[e + r * total] = v;
  }
}

cudaError_t launch_pack(const float* params, const ParamOffsets& off, int H, int L, int planes,
                        __nv_bfloat16* wpack, cudaStream_t s) {
  const size_t total = packed_weight_elems(H, L, planes);
  if (total == 0) return cudaSuccess;
  const int blocks = static_cast<int>((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
  pack_kernel<<<blocks, 256, 0, s>>>(params, off, H, L, planes, wpack);
  return cudaGetLastError();
}

AB_STATUS_SETTER(set_status_score)   // device status word pointer of this unit (ptx.cuh)

}  // namespace ab

#ifdef AB_STATS
extern "C" int ab_debug_trace(unsigned long long* out, int n, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, ab::g_ab_trace, sizeof(unsigned long long) * 2 * n) != cudaSuccess) return -1;
  if (reset) cudaMemset(out, 0, 0);
  static unsigned long long z[8 * 1024 * 2];
  if (reset) cudaMemcpyToSymbol(ab::g_ab_trace, z, sizeof(z));
  return n;
}
extern "C" int ab_debug_timeline(unsigned long long* out) {   // [256][8] of the last K2 launch
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, ab::g_ab_tl, sizeof(unsigned long long) * 256 * 8) == cudaSuccess ? 0 : -1;
}
extern "C" int ab_debug_stats(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, ab::g_ab_stats, sizeof(unsigned long long) * 20) != cudaSuccess) return -1;
  if (reset) {
    unsigned long long z[20] = {};
    cudaMemcpyToSymbol(ab::g_ab_stats, z, sizeof(z));
  }
  return 0;
}
#endif

namespace ab {
// Tensor map over the packed weights: a 2-D array of 128-byte rows (64 bf16), SWIZZLE_NONE (the
// data is pre-swizzled), box = 64 bf16 x NCH/2 rows = one CTA's half of a weight stage.
#ifndef AB_TMAP_L2_PROMOTION
#define AB_TMAP_L2_PROMOTION CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return nullptr;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  return encode;
}

bool make_column_tmaps(CUtensorMap* maps, const float* params, const ParamOffsets& off, int H, int L) {
  auto encode = tmap_encoder();
  if (!encode) return false;
  for (int k = 0; k <= kMaxHidden; ++k) std::memset(&maps[k], 0, sizeof(CUtensorMap));
  for (int k = 2; k <= L; ++k) {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(H), static_cast<cuuint64_t>(H)};   // cols, rows
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(H) * 4};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(H / 16), static_cast<cuuint32_t>(H < 256 ? H : 256)};
    cuuint32_t estr[2] = {1, 1};
    if (encode(&maps[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(params + off.W[k]), dims, strides, box,
               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  return true;
}

bool make_weight_tmap(CUtensorMap* map, const __nv_bfloat16* wpack, int H, int L, int planes) {
  auto encode = tmap_encoder();
  if (!encode) return false;
  const int NCH = packed_weight_nch(H, planes);
  const size_t rows = packed_weight_elems(H, L, planes) / 64 * kWeightReplicas;
  if (rows == 0) { std::memset(map, 0, sizeof(*map)); return true; }
  cuuint64_t dims[2] = {64, rows};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(NCH / 2)};
  cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(wpack), dims, strides, box,
                estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, AB_TMAP_L2_PROMOTION,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace ab
