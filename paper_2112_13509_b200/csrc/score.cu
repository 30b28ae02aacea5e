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
// Structure: persistent CTAs (one per SM), 10 warps.
//   warp 0      TMA producer: streams 64-wide K blocks of the packed bf16 weights into an
//               NS-stage shared-memory ring with cp.async.bulk (L2 evict_last: every CTA
//               re-reads the same 1.5 MB at 4x512, so they stay L2-resident).
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer.
//   warps 2..9  epilogue: 2 warps per TMEM lane quadrant, each owning half of the columns.
// Activations ping-pong between buffer X (shared memory, UMMA SW128 K-major layout, used as
// the A operand of SS-MMAs) and buffer Y (TMEM columns 256.., packed bf16 pairs, A operand
// of TS-MMAs); accumulators are two 128-column TMEM chunks so the epilogue of chunk q
// overlaps the MMAs of chunk q+1. The next tile's h1 is built during the last layer.
#include "internal.h"
#include "ptx.cuh"

namespace ab {

template <int H>
struct ScoreCfg {
  static constexpr int NCH = H >= 128 ? 128 : H;  // N of one MMA / one TMEM accumulator chunk
  static constexpr int NQ = H / NCH;              // chunks per layer
  static constexpr int NKB = H / 64;              // 64-element K blocks per layer
  static constexpr int KB_PER_Q = NCH / 64;       // K blocks of the next layer produced by one chunk
  static constexpr int STAGE_BYTES = NCH * 128;   // one (chunk, K block) weight tile
  static constexpr int A_BYTES = kTileM * H * 2;  // bf16 activation tile, buffer X
  static constexpr int HALF = NCH / 2;            // columns per epilogue warp per chunk
  static constexpr int G_CAP = H == 512 ? 3 : 7;  // hidden-layer biases kept in shared memory
  static constexpr int AW_BYTES = 3 * H * 4;      // a_j, W1[:,82], W1[:,83] (structure of arrays)
  static constexpr int WHAT_BYTES = 2 * H * 4;    // w_j, two tile slots
  static constexpr int BIAS_BYTES = G_CAP * H * 4;
  static constexpr int PART_BYTES = 2 * kTileM * 4;
  static constexpr int MISC_BYTES = 512;
  static constexpr int FIXED = A_BYTES + AW_BYTES + WHAT_BYTES + BIAS_BYTES + PART_BYTES + MISC_BYTES;
  static constexpr int BUDGET = 232448 - 1024;    // opt-in maximum minus the 1 KB alignment slack
  static constexpr int NS_FIT = (BUDGET - FIXED) / STAGE_BYTES;
  static constexpr int NS = NS_FIT > 8 ? 8 : NS_FIT;
  static constexpr int SMEM = 1024 + FIXED + NS * STAGE_BYTES;
  static constexpr uint32_t IDESC = umma_idesc_bf16(128, NCH);
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr uint32_t Y_COL = 256;          // TMEM column of activation buffer Y
  static_assert(NS >= 4, "not enough shared memory for the weight pipeline");
  static_assert(SMEM <= 232448, "shared memory budget");
  static_assert(STAGE_BYTES % 1024 == 0 && A_BYTES % 1024 == 0, "SW128 atoms need 1 KB alignment");
};

constexpr int kScoreThreads = 320;
constexpr int kEpiThreads = 256;
constexpr int kEpiWarps = 8;
constexpr uint32_t kEpiBar = 1;

// One output chunk of one layer: NKB weight stages x 4 MMAs (K = 16 each) into accumulator d_t.
// A comes from buffer X (SS: smem descriptor) or buffer Y (TS: TMEM address). For the first
// chunk of a layer, K block b is only consumed once the epilogue has published the matching
// 128-column piece of A (afull[b / KB_PER_Q]), so a layer starts before its input is complete.
template <typename C, bool TS>
__device__ __forceinline__ void mma_chunk(uint32_t d_t, uint64_t a_desc0, uint32_t a_tmem0, uint64_t b_desc0,
                                          uint64_t* full, uint64_t* empty, uint64_t* afull, uint32_t aph,
                                          int& s, uint32_t& ph) {
#pragma unroll 1
  for (int b = 0; b < C::NKB; ++b) {
    if (afull != nullptr && (b % C::KB_PER_Q) == 0) {
      mbar_wait(&afull[b / C::KB_PER_Q], aph);
      tc_fence_after();
    }
    mbar_wait(&full[s], ph);
    tc_fence_after();
    if (elect_one()) {
      const uint64_t bd = b_desc0 + static_cast<uint64_t>(s * (C::STAGE_BYTES >> 4));
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t acc = (b | kk) != 0;
        if (TS)
          umma_ts(d_t, a_tmem0 + (b * 4 + kk) * 8, bd + 2 * kk, C::IDESC, acc);
        else
          umma_ss(d_t, a_desc0 + static_cast<uint64_t>(b * 1024 + 2 * kk), bd + 2 * kk, C::IDESC, acc);
      }
      umma_commit(&empty[s]);
    }
    __syncwarp();
    if (++s == C::NS) { s = 0; ph ^= 1; }
  }
}

template <int H>
__global__ void __launch_bounds__(kScoreThreads, 1) score_kernel(const __grid_constant__ ScoreParams p) {
  using C = ScoreCfg<H>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = base;
  uint8_t* sStage = sA + C::A_BYTES;
  float* sAw = reinterpret_cast<float*>(sStage + C::NS * C::STAGE_BYTES);   // [3][H]: a_j | W1c0 | W1c1
  float* sWhat = sAw + 3 * H;                                             // [2][H]
  float* sBias = sWhat + 2 * H;                                           // [G_CAP][H]
  float* sPart = sBias + C::G_CAP * H;                                    // [2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sPart + 2 * kTileM);
  uint64_t* full = bars;
  uint64_t* empty = full + C::NS;
  uint64_t* dfull = empty + C::NS;
  uint64_t* dempty = dfull + 2;
  uint64_t* afull = dempty + 2;                                           // [NQ]
  uint32_t* sTmem = reinterpret_cast<uint32_t*>(afull + C::NQ);
  unsigned long long* sWkey = reinterpret_cast<unsigned long long*>(sTmem + 2);
  float* sBeta = reinterpret_cast<float*>(sWkey + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = p.G;
  const int tpj = p.tiles_per_job;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&dfull[i], 1); mbar_init(&dempty[i], kEpiWarps); }
    for (int q = 0; q < C::NQ; ++q) mbar_init(&afull[q], kEpiWarps);
    fence_barrier_init();
  }
  if (warp == 1) { tmem_alloc(sTmem, C::TMEM_COLS); tmem_relinquish(); }
  if (warp >= 2) {
    const float* W1 = p.params + p.off.W[1];
    for (int k = threadIdx.x - 64; k < H; k += kEpiThreads) {
      sAw[H + k] = W1[(size_t)k * kZDim + kXDim];
      sAw[2 * H + k] = W1[(size_t)k * kZDim + kXDim + 1];
    }
    const int gs = G < C::G_CAP ? G : C::G_CAP;
    for (int e = threadIdx.x - 64; e < gs * H; e += kEpiThreads) sBias[e] = p.params[p.off.b[e / H + 2] + e % H];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *sTmem;
  const long long first = blockIdx.x, stride = gridDim.x;

  if (warp == 0) {
    // ================================================================ TMA producer
    if (G > 0) {
      const uint64_t pol = l2_policy_evict_last();
      int s = 0;
      uint32_t ph = 0;
      for (long long t = first; t < p.n_tiles; t += stride)
        for (int g = 0; g < G; ++g)
          for (int q = 0; q < C::NQ; ++q)
            for (int b = 0; b < C::NKB; ++b) {
              mbar_wait(&empty[s], ph ^ 1);
              if (elect_one()) {
                mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
                const __nv_bfloat16* src = p.wpack + ((size_t)(g * C::NQ + q) * C::NKB + b) * (C::NCH * 64);
                bulk_g2s(sStage + s * C::STAGE_BYTES, src, C::STAGE_BYTES, &full[s], pol);
              }
              __syncwarp();
              if (++s == C::NS) { s = 0; ph ^= 1; }
            }
    }
  } else if (warp == 1) {
    // ================================================================ MMA issuer (warp-converged;
    // one elected lane issues, so every operand is warp-uniform and lives in uniform registers)
    if (G > 0) {
      int s = 0;
      uint32_t ph = 0, aph = 0, dbits = 0;
      int dq = 0, b0 = 0;
      const uint64_t a_desc0 = umma_desc_sw128(smem_u32(sA));
      const uint64_t b_desc0 = umma_desc_sw128(smem_u32(sStage));
      for (long long t = first; t < p.n_tiles; t += stride) {
        for (int g = 0; g < G; ++g) {
          const int src = (b0 + g) & 1;
          for (int q = 0; q < C::NQ; ++q) {
            mbar_wait(&dempty[dq], ((dbits >> dq) & 1u) ^ 1u);
            dbits ^= 1u << dq;
            tc_fence_after();
            const uint32_t d_t = tmem + dq * C::NCH;
            uint64_t* aw = q == 0 ? afull : nullptr;
            if (src == 0)
              mma_chunk<C, false>(d_t, a_desc0, 0u, b_desc0, full, empty, aw, aph, s, ph);
            else
              mma_chunk<C, true>(d_t, 0ull, tmem + C::Y_COL, b_desc0, full, empty, aw, aph, s, ph);
            if (elect_one()) umma_commit(&dfull[dq]);
            __syncwarp();
            dq ^= 1;
          }
          aph ^= 1;
        }
        b0 = ((b0 + G - 1) & 1) ^ 1;
      }
    }
  } else {
    // ================================================================ epilogue (256 threads)
    const int etid = threadIdx.x - 64;
    const int ew = warp - 2, quad = warp & 3, half = ew >> 2;
    const int row = quad * 32 + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    const long long cshard = p.c_end - p.c_begin;
    const float* w0s = sAw + H;
    const float* w1s = sAw + 2 * H;

    auto load_vecs = [&](int slot, long long tile) {
      const int j = static_cast<int>(tile / tpj);
      const float* a = p.a + (size_t)j * H;
      const float* w = p.what + (size_t)j * H;
      for (int k = etid; k < H; k += kEpiThreads) {
        sAw[k] = a[k];
        sWhat[slot * H + k] = w[k];
      }
      if (etid == 0) sBeta[slot] = p.beta[j];
    };
    auto row_u = [&](long long tile, float& up, float& uc, long long& c) {
      const int ct = static_cast<int>(tile % tpj);
      c = p.c_begin + (long long)ct * kTileM + row;
      const long long cc = c < p.c_end ? c : p.c_end - 1;
      const long long pi = cc / p.Q, qi = cc % p.Q;
      up = static_cast<float>((log2(static_cast<double>(p.S_p[pi])) - 21.0) / 8.0);   // R#8
      uc = static_cast<float>((static_cast<double>(p.S_c[qi]) - 8.5) / 8.0);
    };
    auto store32 = [&](int dst, int c0, const uint32_t (&pk)[16]) {
      if (dst == 0) {  // buffer X: SW128 K-major, 16-byte chunk j of row r stored at chunk j ^ (r % 8)
        const uint32_t rowbase = smem_u32(sA) + (c0 >> 6) * 16384 + row * 128;
        const int j0 = (c0 & 63) >> 3;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          st_shared_v4(rowbase + (((j0 + u) ^ (row & 7)) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
      } else {         // buffer Y: TMEM, column = element pair index
        tmem_st16(lane_base + C::Y_COL + (c0 >> 1), pk);
      }
    };
    // make this warp's part of A-chunk q visible to the tensor core and count the warp in
    auto publish = [&](int dst, int q) {
      if (dst == 0) fence_proxy_async_smem();
      else { tmem_st_wait(); tc_fence_before(); }
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[q]);
    };
    auto build_h1 = [&](float up, float uc, int dst) {
#pragma unroll 1
      for (int q = 0; q < C::NQ; ++q) {
#pragma unroll
        for (int hp = 0; hp < C::HALF / 32; ++hp) {
          const int c0 = q * C::NCH + half * C::HALF + hp * 32;
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 a4 = *reinterpret_cast<const float4*>(sAw + c0 + 4 * i);
            const float4 u4 = *reinterpret_cast<const float4*>(w0s + c0 + 4 * i);
            const float4 v4 = *reinterpret_cast<const float4*>(w1s + c0 + 4 * i);
            pk[2 * i] = pack_bf16x2(relu(fmaf(v4.x, uc, fmaf(u4.x, up, a4.x))),
                                    relu(fmaf(v4.y, uc, fmaf(u4.y, up, a4.y))));
            pk[2 * i + 1] = pack_bf16x2(relu(fmaf(v4.z, uc, fmaf(u4.z, up, a4.z))),
                                        relu(fmaf(v4.w, uc, fmaf(u4.w, up, a4.w))));
          }
          store32(dst, c0, pk);
        }
        publish(dst, q);
      }
    };

    int dq = 0, b0 = 0, it = 0;
    uint32_t dbits = 0;
    long long t = first;
    if (t < p.n_tiles) load_vecs(0, t);
    named_bar_sync(kEpiBar, kEpiThreads);
    if (G > 0 && t < p.n_tiles) {
      float up, uc;
      long long c;
      row_u(t, up, uc, c);
      build_h1(up, uc, 0);
    }
    for (; t < p.n_tiles; t += stride, ++it) {
      const int slot = it & 1;
      const long long tn = t + stride;
      const int j = static_cast<int>(t / tpj);
      float up, uc;
      long long c;
      row_u(t, up, uc, c);
      float dot = 0.f;
      if (G == 0) {
        if (it > 0) { load_vecs(slot, t); named_bar_sync(kEpiBar, kEpiThreads); }
        const float* wv = sWhat + slot * H;
        for (int k = half * (H / 2); k < (half + 1) * (H / 2); ++k)
          dot = fmaf(relu(fmaf(w1s[k], uc, fmaf(w0s[k], up, sAw[k]))), wv[k], dot);
      }
      for (int g = 0; g < G; ++g) {
        const int src = (b0 + g) & 1, dst = src ^ 1;
        const bool last = (g == G - 1);
        const float* bias = g < C::G_CAP ? sBias + g * H : p.params + p.off.b[g + 2];
        for (int q = 0; q < C::NQ; ++q) {
          mbar_wait(&dfull[dq], (dbits >> dq) & 1u);
          dbits ^= 1u << dq;
          tc_fence_after();
          uint32_t acc[2][32];
          const uint32_t dcol = dq * C::NCH + half * C::HALF;
          tmem_ld32(lane_base + dcol, acc[0]);
          if (C::HALF == 64) tmem_ld32(lane_base + dcol + 32, acc[1]);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&dempty[dq]);
          dq ^= 1;
#pragma unroll
          for (int hp = 0; hp < C::HALF / 32; ++hp) {
            const int n0 = q * C::NCH + half * C::HALF + hp * 32;
            const float4* b4 = reinterpret_cast<const float4*>(bias + n0);
            float v[32];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 bb = b4[i];
              v[4 * i + 0] = relu(__uint_as_float(acc[hp][4 * i + 0]) + bb.x);
              v[4 * i + 1] = relu(__uint_as_float(acc[hp][4 * i + 1]) + bb.y);
              v[4 * i + 2] = relu(__uint_as_float(acc[hp][4 * i + 2]) + bb.z);
              v[4 * i + 3] = relu(__uint_as_float(acc[hp][4 * i + 3]) + bb.w);
            }
            if (!last) {
              uint32_t pk[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) pk[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
              store32(dst, n0, pk);
            } else {
              const float4* w4 = reinterpret_cast<const float4*>(sWhat + slot * H + n0);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const float4 ww = w4[i];
                dot = fmaf(v[4 * i], ww.x, dot);
                dot = fmaf(v[4 * i + 1], ww.y, dot);
                dot = fmaf(v[4 * i + 2], ww.z, dot);
                dot = fmaf(v[4 * i + 3], ww.w, dot);
              }
            }
          }
          if (!last) publish(dst, q);
          if (last && q == 0 && tn < p.n_tiles) {
            // next tile's h1 goes into the buffer the last layer does not read
            load_vecs(slot ^ 1, tn);
            named_bar_sync(kEpiBar, kEpiThreads);
            float up2, uc2;
            long long c2;
            row_u(tn, up2, uc2, c2);
            build_h1(up2, uc2, src ^ 1);
          }
        }
      }
      if (G > 0) b0 = ((b0 + G - 1) & 1) ^ 1;

      // ------------------------------------------------ score, arg-max key, per-job reduction
      sPart[half * kTileM + row] = dot;
      named_bar_sync(kEpiBar, kEpiThreads);
      if (half == 0) {
        const float score = sPart[row] + sPart[kTileM + row] + sBeta[slot];
        const bool valid = c < p.c_end;
        if (valid && p.scores) p.scores[(size_t)j * cshard + (c - p.c_begin)] = score;
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
      if (etid == 0) {
        unsigned long long k = sWkey[0];
        for (int i = 1; i < 4; ++i) k = sWkey[i] > k ? sWkey[i] : k;
        if (k) atomicMax(p.keys + j, k);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
}

size_t score_smem_bytes(int H) {
  switch (H) {
    case 64: return ScoreCfg<64>::SMEM;
    case 128: return ScoreCfg<128>::SMEM;
    case 256: return ScoreCfg<256>::SMEM;
    case 512: return ScoreCfg<512>::SMEM;
  }
  return 0;
}

template <int H>
static cudaError_t launch_score_h(const ScoreParams& p, int num_sms, cudaStream_t s) {
  using C = ScoreCfg<H>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(score_kernel<H>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  long long grid = p.n_tiles < num_sms ? p.n_tiles : num_sms;
  if (grid < 1) return cudaSuccess;
  score_kernel<H><<<static_cast<int>(grid), kScoreThreads, C::SMEM, s>>>(p);
  return cudaGetLastError();
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
__global__ void finalize_kernel(int J, const unsigned long long* __restrict__ keys,
                                const unsigned long long* __restrict__ cur_keys, int32_t* best_idx,
                                float* best_score, float* cur_score) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  const unsigned long long k = keys[j];
  if (k == 0ull) {
    best_idx[j] = -1;
    best_score[j] = __uint_as_float(0x7FC00000u);
  } else {
    best_idx[j] = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(k & 0xFFFFFFFFull));
    best_score[j] = unord32(static_cast<uint32_t>(k >> 32));
  }
  if (cur_score) {
    const unsigned long long ck = cur_keys[j];
    cur_score[j] = ck ? unord32(static_cast<uint32_t>(ck >> 32)) : __uint_as_float(0x7FC00000u);
  }
}

cudaError_t launch_finalize(int J, const unsigned long long* keys, const unsigned long long* cur_keys,
                            int32_t* best_idx, float* best_score, float* cur_score, cudaStream_t s) {
  finalize_kernel<<<(J + 255) / 256, 256, 0, s>>>(J, keys, cur_keys, best_idx, best_score, cur_score);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- weight packing (bf16 shadows)
// wpack layout: for GEMM layer g (W_{g+2}), chunk q of NCH output rows, K block b of 64 inputs:
// a contiguous NCH x 128-byte tile in UMMA SW128 K-major order (row n at n*128 bytes, 16-byte
// chunk j stored at chunk j ^ (n % 8)) — exactly what one cp.async.bulk drops into a stage.
__host__ __device__ size_t packed_weight_elems(int H, int L) { return (size_t)(L > 1 ? L - 1 : 0) * H * H; }

__global__ void pack_kernel(const float* __restrict__ params, ParamOffsets off, int H, int L,
                            __nv_bfloat16* __restrict__ wpack) {
  const int NCH = H >= 128 ? 128 : H, NQ = H / NCH, NKB = H / 64;
  const size_t total = packed_weight_elems(H, L);
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const size_t tile_elems = (size_t)NCH * 64;
    const size_t tile = e / tile_elems;
    const int within = static_cast<int>(e % tile_elems);
    const int nl = within / 64, slot = within % 64;         // slot = position inside the 128-byte row
    const int kl = (((slot >> 3) ^ (nl & 7)) << 3) | (slot & 7);   // logical k of that position
    const int b = static_cast<int>(tile % NKB);
    const int q = static_cast<int>((tile / NKB) % NQ);
    const int g = static_cast<int>(tile / ((size_t)NKB * NQ));
    const int n = q * NCH + nl, k = b * 64 + kl;
    wpack[e] = __float2bfloat16_rn(params[off.W[g + 2] + (size_t)n * H + k]);
  }
}

cudaError_t launch_pack(const float* params, const ParamOffsets& off, int H, int L, __nv_bfloat16* wpack,
                        cudaStream_t s) {
  const size_t total = packed_weight_elems(H, L);
  if (total == 0) return cudaSuccess;
  const int blocks = static_cast<int>((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
  pack_kernel<<<blocks, 256, 0, s>>>(params, off, H, L, wpack);
  return cudaGetLastError();
}

}  // namespace ab
