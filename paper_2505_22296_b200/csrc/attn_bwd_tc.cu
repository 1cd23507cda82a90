// tcgen05 attention backward for head_dim 128 with 64-row query tiles (sm_100a).
// attn_block_backward (attention.cpp:167-216): delta = rowsum(dO * O); P = exp(S*scale - lse);
// dV += P^T dO; dS = P (dP - delta) * scale; dQ += dS K; dK += dS^T Q.
//
// One CTA = one 128-row key/value tile x one kv head; it loops over every (query head of the
// GQA group, 64-row query tile) that sees the tile. The bound of this kernel is the SM's
// shared-memory port (128 B/clk), so the design minimises shared-memory operand traffic:
// K and V are copied ONCE into tensor memory and are the A operands of S^T = K Q^T and
// dP^T = V dO^T (TS MMAs read only the 64-query B operand from shared memory: 2 KB instead of
// 6 KB per 16-wide K step). TMEM map (512 columns, lane = key row unless noted):
//   [0, 64)     S^T of the tile: half a (queries 0-31) cols [0,32), half b [32,64);
//               P^T_h (bf16) overwrites cols [32h, 32h+16), dS^T_h (bf16) [32h+16, 32h+32)
//   [64, 128)   dP^T (half a [64,96), half b [96,128)); dQ^T (lane = head-dim index) reuses it
//   [128, 192)  K (bf16 pairs), [192, 256) V
//   [256, 384)  dV accumulator, [384, 512) dK accumulator
// The query tile is processed as two 32-query halves by two softmax-gradient warpgroups, so
// one half's softmax overlaps the other half's MMAs; with one S/dP buffer (the K/V copies take
// the second buffer's columns) the tensor pipe then idles only for the part of a half's
// softmax that outlasts the 128-cycle dP MMA of the other half. Per-iteration MMA order:
//   [wait PR_a] dV_a dK_a [wait PR_b] dQ^T dV_b dK_b | S_a' S_b' [wait dQ^T drained] dP_a' dP_b'
// Shared-memory traffic per 128x64 iteration: 16+16 KB (S, dP B operands) + 16+16 (dV, dK B)
// + 48 (dQ^T = K^T dS^T, SS) + 32 (Q/dO TMA) + 16 (dS^T stores) + 64 (dQ staging + TMA
// reduce) = 224 KB, against 288 KB for the SS design it replaces.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "tc.cuh"

namespace spattn {
namespace {

constexpr int D = 128;
constexpr int BQ = 64;
constexpr int NST = 3;                      // Q/dO pipeline stages
constexpr int NSMW = 8;                     // softmax-gradient warps: (lane quadrant, half)
constexpr int DRAIN0 = NSMW;                // 4 dQ drain warps (also load K/V into TMEM)
constexpr int PRODW = DRAIN0 + 4, TALLOCW = PRODW + 1, MMAW = PRODW + 3;
constexpr int NTHREADS = (PRODW + 4) * 32;  // 512
constexpr int REG_SM = 160, REG_DQ = 96, REG_CTL = 96;
static_assert(NSMW * REG_SM + 4 * REG_DQ + 4 * REG_CTL <= 2048, "register budget");
constexpr int NSTG = 1;                     // dQ staging slots per drain warp
constexpr int KV_TILE = 128 * D * 2;        // 32 KB (two 16 KB column blocks)
constexpr int Q_TILE = BQ * D * 2;          // 16 KB (two 8 KB column blocks)
constexpr int K_OFF = 0, V_OFF = KV_TILE;
constexpr int Q_OFF = 2 * KV_TILE;          // NST x Q tile
constexpr int DO_OFF = Q_OFF + NST * Q_TILE;
constexpr int DS_OFF = DO_OFF + NST * Q_TILE;    // 2 x [128 keys x 64 queries] bf16 (16 KB each)
constexpr int STG_OFF = DS_OFF + 2 * 16384;      // 4 warps x NSTG x [64 queries x 32 fp32] (8 KB)
constexpr int LD_OFF = STG_OFF + 4 * NSTG * 8192;  // lse*log2e, delta: [NST][64] each
constexpr int BAR_OFF = LD_OFF + 2 * NST * 64 * 4;
constexpr uint32_t T_S = 0, T_DP = 64, T_K = 128, T_V = 192, T_DV = 256, T_DK = 384;

enum {
  E_KV = 0,                 // K/V tiles landed (TMA)
  E_KVT = 1,                // K/V copied into TMEM (128 arrivals)
  E_QF = 2,                 // [NST] Q/dO stage full (TMA bytes + 32 producer lanes)
  E_QE = E_QF + NST,        // [NST] stage consumed (MMA commit)
  E_HF = E_QE + NST,        // [2] S^T_h and dP^T_h done
  E_PR = E_HF + 2,          // [2] half h's P^T / dS^T written (128 arrivals)
  E_MD = E_PR + 2,          // [2] dQ^T of iteration i (buffer i&1) done
  E_DQF = E_MD + 2,         // [2] dQ^T drained to registers (128 arrivals)
  E_FIN = E_DQF + 2,
  E_N = E_FIN + 1
};
constexpr int SMEM = BAR_OFF + E_N * 8 + 16;

// 32 consecutive fp32 columns of one row -> 32 bf16 (4 x 16-byte stores)
__device__ __forceinline__ void store_bf16x32(void* dst, const uint32_t (&r)[32]) {
  uint4* o = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int i = 0; i < 4; ++i)
    o[i] = make_uint4(pack_bf16(__uint_as_float(r[8 * i]), __uint_as_float(r[8 * i + 1])),
                      pack_bf16(__uint_as_float(r[8 * i + 2]), __uint_as_float(r[8 * i + 3])),
                      pack_bf16(__uint_as_float(r[8 * i + 4]), __uint_as_float(r[8 * i + 5])),
                      pack_bf16(__uint_as_float(r[8 * i + 6]), __uint_as_float(r[8 * i + 7])));
}

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

// Softmax gradient of one 32-query half for one key (thread): P = 2^(s*scale*log2e - lse*log2e)
// and dS = P (dP - delta) * scale, both packed to bf16 pairs (attention.cpp:199-209). MASK (only
// for tiles crossing the causal diagonal or the row end) zeroes queries outside [ilo, ihi).
// dl2 holds -delta*scale, so dS comes out pre-scaled and dQ / dK need no rescaling.
template <bool MASK>
__device__ __forceinline__ void grad_half(const uint32_t (&rs)[32], const uint32_t (&rp)[32], const float2* nl2,
                                          const float2* dl2, float sl2, float sc, int ilo, int ihi,
                                          uint32_t (&wp)[16], uint32_t (&wd)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float2 nl = nl2[i], dl = dl2[i];
    float2 pp = make_float2(fast_exp2(fmaf(__uint_as_float(rs[2 * i]), sl2, nl.x)),
                            fast_exp2(fmaf(__uint_as_float(rs[2 * i + 1]), sl2, nl.y)));
    if (MASK) {
      pp.x = (2 * i >= ilo && 2 * i < ihi) ? pp.x : 0.f;
      pp.y = (2 * i + 1 >= ilo && 2 * i + 1 < ihi) ? pp.y : 0.f;
    }
    wp[i] = pack_bf16(pp.x, pp.y);
    wd[i] = pack_bf16(pp.x * fmaf(__uint_as_float(rp[2 * i]), sc, dl.x),
                      pp.y * fmaf(__uint_as_float(rp[2 * i + 1]), sc, dl.y));
  }
}

__global__ void __launch_bounds__(NTHREADS, 1)
    attn_bwd_tc_q64_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                           const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                           const __grid_constant__ CUtensorMap tmDQ, BwdArgs a, ProblemSet ps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  if (sbase & 1023) __trap();
  const uint32_t sK = sbase + K_OFF, sV = sbase + V_OFF, sQ = sbase + Q_OFF, sdO = sbase + DO_OFF,
                 sdS = sbase + DS_OFF, sStg = sbase + STG_OFF;
  float* sL = reinterpret_cast<float*>(smem + LD_OFF);  // [NST][64] -lse * log2e (-inf: empty row)
  float* sDl = sL + NST * 64;                           // [NST][64] -delta * scale
  const uint32_t bars = sbase + BAR_OFF;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + BAR_OFF + E_N * 8);
  auto bar = [&](int i) { return bars + 8u * i; };

  const int warp = threadIdx.x / 32;
  long long* trace = (a.trace && blockIdx.x == 0) ? a.trace : nullptr;
#define TR(slot, it) \
  if (trace) trace[(it) * 16 + (slot)] = clock64()
  // head-major order (kv head slowest, heaviest causal key tiles first within a head): the
  // resident CTAs reduce into one kv head's dQ rows, which keeps the fp32 dQ partial sums
  // L2-resident
  const HeadMap hm = a.hm;
  const int ntiles = ps.tile_prefix[ps.n];
  const int tile = blockIdx.x % ntiles;
  const int kvh = blockIdx.x / ntiles;
  const int pi = find_problem(ps, tile);
  const AttnProblem P = ps.p[pi];
  const int n0 = (tile - ps.tile_prefix[pi]) * 128;
  const int g_lo = (kvh + hm.kv_head_base) * hm.rep;
  const int h_lo = max(0, g_lo - hm.q_head_base);
  const int h_hi = min(hm.hq, g_lo + hm.rep - hm.q_head_base);
  int m_begin = 0;
  if (P.causal) m_begin = max(0, n0 - P.off) / BQ * BQ;
  const bool none = (P.causal && n0 - P.off > P.nq - 1) || h_hi <= h_lo || m_begin >= P.nq;
  const int nqt = none ? 0 : (P.nq - m_begin + BQ - 1) / BQ;
  const int T = none ? 0 : (h_hi - h_lo) * nqt;

  if (threadIdx.x == 0) {
    for (int i = 0; i < E_N; ++i) {
      int cnt = 1;
      if (i == E_KVT || (i >= E_PR && i < E_PR + 2) || (i >= E_DQF && i < E_DQF + 2)) cnt = 128;
      if (i >= E_QF && i < E_QF + NST) cnt = 33;  // TMA bytes + the producer's 32 lse/delta lanes
      tc::mbar_init(bar(i), cnt);
    }
    tc::fence_barrier_init();
  }
  if (warp == TALLOCW) tc::tmem_alloc<512>(smem_u32(tmem_slot));
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp >= PRODW) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(REG_CTL));

  // Roles (the scheduler favours the highest warp id, so the single-thread MMA issuer is the
  // last warp): warps 0-7 softmax-gradient (quadrant w&3, query half w>>2), 8-11 dQ drain,
  // 12 TMA producer, 13 TMEM allocator, 15 MMA issuer.
  if (warp == PRODW) {
    // ------------------------------------------------------------------ TMA producer
    // lane 0 issues the TMA loads; all 32 lanes stage the tile's lse/delta (2 query rows each)
    // into the stage's smem slot and arrive on the stage barrier
    const int lane = threadIdx.x % 32;
    if (T > 0) {
      if (lane == 0) {
        tc::mbar_expect_tx(bar(E_KV), 2 * KV_TILE);
        for (int b = 0; b < 2; ++b) {
          tc::tma_load_2d(sK + b * 16384, &tmK, kvh * D + b * 64, P.k_row0 + n0, bar(E_KV));
          tc::tma_load_2d(sV + b * 16384, &tmV, kvh * D + b * 64, P.k_row0 + n0, bar(E_KV));
        }
      }
      float pl[2], pd[2];
      auto fetch = [&](int it) {
        const int h = h_lo + it / nqt, m0 = m_begin + (it % nqt) * BQ;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int row = m0 + lane + 32 * k;
          pl[k] = -INFINITY, pd[k] = 0.f;
          if (row < P.nq) {
            const int64_t g = (int64_t)(P.q_row0 + row) * a.lse_row_stride + h;
            pl[k] = __ldg(a.lse + g);
            pd[k] = __ldg(a.delta + g);
          }
        }
      };
      fetch(0);
      for (int it = 0; it < T; ++it) {
        const int st = it % NST;
        const int h = h_lo + it / nqt, m0 = m_begin + (it % nqt) * BQ;
        if (it >= NST) tc::mbar_wait(bar(E_QE + st), ((it - NST) / NST) & 1);
        if (lane == 0) {
          tc::mbar_expect_tx(bar(E_QF + st), 2 * Q_TILE);
          for (int b = 0; b < 2; ++b) {
            tc::tma_load_2d(sQ + st * Q_TILE + b * 8192, &tmQ, h * D + b * 64, P.q_row0 + m0, bar(E_QF + st));
            tc::tma_load_2d(sdO + st * Q_TILE + b * 8192, &tmDO, h * D + b * 64, P.q_row0 + m0, bar(E_QF + st));
          }
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          sL[st * 64 + lane + 32 * k] = pl[k] == -INFINITY ? -INFINITY : -pl[k] * kLog2e;
          sDl[st * 64 + lane + 32 * k] = -pd[k] * a.scale;  // dS is stored pre-scaled
        }
        if (it + 1 < T) fetch(it + 1);
        tc::mbar_arrive(bar(E_QF + st));  // release: the stores above are visible to waiters
      }
    }
  } else if (warp == MMAW) {
    // ---------------------------------------------------------------------- MMA issuer
    if (tc::elect_one() && T > 0) {
      constexpr uint32_t id_h = tc::idesc_bf16(128, 32, false, false);  // S^T_h, dP^T_h (A in TMEM)
      constexpr uint32_t id_kv = tc::idesc_bf16(128, D, false, true);   // dV, dK (A in TMEM)
      constexpr uint32_t id_q = tc::idesc_bf16(128, BQ, true, true);    // dQ^T
      // S^T_h = K Q_h^T and dP^T_h = V dO_h^T of iteration `it` (query half h = rows 32h..)
      auto s_half = [&](int it, int h) {
        const uint32_t q = sQ + (it % NST) * Q_TILE + h * 4096;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          tc::mma_ts(tmem + T_S + 32 * h, tmem + T_K + ks * 8,
                     tc::sdesc(q + (ks >> 2) * 8192 + (ks & 3) * 32, 16, 1024), id_h, ks > 0);
      };
      auto dp_half = [&](int it, int h) {
        const uint32_t dO = sdO + (it % NST) * Q_TILE + h * 4096;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          tc::mma_ts(tmem + T_DP + 32 * h, tmem + T_V + ks * 8,
                     tc::sdesc(dO + (ks >> 2) * 8192 + (ks & 3) * 32, 16, 1024), id_h, ks > 0);
      };
      // dV += P^T_h dO_h, dK += dS^T_h Q_h (both A operands in TMEM, 2 K-steps of 16 queries)
      auto kv_half = [&](int it, int h) {
        const int st = it % NST;
        const uint32_t q = sQ + st * Q_TILE, dO = sdO + st * Q_TILE;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk)
          tc::mma_ts(tmem + T_DV, tmem + T_S + 32 * h + kk * 8, tc::sdesc(dO + (2 * h + kk) * 2048, 8192, 1024),
                     id_kv, (it > 0 || h > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk)
          tc::mma_ts(tmem + T_DK, tmem + T_S + 32 * h + 16 + kk * 8,
                     tc::sdesc(q + (2 * h + kk) * 2048, 8192, 1024), id_kv, (it > 0 || h > 0 || kk > 0) ? 1u : 0u);
      };
      tc::mbar_wait(bar(E_KVT), 0);
      tc::fence_after();
      tc::mbar_wait(bar(E_QF), 0);
      tc::fence_after();
      s_half(0, 0);
      s_half(0, 1);
      dp_half(0, 0);
      tc::commit(bar(E_HF + 0));
      dp_half(0, 1);
      tc::commit(bar(E_HF + 1));
      for (int it = 0; it < T; ++it) {
        const int b = it & 1, st = it % NST;
        TR(0, it);
        tc::mbar_wait(bar(E_PR + 0), it & 1);
        tc::fence_after();
        TR(1, it);
        kv_half(it, 0);
        tc::mbar_wait(bar(E_PR + 1), it & 1);
        tc::fence_after();
        TR(2, it);
        // dQ^T = K^T dS^T (M = head dim, N = 64 queries, K = 128 keys) into the dP^T columns
        // (both halves' dP^T were consumed before PR); dS^T from smem buffer b
        const uint32_t ds = sdS + b * 16384;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          tc::mma_ss(tmem + T_DP, tc::sdesc(sK + kk * 2048, 16384, 1024), tc::sdesc(ds + kk * 2048, 8192, 1024),
                     id_q, kk > 0 ? 1u : 0u);
        tc::commit(bar(E_MD + b));
        kv_half(it, 1);
        tc::commit(bar(E_QE + st));  // last readers of this Q/dO stage issued
        if (it + 1 < T) {
          tc::mbar_wait(bar(E_QF + (it + 1) % NST), ((it + 1) / NST) & 1);
          tc::fence_after();
          s_half(it + 1, 0);  // the S^T columns' last readers (dV/dK of `it`) are issued
          s_half(it + 1, 1);
          TR(3, it);
          tc::mbar_wait(bar(E_DQF + b), (it >> 1) & 1);  // dQ^T(it) left the dP^T columns
          tc::fence_after();
          TR(4, it);
          dp_half(it + 1, 0);
          tc::commit(bar(E_HF + 0));
          dp_half(it + 1, 1);
          tc::commit(bar(E_HF + 1));
        }
      }
      tc::commit(bar(E_FIN));
    }
  } else if (warp < NSMW) {
    // ----------------------------------- softmax-gradient warpgroups (lane = key, half = w>>2)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(REG_SM));
    const int qd = warp & 3, half = warp >> 2;
    const int t = qd * 32 + (threadIdx.x & 31);  // key row within the tile == TMEM lane
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    const float sl2 = a.scale * kLog2e;
    const int c = n0 + t;
    for (int it = 0; it < T; ++it) {
      const int b = it & 1;
      const int m0 = m_begin + (it % nqt) * BQ + 32 * half;
      const int lb = (it % NST) * 64 + 32 * half;  // this half's lse/delta slot
      int ilo = 0, ihi = min(32, P.nq - m0);
      if (c >= P.nk) ihi = 0;
      if (P.causal) ilo = max(0, c - P.off - m0);
      const bool full = ilo <= 0 && ihi >= 32;
      tc::mbar_wait(bar(E_HF + half), it & 1);
      if (it >= 2) tc::mbar_wait(bar(E_MD + b), ((it - 2) >> 1) & 1);  // dS^T buffer b free
      tc::fence_after();
      uint32_t rs[32], rp[32];
      tc::tmem_ld32(tmem + lane_base + T_S + 32 * half, rs);
      tc::tmem_ld32(tmem + lane_base + T_DP + 32 * half, rp);
      tc::tmem_wait_ld();
      tc::reg_fence(rs);
      tc::reg_fence(rp);
      const float2* nl2 = reinterpret_cast<const float2*>(sL + lb);
      const float2* dl2 = reinterpret_cast<const float2*>(sDl + lb);
      uint32_t wp[16], wd[16];
      if (full)
        grad_half<false>(rs, rp, nl2, dl2, sl2, a.scale, 0, 32, wp, wd);
      else
        grad_half<true>(rs, rp, nl2, dl2, sl2, a.scale, ilo, ihi, wp, wd);
      tc::tmem_st16(tmem + lane_base + T_S + 32 * half, wp);       // P^T_h: A operand of dV
      tc::tmem_st16(tmem + lane_base + T_S + 32 * half + 16, wd);  // dS^T_h: A operand of dK
      const uint32_t ds = sdS + b * 16384;                          // dS^T_h: B operand of dQ^T
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t addr = tc::sw128(ds, t, half * 4 + k);
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};\n" ::"r"(addr), "r"(wd[4 * k]), "r"(wd[4 * k + 1]),
                     "r"(wd[4 * k + 2]), "r"(wd[4 * k + 3]));
      }
      tc::tmem_wait_st();
      tc::fence_proxy_async();
      tc::fence_before();
      tc::mbar_arrive(bar(E_PR + half));
    }
    // dV epilogue: each half's warps own 64 of the 128 columns
    __nv_bfloat16* dvb = a.dv_bf16 ? reinterpret_cast<__nv_bfloat16*>(a.dv_bf16) +
                                         (int64_t)(P.k_row0 + c) * a.dkv_bf16_row_stride + kvh * D
                                   : nullptr;
    if (T > 0) {
      tc::mbar_wait(bar(E_FIN), 0);
      tc::fence_after();
      float* dv = a.dv_acc + (int64_t)(P.k_row0 + c) * a.dkv_row_stride + kvh * D;
#pragma unroll
      for (int ci = 0; ci < 2; ++ci) {
        const int cc = half * 2 + ci;
        uint32_t r[32];
        tc::tmem_ld32(tmem + lane_base + T_DV + cc * 32, r);
        tc::tmem_wait_ld();
        if (c < P.nk) {
          if (dvb) {
            store_bf16x32(dvb + cc * 32, r);
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              red_add_v4(dv + cc * 32 + 4 * i, __uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                         __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
          }
        }
      }
    } else if (dvb && c < P.nk) {  // no query sees this key tile: dV = 0
      uint32_t z[32] = {};
#pragma unroll
      for (int ci = 0; ci < 2; ++ci) store_bf16x32(dvb + (half * 2 + ci) * 32, z);
    }
  } else if (warp >= DRAIN0 && warp < DRAIN0 + 4) {
    // ------------------------------------------- dQ warpgroup (lane = head-dim index)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(REG_DQ));
    const int w = warp - DRAIN0, lane = threadIdx.x % 32;
    const uint32_t lane_base = (uint32_t)(w * 32) << 16;
    if (T > 0) {
      // K and V rows (this thread's key row = TMEM lane) from the swizzled smem tiles into TMEM:
      // column 32b + 4j + i holds the bf16 pair (64b + 8j + 2i, +1), the TS A-operand layout
      tc::mbar_wait(bar(E_KV), 0);
      const int t = w * 32 + lane;
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const uint32_t src = m == 0 ? sK : sV;
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          uint32_t r[32];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                         : "=r"(r[4 * j]), "=r"(r[4 * j + 1]), "=r"(r[4 * j + 2]), "=r"(r[4 * j + 3])
                         : "r"(tc::sw128(src + b * 16384, t, j)));
          tc::tmem_st32(tmem + lane_base + (m == 0 ? T_K : T_V) + 32 * b, r);
        }
      }
      tc::tmem_wait_st();
      tc::fence_before();
      tc::mbar_arrive(bar(E_KVT));
    }
    const uint32_t stg0 = sStg + w * NSTG * 8192;  // NSTG x [64 queries x 32 fp32], 128B-swizzled rows
    for (int it = 0; it < T; ++it) {
      const int b = it & 1;
      const int h = h_lo + it / nqt, m0 = m_begin + (it % nqt) * BQ;
      tc::mbar_wait(bar(E_MD + b), (it >> 1) & 1);
      tc::fence_after();
      uint32_t r[2][32];
      tc::tmem_ld32(tmem + lane_base + T_DP, r[0]);
      tc::tmem_ld32(tmem + lane_base + T_DP + 32, r[1]);
      tc::tmem_wait_ld();
      tc::fence_before();
      tc::mbar_arrive(bar(E_DQF + b));
      const uint32_t stg = stg0 + (it % NSTG) * 8192;
      if (lane == 0) tc::bulk_wait_read<NSTG - 1>();  // the slot's previous reduce has read it
      __syncwarp();
#pragma unroll
      for (int qq = 0; qq < BQ; ++qq) {
        const uint32_t addr = tc::sw128(stg, qq, lane >> 2) + (lane & 3) * 4;
        asm volatile("st.shared.f32 [%0], %1;\n" ::"r"(addr), "f"(__uint_as_float(r[qq >> 5][qq & 31])));
      }
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tc::tma_reduce_add_2d(&tmDQ, stg, h * D + w * 32, P.q_row0 + m0);
        tc::bulk_commit();
      }
    }
    if (lane == 0) tc::bulk_wait_read<0>();
    const int ck = n0 + w * 32 + lane;
    __nv_bfloat16* dkb = a.dk_bf16 ? reinterpret_cast<__nv_bfloat16*>(a.dk_bf16) +
                                         (int64_t)(P.k_row0 + ck) * a.dkv_bf16_row_stride + kvh * D
                                   : nullptr;
    if (T > 0) {  // dK epilogue (lane = key row)
      tc::mbar_wait(bar(E_FIN), 0);
      tc::fence_after();
      float* dk = a.dk_acc + (int64_t)(P.k_row0 + ck) * a.dkv_row_stride + kvh * D;
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t r[32];
        tc::tmem_ld32(tmem + lane_base + T_DK + cc * 32, r);
        tc::tmem_wait_ld();
        if (ck < P.nk) {
          if (dkb) {
            store_bf16x32(dkb + cc * 32, r);
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              red_add_v4(dk + cc * 32 + 4 * i, __uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                         __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
          }
        }
      }
    } else if (dkb && ck < P.nk) {  // no query sees this key tile: dK = 0
      uint32_t z[32] = {};
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) store_bf16x32(dkb + cc * 32, z);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == TALLOCW) tc::tmem_dealloc<512>(tmem);
#undef TR
}

int max_rows(const ProblemSet& ps, bool q) {
  int m = 0;
  for (int i = 0; i < ps.n; ++i) m = max(m, q ? ps.p[i].q_row0 + ps.p[i].nq : ps.p[i].k_row0 + ps.p[i].nk);
  return m;
}

}  // namespace

long long* g_bwd_trace = nullptr;  // profiling (spattn_debug_bwd_trace): clock64 events of CTA 0
void set_bwd_trace(void* p) { g_bwd_trace = static_cast<long long*>(p); }

bool tc_bwd_q64_supported(const BwdArgs& a) {
  auto al = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; };
  return a.d == D && al(a.q) && al(a.k) && al(a.v) && al(a.dout) && al(a.dq_acc) &&
         (a.q_row_stride * 2) % 16 == 0 && (a.kv_row_stride * 2) % 16 == 0 &&
         a.o_row_stride == a.q_row_stride && (a.dq_row_stride * 4) % 16 == 0 && a.dkv_row_stride % 4 == 0;
}

void launch_attn_bwd_tc_q64(const BwdArgs& a, const ProblemSet& in, cudaStream_t s) {
  ProblemSet ps = in;
  BwdArgs args = a;
  args.debug = 0;
  args.trace = g_bwd_trace;
  ps.tile_prefix[0] = 0;
  for (int i = 0; i < ps.n; ++i) ps.tile_prefix[i + 1] = ps.tile_prefix[i] + (ps.p[i].nk + 127) / 128;
  const int tiles = ps.tile_prefix[ps.n];
  if (tiles == 0 || a.hm.hq == 0 || a.hm.hkv == 0) return;
  CUtensorMap tq, tk, tv, tdo, tdq;
  const uint64_t qw = (uint64_t)a.q_row_stride, kw = (uint64_t)a.kv_row_stride;
  const uint64_t qrows = max(1, max_rows(ps, true)), krows = max(1, max_rows(ps, false));
  if (!make_tma_2d(&tq, a.q, qw, qrows, qw, BQ) || !make_tma_2d(&tk, a.k, kw, krows, kw, 128) ||
      !make_tma_2d(&tv, a.v, kw, krows, kw, 128) || !make_tma_2d(&tdo, a.dout, qw, qrows, qw, BQ) ||
      !make_tma_2d_f32(&tdq, a.dq_acc, (uint64_t)a.hm.hq * D, qrows, (uint64_t)a.dq_row_stride, BQ))
    launch_error("attn_bwd_tc_q64", "TMA descriptor encode failed (q/k/v/dout/dq base, strides or extents)");
  ensure_smem_for(attn_bwd_tc_q64_kernel, SMEM);
  attn_bwd_tc_q64_kernel<<<dim3(tiles * a.hm.hkv), NTHREADS, SMEM, s>>>(tq, tk, tv, tdo, tdq, args, ps);
  note_launch();
}

}  // namespace spattn
