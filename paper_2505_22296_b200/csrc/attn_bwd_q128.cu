// tcgen05 attention backward for head_dim 128 with 128-row query tiles (sm_100a).
// attn_block_backward (attention.cpp:167-216): delta = rowsum(dO * O); P = exp(S*scale - lse);
// dV += P^T dO; dS = P (dP - delta) * scale; dQ += dS K; dK += dS^T Q.
//
// Why 128-row query tiles: the backward is bound by the SM's shared-memory port (tensor-core
// operand reads plus LSU traffic, one 128-byte wavefront per clock; profiles/r2_bwd.md). With
// N = 128 every MMA reads its A operand once per 128 queries instead of once per 64.
//
// One CTA = one 128-row key/value tile x one kv head; it loops over every (query head of the
// GQA group, 128-row query tile) that sees the tile. TMEM (512 columns) holds ONE buffer per
// product, so the softmax-gradient work is split into two phases that each overlap MMAs:
//   [0, 128)    S^T (lane = key, col = query); phase A writes P^T (bf16) over cols
//               [64c, 64c+32) of query half c (A operand of dV)
//   [128, 256)  dV accumulator
//   [256, 384)  dP^T; dQ (lane = QUERY, col = head dim) reuses the columns once phase B has
//               read dP^T
//   [384, 512)  dK accumulator
// Phase A(i): P = exp2(S*scale*log2e - lse*log2e) -> P^T in TMEM; P stays in registers (fp32).
// Phase B(i): dS = P (dP - delta) -> dS^T to one smem tile, read MN-major as the A operand of
// dQ = dS K and K-major as the A operand of dK += dS^T Q. MMA issue order per iteration i:
//   S(i+1)  dQ(i)  dK(i)  dP(i+1)  dV(i+1)
// dQ goes first so its drain (lane = query: the four drain warps load a whole 128-column row,
// release the columns, then stage 16-byte rows for the TMA reduce-add) overlaps dK(i); phase
// B(i+1) starts as soon as dP(i+1) lands, and dV(i+1), which waits for phase A, is off that
// chain. Eight softmax warps (two per TMEM lane quadrant, one 64-query half each; 144
// registers), four drain warps (168), producer / allocator / MMA issuer (56).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "tc.cuh"

namespace spattn {
namespace {

constexpr int D = 128, BQ = 128;
#ifndef Q128_POLY
#define Q128_POLY 0
#endif
constexpr bool kPolyExp = Q128_POLY;
constexpr int NCW = 8;                               // softmax-gradient warps
constexpr int DRAIN0 = NCW, PRODW = DRAIN0 + 4, TALLOCW = PRODW + 1, MMAW = PRODW + 3;
constexpr int NTHREADS = (PRODW + 4) * 32;           // 512
// registers per thread after setmaxnreg (the launch gives 128 to all 512 threads): the drain
// warps hold a whole 128-column dQ row so they release the TMEM columns in one round trip
constexpr int REG_C = 144, REG_DQ = 168, REG_CTL = 56;
static_assert(NCW * REG_C + 4 * REG_DQ + 4 * REG_CTL <= 2048, "register budget");
constexpr int NQ = 2;                                // Q stages (S(i+1) is issued before dK(i))
constexpr int TILE = 128 * D * 2;                    // 32 KB: two 16 KB 128B-swizzled column blocks
constexpr int K_OFF = 0, V_OFF = TILE, Q_OFF = 2 * TILE, DO_OFF = Q_OFF + NQ * TILE;
constexpr int DS_OFF = DO_OFF + TILE;                // dS^T [128 keys][128 queries] bf16: 2 blocks
constexpr int STG_OFF = DS_OFF + TILE;               // 4 drain warps x 2 slots x [32 rows x 32 fp32]
constexpr int LSE_OFF = STG_OFF + 4 * 2 * 4096;      // [NQ][128] -lse*log2e
constexpr int DL_OFF = LSE_OFF + NQ * 128 * 4;       // [128] -delta*scale (rewritten once phase B read it)
constexpr int BAR_OFF = DL_OFF + 128 * 4;
constexpr uint32_t T_S = 0, T_DV = 128, T_DP = 256, T_DK = 384;

enum {
  E_KV = 0,
  E_QF = 1,           // [NQ] Q stage + lse landed (TMA bytes + 32 producer lanes)
  E_QE = E_QF + NQ,   // [NQ] Q stage read by S and dK
  E_DOF = E_QE + NQ,  // dO + delta landed
  E_DOE,              // dO read by dV and dP
  E_SR,               // S^T(i) in TMEM
  E_PR,               // P^T(i) written (256 arrivals)
  E_DPR,              // dP^T(i) in TMEM
  E_DSR,              // dS^T(i) written to TMEM and smem (256 arrivals)
  E_MD,               // dQ(i) in TMEM (dS smem free again)
  E_DQF,              // dQ(i) read out of TMEM (128 arrivals)
  E_FIN,
  E_N
};
constexpr int SMEM = BAR_OFF + E_N * 8 + 16;
static_assert(SMEM <= 232448 - 1024, "shared memory");

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

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <class PS>
__global__ void __launch_bounds__(NTHREADS, 1)
    attn_bwd_q128_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                         const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                         const __grid_constant__ CUtensorMap tmDQ, BwdArgs a, PS ps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  if (sbase & 1023) __trap();
  const uint32_t sK = sbase + K_OFF, sV = sbase + V_OFF, sQ = sbase + Q_OFF, sdO = sbase + DO_OFF,
                 sdS = sbase + DS_OFF, sStg = sbase + STG_OFF;
  float* sLse = reinterpret_cast<float*>(smem + LSE_OFF);
  float* sDl = reinterpret_cast<float*>(smem + DL_OFF);
  const uint32_t bars = sbase + BAR_OFF;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + BAR_OFF + E_N * 8);
  auto bar = [&](int i) { return bars + 8u * i; };

  const int warp = threadIdx.x / 32;
  long long* trace = (a.trace && blockIdx.x == 0) ? a.trace : nullptr;
#define TR(slot, it) \
  if (trace) trace[(it) * 16 + (slot)] = gtimer()
#define TC(slot, it) \
  if (trace) trace[(it) * 16 + (slot)] = clock64()
  // head-major order (kv head slowest, heaviest causal key tiles first within a head): the
  // resident CTAs reduce into one kv head's dQ rows
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
      if ((i >= E_QF && i < E_QF + NQ) || i == E_DOF) cnt = 33;
      if (i == E_PR || i == E_DSR) cnt = 32 * NCW;
      if (i == E_DQF) cnt = 128;
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

  if (warp == PRODW) {
    // ------------------------------------------------------------------ TMA producer
    const int lane = threadIdx.x % 32;
    if (T > 0) {
      if (lane == 0) {
        tc::mbar_expect_tx(bar(E_KV), 2 * TILE);
        for (int b = 0; b < 2; ++b) {
          tc::tma_load_2d(sK + b * 16384, &tmK, kvh * D + b * 64, P.k_row0 + n0, bar(E_KV));
          tc::tma_load_2d(sV + b * 16384, &tmV, kvh * D + b * 64, P.k_row0 + n0, bar(E_KV));
        }
      }
      // lse / delta of iteration it, 4 query rows per lane, fetched one iteration ahead
      float pl[4], pd[4];
      auto fetch = [&](int it) {
        const int h = h_lo + it / nqt, m0 = m_begin + (it % nqt) * BQ;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
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
        const int s = it % NQ;
        const int h = h_lo + it / nqt, m0 = m_begin + (it % nqt) * BQ;
        if (it >= NQ) tc::mbar_wait(bar(E_QE + s), ((it - NQ) / NQ) & 1);
        if (lane == 0) {
          tc::mbar_expect_tx(bar(E_QF + s), TILE);
          for (int b = 0; b < 2; ++b)
            tc::tma_load_2d(sQ + s * TILE + b * 16384, &tmQ, h * D + b * 64, P.q_row0 + m0, bar(E_QF + s));
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
          sLse[s * 128 + lane + 32 * k] = pl[k] == -INFINITY ? -INFINITY : -pl[k] * kLog2e;
        tc::mbar_arrive(bar(E_QF + s));
        if (it >= 1) tc::mbar_wait(bar(E_DOE), (it - 1) & 1);
        if (lane == 0) {
          tc::mbar_expect_tx(bar(E_DOF), TILE);
          for (int b = 0; b < 2; ++b)
            tc::tma_load_2d(sdO + b * 16384, &tmDO, h * D + b * 64, P.q_row0 + m0, bar(E_DOF));
        }
        // the delta slot is free once phase B of the previous iteration has read it (dV / dP
        // of this iteration come after dK of the previous, which waits for that phase anyway)
        if (it >= 1) tc::mbar_wait(bar(E_DSR), (it - 1) & 1);
#pragma unroll
        for (int k = 0; k < 4; ++k) sDl[lane + 32 * k] = -pd[k] * a.scale;
        if (it + 1 < T) fetch(it + 1);
        tc::mbar_arrive(bar(E_DOF));
      }
    }
  } else if (warp == MMAW) {
    // ---------------------------------------------------------------------- MMA issuer
    if (tc::elect_one() && T > 0) {
      constexpr uint32_t id_s = tc::idesc_bf16(128, BQ, false, false);  // S^T, dP^T
      constexpr uint32_t id_kv = tc::idesc_bf16(128, D, false, true);   // dV, dK (A in TMEM)
      constexpr uint32_t id_q = tc::idesc_bf16(BQ, D, true, true);      // dQ = dS K
      // (K-step loops are not unrolled: the issuer runs at 56 registers and one MMA per 64
      // tensor cycles leaves ample issue time)
      auto kxq = [&](uint32_t d_col, uint32_t a_tile, uint32_t b_tile) {  // 128 x 128 x d, both K-major
#pragma unroll 1
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t o = (ks >> 2) * 16384 + (ks & 3) * 32;
          tc::mma_ss(tmem + d_col, tc::sdesc(a_tile + o, 16, 1024), tc::sdesc(b_tile + o, 16, 1024), id_s, ks > 0);
        }
      };
      // acc (+)= (P^T or dS^T in TMEM cols [a_col + 64c, +32)) . (dO or Q, MN-major), K = 128 queries
      auto tmem_a = [&](uint32_t d_col, uint32_t a_col, uint32_t b_tile, bool first) {
#pragma unroll 1
        for (int kk = 0; kk < BQ / 16; ++kk)
          tc::mma_ts(tmem + d_col, tmem + a_col + (kk >> 2) * 64 + (kk & 3) * 8,
                     tc::sdesc(b_tile + kk * 2048, 16384, 1024), id_kv, (!first || kk > 0) ? 1u : 0u);
      };
      tc::mbar_wait(bar(E_KV), 0);
      // prologue: S(0), dP(0), dV(0)
      tc::mbar_wait(bar(E_QF), 0);
      tc::fence_after();
      kxq(T_S, sK, sQ);
      tc::commit(bar(E_SR));
      tc::mbar_wait(bar(E_DOF), 0);
      tc::fence_after();
      kxq(T_DP, sV, sdO);
      tc::commit(bar(E_DPR));
      tc::mbar_wait(bar(E_PR), 0);
      tc::fence_after();
      tmem_a(T_DV, T_S, sdO, true);
      tc::commit(bar(E_DOE));
      for (int it = 0; it < T; ++it) {
        const int s = it % NQ;
        TC(0, it);
        if (it + 1 < T) {  // S^T(i+1): P^T(i) was read by dV(i), issued before
          tc::mbar_wait(bar(E_QF + (it + 1) % NQ), ((it + 1) / NQ) & 1);
          tc::fence_after();
          kxq(T_S, sK, sQ + ((it + 1) % NQ) * TILE);
          tc::commit(bar(E_SR));
        }
        tc::mbar_wait(bar(E_DSR), it & 1);
        tc::fence_after();
        TC(1, it);
        // dQ = dS K first (M = 128 queries: the dS^T smem tile read MN-major; B = K MN-major) into
        // the dP^T columns phase B has consumed, so its drain starts one product earlier
#pragma unroll 1
        for (int kk = 0; kk < 8; ++kk)
          tc::mma_ss(tmem + T_DP, tc::sdesc(sdS + kk * 2048, 16384, 1024), tc::sdesc(sK + kk * 2048, 16384, 1024),
                     id_q, kk > 0 ? 1u : 0u);
        tc::commit(bar(E_MD));
        // dK += dS^T Q with dS^T read K-major from the same smem tile (queries 64c.. in block c)
#pragma unroll 1
        for (int kk = 0; kk < BQ / 16; ++kk)
          tc::mma_ss(tmem + T_DK, tc::sdesc(sdS + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                     tc::sdesc(sQ + s * TILE + kk * 2048, 16384, 1024), id_kv, (it > 0 || kk > 0) ? 1u : 0u);
        tc::commit(bar(E_QE + s));  // Q(i) and the dS^T smem tile are free
        if (it + 1 < T) {
          // dP(i+1) first: phase B(i+1) is on the critical path, dV(i+1) (after phase A) is not
          tc::mbar_wait(bar(E_DOF), (it + 1) & 1);
          tc::mbar_wait(bar(E_DQF), it & 1);  // dQ(i) left the dP^T columns
          tc::fence_after();
          TC(3, it);
          kxq(T_DP, sV, sdO);
          tc::commit(bar(E_DPR));
          tc::mbar_wait(bar(E_PR), (it + 1) & 1);  // P^T(i+1)
          tc::fence_after();
          TC(2, it);
          tmem_a(T_DV, T_S, sdO, false);  // dV += P^T dO
          tc::commit(bar(E_DOE));
        }
      }
      tc::commit(bar(E_FIN));
    }
  } else if (warp < NCW) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(REG_C));
    // ----------------------------------- softmax gradient (lane = key, query half c = w >> 2)
    const int qd = warp & 3, c = warp >> 2;
    const int t = qd * 32 + (threadIdx.x & 31);  // key row in the tile == TMEM lane
    const uint32_t lb = (uint32_t)(qd * 32) << 16;
    const float sl2 = a.scale * kLog2e;
    const int key = n0 + t;
    for (int it = 0; it < T; ++it) {
      const int m0 = m_begin + (it % nqt) * BQ + 64 * c;
      // causal admission: query m0 + j sees this key iff j >= ilo. Queries past the problem end
      // carry lse = -inf from the producer (P = 0), so only the causal bound and keys past the
      // problem end (ilo = 64: nothing admitted) need a mask.
      int ilo = P.causal ? max(0, key - P.off - m0) : 0;
      if (key >= P.nk) ilo = 64;
      const bool full = ilo == 0;
      // phase A: P = exp2(s*scale*log2e - lse*log2e), kept in registers, P^T to TMEM
      tc::mbar_wait(bar(E_SR), it & 1);
      tc::fence_after();
      if (warp == 0 && t == 0) TR(4, it);
      if (warp == 0 && t == 0) TC(10, it);
      const float4* nl4 = reinterpret_cast<const float4*>(sLse + (it % NQ) * 128 + 64 * c);
      // P stays in registers in fp32 for phase B (dS = P (dP - delta) from the unrounded P)
      float pf[64];
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        // queries 32*h2.. of the half: their S^T columns [64c + 32h2, +32) are read before the
        // P^T columns [64c + 16h2, +16) they map to are written
        uint32_t rs[32];
        float p[32];
        tc::tmem_ld32(tmem + lb + T_S + 64 * c + 32 * h2, rs);
        tc::tmem_wait_ld();
        tc::reg_fence(rs);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 nl = nl4[8 * h2 + j];
          const float nv[4] = {nl.x, nl.y, nl.z, nl.w};
          // half of the exponentials on the FMA pipe (cubic exp2, rel. error 8e-5, far below the
          // bf16 rounding of P), half on the MUFU: 16 ex2/clk/SM would otherwise bound phase A
          if ((j & 1) == 0 || !kPolyExp) {
#pragma unroll
            for (int e = 0; e < 4; ++e) p[4 * j + e] = fast_exp2(fmaf(__uint_as_float(rs[4 * j + e]), sl2, nv[e]));
          } else {
#pragma unroll
            for (int e = 0; e < 4; e += 2) {
              const float2 r2 = poly_exp2x2(fmaf(__uint_as_float(rs[4 * j + e]), sl2, nv[e]),
                                            fmaf(__uint_as_float(rs[4 * j + e + 1]), sl2, nv[e + 1]));
              p[4 * j + e] = r2.x, p[4 * j + e + 1] = r2.y;
            }
          }
        }
        if (!full) {
#pragma unroll
          for (int e = 0; e < 32; ++e) p[e] = 32 * h2 + e >= ilo ? p[e] : 0.f;
        }
        uint32_t wp[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) wp[i] = pack_bf16(p[2 * i], p[2 * i + 1]);
#pragma unroll
        for (int e = 0; e < 32; ++e) pf[32 * h2 + e] = p[e];
        tc::tmem_st16(tmem + lb + T_S + 64 * c + 16 * h2, wp);
      }
      tc::tmem_wait_st();
      tc::fence_before();
      tc::mbar_arrive(bar(E_PR));
      if (warp == 0 && t == 0) TR(9, it);
      if (warp == 0 && t == 0) TC(11, it);
      // phase B: dS = P (dP*scale - delta*scale) -> dS^T to TMEM (dK) and smem (dQ)
      tc::mbar_wait(bar(E_DPR), it & 1);
      if (it >= 1) tc::mbar_wait(bar(E_QE + (it - 1) % NQ), ((it - 1) / NQ) & 1);  // dQ / dK(i-1) read dS^T
      tc::fence_after();
      if (warp == 0 && t == 0) TR(5, it);
      if (warp == 0 && t == 0) TC(12, it);
      const float4* dl4 = reinterpret_cast<const float4*>(sDl + 64 * c);
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        uint32_t rp[32], wd[16];
        tc::tmem_ld32(tmem + lb + T_DP + 64 * c + 32 * h2, rp);
        tc::tmem_wait_ld();
        tc::reg_fence(rp);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 dl = dl4[8 * h2 + j];
          const float dv[4] = {dl.x, dl.y, dl.z, dl.w};
#pragma unroll
          for (int e = 0; e < 4; e += 2) {
            const int w2 = (4 * j + e) / 2;  // pair index within this 32-query chunk
            const int q = 32 * h2 + 4 * j + e;
            wd[w2] = pack_bf16(pf[q] * fmaf(__uint_as_float(rp[4 * j + e]), a.scale, dv[e]),
                               pf[q + 1] * fmaf(__uint_as_float(rp[4 * j + e + 1]), a.scale, dv[e + 1]));
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // dS^T rows of the smem tile: A of dQ (MN-major) and of dK (K-major)
          const uint32_t addr = tc::sw128(sdS + c * 16384, t, 4 * h2 + k);
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};\n" ::"r"(addr), "r"(wd[4 * k]), "r"(wd[4 * k + 1]),
                       "r"(wd[4 * k + 2]), "r"(wd[4 * k + 3]));
        }
      }
      tc::fence_proxy_async();
      tc::fence_before();
      tc::mbar_arrive(bar(E_DSR));
      if (warp == 0 && t == 0) TR(6, it);
      if (warp == 0 && t == 0) TC(13, it);
    }
    // dV epilogue: half c owns columns [64c, 64c+64)
    __nv_bfloat16* dvb = a.dv_bf16 ? reinterpret_cast<__nv_bfloat16*>(a.dv_bf16) +
                                         (int64_t)(P.k_row0 + key) * a.dkv_bf16_row_stride + kvh * D
                                   : nullptr;
    if (T > 0) {
      tc::mbar_wait(bar(E_FIN), 0);
      tc::fence_after();
      float* dv = a.dv_acc + (int64_t)(P.k_row0 + key) * a.dkv_row_stride + kvh * D;
#pragma unroll
      for (int ci = 0; ci < 2; ++ci) {
        const int cc = 2 * c + ci;
        uint32_t r[32];
        tc::tmem_ld32(tmem + lb + T_DV + cc * 32, r);
        tc::tmem_wait_ld();
        if (key < P.nk) {
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
    } else if (dvb && key < P.nk) {
      uint32_t z[32] = {};
#pragma unroll
      for (int ci = 0; ci < 2; ++ci) store_bf16x32(dvb + (2 * c + ci) * 32, z);
    }
  } else if (warp >= DRAIN0 && warp < DRAIN0 + 4) {
    // ------------------------------ dQ drain (lane = query row of the dQ tile) + dK epilogue
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(REG_DQ));
    const int w = warp - DRAIN0, lane = threadIdx.x % 32;
    const uint32_t lb = (uint32_t)(w * 32) << 16;
    const uint32_t slot0 = sStg + w * 2 * 4096;  // 2 x [32 rows x 32 fp32], 128B-swizzled rows
    for (int it = 0; it < T; ++it) {
      const int h = h_lo + it / nqt, m0 = m_begin + (it % nqt) * BQ;
      tc::mbar_wait(bar(E_MD), it & 1);
      tc::fence_after();
      if (w == 0 && lane == 0) TR(7, it);
      if (w == 0 && lane == 0) TC(14, it);
      // the whole 128-column row first: dP(i+1) waits for these columns
      uint32_t r[4][32];
#pragma unroll
      for (int j = 0; j < 4; ++j) tc::tmem_ld32(tmem + lb + T_DP + 32 * j, r[j]);
      tc::tmem_wait_ld();
      tc::fence_before();
      tc::mbar_arrive(bar(E_DQF));
      if (w == 0 && lane == 0) TR(8, it);
      if (w == 0 && lane == 0) TC(15, it);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t slot = slot0 + (j & 1) * 4096;
        if (lane == 0) tc::bulk_wait_read<1>();  // the reduce issued two chunks ago has read it
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k)
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};\n" ::"r"(tc::sw128(slot, lane, k)), "r"(r[j][4 * k]),
                       "r"(r[j][4 * k + 1]), "r"(r[j][4 * k + 2]), "r"(r[j][4 * k + 3]));
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tc::tma_reduce_add_2d(&tmDQ, slot, h * D + 32 * j, P.q_row0 + m0 + 32 * w);
          tc::bulk_commit();
        }
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
        tc::tmem_ld32(tmem + lb + T_DK + cc * 32, r);
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
    } else if (dkb && ck < P.nk) {
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

extern long long* g_bwd_trace;

bool tc_bwd_q128_supported(const BwdArgs& a) {
  auto al = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; };
  return a.d == D && al(a.q) && al(a.k) && al(a.v) && al(a.dout) && al(a.dq_acc) &&
         (a.q_row_stride * 2) % 16 == 0 && (a.kv_row_stride * 2) % 16 == 0 &&
         a.o_row_stride == a.q_row_stride && (a.dq_row_stride * 4) % 16 == 0 && a.dkv_row_stride % 4 == 0;
}

void launch_attn_bwd_q128(const BwdArgs& a, const ProblemSet& in, cudaStream_t s) {
  ProblemSet ps;
  copy_problems(ps, in);
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
      !make_tma_2d_f32(&tdq, a.dq_acc, (uint64_t)a.hm.hq * D, qrows, (uint64_t)a.dq_row_stride, 32))
    launch_error("attn_bwd_q128", "TMA descriptor encode failed (q/k/v/dout/dq base, strides or extents)");
  with_problem_set(ps, [&](const auto& set) {
    using PS = std::decay_t<decltype(set)>;
    ensure_smem_for(attn_bwd_q128_kernel<PS>, SMEM);
    attn_bwd_q128_kernel<PS><<<dim3(tiles * a.hm.hkv), NTHREADS, SMEM, s>>>(tq, tk, tv, tdo, tdq, args, set);
  });
  note_launch();
}

}  // namespace spattn
