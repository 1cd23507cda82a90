// tcgen05 attention backward with 64-row query tiles, head_dim 64 or 128 (sm_100a).
//
// One CTA = one 128-row key/value tile x one kv head; it loops over every (query head of the
// GQA group, 64-row query tile) that sees the tile. TMEM (512 columns, lane = key row unless
// noted) is double-buffered per query tile so the softmax-gradient math of tile i overlaps the
// dV/dK/dQ MMAs of tile i-1:
//   S^T_b  = K Q^T          cols [64b, 64b+64)        P^T_b (bf16) written back over it
//   dP^T_b = V dO^T         cols [128+64b, +64)        dQ^T_b (lane = head-dim index) reuses it
//   dV    += P^T_b dO       cols [256, 256+D)          (A operand from TMEM)
//   dK    += dS^T_b Q       cols [256+D, 256+2D)       (A operand from TMEM: dS^T_b)
//   dQ^T_b = K^T dS^T_b     M = 128 (head dim; for D = 64 rows 64-127 are padding that reads
//                           the V tile and is never drained), N = 64 queries, K = 128 keys
// MMA issue order: S(i), dP(i), [dV dK dQ](i-1), S(i+1), ... The dQ warpgroup drains dQ^T
// (warp w owns head-dim columns 32w..32w+31) through an 8 KB smem slot per warp into the fp32
// accumulator with TMA reduce-add. attn_block_backward (attention.cpp:167-216).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include "tc.cuh"

namespace spattn {
namespace {

constexpr int BQ = 64;
// Warp roles: NSMW softmax-gradient warps (4: one per TMEM lane quadrant, 64 queries per thread;
// 8 — two per quadrant, one 32-query chunk each — measured no faster for either head dim:
// 711 vs 746 TFLOP/s at d=64, L=32K), 4 dQ drain warps, the TMA producer, the TMEM allocator and
// (last) the MMA issuer.
template <int D>
struct Roles {
  static constexpr int NSMW = 4;
  static constexpr int DRAIN0 = NSMW;
  static constexpr int PRODW = DRAIN0 + 4, TALLOCW = PRODW + 1, MMAW = PRODW + 3;
  static constexpr int NTHREADS = (PRODW + 4) * 32;
  // registers per thread: softmax / drain / control, sum over warps <= 2048
  static constexpr int REG_SM = NSMW == 4 ? 232 : 160, REG_DQ = NSMW == 4 ? 120 : 96,
                       REG_CTL = NSMW == 4 ? 152 : 96;
  static_assert(NSMW * REG_SM + 4 * REG_DQ + 4 * REG_CTL <= 2048, "register budget");
};
constexpr int NSTG = 1;                     // dQ staging slots per drain warp

enum {
  E_KV = 0,
  E_QF = 1,                 // [NST_MAX]
  E_QE = E_QF + 4,          // [NST_MAX]
  E_SF = E_QE + 4,          // [2]
  E_DPF = E_SF + 2,         // [2]
  E_PR = E_DPF + 2,         // [2] 32 * NSMW arrivals
  E_MD = E_PR + 2,          // [2]
  E_DQF = E_MD + 2,         // [2] 128 arrivals
  E_FIN = E_DQF + 2,
  E_N = E_FIN + 1
};

// Shared-memory layout per head dim (128-byte-swizzled 64-column blocks: 16 KB per 128 K/V rows,
// 8 KB per 64 Q/dO rows). head_dim 64 has room for a deeper Q/dO pipeline.
template <int D>
struct Q64 {
  static constexpr int NB = D / 64;                 // 64-column blocks per row
  static constexpr int NST = D == 64 ? 4 : 3;       // Q/dO pipeline stages
  static constexpr int KV_TILE = 128 * D * 2;
  static constexpr int Q_TILE = BQ * D * 2;
  static constexpr int K_OFF = 0, V_OFF = KV_TILE;
  static constexpr int Q_OFF = 2 * KV_TILE;
  static constexpr int DO_OFF = Q_OFF + NST * Q_TILE;
  static constexpr int DS_OFF = DO_OFF + NST * Q_TILE;    // 2 x [128 keys x 64 queries] bf16
  static constexpr int STG_OFF = DS_OFF + 2 * 16384;      // 4 warps x NSTG x [64 queries x 32 fp32]
  static constexpr int LD_OFF = STG_OFF + 4 * NSTG * 8192;  // lse*log2e, delta: [NST][64] each
  static constexpr int BAR_OFF = LD_OFF + 2 * NST * 64 * 4;
  static constexpr int SMEM = BAR_OFF + E_N * 8 + 16;
  static_assert(NST <= 4, "barrier slots");
};

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

// Softmax gradient of one 32-query chunk for one key (thread): P = 2^(s*scale*log2e - lse*log2e)
// and dS = P (dP - delta), both packed to bf16 pairs (attention.cpp:199-209). MASK (only for
// tiles crossing the causal diagonal or the row end) zeroes queries outside [ilo, ihi).
// dS is produced already multiplied by the softmax scale (dl4 holds -delta*scale): the dQ and
// dK accumulators then need no rescaling (dS scale = scale * P (dP - delta)).
// The per-query -lse*log2e / -delta*scale come from shared memory as warp-uniform 16-byte loads
// (four queries per load): this kernel is bound by shared-memory wavefronts (tensor-core
// operand reads + these loads + the dS^T and dQ stores), and each load instruction is one
// wavefront whatever its width.
template <bool MASK>
__device__ __forceinline__ void grad_chunk(const uint32_t (&rs)[32], const uint32_t (&rp)[32], const float4* nl4,
                                           const float4* dl4, float sl2, float sc, int ilo, int ihi,
                                           uint32_t (&wp)[16], uint32_t (&wd)[16]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 nl = nl4[j], dl = dl4[j];
    const float nv[4] = {nl.x, nl.y, nl.z, nl.w}, dv[4] = {dl.x, dl.y, dl.z, dl.w};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = 2 * j + h;
      float px = fast_exp2(fmaf(__uint_as_float(rs[2 * i]), sl2, nv[2 * h]));
      float py = fast_exp2(fmaf(__uint_as_float(rs[2 * i + 1]), sl2, nv[2 * h + 1]));
      if (MASK) {
        px = (2 * i >= ilo && 2 * i < ihi) ? px : 0.f;
        py = (2 * i + 1 >= ilo && 2 * i + 1 < ihi) ? py : 0.f;
      }
      wp[i] = pack_bf16(px, py);
      wd[i] = pack_bf16(px * fmaf(__uint_as_float(rp[2 * i]), sc, dv[2 * h]),
                        py * fmaf(__uint_as_float(rp[2 * i + 1]), sc, dv[2 * h + 1]));
    }
  }
}

// Profiling switches (wrong results by design) exist only in -DSPATTN_PROFILING builds.
#ifdef SPATTN_PROFILING
#define BWD_DBG(bit) ((a.debug & (bit)) != 0)
#else
#define BWD_DBG(bit) false
#endif

template <int D, class PS>
__global__ void __launch_bounds__(Roles<D>::NTHREADS, 1)
    attn_bwd_tc_q64_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                           const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                           const __grid_constant__ CUtensorMap tmDQ, BwdArgs a, PS ps) {
  using L = Q64<D>;
  using R = Roles<D>;
  constexpr int NSMW = R::NSMW, DRAIN0 = R::DRAIN0, PRODW = R::PRODW, TALLOCW = R::TALLOCW, MMAW = R::MMAW,
                REG_SM = R::REG_SM, REG_DQ = R::REG_DQ, REG_CTL = R::REG_CTL;
  constexpr int NST = L::NST, KV_TILE = L::KV_TILE, Q_TILE = L::Q_TILE, K_OFF = L::K_OFF, V_OFF = L::V_OFF,
                Q_OFF = L::Q_OFF, DO_OFF = L::DO_OFF, DS_OFF = L::DS_OFF, STG_OFF = L::STG_OFF,
                LD_OFF = L::LD_OFF, BAR_OFF = L::BAR_OFF, NB = L::NB;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  if (sbase & 1023) __trap();
  const uint32_t sK = sbase + K_OFF, sV = sbase + V_OFF, sQ = sbase + Q_OFF, sdO = sbase + DO_OFF,
                 sdS = sbase + DS_OFF, sStg = sbase + STG_OFF;
  float* sL = reinterpret_cast<float*>(smem + LD_OFF);  // [NST][64] -lse * log2e (-inf: empty row)
  float* sDl = sL + NST * 64;                           // [NST][64] delta
  const uint32_t bars = sbase + BAR_OFF;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + BAR_OFF + E_N * 8);
  auto bar = [&](int i) { return bars + 8u * i; };

  const int warp = threadIdx.x / 32;
  long long* trace = (a.trace && blockIdx.x == 0) ? a.trace : nullptr;
  // debug bit 4: record only the iteration-start event (minimal perturbation)
  const bool tr_all = !BWD_DBG(4);
#define TR(slot, it) \
  if (trace && (tr_all || (slot) == 0)) trace[(it) * 16 + (slot)] = clock64()
  // 1-D grid, kv head fastest: the heaviest causal key tiles of every head run first (LPT)
  const HeadMap hm = a.hm;
  const int ntiles = ps.tile_prefix[ps.n];
  // head-major order (kv head slowest, heaviest causal key tiles first within a head): the
  // resident CTAs then reduce into one kv head's dQ rows (64 MB at c2) instead of all of them
  // (512 MB), which keeps the fp32 dQ partial sums L2-resident (measured 22.3 -> 21.4 ms at c2).
  // debug bit 8 restores the tile-major order for A/B runs.
  const bool head_major = !BWD_DBG(8);
  const int tile = head_major ? blockIdx.x % ntiles : blockIdx.x / hm.hkv;
  const int kvh = head_major ? blockIdx.x / ntiles : blockIdx.x % hm.hkv;
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
      const bool many = (i >= E_PR && i < E_PR + 2) || (i >= E_DQF && i < E_DQF + 2);
      // a stage is full after the TMA bytes and the producer warp's 32 lse/delta stores
      const bool stage = i >= E_QF && i < E_QF + NST;
      const bool pr = i >= E_PR && i < E_PR + 2;
      tc::mbar_init(bar(i), pr ? 32 * NSMW : many ? 128 : stage ? 33 : 1);
    }
    tc::fence_barrier_init();
  }
  if (warp == TALLOCW) tc::tmem_alloc<512>(smem_u32(tmem_slot));
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tDV = tmem + 256, tDK = tmem + 256 + D;
  if (warp >= PRODW) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(REG_CTL));

  // Roles. The scheduler favours the highest warp id, so the single-thread MMA issuer is the
  // last warp and the producer sits above the math warps: warps 0-3 softmax-gradient, 4-7 dQ
  // drain, 8 TMA producer, 9 TMEM allocator, 11 MMA issuer.
  if (warp == PRODW) {
    // ------------------------------------------------------------------ TMA producer
    // lane 0 issues the TMA loads; all 32 lanes stage this tile's lse/delta (2 query rows each)
    // into the stage's smem slot and arrive on the stage barrier, so the softmax warpgroup
    // never waits on global-memory latency
    const int lane = threadIdx.x % 32;
    if (T > 0) {
      if (lane == 0) {
        tc::mbar_expect_tx(bar(E_KV), 2 * KV_TILE);
        for (int b = 0; b < NB; ++b) {
          tc::tma_load_2d(sK + b * 16384, &tmK, kvh * D + b * 64, P.k_row0 + n0, bar(E_KV));
          tc::tma_load_2d(sV + b * 16384, &tmV, kvh * D + b * 64, P.k_row0 + n0, bar(E_KV));
        }
      }
      // lse/delta of iteration it are fetched into registers one iteration ahead, so their
      // global latency overlaps the wait for the stage instead of following it
      float pl[2], pd[2];
      auto fetch = [&](int it) {
        const int h = h_lo + it / nqt, m0 = m_begin + (it % nqt) * BQ;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int row = m0 + lane + 32 * k;
          pl[k] = -INFINITY, pd[k] = 0.f;  // stored negated: p = 2^(s*scale*log2e + l2)
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
        if (lane == 0) TR(14, it);
        if (it >= NST) tc::mbar_wait(bar(E_QE + st), ((it - NST) / NST) & 1);
        if (lane == 0) {
          TR(15, it);
          tc::mbar_expect_tx(bar(E_QF + st), 2 * Q_TILE);
          for (int b = 0; b < NB; ++b) {
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
      constexpr uint32_t id_s = tc::idesc_bf16(128, BQ, false, false);  // S^T, dP^T
      constexpr uint32_t id_kv = tc::idesc_bf16(128, D, false, true);   // dV, dK
      constexpr uint32_t id_q = tc::idesc_bf16(128, BQ, true, true);    // dQ^T
      auto tail = [&](int i) {  // dV, dK, dQ^T of iteration i
        const int b = i & 1, st = i % NST;
        const uint32_t q = sQ + st * Q_TILE, dO = sdO + st * Q_TILE, ds = sdS + b * 16384;
        TR(5, i);
        tc::mbar_wait(bar(E_PR + b), (i >> 1) & 1);
        TR(6, i);
        tc::fence_after();
        // P^T / dS^T of query chunk c (32 queries) sit in that chunk's own S^T columns:
        // P^T at [64b + 32c, +16), dS^T at [64b + 32c + 16, +16) (16 queries = 8 columns per K step)
#pragma unroll
        for (int kk = 0; kk < BQ / 16; ++kk)
          tc::mma_ts(tDV, tmem + 64 * b + (kk >> 1) * 32 + (kk & 1) * 8, tc::sdesc(dO + kk * 2048, 8192, 1024),
                     id_kv, (i > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < BQ / 16; ++kk)
          tc::mma_ts(tDK, tmem + 64 * b + (kk >> 1) * 32 + 16 + (kk & 1) * 8, tc::sdesc(q + kk * 2048, 8192, 1024),
                     id_kv, (i > 0 || kk > 0) ? 1u : 0u);
        tc::commit(bar(E_QE + st));
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          tc::mma_ss(tmem + 128 + 64 * b, tc::sdesc(sK + kk * 2048, 16384, 1024),
                     tc::sdesc(ds + kk * 2048, 8192, 1024), id_q, kk > 0 ? 1u : 0u);
        tc::commit(bar(E_MD + b));
        TR(7, i);
      };
      tc::mbar_wait(bar(E_KV), 0);
      for (int it = 0; it < T; ++it) {
        const int b = it & 1, st = it % NST;
        const uint32_t q = sQ + st * Q_TILE, dO = sdO + st * Q_TILE;
        TR(0, it);
        tc::mbar_wait(bar(E_QF + st), (it / NST) & 1);
        TR(1, it);
        tc::fence_after();
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t ko = (ks >> 2) * 16384 + (ks & 3) * 32, qo = (ks >> 2) * 8192 + (ks & 3) * 32;
          tc::mma_ss(tmem + 64 * b, tc::sdesc(sK + ko, 16, 1024), tc::sdesc(q + qo, 16, 1024), id_s, ks > 0);
        }
        tc::commit(bar(E_SF + b));
        TR(2, it);
        if (it >= 2 && !BWD_DBG(64)) {  // dQ^T of it-2 (same columns) must be drained (debug 64: skip, wrong dq)
          tc::mbar_wait(bar(E_DQF + b), ((it - 2) >> 1) & 1);
          tc::fence_after();
        }
        TR(3, it);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t ko = (ks >> 2) * 16384 + (ks & 3) * 32, qo = (ks >> 2) * 8192 + (ks & 3) * 32;
          tc::mma_ss(tmem + 128 + 64 * b, tc::sdesc(sV + ko, 16, 1024), tc::sdesc(dO + qo, 16, 1024), id_s,
                     ks > 0);
        }
        tc::commit(bar(E_DPF + b));
        TR(4, it);
        if (it >= 1) tail(it - 1);
      }
      tail(T - 1);
      tc::commit(bar(E_FIN));
    }
  } else if (warp < NSMW) {
    // ----------------------------------------------- softmax-gradient warpgroup (lane = key)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(REG_SM));
    const int t = (warp & 3) * 32 + (threadIdx.x & 31);  // key row within the tile == TMEM lane
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    // query chunks of 32 this warp owns: both (4 warps) or chunk warp/4 (8 warps)
    const int cc_lo = NSMW == 8 ? warp >> 2 : 0, cc_hi = NSMW == 8 ? cc_lo + 1 : 2;
    const float sl2 = a.scale * kLog2e;
    const int c = n0 + t;
    for (int it = 0; it < T; ++it) {
      const int b = it & 1;
      const int m0 = m_begin + (it % nqt) * BQ;
      const int lb = (it % NST) * 64;  // this tile's lse/delta slot (complete once S^T is)
      if (warp == 0 && t == 0) TR(8, it);
      int ilo = 0, ihi = min(BQ, P.nq - m0);
      if (c >= P.nk) ihi = 0;
      if (P.causal) ilo = max(0, c - P.off - m0);
      tc::mbar_wait(bar(E_SF + b), (it >> 1) & 1);
      tc::mbar_wait(bar(E_DPF + b), (it >> 1) & 1);
      if (it >= 2) tc::mbar_wait(bar(E_MD + b), ((it - 2) >> 1) & 1);  // dS^T_b read by dK/dQ
      tc::fence_after();
      if (warp == 0 && t == 0) TR(9, it);
      const uint32_t ds = sdS + b * 16384;
      // chunk c (32 queries) of S^T / dP^T: the first chunk is loaded up front, the second (4
      // warps) after the first is computed; each chunk's P^T / dS^T go back into its own S^T
      // columns, which its loads have already emptied
      const float4* lse4 = reinterpret_cast<const float4*>(sL + lb);   // -lse*log2e per query
      const float4* dl4 = reinterpret_cast<const float4*>(sDl + lb);   // -delta*scale per query
#pragma unroll
      for (int cc = cc_lo; cc < cc_hi; ++cc) {
        uint32_t rs[32], rp[32];
        tc::tmem_ld32(tmem + lane_base + 64 * b + cc * 32, rs);
        tc::tmem_ld32(tmem + lane_base + 128 + 64 * b + cc * 32, rp);
        tc::tmem_wait_ld();
        tc::reg_fence(rs);
        tc::reg_fence(rp);
        uint32_t wp[16], wd[16];
        if (BWD_DBG(16)) {  // profiling: no softmax-gradient math (wrong results)
#pragma unroll
          for (int i = 0; i < 16; ++i) wp[i] = rs[i] ^ rp[i], wd[i] = rs[i + 16] ^ rp[i + 16];
        } else {
          grad_chunk<true>(rs, rp, lse4 + cc * 8, dl4 + cc * 8, sl2, a.scale, ilo - cc * 32, ihi - cc * 32, wp,
                           wd);
        }
        tc::tmem_st16(tmem + lane_base + 64 * b + cc * 32, wp);       // P^T: A operand of dV
        tc::tmem_st16(tmem + lane_base + 64 * b + cc * 32 + 16, wd);  // dS^T: A operand of dK
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // dS^T: B operand of dQ^T
          const uint32_t addr = tc::sw128(ds, t, cc * 4 + k);
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};\n" ::"r"(addr), "r"(wd[4 * k]),
                       "r"(wd[4 * k + 1]), "r"(wd[4 * k + 2]), "r"(wd[4 * k + 3]));
        }
      }
      tc::tmem_wait_st();
      tc::fence_proxy_async();
      tc::fence_before();
      tc::mbar_arrive(bar(E_PR + b));
      if (warp == 0 && t == 0) TR(10, it);
    }
    constexpr int NC = D / 32 / (NSMW / 4);  // 32-column chunks of dV per warp
    const int cc0 = NSMW == 8 ? (warp >> 2) * NC : 0;
    __nv_bfloat16* dvb = a.dv_bf16 ? reinterpret_cast<__nv_bfloat16*>(a.dv_bf16) +
                                         (int64_t)(P.k_row0 + c) * a.dkv_bf16_row_stride + kvh * D
                                   : nullptr;
    if (T > 0) {  // dV epilogue
      tc::mbar_wait(bar(E_FIN), 0);
      tc::fence_after();
      float* dv = a.dv_acc + (int64_t)(P.k_row0 + c) * a.dkv_row_stride + kvh * D;
#pragma unroll
      for (int ci = 0; ci < NC; ++ci) {
        const int cc = cc0 + ci;
        uint32_t r[32];
        tc::tmem_ld32(tDV + lane_base + cc * 32, r);
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
      for (int ci = 0; ci < NC; ++ci) store_bf16x32(dvb + (cc0 + ci) * 32, z);
    }
  } else if (warp >= DRAIN0 && warp < DRAIN0 + 4) {
    // ------------------------------------------- dQ warpgroup (lane = head-dim index)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(REG_DQ));
    const int w = warp - DRAIN0, lane = threadIdx.x % 32;
    const uint32_t lane_base = (uint32_t)(w * 32) << 16;
    const uint32_t stg0 = sStg + w * NSTG * 8192;  // NSTG x [64 queries x 32 fp32], 128B-swizzled rows
    for (int it = 0; it < T; ++it) {
      const int b = it & 1;
      const int h = h_lo + it / nqt, m0 = m_begin + (it % nqt) * BQ;
      tc::mbar_wait(bar(E_MD + b), (it >> 1) & 1);
      tc::fence_after();
      if (w == 0 && lane == 0) TR(11, it);
      uint32_t r[2][32];
      tc::tmem_ld32(tmem + lane_base + 128 + 64 * b, r[0]);
      tc::tmem_ld32(tmem + lane_base + 128 + 64 * b + 32, r[1]);
      tc::tmem_wait_ld();
      tc::fence_before();
      tc::mbar_arrive(bar(E_DQF + b));
      if (w == 0 && lane == 0) TR(12, it);
      // (per-lane red.global.add.f32 from registers measured 1.8x slower than this staging, and
      // a quad-transpose via shuffles + red.global.add.v4.f32 1.6x slower: 3620 vs 2229 cycles
      // per iteration — the L2 atomics, not the smem traffic, would bound it)
      if (BWD_DBG(32)) continue;  // profiling: no dQ staging / reduce (wrong dq)
      if (w * 32 >= D) continue;  // head_dim 64: lanes 64-127 of the M=128 dQ^T MMA are padding
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
      if (lane == 0 && !BWD_DBG(1)) {
        tc::tma_reduce_add_2d(&tmDQ, stg, h * D + w * 32, P.q_row0 + m0);
        tc::bulk_commit();
      }
      if (w == 0 && lane == 0) TR(13, it);
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
        tc::tmem_ld32(tDK + lane_base + cc * 32, r);
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
}

int max_rows(const ProblemSet& ps, bool q) {
  int m = 0;
  for (int i = 0; i < ps.n; ++i) m = max(m, q ? ps.p[i].q_row0 + ps.p[i].nq : ps.p[i].k_row0 + ps.p[i].nk);
  return m;
}

}  // namespace

long long* g_bwd_trace = nullptr;  // profiling (spattn_debug_bwd_trace)
void set_bwd_trace(void* p) { g_bwd_trace = static_cast<long long*>(p); }

bool tc_bwd_q64_supported(const BwdArgs& a) {
  auto al = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; };
  return (a.d == 64 || a.d == 128) && al(a.q) && al(a.k) && al(a.v) && al(a.dout) && al(a.dq_acc) &&
         (a.q_row_stride * 2) % 16 == 0 && (a.kv_row_stride * 2) % 16 == 0 &&
         a.o_row_stride == a.q_row_stride && (a.dq_row_stride * 4) % 16 == 0 && a.dkv_row_stride % 4 == 0;
}

template <int D>
void launch_q64_d(const BwdArgs& a, const ProblemSet& in, cudaStream_t s) {
  ProblemSet ps;
  copy_problems(ps, in);
  BwdArgs args = a;
#ifdef SPATTN_PROFILING
  args.debug = getenv("SPATTN_DEBUG") ? atoi(getenv("SPATTN_DEBUG")) : 0;
#else
  args.debug = 0;
#endif
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
  with_problem_set(ps, [&](const auto& set) {
    using PS = std::decay_t<decltype(set)>;
    ensure_smem_for(attn_bwd_tc_q64_kernel<D, PS>, Q64<D>::SMEM);
    attn_bwd_tc_q64_kernel<D, PS><<<dim3(tiles * a.hm.hkv), Roles<D>::NTHREADS, Q64<D>::SMEM, s>>>(tq, tk, tv, tdo, tdq, args,
                                                                                                   set);
  });
  note_launch();
}

void launch_attn_bwd_tc_q64(const BwdArgs& a, const ProblemSet& in, cudaStream_t s) {
  if (a.d == 64)
    launch_q64_d<64>(a, in, s);
  else
    launch_q64_d<128>(a, in, s);
}

}  // namespace spattn
