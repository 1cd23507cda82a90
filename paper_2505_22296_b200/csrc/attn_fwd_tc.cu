// tcgen05 attention forward with two ping-ponged 128-row query tiles per CTA (sm_100a).
//
// One CTA = 256 query rows (tiles A and B) of one head of one problem; 352 threads:
//   warps 0-3  softmax + epilogue of tile A (thread = query row = TMEM lane)
//   warps 4-7  softmax + epilogue of tile B
//   warp 8     TMA producer of Q_A, Q_B (once) and K_j (2-stage ring)
//   warp 9     TMA producer of V_j (2-stage ring) + TMEM allocator
//   warp 10    MMA issuer (highest warp id: the scheduler favours it)
// TMEM (512 columns): S_A [0,128) | S_B [128,256) | O_A [256,256+D) | O_B [256+D, 256+2D).
// P_X is written back as bf16 pairs over the first 64 columns of S_X and consumed from TMEM by
// the P.V MMA (A operand in TMEM), so P never touches shared memory, and each K / V tile staged
// in shared memory serves 256 query rows: per 128x128 tile of work the SMEM port moves 128 KB
// (Q.K^T operands 64 KB, V 32 KB, half a K/V tile of TMA writes 32 KB) instead of the 1-tile
// kernel's 224 KB. MMA order per key tile j:
//   PV_A(j), S_A(j+1), PV_B(j), S_B(j+1)  — the tensor core works on one tile while the other
// tile's softmax runs (in-order execution lets S_X(j+1) overwrite the P_X(j) columns PV_X(j)
// reads). O is rescaled lazily in TMEM (row max grew by > 2^8): when S_X(j) is complete, so is
// PV_X(j-1) (one issuing thread, commits track all earlier MMAs), and PV_X(j) waits for P_X(j).
// attn_block_forward + finalize_piece (attention.cpp:61-115, :151-165); merge mode folds
// merge_piece (:117-149) into the epilogue.
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>

#include "tc.cuh"

namespace spattn {
namespace {

#ifndef SPATTN_PP_POLY_PAIRS
#define SPATTN_PP_POLY_PAIRS 0x8
#endif
// bit e set: the e-th exponential pair of every 8 columns runs on the FMA pipe (poly_exp2x2)
constexpr int kPPPoly = SPATTN_PP_POLY_PAIRS;

template <int D>
struct PPLayout {
  static constexpr int QB = D / 64;
  static constexpr int TILE = 128 * D * 2;
  static constexpr int Q_OFF = 0;         // Q_A | Q_B
  static constexpr int K_OFF = 2 * TILE;  // 2 stages
  static constexpr int V_OFF = 4 * TILE;  // 2 stages
  static constexpr int BAR_OFF = 6 * TILE;
  static constexpr int SMEM = BAR_OFF + 256;
};

// K_i lives in stage i&1 and V_i in stage (i+1)&1, so the commit closing iteration j (after
// S_X(j+1) and PV_X(j)) frees K stage (j+1)&1 and V stage (j+1)&1 together: one barrier F_KVE[s].
enum PPBar {
  F_Q = 0,
  F_KF = 1,    // [2] K stage full
  F_VF = 3,    // [2] V stage full
  F_KVE = 5,   // [2] K/V stage s empty
  F_SF = 7,    // [2] S_X ready (X = A, B)
  F_PF = 9,    // [2] P_X in TMEM (128 arrivals)
  F_PV = 11,   // [2] last PV_X done
  F_N = 13
};

__device__ long long* g_pp_trace = nullptr;  // profiling: per-tile clock64 events of CTA (0,0)
__device__ long long* g_pp_cta = nullptr;    // profiling: per-CTA globaltimer records
__device__ __forceinline__ long long pp_gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int D, class PS>
__global__ void __launch_bounds__(352, 1)
    attn_fwd_pp_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, FwdArgs a, PS ps) {
  using Lay = PPLayout<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  if (sbase & 1023) __trap();
  const uint32_t sQ = sbase + Lay::Q_OFF, sK = sbase + Lay::K_OFF, sV = sbase + Lay::V_OFF;
  const uint32_t bars = sbase + Lay::BAR_OFF;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Lay::BAR_OFF + F_N * 8);
  auto bar = [&](int i) { return bars + 8u * i; };
  const int warp = threadIdx.x / 32;

  // ---- tile decode: heavy causal tiles first, one head's tiles together (K/V reuse in L2)
  const int pi = find_problem(ps, (int)blockIdx.x);
  const AttnProblem P = ps.p[pi];
  int mt = blockIdx.x - ps.tile_prefix[pi];
  if (P.causal) mt = (ps.tile_prefix[pi + 1] - ps.tile_prefix[pi]) - 1 - mt;
  const int m0 = mt * 256;
  const int h = blockIdx.y;
  const HeadMap hm = a.hm;
  const int kvh = (hm.q_head_base + h) / hm.rep - hm.kv_head_base;
  // key tiles each query tile sees (tile B may be empty; tile A never sees more than B when causal)
  auto tiles_of = [&](int x) {
    const int r0 = m0 + 128 * x, valid = min(128, P.nq - r0);
    if (valid <= 0) return 0;
    int n_end = P.nk;
    if (P.causal) n_end = min(P.nk, r0 + valid - 1 + P.off + 1);
    return (max(n_end, 0) + 127) / 128;
  };
  const int ntA = tiles_of(0), ntB = tiles_of(1), nt = max(ntA, ntB);
  long long* trace = (g_pp_trace && blockIdx.x == 0 && blockIdx.y == 0) ? g_pp_trace : nullptr;
#define PTR(slot, j) \
  if (trace) trace[(j) * 32 + (slot)] = clock64()
  long long* ctr = g_pp_cta ? g_pp_cta + 8 * ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) : nullptr;
  if (ctr && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    ctr[0] = pp_gtimer();
    ctr[4] = 2 * nt;
    ctr[5] = smid;
  }

  if (threadIdx.x == 0) {
    for (int i = 0; i < F_N; ++i) tc::mbar_init(bar(i), (i == F_PF || i == F_PF + 1) ? 128 : 1);
    tc::fence_barrier_init();
  }
  if (warp == 9) tc::tmem_alloc<512>(smem_u32(tmem_slot));
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ------------------------------------------------------------ TMA producer: Q, then K
    if (tc::elect_one() && nt > 0) {
      tc::tma_prefetch(&tmQ);
      tc::tma_prefetch(&tmK);
      tc::mbar_expect_tx(bar(F_Q), 2 * Lay::TILE);
      for (int t = 0; t < 2; ++t)
        for (int b = 0; b < Lay::QB; ++b)
          tc::tma_load_2d(sQ + t * Lay::TILE + b * 16384, &tmQ, h * D + b * 64, P.q_row0 + m0 + 128 * t,
                          bar(F_Q));
      for (int j = 0; j < nt; ++j) {
        const int st = j & 1;
        if (j >= 2) tc::mbar_wait(bar(F_KVE + st), ((j - 2) >> 1) & 1);  // commit C_{j-3}
        tc::mbar_expect_tx(bar(F_KF + st), Lay::TILE);
        for (int b = 0; b < Lay::QB; ++b)
          tc::tma_load_2d(sK + st * Lay::TILE + b * 16384, &tmK, kvh * D + b * 64, P.k_row0 + j * 128,
                          bar(F_KF + st));
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------------ TMA producer: V
    if (tc::elect_one() && nt > 0) {
      tc::tma_prefetch(&tmV);
      for (int j = 0; j < nt; ++j) {
        const int st = (j + 1) & 1;
        if (j >= 2) tc::mbar_wait(bar(F_KVE + st), ((j - 1) >> 1) & 1);  // commit C_{j-2}
        tc::mbar_expect_tx(bar(F_VF + st), Lay::TILE);
        for (int b = 0; b < Lay::QB; ++b)
          tc::tma_load_2d(sV + st * Lay::TILE + b * 16384, &tmV, kvh * D + b * 64, P.k_row0 + j * 128,
                          bar(F_VF + st));
      }
    }
  } else if (warp == 10) {
    // ------------------------------------------------------------------------ MMA issuer
    if (tc::elect_one() && nt > 0) {
      constexpr uint32_t id_s = tc::idesc_bf16(128, 128, false, false);
      constexpr uint32_t id_o = tc::idesc_bf16(128, D, false, true);
      auto issue_s = [&](int x, int j) {  // S_x = Q_x K_j^T
        const uint32_t kb = sK + (j & 1) * Lay::TILE, qb = sQ + x * Lay::TILE;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
          tc::mma_ss(tmem + 128 * x, tc::sdesc(qb + off, 16, 1024), tc::sdesc(kb + off, 16, 1024), id_s,
                     ks > 0 ? 1u : 0u);
        }
        tc::commit(bar(F_SF + x));
      };
      auto issue_pv = [&](int x, int j) {  // O_x += P_x V_j, P_x from TMEM
        tc::mbar_wait(bar(F_PF + x), j & 1);
        PTR(16 + x, j);
        tc::fence_after();
        const uint32_t vb = sV + ((j + 1) & 1) * Lay::TILE;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          tc::mma_ts(tmem + 256 + D * x, tmem + 128 * x + kk * 8, tc::sdesc(vb + kk * 2048, 16384, 1024), id_o,
                     (j > 0 || kk > 0) ? 1u : 0u);
      };
      const int ntx[2] = {ntA, ntB};
      tc::mbar_wait(bar(F_Q), 0);
      tc::mbar_wait(bar(F_KF), 0);
      tc::fence_after();
      if (ntA > 0) issue_s(0, 0);
      if (ntB > 0) issue_s(1, 0);
      tc::commit(bar(F_KVE + 0));  // C_{-1}: K_0 read
      for (int j = 0; j < nt; ++j) {
        const bool more = j + 1 < nt;
        PTR(8, j);
        tc::mbar_wait(bar(F_VF + ((j + 1) & 1)), (j >> 1) & 1);
        if (more) tc::mbar_wait(bar(F_KF + ((j + 1) & 1)), ((j + 1) >> 1) & 1);
        tc::fence_after();
        PTR(9, j);
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          if (j < ntx[x]) {
            PTR(4 + 2 * x, j);
            issue_pv(x, j);
            PTR(5 + 2 * x, j);
            if (j + 1 < ntx[x]) {
              issue_s(x, j + 1);
            } else {
              tc::commit(bar(F_PV + x));  // O_x final
            }
          }
        }
        tc::commit(bar(F_KVE + ((j + 1) & 1)));  // C_j: V_j and K_{j+1} read
      }
    }
  } else if (warp < 8) {
    // --------------------------------------------------- softmax warpgroups (A: 0-3, B: 4-7)
    const int x = warp >> 2;  // tile
    const int row = threadIdx.x & 127;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + 128 * x + lane_base, tO = tmem + 256 + D * x + lane_base;
    const float sl2 = a.scale * kLog2e;
    const int r0 = m0 + 128 * x;
    const int qa = r0 + row;
    const int ntx = x == 0 ? ntA : ntB;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < ntx; ++j) {
      tc::mbar_wait(bar(F_SF + x), j & 1);
      tc::fence_after();
      if (row == 0) PTR(2 * x, j);
#ifdef SPATTN_PP_PROBE_BIDLE
      if (x == 1) {  // profiling probe: tile B's softmax does no work (wrong results)
        tc::fence_before();
        tc::mbar_arrive(bar(F_PF + x));
        continue;
      }
#endif
      if (ctr && j == 0 && threadIdx.x == 0) ctr[1] = pp_gtimer();
      float s[128];
      {
        uint32_t r[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tc::tmem_ld32(tS + c * 32, r[c]);
        tc::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 128; ++i) s[i] = __uint_as_float(r[i >> 5][i & 31]);
      }
      if (row == 0) PTR(18 + 4 * x, j);
      const int n0 = j * 128;
      const bool need_mask = (n0 + 128 > P.nk) || (P.causal && n0 + 127 > r0 + P.off);
      if (need_mask) {
        const int lim = P.causal ? min(P.nk - 1, qa + P.off) - n0 : P.nk - 1 - n0;
#pragma unroll
        for (int i = 0; i < 128; ++i) s[i] = i <= lim ? s[i] : -INFINITY;
      }
      // max over raw scores (sl2 > 0): four independent chains, then a tree
      float mx[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) mx[c] = -INFINITY;
#pragma unroll
      for (int i = 0; i < 128; i += 8) {
#pragma unroll
        for (int c = 0; c < 4; ++c) mx[c] = fmaxf(mx[c], fmaxf(s[i + 2 * c], s[i + 2 * c + 1]));
      }
      const float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * sl2;
      if (row == 0 && trace) trace[j * 32 + 19 + 4 * x] = clock64() + (mt > 1e30f ? 1 : 0);
      if (j == 0) {
        m_run = mt;
      } else if (__any_sync(0xffffffffu, mt > m_run + 8.f)) {
        // lazy rescale of O_x and l (O_x holds PV_x(j-1), complete since S_x(j) is)
        const float m_new = fmaxf(m_run, mt);
        const float alpha = (m_run == -INFINITY || m_new == -INFINITY) ? (m_run == m_new ? 1.f : 0.f)
                                                                        : fast_exp2(m_run - m_new);
#pragma unroll 1
        for (int c = 0; c < D / 8; ++c) {
          uint32_t r[8];
          tc::tmem_ld8(tO + c * 8, r);
          tc::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 8; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
          tc::tmem_st8(tO + c * 8, r);
        }
        l_run *= alpha;
        m_run = m_new;
        if (row == 0) PTR(10 + x, j);
      }
      const float muse = m_run == -INFINITY ? 0.f : m_run;
      const uint64_t sc2 = f2_pack(sl2, sl2), nm2 = f2_pack(-muse, -muse);
      uint64_t rs2[2] = {0ull, 0ull};  // packed (even, odd) partial row sums
      uint32_t pw[64];                 // P row as bf16 pairs
#pragma unroll
      for (int e = 0; e < 64; ++e) {
        const float2 av = f2_unpack(f2_fma(f2_pack(s[2 * e], s[2 * e + 1]), sc2, nm2));
        float2 pv;
        if ((kPPPoly >> (e & 3)) & 1) {
          pv = poly_exp2x2(av.x, av.y);
        } else {
          pv.x = fast_exp2(av.x);
          pv.y = fast_exp2(av.y);
        }
        rs2[e & 1] = f2_add(rs2[e & 1], f2_pack(pv.x, pv.y));
        pw[e] = pack_bf16(pv.x, pv.y);
      }
      if (row == 0 && trace) trace[j * 32 + 20 + 4 * x] = clock64() + (pw[63] == 12345u ? 1 : 0);
      // P_x(j) over the first 64 columns of S_x (its scores are in registers now)
      tc::tmem_st32(tS, *reinterpret_cast<uint32_t(*)[32]>(&pw[0]));
      tc::tmem_st32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&pw[32]));
      {
        const float2 r = f2_unpack(f2_add(rs2[0], rs2[1]));
        l_run += r.x + r.y;
      }
      tc::tmem_wait_st();
      if (row == 0) PTR(21 + 4 * x, j);
      tc::fence_before();
      tc::mbar_arrive(bar(F_PF + x));
      if (row == 0) PTR(2 * x + 1, j);
      if (x == 0 && (row & 31) == 0) PTR(12 + (warp & 3), j);
    }
    if (ctr && threadIdx.x == 0) ctr[2] = pp_gtimer();
    // ---- epilogue
    const bool empty = m_run == -INFINITY || !(l_run > 0.f);
    const float inv = empty ? 0.f : 1.f / l_run;
    const float lse_row = empty ? -INFINITY : (m_run + __log2f(l_run)) * kLn2;
    if (ntx > 0) {
      tc::mbar_wait(bar(F_PV + x), 0);
      tc::fence_after();
    }
    const bool valid = qa < P.nq;
    const int64_t grow = (int64_t)(P.q_row0 + qa);
    if (a.acc_o == nullptr) {
      __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(a.o) + grow * a.o_row_stride + h * D;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t r[32];
        if (ntx > 0) {
          tc::tmem_ld32(tO + c * 32, r);
          tc::tmem_wait_ld();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = 0u;
        }
        uint32_t w[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          w[i] = pack_bf16(__uint_as_float(r[2 * i]) * inv, __uint_as_float(r[2 * i + 1]) * inv);
        if (valid) {
          uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
        }
      }
      if (valid) a.lse[grow * a.lse_row_stride + h] = lse_row;
    } else {
      float* lp = a.lse + grow * a.lse_row_stride + h;
      const float la = valid ? *lp : -INFINITY;
      const float lb = lse_row;
      const float mx = fmaxf(la, lb);
      float wa = 1.f, wb = 0.f, ln = la;
      if (mx != -INFINITY) {
        ln = mx + __logf(__expf(la - mx) + __expf(lb - mx));
        wa = __expf(la - ln);
        wb = __expf(lb - ln) * inv;
      }
      float* arow = a.acc_o + grow * a.o_row_stride + h * D;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t r[32];
        if (ntx > 0) {
          tc::tmem_ld32(tO + c * 32, r);
          tc::tmem_wait_ld();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = 0u;
        }
        if (valid) {
          float4* ap = reinterpret_cast<float4*>(arow + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float4 cur = ap[i];
            cur.x = cur.x * wa + __uint_as_float(r[4 * i]) * wb;
            cur.y = cur.y * wa + __uint_as_float(r[4 * i + 1]) * wb;
            cur.z = cur.z * wa + __uint_as_float(r[4 * i + 2]) * wb;
            cur.w = cur.w * wa + __uint_as_float(r[4 * i + 3]) * wb;
            ap[i] = cur;
          }
        }
      }
      if (valid) *lp = ln;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 9) tc::tmem_dealloc<512>(tmem);
  if (ctr && threadIdx.x == 0) ctr[3] = pp_gtimer();
#undef PTR
}

int max_rows_pp(const ProblemSet& ps, bool q) {
  int m = 0;
  for (int i = 0; i < ps.n; ++i) m = max(m, q ? ps.p[i].q_row0 + ps.p[i].nq : ps.p[i].k_row0 + ps.p[i].nk);
  return m;
}

template <int D>
void launch_pp_d(const FwdArgs& a, const ProblemSet& in, cudaStream_t s) {
  ProblemSet ps;
  copy_problems(ps, in);
  ps.tile_prefix[0] = 0;
  for (int i = 0; i < ps.n; ++i) ps.tile_prefix[i + 1] = ps.tile_prefix[i] + (ps.p[i].nq + 255) / 256;
  const int tiles = ps.tile_prefix[ps.n];
  if (tiles == 0 || a.hm.hq == 0) return;
  CUtensorMap tq, tk, tv;
  const uint64_t qw = (uint64_t)a.q_row_stride, kw = (uint64_t)a.kv_row_stride;
  if (!make_tma_2d(&tq, a.q, qw, max_rows_pp(ps, true), qw, 128) ||
      !make_tma_2d(&tk, a.k, kw, max(1, max_rows_pp(ps, false)), kw, 128) ||
      !make_tma_2d(&tv, a.v, kw, max(1, max_rows_pp(ps, false)), kw, 128))
    launch_error("attn_fwd_pp", "TMA descriptor encode failed");
  with_problem_set(ps, [&](const auto& set) {
    using PS = std::decay_t<decltype(set)>;
    ensure_smem_for(attn_fwd_pp_kernel<D, PS>, PPLayout<D>::SMEM);
    attn_fwd_pp_kernel<D, PS><<<dim3(tiles, a.hm.hq), 352, PPLayout<D>::SMEM, s>>>(tq, tk, tv, a, set);
  });
  note_launch();
}

}  // namespace

void set_pp_trace(void* p) { cudaMemcpyToSymbol(g_pp_trace, &p, sizeof(p)); }
void set_pp_cta_trace(void* p) { cudaMemcpyToSymbol(g_pp_cta, &p, sizeof(p)); }

bool tc_fwd_pp_supported(const FwdArgs& a) {
  auto al = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; };
  return (a.d == 64 || a.d == 128) && al(a.q) && al(a.k) && al(a.v) && (a.q_row_stride * 2) % 16 == 0 &&
         (a.kv_row_stride * 2) % 16 == 0;
}

void launch_attn_fwd_tc_pp(const FwdArgs& a, const ProblemSet& ps, cudaStream_t s) {
  if (a.d == 64)
    launch_pp_d<64>(a, ps, s);
  else
    launch_pp_d<128>(a, ps, s);
}

}  // namespace spattn
