// tcgen05 attention forward with two ping-ponged 128-row query tiles per CTA (sm_100a).
//
// One CTA = 256 query rows (tiles A and B) of one head of one problem; 320 threads:
//   warps 0-3  softmax + epilogue of tile A (thread = query row = TMEM lane)
//   warps 4-7  softmax + epilogue of tile B
//   warp 8     TMA producer (Q_A, Q_B once; K_j, V_j into a 2-stage ring) + TMEM allocator
//   warp 9     MMA issuer (highest warp id: the scheduler favours it)
// TMEM (512 columns): S_A [0,128) | S_B [128,256) | O_A [256,256+D) | O_B [256+D, 256+2D).
// P_X is written back as bf16 pairs over the first 64 columns of S_X and consumed from TMEM by
// the P.V MMA (A operand in TMEM), so P never touches shared memory. MMA order per key tile j:
//   PV_A(j), S_A(j+1), PV_B(j), S_B(j+1)  — the tensor core works on one tile while the other
// tile's softmax runs. O is rescaled lazily in TMEM (row max grew by > 2^8).
// attn_block_forward + finalize_piece (attention.cpp:61-115, :151-165); merge mode folds
// merge_piece (:117-149) into the epilogue.
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>

#include "tc.cuh"

namespace spattn {
namespace {

template <int D>
struct PPLayout {
  static constexpr int QB = D / 64;
  static constexpr int TILE = 128 * D * 2;
  static constexpr int QA_OFF = 0;
  static constexpr int QB_OFF = TILE;
  static constexpr int K_OFF = 2 * TILE;  // 2 stages
  static constexpr int V_OFF = 4 * TILE;  // 2 stages
  static constexpr int BAR_OFF = 6 * TILE;
  static constexpr int SMEM = BAR_OFF + 256;
};

enum PPBar {
  F_Q = 0,
  F_KF = 1,    // [2] K stage full
  F_VF = 3,    // [2] V stage full
  F_KVE = 5,   // [2] K/V stage empty
  F_SF = 7,    // [2] S_X ready (X = A, B)
  F_PF = 9,    // [2] P_X in TMEM (128 arrivals)
  F_PV = 11,   // [2] PV_X done
  F_N = 13
};

template <int D>
__global__ void __launch_bounds__(320, 1)
    attn_fwd_pp_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, FwdArgs a, ProblemSet ps) {
  using Lay = PPLayout<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  if (sbase & 1023) __trap();
  const uint32_t sQ = sbase + Lay::QA_OFF, sK = sbase + Lay::K_OFF, sV = sbase + Lay::V_OFF;
  const uint32_t bars = sbase + Lay::BAR_OFF;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Lay::BAR_OFF + F_N * 8);
  auto bar = [&](int i) { return bars + 8u * i; };
  const int warp = threadIdx.x / 32;

  // ---- tile decode: heavy causal tiles first, one head's tiles together (K/V reuse in L2)
  int pi = 0;
  while (pi + 1 < ps.n && ps.tile_prefix[pi + 1] <= (int)blockIdx.x) ++pi;
  const AttnProblem P = ps.p[pi];
  int mt = blockIdx.x - ps.tile_prefix[pi];
  if (P.causal) mt = (ps.tile_prefix[pi + 1] - ps.tile_prefix[pi]) - 1 - mt;
  const int m0 = mt * 256;
  const int h = blockIdx.y;
  const HeadMap hm = a.hm;
  const int kvh = (hm.q_head_base + h) / hm.rep - hm.kv_head_base;
  const int q_valid = min(256, P.nq - m0);
  int n_end = P.nk;
  if (P.causal) n_end = min(P.nk, m0 + q_valid - 1 + P.off + 1);
  n_end = max(n_end, 0);
  const int n_tiles = (n_end + 127) / 128;  // tile A may see fully-masked trailing tiles

  if (threadIdx.x == 0) {
    for (int i = 0; i < F_N; ++i) tc::mbar_init(bar(i), (i == F_PF || i == F_PF + 1) ? 128 : 1);
    tc::fence_barrier_init();
  }
  if (warp == 8) tc::tmem_alloc<512>(smem_u32(tmem_slot));
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ---------------------------------------------------------------------- TMA producer
    if (tc::elect_one()) {
      tc::mbar_expect_tx(bar(F_Q), 2 * Lay::TILE);
      for (int t = 0; t < 2; ++t)
        for (int b = 0; b < Lay::QB; ++b)
          tc::tma_load_2d(sQ + t * Lay::TILE + b * 16384, &tmQ, h * D + b * 64, P.q_row0 + m0 + 128 * t,
                          bar(F_Q));
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j & 1;
        if (j >= 2) tc::mbar_wait(bar(F_KVE + st), ((j - 2) >> 1) & 1);
        const int y = P.k_row0 + j * 128;
        tc::mbar_expect_tx(bar(F_KF + st), Lay::TILE);
        for (int b = 0; b < Lay::QB; ++b)
          tc::tma_load_2d(sK + st * Lay::TILE + b * 16384, &tmK, kvh * D + b * 64, y, bar(F_KF + st));
        tc::mbar_expect_tx(bar(F_VF + st), Lay::TILE);
        for (int b = 0; b < Lay::QB; ++b)
          tc::tma_load_2d(sV + st * Lay::TILE + b * 16384, &tmV, kvh * D + b * 64, y, bar(F_VF + st));
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------------------ MMA issuer
    if (tc::elect_one() && n_tiles > 0) {
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
        tc::fence_after();
        const uint32_t vb = sV + (j & 1) * Lay::TILE;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          tc::mma_ts(tmem + 256 + D * x, tmem + 128 * x + kk * 8, tc::sdesc(vb + kk * 2048, 16384, 1024), id_o,
                     (j > 0 || kk > 0) ? 1u : 0u);
        tc::commit(bar(F_PV + x));
      };
      tc::mbar_wait(bar(F_Q), 0);
      tc::mbar_wait(bar(F_KF), 0);
      tc::fence_after();
      issue_s(0, 0);
      issue_s(1, 0);
      for (int j = 0; j < n_tiles; ++j) {
        const bool more = j + 1 < n_tiles;
        if (j == 0 || true) {
          tc::mbar_wait(bar(F_VF + (j & 1)), (j >> 1) & 1);
          tc::fence_after();
        }
        issue_pv(0, j);
        if (more) {
          tc::mbar_wait(bar(F_KF + ((j + 1) & 1)), ((j + 1) >> 1) & 1);
          tc::fence_after();
          issue_s(0, j + 1);
        }
        issue_pv(1, j);
        tc::commit(bar(F_KVE + (j & 1)));  // K_j, V_j no longer read
        if (more) issue_s(1, j + 1);
      }
    }
  } else {
    // --------------------------------------------------- softmax warpgroups (A: 0-3, B: 4-7)
    const int x = warp >> 2;  // tile
    const int row = threadIdx.x & 127;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + 128 * x + lane_base, tO = tmem + 256 + D * x + lane_base;
    const float sl2 = a.scale * kLog2e;
    const int qa = m0 + 128 * x + row;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      tc::mbar_wait(bar(F_SF + x), j & 1);
      tc::fence_after();
      // two passes over the S_x columns in TMEM (register-light: 32 columns live at a time):
      // row max, then exp2 / row sum / bf16 P written over already-consumed S columns
      const int n0 = j * 128;
      const bool need_mask = (n0 + 128 > P.nk) || (P.causal && n0 + 127 > m0 + 128 * x + P.off);
      const int lim = !need_mask ? 127 : (P.causal ? min(P.nk - 1, qa + P.off) - n0 : P.nk - 1 - n0);
      float mt = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tc::tmem_ld32(tS + c * 32, r);
        tc::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) mt = fmaxf(mt, c * 32 + i <= lim ? __uint_as_float(r[i]) : -INFINITY);
      }
      mt *= sl2;
      if (j == 0) {
        m_run = mt;
      } else if (__any_sync(0xffffffffu, mt > m_run + 8.f)) {
        // lazy rescale of O and l; O must hold P_{j-1} V_{j-1}
        const float m_new = fmaxf(m_run, mt);
        const float alpha = (m_run == -INFINITY || m_new == -INFINITY) ? (m_run == m_new ? 1.f : 0.f)
                                                                        : fast_exp2(m_run - m_new);
        tc::mbar_wait(bar(F_PV + x), (j - 1) & 1);
        tc::fence_after();
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t r[32];
          tc::tmem_ld32(tO + c * 32, r);
          tc::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
          tc::tmem_st32(tO + c * 32, r);
        }
        tc::tmem_wait_st();
        l_run *= alpha;
        m_run = m_new;
      }
      const float muse = m_run == -INFINITY ? 0.f : m_run;
      float rs = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32], w[16];
        tc::tmem_ld32(tS + c * 32, r);
        tc::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int k0 = c * 32 + 2 * i;
          const float x0 = k0 <= lim ? __uint_as_float(r[2 * i]) : -INFINITY;
          const float x1 = k0 + 1 <= lim ? __uint_as_float(r[2 * i + 1]) : -INFINITY;
          const float p0 = fast_exp2(fmaf(x0, sl2, -muse));
          const float p1 = fast_exp2(fmaf(x1, sl2, -muse));
          rs += p0 + p1;
          w[i] = pack_bf16(p0, p1);
        }
        tc::tmem_st16(tS + c * 16, w);
      }
      l_run += rs;
      tc::tmem_wait_st();
      tc::fence_before();
      tc::mbar_arrive(bar(F_PF + x));
    }
    // ---- epilogue
    const bool empty = !(l_run > 0.f);
    const float inv = empty ? 0.f : 1.f / l_run;
    const float lse_row = empty ? -INFINITY : (m_run + __log2f(l_run)) * kLn2;
    if (n_tiles > 0) {
      tc::mbar_wait(bar(F_PV + x), (n_tiles - 1) & 1);
      tc::fence_after();
    }
    const bool valid = qa < P.nq;
    const int64_t grow = (int64_t)(P.q_row0 + qa);
    if (a.acc_o == nullptr) {
      __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(a.o) + grow * a.o_row_stride + h * D;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t r[32];
        if (n_tiles > 0) {
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
        if (n_tiles > 0) {
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
  if (warp == 8) tc::tmem_dealloc<512>(tmem);
}

int max_rows_pp(const ProblemSet& ps, bool q) {
  int m = 0;
  for (int i = 0; i < ps.n; ++i) m = max(m, q ? ps.p[i].q_row0 + ps.p[i].nq : ps.p[i].k_row0 + ps.p[i].nk);
  return m;
}

template <int D>
void launch_pp_d(const FwdArgs& a, const ProblemSet& in, cudaStream_t s) {
  ProblemSet ps = in;
  ps.tile_prefix[0] = 0;
  for (int i = 0; i < ps.n; ++i) ps.tile_prefix[i + 1] = ps.tile_prefix[i] + (ps.p[i].nq + 255) / 256;
  const int tiles = ps.tile_prefix[ps.n];
  if (tiles == 0 || a.hm.hq == 0) return;
  CUtensorMap tq, tk, tv;
  const uint64_t qw = (uint64_t)a.q_row_stride, kw = (uint64_t)a.kv_row_stride;
  if (!make_tma_2d(&tq, a.q, qw, max_rows_pp(ps, true), qw, 128) ||
      !make_tma_2d(&tk, a.k, kw, max(1, max_rows_pp(ps, false)), kw, 128) ||
      !make_tma_2d(&tv, a.v, kw, max(1, max_rows_pp(ps, false)), kw, 128)) {
    cudaGetLastError();
    return;
  }
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(attn_fwd_pp_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         PPLayout<D>::SMEM);
  });
  attn_fwd_pp_kernel<D><<<dim3(tiles, a.hm.hq), 320, PPLayout<D>::SMEM, s>>>(tq, tk, tv, a, ps);
  note_launch();
}

}  // namespace

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
