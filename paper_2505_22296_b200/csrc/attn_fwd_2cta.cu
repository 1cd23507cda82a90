// tcgen05 attention forward for head_dim 128 on CTA PAIRS (cta_group::2, sm_100a).
//
// A cluster of two CTAs owns 256 query rows of one head (128 per CTA). Every MMA is a pair MMA
// (M = 256) issued by the leader: S = Q K^T takes each CTA's Q rows as A and splits the key
// tile's B operand between the CTAs (64 keys each); O += P V takes each CTA's P rows as A and
// splits V by head-dim columns (64 each). So each SM stages and reads only half of every K / V
// tile — the single-CTA kernel's SS MMAs read 128 B/clk of shared memory, exactly the port's
// rate, which this halves for the B operands. Softmax, lazy rescale, the two alternating
// online-softmax streams and the epilogue are per CTA, as in attn_fwd_tc_kernel (attn_tc.cu);
// attn_block_forward + finalize_piece (attention.cpp:61-115, :151-165).
//
// Pair synchronisation: K/V/Q loads of both CTAs complete on the leader's barriers
// (cp.async.bulk.tensor ... cta_group::2); MMA completions multicast to both CTAs
// (tcgen05.commit ... multicast::cluster); the softmax warps of both CTAs release S buffers and
// publish P to the leader with one cluster-scope arrive per warp.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include "tc.cuh"

namespace spattn {

bool make_tma_2d(CUtensorMap* m, const void* base, uint64_t width, uint64_t rows, uint64_t row_stride_elems,
                 uint32_t box_rows);

namespace {

constexpr int D = 128;
constexpr int Q_TILE = 128 * D * 2;   // 32 KB: this CTA's 128 query rows
constexpr int KH = 64 * D * 2;        // 16 KB: half a key tile (64 keys x 128 dims, 2 column blocks)
constexpr int VH = 128 * 64 * 2;      // 16 KB: half a value tile (128 keys x 64 dims)
constexpr int P_TILE = 128 * 128 * 2; // 32 KB
#ifndef FWD_PAIR_KST
#define FWD_PAIR_KST 3
#endif
constexpr int KST = FWD_PAIR_KST;          // K / V pipeline stages (the half tiles leave room for 3)
constexpr int Q_OFF = 0;
constexpr int K_OFF = Q_OFF + Q_TILE;
constexpr int V_OFF = K_OFF + KST * KH;
constexpr int P_OFF = V_OFF + KST * VH;    // 2 buffers
constexpr int BAR_OFF = P_OFF + 2 * P_TILE;
static_assert(BAR_OFF + 256 + 2 * 2 * 128 * 4 <= 227 * 1024, "shared memory");
constexpr int XCH_OFF = BAR_OFF + 256;
constexpr int SMEM = XCH_OFF + 2 * 2 * 128 * 4;

enum Bar { B_Q = 0, B_KF = 1, B_VF = B_KF + KST, B_SF = B_VF + KST, B_SFREE = B_SF + 2, B_PF = B_SFREE + 2,
           B_PV = B_PF + 2, B_N = B_PV + 2 };

template <class PS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(352, 1)
    attn_fwd_pair_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                         const __grid_constant__ CUtensorMap tmV, FwdArgs a, PS ps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  if (sbase & 1023) __trap();
  const uint32_t sQ = sbase + Q_OFF, sK = sbase + K_OFF, sV = sbase + V_OFF, sP = sbase + P_OFF;
  const uint32_t bars = sbase + BAR_OFF;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + BAR_OFF + B_N * 8);
  auto bar = [&](int i) { return bars + 8u * i; };
  const uint32_t rank = tc::cluster_ctarank();
  const bool leader = rank == 0;
  auto lbar = [&](int i) { return tc::mapa(bar(i), 0); };  // the leader's barrier i
#ifdef FWD_PAIR_RELEASE
  auto publish = [&](int i) { tc::mbar_arrive_cluster(lbar(i)); };
#else
  // local arrive on the leader, relaxed cluster-scope arrive from the peer (its data is ordered
  // by the tcgen05 / proxy fences before it)
  auto publish = [&](int i) {
    if (leader)
      tc::mbar_arrive(bar(i));
    else
      tc::mbar_arrive_cluster_relaxed(lbar(i));
  };
#endif

  const int warp = threadIdx.x / 32;
  // ---- pair decode (heavy causal pairs first; one head's pairs run together)
  const int pair = blockIdx.x >> 1;
  const int pi = find_problem(ps, pair);
  const AttnProblem P = ps.p[pi];
  int mt = pair - ps.tile_prefix[pi];
  if (P.causal) mt = (ps.tile_prefix[pi + 1] - ps.tile_prefix[pi]) - 1 - mt;
  const int pm0 = mt * 256;                 // the pair's first query row
  const int m0 = pm0 + 128 * (int)rank;     // this CTA's first query row
  const int h = blockIdx.y;
  const HeadMap hm = a.hm;
  const int kvh = (hm.q_head_base + h) / hm.rep - hm.kv_head_base;
  const int pair_rows = min(256, P.nq - pm0);
  int n_end = P.nk;  // keys the pair needs (the later CTA's causal extent)
  if (P.causal) n_end = min(P.nk, pm0 + pair_rows - 1 + P.off + 1);
  n_end = max(n_end, 0);
  const int n_tiles = (n_end + 127) / 128;

  if (threadIdx.x == 0) {
    for (int i = 0; i < B_N; ++i) {
      const bool pub = (i >= B_SFREE && i < B_SFREE + 2) || (i >= B_PF && i < B_PF + 2);
      tc::mbar_init(bar(i), pub ? 8 : 1);  // 4 softmax warps x 2 CTAs publish to the leader
    }
    tc::fence_barrier_init();
  }
  if (warp == 9) tc::tmem_alloc_pair<512>(smem_u32(tmem_slot));
  tc::fence_before();
  tc::cluster_sync();  // barriers initialised and TMEM allocated in both CTAs
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tO = tmem + 256;

  if (warp == 8) {
    // Q (both CTAs' rows land on the leader's barrier) and this CTA's half of every key tile
    if (tc::elect_one() && n_tiles > 0) {
      tc::tma_prefetch(&tmQ);
      tc::tma_prefetch(&tmK);
      if (leader) tc::mbar_expect_tx(bar(B_Q), 2 * Q_TILE);
      for (int b = 0; b < 2; ++b)
        tc::tma_load_2d_pair(sQ + b * 16384, &tmQ, h * D + b * 64, P.q_row0 + m0, lbar(B_Q));
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % KST;
        if (j >= KST) tc::mbar_wait(bar(B_SF + ((j - KST) & 1)), ((j - KST) >> 1) & 1);  // S(j-KST) read it
        if (leader) tc::mbar_expect_tx(bar(B_KF + st), 2 * KH);
        for (int b = 0; b < 2; ++b)
          tc::tma_load_2d_pair(sK + st * KH + b * 8192, &tmK, kvh * D + b * 64, P.k_row0 + j * 128 + 64 * rank,
                               lbar(B_KF + st));
      }
    }
  } else if (warp == 9) {
    // this CTA's head-dim half of every value tile
    if (tc::elect_one() && n_tiles > 0) {
      tc::tma_prefetch(&tmV);
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % KST;
        if (j >= KST) tc::mbar_wait(bar(B_PV + ((j - KST) & 1)), ((j - KST) >> 1) & 1);  // PV(j-KST) read it
        if (leader) tc::mbar_expect_tx(bar(B_VF + st), 2 * VH);
        tc::tma_load_2d_pair(sV + st * VH, &tmV, kvh * D + 64 * rank, P.k_row0 + j * 128, lbar(B_VF + st));
      }
    }
  } else if (warp == 10) {
    if (leader && tc::elect_one() && n_tiles > 0) {
      constexpr uint32_t id_s = tc::idesc_bf16(256, 128, false, false);
      constexpr uint32_t id_o = tc::idesc_bf16(256, D, false, true);
      auto issue_s = [&](int j) {
        const int st = j & 1, ks_ = j % KST;
        tc::mbar_wait(bar(B_KF + ks_), (j / KST) & 1);
        if (j >= 2) tc::mbar_wait(bar(B_SFREE + st), ((j - 2) >> 1) & 1);
        tc::fence_after();
        const uint32_t kbase = sK + ks_ * KH;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t qo = (ks >> 2) * 16384 + (ks & 3) * 32, ko = (ks >> 2) * 8192 + (ks & 3) * 32;
          tc::mma_ss_pair(tmem + st * 128, tc::sdesc(sQ + qo, 16, 1024), tc::sdesc(kbase + ko, 16, 1024), id_s,
                          ks > 0 ? 1u : 0u);
        }
        tc::commit_pair(bar(B_SF + st), 0x3);
      };
      auto issue_pv = [&](int i) {
        const int st = i & 1, vs = i % KST;
        tc::mbar_wait(bar(B_PF + st), (i >> 1) & 1);
        tc::mbar_wait(bar(B_VF + vs), (i / KST) & 1);
        tc::fence_after();
        const uint32_t pbase = sP + st * P_TILE, vbase = sV + vs * VH;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t aoff = (kk >> 2) * 16384 + (kk & 3) * 32;
          tc::mma_ss_pair(tO + st * D, tc::sdesc(pbase + aoff, 16, 1024), tc::sdesc(vbase + kk * 2048, 16384, 1024),
                          id_o, (i > 1 || kk > 0) ? 1u : 0u);
        }
        tc::commit_pair(bar(B_PV + st), 0x3);
      };
      tc::mbar_wait(bar(B_Q), 0);
      issue_s(0);
      if (n_tiles > 1) issue_s(1);
      for (int j = 0; j < n_tiles; ++j) {
        if (j + 2 < n_tiles) issue_s(j + 2);
        issue_pv(j);
      }
    }
  } else if (warp < 8) {
    // two online-softmax streams over alternating key tiles (attn_fwd_tc_kernel), on this CTA's
    // 128 rows of the pair's S and O
    const int g = warp >> 2;
    const int lane = threadIdx.x & 31;
    const int row = threadIdx.x & 127;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + g * 128 + lane_base, tOg = tO + g * D + lane_base;
    const float sl2 = a.scale * kLog2e;
    const int qa = m0 + row;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = g; j < n_tiles; j += 2) {
      const int it = j >> 1;
      tc::mbar_wait(bar(B_SF + g), it & 1);
      tc::fence_after();
      float x[128];
      {
        uint32_t r[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tc::tmem_ld32(tS + c * 32, r[c]);
        tc::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 128; ++i) x[i] = __uint_as_float(r[i >> 5][i & 31]);
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) publish(B_SFREE + g);
      const int n0 = j * 128;
      const bool need_mask = (n0 + 128 > P.nk) || (P.causal && n0 + 127 > m0 + P.off);
      if (need_mask) {
        const int lim = P.causal ? min(P.nk - 1, qa + P.off) - n0 : P.nk - 1 - n0;
#pragma unroll
        for (int i = 0; i < 128; ++i) x[i] = i <= lim ? x[i] : -INFINITY;
      }
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int i = 0; i < 128; i += 8) {
        mx[0] = fmaxf(mx[0], fmaxf(x[i], x[i + 1]));
        mx[1] = fmaxf(mx[1], fmaxf(x[i + 2], x[i + 3]));
        mx[2] = fmaxf(mx[2], fmaxf(x[i + 4], x[i + 5]));
        mx[3] = fmaxf(mx[3], fmaxf(x[i + 6], x[i + 7]));
      }
      const float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * sl2;
      if (it == 0) {
        m_run = mt;
      } else if (__any_sync(0xffffffffu, mt > m_run + 8.f)) {
        const float m_new = fmaxf(m_run, mt);
        const float alpha = (m_run == -INFINITY || m_new == -INFINITY) ? (m_run == m_new ? 1.f : 0.f)
                                                                        : fast_exp2(m_run - m_new);
        tc::mbar_wait(bar(B_PV + g), (it - 1) & 1);
        tc::fence_after();
#pragma unroll 1
        for (int c = 0; c < D / 8; ++c) {
          uint32_t r[8];
          tc::tmem_ld8(tOg + c * 8, r);
          tc::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 8; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
          tc::tmem_st8(tOg + c * 8, r);
        }
        tc::tmem_wait_st();
        l_run *= alpha;
        m_run = m_new;
      }
      const float muse = m_run == -INFINITY ? 0.f : m_run;
      const uint64_t sc2 = f2_pack(sl2, sl2), nm2 = f2_pack(-muse, -muse);
      uint64_t rs2[2] = {0ull, 0ull};
      uint32_t pw[64];
#pragma unroll
      for (int e = 0; e < 64; ++e) {
        const float2 av = f2_unpack(f2_fma(f2_pack(x[2 * e], x[2 * e + 1]), sc2, nm2));
        float2 pv;
        if ((e & 3) == 3) {
          pv = poly_exp2x2(av.x, av.y);
        } else {
          pv.x = fast_exp2(av.x);
          pv.y = fast_exp2(av.y);
        }
        rs2[e & 1] = f2_add(rs2[e & 1], f2_pack(pv.x, pv.y));
        pw[e] = pack_bf16(pv.x, pv.y);
      }
      if (it > 0) tc::mbar_wait(bar(B_PV + g), (it - 1) & 1);  // PV(j-2) read P buffer g
      const uint32_t pbase = sP + g * P_TILE;
#pragma unroll
      for (int ch = 0; ch < 16; ++ch) {
        const uint32_t addr = tc::sw128(pbase + (ch >> 3) * 16384, row, ch & 7);
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};\n" ::"r"(addr), "r"(pw[4 * ch]), "r"(pw[4 * ch + 1]),
                     "r"(pw[4 * ch + 2]), "r"(pw[4 * ch + 3]));
      }
      {
        const float2 r = f2_unpack(f2_add(rs2[0], rs2[1]));
        l_run += r.x + r.y;
      }
      tc::fence_before();
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) publish(B_PF + g);
    }
    // ---- epilogue: merge the two streams; group g writes output columns [g*D/2, (g+1)*D/2)
    const bool valid = qa < P.nq;
    const int64_t grow = (int64_t)(P.q_row0 + qa);
    float* lp = a.lse + grow * a.lse_row_stride + h;
    const float la = (a.acc_o != nullptr && valid) ? *lp : -INFINITY;
    float* xch = reinterpret_cast<float*>(smem + XCH_OFF);
    xch[g * 128 + row] = m_run;
    xch[256 + g * 128 + row] = l_run;
    asm volatile("bar.sync 1, 256;\n" ::: "memory");
    const float m_o = xch[(g ^ 1) * 128 + row], l_o = xch[256 + (g ^ 1) * 128 + row];
    const float m = fmaxf(m_run, m_o);
    const float w_own = m_run == -INFINITY ? 0.f : fast_exp2(m_run - m);
    const float w_oth = m_o == -INFINITY ? 0.f : fast_exp2(m_o - m);
    const float l = l_run * w_own + l_o * w_oth;
    const bool empty = m == -INFINITY || !(l > 0.f);
    const float inv = empty ? 0.f : 1.f / l;
    const float lse_row = empty ? -INFINITY : (m + __log2f(l)) * kLn2;
    const bool have_own = n_tiles > g, have_oth = n_tiles > (g ^ 1);
    if (n_tiles > 0) {
      tc::mbar_wait(bar(B_PV + ((n_tiles - 1) & 1)), ((n_tiles - 1) >> 1) & 1);  // all MMAs done
      tc::fence_after();
    }
    const uint32_t tOo = tO + (g ^ 1) * D + lane_base;
    constexpr int DH = D / 2;
    auto o_chunk = [&](int c, float* o) {
      uint32_t r[32], q[32];
      if (have_own) tc::tmem_ld32(tOg + g * DH + c * 32, r);
      if (have_oth) tc::tmem_ld32(tOo + g * DH + c * 32, q);
      tc::tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i)
        o[i] = ((have_own ? __uint_as_float(r[i]) * w_own : 0.f) + (have_oth ? __uint_as_float(q[i]) * w_oth : 0.f)) *
               inv;
    };
    if (a.acc_o == nullptr) {
      __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(a.o) + grow * a.o_row_stride + h * D + g * DH;
#pragma unroll
      for (int c = 0; c < DH / 32; ++c) {
        float o[32];
        o_chunk(c, o);
        uint32_t w[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) w[i] = pack_bf16(o[2 * i], o[2 * i + 1]);
        if (valid) {
          uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
        }
      }
      if (valid && g == 0) *lp = lse_row;
    } else {
      const float lb = lse_row;
      const float mx2 = fmaxf(la, lb);
      float wa = 1.f, wb = 0.f, ln = la;
      if (mx2 != -INFINITY) {
        ln = mx2 + __logf(__expf(la - mx2) + __expf(lb - mx2));
        wa = __expf(la - ln);
        wb = __expf(lb - ln);
      }
      float* arow = a.acc_o + grow * a.o_row_stride + h * D + g * DH;
#pragma unroll
      for (int c = 0; c < DH / 32; ++c) {
        float o[32];
        o_chunk(c, o);
        if (valid) {
          float4* ap = reinterpret_cast<float4*>(arow + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float4 cur = ap[i];
            cur.x = cur.x * wa + o[4 * i] * wb;
            cur.y = cur.y * wa + o[4 * i + 1] * wb;
            cur.z = cur.z * wa + o[4 * i + 2] * wb;
            cur.w = cur.w * wa + o[4 * i + 3] * wb;
            ap[i] = cur;
          }
        }
      }
      if (valid && g == 0) *lp = ln;
    }
  }
  tc::fence_before();
  tc::cluster_sync();  // no CTA leaves while its pair may still touch its smem / TMEM
  tc::fence_after();
  if (warp == 9) tc::tmem_dealloc_pair<512>(tmem);
}

int max_rows2(const ProblemSet& ps, bool q) {
  int m = 0;
  for (int i = 0; i < ps.n; ++i) m = max(m, q ? ps.p[i].q_row0 + ps.p[i].nq : ps.p[i].k_row0 + ps.p[i].nk);
  return m;
}

}  // namespace

bool tc_fwd_pair_supported(const FwdArgs& a) {
  auto al = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; };
  return a.d == D && al(a.q) && al(a.k) && al(a.v) && (a.q_row_stride * 2) % 16 == 0 &&
         (a.kv_row_stride * 2) % 16 == 0;
}

void launch_attn_fwd_pair(const FwdArgs& a, const ProblemSet& in, cudaStream_t s) {
  ProblemSet ps;
  copy_problems(ps, in);
  ps.tile_prefix[0] = 0;
  for (int i = 0; i < ps.n; ++i) ps.tile_prefix[i + 1] = ps.tile_prefix[i] + (ps.p[i].nq + 255) / 256;
  const int pairs = ps.tile_prefix[ps.n];
  if (pairs == 0 || a.hm.hq == 0) return;
  CUtensorMap tq, tk, tv;
  const uint64_t qw = (uint64_t)a.q_row_stride, kw = (uint64_t)a.kv_row_stride;
  const uint64_t krows = max(1, max_rows2(ps, false));
  if (!make_tma_2d(&tq, a.q, qw, max_rows2(ps, true), qw, 128) || !make_tma_2d(&tk, a.k, kw, krows, kw, 64) ||
      !make_tma_2d(&tv, a.v, kw, krows, kw, 128))
    launch_error("attn_fwd_pair", "TMA descriptor encode failed");
  with_problem_set(ps, [&](const auto& set) {
    using PS = std::decay_t<decltype(set)>;
    ensure_smem_for(attn_fwd_pair_kernel<PS>, SMEM);
    attn_fwd_pair_kernel<PS><<<dim3(2 * pairs, a.hm.hq), 352, SMEM, s>>>(tq, tk, tv, a, set);
  });
  note_launch();
}

}  // namespace spattn
