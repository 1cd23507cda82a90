// Flash-attention forward/backward over a list of rectangular causal problems, warp-level
// mma.sync (m16n8k16 bf16 -> fp32) with cp.async double buffering and swizzled shared tiles.
//
// This is the portable correctness anchor of the layer; the tcgen05/TMEM kernels in
// attn_tc.cu are checked against it and against the CPU oracle.
//
// Math restated from the reference block kernels (paths under /root/reference/proj):
//   forward  attn_block_forward + finalize_piece  src/attention.cpp:61-115, :151-165
//   merge    merge_piece                          src/attention.cpp:117-149 (LSE form)
//   backward attn_block_backward                  src/attention.cpp:167-216
// Masking is `kpos <= qpos` (attention.cpp:89) expressed per problem as c <= a + off.
#include <cfloat>

#include "common.cuh"

namespace spattn {
namespace {

constexpr int kBM = 64;   // query rows per CTA tile (4 warps x 16)
constexpr int kBN = 64;   // key rows per tile
constexpr int kThreads = 128;

template <int D>
__device__ __forceinline__ void load_tile(uint32_t sbase, const __nv_bfloat16* g, int64_t stride,
                                          int rows_valid, int tid) {
  constexpr int CH = D / 8;  // 16-byte chunks per row
#pragma unroll
  for (int i = tid; i < kBN * CH; i += kThreads) {
    const int r = i / CH, c = i % CH;
    const bool ok = r < rows_valid;
    const __nv_bfloat16* src = ok ? g + r * stride + c * 8 : g;
    cp_async16(swz<D>(sbase, r, c), src, ok ? 16 : 0);
  }
}

// ---------------------------------------------------------------------------------- forward
template <int D, class PS>
__global__ void __launch_bounds__(kThreads) attn_fwd_mma(FwdArgs a, PS ps) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int TILE = kBN * D * 2;
  const uint32_t sQ = smem_u32(smem);
  const uint32_t sK0 = sQ + TILE, sV0 = sQ + 3 * TILE;  // K[2], V[2]

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int g = lane / 4, t = lane % 4;
  const int tile = blockIdx.x;
  const int pi = find_problem(ps, tile);
  const AttnProblem P = ps.p[pi];
  int mt = tile - ps.tile_prefix[pi];
  if (P.causal) mt = (ps.tile_prefix[pi + 1] - ps.tile_prefix[pi]) - 1 - mt;  // heavy first
  const int m0 = mt * kBM;
  const int h = blockIdx.y;
  const HeadMap hm = a.hm;
  const int kvh = (hm.q_head_base + h) / hm.rep - hm.kv_head_base;

  const int q_valid = min(kBM, P.nq - m0);
  int n_end = P.nk;
  if (P.causal) n_end = min(P.nk, m0 + q_valid - 1 + P.off + 1);
  n_end = max(n_end, 0);
  const int n_tiles = (n_end + kBN - 1) / kBN;

  const __nv_bfloat16* qg =
      reinterpret_cast<const __nv_bfloat16*>(a.q) + (int64_t)(P.q_row0 + m0) * a.q_row_stride + h * D;
  const __nv_bfloat16* kg =
      reinterpret_cast<const __nv_bfloat16*>(a.k) + (int64_t)P.k_row0 * a.kv_row_stride + kvh * D;
  const __nv_bfloat16* vg =
      reinterpret_cast<const __nv_bfloat16*>(a.v) + (int64_t)P.k_row0 * a.kv_row_stride + kvh * D;

  load_tile<D>(sQ, qg, a.q_row_stride, q_valid, tid);
  if (n_tiles > 0) {
    load_tile<D>(sK0, kg, a.kv_row_stride, n_end, tid);
    load_tile<D>(sV0, vg, a.kv_row_stride, n_end, tid);
  }
  cp_async_commit();

  const float sl2 = a.scale * kLog2e;
  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
  uint32_t qa[D / 16][4];

  for (int j = 0; j < n_tiles; ++j) {
    const int buf = j & 1;
    if (j + 1 < n_tiles) {
      const int n1 = (j + 1) * kBN;
      load_tile<D>(sK0 + (buf ^ 1) * TILE, kg + (int64_t)n1 * a.kv_row_stride, a.kv_row_stride,
                   n_end - n1, tid);
      load_tile<D>(sV0 + (buf ^ 1) * TILE, vg + (int64_t)n1 * a.kv_row_stride, a.kv_row_stride,
                   n_end - n1, tid);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        const int r = warp * 16 + (lane % 8) + 8 * ((lane / 8) % 2);
        ldsm_x4(swz<D>(sQ, r, ks * 2 + lane / 16), qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
      }
    }
    const uint32_t sK = sK0 + buf * TILE, sV = sV0 + buf * TILE;
    float s[kBN / 8][4];
#pragma unroll
    for (int i = 0; i < kBN / 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks) {
#pragma unroll
      for (int np = 0; np < kBN / 16; ++np) {
        uint32_t b0, b1, b2, b3;
        const int r = np * 16 + (lane % 8) + 8 * (lane / 16);
        ldsm_x4(swz<D>(sK, r, ks * 2 + (lane / 8) % 2), b0, b1, b2, b3);
        mma_bf16(s[2 * np], qa[ks], b0, b1);
        mma_bf16(s[2 * np + 1], qa[ks], b2, b3);
      }
    }
    const int n0 = j * kBN;
    const bool need_mask = (n0 + kBN > P.nk) || (P.causal && n0 + kBN - 1 > m0 + P.off);
#pragma unroll
    for (int nt = 0; nt < kBN / 8; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float x = s[nt][i] * sl2;
        if (need_mask) {
          const int qa_ = m0 + warp * 16 + g + 8 * (i / 2);
          const int c = n0 + nt * 8 + 2 * t + (i % 2);
          if (c >= P.nk || (P.causal && c > qa_ + P.off)) x = -INFINITY;
        }
        s[nt][i] = x;
      }
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < kBN / 8; ++nt) {
      mx[0] = fmaxf(mx[0], fmaxf(s[nt][0], s[nt][1]));
      mx[1] = fmaxf(mx[1], fmaxf(s[nt][2], s[nt][3]));
    }
    float alpha[2], muse[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float mn = fmaxf(m_run[r], mx[r]);
      muse[r] = mn == -INFINITY ? 0.f : mn;
      alpha[r] = fast_exp2(m_run[r] - muse[r]);
      m_run[r] = mn;
    }
    float rs[2] = {0.f, 0.f};
#pragma unroll
    for (int nt = 0; nt < kBN / 8; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float p = fast_exp2(s[nt][i] - muse[i / 2]);
        s[nt][i] = p;
        rs[i / 2] += p;
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) l_run[r] = l_run[r] * alpha[r] + rs[r];
#pragma unroll
    for (int dt = 0; dt < D / 8; ++dt) {
      o[dt][0] *= alpha[0];
      o[dt][1] *= alpha[0];
      o[dt][2] *= alpha[1];
      o[dt][3] *= alpha[1];
    }
#pragma unroll
    for (int kk = 0; kk < kBN / 16; ++kk) {
      uint32_t pa[4];
      pa[0] = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
      pa[1] = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
      pa[2] = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      pa[3] = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        uint32_t b0, b1, b2, b3;
        const int r = kk * 16 + (lane % 8) + 8 * ((lane / 8) % 2);
        ldsm_x4_t(swz<D>(sV, r, dp * 2 + lane / 16), b0, b1, b2, b3);
        mma_bf16(o[2 * dp], pa, b0, b1);
        mma_bf16(o[2 * dp + 1], pa, b2, b3);
      }
    }
    __syncthreads();
  }
  if (n_tiles == 0) cp_async_wait<0>();

  // ---- epilogue: normalise, LSE (natural log), store or merge
  float inv[2], lse_row[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    float l = l_run[r];
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    const bool empty = !(l > 0.f);
    inv[r] = empty ? 0.f : 1.f / l;
    lse_row[r] = empty ? -INFINITY : (m_run[r] + __log2f(l)) * kLn2;
  }
  const int rowA = m0 + warp * 16 + g;  // rows rowA and rowA + 8 within the problem
  if (a.acc_o == nullptr) {
    // Stage bf16 output through the (now idle) Q tile, then coalesced 16-byte stores.
    __syncthreads();
#pragma unroll
    for (int dt = 0; dt < D / 8; ++dt)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int row = warp * 16 + g + 8 * r;
        const uint32_t v = pack_bf16(o[dt][2 * r] * inv[r], o[dt][2 * r + 1] * inv[r]);
        const uint32_t addr = swz<D>(sQ, row, dt) + t * 4;
        asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(addr), "r"(v));
      }
    __syncthreads();
    __nv_bfloat16* og =
        reinterpret_cast<__nv_bfloat16*>(a.o) + (int64_t)(P.q_row0 + m0) * a.o_row_stride + h * D;
    constexpr int CH = D / 8;
    for (int i = tid; i < kBM * CH; i += kThreads) {
      const int r = i / CH, c = i % CH;
      if (r < q_valid) {
        uint4 v;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "r"(swz<D>(sQ, r, c)));
        *reinterpret_cast<uint4*>(og + (int64_t)r * a.o_row_stride + c * 8) = v;
      }
    }
    if (t == 0) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int row = rowA + 8 * r;
        if (row < P.nq) a.lse[(int64_t)(P.q_row0 + row) * a.lse_row_stride + h] = lse_row[r];
      }
    }
  } else {
    // merge_piece in LSE form: acc <- acc*e^(lse_acc-lse') + o*e^(lse_o-lse'),
    // lse' = logaddexp(lse_acc, lse_o); -inf pieces are skipped/adopted (attention.cpp:130-139).
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int row = rowA + 8 * r;
      const bool valid = row < P.nq;
      float* lp = a.lse + (int64_t)(P.q_row0 + row) * a.lse_row_stride + h;
      const float la = valid ? *lp : -INFINITY;
      const float lb = lse_row[r];
      const float mx = fmaxf(la, lb);
      float wa, wb, ln;
      if (mx == -INFINITY) {
        wa = 1.f, wb = 0.f, ln = -INFINITY;
      } else {
        const float ea = __expf(la - mx), eb = __expf(lb - mx);
        ln = mx + __logf(ea + eb);
        wa = __expf(la - ln);
        wb = __expf(lb - ln) * inv[r];
      }
      __syncwarp();
      if (valid) {
        float* ap = a.acc_o + (int64_t)(P.q_row0 + row) * a.o_row_stride + h * D;
#pragma unroll
        for (int dt = 0; dt < D / 8; ++dt) {
          float2* p2 = reinterpret_cast<float2*>(ap + dt * 8 + 2 * t);
          float2 cur = *p2;
          cur.x = cur.x * wa + o[dt][2 * r] * wb;
          cur.y = cur.y * wa + o[dt][2 * r + 1] * wb;
          *p2 = cur;
        }
        if (t == 0) *lp = ln;
      }
    }
  }
}

// --------------------------------------------------------------------------------- backward
// delta[row, h] = sum_d dout * out (attention.cpp:190-191)
__global__ void attn_bwd_pre(BwdArgs a, int rows) {
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  const int hq = a.hm.hq;
  if (warp_global >= rows * hq) return;
  const int row = warp_global / hq, h = warp_global % hq;
  const __nv_bfloat162* o =
      reinterpret_cast<const __nv_bfloat162*>(reinterpret_cast<const __nv_bfloat16*>(a.o) +
                                              (int64_t)row * a.o_row_stride + h * a.d);
  const __nv_bfloat162* d =
      reinterpret_cast<const __nv_bfloat162*>(reinterpret_cast<const __nv_bfloat16*>(a.dout) +
                                              (int64_t)row * a.o_row_stride + h * a.d);
  float acc = 0.f;
  for (int i = lane; i < a.d / 2; i += 32) {
    const float2 x = __bfloat1622float2(o[i]), y = __bfloat1622float2(d[i]);
    acc += x.x * y.x + x.y * y.y;
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (lane == 0) a.delta[(int64_t)row * a.lse_row_stride + h] = acc;
}

template <int D, class PS>
__global__ void __launch_bounds__(kThreads) attn_bwd_mma(BwdArgs a, PS ps) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int TILE = kBN * D * 2;
  const uint32_t sK = smem_u32(smem), sV = sK + TILE, sQ = sK + 2 * TILE, sdO = sK + 3 * TILE;
  const uint32_t sdS = sK + 4 * TILE;  // [kv 64][q 64] bf16, 128-byte rows
  float* sL = reinterpret_cast<float*>(smem + 4 * TILE + kBN * kBM * 2);
  float* sD = sL + kBM;

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int g = lane / 4, t = lane % 4;
  const int pi = find_problem(ps, blockIdx.x);
  const AttnProblem P = ps.p[pi];
  const int n0 = (blockIdx.x - ps.tile_prefix[pi]) * kBN;
  const int kvh = blockIdx.y;
  const HeadMap hm = a.hm;
  const int k_valid = min(kBN, P.nk - n0);
  // queries that can see key n0: a >= n0 - off
  int m_begin = 0;
  if (P.causal) m_begin = max(0, (n0 - P.off) / kBM * kBM);
  if (P.causal && n0 - P.off > P.nq - 1) return;  // no query sees this key tile
  // dq/dk leave this kernel fully scaled: ds = p (dp - delta) * scale (attention.cpp:203)

  const __nv_bfloat16* kg = reinterpret_cast<const __nv_bfloat16*>(a.k) +
                            (int64_t)(P.k_row0 + n0) * a.kv_row_stride + kvh * D;
  const __nv_bfloat16* vg = reinterpret_cast<const __nv_bfloat16*>(a.v) +
                            (int64_t)(P.k_row0 + n0) * a.kv_row_stride + kvh * D;
  load_tile<D>(sK, kg, a.kv_row_stride, k_valid, tid);
  load_tile<D>(sV, vg, a.kv_row_stride, k_valid, tid);
  cp_async_commit();

  // q heads of this kv head's group that live on this rank
  const int g_lo = (kvh + hm.kv_head_base) * hm.rep;
  const int h_lo = max(0, g_lo - hm.q_head_base);
  const int h_hi = min(hm.hq, g_lo + hm.rep - hm.q_head_base);

  const float sl2 = a.scale * kLog2e;
  float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) dk[i][j] = dv[i][j] = 0.f;

  for (int h = h_lo; h < h_hi; ++h) {
    for (int m0 = m_begin; m0 < P.nq; m0 += kBM) {
      const int q_valid = min(kBM, P.nq - m0);
      const int64_t qrow = P.q_row0 + m0;
      load_tile<D>(sQ, reinterpret_cast<const __nv_bfloat16*>(a.q) + qrow * a.q_row_stride + h * D,
                   a.q_row_stride, q_valid, tid);
      load_tile<D>(sdO,
                   reinterpret_cast<const __nv_bfloat16*>(a.dout) + qrow * a.o_row_stride + h * D,
                   a.o_row_stride, q_valid, tid);
      cp_async_commit();
      if (tid < kBM) {
        float l = INFINITY, dl = 0.f;
        if (tid < q_valid) {
          const float x = a.lse[(qrow + tid) * a.lse_row_stride + h];
          l = x == -INFINITY ? INFINITY : x * kLog2e;
          dl = a.delta[(qrow + tid) * a.lse_row_stride + h];
        }
        sL[tid] = l;
        sD[tid] = dl;
      }
      cp_async_wait<0>();
      __syncthreads();

      // S^T (16 kv rows of this warp x 64 queries) and dP^T
      float st[kBM / 8][4], dpt[kBM / 8][4];
#pragma unroll
      for (int i = 0; i < kBM / 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) st[i][j] = dpt[i][j] = 0.f;
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        uint32_t ka[4], va[4];
        const int r = warp * 16 + (lane % 8) + 8 * ((lane / 8) % 2);
        ldsm_x4(swz<D>(sK, r, ks * 2 + lane / 16), ka[0], ka[1], ka[2], ka[3]);
        ldsm_x4(swz<D>(sV, r, ks * 2 + lane / 16), va[0], va[1], va[2], va[3]);
#pragma unroll
        for (int np = 0; np < kBM / 16; ++np) {
          uint32_t b0, b1, b2, b3;
          const int rq = np * 16 + (lane % 8) + 8 * (lane / 16);
          ldsm_x4(swz<D>(sQ, rq, ks * 2 + (lane / 8) % 2), b0, b1, b2, b3);
          mma_bf16(st[2 * np], ka, b0, b1);
          mma_bf16(st[2 * np + 1], ka, b2, b3);
          ldsm_x4(swz<D>(sdO, rq, ks * 2 + (lane / 8) % 2), b0, b1, b2, b3);
          mma_bf16(dpt[2 * np], va, b0, b1);
          mma_bf16(dpt[2 * np + 1], va, b2, b3);
        }
      }
      const bool need_mask = (n0 + kBN > P.nk) || (m0 + kBM > P.nq) ||
                             (P.causal && n0 + kBN - 1 > m0 + P.off);
#pragma unroll
      for (int nt = 0; nt < kBM / 8; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int ql = nt * 8 + 2 * t + (i % 2);
          float p = fast_exp2(st[nt][i] * sl2 - sL[ql]);
          if (need_mask) {
            const int c = n0 + warp * 16 + g + 8 * (i / 2);
            const int qa_ = m0 + ql;
            if (c >= P.nk || qa_ >= P.nq || (P.causal && c > qa_ + P.off)) p = 0.f;
          }
          st[nt][i] = p;
          dpt[nt][i] = p * (dpt[nt][i] - sD[ql]);
        }
      // dV += P^T dO ; dK += dS^T Q
#pragma unroll
      for (int kk = 0; kk < kBM / 16; ++kk) {
        uint32_t pa[4], da[4];
        pa[0] = pack_bf16(st[2 * kk][0], st[2 * kk][1]);
        pa[1] = pack_bf16(st[2 * kk][2], st[2 * kk][3]);
        pa[2] = pack_bf16(st[2 * kk + 1][0], st[2 * kk + 1][1]);
        pa[3] = pack_bf16(st[2 * kk + 1][2], st[2 * kk + 1][3]);
        da[0] = pack_bf16(dpt[2 * kk][0], dpt[2 * kk][1]);
        da[1] = pack_bf16(dpt[2 * kk][2], dpt[2 * kk][3]);
        da[2] = pack_bf16(dpt[2 * kk + 1][0], dpt[2 * kk + 1][1]);
        da[3] = pack_bf16(dpt[2 * kk + 1][2], dpt[2 * kk + 1][3]);
        // dS^T (bf16) to shared for the dQ product
        {
          const int rr = warp * 16 + g;
          asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(sdS + rr * 128 + (((2 * kk) ^ (rr & 7)) << 4) + t * 4),
                       "r"(da[0]));
          asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(sdS + (rr + 8) * 128 + (((2 * kk) ^ ((rr + 8) & 7)) << 4) + t * 4),
                       "r"(da[1]));
          asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(sdS + rr * 128 + (((2 * kk + 1) ^ (rr & 7)) << 4) + t * 4),
                       "r"(da[2]));
          asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(sdS + (rr + 8) * 128 + (((2 * kk + 1) ^ ((rr + 8) & 7)) << 4) + t * 4),
                       "r"(da[3]));
        }
#pragma unroll
        for (int dp = 0; dp < D / 16; ++dp) {
          uint32_t b0, b1, b2, b3;
          const int r = kk * 16 + (lane % 8) + 8 * ((lane / 8) % 2);
          ldsm_x4_t(swz<D>(sdO, r, dp * 2 + lane / 16), b0, b1, b2, b3);
          mma_bf16(dv[2 * dp], pa, b0, b1);
          mma_bf16(dv[2 * dp + 1], pa, b2, b3);
          ldsm_x4_t(swz<D>(sQ, r, dp * 2 + lane / 16), b0, b1, b2, b3);
          mma_bf16(dk[2 * dp], da, b0, b1);
          mma_bf16(dk[2 * dp + 1], da, b2, b3);
        }
      }
      __syncthreads();
      // dQ[q rows of this warp] += dS K, in 32-column slabs, atomically into fp32
      float* dqg = a.dq_acc + qrow * a.dq_row_stride + h * D;
#pragma unroll
      for (int dc = 0; dc < D / 32; ++dc) {
        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          uint32_t af[4];
          const int rk = kk * 16 + (lane % 8) + 8 * (lane / 16);
          const int ch = 2 * warp + (lane / 8) % 2;
          ldsm_x4_t(sdS + rk * 128 + ((ch ^ (rk & 7)) << 4), af[0], af[1], af[2], af[3]);
#pragma unroll
          for (int dp = 0; dp < 2; ++dp) {
            uint32_t b0, b1, b2, b3;
            const int r = kk * 16 + (lane % 8) + 8 * ((lane / 8) % 2);
            ldsm_x4_t(swz<D>(sK, r, dc * 4 + dp * 2 + lane / 16), b0, b1, b2, b3);
            mma_bf16(acc[2 * dp], af, b0, b1);
            mma_bf16(acc[2 * dp + 1], af, b2, b3);
          }
        }
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int ql = warp * 16 + g + 8 * r;
            if (ql < q_valid) {
              float* p = dqg + (int64_t)ql * a.dq_row_stride + dc * 32 + nt * 8 + 2 * t;
              atomicAdd(reinterpret_cast<float2*>(p), make_float2(acc[nt][2 * r] * a.scale, acc[nt][2 * r + 1] * a.scale));
            }
          }
      }
      __syncthreads();
    }
  }
  // dK, dV of this CTA's key rows (fp32 atomics: several problems may share key rows)
  float* dkg = a.dk_acc + (int64_t)(P.k_row0 + n0) * a.dkv_row_stride + kvh * D;
  float* dvg = a.dv_acc + (int64_t)(P.k_row0 + n0) * a.dkv_row_stride + kvh * D;
#pragma unroll
  for (int dt = 0; dt < D / 8; ++dt)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int kl = warp * 16 + g + 8 * r;
      if (kl < k_valid) {
        const int64_t off = (int64_t)kl * a.dkv_row_stride + dt * 8 + 2 * t;
        atomicAdd(reinterpret_cast<float2*>(dkg + off), make_float2(dk[dt][2 * r] * a.scale, dk[dt][2 * r + 1] * a.scale));
        atomicAdd(reinterpret_cast<float2*>(dvg + off), make_float2(dv[dt][2 * r], dv[dt][2 * r + 1]));
      }
    }
}

ProblemSet with_prefix(const ProblemSet& in, int block) {
  ProblemSet ps;
  copy_problems(ps, in);
  ps.tile_prefix[0] = 0;
  for (int i = 0; i < ps.n; ++i) {
    const int n = (i < ps.n) ? ps.p[i].nq : 0;
    ps.tile_prefix[i + 1] = ps.tile_prefix[i] + (n + block - 1) / block;
  }
  return ps;
}

}  // namespace

void launch_attn_fwd_mma(const FwdArgs& a, const ProblemSet& in, cudaStream_t s) {
  const ProblemSet ps = with_prefix(in, kBM);
  const int tiles = ps.tile_prefix[ps.n];
  if (tiles == 0 || a.hm.hq == 0) return;
  dim3 grid(tiles, a.hm.hq);
  with_problem_set(ps, [&](const auto& set) {
    using PS = std::decay_t<decltype(set)>;
    if (a.d == 64) {
      const int sm = 5 * kBN * 64 * 2;
      attn_fwd_mma<64, PS><<<grid, kThreads, sm, s>>>(a, set);
    } else {
      const int sm = 5 * kBN * 128 * 2;
      ensure_smem_for(attn_fwd_mma<128, PS>, sm);
      attn_fwd_mma<128, PS><<<grid, kThreads, sm, s>>>(a, set);
    }
    note_launch();
  });
}

// delta with 16-byte loads: TPH = d/8 lanes per (row, head), 32/TPH (row, head) pairs per warp
// (the one-warp-per-pair kernel above keeps 4-byte loads and reaches ~half the HBM rate)
template <int TPH>
__global__ void __launch_bounds__(256) attn_bwd_pre_v16(BwdArgs a, int rows) {
  const int64_t pair = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / TPH;
  const int sub = threadIdx.x % TPH;
  const int hq = a.hm.hq;
  const bool live = pair < (int64_t)rows * hq;
  float acc = 0.f;
  int64_t row = 0;
  int h = 0;
  if (live) {
    row = pair / hq, h = (int)(pair % hq);
    const int64_t off = row * a.o_row_stride + (int64_t)h * a.d + sub * 8;
    const uint4 x = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.o) + off);
    const uint4 y = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.dout) + off);
    const __nv_bfloat162* xp = reinterpret_cast<const __nv_bfloat162*>(&x);
    const __nv_bfloat162* yp = reinterpret_cast<const __nv_bfloat162*>(&y);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 u = __bfloat1622float2(xp[i]), w = __bfloat1622float2(yp[i]);
      acc += u.x * w.x + u.y * w.y;
    }
  }
#pragma unroll
  for (int sft = TPH / 2; sft > 0; sft >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, sft);
  if (live && sub == 0) a.delta[row * a.lse_row_stride + h] = acc;
}

void launch_attn_bwd_pre(const BwdArgs& a, int rows, cudaStream_t s) {
  const int64_t pairs = (int64_t)rows * a.hm.hq;
  if (pairs == 0) return;
  const bool v16 = (a.d == 64 || a.d == 128) && (a.o_row_stride % 8) == 0 &&
                   reinterpret_cast<uintptr_t>(a.o) % 16 == 0 && reinterpret_cast<uintptr_t>(a.dout) % 16 == 0;
  if (v16 && a.d == 128) {
    attn_bwd_pre_v16<16><<<(unsigned)((pairs * 16 + 255) / 256), 256, 0, s>>>(a, rows);
  } else if (v16) {
    attn_bwd_pre_v16<8><<<(unsigned)((pairs * 8 + 255) / 256), 256, 0, s>>>(a, rows);
  } else {
    attn_bwd_pre<<<(unsigned)((pairs + 7) / 8), 256, 0, s>>>(a, rows);
  }
  note_launch();
}

void launch_attn_bwd_mma(const BwdArgs& a, const ProblemSet& in, cudaStream_t s) {
  ProblemSet ps;
  copy_problems(ps, in);
  ps.tile_prefix[0] = 0;
  for (int i = 0; i < ps.n; ++i) ps.tile_prefix[i + 1] = ps.tile_prefix[i] + (ps.p[i].nk + kBN - 1) / kBN;
  const int tiles = ps.tile_prefix[ps.n];
  if (tiles == 0 || a.hm.hkv == 0 || a.hm.hq == 0) return;
  dim3 grid(tiles, a.hm.hkv);
  with_problem_set(ps, [&](const auto& set) {
    using PS = std::decay_t<decltype(set)>;
    if (a.d == 64) {
      const int sm = 4 * kBN * 64 * 2 + kBN * kBM * 2 + 2 * kBM * 4;
      attn_bwd_mma<64, PS><<<grid, kThreads, sm, s>>>(a, set);
    } else {
      const int sm = 4 * kBN * 128 * 2 + kBN * kBM * 2 + 2 * kBM * 4;
      ensure_smem_for(attn_bwd_mma<128, PS>, sm);
      attn_bwd_mma<128, PS><<<grid, kThreads, sm, s>>>(a, set);
    }
    note_launch();
  });
}

}  // namespace spattn
