// tcgen05 / TMEM / TMA attention kernels for sm_100a.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include <set>
#include <stdexcept>
#include <string>
#include "tc.cuh"

namespace spattn {

// ------------------------------------------------------------------------ host: TMA maps
namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeFn>(nullptr);
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}
}  // namespace

void launch_error(const char* kernel, const char* what) {
  cudaGetLastError();
  throw std::runtime_error(std::string(kernel) + ": " + what);
}

void ensure_smem(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) launch_error("ensure_smem", "cudaGetDevice failed");
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({kernel, dev})) return;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    launch_error("ensure_smem", "cudaFuncSetAttribute(MaxDynamicSharedMemorySize) failed");
  done.insert({kernel, dev});
}

bool make_tma_2d(CUtensorMap* m, const void* base, uint64_t width, uint64_t rows,
                 uint64_t row_stride_elems, uint32_t box_rows) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {width, rows};
  cuuint64_t strides[1] = {row_stride_elems * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_tma_rows_u64(CUtensorMap* m, const void* base, uint64_t width_u64, uint64_t rows,
                       uint64_t row_stride_bytes, uint32_t box_w_u64, uint32_t box_rows) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {width_u64, rows};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_w_u64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_tma_2d_f32(CUtensorMap* m, const void* base, uint64_t width, uint64_t rows,
                     uint64_t row_stride_elems, uint32_t box_rows) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {width, rows};
  cuuint64_t strides[1] = {row_stride_elems * 4};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ------------------------------------------------------------- descriptor self-test GEMMs
// D1 = A . B^T (B K-major, like S = Q K^T) and D2 = A . Bmn (B MN-major, like O = P V) for
// 128x128x128 bf16 tiles, through TMA + tcgen05.mma + TMEM. Validates the descriptor
// encodings the attention kernels use.
namespace {
__global__ void __launch_bounds__(128, 1)
    umma_selftest_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                         const __grid_constant__ CUtensorMap tBmn, float* D1, float* D2, float* D3) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sA = smem_u32(smem), sB = sA + 32768, sC = sA + 65536;
  __shared__ uint64_t bars[2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t bar_load = smem_u32(&bars[0]), bar_mma = smem_u32(&bars[1]);
  if (threadIdx.x == 0) {
    tc::mbar_init(bar_load, 1);
    tc::mbar_init(bar_mma, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(smem_u32(&tmem_base));
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  if (warp == 0 && lane == 0) {
    tc::mbar_expect_tx(bar_load, 3 * 32768);
    for (int b = 0; b < 2; ++b) {
      tc::tma_load_2d(sA + b * 16384, &tA, b * 64, 0, bar_load);
      tc::tma_load_2d(sB + b * 16384, &tB, b * 64, 0, bar_load);
      tc::tma_load_2d(sC + b * 16384, &tBmn, b * 64, 0, bar_load);
    }
    tc::mbar_wait(bar_load, 0);
    tc::fence_after();
    constexpr uint32_t id_k = tc::idesc_bf16(128, 128, false, false);
    constexpr uint32_t id_mn = tc::idesc_bf16(128, 128, false, true);
    for (int ks = 0; ks < 8; ++ks) {
      const uint32_t off = (ks / 4) * 16384 + (ks % 4) * 32;
      tc::mma_ss(tmem, tc::sdesc(sA + off, 16, 1024), tc::sdesc(sB + off, 16, 1024), id_k, ks > 0);
    }
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
      tc::mma_ss(tmem + 128, tc::sdesc(sA + off, 16, 1024), tc::sdesc(sC + kk * 2048, 16384, 1024),
                 id_mn, kk > 0);
    }
    tc::commit(bar_mma);
  }
  __syncwarp();
  tc::mbar_wait(bar_mma, 0);
  tc::fence_after();
  const int row = warp * 32 + lane;
  const uint32_t lanes = (uint32_t)(warp * 32) << 16;
  for (int half = 0; half < 2; ++half)
    for (int c = 0; c < 128; c += 32) {
      uint32_t r[32];
      tc::tmem_ld32(tmem + lanes + half * 128 + c, r);
      tc::tmem_wait_ld();
      float* dst = (half ? D2 : D1) + row * 128 + c;
      for (int i = 0; i < 32; ++i) dst[i] = __uint_as_float(r[i]);
    }
  // D3 = A . Bmn with A taken from TMEM (A row -> lane, two bf16 per column), the form the
  // backward uses for dV += P^T dO. A is staged from the shared tile by each row's thread.
  if (D3) {
    for (int c = 0; c < 2; ++c) {
      uint32_t r[32];
      for (int i = 0; i < 32; ++i) {
        const int k = c * 64 + 2 * i;  // elements k, k+1 of row `row`
        uint32_t w;
        asm volatile("ld.shared.b32 %0, [%1];\n"
                     : "=r"(w)
                     : "r"(tc::sw128(sA + (k >> 6) * 16384, row, (k & 63) >> 3) + (k & 7) * 2));
        r[i] = w;
      }
      tc::tmem_st32(tmem + lanes + 384 + c * 32, r);
    }
    tc::tmem_wait_st();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (warp == 0 && lane == 0) {
      constexpr uint32_t id_mn = tc::idesc_bf16(128, 128, false, true);
      for (int kk = 0; kk < 8; ++kk)
        tc::mma_ts(tmem + 256, tmem + 384 + kk * 8, tc::sdesc(sC + kk * 2048, 16384, 1024), id_mn, kk > 0);
      tc::commit(bar_mma);
    }
    __syncwarp();
    tc::mbar_wait(bar_mma, 1);
    tc::fence_after();
    for (int c = 0; c < 128; c += 32) {
      uint32_t r[32];
      tc::tmem_ld32(tmem + lanes + 256 + c, r);
      tc::tmem_wait_ld();
      for (int i = 0; i < 32; ++i) D3[row * 128 + c + i] = __uint_as_float(r[i]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
}
}  // namespace

int umma_selftest(cudaStream_t s, const void* A, const void* B, const void* Bmn, float* D1, float* D2, float* D3) {
  CUtensorMap tA, tB, tC;
  if (!make_tma_2d(&tA, A, 128, 128, 128, 128) || !make_tma_2d(&tB, B, 128, 128, 128, 128) ||
      !make_tma_2d(&tC, Bmn, 128, 128, 128, 128))
    return -1;
  const int smem = 3 * 32768 + 1024;
  cudaFuncSetAttribute(umma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  umma_selftest_kernel<<<1, 128, smem, s>>>(tA, tB, tC, D1, D2, D3);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

__device__ long long* g_fwd_trace = nullptr;  // profiling: per-tile clock64 events of CTA (0,0)
void set_fwd_trace(void* p) { cudaMemcpyToSymbol(g_fwd_trace, &p, sizeof(p)); }
// profiling: per-CTA globaltimer records [entry, first S in TMEM, loop end, exit, n_tiles, smid]
__device__ long long* g_fwd_cta = nullptr;
void set_fwd_cta_trace(void* p) { cudaMemcpyToSymbol(g_fwd_cta, &p, sizeof(p)); }
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// =================================================================================
// Forward: one CTA = 128 query rows x one head of one problem. Warp roles:
//   warp 0      TMA producer (Q once; K_j, V_j into a 2-stage ring)
//   warp 1      MMA issuer (one elected thread): S_j = Q K_j^T into TMEM S[j%2], then
//               O += P_{j-1} V_{j-1} into TMEM O — S_{j+1} overlaps the softmax of tile j
//   warp 2      TMEM allocator (512 columns: S0 | S1 | O)
//   warps 4..7  softmax + epilogue: thread t owns query row t = TMEM lane t; P_j goes to a
//               double-buffered 128B-swizzled smem tile (the A operand of the PV MMA)
// O is rescaled in TMEM only when a row max grows by more than 2^8 (exponents stay <= 256),
// and lse/out are finalised from TMEM. attn_block_forward + finalize_piece
// (attention.cpp:61-115, :151-165); merge mode folds merge_piece (:117-149) into the epilogue.
namespace {

#ifndef SPATTN_FWD_POLY_PAIRS
#define SPATTN_FWD_POLY_PAIRS 0x8
#endif
#ifndef SPATTN_FWD_POLY_PAIRS_D64
#define SPATTN_FWD_POLY_PAIRS_D64 0x0
#endif
// bit e set: the e-th exponential pair of every 8 columns uses poly_exp2x2 instead of the MUFU.
// head_dim 128: one pair in four (the measured optimum); head_dim 64: none — its half-size MMAs
// leave the MUFU less loaded relative to the chain, and any share on the FMA pipe measured
// slower (L=32K, 8 heads: 1.51-1.52 ms with none, 1.60-1.64 with 1/4, 1.73 with 1/2).
template <int D>
constexpr int fwd_poly_pairs() {
  return D == 64 ? SPATTN_FWD_POLY_PAIRS_D64 : SPATTN_FWD_POLY_PAIRS;
}

template <int D>
struct FwdLayout {
  static constexpr int QB = D / 64;
  static constexpr int TILE = 128 * D * 2;  // Q, K or V tile (128 rows)
  static constexpr int P_TILE = 128 * 128 * 2;
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = Q_OFF + TILE;
  static constexpr int V_OFF = K_OFF + 2 * TILE;
  static constexpr int P_OFF = V_OFF + 2 * TILE;
  static constexpr int BAR_OFF = P_OFF + 2 * P_TILE;
  static constexpr int XCH_OFF = BAR_OFF + 256;  // epilogue exchange of the two streams' (max, sum)
  static constexpr int SMEM = XCH_OFF + 2 * 2 * 128 * 4;  // base is 1024-aligned (checked)
};

// K stage s is released by the S(j) completion barrier (B_SF), V stage s by the PV(j) one (B_PV),
// so the next K load overlaps the current softmax instead of waiting for PV.
// B_PH: the first half (keys 0-63) of P buffer st has been read by PV — the softmax of the
// stream's next tile may overwrite it while PV still reads the second half.
enum FwdBar { B_Q = 0, B_KF = 1, B_VF = 3, B_SF = 5, B_SFREE = 7, B_PF = 9, B_PV = 11, B_PH = 13, B_N = 15 };
#ifndef SPATTN_FWD_PHALF
#define SPATTN_FWD_PHALF 0
#endif

#ifndef SPATTN_FWD_P_TMEM
#define SPATTN_FWD_P_TMEM 0
#endif
// SPATTN_FWD_P_TMEM=1: P is written back over its own S columns in TMEM (bf16 pairs) and
// O += P V is a TS MMA — no P tile in shared memory (the SS kernel moves 224 KB of smem per
// tile: 128 KB operand reads, 64 KB K/V TMA writes, 32 KB P stores). PV(j) must then precede
// S(j+2) (which overwrites those columns), so the issue order is PV-first.
#ifndef SPATTN_FWD_DUAL_ISSUE
#define SPATTN_FWD_DUAL_ISSUE 0
#endif
// SPATTN_FWD_DUAL_ISSUE=1: two MMA issuers (warps 10 and 11), one per softmax stream (the
// streams touch disjoint S / O accumulators, P buffers and K / V stages). It cuts a stream's
// wait for its next S from 765 to 111 cycles, but the two softmax warps of an SMSP then overlap
// their exp phases on the shared MUFU (16/clk/SM) and the tile period stays at ~1590 cycles
// (1564 with one issuer), so the single issuer is the default.
constexpr int kFwdThreads = SPATTN_FWD_DUAL_ISSUE ? 384 : 352;

template <int D, class PS>
__global__ void __launch_bounds__(kFwdThreads, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, FwdArgs a, PS ps) {
  using Lay = FwdLayout<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  if (sbase & 1023) __trap();  // the swizzled operand tiles need 1024-byte alignment
  const uint32_t sQ = sbase + Lay::Q_OFF, sK = sbase + Lay::K_OFF, sV = sbase + Lay::V_OFF,
                 sP = sbase + Lay::P_OFF;
  const uint32_t bars = sbase + Lay::BAR_OFF;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Lay::BAR_OFF + B_N * 8);
  auto bar = [&](int i) { return bars + 8u * i; };

  const int warp = threadIdx.x / 32;
  // ---- tile decode (heavy causal tiles first; one head's tiles run together, sharing K/V in L2)
  const int pi = find_problem(ps, (int)blockIdx.x);
  const AttnProblem P = ps.p[pi];
  int mt = blockIdx.x - ps.tile_prefix[pi];
  if (P.causal) mt = (ps.tile_prefix[pi + 1] - ps.tile_prefix[pi]) - 1 - mt;
  const int m0 = mt * 128;
  const int h = blockIdx.y;
  const HeadMap hm = a.hm;
  const int kvh = (hm.q_head_base + h) / hm.rep - hm.kv_head_base;
  const int q_valid = min(128, P.nq - m0);
  int n_end = P.nk;
  if (P.causal) n_end = min(P.nk, m0 + q_valid - 1 + P.off + 1);
  n_end = max(n_end, 0);
  const int n_tiles = (n_end + 127) / 128;
  long long* trace = (g_fwd_trace && blockIdx.x == 0 && blockIdx.y == 0) ? g_fwd_trace : nullptr;
  long long* ctr = g_fwd_cta ? g_fwd_cta + 8 * ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) : nullptr;
  if (ctr && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    ctr[0] = gtimer();
    ctr[4] = n_tiles;
    ctr[5] = smid;
  }
#define FTR(slot, j) \
  if (trace) trace[(j) * 16 + (slot)] = clock64()

  if (threadIdx.x == 0) {
    for (int i = 0; i < B_N; ++i) {
      const bool sm = (i >= B_SFREE && i < B_SFREE + 2) || (i >= B_PF && i < B_PF + 2);
      tc::mbar_init(bar(i), sm ? 128 : 1);
    }
    tc::fence_barrier_init();
  }
  if (warp == 9) tc::tmem_alloc<512>(smem_u32(tmem_slot));
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tO = tmem + 256;

  // Roles: warps 0-7 softmax + epilogue (two warpgroups, alternate key tiles), 8 TMA producer, 9 TMEM allocator, 10 MMA issuer (the scheduler favours the
  // highest warp id, so the single issuing thread is never starved).
  if (warp == 8) {
    // K producer (and Q): K stage s is refilled as soon as S reading it has completed
    if (tc::elect_one()) {
      tc::tma_prefetch(&tmQ);
      tc::tma_prefetch(&tmK);
      tc::mbar_expect_tx(bar(B_Q), Lay::TILE);
      for (int b = 0; b < Lay::QB; ++b)
        tc::tma_load_2d(sQ + b * 16384, &tmQ, h * D + b * 64, P.q_row0 + m0, bar(B_Q));
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j & 1;
        if (j >= 2) tc::mbar_wait(bar(B_SF + st), ((j - 2) >> 1) & 1);  // S(j-2) done with K stage
        tc::mbar_expect_tx(bar(B_KF + st), Lay::TILE);
        for (int b = 0; b < Lay::QB; ++b)
          tc::tma_load_2d(sK + st * Lay::TILE + b * 16384, &tmK, kvh * D + b * 64, P.k_row0 + j * 128,
                          bar(B_KF + st));
      }
    }
  } else if (warp == 9) {
    // V producer (this warp also owns the TMEM allocation)
    if (tc::elect_one()) {
      tc::tma_prefetch(&tmV);
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j & 1;
        if (j >= 2) tc::mbar_wait(bar(B_PV + st), ((j - 2) >> 1) & 1);  // PV(j-2) done with V stage
        tc::mbar_expect_tx(bar(B_VF + st), Lay::TILE);
        for (int b = 0; b < Lay::QB; ++b)
          tc::tma_load_2d(sV + st * Lay::TILE + b * 16384, &tmV, kvh * D + b * 64, P.k_row0 + j * 128,
                          bar(B_VF + st));
      }
    }
  } else if (warp == 10 || (SPATTN_FWD_DUAL_ISSUE && warp == 11)) {
    if (tc::elect_one()) {
      constexpr uint32_t id_s = tc::idesc_bf16(128, 128, false, false);
      constexpr uint32_t id_o = tc::idesc_bf16(128, D, false, true);
      // S(j) -> S buffer j&1; needs K(j) and the group's previous tile j-2 read out of TMEM
      auto issue_s = [&](int j) {
        const int st = j & 1;
        FTR(0, j);
        tc::mbar_wait(bar(B_KF + st), (j >> 1) & 1);
        FTR(12, j);
        if (j >= 2) tc::mbar_wait(bar(B_SFREE + st), ((j - 2) >> 1) & 1);
        FTR(13, j);
        tc::fence_after();
        const uint32_t kbase = sK + st * Lay::TILE;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
          tc::mma_ss(tmem + st * 128, tc::sdesc(sQ + off, 16, 1024), tc::sdesc(kbase + off, 16, 1024),
                     id_s, ks > 0 ? 1u : 0u);
        }
        tc::commit(bar(B_SF + st));  // also releases K stage st (each commit costs ~27 pipe cycles)
        FTR(1, j);
      };
      // O_{i&1} += P(i) V(i)
      auto issue_pv = [&](int i) {
        const int st = i & 1;
        FTR(2, i);
        tc::mbar_wait(bar(B_PF + st), (i >> 1) & 1);
        FTR(3, i);
        tc::mbar_wait(bar(B_VF + st), (i >> 1) & 1);
        tc::fence_after();
        const uint32_t pbase = sP + st * Lay::P_TILE, vbase = sV + st * Lay::TILE;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (SPATTN_FWD_P_TMEM) {
            tc::mma_ts(tO + st * D, tmem + st * 128 + kk * 8, tc::sdesc(vbase + kk * 2048, 16384, 1024), id_o,
                       (i > 1 || kk > 0) ? 1u : 0u);
          } else {
            const uint32_t aoff = (kk >> 2) * 16384 + (kk & 3) * 32;
            tc::mma_ss(tO + st * D, tc::sdesc(pbase + aoff, 16, 1024),
                       tc::sdesc(vbase + kk * 2048, 16384, 1024), id_o, (i > 1 || kk > 0) ? 1u : 0u);
            if (SPATTN_FWD_PHALF && kk == 3) tc::commit(bar(B_PH + st));
          }
        }
        tc::commit(bar(B_PV + st));  // also releases V stage st
        FTR(4, i);
      };
      // order S0 S1 | S2 PV0 | S3 PV1 | ...: S(j+2) only needs group j&1 to have read S(j) out of
      // TMEM (early in its softmax), so it runs while that softmax is still computing P(j)
      if (SPATTN_FWD_DUAL_ISSUE) {
        const int g = warp - 10;  // this issuer's stream: key tiles j = g (mod 2)
        if (n_tiles > g) {
          tc::mbar_wait(bar(B_Q), 0);
          issue_s(g);
        }
        for (int j = g; j < n_tiles; j += 2) {
          if (!SPATTN_FWD_P_TMEM && j + 2 < n_tiles) issue_s(j + 2);
          issue_pv(j);
          if (SPATTN_FWD_P_TMEM && j + 2 < n_tiles) issue_s(j + 2);
        }
      } else if (SPATTN_FWD_P_TMEM) {
        if (n_tiles > 0) {
          tc::mbar_wait(bar(B_Q), 0);
          issue_s(0);
        }
        if (n_tiles > 1) issue_s(1);
        for (int j = 0; j < n_tiles; ++j) {
          issue_pv(j);  // reads P(j) from S buffer j&1 before S(j+2) overwrites it (pipe order)
          if (j + 2 < n_tiles) issue_s(j + 2);
        }
      } else {
        if (n_tiles > 0) {
          tc::mbar_wait(bar(B_Q), 0);
          issue_s(0);
        }
        if (n_tiles > 1) issue_s(1);
        for (int j = 0; j < n_tiles; ++j) {
          if (j + 2 < n_tiles) issue_s(j + 2);
          issue_pv(j);
        }
      }
    }
  } else if (warp < 8) {
    // Two independent online-softmax streams: warpgroup g owns the key tiles j = g (mod 2), its
    // S buffer g, P buffer g and O accumulator g, with its own running max/sum. Two tiles are in
    // flight at once, so one group's latency chain (TMEM load -> max -> exp -> P store) overlaps
    // the other's; the two partial results are merged in the epilogue.
    const int g = warp >> 2;
    const int row = threadIdx.x & 127;  // query row within the tile == TMEM lane
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + g * 128 + lane_base, tOg = tO + g * D + lane_base;
    const float sl2 = a.scale * kLog2e;
    const int qa = m0 + row;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = g; j < n_tiles; j += 2) {
      const int it = j >> 1;  // this group's iteration
      if (row == 0) FTR(5, j);
      tc::mbar_wait(bar(B_SF + g), it & 1);
      if (row == 0) FTR(6, j);
      if (ctr && j == 0 && threadIdx.x == 0) ctr[1] = gtimer();
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
      if (row == 0) FTR(8, j);
      tc::fence_before();
      tc::mbar_arrive(bar(B_SFREE + g));
      const int n0 = j * 128;
      const bool need_mask = (n0 + 128 > P.nk) || (P.causal && n0 + 127 > m0 + P.off);
      if (need_mask) {
        const int lim = P.causal ? min(P.nk - 1, qa + P.off) - n0 : P.nk - 1 - n0;
#pragma unroll
        for (int i = 0; i < 128; ++i) x[i] = i <= lim ? x[i] : -INFINITY;
      }
#ifndef SPATTN_FWD_MAX_CHAINS
#define SPATTN_FWD_MAX_CHAINS 4
#endif
      // max over raw scores (sl2 > 0); independent 3-input-max chains, then a tree
      constexpr int NCH = SPATTN_FWD_MAX_CHAINS;
      float mx[NCH];
#pragma unroll
      for (int c = 0; c < NCH; ++c) mx[c] = -INFINITY;
#pragma unroll
      for (int i = 0; i < 128; i += 2 * NCH) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) mx[c] = fmaxf(mx[c], fmaxf(x[i + 2 * c], x[i + 2 * c + 1]));
      }
#pragma unroll
      for (int w = NCH / 2; w > 0; w /= 2) {
#pragma unroll
        for (int c = 0; c < w; ++c) mx[c] = fmaxf(mx[c], mx[c + w]);
      }
      const float mt = mx[0] * sl2;
      if (row == 0) FTR(9, j);
      if (it == 0) {
        m_run = mt;
      } else if (__any_sync(0xffffffffu, mt > m_run + 8.f)) {
        // lazy rescale of O_g and l to a new running max (threshold 2^8); O_g holds PV(j-2)
        const float m_new = fmaxf(m_run, mt);
        const float alpha = (m_run == -INFINITY || m_new == -INFINITY) ? (m_run == m_new ? 1.f : 0.f)
                                                                        : fast_exp2(m_run - m_new);
        tc::mbar_wait(bar(B_PV + g), (it - 1) & 1);
        tc::fence_after();
        // (8-column chunks: the 128 scores of this tile are live in registers)
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
      if (row == 0) FTR(10, j);
      const float muse = m_run == -INFINITY ? 0.f : m_run;
      const uint64_t sc2 = f2_pack(sl2, sl2), nm2 = f2_pack(-muse, -muse);
      uint64_t rs2[2] = {0ull, 0ull};  // packed (even, odd) partial row sums
      uint32_t pw[64];                 // P row as bf16 pairs
#pragma unroll
      for (int e = 0; e < 64; ++e) {
        const float2 av = f2_unpack(f2_fma(f2_pack(x[2 * e], x[2 * e + 1]), sc2, nm2));
        // pairs in fwd_poly_pairs<D>() run on the FMA pipe instead of the MUFU (16/clk/SM)
        float2 pv;
#ifdef SPATTN_FWD_PROBE_NOEXP
        pv = av;  // profiling probe: no exponentials (wrong results)
        if (false) {
#else
        if ((fwd_poly_pairs<D>() >> (e & 3)) & 1) {
#endif
          pv = poly_exp2x2(av.x, av.y);
        } else {
          pv.x = fast_exp2(av.x);
          pv.y = fast_exp2(av.y);
        }
        rs2[e & 1] = f2_add(rs2[e & 1], f2_pack(pv.x, pv.y));
        pw[e] = pack_bf16(pv.x, pv.y);
      }
#ifdef SPATTN_FWD_PROBE_NOSTORE
      if (true) {  // profiling probe: P never written (wrong results)
      } else
#endif
      if (SPATTN_FWD_P_TMEM) {
        // P(j) over the first 64 columns of this group's S buffer (its S values are in x[] now)
        tc::tmem_st32(tS, *reinterpret_cast<uint32_t(*)[32]>(&pw[0]));
        tc::tmem_st32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&pw[32]));
        tc::tmem_wait_st();
      } else {
        // P buffer g was last read by PV(j-2): each 64-key half is stored once PV(j-2) has read it
        const uint32_t pbase = sP + g * Lay::P_TILE;
#pragma unroll
        for (int ch = 0; ch < 16; ++ch) {
          if (it > 0 && ch == 0) tc::mbar_wait(bar(SPATTN_FWD_PHALF ? B_PH + g : B_PV + g), (it - 1) & 1);
          if (SPATTN_FWD_PHALF && it > 0 && ch == 8) tc::mbar_wait(bar(B_PV + g), (it - 1) & 1);
          const uint32_t addr = tc::sw128(pbase + (ch >> 3) * 16384, row, ch & 7);
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};\n" ::"r"(addr), "r"(pw[4 * ch]),
                       "r"(pw[4 * ch + 1]), "r"(pw[4 * ch + 2]), "r"(pw[4 * ch + 3]));
        }
      }
      {
        const float2 r = f2_unpack(f2_add(rs2[0], rs2[1]));
        l_run += r.x + r.y;
      }
      if (row == 0) FTR(11, j);
      tc::fence_before();
      tc::fence_proxy_async();
      tc::mbar_arrive(bar(B_PF + g));
      if (row == 0) FTR(7, j);
    }
    if (ctr && threadIdx.x == 0) ctr[2] = gtimer();
    // ---- epilogue: merge the two streams; group g writes output columns [g*D/2, (g+1)*D/2)
    const bool valid = qa < P.nq;
    const int64_t grow = (int64_t)(P.q_row0 + qa);
    float* lp = a.lse + grow * a.lse_row_stride + h;
    const float la = (a.acc_o != nullptr && valid) ? *lp : -INFINITY;  // read before any write
    float* xch = reinterpret_cast<float*>(smem + Lay::XCH_OFF);    // [m: 2][128], [l: 2][128]
    xch[g * 128 + row] = m_run;
    xch[256 + g * 128 + row] = l_run;
    asm volatile("bar.sync 1, 256;\n" ::: "memory");
    const float m_o = xch[(g ^ 1) * 128 + row], l_o = xch[256 + (g ^ 1) * 128 + row];
    const float m = fmaxf(m_run, m_o);
    const float w_own = m_run == -INFINITY ? 0.f : fast_exp2(m_run - m);
    const float w_oth = m_o == -INFINITY ? 0.f : fast_exp2(m_o - m);
    const float l = l_run * w_own + l_o * w_oth;
    const bool empty = m == -INFINITY || !(l > 0.f);  // poly_exp2 never returns exactly 0
    const float inv = empty ? 0.f : 1.f / l;
    const float lse_row = empty ? -INFINITY : (m + __log2f(l)) * kLn2;
    const bool have_own = n_tiles > g, have_oth = n_tiles > (g ^ 1);
    if (n_tiles > 0) {
      tc::mbar_wait(bar(B_PV + ((n_tiles - 1) & 1)), ((n_tiles - 1) >> 1) & 1);  // all MMAs done
      tc::fence_after();
    }
    const uint32_t tOo = tO + (g ^ 1) * D + lane_base;
    constexpr int DH = D / 2;
    // merged, normalised O column chunk c (32 columns) of this group's half
    auto o_chunk = [&](int c, float* o) {
      uint32_t r[32], q[32];
      if (have_own) tc::tmem_ld32(tOg + g * DH + c * 32, r);
      if (have_oth) tc::tmem_ld32(tOo + g * DH + c * 32, q);
      tc::tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i)
        o[i] = ((have_own ? __uint_as_float(r[i]) * w_own : 0.f) +
                (have_oth ? __uint_as_float(q[i]) * w_oth : 0.f)) * inv;
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
      const float mx = fmaxf(la, lb);
      float wa = 1.f, wb = 0.f, ln = la;
      if (mx != -INFINITY) {
        ln = mx + __logf(__expf(la - mx) + __expf(lb - mx));
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
  __syncthreads();
  if (warp == 9) tc::tmem_dealloc<512>(tmem);
  if (ctr && threadIdx.x == 0) ctr[3] = gtimer();
}

int max_rows(const ProblemSet& ps, bool q) {
  int m = 0;
  for (int i = 0; i < ps.n; ++i) m = max(m, q ? ps.p[i].q_row0 + ps.p[i].nq : ps.p[i].k_row0 + ps.p[i].nk);
  return m;
}

template <int D>
void launch_fwd_tc_d(const FwdArgs& a, const ProblemSet& in, cudaStream_t s) {
  ProblemSet ps;
  copy_problems(ps, in);
  ps.tile_prefix[0] = 0;
  for (int i = 0; i < ps.n; ++i) ps.tile_prefix[i + 1] = ps.tile_prefix[i] + (ps.p[i].nq + 127) / 128;
  const int tiles = ps.tile_prefix[ps.n];
  if (tiles == 0 || a.hm.hq == 0) return;
  CUtensorMap tq, tk, tv;
  const uint64_t qw = (uint64_t)a.q_row_stride, kw = (uint64_t)a.kv_row_stride;
  if (!make_tma_2d(&tq, a.q, qw, max_rows(ps, true), qw, 128) ||
      !make_tma_2d(&tk, a.k, kw, max(1, max_rows(ps, false)), kw, 128) ||
      !make_tma_2d(&tv, a.v, kw, max(1, max_rows(ps, false)), kw, 128))
    launch_error("attn_fwd_tc", "TMA descriptor encode failed (q/k/v base, strides or extents)");
  with_problem_set(ps, [&](const auto& set) {
    using PS = std::decay_t<decltype(set)>;
    ensure_smem_for(attn_fwd_tc_kernel<D, PS>, FwdLayout<D>::SMEM);
    attn_fwd_tc_kernel<D, PS><<<dim3(tiles, a.hm.hq), kFwdThreads, FwdLayout<D>::SMEM, s>>>(tq, tk, tv, a, set);
  });
  note_launch();
}

}  // namespace

bool tc_fwd_supported(const FwdArgs& a) {
  const bool aligned = (reinterpret_cast<uintptr_t>(a.q) % 16 == 0) && (reinterpret_cast<uintptr_t>(a.k) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(a.v) % 16 == 0) && (a.q_row_stride * 2) % 16 == 0 &&
                       (a.kv_row_stride * 2) % 16 == 0;
  return (a.d == 64 || a.d == 128) && aligned;
}
void launch_attn_fwd_tc(const FwdArgs& a, const ProblemSet& ps, cudaStream_t s) {
  if (a.d == 64)
    launch_fwd_tc_d<64>(a, ps, s);
  else
    launch_fwd_tc_d<128>(a, ps, s);
}

}  // namespace spattn
