// tcgen05.mma issue-rate probe (profiling helper): back-to-back kind::f16 MMAs from one thread,
// one CTA per SM, optionally with 4 warps streaming st.shared (the softmax P stores) or a
// second SS stream. Reports tensor-pipe cycles per MMA and the implied smem operand bytes/clk.
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2505_22296_b200/csrc \
//   -I include -o tools/umma_bench tools/umma_bench.cu -lcuda
#include <cstdio>
#include "tc.cuh"

using namespace spattn;

template <int MODE>
__global__ void __launch_bounds__(256, 1) probe(long long* out, int iters, const uint8_t* gsrc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t mb;
  __shared__ volatile int done;
  __shared__ __align__(8) uint64_t mb2[2];
  const uint32_t sb = smem_u32(smem);
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    tc::mbar_init(smem_u32(&mb), 1);
    tc::mbar_init(smem_u32(&mb2[0]), 1);
    tc::mbar_init(smem_u32(&mb2[1]), 1);
    tc::fence_barrier_init();
    done = 0;
  }
  if (warp == 0) tc::tmem_alloc<512>(smem_u32(&tslot));
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tslot;
  constexpr int N = (MODE == 1) ? 256 : ((MODE == 4 || MODE == 15) ? 64 : 128);
  if (warp == 7) {
    if (tc::elect_one()) {
      const uint32_t id = tc::idesc_bf16(128, N, false, false);
      long long t0 = clock64(), wsum = 0, isum = 0;
      if (MODE >= 11 && MODE <= 14) {
        constexpr int G = MODE == 12 ? 2 : 8;
        __shared__ __align__(8) uint64_t pre;
        tc::mbar_init(smem_u32(&pre), 1);
        tc::fence_barrier_init();
        tc::mbar_arrive(smem_u32(&pre));  // phase 0 complete
        for (int i = 0; i < iters / 8; ++i) {
          const long long a0 = clock64();
#pragma unroll
          for (int k = 0; k < G; ++k)
            if (MODE != 14)
              tc::mma_ss(tm, tc::sdesc(sb + k * 32, 16, 1024), tc::sdesc(sb + 65536 + k * 32, 16, 1024), id, 1u);
          if (MODE != 13) tc::commit(smem_u32(&mb2[i & 1]));
          const long long a1 = clock64();
          tc::mbar_wait(smem_u32(&pre), 0);
          const long long a2 = clock64();
          isum += a1 - a0;
          wsum += a2 - a1;
        }
        out[2 * gridDim.x + blockIdx.x] = wsum;
        out[3 * gridDim.x + blockIdx.x] = isum;
      }
      for (int i = 0; i < ((MODE >= 11 && MODE <= 14) ? 0 : iters); ++i) {
        const uint32_t ko = (i & 3) * 32;
        if (MODE == 2 || MODE == 15)
          tc::mma_ts(tm, tm + 256 + (i & 3) * 8, tc::sdesc(sb + 65536 + ko, 16, 1024), id, 1u);
        else if (MODE >= 16 && MODE <= 22) {  // one bwd q64 iteration per 8 loop trips (40 MMAs): S^T, dP^T,
          // dV (TS), dK, dQ^T with the kernel's descriptors; i counts iterations here
          const uint32_t sK = sb, sV = sb + 32768, sQ = sb + 65536, sdO = sb + 81920, ds = sb + 98304;
          const uint32_t id_s = tc::idesc_bf16(128, 64, false, false), id_kv = tc::idesc_bf16(128, 128, false, true),
                         id_q = tc::idesc_bf16(128, 64, true, true);
          constexpr bool all = MODE == 16;
          if (all || MODE == 17)
          for (int ks = 0; ks < 8; ++ks) {
            const uint32_t kof = (ks >> 2) * 16384 + (ks & 3) * 32, qo = (ks >> 2) * 8192 + (ks & 3) * 32;
            tc::mma_ss(tm, tc::sdesc(sK + kof, 16, 1024), tc::sdesc(sQ + qo, 16, 1024), id_s, ks > 0);
          }
          if (all || MODE == 18)
          for (int ks = 0; ks < 8; ++ks) {
            const uint32_t kof = (ks >> 2) * 16384 + (ks & 3) * 32, qo = (ks >> 2) * 8192 + (ks & 3) * 32;
            tc::mma_ss(tm + 128, tc::sdesc(sV + kof, 16, 1024), tc::sdesc(sdO + qo, 16, 1024), id_s, ks > 0);
          }
          if (all || MODE == 19)
          for (int kk = 0; kk < 4; ++kk)
            tc::mma_ts(tm + 256, tm + 64 + kk * 8, tc::sdesc(sdO + kk * 2048, 8192, 1024), id_kv, 1u);
          if (all || MODE == 20)
          for (int kk = 0; kk < 4; ++kk)
            tc::mma_ss(tm + 384, tc::sdesc(ds + kk * 32, 16, 1024), tc::sdesc(sQ + kk * 2048, 8192, 1024), id_kv, 1u);
          if (all || MODE == 21)
          for (int kk = 0; kk < 8; ++kk)
            tc::mma_ss(tm + 192, tc::sdesc(sK + kk * 2048, 16384, 1024), tc::sdesc(ds + kk * 2048, 8192, 1024), id_q, kk > 0);
          if (MODE == 22)  // dQ (not transposed): M=64 queries... as two N64 halves is not possible; M=128 rows of dS^T? use K-major A = dS^T^T
          for (int kk = 0; kk < 8; ++kk)
            tc::mma_ss(tm + 192, tc::sdesc(sK + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), tc::sdesc(ds + kk * 2048, 8192, 1024),
                       tc::idesc_bf16(128, 64, false, true), kk > 0);
          if (i + 1 >= iters / 40) break;
        }
        else if (MODE == 8 || MODE == 9 || MODE == 10) {  // the fwd kernel's pattern: groups of 8 into alternating accumulators + 2 commits
          const bool pv = (i >> 3) & 1;
          tc::mma_ss(tm + (pv ? 256 : 0) + ((i >> 4) & 1) * 128, tc::sdesc(sb + ko, 16, 1024),
                     pv ? tc::sdesc(sb + 65536 + (i & 7) * 2048, 16384, 1024) : tc::sdesc(sb + 65536 + ko, 16, 1024),
                     tc::idesc_bf16(128, 128, false, pv), (i & 7) ? 1u : 0u);
          if ((i & 7) == 7 && MODE != 10) {
            tc::commit(smem_u32(&mb2[0]));
            if (MODE == 8) tc::commit(smem_u32(&mb2[1]));
          }
        } else if (MODE == 5)  // B MN-major (the PV shape: V rows are the K dimension)
          tc::mma_ss(tm, tc::sdesc(sb + ko, 16, 1024), tc::sdesc(sb + 65536 + (i & 7) * 2048, 16384, 1024),
                     tc::idesc_bf16(128, 128, false, true), 1u);
        else
          tc::mma_ss(tm, tc::sdesc(sb + ko, 16, 1024), tc::sdesc(sb + 65536 + ko, 16, 1024), id, 1u);
      }
      tc::commit(smem_u32(&mb));
      tc::mbar_wait(smem_u32(&mb), 0);
      long long t1 = clock64();
      out[blockIdx.x] = t1 - t0;
      done = 1;
    }
  } else if (MODE == 6 && warp < 4) {
    // stream tcgen05.ld of 32 columns from the upper TMEM half (the softmax reading S)
    long long n = 0;
    uint32_t acc = 0;
    while (!done) {
      uint32_t r[32];
      tc::tmem_ld32(tm + ((uint32_t)(warp * 32) << 16) + 256 + (n & 7) * 32, r);
      tc::tmem_wait_ld();
      acc ^= r[0] ^ r[31];
      ++n;
    }
    if (threadIdx.x == 0) out[gridDim.x + blockIdx.x] = n + (acc == 12345);
  } else if (MODE == 7 && warp == 0) {
    // bulk global->smem copies of 16 KB into a separate region (the K/V TMA traffic)
    if (tc::elect_one()) {
      __shared__ __align__(8) uint64_t cb;
      tc::mbar_init(smem_u32(&cb), 1);
      tc::fence_barrier_init();
      long long n = 0;
      while (!done) {
        tc::mbar_expect_tx(smem_u32(&cb), 16384);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];\n"
                     ::"r"(sb + 131072 + (uint32_t)(n & 3) * 16384), "l"(gsrc + (blockIdx.x * 4 + (n & 3)) * 16384),
                     "r"(smem_u32(&cb)) : "memory");
        tc::mbar_wait(smem_u32(&cb), n & 1);
        ++n;
      }
      out[gridDim.x + blockIdx.x] = n;
    }
  } else if (MODE == 3 && warp < 4) {
    // stream 16-byte stores over a 32 KB region, like the softmax writing P
    const uint32_t base = sb + 131072;
    long long n = 0;
    while (!done) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t a = base + ((threadIdx.x * 16 + k * 2048 + (int)n * 16) & 32767);
        asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};\n" ::"r"(a), "r"((uint32_t)n));
      }
      ++n;
    }
    if (threadIdx.x == 0) out[gridDim.x + blockIdx.x] = n;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tm);
}

template <int MODE>
void run(const char* name, long long* d, int iters, const uint8_t* g) {
  cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int r = 0; r < 2; ++r) probe<MODE><<<148, 256, 200 * 1024>>>(d, iters, g);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[600];
  cudaMemcpy(h, d, 600 * 8, cudaMemcpyDeviceToHost);
  const int N = (MODE == 1) ? 256 : ((MODE == 4 || MODE == 15) ? 64 : 128);
  const double cyc = (double)h[0] / (MODE >= 16 && MODE <= 22 ? iters / 40 : iters);
  const double ideal = 128.0 * N * 16 * 2 / 8192.0;  // cycles at 8192 dense bf16 flop/clk/SM
  const double bytes = (MODE == 2 || MODE == 15 ? 0 : 128 * 16 * 2) + N * 16 * 2;
  if (MODE >= 16 && MODE <= 22) {
    printf("%-28s %s cycles/iteration %.1f (ideal at 8192 flop/clk: %.0f)\n", name, cudaGetErrorString(e), cyc,
           5.0 * 128 * 64 * 128 * 2 / 8192.0);
    return;
  }
  printf("%-28s %s cycles/MMA %.1f (ideal %.0f) smem operand B/clk %.0f", name, cudaGetErrorString(e),
         cyc, ideal, bytes / cyc);
  if (MODE == 3) printf("  store B/clk %.1f", (double)h[148] * 128 * 16 * 16 / h[0]);
  if (MODE >= 11 && MODE <= 14) printf("  per group of 8: issue+commit %.0f cycles, satisfied mbar_wait %.0f cycles", (double)h[3 * 148] / (iters / 8), (double)h[2 * 148] / (iters / 8));
  if (MODE == 6) printf("  tmem ld B/clk %.1f", (double)h[148] * 128 * 32 * 4 / h[0]);
  if (MODE == 7) printf("  bulk copy B/clk %.1f", (double)h[148] * 16384 / h[0]);
  printf("\n");
}

int main() {
  long long* d;
  cudaMalloc(&d, 600 * 8);
  cudaMemset(d, 0, 600 * 8);
  const int it = 1 << 16;
  uint8_t* g;
  cudaMalloc(&g, 148 * 4 * 16384);
  run<0>("SS M128 N128 K16", d, it, g);
  run<1>("SS M128 N256 K16", d, it, g);
  run<4>("SS M128 N64 K16", d, it, g);
  run<2>("TS M128 N128 K16 (A tmem)", d, it, g);
  run<15>("TS M128 N64 K16 (A tmem)", d, it, g);
  run<16>("bwd q64 iteration (40 MMAs)", d, it, g);
  run<17>("  S^T only (8 SS N64)", d, it, g);
  run<18>("  dP^T only (8 SS N64)", d, it, g);
  run<19>("  dV only (4 TS N128)", d, it, g);
  run<20>("  dK only (4 SS N128 Bmn)", d, it, g);
  run<21>("  dQ^T only (8 SS N64 A mn)", d, it, g);
  run<22>("  dQ^T with K-major A (8 SS N64)", d, it, g);
  run<5>("SS M128 N128 B MN-major", d, it, g);
  run<8>("fwd pattern (8 S, 2 commits, 8 PV)", d, it, g);
  run<9>("fwd pattern, 1 commit", d, it, g);
  run<10>("fwd pattern, no commit", d, it, g);
  run<11>("8 SS + commit + mbar_wait", d, it, g);
  run<12>("2 SS + commit + mbar_wait", d, it, g);
  run<13>("8 SS, no commit + mbar_wait", d, it, g);
  run<14>("commit only + mbar_wait", d, it, g);
  run<3>("SS M128 N128 + st.shared", d, it, g);
  run<6>("SS M128 N128 + tcgen05.ld", d, it, g);
  run<7>("SS M128 N128 + bulk copy", d, it, g);
  return 0;
}
