// ex2 variants throughput + softmax row mix throughput per SM
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdint.h>
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ float2 f2_unpack(uint64_t v) { float2 r; asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v)); return r; }
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) { uint64_t d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) { __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi); return *reinterpret_cast<uint32_t*>(&v); }
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

template <int MODE>
__global__ void probe(float* out, int iters, long long* cyc) {
  float s[128];
  for (int i = 0; i < 128; ++i) s[i] = -0.01f * ((threadIdx.x + i) & 63);
  float l = 0.f; uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {  // f32 ex2 path: FFMA2, 2 MUFU, FADD2, F2FP per pair
      const uint64_t sc2 = f2_pack(1.4427f, 1.4427f), nm2 = f2_pack(-0.5f, -0.5f);
      uint64_t rs2[2] = {0, 0};
#pragma unroll
      for (int e = 0; e < 64; ++e) {
        const float2 av = f2_unpack(f2_fma(f2_pack(s[2 * e], s[2 * e + 1]), sc2, nm2));
        float2 pv; pv.x = ex2(av.x); pv.y = ex2(av.y);
        rs2[e & 1] = f2_add(rs2[e & 1], f2_pack(pv.x, pv.y));
        acc ^= pack_bf16(pv.x, pv.y);
      }
      const float2 r = f2_unpack(f2_add(rs2[0], rs2[1])); l += r.x + r.y;
    }
    if (MODE == 1) {  // f16x2 ex2: FFMA2, F2FP.F16, MUFU.EX2.F16x2, unpack 2 cvt, FADD2, F2FP.BF16
      const uint64_t sc2 = f2_pack(1.4427f, 1.4427f), nm2 = f2_pack(-0.5f, -0.5f);
      uint64_t rs2[2] = {0, 0};
#pragma unroll
      for (int e = 0; e < 64; ++e) {
        const float2 av = f2_unpack(f2_fma(f2_pack(s[2 * e], s[2 * e + 1]), sc2, nm2));
        __half2 h = __floats2half2_rn(av.x, av.y);
        uint32_t hi = *reinterpret_cast<uint32_t*>(&h), ho;
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(ho) : "r"(hi));
        __half2 hv = *reinterpret_cast<__half2*>(&ho);
        float2 pv = __half22float2(hv);
        rs2[e & 1] = f2_add(rs2[e & 1], f2_pack(pv.x, pv.y));
        acc ^= pack_bf16(pv.x, pv.y);
      }
      const float2 r = f2_unpack(f2_add(rs2[0], rs2[1])); l += r.x + r.y;
    }
    if (MODE == 2) {  // bf16x2 ex2: FFMA2, F2FP.BF16, MUFU.EX2.BF16x2, unpack (2 ops), FADD2; P is the ex2 output
      const uint64_t sc2 = f2_pack(1.4427f, 1.4427f), nm2 = f2_pack(-0.5f, -0.5f);
      uint64_t rs2[2] = {0, 0};
#pragma unroll
      for (int e = 0; e < 64; ++e) {
        const float2 av = f2_unpack(f2_fma(f2_pack(s[2 * e], s[2 * e + 1]), sc2, nm2));
        uint32_t bi = pack_bf16(av.x, av.y), bo;
        asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(bo) : "r"(bi));
        float2 pv = make_float2(__uint_as_float(bo << 16), __uint_as_float(bo & 0xffff0000u));
        rs2[e & 1] = f2_add(rs2[e & 1], f2_pack(pv.x, pv.y));
        acc ^= bo;
      }
      const float2 r = f2_unpack(f2_add(rs2[0], rs2[1])); l += r.x + r.y;
    }
    if (MODE == 3) {  // pure f32 MUFU
#pragma unroll
      for (int e = 0; e < 128; ++e) l += 0.f * ex2(s[e]);
    }
    if (MODE == 4) {  // pure f16x2 MUFU
#pragma unroll
      for (int e = 0; e < 64; ++e) {
        uint32_t ho, hi = __float_as_uint(s[2 * e]);
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(ho) : "r"(hi));
        acc ^= ho;
      }
    }
    for (int i = 0; i < 128; ++i) s[i] += 1e-7f * (acc & 1);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = l + acc;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"f32 mix", "f16x2 mix", "bf16x2 mix", "pure ex2 f32", "pure ex2 f16x2"};
  for (int mode = 0; mode < 5; ++mode)
    for (int warps : {4, 8, 16}) {
      int iters = 200;
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) probe<0><<<148, warps * 32>>>(out, iters, cyc);
        if (mode == 1) probe<1><<<148, warps * 32>>>(out, iters, cyc);
        if (mode == 2) probe<2><<<148, warps * 32>>>(out, iters, cyc);
        if (mode == 3) probe<3><<<148, warps * 32>>>(out, iters, cyc);
        if (mode == 4) probe<4><<<148, warps * 32>>>(out, iters, cyc);
      }
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      // elements per SMSP per iteration = (warps/4) * 32 * 128
      double per_tile = (double)c / iters / (warps / 4) * 1.0;  // cycles per (32 rows x 128) per SMSP
      printf("%-16s warps/SMSP %2d: %.0f cycles per 32x128 tile per SMSP (%.2f exps/clk/SM)\n", names[mode], warps / 4,
             per_tile, 4.0 * 4096 / per_tile);
    }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
