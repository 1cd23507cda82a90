// Device helpers shared by the sm_100a kernels of the SP attention layer.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "spattn_internal.h"

namespace spattn {

// The problem a launch's tile (or tile pair) index belongs to: the first pi in [0, n) with
// tile_prefix[pi + 1] > tile (binary search over up to kMaxProblems prefix sums).
template <class PS>
__device__ __forceinline__ int find_problem(const PS& ps, int tile) {
  int lo = 0, hi = ps.n - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (ps.tile_prefix[mid + 1] > tile)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte async global->shared copy; src_bytes < 16 zero-fills the tail (0 = zero row).
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// D(16x8,f32) += A(16x16,bf16,row) * B(16x8,bf16,col)
__device__ __forceinline__ void mma_bf16(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}

// Packed fp32x2 arithmetic (FFMA2/FADD2, sm_100): one issue slot for two results. The softmax
// loops are issue-bound (one instruction per clock per SMSP), so these halve their cost.
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 f2_unpack(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// poly_exp2 (below) on a packed pair.
__device__ __forceinline__ float2 poly_exp2x2(float a0, float a1) {
  const uint64_t magic = f2_pack(12582912.f, 12582912.f);
  const uint64_t x = f2_pack(fmaxf(a0, -126.f), fmaxf(a1, -126.f));
  const uint64_t t = f2_add(x, magic);
  const uint64_t f = f2_sub(x, f2_sub(t, magic));
  uint64_t p = f2_fma(f2_pack(0.05517032742500305f, 0.05517032742500305f), f,
                      f2_pack(0.24260781705379486f, 0.24260781705379486f));
  p = f2_fma(p, f, f2_pack(0.693260908126831f, 0.693260908126831f));
  p = f2_fma(p, f, f2_pack(0.9999282956123352f, 0.9999282956123352f));
  const float2 pv = f2_unpack(p), tv = f2_unpack(t);
  return make_float2(__int_as_float(__float_as_int(pv.x) + (__float_as_int(tv.x) << 23)),
                     __int_as_float(__float_as_int(pv.y) + (__float_as_int(tv.y) << 23)));
}

// 2^x for x <= 0 on the FP32/INT pipes instead of the MUFU (16 results/clk/SM on B200), used for
// a fraction of the softmax exponentials so the two pipes finish together. Round-to-nearest split
// x = j + f, f in [-1/2, 1/2]; 2^f by a degree-3 fit (max relative error 7.6e-5, far below the
// bf16 rounding of P); j added to the exponent field. Inputs below -126 clamp to ~2^-126.
__device__ __forceinline__ float poly_exp2(float x) {
  x = fmaxf(x, -126.f);
  const float t = __fadd_rn(x, 12582912.f);  // 1.5 * 2^23: integer part lands in the low bits
  const float j = __fsub_rn(t, 12582912.f);
  const float f = __fsub_rn(x, j);
  const float p = fmaf(fmaf(fmaf(0.05517032742500305f, f, 0.24260781705379486f), f, 0.693260908126831f), f,
                       0.9999282956123352f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// Shared tile of `rows` x D bf16 stored with 16-byte chunks XOR-swizzled by (row & 7) so that
// ldmatrix row gathers and cp.async row writes are bank-conflict free.
template <int D>
__device__ __forceinline__ uint32_t swz(uint32_t base, int row, int chunk) {
  return base + row * (D * 2) + ((chunk ^ (row & 7)) << 4);
}

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

}  // namespace spattn
