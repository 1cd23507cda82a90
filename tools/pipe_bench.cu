// Throughput probe for the softmax instruction mix (profiling helper):
// MUFU.EX2, F2FP.BF16.F32.PACK_AB (cvt.rn.bf16x2.f32), and the two interleaved.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_bench tools/pipe_bench.cu
#include <cstdio>
#include <cuda_bf16.h>

template <int MODE>
__global__ void probe(float* out, int iters, long long* cyc) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  unsigned acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0 || MODE == 2) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (MODE == 1 || MODE == 2) {
        unsigned r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        acc ^= r;
      }
      if (MODE == 4) a[i] = fmaf(a[i], 1.0001f, -0.0001f);
      if (MODE == 5 && (i & 1) == 0) {  // packed pair: two results per instruction
        unsigned long long x, m, c;
        float2 xv = make_float2(a[i], a[i + 1]), mv = make_float2(1.0001f, 1.0001f), cv = make_float2(-1e-4f, -1e-4f);
        x = *reinterpret_cast<unsigned long long*>(&xv);
        m = *reinterpret_cast<unsigned long long*>(&mv);
        c = *reinterpret_cast<unsigned long long*>(&cv);
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(m), "l"(c));
        xv = *reinterpret_cast<float2*>(&x);
        a[i] = xv.x;
        a[i + 1] = xv.y;
      }
      if (MODE == 3) {  // integer rounding pack on the ALU: 2 IADD + PRMT
        unsigned x = __float_as_uint(a[i]) + 0x8000u, y = __float_as_uint(a[(i + 1) & 7]) + 0x8000u, r;
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(x), "r"(y));
        acc ^= r;
        a[i] = __uint_as_float(__float_as_uint(a[i]) ^ (r & 1));
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  const char* names[] = {"ex2", "cvt.bf16x2", "ex2+cvt", "iadd+prmt pack", "ffma", "ffma2 (per fp32 result)"};
  for (int mode = 0; mode < 6; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) probe<0><<<148, 512>>>(out, iters, cyc);
      if (mode == 1) probe<1><<<148, 512>>>(out, iters, cyc);
      if (mode == 2) probe<2><<<148, 512>>>(out, iters, cyc);
      if (mode == 3) probe<3><<<148, 512>>>(out, iters, cyc);
      if (mode == 4) probe<4><<<148, 512>>>(out, iters, cyc);
      if (mode == 5) probe<5><<<148, 512>>>(out, iters, cyc);
    }
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    // ops per SM = 512 threads * iters * 8
    printf("%-16s %.2f ops/clk/SM\n", names[mode], 512.0 * iters * 8 / c);
  }
  return 0;
}
