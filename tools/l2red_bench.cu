// Microbenchmark: fp32 reduce-add throughput into global memory on B200 (sizes within and
// beyond L2), to choose the dQ accumulation strategy of the attention backward.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2red l2red_bench.cu
// Modes: 0 = TMA bulk tensor reduce-add (box 32 fp32 x 128 rows, 128B swizzle) from smem,
//        1 = red.global.add.v4.f32, a warp covers 512 contiguous bytes (coalesced),
//        2 = red.global.add.v4.f32, lane = row (each warp touches 32 rows; the old dQ path),
//        3 = plain st.global.v4 (reference).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void __launch_bounds__(128) k_tma(const __grid_constant__ CUtensorMap m, int tiles_x, int tiles_y, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  float* s = reinterpret_cast<float*>(smem);
  for (int i = threadIdx.x; i < 4096; i += 128) s[i] = 1.0f;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(s));
    for (int it = 0; it < iters; ++it) {
      const int t = (blockIdx.x + it * gridDim.x) % (tiles_x * tiles_y);
      const int x = (t % tiles_x) * 32, y = (t / tiles_x) * 128;
      asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];\n"
                   :: "l"(reinterpret_cast<uint64_t>(&m)), "r"(x), "r"(y), "r"(src) : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 3;\n" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
}

// each "tile" = 128 rows x 32 fp32 (16 KB) at the same coordinates as the TMA tiles
__global__ void __launch_bounds__(128) k_red(float* g, int ld, int tiles_x, int tiles_y, int iters, int mode) {
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  for (int it = 0; it < iters; ++it) {
    const int t = (blockIdx.x + it * gridDim.x) % (tiles_x * tiles_y);
    const int x = (t % tiles_x) * 32, y = (t / tiles_x) * 128;
    if (mode == 1) {  // warp w: rows w*32..w*32+31; per instruction 4 rows x 128 B (8 lanes/row)
      for (int r = 0; r < 32; r += 4) {
        const int row = y + warp * 32 + r + lane / 8;
        float* p = g + (int64_t)row * ld + x + (lane % 8) * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};\n" :: "l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
      }
    } else if (mode == 2) {  // lane = row, 8 x 16 B per row
      const int row = y + warp * 32 + lane;
      for (int c = 0; c < 8; ++c) {
        float* p = g + (int64_t)row * ld + x + c * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};\n" :: "l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
      }
    } else {
      for (int r = 0; r < 32; r += 4) {
        const int row = y + warp * 32 + r + lane / 8;
        float4* p = reinterpret_cast<float4*>(g + (int64_t)row * ld + x + (lane % 8) * 4);
        *p = make_float4(1.f, 1.f, 1.f, 1.f);
      }
    }
  }
}

int main() {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  EncodeFn enc = reinterpret_cast<EncodeFn>(fp);
  const int sms = 148;
  for (int64_t rows : {4096LL, 32768LL}) {  // 64 MB (fits L2) and 512 MB (does not)
    const int ld = 4096;  // 32 heads x 128 fp32
    float* g;
    CK(cudaMalloc(&g, rows * ld * 4));
    CK(cudaMemset(g, 0, rows * ld * 4));
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) {
      printf("encode failed\n");
      return 1;
    }
    const int tiles_x = ld / 32, tiles_y = (int)(rows / 128);
    const int iters = 400;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 17 * 1024);
    for (int mode = 0; mode < 4; ++mode) {
      for (int grid : {sms, 4 * sms}) {
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(a);
          if (mode == 0) k_tma<<<grid, 128, 17 * 1024>>>(m, tiles_x, tiles_y, iters);
          else k_red<<<grid, 128>>>(g, ld, tiles_x, tiles_y, iters, mode);
          cudaEventRecord(b);
          CK(cudaEventSynchronize(b));
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (rep == 1)
            printf("rows %6lld mode %d grid %4d: %8.1f GB/s (%.3f ms)\n", (long long)rows, mode, grid,
                   (double)grid * iters * 16384 / (ms * 1e-3) / 1e9, ms);
        }
      }
    }
    CK(cudaGetLastError());
    cudaFree(g);
  }
  return 0;
}
