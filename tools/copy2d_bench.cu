// Pitched host<->device copy throughput (profiling helper): the host step moves head-group
// column slices of [L, heads, dim] rows with cudaMemcpy2DAsync; this measures GB/s by row width.
// nvcc -O2 -o tools/copy2d_bench tools/copy2d_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t rows = 32768, pitch = 8192;  // c2 q rows: 32 heads x 128 dims x bf16
  char *h, *d;
  cudaHostAlloc(&h, rows * pitch, cudaHostAllocDefault);
  cudaMalloc(&d, rows * pitch);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int dir = 0; dir < 2; ++dir)
    for (size_t w : {256, 512, 1024, 2048, 4096, 8192}) {
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a, s);
        for (size_t c = 0; c < pitch / w; ++c) {  // the whole buffer, in w-wide column slices
          if (dir == 0)
            cudaMemcpy2DAsync(d + c * w * rows, w, h + c * w, pitch, w, rows, cudaMemcpyHostToDevice, s);
          else
            cudaMemcpy2DAsync(h + c * w, pitch, d + c * w * rows, w, w, rows, cudaMemcpyDeviceToHost, s);
        }
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("%s width %5zu B: %.1f GB/s\n", dir ? "D2H" : "H2D", w, rows * pitch / best / 1e6);
    }
  // both directions at once (two streams), 1 KB slices
  cudaStream_t s2;
  cudaStreamCreate(&s2);
  char *h2, *d2;
  cudaHostAlloc(&h2, rows * pitch, cudaHostAllocDefault);
  cudaMalloc(&d2, rows * pitch);
  cudaEventRecord(a, s);
  cudaStreamWaitEvent(s2, a, 0);
  for (size_t c = 0; c < 8; ++c) {
    cudaMemcpy2DAsync(d + c * 1024 * rows, 1024, h + c * 1024, pitch, 1024, rows, cudaMemcpyHostToDevice, s);
    cudaMemcpy2DAsync(h2 + c * 1024, pitch, d2 + c * 1024 * rows, 1024, 1024, rows, cudaMemcpyDeviceToHost, s2);
  }
  cudaEventRecord(b, s2);
  cudaStreamWaitEvent(s, b, 0);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("duplex 1 KB slices: %.1f GB/s each way\n", rows * pitch / ms / 1e6);
  return 0;
}
