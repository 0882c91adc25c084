// Throughput of cudaMemcpy2DAsync for the e2e chunk shapes (rows x chunk columns
// out of a [rows][S] pinned host array) vs contiguous copies.
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t rows = 100000, S = 65536;
  float ms;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  long long* h;
  cudaHostAlloc(&h, rows * S * 8, cudaHostAllocDefault);
  for (size_t w : {3584, 8192, 16384, 32768}) {
    long long* d;
    cudaMalloc(&d, rows * w * 8);
    cudaEventRecord(a);
    cudaMemcpy2DAsync(h, S * 8, d, w * 8, w * 8, rows, cudaMemcpyDeviceToHost);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double gb = rows * w * 8 / 1e9;
    printf("D2H 2D width %zu cols (%zu KB rows): %.1f GB/s\n", w, w * 8 / 1024, gb / (ms / 1e3));
    cudaEventRecord(a);
    cudaMemcpy2DAsync(d, w * 8, h, S * 8, w * 8, rows, cudaMemcpyHostToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("H2D 2D width %zu cols: %.1f GB/s\n", w, gb / (ms / 1e3));
    cudaFree(d);
  }
  return 0;
}
