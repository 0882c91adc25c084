// Throughput of cudaMemcpy2DAsync for the e2e chunk shapes (rows x chunk columns
// out of a [rows][S] pinned host array) vs contiguous copies, alone and duplex.
#include <cstdio>
#include <cuda_runtime.h>
static float tm(cudaEvent_t a, cudaEvent_t b) {
  float ms;
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  return ms / 1e3f;
}
int main() {
  const size_t rows = 100000, S = 65536;
  cudaEvent_t a, b, c;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventCreate(&c);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  long long* h;
  int* hi;
  cudaHostAlloc(&h, rows * S * 8, cudaHostAllocDefault);
  cudaHostAlloc(&hi, rows * S * 4, cudaHostAllocDefault);
  for (size_t w : {4096, 14336, 32768}) {
    long long* d;
    int* di;
    cudaMalloc(&d, rows * w * 8);
    cudaMalloc(&di, rows * w * 4);
    double gb8 = rows * w * 8 / 1e9, gb4 = rows * w * 4 / 1e9;
    cudaEventRecord(a, s1);
    cudaMemcpy2DAsync(h, S * 8, d, w * 8, w * 8, rows, cudaMemcpyDeviceToHost, s1);
    cudaEventRecord(b, s1);
    printf("w=%zu D2H 2D int64: %.1f GB/s\n", w, gb8 / tm(a, b));
    cudaEventRecord(a, s1);
    cudaMemcpyAsync(h, d, rows * w * 8, cudaMemcpyDeviceToHost, s1);
    cudaEventRecord(b, s1);
    printf("w=%zu D2H contiguous: %.1f GB/s\n", w, gb8 / tm(a, b));
    cudaEventRecord(a, s1);
    cudaMemcpy2DAsync(di, w * 4, hi, S * 4, w * 4, rows, cudaMemcpyHostToDevice, s1);
    cudaEventRecord(b, s1);
    printf("w=%zu H2D 2D int32: %.1f GB/s\n", w, gb4 / tm(a, b));
    // duplex: D2H int64 on s1, H2D int32 on s2
    cudaDeviceSynchronize();
    cudaEventRecord(a, s1);
    cudaStreamWaitEvent(s2, a, 0);
    cudaMemcpy2DAsync(h, S * 8, d, w * 8, w * 8, rows, cudaMemcpyDeviceToHost, s1);
    cudaMemcpy2DAsync(di, w * 4, hi, S * 4, w * 4, rows, cudaMemcpyHostToDevice, s2);
    cudaEventRecord(b, s1);
    cudaEventRecord(c, s2);
    float t1 = tm(a, b), t2 = tm(a, c);
    printf("w=%zu duplex: D2H %.1f GB/s (%.3f s), H2D %.1f GB/s (%.3f s)\n", w, gb8 / t1, t1,
           gb4 / t2, t2);
    cudaFree(d);
    cudaFree(di);
  }
  return 0;
}
