// Do concurrent H2D and D2H copies (two streams, pinned host buffers) overlap on this box?
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t bytes = 866750 * 8;
  double *h1, *h2, *d1, *d2;
  cudaMallocHost(&h1, bytes);
  cudaMallocHost(&h2, bytes);
  cudaMalloc(&d1, bytes);
  cudaMalloc(&d2, bytes);
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, a);
      cudaStreamWaitEvent(b, e0, 0);
      for (int i = 0; i < 10; ++i) {
        if (mode != 1) cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, a);
        if (mode != 0) cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, mode == 2 ? b : a);
      }
      cudaEvent_t eb;
      cudaEventCreate(&eb);
      cudaEventRecord(eb, b);
      cudaStreamWaitEvent(a, eb, 0);
      cudaEventRecord(e1, a);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2)
        printf("{\"mode\": \"%s\", \"us_per_iter\": %.1f}\n", mode == 0 ? "h2d only" : mode == 1 ? "d2h only" : "h2d||d2h", ms * 100);
    }
  }
  return 0;
}
