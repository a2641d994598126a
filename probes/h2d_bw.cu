// H2D / D2H bandwidth for a 6.9 MB FP64 vector: cudaMallocHost vs cudaHostRegister'd malloc,
// one copy vs chunked over 1/2/4 streams (e2e context).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

int main() {
  const size_t bytes = 866750 * 8;
  double *hp, *d;
  cudaMallocHost(&hp, bytes);
  memset(hp, 1, bytes);
  double* hr = (double*)aligned_alloc(4096, (bytes + 4095) / 4096 * 4096);
  memset(hr, 1, bytes);
  cudaHostRegister(hr, (bytes + 4095) / 4096 * 4096, cudaHostRegisterDefault);
  cudaMalloc(&d, bytes);
  cudaStream_t st[4];
  for (int i = 0; i < 4; ++i) cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[2] = {"mallochost", "registered"};
  double* hs[2] = {hp, hr};
  for (int which = 0; which < 2; ++which)
    for (int dir = 0; dir < 2; ++dir)
      for (int ns : {1, 2, 4}) {
        for (int rep = 0; rep < 2; ++rep) {
          cudaDeviceSynchronize();
          cudaEventRecord(a, st[0]);
          for (int it = 0; it < 10; ++it) {
            for (int i = 1; i < ns; ++i) cudaStreamWaitEvent(st[i], a, 0);
            const size_t chunk = (bytes / ns + 15) / 16 * 16;
            for (int i = 0; i < ns; ++i) {
              size_t off = i * chunk, len = off >= bytes ? 0 : (off + chunk > bytes ? bytes - off : chunk);
              if (!len) continue;
              if (dir == 0) cudaMemcpyAsync((char*)d + off, (char*)hs[which] + off, len, cudaMemcpyHostToDevice, st[i]);
              else cudaMemcpyAsync((char*)hs[which] + off, (char*)d + off, len, cudaMemcpyDeviceToHost, st[i]);
            }
          }
          cudaDeviceSynchronize();
          cudaEventRecord(b, st[0]);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (rep == 1)
            printf("{\"host\": \"%s\", \"dir\": \"%s\", \"streams\": %d, \"us\": %.1f, \"GBs\": %.1f}\n", names[which],
                   dir == 0 ? "h2d" : "d2h", ns, ms * 1e3 / 10, bytes / (ms / 10 * 1e-3) / 1e9);
        }
      }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
