// Dependent-issue latency of DFMA / DMUL / DADD on one warp (clock64 around a chain of N
// dependent instructions), with 1..8 independent chains per thread and 1..16 warps per SM:
// the number K3's banded recurrences are bound by (one dependent DFMA per fiber step).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probes/dfma_lat probes/dfma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void chain(double* out, long long* cyc, int iters, double a, double b) {
  double v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = threadIdx.x + c;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int c = 0; c < CH; ++c) v[c] = fma(v[c], a, b);
    }
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int CH>
void run(int warps, int lanes_note) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 8);
  cudaMalloc(&cyc, 8);
  const int iters = 2000;
  chain<CH><<<148, warps * 32>>>(out, cyc, iters, 0.999999, 1e-9);
  chain<CH><<<148, warps * 32>>>(out, cyc, iters, 0.999999, 1e-9);
  long long h = 0;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("chains/thread %d warps/SM %2d: %.2f cycles per dependent DFMA step (%.2f cycles per DFMA warp-instr per SM)\n",
         CH, warps, (double)h / (iters * 8.0), (double)h / (iters * 8.0 * CH * warps));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {1, 2, 4, 8, 16}) {
    run<1>(w, 0);
    run<2>(w, 0);
    run<4>(w, 0);
    run<8>(w, 0);
  }
  return 0;
}
