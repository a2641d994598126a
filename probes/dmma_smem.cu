// Probe: achievable FP64 DMMA rate when A/B fragments are loaded from shared memory each k4 step
// (the inner loop of K1/K1s), as a function of the warp tile (MT x NT m8n8 tiles) and warps/SM.
// Diagnostic only; prints TFLOP/s per configuration.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int MT, int NT, int FOLD = 0, int SYNC = 0>
__global__ void k(double* out, int iters, int K4) {
  extern __shared__ double sm[];
  const int SA = 100, SB = 116;
  double* As = sm;                 // [K][SA]
  double* Bs = sm + 4 * K4 * SA;   // [K][SB]
  for (int i = threadIdx.x; i < 4 * K4 * (SA + SB); i += blockDim.x) sm[i] = 1e-3 * (i % 7);
  __syncthreads();
  const int lane = threadIdx.x & 31, fr = lane >> 2, fc = lane & 3;
  const int warp = threadIdx.x >> 5;
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const double sgn = (warp & 4) ? -1.0 : 1.0;
  double an[MT];
  if (FOLD == 2) {
#pragma unroll
    for (int i = 0; i < MT; ++i) an[i] = fma(sgn, As[(4 * K4 - 1 - fc) * SA + (warp & 3) * 16 + 8 * i + fr], As[fc * SA + (warp & 3) * 16 + 8 * i + fr]);
  }
  for (int it = 0; it < iters; ++it) {
    for (int k4 = 0; k4 < K4; ++k4) {
      const int kk = 4 * k4 + fc;
      double a[MT], b[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        if (FOLD == 2) a[i] = an[i];
        else a[i] = As[kk * SA + (warp & 3) * 16 + 8 * i + fr];
        if (FOLD == 1) a[i] = fma(sgn, As[(4 * K4 - 1 - kk) * SA + (warp & 3) * 16 + 8 * i + fr], a[i]);
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = Bs[kk * SB + 8 * j + fr];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j], a[i], b[j]);
      if (SYNC && (k4 & 3) == 3) __syncthreads();
      if (FOLD == 2) {
        const int kn = (4 * (k4 + 1) + fc) % (4 * K4);
#pragma unroll
        for (int i = 0; i < MT; ++i) an[i] = fma(sgn, As[(4 * K4 - 1 - kn) * SA + (warp & 3) * 16 + 8 * i + fr], As[kn * SA + (warp & 3) * 16 + 8 * i + fr]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 12345.678) out[0] = s;
}

template <int MT, int NT, int FOLD = 0, int SYNC = 0>
void run(int warps, int ctas_per_sm) {
  double* out;
  cudaMalloc(&out, 8);
  const int K4 = 17, iters = 400;
  size_t smem = sizeof(double) * 4 * K4 * (100 + 116);
  cudaFuncSetAttribute(k<MT, NT, FOLD, SYNC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int grid = 148 * ctas_per_sm;
  k<MT, NT, FOLD, SYNC><<<grid, warps * 32, smem>>>(out, 10, K4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MT, NT, FOLD, SYNC><<<grid, warps * 32, smem>>>(out, iters, K4);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double flops = 512.0 * MT * NT * K4 * (double)iters * warps * grid;
  printf("{\"SYNC\": %d, \"FOLD\": %d, \"MT\": %d, \"NT\": %d, \"warps_per_cta\": %d, \"ctas_per_sm\": %d, \"tflops\": %.2f, \"err\": \"%s\"}\n", SYNC, FOLD, MT, NT,
         warps, ctas_per_sm, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
  cudaFree(out);
}

int main() {
  run<2, 9, 0, 0>(8, 2);
  run<2, 9, 0, 1>(8, 2);
  run<2, 9, 1, 1>(8, 2);
  run<2, 9, 0, 1>(16, 1);
  run<4, 9, 0, 1>(8, 1);
  run<2, 9, 0, 0>(16, 1);
  return 0;
}
