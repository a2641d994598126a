// Probe: K1t's stage inner loop (non-KMAJ FWD: swizzled A tiles, fold, fragment-native B via
// LDS.128, 4 k4 steps per stage) on static shared memory, no TMA, no epilogue -- isolates the
// DMMA issue efficiency of the loop from the pipeline. Prints TFLOP/s per variant.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ double lds64(unsigned a) { double v; asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a)); return v; }
__device__ __forceinline__ void lds128(unsigned a, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}

template <int FOLD, int B128, int SYNC, int STAGES_SM, int EPI = 0, int MBW = 0, int RND = 0>
__global__ void __launch_bounds__(256, 2) k(double* out, int iters) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const unsigned sbase = (static_cast<unsigned>(__cvta_generic_to_shared(sm)) + 1023u) & ~1023u;
  for (int i = threadIdx.x; i < 37 * 1024 * STAGES_SM / 8; i += blockDim.x)
    reinterpret_cast<double*>(sm)[i] = RND ? (double)((i * 2654435761u) % 1000003u) / 1000003.0 - 0.5 : 1e-3 * (i % 7);
  const unsigned bar = sbase + 37888 * STAGES_SM;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wm = warp & 3, role = warp >> 2;
  const int fr = lane >> 2, fc = lane & 3;
  unsigned a0[2][2], a1[2][2];
  for (int ti = 0; ti < 2; ++ti) {
    const int plo = 8 * ti + fr;
    for (int jj = 0; jj < 2; ++jj) {
      const int kk = 2 * fc + jj, km = 15 - kk;
      a0[ti][jj] = (kk + 16 * wm) * 128 + ((((plo >> 1) ^ (kk & 7)) << 4) | ((plo & 1) << 3));
      a1[ti][jj] = (km + 16 * wm) * 128 + ((((plo >> 1) ^ (km & 7)) << 4) | ((plo & 1) << 3));
    }
  }
  const double sgn = role ? -1.0 : 1.0;
  double acc[2][9][2];
  for (int i = 0; i < 2; ++i) for (int u = 0; u < 9; ++u) acc[i][u][0] = acc[i][u][1] = 0.0;
  int stage = 0;
  for (int it = 0; it < iters; ++it) {
    if (MBW) asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(bar) : "memory");
    const unsigned A0 = sbase + stage * 37888, A1 = A0 + 8192, B = A1 + 8192 + role * 10240;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double a[2];
#pragma unroll
      for (int ti = 0; ti < 2; ++ti) {
        const unsigned o0 = a0[ti][j & 1] + (j >> 1) * 1024;
        if (FOLD) {
          const unsigned o1 = a1[ti][j & 1] - (j >> 1) * 1024;
          a[ti] = fma(sgn, lds64(A1 + o1), lds64(A0 + o0));
        } else {
          a[ti] = lds64(A0 + o0);
        }
      }
      double b[10];
      if (B128) {
#pragma unroll
        for (int tp = 0; tp < 5; ++tp) lds128(B + ((j * 5 + tp) * 32 + lane) * 16, b[2 * tp], b[2 * tp + 1]);
      } else {
#pragma unroll
        for (int u = 0; u < 9; ++u) b[u] = lds64(B + ((j * 9 + u) * 32 + lane) * 8);
      }
#pragma unroll
      for (int ti = 0; ti < 2; ++ti)
#pragma unroll
        for (int u = 0; u < 9; ++u) dmma(acc[ti][u], a[ti], b[u]);
    }
    if (SYNC) asm volatile("bar.sync 15, 256;" ::: "memory");
    if (++stage == STAGES_SM) stage = 0;
    if (EPI && it % 17 == 16) {  // a tile every 17 stages: store the accumulators, restart
      double* o = out + 1 + ((size_t)(blockIdx.x * 8 + warp) * 32 + lane) * 36 + (size_t)(it / 17 % 4) * 148 * 2 * 8 * 32 * 36;
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int u = 0; u < 9; ++u) {
          if (EPI == 1) { o[(i * 9 + u) * 2] = acc[i][u][0]; o[(i * 9 + u) * 2 + 1] = acc[i][u][1]; }
          acc[i][u][0] = acc[i][u][1] = 0.0;
        }
    }
  }
  double s = 0;
  for (int i = 0; i < 2; ++i) for (int u = 0; u < 9; ++u) s += acc[i][u][0] + acc[i][u][1];
  if (s == 12345.678) out[0] = s;
}

template <int FOLD, int B128, int SYNC, int ST, int EPI = 0, int MBW = 0, int RND = 0>
void run(int ctas) {
  double* out; cudaMalloc(&out, 8 + 8ull * 4 * 148 * 2 * 8 * 32 * 36);
  const size_t smem = 1024 + 37888 * ST + 64;
  cudaFuncSetAttribute(k<FOLD, B128, SYNC, ST, EPI, MBW, RND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int iters = 4000;
  k<FOLD, B128, SYNC, ST, EPI, MBW, RND><<<148 * ctas, 256, smem>>>(out, 10);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<FOLD, B128, SYNC, ST, EPI, MBW, RND><<<148 * ctas, 256, smem>>>(out, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double flops = 512.0 * 2 * 9 * 4 * (double)iters * 8 * 148 * ctas;
  printf("{\"RND\": %d, \"MBW\": %d, \"EPI\": %d, \"FOLD\": %d, \"B128\": %d, \"SYNC\": %d, \"stages\": %d, \"ctas_per_sm\": %d, \"tflops\": %.2f, \"err\": \"%s\"}\n",
         RND, MBW, EPI, FOLD, B128, SYNC, ST, ctas, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  run<1, 1, 1, 2, 0, 0, 0>(2);
  run<1, 1, 1, 2, 0, 0, 1>(2);
  run<0, 0, 0, 2, 0, 0, 1>(2);
  return 0;
}
