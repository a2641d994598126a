// Probe: does FP64 ALU work (DFMA / DADD) issued next to DMMA (mma.sync f64) cost DMMA
// throughput on sm_100a, and how much per instruction? Register-resident loops, one CTA per SM.
//   mode 0: W warps, each 18 independent DMMA per iteration + F independent DFMA (same warp)
//   mode 1: W DMMA-only warps + S side warps doing F*18/... DFMA per iteration (other warps)
// Prints DMMA TFLOP/s and the side work per DMMA.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int F, int MODE, int MUFU>
__global__ void __launch_bounds__(512, 1) mix(double* out, int iters, int wdmma) {
  const int warp = threadIdx.x >> 5;
  double acc[18][2];
#pragma unroll
  for (int u = 0; u < 18; ++u) acc[u][0] = acc[u][1] = 0.0;
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  const double a = 1.0 + 1e-12 * threadIdx.x, b = 1.0 - 1e-12 * threadIdx.x;
  if (MODE == 0 || warp < wdmma) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int u = 0; u < 18; ++u) dmma(acc[u], a, b);
      if (MODE == 0) {
#pragma unroll
        for (int f = 0; f < F; ++f) {
          if (MUFU) {
            double r;
            asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[f & 7]));
            x[f & 7] = r;
          } else {
            x[f & 7] = fma(x[f & 7], 0.999999, 1e-7);
          }
        }
      }
    }
  } else {
    // side warps: F FP64 ops per "iteration" of the DMMA warps, for as long as they run
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int f = 0; f < F; ++f) {
        if (MUFU) {
          double r;
          asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[f & 7]));
          x[f & 7] = r;
        } else {
          x[f & 7] = fma(x[f & 7], 0.999999, 1e-7);
        }
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < 18; ++u) s += acc[u][0] + acc[u][1];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int F, int MODE, int MUFU>
void run(const char* name, int warps, int wdmma, double* out, int sms) {
  const int iters = 4000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mix<F, MODE, MUFU><<<sms, warps * 32>>>(out, 100, wdmma);
  cudaEventRecord(e0);
  mix<F, MODE, MUFU><<<sms, warps * 32>>>(out, iters, wdmma);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const int dw = MODE == 0 ? warps : wdmma;
  const double flops = (double)sms * dw * iters * 18 * 512.0;
  printf("%-34s warps %2d dmma-warps %2d side-ops/iter %2d: DMMA %.2f TF/s (%.3f ms)\n", name, warps, dw, F,
         flops / (ms * 1e-3) / 1e12, ms);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1 << 20);
  run<0, 0, 0>("DMMA only", 8, 8, out, sms);
  run<1, 0, 0>("same warp DFMA", 8, 8, out, sms);
  run<2, 0, 0>("same warp DFMA", 8, 8, out, sms);
  run<4, 0, 0>("same warp DFMA", 8, 8, out, sms);
  run<8, 0, 0>("same warp DFMA", 8, 8, out, sms);
  run<2, 0, 1>("same warp MUFU.RCP64H", 8, 8, out, sms);
  run<8, 0, 1>("same warp MUFU.RCP64H", 8, 8, out, sms);
  run<0, 1, 0>("other warps DFMA (0)", 12, 8, out, sms);
  run<2, 1, 0>("other warps DFMA", 12, 8, out, sms);
  run<4, 1, 0>("other warps DFMA", 12, 8, out, sms);
  run<8, 1, 0>("other warps DFMA", 12, 8, out, sms);
  run<16, 1, 0>("other warps DFMA", 12, 8, out, sms);
  run<4, 1, 1>("other warps MUFU.RCP64H", 12, 8, out, sms);
  run<16, 1, 1>("other warps MUFU.RCP64H", 12, 8, out, sms);
  return 0;
}
