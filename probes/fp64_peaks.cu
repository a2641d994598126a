// FP64 ceiling probes for B200 (sm_100a): DMMA (mma.sync f64) and DFMA register-resident
// loops over all SMs, cuBLAS DGEMM at square and tall-skinny FD shapes, and an HBM copy.
// Output: one JSON object on stdout. These numbers are the roofline denominators the bench
// reports against (MEASURED_PEAKS.json carries no FP64 entry).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cublas_v2.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

static float time_ms(cudaEvent_t e0, cudaEvent_t e1) { float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); return ms; }

int main() {
  int dev = 0, sms = 0, l2 = 0, clk = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  printf("{\"sms\": %d, \"l2_bytes\": %d, \"clock_khz\": %d", sms, l2, clk);

  // DMMA: flops per mma = 2*8*8*4 = 512 per warp.
  const int NACC = 8;
  for (int warps : {4, 8, 16, 32}) {
    int iters = 20000;
    int blocks = sms * 1;
    dmma_loop<NACC><<<blocks, warps * 32>>>(out, 100);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0));
      dmma_loop<NACC><<<blocks, warps * 32>>>(out, iters);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      best = fminf(best, time_ms(e0, e1));
    }
    double flops = 512.0 * NACC * (double)iters * warps * blocks;
    printf(", \"dmma_tflops_w%d\": %.3f", warps, flops / (best * 1e-3) / 1e12);
  }
  for (int warps : {8, 16, 32}) {
    int iters = 20000;
    int blocks = sms;
    dfma_loop<16><<<blocks, warps * 32>>>(out, 100);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0));
      dfma_loop<16><<<blocks, warps * 32>>>(out, iters);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      best = fminf(best, time_ms(e0, e1));
    }
    double flops = 2.0 * 16 * (double)iters * warps * 32 * blocks;
    printf(", \"dfma_tflops_w%d\": %.3f", warps, flops / (best * 1e-3) / 1e12);
  }

  // HBM copy 2 GiB read + 2 GiB write.
  {
    size_t n = (size_t)1 << 27;  // double2 elements = 2 GiB
    double2 *a, *b;
    CK(cudaMalloc(&a, n * sizeof(double2))); CK(cudaMalloc(&b, n * sizeof(double2)));
    CK(cudaMemset(a, 0, n * sizeof(double2)));
    copy_kernel<<<sms * 8, 512>>>(a, b, n);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0)); copy_kernel<<<sms * 8, 512>>>(a, b, n); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      best = fminf(best, time_ms(e0, e1));
    }
    printf(", \"hbm_copy_gbs\": %.1f", 2.0 * n * sizeof(double2) / (best * 1e-3) / 1e9);
    CK(cudaFree(a)); CK(cudaFree(b));
  }

  // cuBLAS DGEMM.
  cublasHandle_t h; cublasCreate(&h);
  auto dgemm = [&](int M, int N, int K, const char* tag) {
    double *A, *B, *C;
    CK(cudaMalloc(&A, (size_t)M * K * 8)); CK(cudaMalloc(&B, (size_t)K * N * 8)); CK(cudaMalloc(&C, (size_t)M * N * 8));
    CK(cudaMemset(A, 0, (size_t)M * K * 8)); CK(cudaMemset(B, 0, (size_t)K * N * 8));
    double al = 1.0, be = 0.0;
    cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, M, N, K, &al, A, M, B, K, &be, C, M);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0));
      cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, M, N, K, &al, A, M, B, K, &be, C, M);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      best = fminf(best, time_ms(e0, e1));
    }
    printf(", \"cublas_dgemm_%s_tflops\": %.3f", tag, 2.0 * M * N * (double)K / (best * 1e-3) / 1e12);
    CK(cudaFree(A)); CK(cudaFree(B)); CK(cudaFree(C));
  };
  dgemm(8192, 8192, 8192, "8192cube");
  dgemm(1 << 22, 65, 65, "M4M_n65");
  dgemm(1 << 22, 264, 259, "M4M_n259");
  dgemm(1 << 22, 516, 516, "M4M_n516");
  dgemm(67081, 259, 259, "M67081_n259");
  dgemm(4225, 65, 65, "M4225_n65");
  cublasDestroy(h);
  printf("}\n");
  return 0;
}
