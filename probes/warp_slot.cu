// Where do the warps of one-warp CTAs land? K3t runs three 1-warp CTAs per SM (shared memory bound);
// if their warps shared a sub-partition (SMSP) they would share its FP64 pipe. Each CTA records
// %smid / %warpid and times a 4-chain DFMA loop; k CTAs per SM are forced by the dynamic shared
// memory size. Compare the loop time with 1, 2, 3, 4 CTAs per SM (same time = separate SMSPs).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probes/warp_slot probes/warp_slot.cu
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__global__ void k(double* out, int* sm, int* wid, long long* cyc, int iters, double a, double b) {
  extern __shared__ double sh[];
  double v[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) v[c] = threadIdx.x + c;
  unsigned s, w;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(w));
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = fma(v[c], a, b);
  }
  const long long t1 = clock64();
  sh[threadIdx.x] = v[0] + v[1] + v[2] + v[3];
  out[blockIdx.x * 32 + threadIdx.x] = sh[threadIdx.x];
  if (threadIdx.x == 0) {
    sm[blockIdx.x] = s;
    wid[blockIdx.x] = w;
    cyc[blockIdx.x] = t1 - t0;
  }
}

int main() {
  for (int per = 1; per <= 4; ++per) {
    const int nb = 148 * per, iters = 20000;
    const int smem = per == 1 ? 200 * 1024 : per == 2 ? 100 * 1024 : per == 3 ? 58 * 1024 : 50 * 1024;
    double* out; int *sm, *wid; long long* cyc;
    cudaMalloc(&out, nb * 32 * 8); cudaMalloc(&sm, nb * 4); cudaMalloc(&wid, nb * 4); cudaMalloc(&cyc, nb * 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<nb, 32, smem>>>(out, sm, wid, cyc, iters, 0.999999, 1e-9);
    k<<<nb, 32, smem>>>(out, sm, wid, cyc, iters, 0.999999, 1e-9);
    std::vector<int> hs(nb), hw(nb); std::vector<long long> hc(nb);
    cudaMemcpy(hs.data(), sm, nb * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hw.data(), wid, nb * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hc.data(), cyc, nb * 8, cudaMemcpyDeviceToHost);
    double mean = 0; long long mx = 0;
    for (int i = 0; i < nb; ++i) { mean += hc[i]; if (hc[i] > mx) mx = hc[i]; }
    printf("%d CTAs/SM: mean %.2f max %.2f cycles per 4-DFMA step;", per, mean / nb / (iters * 8.0), mx / (iters * 8.0));
    printf(" sm 0's CTAs:");
    for (int i = 0; i < nb; ++i) if (hs[i] == hs[0]) printf(" (blk %d warpid %d)", i, hw[i]);
    printf("\n");
    cudaFree(out); cudaFree(sm); cudaFree(wid); cudaFree(cyc);
  }
  return 0;
}
