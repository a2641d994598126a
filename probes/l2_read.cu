// Probe: time to read an L2-resident buffer of config-2 size (6.6 MB) into registers with all SMs
// (16 warps/SM, 8-byte and 16-byte loads), i.e. the floor of a pass's panel-load phase.
#include <cstdio>
#include <cuda_runtime.h>

template <int VEC>
__global__ void rd(const double* __restrict__ x, long long n, double* out) {
  double s = 0;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  if (VEC == 2) {
    const double2* x2 = reinterpret_cast<const double2*>(x);
    for (long long i = tid; i < n / 2; i += nt) { double2 v = __ldg(x2 + i); s += v.x + v.y; }
  } else {
    for (long long i = tid; i < n; i += nt) s += __ldg(x + i);
  }
  if (s == 1234.5) out[0] = s;
}

__global__ void wr(double* __restrict__ x, long long n) {
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n; i += nt) x[i] = (double)i;
}

int main() {
  const long long n = 866750;  // config 2 doubles
  double *x, *o;
  cudaMalloc(&x, n * 8 * 4);
  cudaMalloc(&o, 8);
  cudaMemset(x, 0, n * 8 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    for (int vec : {1, 2}) {
      rd<1><<<148, 512>>>(x, n, o);  // warm into L2
      cudaDeviceSynchronize();
      cudaEventRecord(a);
      for (int it = 0; it < 20; ++it) {
        if (vec == 1) rd<1><<<148, 512>>>(x, n, o);
        else rd<2><<<148, 512>>>(x, n, o);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("{\"read_vec\": %d, \"us_per_pass\": %.2f, \"TBps\": %.2f}\n", vec, ms * 1e3 / 20, n * 8 / (ms / 20 * 1e-3) / 1e12);
    }
    cudaEventRecord(a);
    for (int it = 0; it < 20; ++it) wr<<<148, 512>>>(x, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"write\": 1, \"us_per_pass\": %.2f, \"TBps\": %.2f}\n", ms * 1e3 / 20, n * 8 / (ms / 20 * 1e-3) / 1e12);
    // empty kernel baseline
    cudaEventRecord(a);
    for (int it = 0; it < 20; ++it) rd<1><<<148, 512>>>(x, 0, o);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"empty_us\": %.2f}\n", ms * 1e3 / 20);
  }
  return 0;
}
