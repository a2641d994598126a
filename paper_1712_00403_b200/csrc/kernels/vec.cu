// Vector kernels of the GPU-resident Krylov driver: dot products with a
// deterministic two-level reduction (fixed grid, fixed order) and fused linear combinations.
// HBM-bound streaming (16-24 B per element).
#include "../fdp_internal.h"

namespace fdp {
namespace {

constexpr int kDotBlocks = 296;  // 2 x 148 SMs, fixed so the reduction order is reproducible
constexpr int kDotThreads = 256;

__global__ void dot_partial_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                   long long n, double* __restrict__ partial) {
  __shared__ double sh[kDotThreads / 32];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)kDotThreads + threadIdx.x; i < n;
       i += (long long)gridDim.x * kDotThreads)
    s = fma(x[i], y[i], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < kDotThreads / 32 ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) partial[blockIdx.x] = v;
  }
}

__global__ void dot_final_kernel(const double* __restrict__ partial, double* __restrict__ out) {
  __shared__ double sh[kDotThreads / 32];
  double v = 0.0;
  for (int i = threadIdx.x; i < kDotBlocks; i += kDotThreads) v += partial[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double w = threadIdx.x < kDotThreads / 32 ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w += __shfl_down_sync(0xffffffffu, w, o);
    if (threadIdx.x == 0) out[0] = w;
  }
}

__global__ void lincomb_kernel(double a, const double* x, double b, const double* y, double c,
                               const double* z, double* out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double v = a * x[i];
    if (y) v = fma(b, y[i], v);
    if (z) v = fma(c, z[i], v);
    out[i] = v;
  }
}

__global__ void partsum_kernel(const __grid_constant__ PartSum ps, double* __restrict__ y,
                               double beta, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double v = beta != 0.0 ? beta * y[i] : 0.0;
    for (int j = 0; j < ps.nparts; ++j) v = fma(ps.coef[j], ps.parts[j][i], v);
    y[i] = v;
  }
}

// h[j] = V_j . w for j < m (V_j = V + j ldv): partial sums of 8 vectors per block row, then a
// fixed-order reduction per vector (deterministic)
constexpr int kMdVec = 8;
__global__ void multidot_partial_kernel(const double* __restrict__ V, long long ldv, int m,
                                        const double* __restrict__ w, long long n,
                                        double* __restrict__ partial) {
  __shared__ double sh[kDotThreads / 32][kMdVec];
  const int j0 = blockIdx.y * kMdVec;
  const int nv = min(kMdVec, m - j0);
  double s[kMdVec];
#pragma unroll
  for (int j = 0; j < kMdVec; ++j) s[j] = 0.0;
  for (long long i = blockIdx.x * (long long)kDotThreads + threadIdx.x; i < n;
       i += (long long)gridDim.x * kDotThreads) {
    const double wi = w[i];
#pragma unroll
    for (int j = 0; j < kMdVec; ++j)
      if (j < nv) s[j] = fma(V[(j0 + j) * ldv + i], wi, s[j]);
  }
#pragma unroll
  for (int j = 0; j < kMdVec; ++j) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s[j] += __shfl_down_sync(0xffffffffu, s[j], o);
  }
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int j = 0; j < kMdVec; ++j) sh[threadIdx.x >> 5][j] = s[j];
  __syncthreads();
  if (threadIdx.x < nv) {
    double t = 0.0;
    for (int q = 0; q < kDotThreads / 32; ++q) t += sh[q][threadIdx.x];
    partial[(long long)(j0 + threadIdx.x) * kDotBlocks + blockIdx.x] = t;
  }
}

__global__ void multidot_final_kernel(const double* __restrict__ partial, double* __restrict__ h) {
  __shared__ double sh[kDotThreads / 32];
  const double* p = partial + (long long)blockIdx.x * kDotBlocks;
  double v = 0.0;
  for (int i = threadIdx.x; i < kDotBlocks; i += kDotThreads) v += p[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < kDotThreads / 32; ++q) t += sh[q];
    h[blockIdx.x] = t;
  }
}

// w = beta w + alpha sum_j h[j] V_j (fixed order in j per element)
__global__ void gemv_kernel(const double* __restrict__ V, long long ldv, int m,
                            const double* __restrict__ h, double alpha, double* __restrict__ w,
                            double beta, long long n) {
  extern __shared__ double hs[];
  for (int j = threadIdx.x; j < m; j += blockDim.x) hs[j] = h[j];
  __syncthreads();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < m; ++j) s = fma(hs[j], V[j * ldv + i], s);
    w[i] = beta != 0.0 ? fma(alpha, s, beta * w[i]) : alpha * s;
  }
}

}  // namespace

size_t multidot_scratch_elems(int m) { return (size_t)m * kDotBlocks; }

cudaError_t launch_multidot(const double* V, long long ldv, int m, const double* w, long long n,
                            double* h, double* scratch, cudaStream_t s) {
  if (m <= 0) return cudaSuccess;
  dim3 grid(kDotBlocks, (m + kMdVec - 1) / kMdVec);
  multidot_partial_kernel<<<grid, kDotThreads, 0, s>>>(V, ldv, m, w, n, scratch);
  multidot_final_kernel<<<m, kDotThreads, 0, s>>>(scratch, h);
  return cudaGetLastError();
}

cudaError_t launch_gemv(const double* V, long long ldv, int m, const double* h, double alpha,
                        double* w, double beta, long long n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 8);
  gemv_kernel<<<blocks, 256, (size_t)std::max(m, 1) * sizeof(double), s>>>(V, ldv, m, h, alpha, w, beta, n);
  return cudaGetLastError();
}

cudaError_t launch_partsum(const PartSum& ps, double* y, double beta, long long n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 8);
  partsum_kernel<<<blocks, 256, 0, s>>>(ps, y, beta, n);
  return cudaGetLastError();
}

cudaError_t launch_dot(const double* x, const double* y, long long n, double* result,
                       double* scratch, cudaStream_t s) {
  dot_partial_kernel<<<kDotBlocks, kDotThreads, 0, s>>>(x, y, n, scratch);
  dot_final_kernel<<<1, kDotThreads, 0, s>>>(scratch, result);
  return cudaGetLastError();
}

int dot_scratch_doubles() { return kDotBlocks; }

cudaError_t launch_lincomb(double a, const double* x, double b, const double* y, double c,
                           const double* z, double* out, long long n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 8);
  lincomb_kernel<<<blocks, 256, 0, s>>>(a, x, b, y, c, z, out, n);
  return cudaGetLastError();
}

}  // namespace fdp
