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

// out = k[0] x + k[1] y + k[2] z with the coefficients read from device memory; a term whose
// coefficient is exactly 0 is skipped (its vector is not read), as is a NULL vector
__global__ void lincomb_dev_kernel(const double* __restrict__ k, const double* x, const double* y,
                                   const double* z, double* out, long long n) {
  const double a = k[0], b = y ? k[1] : 0.0, c = z ? k[2] : 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double v = a != 0.0 ? a * x[i] : 0.0;
    if (b != 0.0) v = fma(b, y[i], v);
    if (c != 0.0) v = fma(c, z[i], v);
    out[i] = v;
  }
}

// Paige-Saunders MINRES scalar recurrence on the device (one thread); state layout in fdp.h
__global__ void minres_scalars_kernel(int phase, double* __restrict__ s, double* __restrict__ hist,
                                      int hist_cap) {
  enum { BETA1, BETA, OLDB, DBAR, EPSLN, PHIBAR, CS, SN, ALFA, DOT, ITN, DONE, ITN_DONE, TOL,
         ERR, KV = 16, KY1 = 19, KY2 = 22, KW = 25, KX = 28 };
  if (phase == 0) {  // init: DOT = r1 . P r1
    const double d = s[DOT];
    if (d < 0.0) s[ERR] = 1.0;
    const double b1 = sqrt(fmax(d, 0.0));
    s[BETA1] = b1;
    s[BETA] = b1;
    s[PHIBAR] = b1;
    s[OLDB] = s[DBAR] = s[EPSLN] = 0.0;
    s[CS] = -1.0;
    s[SN] = 0.0;
    s[ITN] = 0.0;
    s[DONE] = b1 == 0.0 ? 1.0 : 0.0;
    s[ITN_DONE] = 0.0;
    return;
  }
  if (phase == 1) {  // iteration start: v = y / beta, y -= (beta / oldb) r1 (itn >= 2)
    const double itn = s[ITN] + 1.0;
    s[ITN] = itn;
    const bool live = s[DONE] == 0.0;
    s[KV] = live ? 1.0 / s[BETA] : 0.0;
    s[KV + 1] = s[KV + 2] = 0.0;
    s[KY1] = 1.0;
    s[KY1 + 1] = (live && itn >= 2.0) ? -s[BETA] / s[OLDB] : 0.0;
    s[KY1 + 2] = 0.0;
    return;
  }
  if (phase == 2) {  // after alfa = v . y: y -= (alfa / beta) r2
    const bool live = s[DONE] == 0.0;
    s[KY2] = 1.0;
    s[KY2 + 1] = live ? -s[ALFA] / s[BETA] : 0.0;
    s[KY2 + 2] = 0.0;
    return;
  }
  // phase 3: after DOT = r2 . P r2 -- the plane rotation, w and x coefficients, stopping test
  const bool live = s[DONE] == 0.0;
  if (!live) {
    s[KW] = s[KW + 1] = s[KW + 2] = 0.0;
    s[KX] = 1.0;
    s[KX + 1] = s[KX + 2] = 0.0;
    return;
  }
  const double d = s[DOT];
  if (d < 0.0) s[ERR] = 1.0;
  const double alfa = s[ALFA];
  const double oldb = s[BETA];
  const double beta = sqrt(fmax(d, 0.0));
  const double cs = s[CS], sn = s[SN], dbar = s[DBAR];
  const double oldeps = s[EPSLN];
  const double delta = cs * dbar + sn * alfa;
  const double gbar = sn * dbar - cs * alfa;
  const double epsln = sn * beta;
  const double dbar2 = -cs * beta;
  const double gamma = fmax(hypot(gbar, beta), 2.220446049250313e-16);
  const double cs2 = gbar / gamma, sn2 = beta / gamma;
  const double phi = cs2 * s[PHIBAR];
  const double phibar = sn2 * s[PHIBAR];
  s[OLDB] = oldb;
  s[BETA] = beta;
  s[EPSLN] = epsln;
  s[DBAR] = dbar2;
  s[CS] = cs2;
  s[SN] = sn2;
  s[PHIBAR] = phibar;
  s[KW] = 1.0 / gamma;
  s[KW + 1] = -oldeps / gamma;
  s[KW + 2] = -delta / gamma;
  s[KX] = 1.0;
  s[KX + 1] = phi;
  s[KX + 2] = 0.0;
  const int itn = (int)s[ITN];
  const double rel = phibar / s[BETA1];
  if (hist && itn < hist_cap) hist[itn] = rel;
  if (rel <= s[TOL]) {
    s[DONE] = 1.0;
    s[ITN_DONE] = itn;
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

// ---- device-indexed Arnoldi helpers (GPU-resident GMRES): counts and indices read from device
// memory so that whole iterations can be captured in one CUDA graph ----
__global__ void copy_indexed_kernel(const double* __restrict__ V, long long ldv, const int* idx,
                                    double* __restrict__ out, long long n) {
  const long long base = (long long)(*idx) * ldv;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = V[base + i];
}

__global__ void store_indexed_kernel(double* __restrict__ V, long long ldv, const int* idx,
                                     const double* __restrict__ w, const double* coef, long long n) {
  const double c = *coef;
  if (c == 0.0) return;
  const long long base = (long long)(*idx) * ldv;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    V[base + i] = c * w[i];
}

__global__ void multidot_partial_dev_kernel(const double* __restrict__ V, long long ldv,
                                            const int* m_ptr, int m_max,
                                            const double* __restrict__ w, long long n,
                                            double* __restrict__ partial) {
  const int m = min(*m_ptr, m_max);
  const int j0 = blockIdx.y * kMdVec;
  if (j0 >= m) return;
  __shared__ double sh[kDotThreads / 32][kMdVec];
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

__global__ void multidot_final_dev_kernel(const double* __restrict__ partial, const int* m_ptr,
                                          int m_max, double* __restrict__ h) {
  if ((int)blockIdx.x >= min(*m_ptr, m_max)) return;
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

__global__ void gemv_dev_kernel(const double* __restrict__ V, long long ldv, const int* m_ptr,
                                int m_max, const double* __restrict__ h, double alpha,
                                double* __restrict__ w, double beta, long long n) {
  extern __shared__ double hs[];
  const int m = min(*m_ptr, m_max);
  for (int j = threadIdx.x; j < m; j += blockDim.x) hs[j] = h[j];
  __syncthreads();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < m; ++j) s = fma(hs[j], V[j * ldv + i], s);
    w[i] = beta != 0.0 ? fma(alpha, s, beta * w[i]) : alpha * s;
  }
}

// GMRES least-squares bookkeeping on the device (one thread), Saad & Schultz with Givens
// rotations; layouts in fdp.h.
__global__ void gmres_scalars_kernel(int phase, int* __restrict__ is, double* __restrict__ ds,
                                     double* __restrict__ H, int ldh, const double* __restrict__ h1,
                                     const double* __restrict__ h2, double* __restrict__ hist,
                                     int m_max) {
  enum { J, DONE, KFIN, MCNT, STORE };
  enum { BETA, TOL, COEF, NRM2, DOT };
  double* cs = ds + 8;
  double* sn = cs + m_max + 1;
  double* g = sn + m_max + 1;
  if (phase == 0) {  // init from DOT = ||P^{-1} b||^2
    const double beta = sqrt(fmax(ds[DOT], 0.0));
    ds[BETA] = beta;
    for (int i = 0; i <= m_max; ++i) g[i] = 0.0;
    g[0] = beta;
    is[J] = 0;
    is[DONE] = beta == 0.0 ? 1 : 0;
    is[KFIN] = 0;
    is[MCNT] = 1;
    is[STORE] = 0;
    ds[COEF] = beta == 0.0 ? 0.0 : 1.0 / beta;
    if (hist) hist[0] = 1.0;
    return;
  }
  if (is[DONE]) {
    ds[COEF] = 0.0;
    return;
  }
  const int j = is[J];
  double* col = H + (long long)j * ldh;
  for (int i = 0; i <= j; ++i) col[i] = h1[i] + h2[i];
  const double hn = sqrt(fmax(ds[NRM2], 0.0));
  col[j + 1] = hn;
  ds[COEF] = hn != 0.0 ? 1.0 / hn : 0.0;
  is[STORE] = j + 1;
  for (int i = 0; i < j; ++i) {
    const double t = cs[i] * col[i] + sn[i] * col[i + 1];
    col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1];
    col[i] = t;
  }
  const double den = hypot(col[j], col[j + 1]);
  cs[j] = col[j] / den;
  sn[j] = col[j + 1] / den;
  col[j] = den;
  col[j + 1] = 0.0;
  g[j + 1] = -sn[j] * g[j];
  g[j] = cs[j] * g[j];
  const double res = fabs(g[j + 1]) / ds[BETA];
  if (hist) hist[j + 1] = res;
  is[J] = j + 1;
  is[MCNT] = j + 2;
  if (res <= ds[TOL] || den == 0.0 || j + 1 >= m_max) {
    is[DONE] = 1;
    is[KFIN] = j + 1;
  }
}

}  // namespace

cudaError_t launch_copy_indexed(const double* V, long long ldv, const int* idx, double* out,
                                long long n, cudaStream_t s) {
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 8);
  copy_indexed_kernel<<<std::max(blocks, 1), 256, 0, s>>>(V, ldv, idx, out, n);
  return cudaGetLastError();
}
cudaError_t launch_store_indexed(double* V, long long ldv, const int* idx, const double* w,
                                 const double* coef, long long n, cudaStream_t s) {
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 8);
  store_indexed_kernel<<<std::max(blocks, 1), 256, 0, s>>>(V, ldv, idx, w, coef, n);
  return cudaGetLastError();
}
cudaError_t launch_multidot_dev(const double* V, long long ldv, const int* m_ptr, int m_max,
                                const double* w, long long n, double* h, double* scratch,
                                cudaStream_t s) {
  if (m_max <= 0) return cudaSuccess;
  dim3 grid(kDotBlocks, (m_max + kMdVec - 1) / kMdVec);
  multidot_partial_dev_kernel<<<grid, kDotThreads, 0, s>>>(V, ldv, m_ptr, m_max, w, n, scratch);
  multidot_final_dev_kernel<<<m_max, kDotThreads, 0, s>>>(scratch, m_ptr, m_max, h);
  return cudaGetLastError();
}
cudaError_t launch_gemv_dev(const double* V, long long ldv, const int* m_ptr, int m_max,
                            const double* h, double alpha, double* w, double beta, long long n,
                            cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 8);
  gemv_dev_kernel<<<blocks, 256, (size_t)std::max(m_max, 1) * sizeof(double), s>>>(V, ldv, m_ptr, m_max, h,
                                                                                   alpha, w, beta, n);
  return cudaGetLastError();
}
cudaError_t launch_gmres_scalars(int phase, int* is, double* ds, double* H, int ldh,
                                 const double* h1, const double* h2, double* hist, int m_max,
                                 cudaStream_t s) {
  gmres_scalars_kernel<<<1, 1, 0, s>>>(phase, is, ds, H, ldh, h1, h2, hist, m_max);
  return cudaGetLastError();
}

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

cudaError_t launch_lincomb_dev(const double* k, const double* x, const double* y, const double* z,
                               double* out, long long n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 8);
  lincomb_dev_kernel<<<blocks, 256, 0, s>>>(k, x, y, z, out, n);
  return cudaGetLastError();
}

cudaError_t launch_minres_scalars(int phase, double* state, double* hist, int hist_cap, cudaStream_t s) {
  minres_scalars_kernel<<<1, 1, 0, s>>>(phase, state, hist, hist_cap);
  return cudaGetLastError();
}

cudaError_t launch_lincomb(double a, const double* x, double b, const double* y, double c,
                           const double* z, double* out, long long n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 8);
  lincomb_kernel<<<blocks, 256, 0, s>>>(a, x, b, y, c, z, out, n);
  return cudaGetLastError();
}

}  // namespace fdp
