// K3: banded Kronecker mass solve / product along the fibers of one mode (PAPER.md P:975-976:
// "the solution of a linear system with matrix P_Q is obtained in a direct way with only O(p n_Q)
// FLOPs"; per-mode application by the identity (A(x)B(x)C)^{-1} vec X of P:422-426).
//
// One thread per fiber (p, q) of the (P, n, Q) view; consecutive threads take consecutive p, so
// for modes >= 2 every step of the recurrence is a coalesced warp access. The last `band`
// solution values live in registers (shift register, BAND is a template parameter).
#include "../fdp_internal.h"

namespace fdp {
namespace {

template <int BAND>
__global__ void mass_solve_kernel(const MassMode mm) {
  const long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nf = (long long)mm.P * mm.Q * mm.batch;
  if (f >= nf) return;
  const int P = mm.P, n = mm.n;
  const long long p = f % P, r = f / P;
  const long long sbase = p + (long long)P * n * (r % mm.Q);  // index within the batch item
  const long long base = sbase + mm.bs * (r / mm.Q);
  const double* __restrict__ in = mm.in;
  double* __restrict__ out = mm.out;
  const double* __restrict__ Lb = mm.Lb;
  const double* __restrict__ invd = mm.invd;

  // forward substitution L y = x  (y written to out)
  double ring[BAND > 0 ? BAND : 1];  // ring[0] = y_{i-1}, ring[1] = y_{i-2}, ...
#pragma unroll
  for (int j = 0; j < BAND; ++j) ring[j] = 0.0;
  for (int i = 0; i < n; ++i) {
    const long long idx = base + (long long)P * i;
    double v = in[idx];
    if (mm.pre) v *= mm.pre[sbase + (long long)P * i];
    const double* Li = Lb + (size_t)i * (BAND + 1);
#pragma unroll
    for (int j = 1; j <= BAND; ++j) v -= Li[BAND - j] * ring[j - 1];
    v *= invd[i];
#pragma unroll
    for (int j = BAND - 1; j > 0; --j) ring[j] = ring[j - 1];
    if (BAND > 0) ring[0] = v;
    out[idx] = v;
  }
  // back substitution L^T z = y:  z_i = (y_i - sum_j L[i+j][i] z_{i+j}) / L[i][i]
#pragma unroll
  for (int j = 0; j < BAND; ++j) ring[j] = 0.0;
  for (int i = n - 1; i >= 0; --i) {
    const long long idx = base + (long long)P * i;
    double v = out[idx];
#pragma unroll
    for (int j = 1; j <= BAND; ++j) {
      if (i + j < n) v -= Lb[(size_t)(i + j) * (BAND + 1) + (BAND - j)] * ring[j - 1];
    }
    v *= invd[i];
#pragma unroll
    for (int j = BAND - 1; j > 0; --j) ring[j] = ring[j - 1];
    if (BAND > 0) ring[0] = v;
    if (mm.post) v *= mm.post[sbase + (long long)P * i];
    out[idx] = v;
  }
}

// y = M x along fibers (FDP_MASS_FORWARD); out must not alias in.
template <int BAND>
__global__ void mass_forward_kernel(const MassMode mm) {
  const long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nf = (long long)mm.P * mm.Q * mm.batch;
  if (f >= nf) return;
  const int P = mm.P, n = mm.n;
  const long long p = f % P, r = f / P;
  const long long base = p + (long long)P * n * (r % mm.Q) + mm.bs * (r / mm.Q);
  for (int i = 0; i < n; ++i) {
    double v = 0.0;
#pragma unroll
    for (int d = -BAND; d <= BAND; ++d) {
      const int j = i + d;
      if (j >= 0 && j < n) v += mm.Mb[(size_t)i * (2 * BAND + 1) + (d + BAND)] * mm.in[base + (long long)P * j];
    }
    mm.out[base + (long long)P * i] = v;
  }
}

template <int BAND>
cudaError_t launch_b(const MassMode& m, cudaStream_t s) {
  const long long nf = (long long)m.P * m.Q * m.batch;
  const int threads = 128;
  const long long blocks = (nf + threads - 1) / threads;
  if (blocks == 0) return cudaSuccess;
  if (m.forward) mass_forward_kernel<BAND><<<(unsigned)blocks, threads, 0, s>>>(m);
  else mass_solve_kernel<BAND><<<(unsigned)blocks, threads, 0, s>>>(m);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_mass_mode(const MassMode& m, cudaStream_t s) {
  switch (m.band) {
    case 0: return launch_b<0>(m, s);
    case 1: return launch_b<1>(m, s);
    case 2: return launch_b<2>(m, s);
    case 3: return launch_b<3>(m, s);
    case 4: return launch_b<4>(m, s);
    case 5: return launch_b<5>(m, s);
    case 6: return launch_b<6>(m, s);
    case 7: return launch_b<7>(m, s);
    case 8: return launch_b<8>(m, s);
    case 9: return launch_b<9>(m, s);
    case 10: return launch_b<10>(m, s);
    case 11: return launch_b<11>(m, s);
    case 12: return launch_b<12>(m, s);
    case 13: return launch_b<13>(m, s);
    case 14: return launch_b<14>(m, s);
    case 15: return launch_b<15>(m, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace fdp
