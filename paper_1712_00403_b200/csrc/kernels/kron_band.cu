// K4: banded m-mode product for the matrix-free Stokes operator (NEXT-1; the Kronecker factors of
// a(.,.) and b(.,.), are banded B-spline Gram / stiffness / mixed matrices).
// Y(p, a, q) = alpha * sum_{j < bw} Wb[a*bw + j] * X(p, lo[a] + j, q) (+ beta * Y), the
// (P, n_in, Q) -> (P, n_out, Q) view of kernels/mode_contract.cu with the factor stored as its
// nonzero band per output row. HBM-bound (bw FMAs per output, the input window of a thread block
// reused through L1) instead of the dense contraction's 2 n_in flops per output.
#include "../fdp_internal.h"

namespace fdp {
namespace {

constexpr int kBandThreads = 256;

__global__ void __launch_bounds__(kBandThreads) kron_band_kernel(const __grid_constant__ BandGroup g) {
  int pi = 0;
  for (int i = 1; i < g.count; ++i)
    if ((int)blockIdx.x >= g.prob[i].blk_begin) pi = i;
  const BandProb& b = g.prob[pi];
  const long long idx = (long long)(blockIdx.x - b.blk_begin) * kBandThreads + threadIdx.x;
  const long long P = b.P;
  const long long total = P * b.nout * b.Q;
  if (idx >= total) return;
  const long long p = idx % P, r = idx / P;
  const int a = (int)(r % b.nout);
  const long long q = r / b.nout;
  const double* __restrict__ x = b.X + p + P * (b.lo[a] + (long long)b.nin * q);
  const double* __restrict__ w = b.Wb + (long long)a * b.bw;
  double s0 = 0.0, s1 = 0.0;
  int j = 0;
  for (; j + 2 <= b.bw; j += 2) {
    s0 = fma(__ldg(w + j), __ldg(x + P * j), s0);
    s1 = fma(__ldg(w + j + 1), __ldg(x + P * (j + 1)), s1);
  }
  if (j < b.bw) s0 = fma(__ldg(w + j), __ldg(x + P * j), s0);
  double v = b.alpha * (s0 + s1);
  double* y = b.Y + p + P * (a + (long long)b.nout * q);
  if (b.beta != 0.0) v += b.beta * *y;
  *y = v;
}

}  // namespace

cudaError_t launch_kron_band(const BandGroup& g, cudaStream_t s) {
  if (g.total_blocks <= 0) return cudaSuccess;
  kron_band_kernel<<<g.total_blocks, kBandThreads, 0, s>>>(g);
  return cudaGetLastError();
}

int kron_band_blocks(long long outputs) { return (int)((outputs + kBandThreads - 1) / kBandThreads); }

}  // namespace fdp
