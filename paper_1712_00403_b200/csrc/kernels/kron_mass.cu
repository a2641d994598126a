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

// <= 64 registers (eight 128-thread blocks per SM): config 5's 266,256 fibers per mode then take
// two waves of 1,184 blocks instead of three of 1,036 (a fiber is a long sequential unit, so a
// nearly empty third wave costs a whole fiber time)
template <int BAND, int U>
__global__ void __launch_bounds__(128, 8) mass_solve_kernel(const MassMode mm) {
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

  // The recurrences are sequential in i but their loads are not: each sweep reads U fiber values
  // ahead (U independent loads in flight per thread instead of one; with one, the HBM latency
  // capped modes >= 2 at about half the copy bandwidth: config 5 1.30 -> 1.10 ms per mode).
  // Mode 1 (P == 1) takes mass_solve_mode1_kernel: read-ahead on its uncoalesced fibers only
  // thrashed L1 (3.1 vs 2.0 ms); the transposed tiles bring it to 1.6 ms.
  // forward substitution L y = x  (y written to out)
  double ring[BAND > 0 ? BAND : 1];  // ring[0] = y_{i-1}, ring[1] = y_{i-2}, ...
#pragma unroll
  for (int j = 0; j < BAND; ++j) ring[j] = 0.0;
  for (int i0 = 0; i0 < n; i0 += U) {
    double xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u;
      xv[u] = i < n ? in[base + (long long)P * i] : 0.0;
      if (mm.pre && i < n) xv[u] *= mm.pre[sbase + (long long)P * i];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u;
      if (i < n) {
        double v = xv[u];
        const double* Li = Lb + (size_t)i * (BAND + 1);
#pragma unroll
        for (int j = 1; j <= BAND; ++j) v -= Li[BAND - j] * ring[j - 1];
        v *= invd[i];
#pragma unroll
        for (int j = BAND - 1; j > 0; --j) ring[j] = ring[j - 1];
        if (BAND > 0) ring[0] = v;
        out[base + (long long)P * i] = v;
      }
    }
  }
  // back substitution L^T z = y:  z_i = (y_i - sum_j L[i+j][i] z_{i+j}) / L[i][i]
#pragma unroll
  for (int j = 0; j < BAND; ++j) ring[j] = 0.0;
  for (int i0 = n - 1; i0 >= 0; i0 -= U) {
    double yv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 - u;
      yv[u] = i >= 0 ? out[base + (long long)P * i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 - u;
      if (i >= 0) {
        double v = yv[u];
#pragma unroll
        for (int j = 1; j <= BAND; ++j) {
          if (i + j < n) v -= Lb[(size_t)(i + j) * (BAND + 1) + (BAND - j)] * ring[j - 1];
        }
        v *= invd[i];
#pragma unroll
        for (int j = BAND - 1; j > 0; --j) ring[j] = ring[j - 1];
        if (BAND > 0) ring[0] = v;
        if (mm.post) v *= mm.post[sbase + (long long)P * i];
        out[base + (long long)P * i] = v;
      }
    }
  }
}

// Mode 1 (P == 1: each fiber contiguous): one warp per 32 consecutive fibers, chunks of 32
// elements staged through a padded shared-memory tile so that every global access is a coalesced
// 256-byte row segment, the recurrence of lane l running down row l of the tile (stride 33:
// conflict-free). Same arithmetic, same order as mass_solve_kernel.
constexpr int kM1Warps = 4;
template <int BAND>
__global__ void __launch_bounds__(kM1Warps * 32)
mass_solve_mode1_kernel(const MassMode mm) {
  __shared__ double tile[kM1Warps][32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long nf = (long long)mm.Q * mm.batch;
  const long long f0 = ((long long)blockIdx.x * kM1Warps + w) * 32;
  if (f0 >= nf) return;
  const int n = mm.n;
  double (*T)[33] = tile[w];
  // lane r holds fiber f0 + r's element-0 offsets (global, and within its batch item), shared
  // with the warp by shuffles
  long long my_g = 0, my_s = 0;
  const bool my_ok = f0 + lane < nf;
  if (my_ok) {
    const long long f = f0 + lane, q = f % mm.Q, b = f / mm.Q;
    my_s = (long long)n * q;
    my_g = my_s + mm.bs * b;
  }
  const double* __restrict__ Lb = mm.Lb;
  const double* __restrict__ invd = mm.invd;
  double ring[BAND > 0 ? BAND : 1];
#pragma unroll
  for (int j = 0; j < BAND; ++j) ring[j] = 0.0;
  // forward substitution L y = x, y -> out
  for (int k0 = 0; k0 < n; k0 += 32) {
    const int k = k0 + lane;
    double v[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {  // 32 independent coalesced row segments in flight
      const long long g = __shfl_sync(0xffffffffu, my_g, r);
      const long long sb = __shfl_sync(0xffffffffu, my_s, r);
      const bool ok = __shfl_sync(0xffffffffu, my_ok, r) && k < n;
      v[r] = ok ? mm.in[g + k] : 0.0;
      if (ok && mm.pre) v[r] *= mm.pre[sb + k];
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) T[r][lane] = v[r];
    __syncwarp();
    const int kend = min(32, n - k0);
    // steps in groups of 4 whose tile values and band coefficients are loaded before the group's
    // dependent chain (one step at a time, the L1 latency of the coefficient loads sat on the
    // chain: 51% of the warps' stalls were long-scoreboard waits)
    int kk = 0;
    for (; kk + 4 <= kend; kk += 4) {
      double xv[4], cf[4][BAND > 0 ? BAND : 1], dv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = k0 + kk + u;
        xv[u] = T[lane][kk + u];
        dv[u] = __ldg(invd + i);
#pragma unroll
        for (int j = 1; j <= BAND; ++j) cf[u][j - 1] = __ldg(Lb + (size_t)i * (BAND + 1) + (BAND - j));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        double x = xv[u];
#pragma unroll
        for (int j = 1; j <= BAND; ++j) x -= cf[u][j - 1] * ring[j - 1];
        x *= dv[u];
#pragma unroll
        for (int j = BAND - 1; j > 0; --j) ring[j] = ring[j - 1];
        if (BAND > 0) ring[0] = x;
        T[lane][kk + u] = x;
      }
    }
    for (; kk < kend; ++kk) {
      const int i = k0 + kk;
      double x = T[lane][kk];
      const double* Li = Lb + (size_t)i * (BAND + 1);
#pragma unroll
      for (int j = 1; j <= BAND; ++j) x -= Li[BAND - j] * ring[j - 1];
      x *= invd[i];
#pragma unroll
      for (int j = BAND - 1; j > 0; --j) ring[j] = ring[j - 1];
      if (BAND > 0) ring[0] = x;
      T[lane][kk] = x;
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const long long g = __shfl_sync(0xffffffffu, my_g, r);
      const bool ok = __shfl_sync(0xffffffffu, my_ok, r) && k < n;
      if (ok) mm.out[g + k] = T[r][lane];
    }
    __syncwarp();
  }
  // back substitution L^T z = y over the chunks in reverse
#pragma unroll
  for (int j = 0; j < BAND; ++j) ring[j] = 0.0;
  for (int k0 = ((n - 1) / 32) * 32; k0 >= 0; k0 -= 32) {
    const int k = k0 + lane;
    double v[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const long long g = __shfl_sync(0xffffffffu, my_g, r);
      const bool ok = __shfl_sync(0xffffffffu, my_ok, r) && k < n;
      v[r] = ok ? mm.out[g + k] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) T[r][lane] = v[r];
    __syncwarp();
    const int kend = min(32, n - k0);
    int kk = kend - 1;
    for (; kk - 3 >= 0; kk -= 4) {  // groups of 4 steps, inputs loaded first (see above)
      double xv[4], cf[4][BAND > 0 ? BAND : 1], dv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = k0 + kk - u;
        xv[u] = T[lane][kk - u];
        dv[u] = __ldg(invd + i);
#pragma unroll
        for (int j = 1; j <= BAND; ++j)
          cf[u][j - 1] = i + j < n ? __ldg(Lb + (size_t)(i + j) * (BAND + 1) + (BAND - j)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        double x = xv[u];
#pragma unroll
        for (int j = 1; j <= BAND; ++j) x -= cf[u][j - 1] * ring[j - 1];
        x *= dv[u];
#pragma unroll
        for (int j = BAND - 1; j > 0; --j) ring[j] = ring[j - 1];
        if (BAND > 0) ring[0] = x;
        T[lane][kk - u] = x;
      }
    }
    for (; kk >= 0; --kk) {
      const int i = k0 + kk;
      double x = T[lane][kk];
#pragma unroll
      for (int j = 1; j <= BAND; ++j) {
        if (i + j < n) x -= Lb[(size_t)(i + j) * (BAND + 1) + (BAND - j)] * ring[j - 1];
      }
      x *= invd[i];
#pragma unroll
      for (int j = BAND - 1; j > 0; --j) ring[j] = ring[j - 1];
      if (BAND > 0) ring[0] = x;
      T[lane][kk] = x;
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const long long g = __shfl_sync(0xffffffffu, my_g, r);
      const long long sb = __shfl_sync(0xffffffffu, my_s, r);
      const bool ok = __shfl_sync(0xffffffffu, my_ok, r) && k < n;
      if (ok) {
        double x = T[r][lane];
        if (mm.post) x *= mm.post[sb + k];
        mm.out[g + k] = x;
      }
    }
    __syncwarp();
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
  else if (m.P == 1) {
    const long long warps = (nf + 31) / 32;
    mass_solve_mode1_kernel<BAND><<<(unsigned)((warps + kM1Warps - 1) / kM1Warps), kM1Warps * 32, 0, s>>>(m);
  }
  else mass_solve_kernel<BAND, 8><<<(unsigned)blocks, threads, 0, s>>>(m);
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
