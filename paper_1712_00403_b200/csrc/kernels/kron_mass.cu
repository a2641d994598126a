// K3: banded Kronecker mass solve / product along the fibers of one mode (PAPER.md P:975-976:
// "the solution of a linear system with matrix P_Q is obtained in a direct way with only O(p n_Q)
// FLOPs"; per-mode application by the identity (A(x)B(x)C)^{-1} vec X of P:422-426).
//
// One thread per fiber (p, q) of the (P, n, Q) view; consecutive threads take consecutive p, so
// for modes >= 2 every step of the recurrence is a coalesced warp access. The last `band`
// solution values live in registers (shift register, BAND is a template parameter).
#include "../fdp_internal.h"

#include <cuda.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

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

// K3t: the whole solve of a tile of F fibers in shared memory — one HBM read and one HBM write
// per element instead of the two of each that the forward/back sweeps above cost (y round-trips
// through `out`). One warp per CTA. Mode 1 (P == 1): lane 0 arms an mbarrier and the lanes issue
// one bulk copy per fiber (n doubles) into a fiber-major tile whose fiber stride NP is 2 mod 4
// doubles (16-byte aligned rows; the 14-16 fibers' accesses spread over the bank groups); modes
// >= 2: lane 0 issues `nbox` 4-D TMA tensor-map boxes {F fibers, boxn rows} (tile element (i, r)
// at i F + r; a ragged last p-block is zero-filled on load and clipped on store). Lanes r < nf
// run fiber r's recurrences in place and the tile leaves with bulk stores. The scaled band
// coefficients cf / cb (kron_mass_setup) make each step one multiply and BAND FMAs whose
// dependent chain is a single FMA on the newest value:
//   forward  y_i = x_i d_i - sum_{j=BAND..1} (L_{i,i-j} d_i) y_{i-j}
//   backward z_i = y_i d_i - sum_{j=BAND..1} (L_{i+j,i} d_i) z_{i+j},   d_i = 1 / L_ii
// (the same solve as mass_solve_kernel up to rounding order). Round 2's ncu source view: the warp
// issues one instruction per ~3.7 cycles and a quarter of them are the coefficient loads through
// L1 (~4 issue cycles each); K3u below keeps the rows in shared memory and takes the shapes it can.
// Steps go in groups of G = 4 whose
// tile values and coefficients sit in one of three register buffers loaded two groups ahead (one
// group ahead, the compiler sank the loads onto the consumers and the warps stalled on them).
// F = 14 leaves the L1 room for both coefficient arrays next to three tiles per SM.
__device__ __forceinline__ unsigned k3_smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void k3_bulk_load(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void k3_bulk_store(void* dst, unsigned src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void k3_map_load(unsigned dst, const CUtensorMap* map, unsigned bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void k3_map_store(const CUtensorMap* map, unsigned src, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
          reinterpret_cast<unsigned long long>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(src)
      : "memory");
}

__device__ __forceinline__ void k3_bulk_prefetch(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void k3_map_prefetch(const CUtensorMap* map, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                   reinterpret_cast<unsigned long long>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}

struct TileArgs {
  int NP;     // mode 1: fiber stride of the tile (doubles)
  int boxn;   // modes >= 2: rows per tensor-map box
  int nbox;   // boxes per tile
};

template <int BAND, int F, bool M1, bool SC>
__global__ void __launch_bounds__(32) mass_tile_kernel(const MassMode mm, const __grid_constant__ CUtensorMap map_in,
                                                      const __grid_constant__ CUtensorMap map_out,
                                                      const TileArgs ta) {
  extern __shared__ __align__(128) double T[];
  __shared__ __align__(8) unsigned long long bar;
  constexpr int CS = (BAND + 2) & ~1;  // coefficient row: BAND band values then d_i (padded even)
  constexpr int G = 4;
  const int lane = threadIdx.x;
  const int n = mm.n;
  const long long P = mm.P;
  long long gbase = 0, sbase = 0;  // lane's own fiber (M1) / the tile's first fiber (modes >= 2)
  int nf, p0 = 0, q = 0, bi = 0;
  if (M1) {
    const long long nfib = (long long)mm.Q * mm.batch, f0 = (long long)blockIdx.x * F;
    nf = (int)min((long long)F, nfib - f0);
    if (lane < nf) {
      const long long f = f0 + lane;
      sbase = (long long)n * (f % mm.Q);
      gbase = sbase + mm.bs * (f / mm.Q);
    }
  } else {
    const long long pblocks = (P + F - 1) / F, t = blockIdx.x;
    p0 = (int)((t % pblocks) * F);
    const long long rest = t / pblocks;
    q = (int)(rest % mm.Q);
    bi = (int)(rest / mm.Q);
    nf = (int)min((long long)F, P - p0);
    sbase = p0 + P * n * q;
  }
  const unsigned tb = k3_smem_u32(T), bb = k3_smem_u32(&bar);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const unsigned bytes = M1 ? (unsigned)(n * nf * 8) : (unsigned)(ta.nbox * ta.boxn * F * 8);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(bytes) : "memory");
    if (!M1)
      for (int k = 0; k < ta.nbox; ++k)
        k3_map_load(tb + (unsigned)(k * ta.boxn * F * 8), &map_in, bb, p0, k * ta.boxn, q, bi);
  }
  __syncwarp();
  if (M1 && lane < nf) k3_bulk_load(tb + (unsigned)(lane * ta.NP * 8), mm.in + gbase, (unsigned)n * 8, bb);
  asm volatile(
      "{\n.reg .pred p;\nK3W_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      "@!p bra K3W_%=;\n}\n" ::"r"(bb)
      : "memory");

  if (lane < nf) {
    const int r = lane;
    double* const Tr = M1 ? T + r * ta.NP : T + r;  // element i at Tr[i * ist]
    const int ist = M1 ? 1 : F;
    const long long pofs = M1 ? sbase : sbase + r;  // pre / post scaling offset
    const long long pstr = M1 ? 1 : P;
    const double* __restrict__ pre = SC ? mm.pre : nullptr;  // SC: a P^G scaling is present
    const double* __restrict__ post = SC ? mm.post : nullptr;
    double ring[BAND];  // ring[j-1] = value j steps back
    struct Buf {
      double x[G];
      double c[G][CS];
    };
    Buf A, B, C;
    const int ng = n / G;
    // ---- forward ----
    const double* __restrict__ cf = mm.cf;
    auto load_f = [&](Buf& bf, int g) {
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const int i = g * G + u;
        if (M1) {  // fiber-major tile: element pairs as 16-byte shared loads (i even, NP even)
          if ((u & 1) == 0) {
            const double2 t = *reinterpret_cast<const double2*>(Tr + i);
            bf.x[u] = t.x;
            bf.x[u + 1] = t.y;
          }
        } else {
          bf.x[u] = Tr[i * ist];
        }
        if (pre) bf.x[u] *= __ldg(pre + pofs + pstr * i);
#pragma unroll
        for (int k = 0; k < CS; k += 2) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(cf + (size_t)i * CS + k));
          bf.c[u][k] = v.x;
          bf.c[u][k + 1] = v.y;
        }
      }
    };
    double Tf1 = 0.0;  // M1: the previous output of the pair being assembled
    auto step_f = [&](const Buf& bf, int g) {
#pragma unroll
      for (int u = 0; u < G; ++u) {
        double v = bf.x[u] * bf.c[u][BAND];
#pragma unroll
        for (int k = 0; k < BAND; ++k) v = fma(-bf.c[u][k], ring[BAND - 1 - k], v);
#pragma unroll
        for (int j = BAND - 1; j > 0; --j) ring[j] = ring[j - 1];
        ring[0] = v;
        if (M1) {
          if (u & 1) *reinterpret_cast<double2*>(Tr + g * G + u - 1) = make_double2(Tf1, v);
          Tf1 = v;
        } else {
          Tr[(g * G + u) * ist] = v;
        }
      }
    };
#pragma unroll
    for (int j = 0; j < BAND; ++j) ring[j] = 0.0;
    if (ng > 0) load_f(A, 0);
    if (ng > 1) load_f(B, 1);
    int g = 0;
    for (; g + 3 <= ng; g += 3) {
      load_f(C, g + 2);
      step_f(A, g);
      load_f(A, min(g + 3, ng - 1));
      step_f(B, g + 1);
      load_f(B, min(g + 4, ng - 1));
      step_f(C, g + 2);
    }
    if (g < ng) step_f(A, g);
    if (g + 1 < ng) step_f(B, g + 1);
    for (int i = ng * G; i < n; ++i) {
      double v = Tr[i * ist];
      if (pre) v *= __ldg(pre + pofs + pstr * i);
      const double* c = cf + (size_t)i * CS;
      v *= __ldg(c + BAND);
#pragma unroll
      for (int k = 0; k < BAND; ++k) v = fma(-__ldg(c + k), ring[BAND - 1 - k], v);
#pragma unroll
      for (int j = BAND - 1; j > 0; --j) ring[j] = ring[j - 1];
      ring[0] = v;
      Tr[i * ist] = v;
    }
    // ---- backward: the n % G top steps singly, then groups h = ng-1 .. 0 (steps 4h+3 .. 4h) ----
    const double* __restrict__ cb = mm.cb;
#pragma unroll
    for (int j = 0; j < BAND; ++j) ring[j] = 0.0;
    for (int i = n - 1; i >= ng * G; --i) {
      const double* c = cb + (size_t)i * CS;
      double v = Tr[i * ist] * __ldg(c + BAND);
#pragma unroll
      for (int k = 0; k < BAND; ++k) v = fma(-__ldg(c + k), ring[BAND - 1 - k], v);
#pragma unroll
      for (int j = BAND - 1; j > 0; --j) ring[j] = ring[j - 1];
      ring[0] = v;
      Tr[i * ist] = post ? v * __ldg(post + pofs + pstr * i) : v;
    }
    auto load_b = [&](Buf& bf, int h) {
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const int i = h * G + G - 1 - u;
        if (M1) {  // steps i, i - 1 from one 16-byte load at i - 1 (i odd)
          if ((u & 1) == 0) {
            const double2 t = *reinterpret_cast<const double2*>(Tr + i - 1);
            bf.x[u] = t.y;
            bf.x[u + 1] = t.x;
          }
        } else {
          bf.x[u] = Tr[i * ist];
        }
#pragma unroll
        for (int k = 0; k < CS; k += 2) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(cb + (size_t)i * CS + k));
          bf.c[u][k] = v.x;
          bf.c[u][k + 1] = v.y;
        }
      }
    };
    double Tr1 = 0.0;  // M1: the previous (higher-i) output of the pair being assembled
    auto step_b = [&](const Buf& bf, int h) {
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const int i = h * G + G - 1 - u;
        double v = bf.x[u] * bf.c[u][BAND];
#pragma unroll
        for (int k = 0; k < BAND; ++k) v = fma(-bf.c[u][k], ring[BAND - 1 - k], v);
#pragma unroll
        for (int j = BAND - 1; j > 0; --j) ring[j] = ring[j - 1];
        ring[0] = v;
        const double o = post ? v * __ldg(post + pofs + pstr * i) : v;
        if (M1) {  // (i, i + 1) written together at the odd step u (i even)
          if (u & 1) *reinterpret_cast<double2*>(Tr + i) = make_double2(o, Tr1);
          Tr1 = o;
        } else {
          Tr[i * ist] = o;
        }
      }
    };
    if (ng > 0) load_b(A, ng - 1);
    if (ng > 1) load_b(B, ng - 2);
    int h = ng - 1;
    for (; h - 2 >= 0; h -= 3) {
      load_b(C, h - 2);
      step_b(A, h);
      load_b(A, max(h - 3, 0));
      step_b(B, h - 1);
      load_b(B, max(h - 4, 0));
      step_b(C, h - 2);
    }
    if (h >= 0) step_b(A, h);
    if (h - 1 >= 0) step_b(B, h - 1);
  }
  // generic-proxy smem writes -> visible to the bulk-copy (async) proxy, then the stores
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (M1) {
    if (lane < nf) k3_bulk_store(mm.out + gbase, tb + (unsigned)(lane * ta.NP * 8), (unsigned)n * 8);
  } else if (lane == 0) {
    for (int k = 0; k < ta.nbox; ++k)
      k3_map_store(&map_out, tb + (unsigned)(k * ta.boxn * F * 8), p0, k * ta.boxn, q, bi);
  }
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem stays valid until read
}

// K3t applies when the copies' 16-byte rules hold (mode 1: n even; modes >= 2: P even, for the
// tensor maps' strides; 16-byte aligned in / out, even batch stride), BAND <= kTileMaxBand and
// the tile fits the per-CTA shared memory.
constexpr int kTileMaxSmem = 227 * 1024;
constexpr int kTileMaxBand = 8;
inline int tile_f() {
  static const int f = [] {
    const char* e = std::getenv("FDP_K3_F");
    const int v = e ? std::atoi(e) : 14;
    return v == 16 ? 16 : 14;
  }();
  return f;
}
inline int tile_np(int n) { return (n / 2) % 2 ? n : n + 2; }  // n even: n or n + 2, = 2 mod 4
inline TileArgs tile_args(const MassMode& m) {
  TileArgs ta{};
  ta.NP = tile_np(m.n);
  ta.nbox = (m.n + 255) / 256;
  // rows per box a multiple of 8: every box's shared-memory destination 128-byte aligned (F even)
  ta.boxn = ((m.n + ta.nbox - 1) / ta.nbox + 7) / 8 * 8;
  return ta;
}
inline size_t tile_smem(const MassMode& m, int F) {
  const TileArgs ta = tile_args(m);
  return m.P == 1 ? (size_t)F * ta.NP * 8 : (size_t)F * ta.boxn * ta.nbox * 8;
}
inline bool tile_ok(const MassMode& m) {
  static const bool sweep = std::getenv("FDP_K3_SWEEP") != nullptr;  // diagnostic: the sweep kernels
  static const bool all = std::getenv("FDP_K3_TILE_ALL") != nullptr;  // diagnostic: K3t in modes >= 2
  if (m.forward || !m.cf || !m.cb || sweep || m.band < 1 || m.band > kTileMaxBand) return false;
  // modes >= 2: the coalesced sweep kernel (0.9 ms per config-5 mode at 4.4 GB) beats K3t (1.2 ms
  // at 2.2 GB: three 14-fiber tiles per SM leave the recurrences issue-bound)
  if (m.P != 1 && !all) return false;
  const bool a16 = ((reinterpret_cast<uintptr_t>(m.in) | reinterpret_cast<uintptr_t>(m.out)) & 15) == 0;
  if (!a16 || (m.batch > 1 && (m.bs & 1))) return false;
  if (m.P == 1 ? (m.n & 1) : (m.P & 1)) return false;
  if ((long long)m.Q * m.batch >= (1LL << 31)) return false;
  return tile_smem(m, tile_f()) <= (size_t)kTileMaxSmem;
}

template <int BAND, int F>
cudaError_t launch_tile(const MassMode& m, cudaStream_t s) {
  const TileArgs ta = tile_args(m);
  const size_t smem = tile_smem(m, F);
  const bool m1 = m.P == 1;
  CUtensorMap map_in, map_out;
  std::memset(&map_in, 0, sizeof(map_in));
  std::memset(&map_out, 0, sizeof(map_out));
  if (!m1 && (!mass_tile_map(&map_in, m.in, m.P, m.n, m.Q, m.batch, m.bs, F, ta.boxn) ||
              !mass_tile_map(&map_out, m.out, m.P, m.n, m.Q, m.batch, m.bs, F, ta.boxn)))
    return cudaErrorNotSupported;
  const long long tiles = m1 ? ((long long)m.Q * m.batch + F - 1) / F
                             : ((long long)m.P + F - 1) / F * m.Q * m.batch;
  const bool sc = m.pre || m.post;
  auto kern = m1 ? (sc ? mass_tile_kernel<BAND, F, true, true> : mass_tile_kernel<BAND, F, true, false>)
                 : (sc ? mass_tile_kernel<BAND, F, false, true> : mass_tile_kernel<BAND, F, false, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // the smallest carveout that holds three tiles (the rest of the 256 KB is L1, where the forward
  // and backward coefficient arrays live: 2 x 24.8 KB at n = 516, band 4)
  const int pct = (int)std::min<size_t>(100, (3 * (smem + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024));
  if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)tiles, 32, smem, s>>>(m, map_in, map_out, ta);
  return cudaGetLastError();
}

template <int BAND>
cudaError_t launch_tile_b(const MassMode& m, cudaStream_t s) {
  if constexpr (BAND >= 1 && BAND <= kTileMaxBand)
    return tile_f() == 16 ? launch_tile<BAND, 16>(m, s) : launch_tile<BAND, 14>(m, s);
  return cudaErrorNotSupported;
}

// K3u: K3t rebuilt around the instruction stream. The ncu source view of K3t shows one warp per
// sub-partition issuing an instruction every ~3.7 cycles: three of every twelve are coefficient
// loads through L1 with 64-bit address arithmetic, and each costs ~4 issue cycles, so a step takes
// ~40 cycles where its five FP64 instructions need 10. K3u is one persistent 4-warp CTA per SM:
//   * the scaled band rows R_i = (L_{i,i-BAND..i-1} d_i, d_i) (`cf`, the only table: both
//     substitutions read ROW i at step i) are copied to shared memory once per CTA and read with
//     warp-uniform 16-byte loads, no L1 and no per-step address arithmetic;
//   * each warp owns a tile of 12 fibers (4 x 12 x n doubles + the table fill the 227 KB) and walks
//     its own tile sequence with its own mbarrier, so the four warps' loads, solves and stores
//     overlap each other;
//   * both substitutions are right-looking, so the BAND FMAs of a step are independent of each
//     other and the dependent chain is the single FMA on the newest value:
//       forward   y_i = A_i - R_{i,BAND-1} y_{i-1};  A_{i+m} -= R_{i+m,BAND-1-m} y_{i-1} (m < BAND-1);
//                 A_{i+BAND-1} = x_{i+BAND-1} d_{i+BAND-1} - R_{i+BAND-1,0} y_{i-1}
//       backward  (z_i = d_i r_i)  r_j = A_j;  A_{j-m} -= R_{j,BAND-m} r_j (m = 1..BAND-1);
//                 A_{j-BAND} = y_{j-BAND} - R_{j,0} r_j
//     (the forward sums accumulate in K3t's order; the backward works on r = z / d so that the
//     row-scaled table serves it too).
// Steps go in groups of G = 4 rows whose tile values and coefficients sit in one of three register
// buffers loaded ahead. Needs n % 4 == 0, n >= 16, 1 <= BAND <= 5 (the forward window of BAND rows
// spans two groups); other shapes keep K3t / the sweeps.
constexpr int kUWarps = 4;  // measured: 6 warps x 8 fibers 3.30 ms, 8 x 6 3.87 ms vs 2.36 ms (config 5, all modes)
constexpr int kUF = 12;
struct UArgs {
  int NP;         // mode 1: fiber stride of the tile (doubles)
  int boxn;       // modes >= 2: rows per tensor-map box
  int nbox;       // boxes per tile
  int tile_d;     // doubles per warp tile (128-byte multiple)
  int tab_d;      // doubles of the coefficient table region (128-byte multiple)
  long long tiles;
  int prefetch;   // L2 prefetch of the warp's next tile: 0 off, 1 at load time, 2 between the substitutions
};

template <int BAND, bool M1, bool SC>
__global__ void __launch_bounds__(kUWarps * 32, 1)
    mass_utile_kernel(const MassMode mm, const __grid_constant__ CUtensorMap map_in,
                      const __grid_constant__ CUtensorMap map_out, const UArgs ua) {
  extern __shared__ __align__(128) double S[];
  __shared__ __align__(8) unsigned long long bars[kUWarps];
  constexpr int CS = (BAND + 2) & ~1;
  constexpr int G = 4;
  constexpr int F = kUF;
  const int n = mm.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long P = mm.P;
  // the table in shared memory. BAND odd: the rows of cf as they are (BAND coefficients and d_i,
  // 16-byte aligned); BAND even: the d_i split off into their own array behind the rows, so that a
  // group of four rows costs BAND / 2 loads per row plus two for its four d_i (instead of a padded
  // third load per row)
  constexpr bool SPLIT = (BAND & 1) == 0;
  constexpr int RS = SPLIT ? BAND : CS;  // row stride
  if (SPLIT) {
    for (int i = threadIdx.x; i < n * CS; i += kUWarps * 32) {
      const int row = i / CS, k = i - row * CS;
      const double v = __ldg(mm.cf + i);
      if (k < BAND) S[row * BAND + k] = v;
      else if (k == BAND) S[n * BAND + row] = v;
    }
  } else {
    const double2* __restrict__ src = reinterpret_cast<const double2*>(mm.cf);
    double2* dst = reinterpret_cast<double2*>(S);
    for (int i = threadIdx.x; i < n * CS / 2; i += kUWarps * 32) dst[i] = __ldg(src + i);
  }
  const double* const R = S;
  const double* const E = S + (size_t)n * BAND;  // SPLIT: d_i
  double* const T = S + ua.tab_d + (size_t)warp * ua.tile_d;
  const unsigned tb = k3_smem_u32(T), bb = k3_smem_u32(&bars[warp]);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int ng = n / G;
  const double* __restrict__ pre = SC ? mm.pre : nullptr;
  const double* __restrict__ post = SC ? mm.post : nullptr;
  unsigned phase = 0;
  for (long long t = (long long)blockIdx.x * kUWarps + warp; t < ua.tiles; t += (long long)gridDim.x * kUWarps) {
    long long gbase = 0, sbase = 0;  // lane's own fiber (M1) / the tile's first fiber (modes >= 2)
    int nf, p0 = 0, q = 0, bi = 0;
    if (M1) {
      const long long nfib = (long long)mm.Q * mm.batch, f0 = t * F;
      nf = (int)min((long long)F, nfib - f0);
      if (lane < nf) {
        const long long f = f0 + lane;
        sbase = (long long)n * (f % mm.Q);
        gbase = sbase + mm.bs * (f / mm.Q);
      }
    } else {
      const long long pblocks = (P + F - 1) / F;
      p0 = (int)((t % pblocks) * F);
      const long long rest = t / pblocks;
      q = (int)(rest % mm.Q);
      bi = (int)(rest / mm.Q);
      nf = (int)min((long long)F, P - p0);
      sbase = p0 + P * n * q;
    }
    if (lane == 0) {
      const unsigned bytes = M1 ? (unsigned)(n * nf * 8) : (unsigned)(ua.nbox * ua.boxn * F * 8);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(bytes) : "memory");
      if (!M1)
        for (int k = 0; k < ua.nbox; ++k)
          k3_map_load(tb + (unsigned)(k * ua.boxn * F * 8), &map_in, bb, p0, k * ua.boxn, q, bi);
    }
    __syncwarp();
    if (M1 && lane < nf) k3_bulk_load(tb + (unsigned)(lane * ua.NP * 8), mm.in + gbase, (unsigned)n * 8, bb);
    // the warp's next tile on its way into L2 while this one is solved; issued between the two
    // substitutions: at load time (a whole tile solve, ~13 us, ahead) ncu showed 1.25-1.6x the
    // algorithmic DRAM reads - part of the prefetched lines were evicted before their load
    auto prefetch_next = [&]() {
      const long long tn = t + (long long)gridDim.x * kUWarps;
      if (tn < ua.tiles) {
        if (M1) {
          const long long nfib = (long long)mm.Q * mm.batch, f = tn * F + lane;
          if (lane < F && f < nfib)
            k3_bulk_prefetch(mm.in + (long long)n * (f % mm.Q) + mm.bs * (f / mm.Q), (unsigned)n * 8);
        } else if (lane == 0) {
          const long long pblocks = (P + F - 1) / F, rest = tn / pblocks;
          for (int k = 0; k < ua.nbox; ++k)
            k3_map_prefetch(&map_in, (int)((tn % pblocks) * F), k * ua.boxn, (int)(rest % mm.Q), (int)(rest / mm.Q));
        }
      }
    };
    if (ua.prefetch == 1) prefetch_next();
    asm volatile(
        "{\n.reg .pred p;\nK3U_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra K3U_%=;\n}\n" ::"r"(bb),
        "r"(phase)
        : "memory");
    phase ^= 1u;

    if (lane < nf) {
      const int r = lane;
      double* const Tr = M1 ? T + r * ua.NP : T + r;  // element i at Tr[i * ist]
      constexpr int ist = M1 ? 1 : F;
      const long long pofs = M1 ? sbase : sbase + r;  // pre / post scaling offset
      const long long pstr = M1 ? 1 : P;
      struct Buf {
        double x[G];      // forward: x_i (then x_i d_i); backward: y_{j-BAND}
        double c[G][CS];  // R_i (unused in the constant-row phases)
      };
      Buf A, B, C;
      auto load_c = [&](Buf& bf, int i, int u) {
#pragma unroll
        for (int k = 0; k < RS; k += 2) {
          const double2 v = *reinterpret_cast<const double2*>(R + (size_t)i * RS + k);
          bf.c[u][k] = v.x;
          bf.c[u][k + 1] = v.y;
        }
      };
      // SPLIT: the d_i of rows 4 gq .. 4 gq + 3 into slots u = 0..3 (rev: 3..0)
      auto load_e = [&](Buf& bf, int gq, bool rev) {
        if (SPLIT) {
          const double2 a = *reinterpret_cast<const double2*>(E + gq * G);
          const double2 b = *reinterpret_cast<const double2*>(E + gq * G + 2);
          bf.c[rev ? 3 : 0][BAND] = a.x;
          bf.c[rev ? 2 : 1][BAND] = a.y;
          bf.c[rev ? 1 : 2][BAND] = b.x;
          bf.c[rev ? 0 : 3][BAND] = b.y;
        }
      };
      auto coef = [&](int i, int k) { return R[(size_t)i * RS + k]; };
      auto dinv = [&](int i) { return SPLIT ? E[i] : R[(size_t)i * RS + BAND]; };
      // ---------------- forward ----------------
      auto load_f = [&](Buf& bf, int g) {
#pragma unroll
        for (int u = 0; u < G; ++u) {
          const int i = g * G + u;
          load_c(bf, i, u);
          if (M1) {
            if ((u & 1) == 0) {
              const double2 v = *reinterpret_cast<const double2*>(Tr + i);
              bf.x[u] = v.x;
              bf.x[u + 1] = v.y;
            }
          } else {
            bf.x[u] = Tr[i * ist];
          }
        }
        load_e(bf, g, false);
        if (pre) {
#pragma unroll
          for (int u = 0; u < G; ++u) bf.x[u] *= __ldg(pre + pofs + pstr * (g * G + u));
        }
      };
      // x_i d_i of a buffer, a group after its loads were issued (next to the loads, the multiplies
      // stalled the warp on the load latency)
      auto scale_f = [&](Buf& bf) {
#pragma unroll
        for (int u = 0; u < G; ++u) bf.x[u] *= bf.c[u][BAND];
      };
      double acc[BAND > 1 ? BAND - 1 : 1];
      double yp = 0.0, ylo = 0.0;
      auto step_f = [&](const Buf& cur, Buf& nxt, int g) {
        scale_f(nxt);
#pragma unroll
        for (int u = 0; u < G; ++u) {
          // row i + m of the window: cur for u + m < G, else nxt
          auto cf_ = [&](int m, int k) { return (u + m < G) ? cur.c[(u + m) % G][k] : nxt.c[(u + m) % G][k]; };
          double y;
          if (BAND == 1) {
            y = fma(-cf_(0, 0), yp, cur.x[u]);
          } else {
            y = fma(-cf_(0, BAND - 1), yp, acc[0]);
#pragma unroll
            for (int m = 1; m < BAND - 1; ++m) acc[m - 1] = fma(-cf_(m, BAND - 1 - m), yp, acc[m]);
            const double xn = (u + BAND - 1 < G) ? cur.x[(u + BAND - 1) % G] : nxt.x[(u + BAND - 1) % G];
            acc[BAND - 2] = fma(-cf_(BAND - 1, 0), yp, xn);
          }
          yp = y;
          if (M1) {
            if (u & 1) *reinterpret_cast<double2*>(Tr + g * G + u - 1) = make_double2(ylo, y);
            ylo = y;
          } else {
            Tr[(g * G + u) * ist] = y;
          }
        }
      };
      // groups g0 .. g1-1 right-looking, three register buffers loaded two groups ahead
      auto run_f = [&](int g0, int g1) {
        load_f(A, g0);
        load_f(B, min(g0 + 1, ng - 1));
        scale_f(A);
        int g = g0;
        for (; g + 3 <= g1; g += 3) {
          load_f(C, min(g + 2, ng - 1));
          step_f(A, B, g);
          load_f(A, min(g + 3, ng - 1));
          step_f(B, C, g + 1);
          load_f(B, min(g + 4, ng - 1));
          step_f(C, A, g + 2);
        }
        if (g < g1) {
          load_f(C, min(g + 2, ng - 1));
          step_f(A, B, g);
          if (g + 1 < g1) step_f(B, C, g + 1);
        }
      };
      {
        const int ngm = ng - 1;  // groups 0 .. ng-2 run right-looking (their windows end in group ng-1)
#pragma unroll
        for (int m = 0; m < BAND - 1; ++m) {
          double v = Tr[m * ist] * dinv(m);
          if (pre) v *= __ldg(pre + pofs + pstr * m);
          acc[m] = v;
        }
        run_f(0, ngm);
        // the last group left-looking from the tile
        for (int i = ngm * G; i < n; ++i) {
          double v = Tr[i * ist];
          if (pre) v *= __ldg(pre + pofs + pstr * i);
          v *= dinv(i);
#pragma unroll
          for (int k = 0; k < BAND; ++k) {
            const int j = i - BAND + k;
            if (j >= 0) v = fma(-coef(i, k), Tr[j * ist], v);
          }
          Tr[i * ist] = v;
        }
      }
      if (ua.prefetch == 2) prefetch_next();
      // ---------------- backward ----------------
      auto load_b = [&](Buf& bf, int h) {
#pragma unroll
        for (int u = 0; u < G; ++u) {
          const int j = h * G + G - 1 - u;
          load_c(bf, j, u);
          if (M1 && (BAND & 1) == 0) {  // rows j - BAND, j - BAND - 1 from one 16-byte load (j odd at even u)
            if ((u & 1) == 0) {
              const double2 v = *reinterpret_cast<const double2*>(Tr + max(j - 1 - BAND, 0));
              bf.x[u] = v.y;
              bf.x[u + 1] = v.x;
            }
          } else {
            bf.x[u] = Tr[max(j - BAND, 0) * ist];
          }
        }
        load_e(bf, h, true);
      };
      double ab[BAND];
      double ohi = 0.0;
      auto step_b = [&](const Buf& bf, int h) {
#pragma unroll
        for (int u = 0; u < G; ++u) {
          const int j = h * G + G - 1 - u;
          auto cb_ = [&](int k) { return bf.c[u][k]; };
          const double rj = ab[0];
#pragma unroll
          for (int m = 1; m < BAND; ++m) ab[m - 1] = fma(-cb_(BAND - m), rj, ab[m]);
          ab[BAND - 1] = fma(-cb_(0), rj, bf.x[u]);
          double o = rj * cb_(BAND);
          if (post) o *= __ldg(post + pofs + pstr * j);
          if (M1) {  // (j, j + 1) written together at the odd step u (j even)
            if (u & 1) *reinterpret_cast<double2*>(Tr + j) = make_double2(o, ohi);
            ohi = o;
          } else {
            Tr[j * ist] = o;
          }
        }
      };
      // groups h1-1 .. h0, descending
      auto run_b = [&](int h0, int h1) {
        load_b(A, h1 - 1);
        load_b(B, max(h1 - 2, 0));
        int h = h1 - 1;
        for (; h - 2 >= h0; h -= 3) {
          load_b(C, h - 2);
          step_b(A, h);
          load_b(A, max(h - 3, 0));
          step_b(B, h - 1);
          load_b(B, max(h - 4, 0));
          step_b(C, h - 2);
        }
        if (h >= h0) step_b(A, h);
        if (h - 1 >= h0) step_b(B, h - 1);
      };
      {
#pragma unroll
        for (int m = 0; m < BAND; ++m) ab[m] = Tr[(n - 1 - m) * ist];
        run_b(0, ng);
      }
    }
    // generic-proxy smem writes -> visible to the bulk-copy (async) proxy, then the stores
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (M1) {
      if (lane < nf) k3_bulk_store(mm.out + gbase, tb + (unsigned)(lane * ua.NP * 8), (unsigned)n * 8);
    } else if (lane == 0) {
      for (int k = 0; k < ua.nbox; ++k)
        k3_map_store(&map_out, tb + (unsigned)(k * ua.boxn * F * 8), p0, k * ua.boxn, q, bi);
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // the tile is free for the next load
    __syncwarp();
  }
}

inline int utile_mode() {  // FDP_K3_U: 0 off, 1 mode 1 only, 2 every mode (default)
  static const int v = [] {
    const char* e = std::getenv("FDP_K3_U");
    return e ? std::atoi(e) : 2;
  }();
  return v;
}
inline int sm_count() {
  static const int v = [] {
    int dev = 0, c = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      c = 148;
    return c > 0 ? c : 148;
  }();
  return v;
}
inline UArgs utile_args(const MassMode& m) {
  UArgs ua{};
  const int cs = mass_coef_stride(m.band);
  ua.NP = tile_np(m.n);
  ua.nbox = (m.n + 255) / 256;
  ua.boxn = ((m.n + ua.nbox - 1) / ua.nbox + 7) / 8 * 8;
  const long long td = m.P == 1 ? (long long)kUF * ua.NP : (long long)kUF * ua.boxn * ua.nbox;
  ua.tile_d = (int)((td + 15) / 16 * 16);
  ua.tab_d = (m.n * ((m.band & 1) ? cs : m.band + 1) + 15) / 16 * 16;
  static const int pf = [] {  // FDP_K3_NO_PF=1: off; FDP_K3_PF=1: at load time (diagnostics)
    if (std::getenv("FDP_K3_NO_PF")) return 0;
    const char* e = std::getenv("FDP_K3_PF");
    return e ? std::atoi(e) : 2;
  }();
  ua.prefetch = pf;
  ua.tiles = m.P == 1 ? ((long long)m.Q * m.batch + kUF - 1) / kUF
                      : ((long long)m.P + kUF - 1) / kUF * m.Q * m.batch;
  return ua;
}
inline bool utile_ok(const MassMode& m) {
  static const bool sweep = std::getenv("FDP_K3_SWEEP") != nullptr;
  const int um = utile_mode();
  if (m.forward || !m.cf || sweep || um < 1 || m.band < 1 || m.band > 5) return false;
  if (m.P != 1 && um < 2) return false;
  if ((m.n & 3) || m.n < 16 || m.n > (1 << 16)) return false;
  const bool a16 = ((reinterpret_cast<uintptr_t>(m.in) | reinterpret_cast<uintptr_t>(m.out)) & 15) == 0;
  if (!a16 || (m.batch > 1 && (m.bs & 1))) return false;
  if (m.P != 1 && (m.P & 1)) return false;
  const UArgs ua = utile_args(m);
  if (ua.tiles < 1 || ua.tiles >= (1LL << 31) * kUF) return false;
  return ((size_t)ua.tab_d + (size_t)kUWarps * ua.tile_d) * 8 <= (size_t)kTileMaxSmem;
}

template <int BAND>
cudaError_t launch_utile(const MassMode& m, cudaStream_t s) {
  if constexpr (BAND >= 1 && BAND <= 5) {
    const UArgs ua = utile_args(m);
    const size_t smem = ((size_t)ua.tab_d + (size_t)kUWarps * ua.tile_d) * 8;
    const bool m1 = m.P == 1;
    CUtensorMap map_in, map_out;
    std::memset(&map_in, 0, sizeof(map_in));
    std::memset(&map_out, 0, sizeof(map_out));
    if (!m1 && (!mass_tile_map(&map_in, m.in, m.P, m.n, m.Q, m.batch, m.bs, kUF, ua.boxn) ||
                !mass_tile_map(&map_out, m.out, m.P, m.n, m.Q, m.batch, m.bs, kUF, ua.boxn)))
      return cudaErrorNotSupported;
    const bool sc = m.pre || m.post;
    auto kern = m1 ? (sc ? mass_utile_kernel<BAND, true, true> : mass_utile_kernel<BAND, true, false>)
                   : (sc ? mass_utile_kernel<BAND, false, true> : mass_utile_kernel<BAND, false, false>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    const long long ctas = std::min<long long>(sm_count(), (ua.tiles + kUWarps - 1) / kUWarps);
    kern<<<(unsigned)ctas, kUWarps * 32, smem, s>>>(m, map_in, map_out, ua);
    return cudaGetLastError();
  }
  return cudaErrorNotSupported;
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
  if (m.forward) {
    mass_forward_kernel<BAND><<<(unsigned)blocks, threads, 0, s>>>(m);
  } else if (utile_ok(m) && launch_utile<BAND>(m, s) != cudaErrorNotSupported) {
    // K3u launched (or failed to launch: the error is read below)
  } else if (tile_ok(m) && launch_tile_b<BAND>(m, s) != cudaErrorNotSupported) {
    // K3t launched (or failed to launch: the error is read below)
  } else if (m.P == 1) {
    const long long warps = (nf + 31) / 32;
    mass_solve_mode1_kernel<BAND><<<(unsigned)((warps + kM1Warps - 1) / kM1Warps), kM1Warps * 32, 0, s>>>(m);
  } else {
    mass_solve_kernel<BAND, 8><<<(unsigned)blocks, threads, 0, s>>>(m);
  }
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
