// Slab-decomposition pack / unpack: the transposes around the mode-3
// contraction when the i3 axis is partitioned over G ranks. Streaming, HBM-bound (16 B/element).
//
// z-slab tensor of rank g: (n1, n2, nz) with i1 fastest. Piece for rank h: the i2-range
// [y0_h, y1_h) of every local plane, laid out [i3 local][i2 - y0_h][i1], stored at offset
// n1 * nz * y0_h of the send buffer. Received pieces concatenated in rank order then form the
// y-slab tensor (n1, ny, n3) of the receiver without any further copy (the source's planes are
// contiguous there), which is why only the z-slab side needs this kernel.
#include "../fdp_internal.h"

namespace fdp {
namespace {

__device__ __forceinline__ void part(long long n, int G, int r, long long& lo, long long& len) {
  const long long q = n / G, rem = n % G;
  lo = r * q + (r < rem ? r : rem);
  len = q + (r < rem ? 1 : 0);
}

// dir 0: pack (slab -> pieces), dir 1: unpack (pieces -> slab)
__global__ void slab_copy_kernel(const double* __restrict__ src, double* __restrict__ dst, int n1,
                                 int n2, int nz, int G, int dir, const double* __restrict__ scale) {
  const long long total = (long long)n1 * n2 * nz;
  const long long q = n2 / G, rem = n2 % G;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i1 = (int)(e % n1);
    const long long r = e / n1;
    const int i2 = (int)(r % n2);
    const int i3 = (int)(r / n2);
    // owner rank of i2 under the even split (first rem ranks hold q+1)
    int h;
    if (i2 < rem * (q + 1)) h = (int)(i2 / (q + 1));
    else h = (int)(rem + (i2 - rem * (q + 1)) / q);
    long long y0, ny;
    part(n2, G, h, y0, ny);
    const long long po = (long long)n1 * nz * y0 + i1 + (long long)n1 * ((i2 - y0) + ny * i3);
    if (dir == 0) {
      dst[po] = src[e];
    } else {
      double v = src[po];
      if (scale) v *= scale[e];
      dst[e] = v;
    }
  }
}

__global__ void slab_scatter_kernel(const double* __restrict__ src, const ScatterDesc sd, int nq,
                                    int a_outer) {
  const long long total = (long long)sd.n1 * sd.na * nq;
  const int G = sd.G, na = sd.na;
  const int qd = na / G, rem = na % G;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i1 = (int)(e % sd.n1);
    const long long t = e / sd.n1;
    int a, q;
    if (a_outer) {
      q = (int)(t % nq);
      a = (int)(t / nq);
    } else {
      a = (int)(t % na);
      q = (int)(t / na);
    }
    const int o = (qd == 0 || a < rem * (qd + 1)) ? a / (qd + 1) : rem + (a - rem * (qd + 1)) / qd;
    const int lo = o * qd + (o < rem ? o : rem);
    const int len = qd + (o < rem ? 1 : 0);
    sd.peers[o][i1 + (long long)sd.n1 * ((long long)(a - lo) * (sd.a0 + sd.a1 * len) +
                                         (long long)(q + sd.qoff) * (sd.q0 + sd.q1 * len))] = src[e];
  }
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void peer_barrier_kernel(unsigned long long* const* flags, unsigned long long* counter,
                                    int G, int rank) {
  const int lane = threadIdx.x;
  unsigned long long epoch = 0;
  if (lane == 0) {
    epoch = *counter + 1;
    *counter = epoch;
  }
  epoch = __shfl_sync(0xffffffffu, epoch, 0);
  __threadfence_system();  // this rank's earlier peer stores (previous kernels) before the signal
  if (lane < G) st_release_sys(flags[lane] + rank, epoch);
  if (lane < G) {
    const unsigned long long* mine = flags[rank] + lane;
    while (ld_acquire_sys(mine) < epoch) {
    }
  }
  __syncwarp();
  __threadfence_system();
}

}  // namespace

cudaError_t launch_slab_scatter(const double* src, const ScatterDesc& sd, int nq, int a_outer,
                                cudaStream_t s) {
  const long long total = (long long)sd.n1 * sd.na * nq;
  if (total == 0) return cudaSuccess;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  slab_scatter_kernel<<<blocks, 256, 0, s>>>(src, sd, nq, a_outer);
  return cudaGetLastError();
}

cudaError_t launch_peer_barrier(unsigned long long* const* flags, unsigned long long* counter,
                                int G, int rank, cudaStream_t s) {
  if (G < 1 || G > 32) return cudaErrorInvalidValue;
  peer_barrier_kernel<<<1, 32, 0, s>>>(flags, counter, G, rank);
  return cudaGetLastError();
}

cudaError_t launch_slab_copy(const double* src, double* dst, int n1, int n2, int nz, int G, int dir,
                             const double* scale, cudaStream_t s) {
  const long long total = (long long)n1 * n2 * nz;
  if (total == 0) return cudaSuccess;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  slab_copy_kernel<<<blocks, 256, 0, s>>>(src, dst, n1, n2, nz, G, dir, scale);
  return cudaGetLastError();
}

}  // namespace fdp
