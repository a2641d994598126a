// K1s: small-n mode contraction (n <= 96) on FP64 tensor cores (mma.sync.m8n8k4.f64 -> DMMA).
//
// Same arithmetic as K1 (Algorithm 1 steps 2-4; m-mode product P:389-398),
// organised for the latency-bound small configs (configs 1-3: n = 32..68, <= 1.3 M dofs):
//   * one persistent CTA per SM (8 warps); the problem's W = U_d (or U_d^T) is loaded into shared
//     memory once per CTA, before griddepcontrol.wait, so it overlaps the previous kernel's tail
//     (programmatic dependent launch);
//   * each warp streams 8-row A panels covering the whole K extent (one cp.async group per panel,
//     double-buffered), computes the 8 x 8*NT output tile with NT independent DMMA accumulators
//     per k4 step, and writes it through the epilogue;
//   * work is balanced at 8-row granularity over all warps of the grid;
//   * EPI_FUSED: mode-D forward contraction, division by Lambda (step 3) and the mode-D
//     backward contraction in one pass: the 8 x n intermediate stays in shared memory and the
//     second GEMM reads U_D^T as a transposed view of the same W tile.
#include "../fdp_internal.h"

namespace fdp {
namespace {

constexpr int SW = 16;          // warps per CTA (4 per SM sub-partition share its DMMA pipe)
constexpr int STH = SW * 32;

__device__ __forceinline__ void cp_async8z(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async16g(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int NT, bool KMAJ>
struct SS {
  static constexpr int BN = 8 * NT;
  static constexpr int KP = ((BN + 15) / 16) * 16;   // >= kpad of any n <= BN
  static constexpr int SB = KP + 4;                  // W row stride (== 4 mod 16)
  static constexpr int SA = KP + 4;                  // [8][SA] panel / fused intermediate
  static constexpr int ABUF = 8 * SA;
  static constexpr int W_ELEMS = KP * SB;
  static constexpr size_t BYTES = sizeof(double) * (W_ELEMS + SW * ABUF);
};

template <int NT, bool KMAJ>
__global__ void __launch_bounds__(STH, 1) mode_small_kernel(const __grid_constant__ ModeGroup grp) {
  using S = SS<NT, KMAJ>;
  extern __shared__ __align__(16) double sm[];
  double* Ws = sm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* A = sm + S::W_ELEMS + warp * S::ABUF;  // this warp's 8-row panel ([8][SA])

  int pi = 0;
#pragma unroll
  for (int i = 1; i < kMaxGroup; ++i)
    if (i < grp.count && (int)blockIdx.x >= grp.prob[i].cta_begin) pi = i;
  const ModeProb& pb = grp.prob[pi];
  const int n = pb.n, P = pb.P, Qn = pb.Q;
  const int Pn = P * n;                       // < 2^31: the host routes only small tensors here
  const int Mi = P * Qn;                      // rows per batch item
  const long long M = (long long)Mi * pb.batch;
  const int kpad = ((n + 15) / 16) * 16;
  const int k4n = (n + 3) / 4;

  unsigned long long* trace = grp.trace ? grp.trace + ((size_t)blockIdx.x * SW + warp) * kTracePhases : nullptr;
  if (trace && lane == 0) trace[0] = gtimer();
  // ---- W (independent of the previous kernel): rows 0..kpad-1, cols 0..BN-1 ----
  {
    const double* W = pb.W;
    const int ldw = pb.ldw;
    // rows needed: kpad for x_d W; the fused second GEMM reads W^T rows up to BN-1 as well
    const int rows = (pb.epi == EPI_FUSED && S::BN > kpad) ? S::BN : kpad;
    const int chunks = rows * (S::BN / 2);
    for (int c = tid; c < chunks; c += STH) {
      const int r = c / (S::BN / 2), cc = (c % (S::BN / 2)) * 2;
      cp_async16g(&Ws[r * S::SB + cc], W + (size_t)r * ldw + cc);
    }
    commit();
  }
  // PDL: everything below may read what the previous kernel wrote.
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (trace && lane == 0) trace[1] = gtimer();

  const double* __restrict__ X = pb.X;
  // tile t -> CTA t % ctas, then warp (t / ctas) % SW: consecutive tiles land on different SMs,
  // so every SM sub-partition gets within one tile of the same DMMA work.
  const int gw = (blockIdx.x - pb.cta_begin) + pb.ctas * warp;
  const int nw = pb.ctas * SW;
  const long long ntiles = pb.tiles_m;

  // element offset of GEMM row m within its batch item, and the item's offset for tensor `bs`
  auto row_index = [&](long long m, int& within, long long& item) {
    const int b = (int)(m / Mi);
    const int mi = (int)(m - (long long)b * Mi);
    if (KMAJ) {
      within = n * mi;                       // P == 1: row = fiber q = mi
    } else {
      const int q = mi / P, p = mi - q * P;
      within = p + Pn * q;
    }
    item = b;
  };

  auto load_panel = [&](long long t) {
    const long long m0 = t * 8;
    if (KMAJ) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const long long m = m0 + r;
        const bool rv = m < M;
        int w = 0;
        long long b = 0;
        if (rv) row_index(m, w, b);
        const double* src = X + (w + pb.xbs * b);
        for (int k = lane; k < kpad; k += 32)
          cp_async8z(&A[r * S::SA + k], rv && k < n ? src + k : X, rv && k < n);
      }
    } else {
      const int r = lane & 7;
      const long long m = m0 + r;
      const bool rv = m < M;
      int w = 0;
      long long b = 0;
      if (rv) row_index(m, w, b);
      const double* src = X + (w + pb.xbs * b);
      for (int k = lane >> 3; k < kpad; k += 4)
        cp_async8z(&A[r * S::SA + k], rv && k < n ? src + (long long)P * k : X, rv && k < n);
    }
    commit();
  };

  const int fr = lane >> 2, fc = lane & 3;
  const bool FUSED = pb.epi == EPI_FUSED;  // uniform per CTA (one problem per CTA)
  wait_group<0>();  // W landed (this thread's part)
  __syncthreads();  // W visible to all warps
  if (trace && lane == 0) trace[2] = gtimer();

  for (long long t = gw; t < ntiles; t += nw) {
    load_panel(t);
    wait_group<0>();
    __syncwarp();
    const bool tr = trace && lane == 0 && t == gw;
    if (tr) trace[3] = gtimer();

    double acc[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;
    for (int k4 = 0; k4 < k4n; ++k4) {
      const int k = 4 * k4 + fc;
      const double a = A[fr * S::SA + k];
      double b[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = Ws[k * S::SB + 8 * j + fr];
#pragma unroll
      for (int j = 0; j < NT; ++j) dmma(acc[j], a, b[j]);
    }

    if (tr) trace[4] = gtimer();
    // row bookkeeping for the output row m = 8t + fr
    const long long m = t * 8 + fr;
    const bool mv = m < M;
    int sidx = 0;
    long long item = 0;
    double lrow = 0.0;
    if (mv) {
      row_index(m, sidx, item);
      if (!KMAJ && (FUSED || pb.epi == EPI_LAMBDA)) {
        const int p = (int)((m - item * Mi) % P);
        lrow = pb.lam1 ? pb.lam0[p % pb.n1] + pb.lam1[p / pb.n1] : pb.lam0[p];
      }
    }

    if (FUSED) {
      // T = acc / Lambda -> this warp's panel buffer ([8][SA]); zero beyond n.
      __syncwarp();
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int a = 8 * j + 2 * fc + h;
          A[fr * S::SA + a] = (mv && a < n) ? acc[j][h] / (lrow + pb.lamcol[a]) : 0.0;
        }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;
      for (int k4 = 0; k4 < k4n; ++k4) {
        const int k = 4 * k4 + fc;
        const double a = A[fr * S::SA + k];
        double b[NT];
#pragma unroll
        for (int j = 0; j < NT; ++j) b[j] = Ws[(8 * j + fr) * S::SB + k];  // (U^T)[k][a] = U[a][k]
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[j], a, b[j]);
      }
    }

    if (mv) {
      double* __restrict__ Y = pb.Y + pb.ybs * item + sidx;
      const int epi = FUSED ? EPI_NONE : pb.epi;
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int a = 8 * j + 2 * fc + h;
          if (a < n) {
            double v = acc[j][h];
            if (epi == EPI_LAMBDA) v = v / (lrow + pb.lamcol[a]);
            else if (epi == EPI_SCALE) v = v * pb.scale[sidx + P * a];
            Y[P * a] = v;
          }
        }
    }
    __syncwarp();  // all lanes done with the panel before it is refilled
    if (tr) trace[5] = gtimer();
  }
}

template <int NT, bool KMAJ>
cudaError_t launch_s(const ModeGroup* g, cudaStream_t s) {
  using S = SS<NT, KMAJ>;
  if (!g)
    return cudaFuncSetAttribute(mode_small_kernel<NT, KMAJ>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::BYTES);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g->total_ctas);
  cfg.blockDim = dim3(STH);
  cfg.dynamicSmemBytes = S::BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, mode_small_kernel<NT, KMAJ>, *g);
}

template <bool KMAJ>
cudaError_t dispatch_small(const ModeGroup* g, int NT, cudaStream_t s) {
  switch (NT) {
    case 1: return launch_s<1, KMAJ>(g, s);
    case 2: return launch_s<2, KMAJ>(g, s);
    case 3: return launch_s<3, KMAJ>(g, s);
    case 4: return launch_s<4, KMAJ>(g, s);
    case 5: return launch_s<5, KMAJ>(g, s);
    case 6: return launch_s<6, KMAJ>(g, s);
    case 7: return launch_s<7, KMAJ>(g, s);
    case 8: return launch_s<8, KMAJ>(g, s);
    case 9: return launch_s<9, KMAJ>(g, s);
    case 10: return launch_s<10, KMAJ>(g, s);
    case 11: return launch_s<11, KMAJ>(g, s);
    case 12: return launch_s<12, KMAJ>(g, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

cudaError_t launch_mode_small(const ModeGroup& g, int NT, bool kmaj, cudaStream_t s) {
  if (g.total_ctas <= 0) return cudaSuccess;
  return kmaj ? dispatch_small<true>(&g, NT, s) : dispatch_small<false>(&g, NT, s);
}

cudaError_t prepare_mode_small(int NT) {
  cudaError_t e;
  if ((e = dispatch_small<true>(nullptr, NT, 0)) != cudaSuccess) return e;
  return dispatch_small<false>(nullptr, NT, 0);
}

}  // namespace fdp
