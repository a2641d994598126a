// K1p: the middle of Algorithm 1 one plane at a time, D = 3.
//
// After the mode-1 forward pass has written its output plane-major (plane a1 = the n2 x n3 slice
// of fixed spectral index a1, contiguous, i2 fastest; TIO_OUT_T), every remaining step before the
// mode-1 backward pass acts inside one such plane:
//     mode-2 forward  x_2 U_2^T      rows = i3 lines of the plane
//     mode-3 forward  x_3 U_3^T      rows = a2 columns, then the division by
//                                    Lambda = lambda_1[a1] + lambda_2[a2] + lambda_3[a3],
//     mode-3 backward x_3 U_3        then this backward transform (same columns, same warp)
//     mode-2 backward x_2 U_2        rows = i3 lines
// so one CTA loads a plane into shared memory once, runs the four folded contractions
// (tile_compute_store_fold's arithmetic) in place with a CTA barrier between the
// row and column steps, and writes the plane back: one launch instead of three, and the plane's
// 4 contractions never leave the SM. The P_Q passes of modes 2 and 3 (dense centrosymmetric
// M_d^{-1}, FOLD_SYM) ride along as planes of kind 1, whose result is stored in the
// natural layout (i1 fastest) with the P^G scaling D_Q^{-1/2}.
//
// Shared memory: the folded forward matrices of modes 2 and 3 (E | O blocks, row stride SBF) and
// the plane (row stride SP == 4 mod 16 doubles: the 8x4 A-fragment reads of both the row and the
// column steps are bank-conflict free). 8 warps per CTA, two CTAs per SM at n <= 68.
#include "../fdp_internal.h"

namespace fdp {
namespace {

constexpr int PW = 8;
constexpr int PTH = PW * 32;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int NT>
struct PS {
  static constexpr int NTE = NT / 2;
  static constexpr int KPF = 4 * NT;                       // rows of one folded block (8 NTE)
  static constexpr int SBF = ((KPF + 15) / 16) * 16 + 4;  // W row stride
  static constexpr int WB = 2 * KPF * SBF;                 // one folded matrix (E | O)
};

enum PlaneStep : int { PT_FWD = 0, PT_FUSED = 1, PT_BWDT = 2, PT_SYM = 3 };

// One 8-row tile of a folded contraction over the shared-memory plane, in place. Row r of the
// tile, element k at Pl[r * rs + k * ks]; n = contracted extent; rows >= nrows are computed on
// whatever the buffer holds and never written. W: folded forward (or FOLD_SYM) matrix in shared
// memory, block O at W + KPF * SBF.
//   PT_FWD:   y_E = W_E^T s, y_O = W_O^T d            -> spectral [E | O] along k
//   PT_FUSED: PT_FWD, / (lrow + lamcol[a]), then the backward transform with W read transposed
//   PT_BWDT:  backward transform, W read transposed    -> spatial along k
//   PT_SYM:   e = W_E^T s, o = W_O^T d, output butterfly (y = A x, A centrosymmetric)
template <int NT, int MT>
__device__ __noinline__ void plane_tile(double* Pl, int rs, int ks, int r0, int nrows, int n,
                                           const double* W, int step, double lbase,
                                           const double* lrowv, const double* lamcol, int lane) {
  // MT row tiles of 8 per warp share every B fragment (MT = 2: half the B loads per DMMA and two
  // independent accumulator chains per fragment)
  using S = PS<NT>;
  constexpr int NTE = S::NTE, SBF = S::SBF;
  const double* WO = W + S::KPF * SBF;
  const int ne = (n + 1) >> 1, no = n >> 1;
  const bool full_o = ((no + 7) >> 3) == NTE;
  const int fr = lane >> 2, fc = lane & 3;
  double* Ar[MT];
  bool rv[MT];
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int r = r0 + 8 * i + fr;
    rv[i] = r < nrows;
    Ar[i] = Pl + (long long)r * rs;
  }
  double ae[MT][NTE][2], ao[MT][NTE][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NTE; ++j) ae[i][j][0] = ae[i][j][1] = ao[i][j][0] = ao[i][j][1] = 0.0;

  if (step != PT_BWDT) {
    const int k4n = (ne + 3) >> 2;
    // running pointers: x_k and x_{n-1-k} of each row, the k-th rows of W_E / W_O
    const double* px0[MT];
    const double* px1[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      px0[i] = Ar[i] + fc * ks;
      px1[i] = Ar[i] + (n - 1 - fc) * ks;
    }
    const double* pwe = W + fc * SBF + fr;
    const double* pwo = WO + fc * SBF + fr;
    const int kstep = 4 * ks;
#pragma unroll 2
    for (int k4 = 0; k4 < k4n; ++k4) {
      double sv[MT], dv[MT];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const double x0 = *px0[i], x1 = *px1[i];
        px0[i] += kstep;
        px1[i] -= kstep;
        sv[i] = x0 + x1;
        dv[i] = x0 - x1;
      }
      double be[NTE], bo[NTE];
#pragma unroll
      for (int j = 0; j < NTE; ++j) {
        be[j] = pwe[8 * j];
        bo[j] = pwo[8 * j];
      }
      pwe += 4 * SBF;
      pwo += 4 * SBF;
#pragma unroll
      for (int j = 0; j < NTE; ++j)
#pragma unroll
        for (int i = 0; i < MT; ++i) dmma(ae[i][j], sv[i], be[j]);
#pragma unroll
      for (int j = 0; j < NTE; ++j)
        if (j < NTE - 1 || full_o)
#pragma unroll
          for (int i = 0; i < MT; ++i) dmma(ao[i][j], dv[i], bo[j]);
    }
    __syncwarp();
    if (step == PT_FWD || step == PT_FUSED) {
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        if (!rv[i]) continue;
        const double lrow = step == PT_FUSED ? lbase + lrowv[r0 + 8 * i + fr] : 0.0;
#pragma unroll
        for (int j = 0; j < NTE; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int a = 8 * j + 2 * fc + h;
            if (a < ne) Ar[i][a * ks] = step == PT_FUSED ? fdp_div(ae[i][j][h], lrow + lamcol[a]) : ae[i][j][h];
            if (a < no) Ar[i][(ne + a) * ks] = step == PT_FUSED ? fdp_div(ao[i][j][h], lrow + lamcol[ne + a]) : ao[i][j][h];
          }
      }
      __syncwarp();
      if (step == PT_FWD) return;
    }
  }
  if (step != PT_SYM) {
    // backward from the spectral row: e over [0, ne), o over [ne, n); W_f read transposed
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NTE; ++j) ae[i][j][0] = ae[i][j][1] = ao[i][j][0] = ao[i][j][1] = 0.0;
    {
      const int k4n = (ne + 3) >> 2;
#pragma unroll 2
      for (int k4 = 0; k4 < k4n; ++k4) {
        const int k = 4 * k4 + fc;
        double a[MT];
#pragma unroll
        for (int i = 0; i < MT; ++i) a[i] = k < n ? Ar[i][k * ks] : 0.0;
        double b[NTE];
#pragma unroll
        for (int j = 0; j < NTE; ++j) b[j] = W[(8 * j + fr) * SBF + k];
#pragma unroll
        for (int j = 0; j < NTE; ++j)
#pragma unroll
          for (int i = 0; i < MT; ++i) dmma(ae[i][j], a[i], b[j]);
      }
    }
    {
      const int k4n = (no + 3) >> 2;
#pragma unroll 2
      for (int k4 = 0; k4 < k4n; ++k4) {
        const int k = 4 * k4 + fc;
        double a[MT];
#pragma unroll
        for (int i = 0; i < MT; ++i) a[i] = ne + k < n ? Ar[i][(ne + k) * ks] : 0.0;
        double b[NTE];
#pragma unroll
        for (int j = 0; j < NTE; ++j) b[j] = WO[(8 * j + fr) * SBF + k];
#pragma unroll
        for (int j = 0; j < NTE; ++j)
          if (j < NTE - 1 || full_o)
#pragma unroll
            for (int i = 0; i < MT; ++i) dmma(ao[i][j], a[i], b[j]);
      }
    }
    __syncwarp();
  }
  // x_c = e_c + o_c, x_{n-1-c} = e_c - o_c; the transposed forward matrix halves the middle row
  // of an odd n (undone here)
  const bool mid2 = step != PT_SYM && (n & 1);
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    if (!rv[i]) continue;
#pragma unroll
    for (int j = 0; j < NTE; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 8 * j + 2 * fc + h;
        if (c < ne) {
          const double e = (mid2 && c == no) ? 2.0 * ae[i][j][h] : ae[i][j][h];
          Ar[i][c * ks] = e + ao[i][j][h];
          Ar[i][(n - 1 - c) * ks] = e - ao[i][j][h];
        }
      }
  }
  __syncwarp();
}

// One leftover row (the rows past the last full 8-row tile) of a plane step on the FP64 FMA pipe,
// by one warp: the same folded arithmetic as plane_tile, lanes over the output index, each dot
// product split over four independent accumulators (the k loop is latency-bound otherwise).
template <int NT>
__device__ __forceinline__ double dot4(const double* w, int wstride, const double* x, int xstride,
                                       int len) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int k = 0;
  for (; k + 4 <= len; k += 4) {
    s0 = fma(w[k * wstride], x[k * xstride], s0);
    s1 = fma(w[(k + 1) * wstride], x[(k + 1) * xstride], s1);
    s2 = fma(w[(k + 2) * wstride], x[(k + 2) * xstride], s2);
    s3 = fma(w[(k + 3) * wstride], x[(k + 3) * xstride], s3);
  }
  for (; k < len; ++k) s0 = fma(w[k * wstride], x[k * xstride], s0);
  return (s0 + s1) + (s2 + s3);
}

template <int NT>
__device__ __noinline__ void plane_row(double* Pl, int rs, int ks, int r, int n, const double* W,
                                          int step, double lbase, const double* lrowv,
                                          const double* lamcol, double* scratch, int lane) {
  using S = PS<NT>;
  constexpr int SBF = S::SBF;
  const double* WO = W + S::KPF * SBF;
  const int ne = (n + 1) >> 1, no = n >> 1;
  double* Ar = Pl + (long long)r * rs;
  double* sv = scratch;        // s (ne) then d (no): the butterflies of the row, contiguous
  double* dv = scratch + 48;
  constexpr int MAXJ = 2;  // ne <= 48: at most two outputs per lane
  double e[MAXJ], o[MAXJ];
  if (step != PT_BWDT) {
    for (int k = lane; k < ne; k += 32) {
      const double x0 = Ar[k * ks], x1 = Ar[(n - 1 - k) * ks];
      sv[k] = x0 + x1;
      if (k < no) dv[k] = x0 - x1;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < MAXJ; ++q) {
      const int a = lane + 32 * q;
      e[q] = a < ne ? dot4<NT>(W + a, SBF, sv, 1, ne) : 0.0;
      o[q] = a < no ? dot4<NT>(WO + a, SBF, dv, 1, no) : 0.0;
    }
    __syncwarp();
    if (step == PT_FWD || step == PT_FUSED) {
      const double lrow = step == PT_FUSED ? lbase + lrowv[r] : 0.0;
#pragma unroll
      for (int q = 0; q < MAXJ; ++q) {
        const int a = lane + 32 * q;
        if (a < ne) Ar[a * ks] = step == PT_FUSED ? fdp_div(e[q], lrow + lamcol[a]) : e[q];
        if (a < no) Ar[(ne + a) * ks] = step == PT_FUSED ? fdp_div(o[q], lrow + lamcol[ne + a]) : o[q];
      }
      __syncwarp();
      if (step == PT_FWD) return;
    }
  }
  if (step != PT_SYM) {  // backward, W_f read transposed (row c of W against the spectral row)
    for (int k = lane; k < n; k += 32) sv[k] = Ar[k * ks];
    __syncwarp();
#pragma unroll
    for (int q = 0; q < MAXJ; ++q) {
      const int c = lane + 32 * q;
      e[q] = c < ne ? dot4<NT>(W + c * SBF, 1, sv, 1, ne) : 0.0;
      o[q] = c < no ? dot4<NT>(WO + c * SBF, 1, sv + ne, 1, no) : 0.0;
    }
    __syncwarp();
  }
  const bool mid2 = step != PT_SYM && (n & 1);
#pragma unroll
  for (int q = 0; q < MAXJ; ++q) {
    const int c = lane + 32 * q;
    if (c < ne) {
      const double ev = (mid2 && c == no) ? 2.0 * e[q] : e[q];
      const double ov = c < no ? o[q] : 0.0;
      Ar[c * ks] = ev + ov;
      Ar[(n - 1 - c) * ks] = ev - ov;
    }
  }
  __syncwarp();
}

template <int NT>
__device__ __forceinline__ void plane_step(double* Pl, int rs, int ks, int nrows, int n,
                                           const double* W, int step, double lbase,
                                           const double* lrowv, const double* lamcol,
                                           double* scratch, int warp, int lane) {
  // 16-row tiles over the full 8-row tiles (an odd last one masked to its 8 rows), the leftover
  // rows (nrows % 8) on the FMA pipe by the warps without a tile
  const int full = nrows >> 3;
  const int t16 = (full + 1) >> 1;
  int first;
  for (int t = warp; t < t16; t += PW)
    plane_tile<NT, 2>(Pl, rs, ks, 16 * t, 8 * full, n, W, step, lbase, lrowv, lamcol, lane);
  first = t16 % PW;
  for (int r = 8 * full + ((warp + PW - first) % PW); r < nrows; r += PW)
    plane_row<NT>(Pl, rs, ks, r, n, W, step, lbase, lrowv, lamcol, scratch + warp * 96, lane);
}

template <int NT>
__global__ void __launch_bounds__(PTH, 2) mode_plane_kernel(const __grid_constant__ PlaneGroup grp) {
  using S = PS<NT>;
  extern __shared__ __align__(16) double sm[];
  double* W2 = sm;
  double* W3 = sm + S::WB;
  double* Sc = sm + 2 * S::WB;        // per-warp scratch rows of the leftover-row path (96 each)
  double* Lm = Sc + PW * 96;          // lambda_1 | lambda_2 | lambda_3 of the current problem
  double* Pl = Lm + 3 * 96;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int CPR = S::KPF / 2;  // 16-byte chunks per W row (8 NTE doubles)

  // the eigenvalues next to W (a cold-L2 apply otherwise pays an HBM round trip per warp in the
  // Lambda epilogue)
  auto load_lam = [&](const PlaneProb& pb) {
    if (pb.kind != 0 && pb.kind != 2) return;
    if (pb.lam1)
      for (int i = tid; i < pb.n1; i += PTH) cp_async8(&Lm[i], pb.lam1 + i);
    for (int i = tid; i < pb.n2; i += PTH) cp_async8(&Lm[96 + i], pb.lam2 + i);
    for (int i = tid; i < pb.n3; i += PTH) cp_async8(&Lm[192 + i], pb.lam3 + i);
  };
  auto load_w = [&](const PlaneProb& pb) {
    load_lam(pb);
    for (int c = tid; c < 2 * S::KPF * CPR; c += PTH) {
      const int rr = c / CPR, cc = (c % CPR) * 2;
      const int g2 = rr < S::KPF ? rr : pb.foldh2 + (rr - S::KPF);
      const int g3 = rr < S::KPF ? rr : pb.foldh3 + (rr - S::KPF);
      cp_async16(&W2[rr * S::SBF + cc], pb.W2 + (size_t)g2 * pb.ldw2 + cc);
      cp_async16(&W3[rr * S::SBF + cc], pb.W3 + (size_t)g3 * pb.ldw3 + cc);
    }
  };
  auto prob_of = [&](int gp) {
    int pi = 0;
    for (int i = 1; i < grp.count; ++i)
      if (gp >= grp.prob[i].plane_begin) pi = i;
    return pi;
  };

  unsigned long long* tr = (grp.trace && tid == 0) ? grp.trace + (size_t)blockIdx.x * 8 : nullptr;
  if (tr) tr[0] = gtimer();
  int cur = -1;
  if ((int)blockIdx.x < grp.total) {  // W of the first plane: independent of the previous kernel
    cur = prob_of(blockIdx.x);
    load_w(grp.prob[cur]);
    commit();
  }
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (tr) tr[1] = gtimer();

  for (int gp = blockIdx.x; gp < grp.total; gp += gridDim.x) {
    if (gp != (int)blockIdx.x) tr = nullptr;
    const int pi = prob_of(gp);
    const PlaneProb& pb = grp.prob[pi];
    if (pi != cur) {
      load_w(pb);
      commit();
      cur = pi;
    }
    const int n1 = pb.n1, n2 = pb.n2, n3 = pb.n3, sp = pb.sp;
    const int Mi = n2 * n3;
    const int local = gp - pb.plane_begin;
    const int a1 = local % n1, b = local / n1;
    const bool d2 = pb.kind >= 2;  // D = 2: natural-layout input, optional pre-scaling
    const double* src = d2 ? pb.X + pb.xbs * (long long)b
                           : pb.T + pb.tbs * (long long)b + (long long)a1 * pb.pstride;
    if (d2 && pb.pre) {
      for (int e = tid; e < Mi; e += PTH) {
        const int i3 = e / n2, i2 = e - i3 * n2;
        Pl[i3 * sp + i2] = __ldg(src + e) * __ldg(pb.pre + e);
      }
    } else {
      for (int e = tid; e < Mi; e += PTH) {
        const int i3 = e / n2, i2 = e - i3 * n2;
        cp_async8(&Pl[i3 * sp + i2], src + e);
      }
    }
    commit();
    wait_all();
    __syncthreads();
    if (tr) tr[2] = gtimer();

    const bool fd = pb.kind == 0 || pb.kind == 2;
    // mode 2 on the i3 rows
    plane_step<NT>(Pl, sp, 1, n3, n2, W2, fd ? PT_FWD : PT_SYM, 0.0, nullptr, nullptr, Sc, warp, lane);
    __syncthreads();
    if (tr) tr[3] = gtimer();
    // mode 3 on the a2 columns (FD: forward, Lambda, backward; D = 2: Lambda = lambda_1[row]
    // + lambda_2[column], no plane term)
    const double lb = pb.kind == 0 ? Lm[a1] : 0.0;
    plane_step<NT>(Pl, 1, sp, n2, n3, W3, fd ? PT_FUSED : PT_SYM, lb, Lm + 96, Lm + 192, Sc, warp, lane);
    __syncthreads();
    if (tr) tr[4] = gtimer();
    if (fd) {  // mode-2 backward on the i3 rows
      plane_step<NT>(Pl, sp, 1, n3, n2, W2, PT_BWDT, 0.0, nullptr, nullptr, Sc, warp, lane);
      __syncthreads();
      if (tr) tr[5] = gtimer();
    }
    if (d2) {  // D = 2: natural-layout output, optional post-scaling
      double* dst = pb.Y + pb.ybs * (long long)b;
      for (int e = tid; e < Mi; e += PTH) {
        const int i3 = e / n2, i2 = e - i3 * n2;
        const double v = Pl[i3 * sp + i2];
        dst[e] = pb.scale ? v * __ldg(pb.scale + e) : v;
      }
    } else if (fd) {
      double* dst = pb.T + pb.tbs * (long long)b + (long long)a1 * pb.pstride;  // in place
      for (int e = tid; e < Mi; e += PTH) {
        const int i3 = e / n2, i2 = e - i3 * n2;
        dst[e] = Pl[i3 * sp + i2];
      }
    } else {  // P_Q result in the natural layout (i1 = a1 fastest), optional D_Q^{-1/2}
      double* dst = pb.Y + pb.ybs * (long long)b;
      for (int e = tid; e < Mi; e += PTH) {
        const int i3 = e / n2, i2 = e - i3 * n2;
        const long long o = a1 + (long long)n1 * e;
        const double v = Pl[i3 * sp + i2];
        dst[o] = pb.scale ? v * pb.scale[o] : v;
      }
    }
    __syncthreads();  // the plane buffer is refilled next
    if (tr) {
      tr[6] = gtimer();
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      tr[7] = ((unsigned long long)pb.kind << 32) | ((unsigned long long)smid << 16) | (unsigned)gp;
    }
  }
  wait_all();
}

template <int NT>
cudaError_t launch_p(const PlaneGroup* g, size_t smem, cudaStream_t s) {
  if (!g)
    return cudaFuncSetAttribute(mode_plane_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g->grid);
  cfg.blockDim = dim3(PTH);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, mode_plane_kernel<NT>, *g);
}

cudaError_t dispatch_p(const PlaneGroup* g, int NT, size_t smem, cudaStream_t s) {
  switch (NT) {
    case 2: return launch_p<2>(g, smem, s);
    case 4: return launch_p<4>(g, smem, s);
    case 6: return launch_p<6>(g, smem, s);
    case 8: return launch_p<8>(g, smem, s);
    case 10: return launch_p<10>(g, smem, s);
    case 12: return launch_p<12>(g, smem, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

size_t plane_smem_bytes(int NT, int sp, int rows) {
  const int KPF = 4 * NT, SBF = ((KPF + 15) / 16) * 16 + 4;
  return sizeof(double) * ((size_t)2 * 2 * KPF * SBF + PW * 96 + 3 * 96 + (size_t)sp * rows);
}

int plane_stride(int n2) {
  int sp = n2;
  while (sp % 16 != 4) ++sp;
  return sp;
}

cudaError_t launch_mode_plane(const PlaneGroup& g, int NT, size_t smem, cudaStream_t s) {
  if (g.total <= 0) return cudaSuccess;
  return dispatch_p(&g, NT, smem, s);
}

cudaError_t prepare_mode_plane(int NT, size_t smem) { return dispatch_p(nullptr, NT, smem, 0); }

}  // namespace fdp
