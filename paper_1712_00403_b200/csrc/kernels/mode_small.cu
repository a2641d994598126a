// K1s: small-n mode contraction (n <= 96) on FP64 tensor cores (mma.sync.m8n8k4.f64 -> DMMA).
//
// Same arithmetic as K1 (Algorithm 1 steps 2-4; m-mode product P:389-398),
// organised for the latency-bound small configs (configs 1-3: n = 32..68, <= 1.3 M dofs):
//   * one persistent CTA per SM (16 warps); the problem's W = U_d (or U_d^T) is loaded into shared
//     memory once per CTA, before griddepcontrol.wait, so it overlaps the previous kernel's tail
//     (programmatic dependent launch);
//   * each warp owns 8-row tiles covering the whole K extent: loads the panel (LDG -> STS),
//     computes the 8 x 8*NT output tile with NT independent DMMA accumulators per k4 step, and
//     writes it through the epilogue; tiles are dealt round-robin over SMs first so every SM
//     sub-partition gets within one tile of the same DMMA work;
//   * EPI_FUSED: mode-D forward contraction, division by Lambda (step 3) and the mode-D
//     backward contraction in one pass: the 8 x n intermediate stays in shared memory and the
//     second GEMM reads U_D^T as a transposed view of the same W tile;
#include <cstdlib>

#include "../fdp_internal.h"

namespace fdp {
namespace {

constexpr int SW = 16;          // warps per CTA (4 per SM sub-partition share its DMMA pipe)
constexpr int STH = SW * 32;

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

template <int NT>
struct SS {
  static constexpr int BN = 8 * NT;
  static constexpr int KP = ((BN + 15) / 16) * 16;   // >= kpad of any n <= BN
  static constexpr int SB = KP + 4;                  // W row stride (== 4 mod 16)
  static constexpr int SA = KP + 4;                  // [8][SA] panel / fused intermediate
  static constexpr int ABUF = 8 * SA;
  static constexpr int W_ELEMS = KP * SB;
  static constexpr size_t BYTES = sizeof(double) * (W_ELEMS + SW * ABUF);
  // folded W (NT = 2 * NTE): blocks E and O of KPF rows x 8*NTE columns, row stride SBF
  static constexpr int KPF = 4 * NT;
  static constexpr int SBF = ((KPF + 15) / 16) * 16 + 4;
  static_assert(2 * KPF * SBF <= W_ELEMS, "folded W must fit the dense W footprint");
};

// Load W (rows 0..rows-1, cols 0..BN-1 of the padded global matrix) into shared memory.
template <int NT>
__device__ __forceinline__ void load_w(double* Ws, const ModeProb& pb, int tid) {
  using S = SS<NT>;
  const int kpad = ((pb.n + 15) / 16) * 16;
  // the fused second GEMM reads W^T rows up to BN-1 as well
  const int rows = (pb.epi == EPI_FUSED && S::BN > kpad) ? S::BN : kpad;
  const int chunks = rows * (S::BN / 2);
  for (int c = tid; c < chunks; c += STH) {
    const int r = c / (S::BN / 2), cc = (c % (S::BN / 2)) * 2;
    cp_async16g(&Ws[r * S::SB + cc], pb.W + (size_t)r * pb.ldw + cc);
  }
  commit();
}

// Folded W: block E = global rows [0, KPF), block O = global rows [foldh, foldh + KPF), columns
// [0, 8*NTE) of each.
template <int NT, int NTHREADS = STH>
__device__ __forceinline__ void load_w_fold(double* Ws, const ModeProb& pb, int tid) {
  using S = SS<NT>;
  constexpr int CPR = S::KPF / 2;  // 16-byte chunks per row (8*NTE doubles)
  for (int c = tid; c < 2 * S::KPF * CPR; c += NTHREADS) {
    const int r = c / CPR, cc = (c % CPR) * 2;
    const int gr = r < S::KPF ? r : pb.foldh + (r - S::KPF);
    cp_async16g(&Ws[r * S::SBF + cc], pb.W + (size_t)gr * pb.ldw + cc);
  }
  commit();
}

// Geometry of one problem, per thread.
struct Geo {
  int n, nout, P, Q, Pn, Pno, Mi, kpad, k4n, nch;
  long long M;
  __device__ explicit Geo(const ModeProb& pb) {
    n = pb.n;
    nout = pb.nout;
    P = pb.P;
    Q = pb.Q;
    Pn = P * n;
    Pno = P * nout;
    Mi = P * Q;
    M = (long long)Mi * pb.batch;
    kpad = ((n + 15) / 16) * 16;
    k4n = (n + 3) / 4;
    nch = (kpad + 31) / 32;
  }
};

// element offset of GEMM row m within its batch item (32-bit: the host routes here only problems
// with M < 2^31) and the batch item index; ld = fiber stride of the tensor (KMAJ)
template <bool KMAJ>
__device__ __forceinline__ void row_index(const Geo& g, int m, int& within, int& item, int ld,
                                          int pn) {
  const unsigned b = (unsigned)m / (unsigned)g.Mi;
  const int mi = m - (int)b * g.Mi;
  if (KMAJ) {
    within = ld * mi;  // P == 1: row = fiber q = mi
  } else {
    const unsigned q = (unsigned)mi / (unsigned)g.P;
    within = (mi - (int)q * g.P) + pn * (int)q;  // pn = P * (extent of the mode in that tensor)
  }
  item = (int)b;
}

template <bool COHERENT>
__device__ __forceinline__ double ldx(const double* p) {
  return COHERENT ? __ldcg(p) : __ldg(p);
}

template <int NT, bool KMAJ, bool SC = false>
__device__ __forceinline__ void tile_compute_store(const ModeProb& pb, const Geo& g,
                                                   const double* Ws, double* A, long long t,
                                                   int lane, unsigned long long* tr);
template <int NT, bool KMAJ, int MT = 1>
__device__ __forceinline__ void tile_compute_store_fold(const ModeProb& pb, const Geo& g,
                                                        const double* Ws, double* A, long long t,
                                                        int lane, unsigned long long* tr);

// One 8-row tile: panel load (LDG -> STS, zero fill beyond n / M), DMMAs, epilogue.
// COHERENT: the input was written earlier in the same launch (plane pipeline): L2-coherent loads.
// Rows 8t .. 8t+7 of the tile's panel into A ([8][SA]; LDG -> STS, zero fill beyond n / M).
template <int NT, bool KMAJ, bool COHERENT>
__device__ __forceinline__ void load_tile_rows(const ModeProb& pb, const Geo& g, double* A,
                                               long long t, int lane) {
  using S = SS<NT>;
  const double* __restrict__ X = pb.X;
  const int m0 = (int)(t * 8);
  if (KMAJ) {
    int mi, b0;
    row_index<true>(g, m0, mi, b0, 1, 0);  // fiber index of the tile's first row
    const double* src[8];
    const double* pre[8];
    bool rv[8];
    const bool scaled = pb.pre != nullptr;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      rv[r] = (long long)m0 + r < g.M;
      src[r] = X + ((long long)pb.xld * mi + pb.xbs * b0);
      pre[r] = scaled ? pb.pre + (long long)pb.xld * mi : nullptr;
      if (++mi == g.Mi) { mi = 0; ++b0; }
    }
    if (pb.vx) {
      // 16-byte loads: rows of an even-stride (padded) tensor; element n of an odd-n row is the
      // zero pad column
      double2 v[2][8];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int k = 64 * c + 2 * lane;
#pragma unroll
        for (int r = 0; r < 8; ++r)
          v[c][r] = (rv[r] && k < g.n) ? (COHERENT ? __ldcg(reinterpret_cast<const double2*>(src[r] + k))
                                                 : __ldg(reinterpret_cast<const double2*>(src[r] + k)))
                                      : make_double2(0.0, 0.0);
        if (scaled) {
#pragma unroll
          for (int r = 0; r < 8; ++r)
            if (rv[r] && k < g.n) {
              const double2 w = __ldg(reinterpret_cast<const double2*>(pre[r] + k));
              v[c][r].x *= w.x;
              v[c][r].y *= (k + 1 < g.n) ? w.y : 0.0;  // the pad column stays 0
            }
        }
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int k = 64 * c + 2 * lane;
        if (k < g.kpad) {
#pragma unroll
          for (int r = 0; r < 8; ++r) *reinterpret_cast<double2*>(&A[r * S::SA + k]) = v[c][r];
        }
      }
    } else {
      double v[3][8];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int k = 32 * c + lane;
#pragma unroll
        for (int r = 0; r < 8; ++r) v[c][r] = (c < g.nch && rv[r] && k < g.n) ? ldx<COHERENT>(src[r] + k) : 0.0;
        if (scaled) {
#pragma unroll
          for (int r = 0; r < 8; ++r)
            if (c < g.nch && rv[r] && k < g.n) v[c][r] *= __ldg(pre[r] + k);
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int k = 32 * c + lane;
        if (c < g.nch && k < g.kpad) {
#pragma unroll
          for (int r = 0; r < 8; ++r) A[r * S::SA + k] = v[c][r];
        }
      }
    }
  } else if (pb.vx) {
    // 16-byte loads of row pairs (p, p+1), p even, of an even-P tensor; lane = (pair, k)
    const int rp = lane & 3, kk = lane >> 2;
    const int m = m0 + 2 * rp;
    const bool rv = (long long)m < g.M;  // M is even here, so the pair is all or nothing
    int w = 0, b = 0;
    if (rv) row_index<false>(g, m, w, b, 0, g.Pn);
    const double* src = X + (w + pb.xbs * b);
    double2 v[12];
#pragma unroll
    for (int j = 0; j < 12; ++j) {
      const int k = kk + 8 * j;
      v[j] = (k < g.n && rv) ? (COHERENT ? __ldcg(reinterpret_cast<const double2*>(src + (long long)g.P * k))
                                         : __ldg(reinterpret_cast<const double2*>(src + (long long)g.P * k)))
                             : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int j = 0; j < 12; ++j) {
      const int k = kk + 8 * j;
      if (k < g.kpad) {
        A[(2 * rp) * S::SA + k] = v[j].x;
        A[(2 * rp + 1) * S::SA + k] = v[j].y;
      }
    }
  } else {
    const int r = lane & 7;
    const int m = m0 + r;
    const bool rv = (long long)m < g.M;
    int w = 0, b = 0;
    if (rv) row_index<false>(g, m, w, b, 0, g.Pn);
    const double* src = X + (w + pb.xbs * b);
    double v[24];
#pragma unroll
    for (int j = 0; j < 24; ++j) {
      const int k = (lane >> 3) + 4 * j;
      v[j] = (k < g.n && rv) ? ldx<COHERENT>(src + (long long)g.P * k) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 24; ++j) {
      const int k = (lane >> 3) + 4 * j;
      if (k < g.kpad) A[r * S::SA + k] = v[j];
    }
  }
}

template <int NT, bool KMAJ, bool COHERENT, bool SC = false, bool FOLD = false>
__device__ __forceinline__ void do_tile(const ModeProb& pb, const Geo& g, const double* Ws,
                                        double* A, long long t, int lane,
                                        unsigned long long* tr) {
  load_tile_rows<NT, KMAJ, COHERENT>(pb, g, A, t, lane);
  __syncwarp();
  if (tr) tr[3] = gtimer();
  if constexpr (FOLD)
    tile_compute_store_fold<NT, KMAJ>(pb, g, Ws, A, t, lane, tr);
  else
    tile_compute_store<NT, KMAJ, SC>(pb, g, Ws, A, t, lane, tr);
}

template <int NT, bool KMAJ, bool SC>
__device__ __forceinline__ void tile_compute_store(const ModeProb& pb, const Geo& g,
                                                   const double* Ws, double* A, long long t,
                                                   int lane, unsigned long long* tr) {
  using S = SS<NT>;
  const int m0 = (int)(t * 8);
  const int fr = lane >> 2, fc = lane & 3;
  double acc[NT][2];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;
  for (int k4 = 0; k4 < g.k4n; ++k4) {
    const int k = 4 * k4 + fc;
    const double a = A[fr * S::SA + k];
    double b[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) b[j] = Ws[k * S::SB + 8 * j + fr];
#pragma unroll
    for (int j = 0; j < NT; ++j) dmma(acc[j], a, b[j]);
  }
  if (tr) tr[4] = gtimer();

  // row bookkeeping for the output row m = 8t + fr
  const int m = m0 + fr;
  const bool mv = (long long)m < g.M;
  const bool FUSED = pb.epi == EPI_FUSED;
  int sidx = 0, item = 0;
  double lrow = 0.0;
  bool pad_row = false;  // padding row (i1 >= n1v) of a padded intermediate: output stays 0
  if (mv) {
    row_index<KMAJ>(g, m, sidx, item, pb.yld, g.Pno);
    if (!KMAJ && (FUSED || pb.epi == EPI_LAMBDA)) {
      const int mi = m - item * g.Mi;
      const int p = mi - (int)((unsigned)mi / (unsigned)g.P) * g.P;
      const unsigned i2 = (unsigned)p / (unsigned)pb.n1;
      const int i1 = p - (int)i2 * pb.n1;
      pad_row = i1 >= pb.n1v;
      if (!pad_row) lrow = pb.lam1 ? pb.lam0[i1] + pb.lam1[i2] : pb.lam0[p];
    }
  }

  if (FUSED) {
    // T = acc / Lambda -> this warp's panel buffer ([8][SA]); zero beyond n and on pad rows.
    __syncwarp();
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = 8 * j + 2 * fc + h;
        A[fr * S::SA + a] = (mv && !pad_row && a < g.n) ? fdp_div(acc[j][h], lrow + pb.lamcol[a]) : 0.0;
      }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;
    for (int k4 = 0; k4 < g.k4n; ++k4) {
      const int k = 4 * k4 + fc;
      const double a = A[fr * S::SA + k];
      double b[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = Ws[(8 * j + fr) * S::SB + k];  // (U^T)[k][a] = U[a][k]
#pragma unroll
      for (int j = 0; j < NT; ++j) dmma(acc[j], a, b[j]);
    }
  }

  // epilogue values (Lambda / scale applied), then stores
  const int epi = FUSED ? EPI_NONE : pb.epi;
  const int ncols = KMAJ ? pb.yld : g.nout;  // padded KMAJ outputs also get their zero pad column
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int a = 8 * j + 2 * fc + h;
      double v = acc[j][h];
      if (epi == EPI_LAMBDA) v = (pad_row || a >= g.n) ? 0.0 : fdp_div(v, lrow + pb.lamcol[a]);
      else if (epi == EPI_SCALE && mv && a < g.n) v = v * pb.scale[sidx + g.P * a];
      acc[j][h] = v;
    }
  double* __restrict__ Y = pb.Y + pb.ybs * (long long)item + sidx;
  if (epi == EPI_AXPBY && mv) {  // kron-operator terms: Y = alpha * result + beta * Y (scalar path)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = 8 * j + 2 * fc + h;
        if (a < ncols) {
          double* yp = Y + (KMAJ ? 1 : g.P) * a;
          *yp = pb.alpha * acc[j][h] + (pb.beta != 0.0 ? pb.beta * *yp : 0.0);
        }
      }
    __syncwarp();
    return;
  }
  if (SC) {  // peer-store scatter of the slab exchange (scalar stores)
    if (mv) {
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int a = 8 * j + 2 * fc + h;
          if (a < g.nout) *scatter_ptr(pb, m, a) = acc[j][h];
        }
    }
  } else if (pb.vy && KMAJ) {
    // (a, a+1) adjacent in a row of an even-stride tensor
    if (mv) {
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int a = 8 * j + 2 * fc;
        if (a < ncols) *reinterpret_cast<double2*>(Y + a) = make_double2(acc[j][0], acc[j][1]);
      }
    }
  } else if (pb.vy) {
    // rows (p, p+1), p even, are adjacent: swap halves with the partner lane (fr ^ 1) and store
    // 16-byte row pairs; even fr stores column c0, odd fr column c0 + 1 of the pair (fr & ~1)
    const bool odd = fr & 1;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const double send = odd ? acc[j][0] : acc[j][1];
      const double got = __shfl_xor_sync(0xffffffffu, send, 4);
      const int c = 8 * j + 2 * fc + (odd ? 1 : 0);
      if (mv && c < ncols) {
        double* dst = odd ? Y - 1 : Y;
        *reinterpret_cast<double2*>(dst + (long long)g.P * c) =
            odd ? make_double2(got, acc[j][1]) : make_double2(acc[j][0], got);
      }
    }
  } else if (mv) {
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = 8 * j + 2 * fc + h;
        if (a < ncols) Y[(KMAJ ? 1 : g.P) * a] = acc[j][h];
      }
  }
  __syncwarp();  // all lanes done with the panel before it is refilled
  if (tr) tr[5] = gtimer();
}


// Even-odd folded transform of one 8-row tile (pb.fold != 0). For a persymmetric
// pencil (J K J = K, J M J = M, J the index reversal) the eigenvectors split into ne = ceil(n/2)
// symmetric and no = floor(n/2) antisymmetric ones, so with s_k = x_k + x_{n-1-k} (k < ne) and
// d_k = x_k - x_{n-1-k} (k < no):
//   forward   y_E = W_E^T s,  y_O = W_O^T d                       (spectral order [E | O])
//   backward  e = W_E y_E, o = W_O y_O;  x_k = e_k + o_k,  x_{n-1-k} = e_k - o_k
// -- the same x as the dense m-mode product of P:389-398 (Algorithm 1 steps 2 and 4)
// in about half the DMMAs. W_E / W_O carry the 1/sqrt(2) normalisation (the middle row of an odd
// n: 1/2 in the forward matrix, 1 in the backward one). FOLD_FUSED (small D-th mode): forward,
// division by Lambda and backward in one pass, the backward reading the forward W
// transposed; its middle output (odd n) is doubled to undo the forward's 1/2. FOLD_SYM: y = A x
// for a centrosymmetric A (the dense M_d^{-1} passes of P_Q): e = W_E^T s,
// o = W_O^T d and the backward's output butterfly.
template <int NT, bool KMAJ, int MT>
__device__ __forceinline__ void tile_compute_store_fold(const ModeProb& pb, const Geo& g,
                                                        const double* Ws, double* A, long long t,
                                                        int lane, unsigned long long* tr) {
  // MT 8-row DMMA tiles per warp (rows 8 MT t .. 8 MT t + 8 MT - 1 of the panel A) share every B
  // fragment
  using S = SS<NT>;
  constexpr int NTE = NT / 2;
  constexpr int SBF = S::SBF;
  const double* WO = Ws + S::KPF * SBF;
  const int n = g.n, ne = (n + 1) >> 1, no = n >> 1;
  const bool full_o = ((no + 7) >> 3) == NTE;  // else the last O tile is empty
  const int m0 = (int)(t * 8 * MT);
  const int fr = lane >> 2, fc = lane & 3;
  const int mode = pb.fold;
  double ae[MT][NTE][2], ao[MT][NTE][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NTE; ++j) ae[i][j][0] = ae[i][j][1] = ao[i][j][0] = ao[i][j][1] = 0.0;

  if (mode != FOLD_BWD) {
    const int k4n = (ne + 3) >> 2;
    for (int k4 = 0; k4 < k4n; ++k4) {
      const int k = 4 * k4 + fc;
      double sv[MT], dv[MT];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const double* Ar = A + (8 * i + fr) * S::SA;
        const double x0 = Ar[k], x1 = Ar[n - 1 - k];  // k <= ne + 2 < n (n >= 8)
        sv[i] = x0 + x1;
        dv[i] = x0 - x1;
      }
      double be[NTE], bo[NTE];
#pragma unroll
      for (int j = 0; j < NTE; ++j) {
        be[j] = Ws[k * SBF + 8 * j + fr];
        bo[j] = WO[k * SBF + 8 * j + fr];
      }
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
  }

  // per row group i: row bookkeeping, then (FUSED) the spectral panel or (FWD) the stores
  int sidx[MT], item[MT];
  bool mv[MT], pad_row[MT];
  double lrow[MT];
  long long cs = KMAJ ? 1 : g.P;
  bool kout = KMAJ;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int m = m0 + 8 * i + fr;
    mv[i] = (long long)m < g.M;
    sidx[i] = item[i] = 0;
    lrow[i] = 0.0;
    pad_row[i] = false;
    if (mv[i]) {
      row_index<KMAJ>(g, m, sidx[i], item[i], pb.yld, g.Pno);
      if (!KMAJ && (mode == FOLD_FUSED || pb.epi == EPI_LAMBDA)) {
        const int mi = m - item[i] * g.Mi;
        const int p = mi - (int)((unsigned)mi / (unsigned)g.P) * g.P;
        const unsigned i2 = (unsigned)p / (unsigned)pb.n1;
        const int i1 = p - (int)i2 * pb.n1;
        pad_row[i] = i1 >= pb.n1v;
        if (!pad_row[i]) lrow[i] = pb.lam1 ? pb.lam0[i1] + pb.lam1[i2] : pb.lam0[p];
      }
      // output addressing: row base sidx, column stride cs; kout = rows contiguous in the output
      if (pb.tio != TIO_NONE) {
        const int mi = m - item[i] * g.Mi;
        if (pb.tio == TIO_OUT_T) { sidx[i] = mi; cs = pb.tio_ld; kout = false; }
        else {
          sidx[i] = pb.yld * mi;
          cs = 1;
          kout = true;
          if (mi >= pb.tio_rows) mv[i] = false;  // the plane-major pad row
        }
      }
    }
  }
  if (pb.tio == TIO_OUT_T) { cs = pb.tio_ld; kout = false; }
  else if (pb.tio == TIO_OUT_K) { cs = 1; kout = true; }
  const bool vrow = !KMAJ && pb.vy && pb.tio == TIO_NONE;  // 16-byte row-pair stores

  if (mode == FOLD_FUSED) {
    // spectral panel [E | O] <- y / Lambda (positions >= n keep the load's zero fill)
    __syncwarp();
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      double* Ar = A + (8 * i + fr) * S::SA;
      const bool ok = mv[i] && !pad_row[i];
#pragma unroll
      for (int j = 0; j < NTE; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int a = 8 * j + 2 * fc + h;
          if (a < ne) Ar[a] = ok ? fdp_div(ae[i][j][h], lrow[i] + pb.lamcol[a]) : 0.0;
          if (a < no) Ar[ne + a] = ok ? fdp_div(ao[i][j][h], lrow[i] + pb.lamcol[ne + a]) : 0.0;
        }
    }
    __syncwarp();
  }

  if (mode == FOLD_FWD) {
    if (tr) tr[4] = gtimer();
    const int ncols = kout ? pb.yld : n;  // row-major rows: their pad columns get their zeros
    const bool lam = pb.epi == EPI_LAMBDA;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      // spectral outputs: E column a -> a, O column a -> ne + a
      double* __restrict__ Y = pb.Y + pb.ybs * (long long)item[i] + sidx[i];
      if (lam) {
#pragma unroll
        for (int j = 0; j < NTE; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int a = 8 * j + 2 * fc + h;
            ae[i][j][h] = (pad_row[i] || a >= ne) ? 0.0 : fdp_div(ae[i][j][h], lrow[i] + pb.lamcol[a]);
            ao[i][j][h] = (pad_row[i] || a >= no) ? 0.0 : fdp_div(ao[i][j][h], lrow[i] + pb.lamcol[ne + a]);
          }
      }
      if (vrow) {
        // rows (p, p+1), p even, adjacent: pair up with the partner lane (fr ^ 1)
        const bool odd = fr & 1;
        double* base = odd ? Y - 1 : Y;
#pragma unroll
        for (int j = 0; j < NTE; ++j) {
          const int c = 8 * j + 2 * fc + (odd ? 1 : 0);
          const double se = odd ? ae[i][j][0] : ae[i][j][1];
          const double ge = __shfl_xor_sync(0xffffffffu, se, 4);
          const double so = odd ? ao[i][j][0] : ao[i][j][1];
          const double go = __shfl_xor_sync(0xffffffffu, so, 4);
          if (mv[i] && c < ne)
            *reinterpret_cast<double2*>(base + (long long)g.P * c) =
                odd ? make_double2(ge, ae[i][j][1]) : make_double2(ae[i][j][0], ge);
          if (mv[i] && c < no)
            *reinterpret_cast<double2*>(base + (long long)g.P * (ne + c)) =
                odd ? make_double2(go, ao[i][j][1]) : make_double2(ao[i][j][0], go);
        }
      } else if (mv[i]) {
#pragma unroll
        for (int j = 0; j < NTE; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int a = 8 * j + 2 * fc + h;
            if (a < ne) Y[cs * a] = ae[i][j][h];
            if (ne + a < ncols && (a < no || kout)) Y[cs * (ne + a)] = ao[i][j][h];
          }
      }
    }
    __syncwarp();
    if (tr) tr[5] = gtimer();
    return;
  }

  // backward: e over the E part of the spectral panel, o over the O part (FOLD_SYM: e and o are
  // the forward-style products already in ae / ao)
  const bool trw = mode == FOLD_FUSED;  // the forward W read transposed
  if (mode != FOLD_SYM) {
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NTE; ++j) ae[i][j][0] = ae[i][j][1] = ao[i][j][0] = ao[i][j][1] = 0.0;
    {
      const int k4n = (ne + 3) >> 2;
      for (int k4 = 0; k4 < k4n; ++k4) {
        const int k = 4 * k4 + fc;
        double a[MT];
#pragma unroll
        for (int i = 0; i < MT; ++i) a[i] = A[(8 * i + fr) * S::SA + k];
        double b[NTE];
#pragma unroll
        for (int j = 0; j < NTE; ++j) b[j] = trw ? Ws[(8 * j + fr) * SBF + k] : Ws[k * SBF + 8 * j + fr];
#pragma unroll
        for (int j = 0; j < NTE; ++j)
#pragma unroll
          for (int i = 0; i < MT; ++i) dmma(ae[i][j], a[i], b[j]);
      }
    }
    {
      const int k4n = (no + 3) >> 2;
      for (int k4 = 0; k4 < k4n; ++k4) {
        const int k = 4 * k4 + fc;
        double a[MT];
#pragma unroll
        for (int i = 0; i < MT; ++i) a[i] = A[(8 * i + fr) * S::SA + ne + k];  // <= n + 2: zeroed pad
        double b[NTE];
#pragma unroll
        for (int j = 0; j < NTE; ++j) b[j] = trw ? WO[(8 * j + fr) * SBF + k] : WO[k * SBF + 8 * j + fr];
#pragma unroll
        for (int j = 0; j < NTE; ++j)
          if (j < NTE - 1 || full_o)
#pragma unroll
            for (int i = 0; i < MT; ++i) dmma(ao[i][j], a[i], b[j]);
      }
    }
  }
  if (tr) tr[4] = gtimer();
  // x_c = e_c + o_c, x_{n-1-c} = e_c - o_c (c < ne; the middle of an odd n is written twice with
  // the same value)
  const bool scale = pb.epi == EPI_SCALE;
  const bool mid2 = trw && (n & 1);
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    double xd[NTE][2], xm[NTE][2];
#pragma unroll
    for (int j = 0; j < NTE; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 8 * j + 2 * fc + h;
        double e = ae[i][j][h];
        if (mid2 && c == no) e *= 2.0;
        double v0 = e + ao[i][j][h], v1 = e - ao[i][j][h];
        if (scale && mv[i] && c < ne) {
          v0 *= pb.scale[sidx[i] + cs * c];
          v1 *= pb.scale[sidx[i] + cs * (n - 1 - c)];
        }
        xd[j][h] = v0;
        xm[j][h] = v1;
      }
    double* __restrict__ Y = pb.Y + pb.ybs * (long long)item[i] + sidx[i];
    if (vrow) {
      const bool odd = fr & 1;
      double* base = odd ? Y - 1 : Y;
#pragma unroll
      for (int j = 0; j < NTE; ++j) {
        const int c = 8 * j + 2 * fc + (odd ? 1 : 0);
        const double sd = odd ? xd[j][0] : xd[j][1];
        const double gd = __shfl_xor_sync(0xffffffffu, sd, 4);
        const double sm_ = odd ? xm[j][0] : xm[j][1];
        const double gm = __shfl_xor_sync(0xffffffffu, sm_, 4);
        if (mv[i] && c < ne) {
          *reinterpret_cast<double2*>(base + (long long)g.P * c) =
              odd ? make_double2(gd, xd[j][1]) : make_double2(xd[j][0], gd);
          *reinterpret_cast<double2*>(base + (long long)g.P * (n - 1 - c)) =
              odd ? make_double2(gm, xm[j][1]) : make_double2(xm[j][0], gm);
        }
      }
    } else if (mv[i]) {
#pragma unroll
      for (int j = 0; j < NTE; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = 8 * j + 2 * fc + h;
          if (c < ne) {
            Y[cs * c] = xd[j][h];
            Y[cs * (n - 1 - c)] = xm[j][h];
          }
        }
      if (kout && fc == 0)
        for (int c = n; c < pb.yld; ++c) Y[c] = 0.0;  // zero pad column of a padded row
    }
  }
  __syncwarp();
  if (tr) tr[5] = gtimer();
}

template <int NT, bool KMAJ, int G, bool SC = false, bool FOLD = false>
__global__ void __launch_bounds__(STH, 1) mode_small_kernel(const __grid_constant__ ModeGroupT<G> grp) {
  using S = SS<NT>;
  extern __shared__ __align__(16) double sm[];
  double* Ws = sm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* A = sm + S::W_ELEMS + warp * S::ABUF;  // this warp's 8-row panel ([8][SA])

  int pi = 0;
#pragma unroll
  for (int i = 1; i < G; ++i)
    if (i < grp.count && (int)blockIdx.x >= grp.prob[i].cta_begin) pi = i;
  const ModeProb& pb = grp.prob[pi];
  const Geo g(pb);

  unsigned long long* trace = grp.trace ? grp.trace + ((size_t)blockIdx.x * SW + warp) * kTracePhases : nullptr;
  if (trace && lane == 0) trace[0] = gtimer();
  // independent of the previous kernel
  if constexpr (FOLD) {
    load_w_fold<NT>(Ws, pb, tid);
    for (int i = lane; i < S::ABUF; i += 32) A[i] = 0.0;  // panel pad columns read as zeros
  } else {
    load_w<NT>(Ws, pb, tid);
  }
  // PDL: everything below may read what the previous kernel wrote.
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (trace && lane == 0) trace[1] = gtimer();
  wait_group<0>();
  __syncthreads();  // W visible to all warps
  if (trace && lane == 0) trace[2] = gtimer();

  // tile t -> CTA t % ctas, then warp (t / ctas) % SW
  const int gw = (blockIdx.x - pb.cta_begin) + pb.ctas * warp;
  const int nw = pb.ctas * SW;
  for (long long t = gw; t < pb.tiles_m; t += nw)
    do_tile<NT, KMAJ, false, SC, FOLD>(pb, g, Ws, A, t, lane, (trace && lane == 0 && t == gw) ? trace : nullptr);
}

template <int NT, bool KMAJ>
cudaError_t launch_s(const ModeGroup* g, cudaStream_t s) {
  using S = SS<NT>;
  if (!g) {
    cudaError_t e = cudaFuncSetAttribute(mode_small_kernel<NT, KMAJ, kSmallGroup>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::BYTES);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(mode_small_kernel<NT, KMAJ, kMaxGroup>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::BYTES);
    if (e == cudaSuccess && !KMAJ)
      e = cudaFuncSetAttribute(mode_small_kernel<NT, false, kSmallGroup, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::BYTES);
    if constexpr (NT % 2 == 0) {
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(mode_small_kernel<NT, KMAJ, kSmallGroup, false, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::BYTES);
    }
    return e;
  }
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
  bool sc = false;
  for (int i = 0; i < g->count; ++i) sc = sc || g->prob[i].peers != nullptr;
  if (g->prob[0].fold != FOLD_NONE) {  // even-odd folded group (host-checked: all problems)
    if (sc || NT % 2 || g->count > kSmallGroup) return cudaErrorInvalidValue;
    if constexpr (NT % 2 == 0) {
      return cudaLaunchKernelEx(&cfg, mode_small_kernel<NT, KMAJ, kSmallGroup, false, true>,
                                narrow_group<kSmallGroup>(*g));
    }
    return cudaErrorInvalidValue;
  }
  if (sc) {  // peer-store problems (slab exchange): non-KMAJ, single-buffered kernel
    if (KMAJ || g->count > kSmallGroup) return cudaErrorInvalidValue;
    return cudaLaunchKernelEx(&cfg, mode_small_kernel<NT, false, kSmallGroup, true>,
                              narrow_group<kSmallGroup>(*g));
  }
  if (g->count <= kSmallGroup) {
    return cudaLaunchKernelEx(&cfg, mode_small_kernel<NT, KMAJ, kSmallGroup>,
                              narrow_group<kSmallGroup>(*g));
  }
  return cudaLaunchKernelEx(&cfg, mode_small_kernel<NT, KMAJ, kMaxGroup>, *g);
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
  if ((e = dispatch_small<false>(nullptr, NT, 0)) != cudaSuccess) return e;
  return cudaSuccess;
}

}  // namespace fdp
