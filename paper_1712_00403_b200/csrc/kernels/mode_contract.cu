// K1: mode-d contraction on FP64 tensor cores (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4 on
// sm_100a; tcgen05 has no f64 kind, DESIGN.md §"FP64 tensor cores").
//
// Implements one stage of Algorithm 1 steps 2 and 4: the m-mode product
// of P:389-398 against an n x n eigenvector matrix, for up to kMaxGroup independent problems
// (velocity components / batch) in one grouped launch. Optional fused epilogues: division by the
// Kronecker-sum spectrum Lambda (step 3) and the P^G post-scaling D^{-1/2}.
//
// CTA tile: BM = 4 warps x (8*MT) rows  by  BN = 8*NT columns, K in chunks of BK = 16 through a
// STAGES-deep cp.async ring in shared memory. Each warp owns MT x NT DMMA accumulators (FP64
// registers). Shared-memory strides are == 4 (mod 16) doubles so the 8x4 / 4x8 fragment loads
// are bank-conflict free.
#include <cstdlib>

#include "../fdp_internal.h"

namespace fdp {
namespace {

#ifndef FDP_K1_BK
#define FDP_K1_BK 16
#endif
// 2 stages x 4 CTAs per SM (registers capped at 128 by the launch bound; 16 resident warps)
// measured 2% faster than 3 stages x 3 CTAs (154-164 registers) on configs 4 and 5
#ifndef FDP_K1_STAGES
#define FDP_K1_STAGES 2
#endif
#ifndef FDP_K1_MINB
#define FDP_K1_MINB 4
#endif
constexpr int BK = FDP_K1_BK;
// folded forward: two A tiles per stage; K chunks of 8 keep 4 CTAs (16 warps) per SM
#ifndef FDP_K1F_BK
#define FDP_K1F_BK 8
#endif
constexpr int kFoldBK = FDP_K1F_BK;
#ifndef FDP_K1F_STAGES
#define FDP_K1F_STAGES 2
#endif
constexpr int kFoldStages = FDP_K1F_STAGES;
constexpr int STAGES = FDP_K1_STAGES;
constexpr int WARPS = kK1Warps;
constexpr int THREADS = WARPS * 32;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int MT, int NT, bool KMAJ>
struct Smem {
  static constexpr int BM = WARPS * 8 * MT;
  static constexpr int BN = 8 * NT;
  static constexpr int SA = KMAJ ? (BK + 4) : (BM + 4);      // KMAJ: [BM][SA]; else [BK][SA]
  static constexpr int A_ELEMS = KMAJ ? BM * SA : BK * SA;
  static constexpr int SB = ((BN + 15) / 16) * 16 + 4;       // [BK][SB]
  static constexpr int B_ELEMS = BK * SB;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr size_t BYTES = sizeof(double) * STAGE * STAGES;
};

template <int MT, int NT, bool KMAJ, int G, bool SC = false>
__global__ void __launch_bounds__(THREADS, FDP_K1_MINB)
mode_contract_kernel(const __grid_constant__ ModeGroupT<G> grp) {
  using S = Smem<MT, NT, KMAJ>;
  constexpr int BM = S::BM, BN = S::BN;
  extern __shared__ __align__(16) double smem[];

  // ---- which problem / tile ----
  int pi = 0;
#pragma unroll
  for (int i = 1; i < G; ++i)
    if (i < grp.count && (int)blockIdx.x >= grp.prob[i].cta_begin) pi = i;
  const ModeProb& pb = grp.prob[pi];
  const int t = blockIdx.x - pb.cta_begin;
  const int tn = t % pb.tiles_n;
  const int tm = t / pb.tiles_n;
  const long long m0 = (long long)tm * BM;
  const int n0 = tn * BN;
  const long long M = (long long)pb.P * pb.Q * pb.batch;
  const int P = pb.P, n = pb.n, ldw = pb.ldw, nout = pb.nout;
  const long long Pn = (long long)P * n, Pno = (long long)P * nout;
  const double* __restrict__ X = pb.X;
  const double* __restrict__ W = pb.W;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // ---- per-thread load assignments (fixed across the K loop) ----
  // KMAJ: thread loads k = tid % BK of rows m = tid/BK + (THREADS/BK)*j, j < BM*BK/THREADS.
  // else : thread loads row m = tid % BM for k = tid/BM + (THREADS/BM)*j.
  constexpr int RSTEP = THREADS / BK;  // KMAJ rows covered per pass
  constexpr int A_ROWS_PER_THREAD = KMAJ ? BM / RSTEP : 1;
  long long a_off[A_ROWS_PER_THREAD];
  bool a_ok[A_ROWS_PER_THREAD];
  const int Qn = pb.Q;
  if (KMAJ) {
#pragma unroll
    for (int j = 0; j < A_ROWS_PER_THREAD; ++j) {
      long long m = m0 + tid / BK + RSTEP * j;
      a_ok[j] = m < M;
      // P == 1: row m = q + Q*b at xld*q + xbs*b, contiguous in k
      a_off[j] = a_ok[j] ? (long long)pb.xld * (m % Qn) + pb.xbs * (m / Qn) : 0;
    }
  } else {
    long long m = m0 + tid % BM;
    a_ok[0] = m < M;
    if (a_ok[0]) {
      const long long p = m % P, r = m / P;
      a_off[0] = p + Pn * (r % Qn) + pb.xbs * (r / Qn);
    } else {
      a_off[0] = 0;
    }
  }

  auto load_stage = [&](int stage, int k0) {
    double* As = smem + stage * S::STAGE;
    double* Bs = As + S::A_ELEMS;
    if (KMAJ) {
      const int k = tid % BK;
      const bool kv = (k0 + k) < n;
#pragma unroll
      for (int j = 0; j < A_ROWS_PER_THREAD; ++j) {
        const int mr = tid / BK + RSTEP * j;
        const bool v = a_ok[j] && kv;
        cp_async8(&As[mr * S::SA + k], X + (v ? a_off[j] + k0 + k : 0), v);
      }
    } else {
      constexpr int KSTEP = THREADS / BM;  // rows of k handled per pass
      const int mr = tid % BM;
#pragma unroll
      for (int kk = tid / BM; kk < BK; kk += KSTEP) {
        const bool v = a_ok[0] && (k0 + kk) < n;
        cp_async8(&As[kk * S::SA + mr], X + (v ? a_off[0] + (long long)P * (k0 + kk) : 0), v);
      }
    }
    // B: BK rows x BN cols from W (always in bounds: W is kpad x ldw, zero padded).
    constexpr int CHUNKS = BK * BN / 2;  // 16-byte chunks
#pragma unroll
    for (int c = tid; c < CHUNKS; c += THREADS) {
      const int kr = c / (BN / 2), cc = (c % (BN / 2)) * 2;
      cp_async16(&Bs[kr * S::SB + cc], W + (size_t)(k0 + kr) * ldw + n0 + cc);
    }
  };

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int KT = (n + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s * BK);
    cp_async_commit();
  }

  const int fr = lane >> 2, fc = lane & 3;  // fragment row (0..7) / k or col index (0..3)
  const int wm = warp * 8 * MT;

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < KT) load_stage(nk % STAGES, nk * BK);
      cp_async_commit();
    }
    const double* As = smem + (kt % STAGES) * S::STAGE;
    const double* Bs = As + S::A_ELEMS;
    const int kvalid = min(BK, n - kt * BK);
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      if (k4 < kvalid) {
        double a[MT], b[NT];
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const int mr = wm + 8 * i + fr;
          a[i] = KMAJ ? As[mr * S::SA + k4 + fc] : As[(k4 + fc) * S::SA + mr];
        }
#pragma unroll
        for (int j = 0; j < NT; ++j) b[j] = Bs[(k4 + fc) * S::SB + 8 * j + fr];
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma(acc[i][j], a[i], b[j]);
      }
    }
  }
  cp_async_wait<0>();

  // ---- epilogue: C[m][a], m = wm + 8i + fr, a = 8j + 2fc + {0,1} ----
  const int epi = pb.epi;
  double* __restrict__ Y = pb.Y;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const long long m = m0 + wm + 8 * i + fr;
    if (m >= M) continue;
    long long row_off;
    long long sidx;  // index within the batch item (for EPI_SCALE)
    double lrow = 0.0;
    bool pad_row = false;
    if (KMAJ) {
      sidx = (long long)pb.yld * (m % Qn);
      row_off = sidx + pb.ybs * (m / Qn);
    } else {
      const long long p = m % P, r = m / P;
      sidx = p + Pno * (r % Qn);
      row_off = sidx + pb.ybs * (r / Qn);
      if (epi == EPI_LAMBDA) {
        const int i1 = (int)(p % pb.n1);
        pad_row = i1 >= pb.n1v;  // padding row of a padded intermediate: stays 0
        if (!pad_row) lrow = pb.lam1 ? pb.lam0[i1] + pb.lam1[p / pb.n1] : pb.lam0[p];
      }
    }
    const int ncols = KMAJ ? pb.yld : nout;  // padded outputs also get their zero pad column
#pragma unroll
    for (int j = 0; j < NT; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = n0 + 8 * j + 2 * fc + h;
        if (a < ncols) {
          double v = acc[i][j][h];
          // SC (compile-time): peer-store scatter of the slab exchange; other launches keep the
          // plain addressing (the scatter branch cost 5% on config 4 when always compiled in)
          double* yp = SC ? scatter_ptr(pb, m, a) : Y + row_off + (long long)P * a;
          if (epi == EPI_LAMBDA) v = pad_row ? 0.0 : fdp_div(v, lrow + pb.lamcol[a]);
          else if (epi == EPI_SCALE) v = v * pb.scale[sidx + (long long)P * a];
          else if (epi == EPI_AXPBY) v = pb.alpha * v + (pb.beta != 0.0 ? pb.beta * *yp : 0.0);
          *yp = v;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// K1f: the even-odd folded transform (mode_small.cu tile_compute_store_fold has the
// algebra) on the K1 tiling, for extents n > 96.
//   FOLD = FOLD_FWD: a CTA's column tile lies in the E block (tn < tiles_ne: spectral columns
//     [0, ne), operand s_k = x_k + x_{n-1-k}) or the O block (columns ne + [0, no), operand
//     d_k = x_k - x_{n-1-k}); each pipeline stage holds the direct A tile (k0 .. k0+BK-1) and the
//     mirrored one (n-k0-BK .. n-k0-1), combined at the fragment load. K = ne or no: about half
//     the dense DMMAs. Optional EPI_LAMBDA (spectral order [E | O]).
//   FOLD = FOLD_BWD: a CTA owns spatial columns c in [n0, n0 + BN) of [0, ne) and accumulates
//     e = W_E y_E over the E half of the spectral row and o = W_O y_O over the O half in two
//     register sets, then writes x_c = e + o and x_{n-1-c} = e - o (optional EPI_SCALE).
// ---------------------------------------------------------------------------------------------
template <int MT, int NT, bool KMAJ, int FOLD, int BKF>
struct SmemF {
  static constexpr int BM = WARPS * 8 * MT;
  static constexpr int BN = 8 * NT;
  static constexpr int SA = KMAJ ? (BKF + 4) : (BM + 4);
  static constexpr int A1 = KMAJ ? BM * SA : BKF * SA;       // one A tile
  static constexpr int A_ELEMS = A1 * (FOLD == FOLD_FWD || FOLD == FOLD_SYM ? 2 : 1);
  static constexpr int SB = ((BN + 15) / 16) * 16 + 4;
  static constexpr int B_ELEMS = BKF * SB;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr size_t BYTES = sizeof(double) * STAGE * kFoldStages;
};

template <int MT, int NT, bool KMAJ, int FOLD, int BKF, bool SC = false>
__global__ void __launch_bounds__(THREADS, FDP_K1_MINB)
mode_contract_fold_kernel(const __grid_constant__ ModeGroupT<kSmallGroup> grp) {
  using S = SmemF<MT, NT, KMAJ, FOLD, BKF>;
  using SF = S;
  constexpr int BM = S::BM, BN = S::BN;
  extern __shared__ __align__(16) double smem[];

  int pi = 0;
#pragma unroll
  for (int i = 1; i < kSmallGroup; ++i)
    if (i < grp.count && (int)blockIdx.x >= grp.prob[i].cta_begin) pi = i;
  const ModeProb& pb = grp.prob[pi];
  const int t = blockIdx.x - pb.cta_begin;
  const int tn = t % pb.tiles_n;
  const int tm = t / pb.tiles_n;
  const long long m0 = (long long)tm * BM;
  const long long M = (long long)pb.P * pb.Q * pb.batch;
  const int P = pb.P, n = pb.n, ldw = pb.ldw, nout = pb.nout;
  const int ne = (n + 1) >> 1, no = n >> 1;
  const long long Pn = (long long)P * n, Pno = (long long)P * nout;
  const double* __restrict__ X = pb.X;
  const double* __restrict__ W = pb.W;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // FOLD_FWD: E or O column tile
  const bool isE = FOLD != FOLD_FWD || tn < pb.tiles_ne;
  const int n0 = (FOLD == FOLD_FWD && !isE ? tn - pb.tiles_ne : tn) * BN;

  constexpr int RSTEP = THREADS / BKF;
  constexpr int A_ROWS_PER_THREAD = KMAJ ? BM / RSTEP : 1;
  long long a_off[A_ROWS_PER_THREAD];
  bool a_ok[A_ROWS_PER_THREAD];
  const int Qn = pb.Q;
  if (KMAJ) {
#pragma unroll
    for (int j = 0; j < A_ROWS_PER_THREAD; ++j) {
      long long m = m0 + tid / BKF + RSTEP * j;
      a_ok[j] = m < M;
      a_off[j] = a_ok[j] ? (long long)pb.xld * (m % Qn) + pb.xbs * (m / Qn) : 0;
    }
  } else {
    long long m = m0 + tid % BM;
    a_ok[0] = m < M;
    if (a_ok[0]) {
      const long long p = m % P, r = m / P;
      a_off[0] = p + Pn * (r % Qn) + pb.xbs * (r / Qn);
    } else {
      a_off[0] = 0;
    }
  }

  // A tile of columns kb .. kb+BKF-1 (zero outside [0, n)) into As
  auto load_a = [&](double* As, int kb) {
    if (KMAJ) {
      const int k = tid % BKF;
      const int kk = kb + k;
      const bool kv = kk >= 0 && kk < n;
#pragma unroll
      for (int j = 0; j < A_ROWS_PER_THREAD; ++j) {
        const int mr = tid / BKF + RSTEP * j;
        const bool v = a_ok[j] && kv;
        cp_async8(&As[mr * S::SA + k], X + (v ? a_off[j] + kk : 0), v);
      }
    } else {
      constexpr int KSTEP = THREADS / BM;
      const int mr = tid % BM;
#pragma unroll
      for (int k = tid / BM; k < BKF; k += KSTEP) {
        const int kk = kb + k;
        const bool v = a_ok[0] && kk >= 0 && kk < n;
        cp_async8(&As[k * S::SA + mr], X + (v ? a_off[0] + (long long)P * kk : 0), v);
      }
    }
  };
  // one stage: A (direct; FOLD_FWD also the mirror block) and the W rows wrow0 + k0 ..
  auto load_stage = [&](int stage, int k0, int aoff, int wrow0) {
    double* As = smem + stage * SF::STAGE;
    double* Bs = As + SF::A_ELEMS;
    load_a(As, aoff + k0);
    if (FOLD == FOLD_FWD || FOLD == FOLD_SYM) load_a(As + S::A1, n - k0 - BKF);
    constexpr int CHUNKS = BKF * BN / 2;
#pragma unroll
    for (int c = tid; c < CHUNKS; c += THREADS) {
      const int kr = c / (BN / 2), cc = (c % (BN / 2)) * 2;
      cp_async16(&Bs[kr * S::SB + cc], W + (size_t)(wrow0 + k0 + kr) * ldw + n0 + cc);
    }
  };

  const int fr = lane >> 2, fc = lane & 3;
  const int wm = warp * 8 * MT;
  constexpr bool TWO = FOLD == FOLD_BWD || FOLD == FOLD_SYM;  // e and o accumulator sets
  double acc[MT][NT][2], acc2[TWO ? MT : 1][TWO ? NT : 1][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if constexpr (TWO) {
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc2[i][j][0] = acc2[i][j][1] = 0.0;
  }

  // K loop over K columns of the operand starting at aoff, W rows from wrow0, into accumulator c
  auto kloop = [&](double (&c)[MT][NT][2], int K, int aoff, int wrow0, double sgn) {
    const int KT = (K + BKF - 1) / BKF;
#pragma unroll
    for (int st = 0; st < kFoldStages - 1; ++st) {
      if (st < KT) load_stage(st, st * BKF, aoff, wrow0);
      cp_async_commit();
    }
    for (int kt = 0; kt < KT; ++kt) {
      cp_async_wait<kFoldStages - 2>();
      __syncthreads();
      {
        const int nk = kt + kFoldStages - 1;
        if (nk < KT) load_stage(nk % kFoldStages, nk * BKF, aoff, wrow0);
        cp_async_commit();
      }
      const double* As = smem + (kt % kFoldStages) * SF::STAGE;
      const double* As2 = As + S::A1;
      const double* Bs = As + SF::A_ELEMS;
      const int kvalid = min(BKF, K - kt * BKF);
#pragma unroll
      for (int k4 = 0; k4 < BKF; k4 += 4) {
        if (k4 < kvalid) {
          double a[MT], b[NT];
#pragma unroll
          for (int i = 0; i < MT; ++i) {
            const int mr = wm + 8 * i + fr;
            const int kk = k4 + fc;
            a[i] = KMAJ ? As[mr * S::SA + kk] : As[kk * S::SA + mr];
            if (FOLD == FOLD_FWD || FOLD == FOLD_SYM) {
              const int km = BKF - 1 - kk;  // mirror block holds n-k0-BKF .. n-k0-1
              a[i] += sgn * (KMAJ ? As2[mr * S::SA + km] : As2[km * S::SA + mr]);
            }
          }
#pragma unroll
          for (int j = 0; j < NT; ++j) b[j] = Bs[(k4 + fc) * S::SB + 8 * j + fr];
#pragma unroll
          for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma(c[i][j], a[i], b[j]);
        }
      }
    }
    cp_async_wait<0>();
    __syncthreads();  // the next phase refills the ring
  };

  if constexpr (FOLD == FOLD_FWD) {
    kloop(acc, isE ? ne : no, 0, isE ? 0 : pb.foldh, isE ? 1.0 : -1.0);
  } else if constexpr (FOLD == FOLD_SYM) {  // y = A x, A centrosymmetric: e = W_E^T s, o = W_O^T d
    kloop(acc, ne, 0, 0, 1.0);
    kloop(acc2, no, 0, pb.foldh, -1.0);
  } else {
    kloop(acc, ne, 0, 0, 0.0);              // e over the E half of the spectral row
    kloop(acc2, no, ne, pb.foldh, 0.0);     // o over the O half
  }

  // ---- epilogue ----
  const int epi = pb.epi;
  double* __restrict__ Y = pb.Y;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const long long m = m0 + wm + 8 * i + fr;
    if (m >= M) continue;
    long long row_off, sidx;
    double lrow = 0.0;
    bool pad_row = false;
    if (KMAJ) {
      sidx = (long long)pb.yld * (m % Qn);
      row_off = sidx + pb.ybs * (m / Qn);
    } else {
      const long long p = m % P, r = m / P;
      sidx = p + Pno * (r % Qn);
      row_off = sidx + pb.ybs * (r / Qn);
      if (epi == EPI_LAMBDA) {
        const int i1 = (int)(p % pb.n1);
        pad_row = i1 >= pb.n1v;
        if (!pad_row) lrow = pb.lam1 ? pb.lam0[i1] + pb.lam1[p / pb.n1] : pb.lam0[p];
      }
    }
    const long long cs = KMAJ ? 1 : P;
    if constexpr (FOLD == FOLD_FWD) {
      const int ncols = KMAJ ? pb.yld : nout;  // KMAJ rows: their pad columns get their zeros
      const int coff = isE ? 0 : ne, cval = isE ? ne : no;
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int a = n0 + 8 * j + 2 * fc + h;
          const int oc = coff + a;
          if (oc < ncols && (a < cval || (KMAJ && !isE))) {
            double v = a < cval ? acc[i][j][h] : 0.0;
            if (epi == EPI_LAMBDA) v = (pad_row || a >= cval) ? 0.0 : fdp_div(v, lrow + pb.lamcol[oc]);
            // SC: peer-store scatter of the slab exchange
            if (SC) *scatter_ptr(pb, m, oc) = v;
            else Y[row_off + cs * oc] = v;
          }
        }
    } else {
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = n0 + 8 * j + 2 * fc + h;
          if (c < ne) {
            double v0 = acc[i][j][0 + h] + acc2[i][j][h];
            double v1 = acc[i][j][h] - acc2[i][j][h];
            if (epi == EPI_SCALE) {
              v0 *= pb.scale[sidx + cs * c];
              v1 *= pb.scale[sidx + cs * (n - 1 - c)];
            }
            if (SC) {
              *scatter_ptr(pb, m, c) = v0;
              *scatter_ptr(pb, m, n - 1 - c) = v1;
            } else {
              Y[row_off + cs * c] = v0;
              Y[row_off + cs * (n - 1 - c)] = v1;
            }
          }
        }
      if (KMAJ && !SC && n0 == 0 && fc == 0)
        for (int c = n; c < pb.yld; ++c) Y[row_off + c] = 0.0;  // zero pad column of a padded row
    }
  }
}

template <int MT, int NT, bool KMAJ>
cudaError_t launch_t(const ModeGroup* g, cudaStream_t s) {
  using S = Smem<MT, NT, KMAJ>;
  if (!g) {  // prepare: raise the dynamic shared-memory limit (outside any stream capture)
    cudaError_t e = cudaFuncSetAttribute(mode_contract_kernel<MT, NT, KMAJ, kSmallGroup>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::BYTES);
    if (e == cudaSuccess && !KMAJ)
      e = cudaFuncSetAttribute(mode_contract_kernel<MT, NT, false, kSmallGroup, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::BYTES);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(mode_contract_kernel<MT, NT, KMAJ, kMaxGroup>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::BYTES);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(mode_contract_fold_kernel<MT, NT, KMAJ, FOLD_FWD, kFoldBK>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)SmemF<MT, NT, KMAJ, FOLD_FWD, kFoldBK>::BYTES);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(mode_contract_fold_kernel<MT, NT, KMAJ, FOLD_BWD, BK>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)SmemF<MT, NT, KMAJ, FOLD_BWD, BK>::BYTES);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(mode_contract_fold_kernel<MT, NT, KMAJ, FOLD_SYM, kFoldBK>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)SmemF<MT, NT, KMAJ, FOLD_SYM, kFoldBK>::BYTES);
    if (!KMAJ && e == cudaSuccess)
      e = cudaFuncSetAttribute(mode_contract_fold_kernel<MT, NT, false, FOLD_FWD, kFoldBK, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)SmemF<MT, NT, false, FOLD_FWD, kFoldBK>::BYTES);
    if (!KMAJ && e == cudaSuccess)
      e = cudaFuncSetAttribute(mode_contract_fold_kernel<MT, NT, false, FOLD_BWD, BK, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)SmemF<MT, NT, false, FOLD_BWD, BK>::BYTES);
    return e;
  }
  if (g->prob[0].fold != FOLD_NONE) {  // folded K1 group (host-checked: all problems, one kind)
    const int f = g->prob[0].fold;
    if (g->count > kSmallGroup || (f != FOLD_FWD && f != FOLD_BWD && f != FOLD_SYM))
      return cudaErrorInvalidValue;
    if (f == FOLD_SYM) {  // the dense P_Q passes of a K1-sized pressure factor
      mode_contract_fold_kernel<MT, NT, KMAJ, FOLD_SYM, kFoldBK>
          <<<g->total_ctas, THREADS, SmemF<MT, NT, KMAJ, FOLD_SYM, kFoldBK>::BYTES, s>>>(narrow_group<kSmallGroup>(*g));
      return cudaGetLastError();
    }
    bool scf = false;
    for (int i = 0; i < g->count; ++i) scf = scf || g->prob[i].peers != nullptr;
    if (scf) {  // peer-store problems: non-KMAJ, batch 1
      if (KMAJ) return cudaErrorInvalidValue;
      if (f == FOLD_FWD)
        mode_contract_fold_kernel<MT, NT, false, FOLD_FWD, kFoldBK, true>
            <<<g->total_ctas, THREADS, SmemF<MT, NT, false, FOLD_FWD, kFoldBK>::BYTES, s>>>(narrow_group<kSmallGroup>(*g));
      else
        mode_contract_fold_kernel<MT, NT, false, FOLD_BWD, BK, true>
            <<<g->total_ctas, THREADS, SmemF<MT, NT, false, FOLD_BWD, BK>::BYTES, s>>>(narrow_group<kSmallGroup>(*g));
      return cudaGetLastError();
    }
    if (f == FOLD_FWD)
      mode_contract_fold_kernel<MT, NT, KMAJ, FOLD_FWD, kFoldBK>
          <<<g->total_ctas, THREADS, SmemF<MT, NT, KMAJ, FOLD_FWD, kFoldBK>::BYTES, s>>>(narrow_group<kSmallGroup>(*g));
    else
      mode_contract_fold_kernel<MT, NT, KMAJ, FOLD_BWD, BK>
          <<<g->total_ctas, THREADS, SmemF<MT, NT, KMAJ, FOLD_BWD, BK>::BYTES, s>>>(narrow_group<kSmallGroup>(*g));
    return cudaGetLastError();
  }
  bool sc = false;
  for (int i = 0; i < g->count; ++i) sc = sc || g->prob[i].peers != nullptr;
  if (sc) {  // peer-store problems: batch 1, non-KMAJ, launched one at a time (run1)
    if (KMAJ || g->count > kSmallGroup) return cudaErrorInvalidValue;
    mode_contract_kernel<MT, NT, false, kSmallGroup, true><<<g->total_ctas, THREADS, S::BYTES, s>>>(
        narrow_group<kSmallGroup>(*g));
  } else if (g->count <= kSmallGroup)
    mode_contract_kernel<MT, NT, KMAJ, kSmallGroup><<<g->total_ctas, THREADS, S::BYTES, s>>>(
        narrow_group<kSmallGroup>(*g));
  else
    mode_contract_kernel<MT, NT, KMAJ, kMaxGroup><<<g->total_ctas, THREADS, S::BYTES, s>>>(*g);
  return cudaGetLastError();
}

template <int MT, bool KMAJ>
cudaError_t dispatch_nt(const ModeGroup* g, int NT, cudaStream_t s) {
  switch (NT) {
    case 1: return launch_t<MT, 1, KMAJ>(g, s);
    case 2: return launch_t<MT, 2, KMAJ>(g, s);
    case 3: return launch_t<MT, 3, KMAJ>(g, s);
    case 4: return launch_t<MT, 4, KMAJ>(g, s);
    case 5: return launch_t<MT, 5, KMAJ>(g, s);
    case 6: return launch_t<MT, 6, KMAJ>(g, s);
    case 7: return launch_t<MT, 7, KMAJ>(g, s);
    case 8: return launch_t<MT, 8, KMAJ>(g, s);
    case 9: return launch_t<MT, 9, KMAJ>(g, s);
    case 10: return launch_t<MT, 10, KMAJ>(g, s);
    case 11: return launch_t<MT, 11, KMAJ>(g, s);
    case 12: return launch_t<MT, 12, KMAJ>(g, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

TileCfg choose_tile(int n) {
  TileCfg c;
  const int n8 = (n + 7) / 8;
  int split = (n8 + 11) / 12;            // number of column tiles, each <= 12 n8-tiles
  c.NT = (n8 + split - 1) / split;
  c.tiles_n = (n8 + c.NT - 1) / c.NT;
  c.MT = 2;
  c.ldw = c.tiles_n * 8 * c.NT;
  c.kpad = ((n + 31) / 32) * 32;  // covers any K-tile depth <= 32
  return c;
}

cudaError_t launch_mode_group(const ModeGroup& g, const TileCfg& cfg, bool kmaj, cudaStream_t s) {
  if (g.total_ctas <= 0) return cudaSuccess;
  if (cfg.MT != 2) return cudaErrorInvalidValue;
  return kmaj ? dispatch_nt<2, true>(&g, cfg.NT, s) : dispatch_nt<2, false>(&g, cfg.NT, s);
}

cudaError_t prepare_mode_kernels(const TileCfg& cfg) {
  if (cfg.MT != 2) return cudaErrorInvalidValue;
  cudaError_t e = dispatch_nt<2, true>(nullptr, cfg.NT, 0);
  if (e != cudaSuccess) return e;
  return dispatch_nt<2, false>(nullptr, cfg.NT, 0);
}

// ---------------------------------------------------------------------------------------------
// K2: streaming diagonal scaling y = x o s (period N over the batch), double2-vectorised when
// aligned. HBM-bound: 24 B per element (read x, s (L2-resident across the batch), write y).
// ---------------------------------------------------------------------------------------------
namespace {
__global__ void scale_kernel(const double* __restrict__ x, double* __restrict__ y,
                             const double* __restrict__ s, long long N, long long total,
                             long long xs, long long ys) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (; i < total; i += stride) {
    const long long b = i / N, j = i - b * N;
    y[b * ys + j] = x[b * xs + j] * s[j];
  }
}
}  // namespace

cudaError_t launch_scale(const double* x, double* y, const double* s, long long N, long long batch,
                         long long xs, long long ys, cudaStream_t st) {
  long long total = N * batch;
  if (total == 0) return cudaSuccess;
  int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  scale_kernel<<<blocks, 256, 0, st>>>(x, y, s, N, total, xs, ys);
  return cudaGetLastError();
}

}  // namespace fdp
