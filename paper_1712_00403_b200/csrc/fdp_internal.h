// Internal declarations shared by the host (C++) and device (CUDA) translation units of libfdp.
// Nothing here crosses the C ABI (include/fdp.h).
#pragma once

#include <cstdint>
#include <cstddef>
#include <string>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/fdp.h"

namespace fdp {

// ---------------------------------------------------------------------------------------------
// Mode-d contraction (PAPER.md P:389-398 m-mode product; Algorithm 1 steps 2/4).
// The tensor is viewed as (P, n, Q): element (p, k, q) at p + P*(k + n*q), i1 fastest, with the
// batch folded into Q. Output Y(p, a, q) = sum_k X(p, k, q) * W[k*ldw + a].
//   forward transform  (x_d U_d^T): W[k][a] = U_d[k][a]
//   backward transform (x_d U_d)  : W[k][a] = U_d[a][k]
// Flattened GEMM rows m = p + P*q; "KMAJ" (P == 1, mode 1) rows are contiguous along k.
// ---------------------------------------------------------------------------------------------
// FOLD_SYM: y = A x for a centrosymmetric A (J A J = A) in one folded pass (dense P_Q^{-1} modes)
enum Fold : int { FOLD_NONE = 0, FOLD_FWD = 1, FOLD_BWD = 2, FOLD_FUSED = 3, FOLD_SYM = 4 };

enum TransIO : int { TIO_NONE = 0, TIO_OUT_T = 1, TIO_OUT_K = 2 };

enum Epilogue : int {
  EPI_NONE = 0,
  EPI_LAMBDA = 1,  // divide by Lambda[i] = lamrow(p) + lamcol[a]   (Algorithm 1 step 3)
  EPI_SCALE = 2,   // multiply by dscale[index within item]           (P^G post-scaling)
  EPI_FUSED = 3,   // small-n only: x_D U_D^T, divide by Lambda, x_D U_D in one pass
  EPI_AXPBY = 4,   // Y = alpha * result + beta * Y (Kronecker operator terms accumulate)
};

struct ModeProb {
  const double* X;
  double* Y;
  const double* W;        // kpad x ldw row-major, zero padded
  const double* scale;    // EPI_SCALE: length N (one batch item)
  const double* lam0;     // EPI_LAMBDA: coef-scaled eigenvalues c_d*lambda_d, d = 1 (index i1)
  const double* lam1;     //             d = 2 (3D only; nullptr in 2D)
  const double* lamcol;   //             d = D (the contracted, last direction)
  const double* rlam;     // EPI_LAMBDA on K1t: 1 / Lambda in the output layout of one item, or NULL
  long long N;            // elements per batch item (of this tensor)
  long long xbs, ybs;     // batch-item strides of X and Y (elements)
  int P, n, Q;            // per item; GEMM rows M = P * Q * batch; n = contracted extent
  int nout;               // output extent of the mode (= n for the square FD transforms)
  double alpha, beta;     // EPI_AXPBY
  int batch;
  int ldw;
  int n1;                 // leading dimension of direction 1 (Lambda row decomposition)
  int n1v;                // valid extent of direction 1 (rows with i1 >= n1v are padding)
  int xld, yld;           // KMAJ (mode 1): row (fiber) strides of X and Y (n1 or padded n1p)
  int vx, vy;             // 16-byte vector loads of X / stores of Y are aligned (host-checked)
  int epi;
  int tiles_m, tiles_n;
  int cta_begin;          // first CTA of this problem in the grouped grid
  int fd_work;            // host-side accounting only: 1 = FD contraction, 0 = dense P_Q pass
  int ctas;               // small-n kernel: CTAs assigned to this problem
  // Even-odd folding of a persymmetric mode (DESIGN.md §5 "folded transforms"): 0 = dense W,
  // FOLD_FWD / FOLD_BWD / FOLD_FUSED = the folded forward, backward or fused (forward, Lambda,
  // backward) transform. W then holds two blocks, E (rows [0, foldh)) and O (rows [foldh, 2 foldh)),
  // and the mode's spectral index runs over [E (ceil(n/2)) | O (floor(n/2))].
  int fold;
  int foldh;
  int fold_k1;            // folded problem of the K1 kernel (n > 96): 1; small-path fold: 0
  int tiles_ne;           // K1 FOLD_FWD: column tiles of the E block (the rest are O tiles)
  // Transposed I/O of the plane path (folded problems only): TIO_OUT_T (KMAJ
  // kernel): output row m, column a at Y[item * ybs + mi + Mi * a] (the plane-major layout, mi the
  // row within its item, Mi = P * Q rows per item); TIO_OUT_K (non-KMAJ kernel reading a
  // plane-major tensor as P = Mi, Q = 1): output at Y[item * ybs + yld * mi + a].
  int tio;
  int tio_ld;             // TIO_OUT_T: column stride of the output (the plane stride, even)
  int tio_rows;           // TIO_OUT_K: rows per item that exist (rows >= tio_rows are the
                          // plane-major layout's pad row: computed, never stored)
  // KMAJ small-path loads: optional input scaling x <- pre o x (pre indexed like the input within
  // one item: the P^G pre-scaling D^{-1/2} fused into the first pass)
  const double* pre;
  // K1t (kernels/mode_tma.cu): fragment-native folded W chunks of this transform, or NULL when
  // the TMA kernel cannot take it (see mode_tma.h)
  const double* Wt;
  // Peer-store scatter (slab exchange fused into the epilogue): when peers != NULL,
  // output element (GEMM row m, column a) of a batch-1, non-KMAJ problem is stored at
  // peers[o] + r + sc_n1 * ((a - lo_o) * (sc_a0 + sc_a1 * len_o) + (q + sc_qoff) * (sc_q0 + sc_q1 * len_o))
  // with r = m % sc_n1, q = m / sc_n1, and [lo_o, lo_o + len_o) the share of rank o that owns a
  // under the even split of sc_na over sc_G ranks (first sc_na % sc_G ranks one extra).
  double* const* peers;
  int sc_G, sc_na, sc_n1, sc_qoff, sc_a0, sc_a1, sc_q0, sc_q1;
};

#ifdef __CUDACC__
__device__ __forceinline__ double* scatter_ptr(const ModeProb& pb, long long m, int a) {
  const int G = pb.sc_G, na = pb.sc_na;
  const int q = na / G, rem = na % G;
  const int o = (q == 0 || a < rem * (q + 1)) ? a / (q + 1) : rem + (a - rem * (q + 1)) / q;
  const int lo = o * q + (o < rem ? o : rem);
  const int len = q + (o < rem ? 1 : 0);
  const long long r = m % pb.sc_n1, qq = m / pb.sc_n1;
  return pb.peers[o] + r +
         (long long)pb.sc_n1 * ((long long)(a - lo) * (pb.sc_a0 + pb.sc_a1 * len) +
                                (qq + pb.sc_qoff) * (pb.sc_q0 + pb.sc_q1 * len));
}
#endif

// Quotient a / b for the Lambda^{-1} epilogues (b = Lambda > 0, normal): hardware reciprocal
// approximation (~2^-23), one Newton step (~2^-46) and one Markstein correction of the quotient
// -- 5 FP64 ops (they share the FP64 datapath with DMMA) and no slow-path branch; within one
// ulp of the IEEE quotient (C-11).
#ifdef __CUDACC__
__device__ __forceinline__ double fdp_div(double a, double b) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(b));
  y = fma(fma(-b, y, 1.0), y, y);
  const double q = a * y;
  return fma(fma(-b, q, a), y, q);
}
#endif

// Problems of one grouped launch, passed by value as the kernel parameter. Kernels are compiled
// for two capacities: kSmallGroup (the FD stages: <= 4 problems, a small parameter block keeps the
// launch cheap) and kMaxGroup (multi-operator Kronecker stages); the host fills a ModeGroup and
// the launcher narrows it when it fits.
constexpr int kMaxGroup = 32;   // kernel parameters stay < 32 KB
constexpr int kSmallGroup = 4;
template <int G>
struct ModeGroupT {
  ModeProb prob[G];
  int count;
  int total_ctas;
  // diagnostics: when non-null, lane 0 of every warp records %globaltimer at kTracePhases points
  // of its first tile into trace[(blockIdx * warps + warp) * kTracePhases + phase]
  unsigned long long* trace;
};
using ModeGroup = ModeGroupT<kMaxGroup>;
template <int G>
inline ModeGroupT<G> narrow_group(const ModeGroup& g) {
  ModeGroupT<G> o;
  for (int i = 0; i < G; ++i) o.prob[i] = g.prob[i];
  o.count = g.count;
  o.total_ctas = g.total_ctas;
  o.trace = g.trace;
  return o;
}
constexpr int kTracePhases = 6;

// K1 CTA: kK1Warps warps stacked along M (BM = kK1Warps * 8 * MT rows).
#ifndef FDP_K1_WARPS
#define FDP_K1_WARPS 4
#endif
constexpr int kK1Warps = FDP_K1_WARPS;

// Tile configuration chosen for a problem size n (same for all problems of one launch).
struct TileCfg {
  int MT;      // m8 tiles per warp (warps stacked along M: BM = 4*8*MT)
  int NT;      // n8 tiles per warp (BN = 8*NT)
  int tiles_n; // ceil(n / BN)
  int ldw;     // tiles_n * BN
  int kpad;    // round_up(n, 16)
};
TileCfg choose_tile(int n);

// Launch one grouped mode-contraction stage. kmaj: P == 1 for every problem (mode 1).
cudaError_t launch_mode_group(const ModeGroup& g, const TileCfg& cfg, bool kmaj, cudaStream_t s);

// Small-n path (n <= 96, one column tile): persistent row-streaming kernel, W resident in shared
// memory, whole-K A panels per warp (8 rows) double-buffered with cp.async, programmatic
// dependent launch. Problems with epi == EPI_FUSED do mode-D forward, Lambda^{-1} and mode-D
// backward in one pass (the middle of Algorithm 1). The caller fills prob[i].ctas
// (CTAs per problem, sum = total_ctas) and prob[i].tiles_m = ceil(M/8).
constexpr int kSmallMaxN = 96;

// Folded problems (prob.fold != 0, every problem of the group) take the even-odd kernel; NT is
// then 2 * ceil(ceil(n/2) / 8) (even).
cudaError_t launch_mode_small(const ModeGroup& g, int NT, bool kmaj, cudaStream_t s);

// Plane kernel (kernels/mode_plane.cu). D = 3: per plane a1 of a plane-major tensor (written by a
// TIO_OUT_T mode-1 pass), the folded mode-2 forward, mode-3 forward / Lambda^{-1} / backward and
// mode-2 backward in shared memory (kind 0, in place), or the FOLD_SYM mode-2 and mode-3 passes
// of P_Q with the result stored in the natural layout (kind 1). D = 2: the whole component is one
// plane (rows = i2 lines): the complete folded FD apply (kind 2) or P_Q (kind 3) in one launch,
// natural-layout input and output.
struct PlaneProb {
  double* T;              // plane-major tensor: item b, plane a1 at T + b * tbs + a1 * n2 * n3
  long long tbs;
  const double* W2;       // folded forward (kind 0) or FOLD_SYM (kind 1) matrices, global layout
  const double* W3;
  int ldw2, foldh2, ldw3, foldh3;
  const double* lam1;     // kind 0: coef-scaled eigenvalues, folded spectral order
  const double* lam2;
  const double* lam3;
  int n1, n2, n3, batch;
  int pstride;            // plane stride of the plane-major tensor (n2 n3 rounded up to even)
  int sp;                 // shared-memory row stride of the plane
  int kind;
  double* Y;              // kinds 1-3: output (natural layout), batch stride ybs, optional scale
  long long ybs;
  const double* scale;
  int plane_begin;        // first plane of this problem in the grouped grid
  // kinds 2 / 3 (D = 2, the whole component is the plane): input in the natural layout (i1
  // fastest = the plane's rows), batch stride xbs, optional pre-scaling
  const double* X;
  long long xbs;
  const double* pre;
};
constexpr int kPlaneMax = 8;
struct PlaneGroup {
  PlaneProb prob[kPlaneMax];
  int count;
  int total;              // planes over all problems
  int grid;               // CTAs (persistent over planes)
  // diagnostics: thread 0 of every CTA records %globaltimer at 8 points of its first plane into
  // trace[blockIdx * 8 + point] when non-null
  unsigned long long* trace;
};
size_t plane_smem_bytes(int NT, int sp, int rows);
int plane_stride(int n2);
cudaError_t launch_mode_plane(const PlaneGroup& g, int NT, size_t smem, cudaStream_t s);
cudaError_t prepare_mode_plane(int NT, size_t smem);
cudaError_t prepare_mode_small(int NT);

// Banded m-mode products (kernels/kron_band.cu): factor rows stored as their nonzero band.
struct BandProb {
  const double* X;
  double* Y;
  const double* Wb;   // nout x bw: Wb[a*bw + j] = F[a][lo[a] + j]
  const int* lo;      // first input index of row a's band (lo[a] + bw <= nin)
  int bw, P, nin, nout, Q;
  double alpha, beta; // Y = alpha * result + beta * Y
  int blk_begin;
};
constexpr int kBandMax = 32;
struct BandGroup {
  BandProb prob[kBandMax];
  int count;
  int total_blocks;
};
cudaError_t launch_kron_band(const BandGroup& g, cudaStream_t s);
int kron_band_blocks(long long outputs);

// y[b*ys + i] = x[b*xs + i] * s[i], i < N  (P^G pre-scaling), over `batch` items.
cudaError_t launch_scale(const double* x, double* y, const double* s, long long N, long long batch,
                         long long xs, long long ys, cudaStream_t st);
// Set the dynamic shared-memory attribute of the kernels a tile config uses (call outside capture).
cudaError_t prepare_mode_kernels(const TileCfg& cfg);

// y = beta * y + sum_i coef[i] parts[i] (n elements); up to kMaxParts inputs per launch.
constexpr int kMaxParts = 48;
struct PartSum {
  const double* parts[kMaxParts];
  double coef[kMaxParts];
  int nparts;
};
size_t multidot_scratch_elems(int m);
cudaError_t launch_multidot(const double* V, long long ldv, int m, const double* w, long long n,
                            double* h, double* scratch, cudaStream_t s);
cudaError_t launch_gemv(const double* V, long long ldv, int m, const double* h, double alpha,
                        double* w, double beta, long long n, cudaStream_t s);
cudaError_t launch_copy_indexed(const double* V, long long ldv, const int* idx, double* out,
                                long long n, cudaStream_t s);
cudaError_t launch_store_indexed(double* V, long long ldv, const int* idx, const double* w,
                                 const double* coef, long long n, cudaStream_t s);
cudaError_t launch_multidot_dev(const double* V, long long ldv, const int* m_ptr, int m_max,
                                const double* w, long long n, double* h, double* scratch,
                                cudaStream_t s);
cudaError_t launch_gemv_dev(const double* V, long long ldv, const int* m_ptr, int m_max,
                            const double* h, double alpha, double* w, double beta, long long n,
                            cudaStream_t s);
cudaError_t launch_gmres_scalars(int phase, int* is, double* ds, double* H, int ldh,
                                 const double* h1, const double* h2, double* hist, int m_max,
                                 cudaStream_t s);
cudaError_t launch_lincomb_dev(const double* k, const double* x, const double* y, const double* z,
                               double* out, long long n, cudaStream_t s);
cudaError_t launch_minres_scalars(int phase, double* state, double* hist, int hist_cap, cudaStream_t s);
cudaError_t launch_partsum(const PartSum& ps, double* y, double beta, long long n, cudaStream_t s);

// Geometry-aware setup (host_geo.cpp), wrapped by the C ABI in abi.cpp
fdp_status geometry_coeffs_impl(int kind, int D, int k, int nq, const double* x, double* c_out);
fdp_status separable_fit_impl(int D, const int32_t* nq, const double* const* c, int max_sweeps,
                              double tol, double* tau, double* mu, int* sweeps);

// Vector kernels (vec.cu)
cudaError_t launch_dot(const double* x, const double* y, long long n, double* result,
                       double* scratch, cudaStream_t s);
int dot_scratch_doubles();
cudaError_t launch_lincomb(double a, const double* x, double b, const double* y, double c,
                           const double* z, double* out, long long n, cudaStream_t s);
int iga_mixed_build(int deg_t, int alpha_t, int flags_t, int deg_r, int alpha_r, int flags_r,
                    int n_el, int dtest, int dtrial, int q, const double* wq, double* out,
                    int* n_test, int* n_trial, std::string* err);
int iga_mass_diag_factor_build(int deg, int alpha, int n_el, int flags, int q, double* out,
                               int* n_out, std::string* err);
int iga_quadrature_build(int n_el, int q, double* x, double* w);

// Slab pack (dir 0: z-slab -> piece buffer) / unpack (dir 1, optional scale on the z-slab).
// Peer scatter-copy (pressure blocks of the peer-store slab exchange): src is the local tensor
// with the split axis `a` (extent na) and the other axis `q` (extent nq), i1 fastest; a_outer = 0:
// src (n1, na, nq), a_outer = 1: src (n1, nq, na). Destinations as ModeProb's scatter fields.
struct ScatterDesc {
  double* const* peers;
  int G, na, n1, qoff, a0, a1, q0, q1;
};
cudaError_t launch_slab_scatter(const double* src, const ScatterDesc& sd, int nq, int a_outer,
                                cudaStream_t s);
// Cross-GPU barrier over peer flags (one warp): bumps the caller's epoch counter, release-stores
// it into slot `rank` of every rank's flag array (flags[o], device pointers, mapped via IPC) and
// acquire-spins until all G slots of its own array reach it (system-scope fences).
cudaError_t launch_peer_barrier(unsigned long long* const* flags, unsigned long long* counter,
                                int G, int rank, cudaStream_t s);
cudaError_t launch_slab_copy(const double* src, double* dst, int n1, int n2, int nz, int G, int dir,
                             const double* scale, cudaStream_t s);

// ---------------------------------------------------------------------------------------------
// Banded Kronecker mass solve: per mode, along every fiber of the (P, n, Q) view,
// forward substitution with the banded Cholesky factor L then back substitution with L^T.
// Lb[i*(b+1) + j] = L[i][i-b+j] (j = b is the diagonal, entries with i-b+j < 0 are 0);
// invd[i] = 1/L[i][i]. pre/post: optional scale vectors (length N = P*n*Q/batch) applied on the
// first read / last write.
// ---------------------------------------------------------------------------------------------
struct MassMode {
  const double* in;
  double* out;
  const double* Lb;
  const double* invd;
  const double* Mb;       // FORWARD: band of M, Mb[i*(2b+1) + (j-i+b)] = M[i][j]
  // K3t scaled coefficients, rows of mass_coef_stride(band) doubles (NULL: the sweep kernels):
  // cf[i][k] = L[i][i-band+k] / L[i][i], cb[i][k] = L[i+band-k][i] / L[i][i] (0 past n-1),
  // cf[i][band] = cb[i][band] = 1 / L[i][i]
  const double* cf;
  const double* cb;
  const double* pre;
  const double* post;
  long long N;            // elements per batch item
  long long bs;           // batch-item stride of in/out (elements)
  int P, n, Q, batch;
  int band;
  int forward;            // 1: y = M x along fibers (FDP_MASS_FORWARD)
};
cudaError_t launch_mass_mode(const MassMode& m, cudaStream_t s);
inline int mass_coef_stride(int band) { return (band + 2) & ~1; }
// K3t tensor map (abi_tma.cpp) of the (P, n, Q, batch) fiber view of X with box {F, boxn, 1, 1};
// false when the encoder is unavailable or the view breaks a tensor-map rule.
bool mass_tile_map(CUtensorMap* map, const double* X, int P, int n, long long Q, long long batch,
                   long long bs, int F, int boxn);

// ---------------------------------------------------------------------------------------------
// Host numerics (host_eig.cpp, host_iga.cpp): own implementations, no LAPACK.
// ---------------------------------------------------------------------------------------------
// Generalized symmetric-definite eigenproblem K U = M U diag(lam), U^T M U = I.
// Column-major n x n. Returns 0, or FDP_ERR_NOT_SPD / FDP_ERR_SINGULAR-like codes.
int gen_eig(int n, const double* K, const double* M, double* U, double* lam, std::string* err);
// Banded Cholesky of a symmetric positive definite column-major matrix with half bandwidth b.
int band_cholesky(int n, int b, const double* M, std::vector<double>* Lb, std::vector<double>* invd,
                  std::string* err);
int detect_bandwidth(int n, const double* M);
int spd_inverse_from_band(int n, int b, const std::vector<double>& Lb, std::vector<double>* X);

int iga_build(int deg, int alpha, int n_el, int flags, double c_pen, int q, double* K, double* M,
              int* n_out, std::string* err);
int iga_greville_build(int deg, int alpha, int n_el, int flags, double* g, int* n_out,
                       std::string* err);

}  // namespace fdp
