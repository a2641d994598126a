// C ABI of libfdp (include/fdp.h): handle lifetime, argument validation, error reporting and the
// launch orchestration of the preconditioner application (§4-§5: P_D of P:591-598,
// Algorithm 1 of P:1003-1011, P_Q solve of P:975-976, diagonal scaling of P:1038-1059).
#include "abi_impl.h"

extern "C" const char* fdp_status_string(fdp_status s) {
  switch (s) {
    case FDP_OK: return "FDP_OK";
    case FDP_ERR_INVALID_ARG: return "FDP_ERR_INVALID_ARG";
    case FDP_ERR_SHAPE: return "FDP_ERR_SHAPE";
    case FDP_ERR_NOT_SPD: return "FDP_ERR_NOT_SPD";
    case FDP_ERR_SINGULAR: return "FDP_ERR_SINGULAR";
    case FDP_ERR_CUDA: return "FDP_ERR_CUDA";
    case FDP_ERR_OOM: return "FDP_ERR_OOM";
    case FDP_ERR_NCCL: return "FDP_ERR_NCCL";
    case FDP_ERR_UNSUPPORTED: return "FDP_ERR_UNSUPPORTED";
  }
  return "FDP_ERR_UNKNOWN";
}
extern "C" const char* fdp_last_error(void) { return g_last_error.c_str(); }
extern "C" const char* fdp_version(void) { return "fdp 0.1 sm_100a"; }
// ------------------------------------------------------------------------------------------------
// FD handle
// ------------------------------------------------------------------------------------------------


// ------------------------------------------------------------------------------------------------
// Even-odd folding (DESIGN.md §5 "folded transforms"). J = index reversal. A persymmetric pencil
// (J K J = K, J M J = M: every pencil of the cube configurations, open uniform knots with the
// same boundary treatment at both ends) is block-diagonalised by the orthogonal
//   Q = [q^E_0 .. q^E_{ne-1} | q^O_0 .. q^O_{no-1}],  q^E_k = (e_k + e_{n-1-k}) / sqrt2 (k < no),
//   q^E_h = e_h (odd n, h = no),  q^O_k = (e_k - e_{n-1-k}) / sqrt2,
// so K U = M U Lambda splits into the ne x ne and no x no pencils Q_E^T (K, M) Q_E and
// Q_O^T (K, M) Q_O (P:990-996 on each block), U = Q diag(V_E, V_O), U^T M U = I unchanged.
// ------------------------------------------------------------------------------------------------
bool persymmetric(int n, const double* A, double rtol) {
  double mx = 0.0, dev = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const double a = A[i + (size_t)n * j];
      mx = std::max(mx, std::fabs(a));
      dev = std::max(dev, std::fabs(a - A[(n - 1 - i) + (size_t)n * (n - 1 - j)]));
    }
  return dev <= rtol * mx;
}

// Q_X^T A Q_X (X = E: sign +1, X = O: sign -1), column-major m x m
static std::vector<double> fold_block(int n, const double* A, int sign) {
  const int no = n / 2, m = sign > 0 ? (n + 1) / 2 : no;
  const double r2 = std::sqrt(0.5);
  auto a = [&](int i, int j) { return A[i + (size_t)n * j]; };
  std::vector<double> B((size_t)m * m);
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < m; ++i) {
      const bool mi = i == no, mj = j == no;  // middle of an odd n (E only)
      double v;
      if (mi && mj) v = a(no, no);
      else if (mi) v = r2 * (a(no, j) + a(no, n - 1 - j));
      else if (mj) v = r2 * (a(i, no) + a(n - 1 - i, no));
      else
        v = 0.5 * (a(i, j) + sign * a(i, n - 1 - j) + sign * a(n - 1 - i, j) + a(n - 1 - i, n - 1 - j));
      B[i + (size_t)m * j] = v;
    }
  return B;
}

void fold_sym_matrix(int n, const double* A, int foldh, int ldw, std::vector<double>* w) {
  // y = A x: e_c = sum_k W_E[k][c] s_k, o_c = sum_k W_O[k][c] d_k, y_c = e_c + o_c,
  // y_{n-1-c} = e_c - o_c with W_E[k][c] = (A[c][k] + A[c][n-1-k]) / 2 (the middle row k = h:
  // A[c][h] / 2, since s_h = 2 x_h), W_O[k][c] = (A[c][k] - A[c][n-1-k]) / 2.
  const int ne = (n + 1) / 2, no = n / 2;
  w->assign((size_t)2 * foldh * ldw, 0.0);
  auto a = [&](int i, int j) { return A[i + (size_t)n * j]; };
  for (int k = 0; k < ne; ++k)
    for (int c = 0; c < ne; ++c)
      (*w)[(size_t)k * ldw + c] = k == no ? 0.5 * a(c, k) : 0.5 * (a(c, k) + a(c, n - 1 - k));
  for (int k = 0; k < no; ++k)
    for (int c = 0; c < no; ++c)
      (*w)[(size_t)(foldh + k) * ldw + c] = 0.5 * (a(c, k) - a(c, n - 1 - k));
}

// Folded eigen-data of a persymmetric pencil: forward / backward matrices in the folded layout and
// coef * [lambda_E | lambda_O].
static int fold_eig(int n, const double* K, const double* M, double coef, int foldh, int ldw,
                    int ldwb, std::vector<double>* wf, std::vector<double>* wb,
                    std::vector<double>* lam, std::string* err) {
  const int ne = (n + 1) / 2, no = n / 2;
  const double r2 = std::sqrt(0.5);
  std::vector<double> KE = fold_block(n, K, 1), ME = fold_block(n, M, 1);
  std::vector<double> KO = fold_block(n, K, -1), MO = fold_block(n, M, -1);
  std::vector<double> VE((size_t)ne * ne), VO((size_t)no * no), lE(ne), lO(no);
  int st = gen_eig(ne, KE.data(), ME.data(), VE.data(), lE.data(), err);
  if (!st && no > 0) st = gen_eig(no, KO.data(), MO.data(), VO.data(), lO.data(), err);
  if (st) return st;
  wf->assign((size_t)2 * foldh * ldw, 0.0);
  wb->assign((size_t)2 * foldh * ldwb, 0.0);
  // forward W_E[k][a] = V_E[k][a] / sqrt2 (k < no), V_E[h][a] / 2 (middle: s_h = 2 x_h);
  // backward W_E[a][c] = V_E[c][a] / sqrt2 (c < no), V_E[h][a] (middle)
  for (int k = 0; k < ne; ++k)
    for (int a = 0; a < ne; ++a) {
      const double v = VE[k + (size_t)ne * a];
      (*wf)[(size_t)k * ldw + a] = k == no ? 0.5 * v : r2 * v;
      (*wb)[(size_t)a * ldwb + k] = k == no ? v : r2 * v;
    }
  for (int k = 0; k < no; ++k)
    for (int a = 0; a < no; ++a) {
      const double v = r2 * VO[k + (size_t)no * a];
      (*wf)[(size_t)(foldh + k) * ldw + a] = v;
      (*wb)[(size_t)(foldh + a) * ldwb + k] = v;
    }
  lam->resize(n);
  for (int a = 0; a < ne; ++a) (*lam)[a] = coef * lE[a];
  for (int a = 0; a < no; ++a) (*lam)[ne + a] = coef * lO[a];
  return 0;
}

static void free_fd(fdp_fd h) {
  if (!h) return;
  for (int d = 0; d < 3; ++d) {
    cudaFree(h->Wf[d]);
    cudaFree(h->Wb[d]);
    cudaFree(h->lamc[d]);
    cudaFree(h->WfF[d]);
    cudaFree(h->WbF[d]);
    cudaFree(h->lamcF[d]);
    cudaFree(h->WtF[d]);
    cudaFree(h->WtB[d]);
  }
  cudaFree(h->rlam);
  cudaFree(h->ws);
  delete h;
}

extern "C" fdp_status fd_setup(int D, const int32_t* n, const double* const* K,
                               const double* const* M, const double* coef, int device,
                               int64_t max_batch, fdp_fd* out) {
  try {
    if (!out) return fail(FDP_ERR_INVALID_ARG, "fd_setup: out is NULL");
    *out = nullptr;
    if (D < 2 || D > 3) return fail(FDP_ERR_UNSUPPORTED, "fd_setup: D must be 2 or 3");
    if (!n || !K || !M || !coef) return fail(FDP_ERR_INVALID_ARG, "fd_setup: NULL argument");
    if (max_batch < 0) return fail(FDP_ERR_SHAPE, "fd_setup: max_batch < 0");
    long long N = 1;
    for (int d = 0; d < D; ++d) {
      if (n[d] < 1 || n[d] > 2048) return fail(FDP_ERR_SHAPE, "fd_setup: n[d] must be in [1, 2048]");
      if (!K[d] || !M[d]) return fail(FDP_ERR_INVALID_ARG, "fd_setup: NULL K[d] or M[d]");
      if (!(coef[d] > 0.0)) return fail(FDP_ERR_INVALID_ARG, "fd_setup: coef[d] must be > 0");
      if (!symmetric(n[d], K[d]) || !symmetric(n[d], M[d]))
        return fail(FDP_ERR_NOT_SPD, "fd_setup: K[d] or M[d] not symmetric");
      N *= n[d];
    }
    if (is_device_ptr(K[0]) || is_device_ptr(M[0]))
      return fail(FDP_ERR_INVALID_ARG, "fd_setup: K and M must be host arrays");
    std::unique_ptr<fdp_fd_s> h(new (std::nothrow) fdp_fd_s);
    if (!h) return fail(FDP_ERR_OOM, "fd_setup: host allocation");
    h->D = D;
    h->N = N;
    h->device = device;
    for (int d = 0; d < D; ++d) {
      h->n[d] = n[d];
      h->coef[d] = coef[d];
    }
    // Algorithm 1 step 1: generalized eigendecompositions on the host.
    double lmin = 0.0, lmax = 0.0;
    for (int d = 0; d < D; ++d) {
      const int nd = n[d];
      h->U_host[d].resize((size_t)nd * nd);
      h->lam_host[d].resize(nd);
      std::string err;
      int st = gen_eig(nd, K[d], M[d], h->U_host[d].data(), h->lam_host[d].data(), &err);
      if (st) return fail((fdp_status)st, "fd_setup: " + err);
      h->dK[d].resize(nd);
      h->dM[d].resize(nd);
      for (int i = 0; i < nd; ++i) {
        h->dK[d][i] = K[d][i + (size_t)nd * i];
        h->dM[d][i] = M[d][i + (size_t)nd * i];
      }
      lmin += coef[d] * h->lam_host[d].front();
      lmax += coef[d] * h->lam_host[d].back();
    }
    if (!(lmin > 1e-12 * lmax))
      return fail(FDP_ERR_SINGULAR, "fd_setup: Kronecker-sum spectrum not positive (min Lambda <= 1e-12 max Lambda)");

    DeviceGuard dg(device);
    if (!dg.ok) return fail(FDP_ERR_CUDA, "fd_setup: cannot select device");
    fdp_fd raw = h.release();
    for (int d = 0; d < D; ++d) {
      const int nd = n[d];
      TileCfg c = choose_tile(nd);
      raw->cfg[d] = c;
      const int wrows = std::max(c.kpad, c.ldw);  // the fused small kernel reads W^T rows < ldw
      std::vector<double> wf((size_t)wrows * c.ldw, 0.0), wb((size_t)wrows * c.ldw, 0.0);
      const std::vector<double>& U = raw->U_host[d];  // column-major: U[i + n*j]
      for (int k = 0; k < nd; ++k)
        for (int a = 0; a < nd; ++a) {
          wf[(size_t)k * c.ldw + a] = U[k + (size_t)nd * a];  // W[k][a] = U[k][a]
          wb[(size_t)k * c.ldw + a] = U[a + (size_t)nd * k];  // W[k][a] = U[a][k]
        }
      std::vector<double> lc(nd);
      for (int i = 0; i < nd; ++i) lc[i] = coef[d] * raw->lam_host[d][i];
      fdp_status st;
      if ((st = dalloc(&raw->Wf[d], wf.size())) || (st = dalloc(&raw->Wb[d], wb.size())) ||
          (st = dalloc(&raw->lamc[d], lc.size()))) {
        free_fd(raw);
        return st;
      }
      // folded copy for a persymmetric pencil (FDP_NO_FOLD=1 disables): small-path extents use
      // the small kernels (fold 1), larger ones the folded K1 kernels (fold 2)
      const bool persym = std::getenv("FDP_NO_FOLD") == nullptr && nd >= 8 &&
                          persymmetric(nd, K[d], 1e-12) && persymmetric(nd, M[d], 1e-12);
      const bool small_fold = persym && std::getenv("FDP_NO_SMALL") == nullptr &&
                              nd <= kSmallMaxN && c.tiles_n == 1;
      // (FDP_NO_SMALL=1 routes every extent through K1, so the folded K1 kernels also take the
      // small extents then)
      const bool k1_fold = persym && !small_fold &&
                           (nd > kSmallMaxN || std::getenv("FDP_NO_SMALL") != nullptr);
      std::vector<double> lcf = lc;
      if (small_fold || k1_fold) {
        int nt = 0, foldh, ldwf, ldwb;
        if (small_fold) {
          nt = fold_nt(nd);
          foldh = ldwf = ldwb = 4 * nt;  // KPF rows / 8 * NTE columns of the kernel
        } else {
          const int ne = (nd + 1) / 2, no = nd / 2;
          TileCfg cf{}, cb{};
          const int n8e = (ne + 7) / 8, n8o = (no + 7) / 8;
          cf.MT = cb.MT = 2;
          cf.NT = (n8e + (n8e + 11) / 12 - 1) / ((n8e + 11) / 12);   // <= 12 n8-tiles per column tile
          const int te = (n8e + cf.NT - 1) / cf.NT, to = (n8o + cf.NT - 1) / cf.NT;
          cf.tiles_n = te + to;
          cf.ldw = std::max(te, to) * 8 * cf.NT;
          cb.NT = (n8e + (n8e + 5) / 6 - 1) / ((n8e + 5) / 6);       // <= 6: two accumulator sets
          cb.tiles_n = (n8e + cb.NT - 1) / cb.NT;
          cb.ldw = cb.tiles_n * 8 * cb.NT;
          cf.kpad = cb.kpad = c.kpad;
          raw->cfgFf[d] = cf;
          raw->cfgFb[d] = cb;
          raw->tiles_ne[d] = te;
          foldh = ((ne + 31) / 32) * 32;
          ldwf = cf.ldw;
          ldwb = cb.ldw;
        }
        std::vector<double> wff, wbf;
        std::string err;
        const int fst = fold_eig(nd, K[d], M[d], coef[d], foldh, ldwf, ldwb, &wff, &wbf, &lcf, &err);
        if (fst) {
          free_fd(raw);
          return fail((fdp_status)fst, "fd_setup (folded): " + err);
        }
        if (k1_fold) {  // K1t fragment-native chunks (mode 1 is the KMAJ pass)
          const std::vector<double> tf = tma_wt_build(nd, foldh, ldwf, wff, d == 0);
          const std::vector<double> tb = tma_wt_build(nd, foldh, ldwb, wbf, d == 0);
          fdp_status as;
          if ((as = dalloc(&raw->WtF[d], tf.size())) || (as = dalloc(&raw->WtB[d], tb.size()))) {
            free_fd(raw);
            return as;
          }
          cudaError_t e;
          if ((e = cudaMemcpy(raw->WtF[d], tf.data(), tf.size() * 8, cudaMemcpyHostToDevice)) ||
              (e = cudaMemcpy(raw->WtB[d], tb.data(), tb.size() * 8, cudaMemcpyHostToDevice)) ||
              (e = prepare_mode_tma())) {
            free_fd(raw);
            return cuda_fail(e, "fd_setup: K1t chunks");
          }
        }
        raw->fold[d] = small_fold ? 1 : 2;
        raw->fold_nt[d] = nt;
        raw->foldh[d] = foldh;
        raw->ldwF[d] = ldwf;
        raw->ldwFb[d] = ldwb;
        fdp_status fs;
        if ((fs = dalloc(&raw->WfF[d], wff.size())) || (fs = dalloc(&raw->WbF[d], wbf.size()))) {
          free_fd(raw);
          return fs;
        }
        cudaError_t e;
        if ((e = cudaMemcpy(raw->WfF[d], wff.data(), wff.size() * 8, cudaMemcpyHostToDevice)) ||
            (e = cudaMemcpy(raw->WbF[d], wbf.data(), wbf.size() * 8, cudaMemcpyHostToDevice)) ||
            (e = small_fold ? prepare_mode_small(nt) : prepare_mode_kernels(raw->cfgFf[d])) ||
            (e = small_fold ? prepare_mode_plane(nt, 227 * 1024) : prepare_mode_kernels(raw->cfgFb[d]))) {
          free_fd(raw);
          return cuda_fail(e, "fd_setup: folded upload");
        }
      }
      {
        fdp_status fs = dalloc(&raw->lamcF[d], lcf.size());
        if (fs) {
          free_fd(raw);
          return fs;
        }
        cudaError_t e = cudaMemcpy(raw->lamcF[d], lcf.data(), lcf.size() * 8, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
          free_fd(raw);
          return cuda_fail(e, "fd_setup: upload");
        }
      }
      cudaError_t e;
      if ((e = cudaMemcpy(raw->Wf[d], wf.data(), wf.size() * 8, cudaMemcpyHostToDevice)) ||
          (e = cudaMemcpy(raw->Wb[d], wb.data(), wb.size() * 8, cudaMemcpyHostToDevice)) ||
          (e = cudaMemcpy(raw->lamc[d], lc.data(), lc.size() * 8, cudaMemcpyHostToDevice)) ||
          (e = prepare_mode_kernels(c)) || (e = prepare_mode_small(c.NT))) {
        free_fd(raw);
        return cuda_fail(e, "fd_setup: upload");
      }
    }
    if (raw->fold[D - 1] == 2 && D >= 2) {
      // the Lambda pass on K1t multiplies by a stored 1 / Lambda (DESIGN.md §5 "K1t", C-11)
      const int n1p = n1pad(raw), nmid = D == 3 ? raw->n[1] : 1;
      fdp_status st = dalloc(&raw->rlam, (size_t)n1p * nmid * raw->n[D - 1]);
      cudaError_t e = st ? cudaSuccess
                         : launch_rlam(raw->rlam, raw->lamcF[0], D == 3 ? raw->lamcF[1] : nullptr, raw->lamcF[D - 1],
                                       n1p, raw->n[0], nmid, raw->n[D - 1], nullptr);
      if (!st && e == cudaSuccess) e = cudaDeviceSynchronize();
      if (st || e != cudaSuccess) {
        free_fd(raw);
        return st ? st : cuda_fail(e, "fd_setup: 1/Lambda");
      }
    }
    if (max_batch > 0) {
      fdp_status st = dalloc(&raw->ws, (size_t)(2 * max_batch * Npad(raw) + kWsSlack));
      if (st) {
        free_fd(raw);
        return st;
      }
      raw->ws_batch = max_batch;
    }
    *out = raw;
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fd_get_eigs(fdp_fd h, int d, double* U_out, double* lambda_out) {
  try {
    if (!h) return fail(FDP_ERR_INVALID_ARG, "fd_get_eigs: NULL handle");
    if (d < 0 || d >= h->D) return fail(FDP_ERR_SHAPE, "fd_get_eigs: d out of range");
    if (U_out) std::memcpy(U_out, h->U_host[d].data(), h->U_host[d].size() * 8);
    if (lambda_out) std::memcpy(lambda_out, h->lam_host[d].data(), h->lam_host[d].size() * 8);
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

// out[i] = sum_t c_t prod_d f_td[i_d] (i1 fastest) for per-direction diagonals f_td
void kron_diag_accumulate(int D, const int* n, const std::vector<const double*>& f, double c,
                                 double* out) {
  long long N = 1;
  for (int d = 0; d < D; ++d) N *= n[d];
  for (long long i = 0; i < N; ++i) {
    long long t = i;
    double v = c;
    for (int d = 0; d < D; ++d) {
      v *= f[d][t % n[d]];
      t /= n[d];
    }
    out[i] += v;
  }
}

extern "C" fdp_status iga_geometry_coeffs(int kind, int D, int k, int nq, const double* x,
                                          double* c_out) {
  try {
    const fdp_status st = geometry_coeffs_impl(kind, D, k, nq, x, c_out);
    if (st == FDP_ERR_UNSUPPORTED) return fail(st, "iga_geometry_coeffs: the annulus map is 3D only");
    if (st) return fail(st, "iga_geometry_coeffs: bad kind, k, nq or NULL pointer");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status iga_separable_fit(int D, const int32_t* nq, const double* const* c,
                                        int max_sweeps, double tol, double* tau, double* mu,
                                        int* sweeps) {
  try {
    const fdp_status st = separable_fit_impl(D, nq, c, max_sweeps, tol, tau, mu, sweeps);
    if (st) return fail(st, "iga_separable_fit: bad arguments or a sample <= 0 (logs undefined)");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fd_operator_diagonal(fdp_fd h, double* out) {
  try {
    if (!h || !out) return fail(FDP_ERR_INVALID_ARG, "fd_operator_diagonal: NULL argument");
    std::fill(out, out + h->N, 0.0);
    for (int d = 0; d < h->D; ++d) {
      std::vector<const double*> f(h->D);
      for (int e = 0; e < h->D; ++e) f[e] = e == d ? h->dK[e].data() : h->dM[e].data();
      kron_diag_accumulate(h->D, h->n, f, h->coef[d], out);
    }
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" int64_t fd_size(fdp_fd h) { return h ? h->N : 0; }
extern "C" size_t fd_workspace_bytes(fdp_fd h, int64_t batch) {
  try {
    return h && batch > 0 ? (size_t)(2 * batch * Npad(h) + kWsSlack) * sizeof(double) : 0;
  } catch (...) {
    return 0;
  }
}

// One FD problem inside a grouped stage: mode d (0-based), direction fwd/bwd. xld / yld: fiber
// strides of X / Y (n1, or n1p for padded intermediates); mode >= 1 always runs on padded
// intermediates (P counts the n1p leading rows, pad rows stay zero).
static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
static ModeProb make_mode_prob(const fdp_fd_s* h, int d, bool fwd, const double* X, long long xbs,
                               double* Y, long long ybs, int64_t batch, int epi, const double* scale,
                               int xld, int yld) {
  ModeProb p{};
  const int n1p = n1pad(h);
  long long P = 1, Q = 1;
  for (int e = 0; e < d; ++e) P *= (e == 0 ? n1p : h->n[e]);
  for (int e = d + 1; e < h->D; ++e) Q *= h->n[e];
  p.X = X;
  p.Y = Y;
  p.W = fwd ? h->Wf[d] : h->Wb[d];
  p.N = h->N;
  p.xbs = xbs;
  p.ybs = ybs;
  p.P = (int)P;
  p.n = p.nout = h->n[d];
  p.Q = (int)Q;
  p.batch = (int)batch;
  p.ldw = h->cfg[d].ldw;
  p.n1 = n1p;
  p.n1v = h->n[0];
  p.xld = xld;
  p.yld = yld;
  if (d == 0) {
    p.vx = (xld % 2 == 0) && (xbs % 2 == 0) && aligned16(X);
    p.vy = (yld % 2 == 0) && (ybs % 2 == 0) && aligned16(Y);
  } else {
    p.vx = (P % 2 == 0) && (xbs % 2 == 0) && aligned16(X);
    p.vy = (P % 2 == 0) && (ybs % 2 == 0) && aligned16(Y);
  }
  if (std::getenv("FDP_NO_VEC")) p.vx = p.vy = 0;
  p.epi = epi;
  p.scale = scale;
  if (epi == EPI_LAMBDA || epi == EPI_FUSED) {  // spectral order of the (possibly folded) modes
    p.lam0 = h->lamcF[0];
    p.lam1 = h->D == 3 ? h->lamcF[1] : nullptr;
    p.lamcol = h->lamcF[h->D - 1];
    if (epi == EPI_LAMBDA && d == h->D - 1 && yld == n1p) p.rlam = h->rlam;
  }
  const int BM = kK1Warps * 8 * h->cfg[d].MT;
  const long long M = P * Q * batch;
  p.tiles_m = (int)((M + BM - 1) / BM);
  p.tiles_n = h->cfg[d].tiles_n;
  p.fd_work = 1;
  if (h->fold[d]) {
    p.fold = epi == EPI_FUSED ? FOLD_FUSED : (fwd ? FOLD_FWD : FOLD_BWD);
    p.W = fwd ? h->WfF[d] : h->WbF[d];
    p.ldw = fwd ? h->ldwF[d] : h->ldwFb[d];
    p.foldh = h->foldh[d];
    if (h->fold[d] == 2) {
      p.fold_k1 = 1;
      p.tiles_n = fwd ? h->cfgFf[d].tiles_n : h->cfgFb[d].tiles_n;
      p.tiles_ne = h->tiles_ne[d];
      p.Wt = fwd ? h->WtF[d] : h->WtB[d];
    }
  }
  return p;
}

// Small-path grid: one CTA per SM, split over the problems of a group in proportion to their
// DMMA work (prob.ctas, prob.cta_begin, total_ctas). prob.tiles_m must hold the 8-row tile count.
static void alloc_small_ctas(ModeGroup& g, const std::vector<double>& w) {
  const int total = num_sms();
  double wsum = 0.0;
  for (int j = 0; j < g.count; ++j) wsum += w[j];
  if (!(wsum > 0.0)) wsum = 1.0;
  int used = 0;
  for (int j = 0; j < g.count; ++j) {
    ModeProb& p = g.prob[j];
    int c = std::max(1, (int)(total * w[j] / wsum));
    c = std::min(c, std::max(1, (p.tiles_m + 7) / 8));  // no more warps than 8-row tiles
    p.ctas = c;
    used += c;
  }
  while (used < total) {  // leftover CTAs to the problems with the most work per CTA
    int best = -1;
    double bw = 0.0;
    for (int j = 0; j < g.count; ++j) {
      const double per = w[j] / g.prob[j].ctas;
      if (g.prob[j].ctas * 8 < g.prob[j].tiles_m && per > bw) { bw = per; best = j; }
    }
    if (best < 0) break;
    ++g.prob[best].ctas;
    ++used;
  }
  int begin = 0;
  for (int j = 0; j < g.count; ++j) {
    g.prob[j].cta_begin = begin;
    begin += g.prob[j].ctas;
  }
  g.total_ctas = begin;
}

static bool small_ok(const ModeProb& p) {
  return p.n <= kSmallMaxN && p.tiles_n == 1 && (long long)p.P * p.Q * p.batch + 8 < (1LL << 31);
}

static double recorded_flops(const ModeProb& p) {
  // algorithmic FLOPs of the transform as executed: dense 2 R n^2 per m-mode product (R = rows),
  // folded 2 R (ne^2 + no^2); dense-inverse pressure passes ride along but are
  // not FD work: their bytes only
  if (!p.fd_work) return 0.0;
  const double rows = (double)p.P * p.Q * p.batch;
  const double ne = (p.n + 1) / 2, no = p.n / 2;
  const double per = p.fold ? 2.0 * rows * (ne * ne + no * no) : 2.0 * rows * p.n * p.n;
  return (p.epi == EPI_FUSED ? 2.0 : 1.0) * per;
}
static double recorded_bytes(const ModeProb& p) {
  const double elems = (double)p.P * p.Q * p.batch * p.n;
  return 16.0 * elems + (p.epi == EPI_SCALE ? 8.0 * p.N : 0.0);
}

// diagnostics (fdp_debug_trace): per-warp phase timestamps of small-path launches
static unsigned long long* g_trace = nullptr;
static size_t g_trace_cap = 0, g_trace_used = 0;

cudaError_t launch_stage(std::vector<ModeProb>& probs_in, const std::vector<TileCfg>& cfgs_in,
                         bool kmaj, cudaStream_t s, int* nlaunch, Recorder* rec) {
  // drop empty problems (e.g. a rank that owns no plane of a short axis)
  std::vector<ModeProb> probs;
  std::vector<TileCfg> cfgs;
  for (size_t i = 0; i < probs_in.size(); ++i)
    if ((long long)probs_in[i].P * probs_in[i].Q * probs_in[i].batch > 0) {
      probs.push_back(probs_in[i]);
      cfgs.push_back(cfgs_in[i]);
    }
  std::vector<bool> done(probs.size(), false);
  for (size_t i = 0; i < probs.size(); ++i) {
    if (done[i]) continue;
    ModeGroup g{};
    g.count = 0;
    int ctas = 0;
    for (size_t j = i; j < probs.size() && g.count < kMaxGroup; ++j) {
      if (done[j] || cfgs[j].NT != cfgs[i].NT || cfgs[j].MT != cfgs[i].MT ||
          (probs[j].fold != FOLD_NONE) != (probs[i].fold != FOLD_NONE) ||
          probs[j].fold_k1 != probs[i].fold_k1 || (probs[i].fold_k1 && g.count >= kSmallGroup))
        continue;
      ModeProb p = probs[j];
      p.cta_begin = ctas;
      ctas += p.tiles_m * p.tiles_n;
      g.prob[g.count++] = p;
      done[j] = true;
    }
    g.total_ctas = ctas;
    // small-n path: every problem fits one column tile of <= 96 columns
    bool small = std::getenv("FDP_NO_SMALL") == nullptr;
    for (int j = 0; j < g.count; ++j) small = small && small_ok(g.prob[j]);
    if (small) {
      std::vector<double> w(g.count);
      for (int j = 0; j < g.count; ++j) {
        ModeProb& p = g.prob[j];
        const long long M = (long long)p.P * p.Q * p.batch;
        p.tiles_m = (int)((M + 7) / 8);
        const int kn = p.fold ? (p.n + 1) / 2 : p.n;  // folded: about half the k4 steps
        w[j] = (double)p.tiles_m * ((kn + 3) / 4) * (p.epi == EPI_FUSED ? 2 : 1);
      }
      alloc_small_ctas(g, w);
    } else {
      for (int j = 0; j < g.count; ++j)  // fused and small-fold passes need the small path
        if (g.prob[j].epi == EPI_FUSED || (g.prob[j].fold && !g.prob[j].fold_k1))
          return cudaErrorInvalidValue;
    }
    if (rec) {
      double fl = 0.0, by = 0.0;
      for (int j = 0; j < g.count; ++j) {
        fl += recorded_flops(g.prob[j]);
        by += recorded_bytes(g.prob[j]);
      }
      cudaError_t e0 = rec->before(0, fl, by);
      if (e0 != cudaSuccess) return e0;
    }
    g.trace = nullptr;
    if (small && g_trace) {
      const size_t need = (size_t)g.total_ctas * 16 * kTracePhases;
      if (g_trace_used + need <= g_trace_cap) {
        g.trace = g_trace + g_trace_used;
        g_trace_used += need;
      }
    }
    // folded K1 problems whose operands a tensor map can describe: the TMA kernel K1t
    bool tma = !small && g.prob[0].fold_k1 && g.count <= kTmaMaxProbs;
    for (int j = 0; j < g.count && tma; ++j)
      tma = tma_eligible(g.prob[j], kmaj) && tma_input_ok(g.prob[j], kmaj);
    if (!small && !tma && g.prob[0].fold_k1) ++g_k1_launches[0];
    cudaError_t e = small ? launch_mode_small(g, cfgs[i].NT, kmaj, s)
                    : tma ? launch_tma_stage(g.prob, g.count, kmaj, s)
                          : launch_mode_group(g, cfgs[i], kmaj, s);
    if (e != cudaSuccess) return e;
    if (nlaunch) ++*nlaunch;
  }
  return cudaSuccess;
}

// Enqueue FD solves for several handles (block components) on stream s.
// in[k], out[k] with batch strides ibs/obs; T[k] workspace with stride N_k. dscale[k] may be NULL.
// Pre-scaling (if any) must already have been applied by the caller (into out[k]) and `in` point
// at it.
// Plane path: D = 3 and every mode of every component folded with one kernel NT
// for modes 2 and 3; returns that NT, or 0 when the path does not apply.
static int plane_nt(const std::vector<const fdp_fd_s*>& hs, const PresPlane* pq) {
  if (std::getenv("FDP_NO_PLANE") || std::getenv("FDP_NO_FUSE") || std::getenv("FDP_NO_SMALL"))
    return 0;
  if (hs.empty() || hs.size() + (pq ? 1 : 0) > (size_t)kPlaneMax) return 0;
  if (hs[0]->D == 2) {  // the whole component is the plane: both modes folded, one kernel NT
    const int nt = hs[0]->fold_nt[0];
    for (const fdp_fd_s* h : hs)
      if (h->D != 2 || h->fold[0] != 1 || h->fold[1] != 1 || h->fold_nt[0] != nt || h->fold_nt[1] != nt)
        return 0;
    if (pq && !(pq->q_fold[0] == 1 && pq->q_fold[1] == 1)) return 0;
    return nt;
  }
  if (hs[0]->D != 3) return 0;
  const int nt = hs[0]->fold_nt[1];
  for (const fdp_fd_s* h : hs) {
    if (h->fold[0] != 1 || h->fold[1] != 1 || h->fold[2] != 1) return 0;
    if (h->fold_nt[1] != nt || h->fold_nt[2] != nt || h->fold_nt[0] != hs[0]->fold_nt[0]) return 0;
  }
  if (pq && !(pq->q_fold[0] == 1 && pq->q_fold[1] == 1 && pq->q_fold[2] == 1)) return 0;
  return nt;
}

// Plane buffer rows: n3, or more when an odd count of 8-row tiles makes the last (masked) 16-row
// tile of the row step read past row n3, or that of the column step read past the last row's
// end (columns up to 16 * t16(n2) - 1 of the last row).
static int plane_rows(int n2, int n3, int sp) {
  auto t16 = [](int n) { return ((n >> 3) + 1) >> 1; };
  return std::max({n3, 16 * t16(n3), n3 - 1 + (16 * t16(n2) + sp - 1) / sp});
}

bool plane_path(const std::vector<const fdp_fd_s*>& hs, const PresPlane* pq, int64_t batch) {
  if (plane_nt(hs, pq) <= 0 || (long long)hs[0]->N * batch >= (1LL << 31)) return false;
  if (hs[0]->D == 2) return true;
  // 3D: at least one plane per SM, else the five small-path passes spread the work wider (one
  // config-2 component alone: 36 us in five passes against 40 us with its 65 planes)
  long long planes = 0;
  for (const fdp_fd_s* h : hs) planes += (long long)h->n[0] * batch;
  if (pq) planes += (long long)pq->n[0] * batch;
  return planes >= num_sms();
}

// fuse_prescale: the inputs are not yet scaled by D^{-1/2} (dscale[k] / pq->pre): the mode-1
// pass scales while it loads (P^G pre-scaling; saves the separate streaming launch)
static cudaError_t enqueue_fd_plane(const std::vector<const fdp_fd_s*>& hs,
                                    const std::vector<const double*>& in, long long ibs,
                                    const std::vector<double*>& out, long long obs,
                                    const std::vector<double*>& T,
                                    const std::vector<const double*>& dscale, int64_t batch,
                                    int nt, cudaStream_t s, int* nlaunch, Recorder* rec,
                                    const PresPlane* pq, bool fuse_prescale) {
  const size_t K = hs.size();
  if (hs[0]->D == 2) {  // one launch: each component (and P_Q) a plane per batch item
    PlaneGroup g{};
    int sp = 4, rows = 8, begin = 0;
    double fl = 0.0, by = 0.0;
    for (size_t k = 0; k < K; ++k) {
      const fdp_fd_s* h = hs[k];
      PlaneProb& q = g.prob[g.count++];
      q.kind = 2;
      q.X = in[k];
      q.xbs = ibs;
      q.pre = fuse_prescale ? dscale[k] : nullptr;
      q.Y = out[k];
      q.ybs = obs;
      q.scale = dscale[k];
      q.W2 = h->WfF[0];
      q.W3 = h->WfF[1];
      q.ldw2 = h->ldwF[0];
      q.foldh2 = h->foldh[0];
      q.ldw3 = h->ldwF[1];
      q.foldh3 = h->foldh[1];
      q.lam2 = h->lamcF[0];  // Lambda = lambda_1[row of the column step] + lambda_2[column]
      q.lam3 = h->lamcF[1];
      q.n1 = 1;
      q.n2 = h->n[0];
      q.n3 = h->n[1];
      q.batch = (int)batch;
      q.sp = plane_stride(q.n2);
      q.plane_begin = begin;
      begin += (int)batch;
      sp = std::max(sp, q.sp);
      rows = std::max(rows, plane_rows(q.n2, q.n3, q.sp));
      for (int d = 0; d < 2; ++d) {
        const double ne = (h->n[d] + 1) / 2, no = h->n[d] / 2;
        fl += 2.0 * 2.0 * (double)(h->N / h->n[d]) * batch * (ne * ne + no * no);
      }
      by += 16.0 * h->N * batch;
    }
    if (pq) {
      PlaneProb& q = g.prob[g.count++];
      q.kind = 3;
      q.X = pq->rq;
      q.xbs = pq->rbs;
      q.pre = fuse_prescale ? pq->pre : nullptr;
      q.Y = pq->out;
      q.ybs = pq->obs;
      q.scale = pq->scale;
      q.W2 = pq->Wq[0];
      q.W3 = pq->Wq[1];
      q.ldw2 = pq->q_ldw[0];
      q.foldh2 = pq->q_foldh[0];
      q.ldw3 = pq->q_ldw[1];
      q.foldh3 = pq->q_foldh[1];
      q.n1 = 1;
      q.n2 = pq->n[0];
      q.n3 = pq->n[1];
      q.batch = (int)batch;
      q.sp = plane_stride(q.n2);
      q.plane_begin = begin;
      begin += (int)batch;
      sp = std::max(sp, q.sp);
      rows = std::max(rows, plane_rows(q.n2, q.n3, q.sp));
      by += 16.0 * pq->n[0] * pq->n[1] * batch;
    }
    g.total = begin;
    const size_t smem = plane_smem_bytes(nt, sp, rows);
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    const int per_sm = smem <= 112 * 1024 ? 2 : 1;
    g.grid = std::min(g.total, per_sm * num_sms());
    if (rec) {
      cudaError_t e0 = rec->before(0, fl, by);
      if (e0 != cudaSuccess) return e0;
    }
    g.trace = nullptr;
    cudaError_t e = launch_mode_plane(g, nt, smem, s);
    if (e != cudaSuccess) return e;
    if (nlaunch) ++*nlaunch;
    return cudaSuccess;
  }
  // L1: mode-1 forward, plane-major output (velocity into T[k], pressure M_1^{-1} into Tq)
  {
    std::vector<ModeProb> probs;
    std::vector<TileCfg> cfgs;
    for (size_t k = 0; k < K; ++k) {
      const fdp_fd_s* h = hs[k];
      const long long Mi = (long long)h->n[1] * h->n[2], Mp = Mi + (Mi & 1);
      ModeProb p = make_mode_prob(h, 0, true, in[k], ibs, T[k], h->n[0] * Mp, batch, EPI_NONE,
                                  nullptr, h->n[0], h->n[0]);
      p.tio = TIO_OUT_T;
      p.tio_ld = (int)Mp;
      p.vy = 0;
      if (fuse_prescale) p.pre = dscale[k];
      probs.push_back(p);
      TileCfg c = h->cfg[0];
      c.NT = h->fold_nt[0];
      cfgs.push_back(c);
    }
    if (pq) {
      ModeProb p{};
      p.X = pq->rq;
      p.xbs = pq->rbs;
      const long long Mqi = (long long)pq->n[1] * pq->n[2], Mqp = Mqi + (Mqi & 1);
      p.Y = pq->Tq;
      p.ybs = pq->n[0] * Mqp;
      p.W = pq->Wq[0];
      p.ldw = pq->q_ldw[0];
      p.foldh = pq->q_foldh[0];
      p.fold = FOLD_SYM;
      p.tio = TIO_OUT_T;
      p.tio_ld = (int)Mqp;
      p.N = (long long)pq->n[0] * pq->n[1] * pq->n[2];
      p.P = 1;
      p.n = p.nout = pq->n[0];
      p.Q = pq->n[1] * pq->n[2];
      p.batch = (int)batch;
      p.n1 = p.n1v = pq->n[0];
      p.xld = p.yld = pq->n[0];
      p.tiles_n = 1;
      if (fuse_prescale) p.pre = pq->pre;
      probs.push_back(p);
      cfgs.push_back(cfgs[0]);
    }
    cudaError_t e = launch_stage(probs, cfgs, true, s, nlaunch, rec);
    if (e != cudaSuccess) return e;
  }
  // L2: the planes
  {
    PlaneGroup g{};
    int sp = 4, rows = 8, begin = 0;
    double fl = 0.0, by = 0.0;
    for (size_t k = 0; k < K; ++k) {
      const fdp_fd_s* h = hs[k];
      PlaneProb& q = g.prob[g.count++];
      const long long Mi = (long long)h->n[1] * h->n[2], Mp = Mi + (Mi & 1);
      q.T = T[k];
      q.tbs = h->n[0] * Mp;
      q.pstride = (int)Mp;
      q.W2 = h->WfF[1];
      q.W3 = h->WfF[2];
      q.ldw2 = h->ldwF[1];
      q.foldh2 = h->foldh[1];
      q.ldw3 = h->ldwF[2];
      q.foldh3 = h->foldh[2];
      q.lam1 = h->lamcF[0];
      q.lam2 = h->lamcF[1];
      q.lam3 = h->lamcF[2];
      q.n1 = h->n[0];
      q.n2 = h->n[1];
      q.n3 = h->n[2];
      q.batch = (int)batch;
      q.sp = plane_stride(q.n2);
      q.kind = 0;
      q.plane_begin = begin;
      begin += q.n1 * (int)batch;
      sp = std::max(sp, q.sp);
      rows = std::max(rows, plane_rows(q.n2, q.n3, q.sp));
      for (int d = 1; d < 3; ++d) {  // forward + backward folded transforms of modes 2 and 3
        const double ne = (h->n[d] + 1) / 2, no = h->n[d] / 2;
        fl += 2.0 * 2.0 * (double)(h->N / h->n[d]) * batch * (ne * ne + no * no);
      }
      by += 16.0 * h->N * batch;
    }
    if (pq) {
      PlaneProb& q = g.prob[g.count++];
      const long long Mqi = (long long)pq->n[1] * pq->n[2], Mqp = Mqi + (Mqi & 1);
      q.T = pq->Tq;
      q.tbs = pq->n[0] * Mqp;
      q.pstride = (int)Mqp;
      q.W2 = pq->Wq[1];
      q.W3 = pq->Wq[2];
      q.ldw2 = pq->q_ldw[1];
      q.foldh2 = pq->q_foldh[1];
      q.ldw3 = pq->q_ldw[2];
      q.foldh3 = pq->q_foldh[2];
      q.n1 = pq->n[0];
      q.n2 = pq->n[1];
      q.n3 = pq->n[2];
      q.batch = (int)batch;
      q.sp = plane_stride(q.n2);
      q.kind = 1;
      q.Y = pq->out;
      q.ybs = pq->obs;
      q.scale = pq->scale;
      q.plane_begin = begin;
      begin += q.n1 * (int)batch;
      sp = std::max(sp, q.sp);
      rows = std::max(rows, plane_rows(q.n2, q.n3, q.sp));
      by += 16.0 * pq->n[0] * pq->n[1] * pq->n[2] * batch;
    }
    g.total = begin;
    const size_t smem = plane_smem_bytes(nt, sp, rows);
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    const int per_sm = smem <= 112 * 1024 ? 2 : 1;
    g.grid = std::min(g.total, per_sm * num_sms());
    if (rec) {
      cudaError_t e0 = rec->before(0, fl, by);
      if (e0 != cudaSuccess) return e0;
    }
    g.trace = nullptr;
    if (g_trace) {
      const size_t need = (size_t)g.grid * 8;
      if (g_trace_used + need <= g_trace_cap) {
        g.trace = g_trace + g_trace_used;
        g_trace_used += need;
      }
    }
    cudaError_t e = launch_mode_plane(g, nt, smem, s);
    if (e != cudaSuccess) return e;
    if (nlaunch) ++*nlaunch;
  }
  // L3: mode-1 backward reading the plane-major tensor (P = n2 n3, Q = 1), natural-layout output
  {
    std::vector<ModeProb> probs;
    std::vector<TileCfg> cfgs;
    for (size_t k = 0; k < K; ++k) {
      const fdp_fd_s* h = hs[k];
      const bool sc = dscale[k] != nullptr;
      const long long Mi = (long long)h->n[1] * h->n[2], Mp = Mi + (Mi & 1);
      ModeProb p = make_mode_prob(h, 0, false, T[k], h->n[0] * Mp, out[k], obs, batch,
                                  sc ? EPI_SCALE : EPI_NONE, dscale[k], h->n[0], h->n[0]);
      // rows = the even plane stride (pad row masked at the store): 16-byte row-pair loads
      p.P = (int)Mp;
      p.Q = 1;
      p.vx = (reinterpret_cast<uintptr_t>(T[k]) & 15) == 0 && ((h->n[0] * Mp) % 2 == 0) &&
             std::getenv("FDP_NO_VEC") == nullptr;
      p.vy = 0;
      p.tio = TIO_OUT_K;
      p.tio_rows = (int)Mi;
      probs.push_back(p);
      TileCfg c = h->cfg[0];
      c.NT = h->fold_nt[0];
      cfgs.push_back(c);
    }
    cudaError_t e = launch_stage(probs, cfgs, false, s, nlaunch, rec);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t enqueue_fd(const std::vector<const fdp_fd_s*>& hs,
                              const std::vector<const double*>& in, long long ibs,
                              const std::vector<double*>& out, long long obs,
                              const std::vector<double*>& T,
                              const std::vector<const double*>& dscale, int64_t batch,
                              cudaStream_t s, int* nlaunch, Recorder* rec, const StageHook& hook,
                              const PresPlane* pq, bool fuse_prescale) {
  const int D = hs[0]->D;
  const size_t K = hs.size();
  if ((pq || !hook) && plane_path(hs, pq, batch))
    return enqueue_fd_plane(hs, in, ibs, out, obs, T, dscale, batch, plane_nt(hs, pq), s, nlaunch,
                            rec, pq, fuse_prescale);
  if (fuse_prescale) return cudaErrorInvalidValue;  // callers check plane_path first
  // Stage list: forward d = 0..D-1, backward d = D-1..0. When every mode of every component is
  // small (single column tile, n <= 96) the mode-D forward / Lambda / mode-D backward triple is
  // one fused pass. Destinations alternate so that the last pass lands in `out`.
  bool fuse = std::getenv("FDP_NO_FUSE") == nullptr && std::getenv("FDP_NO_SMALL") == nullptr;
  for (size_t k = 0; k < K; ++k)
    for (int d = 0; d < D; ++d)
      fuse = fuse && hs[k]->n[d] <= kSmallMaxN && hs[k]->cfg[d].tiles_n == 1;
  struct Stage { int d; bool fwd; bool fused; };
  std::vector<Stage> stages;
  for (int d = 0; d < D; ++d) stages.push_back({d, true, fuse && d == D - 1});
  for (int d = D - 1; d >= 0; --d)
    if (!(fuse && d == D - 1)) stages.push_back({d, false, false});
  const int npass = (int)stages.size();
  for (int pass = 0; pass < npass; ++pass) {
    const Stage& st = stages[pass];
    const int d = st.d;
    const bool first = pass == 0, last = pass == npass - 1;
    std::vector<ModeProb> probs;
    std::vector<TileCfg> cfgs;
    for (size_t k = 0; k < K; ++k) {
      // T[k] holds two padded intermediates (batch x Np each): passes alternate between them
      const long long np = Npad(hs[k]);
      double* buf0 = T[k];
      double* buf1 = T[k] + np * batch;
      const double* src = first ? in[k] : ((pass - 1) % 2 == 0 ? buf0 : buf1);
      const long long sbs = first ? ibs : np;
      double* dst = last ? out[k] : (pass % 2 == 0 ? buf0 : buf1);
      const long long dbs = last ? obs : np;
      const int xld = first ? hs[k]->n[0] : n1pad(hs[k]);
      const int yld = last ? hs[k]->n[0] : n1pad(hs[k]);
      int epi = EPI_NONE;
      const double* sc = nullptr;
      if (st.fused) epi = EPI_FUSED;
      else if (st.fwd && d == D - 1) epi = EPI_LAMBDA;
      if (!st.fwd && d == 0 && dscale[k]) { epi = EPI_SCALE; sc = dscale[k]; }
      probs.push_back(make_mode_prob(hs[k], d, st.fwd, src, sbs, dst, dbs, batch, epi, sc, xld, yld));
      TileCfg c = hs[k]->cfg[d];
      if (hs[k]->fold[d] == 1) c.NT = hs[k]->fold_nt[d];
      if (hs[k]->fold[d] == 2) c = st.fwd ? hs[k]->cfgFf[d] : hs[k]->cfgFb[d];
      cfgs.push_back(c);
      // K1t reads its first pass through a tensor map: a C-ABI input with odd rows or an
      // unaligned base is first copied into the second intermediate with padded rows
      ModeProb& pk = probs.back();
      if (first && d == 0 && tma_eligible(pk, true) && !tma_input_ok(pk, true)) {
        const long long rows = hs[k]->N / hs[k]->n[0];
        if (rec) {
          cudaError_t e0 = rec->before(1, 0.0, 16.0 * hs[k]->N * batch);
          if (e0 != cudaSuccess) return e0;
        }
        cudaError_t e = launch_pad_rows(src, sbs, buf1, np, hs[k]->n[0], n1pad(hs[k]), rows, batch, s);
        if (e != cudaSuccess) return e;
        if (nlaunch) ++*nlaunch;
        pk.X = buf1;
        pk.xld = n1pad(hs[k]);
        pk.xbs = np;
      }
    }
    if (hook) hook(pass, st.fwd, d, probs, cfgs);
    cudaError_t e = launch_stage(probs, cfgs, d == 0, s, nlaunch, rec);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

extern "C" fdp_status fd_apply(fdp_fd h, const double* b, double* x, const double* dscale,
                               int64_t batch, void* workspace, void* stream) {
  try {
    if (!h) return fail(FDP_ERR_INVALID_ARG, "fd_apply: NULL handle");
    if (batch < 0) return fail(FDP_ERR_SHAPE, "fd_apply: batch < 0");
    if (batch == 0) return FDP_OK;
    if (!is_device_ptr(b) || !is_device_ptr(x))
      return fail(FDP_ERR_INVALID_ARG, "fd_apply: b and x must be device pointers");
    if (dscale && !is_device_ptr(dscale))
      return fail(FDP_ERR_INVALID_ARG, "fd_apply: dscale must be a device pointer");
    double* T = static_cast<double*>(workspace);
    if (!T) {
      if (batch > h->ws_batch) return fail(FDP_ERR_SHAPE, "fd_apply: batch exceeds handle max_batch and no workspace given");
      T = h->ws;
    } else if (!is_device_ptr(T)) {
      return fail(FDP_ERR_INVALID_ARG, "fd_apply: workspace must be device memory");
    }
    DeviceGuard dg(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const double* src = b;
    // plane path: the mode-1 pass applies D^{-1/2} while loading; otherwise a streaming launch
    const bool fuse = dscale && plane_path({h}, nullptr, batch);
    if (dscale && !fuse) {  // x <- D^{-1/2} b, then the transforms read x
      FDP_CUDA(launch_scale(b, x, dscale, h->N, batch, h->N, h->N, s), "fd_apply: prescale");
      src = x;
    }
    FDP_CUDA(enqueue_fd({h}, {src}, h->N, {x}, h->N, {T}, {dscale}, batch, s, nullptr, nullptr,
                        nullptr, nullptr, fuse),
             "fd_apply");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fd_destroy(fdp_fd h) {
  try {
    if (!h) return FDP_OK;
    DeviceGuard dg(h->device);
    free_fd(h);
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}


// Diagnostics only (not part of include/fdp.h): route per-warp phase timestamps of subsequent
// small-path launches into a device buffer of `cap` uint64 (NULL disables). Invalidates nothing:
// callers must use fresh buffers / handles so graphs are re-captured.
extern "C" int fdp_debug_trace(unsigned long long* dev_buf, size_t cap) {
  try {
    g_trace = dev_buf;
    g_trace_cap = dev_buf ? cap : 0;
    g_trace_used = 0;
    return 0;
  } catch (...) {
    return -1;
  }
}
// ------------------------------------------------------------------------------------------------
// Kronecker mass handle
// ------------------------------------------------------------------------------------------------

static void free_mass(fdp_mass h) {
  if (!h) return;
  for (int d = 0; d < 3; ++d) {
    cudaFree(h->Lb[d]);
    cudaFree(h->invd[d]);
    cudaFree(h->Mb[d]);
    cudaFree(h->cf[d]);
    cudaFree(h->cb[d]);
  }
  delete h;
}

extern "C" fdp_status kron_mass_setup(int D, const int32_t* n, const double* const* M, int device,
                                      fdp_mass* out) {
  try {
    if (!out) return fail(FDP_ERR_INVALID_ARG, "kron_mass_setup: out is NULL");
    *out = nullptr;
    if (D < 2 || D > 3) return fail(FDP_ERR_UNSUPPORTED, "kron_mass_setup: D must be 2 or 3");
    if (!n || !M) return fail(FDP_ERR_INVALID_ARG, "kron_mass_setup: NULL argument");
    std::unique_ptr<fdp_mass_s> h(new (std::nothrow) fdp_mass_s);
    if (!h) return fail(FDP_ERR_OOM, "kron_mass_setup: host allocation");
    h->D = D;
    h->device = device;
    h->N = 1;
    std::vector<double> Lb[3], invd[3], Mb[3];
    for (int d = 0; d < D; ++d) {
      if (n[d] < 1 || n[d] > 1 << 20) return fail(FDP_ERR_SHAPE, "kron_mass_setup: n[d] out of range");
      if (!M[d]) return fail(FDP_ERR_INVALID_ARG, "kron_mass_setup: NULL M[d]");
      if (!symmetric(n[d], M[d])) return fail(FDP_ERR_NOT_SPD, "kron_mass_setup: M[d] not symmetric");
      h->n[d] = n[d];
      h->N *= n[d];
      const int b = detect_bandwidth(n[d], M[d]);
      if (b > 15) return fail(FDP_ERR_UNSUPPORTED, "kron_mass_setup: half bandwidth > 15");
      h->band[d] = b;
      std::string err;
      int st = band_cholesky(n[d], b, M[d], &Lb[d], &invd[d], &err);
      if (st) return fail((fdp_status)st, "kron_mass_setup: " + err);
      Mb[d].assign((size_t)n[d] * (2 * b + 1), 0.0);
      for (int i = 0; i < n[d]; ++i)
        for (int j = std::max(0, i - b); j <= std::min(n[d] - 1, i + b); ++j)
          Mb[d][(size_t)i * (2 * b + 1) + (j - i + b)] = M[d][i + (size_t)n[d] * j];
    }
    DeviceGuard dg(device);
    if (!dg.ok) return fail(FDP_ERR_CUDA, "kron_mass_setup: cannot select device");
    fdp_mass raw = h.release();
    for (int d = 0; d < D; ++d) raw->Lb_host[d] = Lb[d];
    for (int d = 0; d < D; ++d) {
      fdp_status st;
      // K3t coefficients: the band rows scaled by 1 / L_ii (forward by row, backward by column)
      const int b = raw->band[d], nd = raw->n[d], cs = mass_coef_stride(b);
      std::vector<double> cf((size_t)nd * cs, 0.0), cb((size_t)nd * cs, 0.0);
      for (int i = 0; i < nd; ++i) {
        for (int k = 0; k < b; ++k) {
          cf[(size_t)i * cs + k] = Lb[d][(size_t)i * (b + 1) + k] * invd[d][i];
          const int i2 = i + b - k;
          if (i2 < nd) cb[(size_t)i * cs + k] = Lb[d][(size_t)i2 * (b + 1) + k] * invd[d][i];
        }
        cf[(size_t)i * cs + b] = cb[(size_t)i * cs + b] = invd[d][i];
      }
      if ((st = dalloc(&raw->Lb[d], Lb[d].size())) || (st = dalloc(&raw->invd[d], invd[d].size())) ||
          (st = dalloc(&raw->Mb[d], Mb[d].size())) || (st = dalloc(&raw->cf[d], cf.size())) ||
          (st = dalloc(&raw->cb[d], cb.size()))) {
        free_mass(raw);
        return st;
      }
      cudaError_t e;
      if ((e = cudaMemcpy(raw->Lb[d], Lb[d].data(), Lb[d].size() * 8, cudaMemcpyHostToDevice)) ||
          (e = cudaMemcpy(raw->invd[d], invd[d].data(), invd[d].size() * 8, cudaMemcpyHostToDevice)) ||
          (e = cudaMemcpy(raw->Mb[d], Mb[d].data(), Mb[d].size() * 8, cudaMemcpyHostToDevice)) ||
          (e = cudaMemcpy(raw->cf[d], cf.data(), cf.size() * 8, cudaMemcpyHostToDevice)) ||
          (e = cudaMemcpy(raw->cb[d], cb.data(), cb.size() * 8, cudaMemcpyHostToDevice))) {
        free_mass(raw);
        return cuda_fail(e, "kron_mass_setup: upload");
      }
    }
    *out = raw;
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" int64_t kron_mass_size(fdp_mass h) { return h ? h->N : 0; }

// Enqueue the D per-mode passes of the mass inverse (or forward product) for in -> out.
cudaError_t enqueue_mass(const fdp_mass_s* h, int mode, const double* in, double* out,
                                long long bs, const double* dscale, int64_t batch, cudaStream_t s,
                                int* nlaunch, Recorder* rec) {
  for (int d = 0; d < h->D; ++d) {
    MassMode m{};
    long long P = 1, Q = 1;
    for (int e = 0; e < d; ++e) P *= h->n[e];
    for (int e = d + 1; e < h->D; ++e) Q *= h->n[e];
    m.in = d == 0 ? in : out;
    m.out = out;
    m.Lb = h->Lb[d];
    m.invd = h->invd[d];
    m.Mb = h->Mb[d];
    m.cf = h->cf[d];
    m.cb = h->cb[d];
    m.pre = (d == 0 && mode == FDP_MASS_INVERSE) ? dscale : nullptr;
    m.post = (d == h->D - 1 && mode == FDP_MASS_INVERSE) ? dscale : nullptr;
    m.N = h->N;
    m.bs = bs;
    m.P = (int)P;
    m.n = h->n[d];
    m.Q = (int)Q;
    m.batch = (int)batch;
    m.band = h->band[d];
    m.forward = mode == FDP_MASS_FORWARD;
    if (rec) {
      const double elems = (double)h->N * batch;
      cudaError_t e0 = rec->before(2, 2.0 * 2.0 * (2 * m.band + 1) * elems,
                                   16.0 * elems + (m.pre || m.post ? 8.0 * h->N : 0.0));
      if (e0 != cudaSuccess) return e0;
    }
    cudaError_t e = launch_mass_mode(m, s);
    if (e != cudaSuccess) return e;
    if (nlaunch) ++*nlaunch;
  }
  return cudaSuccess;
}

extern "C" fdp_status kron_mass_apply(fdp_mass h, int mode, const double* b, double* x,
                                      const double* dscale, int64_t batch, void* stream) {
  try {
    if (!h) return fail(FDP_ERR_INVALID_ARG, "kron_mass_apply: NULL handle");
    if (mode != FDP_MASS_INVERSE && mode != FDP_MASS_FORWARD)
      return fail(FDP_ERR_INVALID_ARG, "kron_mass_apply: bad mode");
    if (batch < 0) return fail(FDP_ERR_SHAPE, "kron_mass_apply: batch < 0");
    if (batch == 0) return FDP_OK;
    if (!is_device_ptr(b) || !is_device_ptr(x))
      return fail(FDP_ERR_INVALID_ARG, "kron_mass_apply: b and x must be device pointers");
    if (mode == FDP_MASS_FORWARD) {
      if (dscale) return fail(FDP_ERR_INVALID_ARG, "kron_mass_apply: FORWARD takes no dscale");
      if (b == x) return fail(FDP_ERR_INVALID_ARG, "kron_mass_apply: FORWARD cannot run in place");
    }
    if (dscale && !is_device_ptr(dscale))
      return fail(FDP_ERR_INVALID_ARG, "kron_mass_apply: dscale must be a device pointer");
    DeviceGuard dg(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (mode == FDP_MASS_FORWARD) {
      // out-of-place stencil per mode: b -> x (d=0), x -> tmp (d=1), tmp -> x (d=2) ...
      double* tmp = nullptr;
      FDP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), (size_t)(h->N * batch) * 8, s),
               "kron_mass_apply: temporary");
      const double* src = b;
      for (int d = 0; d < h->D; ++d) {
        double* dst = ((h->D - d) % 2 == 1) ? x : tmp;
        MassMode m{};
        long long P = 1, Q = 1;
        for (int e = 0; e < d; ++e) P *= h->n[e];
        for (int e = d + 1; e < h->D; ++e) Q *= h->n[e];
        m.in = src;
        m.out = dst;
        m.Mb = h->Mb[d];
        m.N = h->N;
        m.bs = h->N;
        m.P = (int)P;
        m.n = h->n[d];
        m.Q = (int)Q;
        m.batch = (int)batch;
        m.band = h->band[d];
        m.forward = 1;
        cudaError_t e = launch_mass_mode(m, s);
        if (e != cudaSuccess) {
          cudaFreeAsync(tmp, s);
          return cuda_fail(e, "kron_mass_apply");
        }
        src = dst;
      }
      FDP_CUDA(cudaFreeAsync(tmp, s), "kron_mass_apply: free");
      return FDP_OK;
    }
    FDP_CUDA(enqueue_mass(h, mode, b, x, h->N, dscale, batch, s, nullptr), "kron_mass_apply");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status kron_mass_destroy(fdp_mass h) {
  try {
    if (!h) return FDP_OK;
    DeviceGuard dg(h->device);
    free_mass(h);
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

// One problem as its own stage (batch-1 helpers: slab phases, Kronecker operators).
cudaError_t run1(ModeProb p, const TileCfg& c, bool kmaj, cudaStream_t s) {
  std::vector<ModeProb> v{p};
  std::vector<TileCfg> cv{c};
  return launch_stage(v, cv, kmaj, s, nullptr, nullptr);
}
