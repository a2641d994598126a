// C ABI: host-only spline helpers (univariate K/M, Greville points, generalized eigenproblem,
// quadrature and mixed weighted matrices).
#include "abi_impl.h"

// ------------------------------------------------------------------------------------------------
// host helpers
// ------------------------------------------------------------------------------------------------
extern "C" fdp_status iga_univariate(int deg, int alpha, int n_el, int flags, double c_pen, int q,
                                     double* K, double* M, int32_t* n_out) {
  try {
    if (!n_out) return fail(FDP_ERR_INVALID_ARG, "iga_univariate: n_out is NULL");
    std::string err;
    int n = 0;
    int st = iga_build(deg, alpha, n_el, flags, c_pen, q, K, M, &n, &err);
    if (st) return fail((fdp_status)st, err);
    *n_out = n;
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status iga_greville(int deg, int alpha, int n_el, int flags, double* g,
                                   int32_t* n_out) {
  try {
    if (!n_out) return fail(FDP_ERR_INVALID_ARG, "iga_greville: n_out is NULL");
    std::string err;
    int n = 0;
    int st = iga_greville_build(deg, alpha, n_el, flags, g, &n, &err);
    if (st) return fail((fdp_status)st, err);
    *n_out = n;
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_kron_diag(int D, const int32_t* n, int T, const double* const* f,
                                    const double* c, int invert, double* out) {
  try {
    if (!n || !f || !c || !out) return fail(FDP_ERR_INVALID_ARG, "fdp_kron_diag: NULL argument");
    if (D < 1 || D > 3 || T < 1) return fail(FDP_ERR_SHAPE, "fdp_kron_diag: D in [1,3], T >= 1");
    int nn[3] = {1, 1, 1};
    long long N = 1;
    for (int d = 0; d < D; ++d) {
      if (n[d] < 1) return fail(FDP_ERR_SHAPE, "fdp_kron_diag: n[d] < 1");
      nn[d] = n[d];
      N *= n[d];
    }
    // per term: the outer product of the direction factors, accumulated slice by slice
    std::fill(out, out + N, 0.0);
    std::vector<double> row((size_t)nn[0]);
    for (int t = 0; t < T; ++t) {
      const double* f1 = f[(size_t)t * D];
      const double* f2 = D > 1 ? f[(size_t)t * D + 1] : nullptr;
      const double* f3 = D > 2 ? f[(size_t)t * D + 2] : nullptr;
      for (int i1 = 0; i1 < nn[0]; ++i1) row[i1] = c[t] * (f1 ? f1[i1] : 1.0);
      for (int i3 = 0; i3 < nn[2]; ++i3)
        for (int i2 = 0; i2 < nn[1]; ++i2) {
          const double w = (f2 ? f2[i2] : 1.0) * (f3 ? f3[i3] : 1.0);
          double* o = out + ((long long)i3 * nn[1] + i2) * nn[0];
          for (int i1 = 0; i1 < nn[0]; ++i1) o[i1] += row[i1] * w;
        }
    }
    if (invert)
      for (long long i = 0; i < N; ++i) {
        if (out[i] == 0.0) return fail(FDP_ERR_INVALID_ARG, "fdp_kron_diag: zero value with invert");
        out[i] = 1.0 / out[i];
      }
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_gen_eig(int n, const double* K, const double* M, double* U,
                                  double* lambda) {
  try {
    if (n < 1) return fail(FDP_ERR_SHAPE, "fdp_gen_eig: n < 1");
    if (!K || !M || !U || !lambda) return fail(FDP_ERR_INVALID_ARG, "fdp_gen_eig: NULL argument");
    std::string err;
    int st = gen_eig(n, K, M, U, lambda, &err);
    if (st) return fail((fdp_status)st, "fdp_gen_eig: " + err);
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

// ------------------------------------------------------------------------------------------------
// host helpers: quadrature points and mixed univariate matrices
// ------------------------------------------------------------------------------------------------
extern "C" fdp_status iga_quadrature(int n_el, int q, double* x, double* w) {
  try {
    if (n_el < 1 || q < 1) return fail(FDP_ERR_SHAPE, "iga_quadrature: n_el, q >= 1");
    iga_quadrature_build(n_el, q, x, w);
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status iga_mixed(int deg_test, int alpha_test, int flags_test, int deg_trial,
                                int alpha_trial, int flags_trial, int n_el, int dtest, int dtrial,
                                int q, const double* wq, double* out, int32_t* n_test,
                                int32_t* n_trial) {
  try {
    if (!n_test || !n_trial) return fail(FDP_ERR_INVALID_ARG, "iga_mixed: NULL size outputs");
    std::string err;
    int a = 0, b = 0;
    int st = iga_mixed_build(deg_test, alpha_test, flags_test, deg_trial, alpha_trial, flags_trial,
                             n_el, dtest, dtrial, q, wq, out, &a, &b, &err);
    if (st) return fail((fdp_status)st, err);
    *n_test = a;
    *n_trial = b;
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status iga_mass_diag_factor(int deg, int alpha, int n_el, int flags, int q, double* out,
                                           int32_t* n_out) {
  try {
    if (!n_out) return fail(FDP_ERR_INVALID_ARG, "iga_mass_diag_factor: n_out is NULL");
    std::string err;
    int n = 0;
    const int st = iga_mass_diag_factor_build(deg, alpha, n_el, flags, q, out, &n, &err);
    if (st) return fail((fdp_status)st, "iga_mass_diag_factor: " + err);
    *n_out = n;
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}
