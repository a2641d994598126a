// Geometry-aware pencils, host setup code.
//
//  * iga_geometry_coeffs: diagonal entries c^k_dd of C_k^TH = nu (J^{-1} J^{-T} + D_k D_k^T) |det J|,
//    D_k = J^{-1} e_k (PAPER.md eq. (Q_TH)), nu = 1, at a tensor grid of points, for the
//    identity map or the eighth of the thick annulus (N3-3). J is formed
//    from the map's derivatives and inverted by cofactors.
//  * iga_separable_fit: c^k_dd ~ tau_d(eta_d) prod_{m != d} mu_m(eta_m) (Appendix)
//    by log-domain alternating least squares (N3-2).
#include <cmath>
#include <cstring>
#include <vector>

#include "fdp_internal.h"

namespace {

// J[a][b] = dG_a / d eta_b
void jacobian(int kind, const double* e, double J[3][3]) {
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) J[a][b] = a == b ? 1.0 : 0.0;
  if (kind == FDP_GEOM_ANNULUS) {
    const double a = M_PI / 4.0, r = 1.0 + e[0], th = a * e[1];
    const double c = std::cos(th), s = std::sin(th);
    J[0][0] = c;
    J[0][1] = -a * r * s;
    J[1][0] = s;
    J[1][1] = a * r * c;
  }
}

double inverse3(const double J[3][3], double Ji[3][3]) {
  const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
  Ji[0][0] = c00 / det;
  Ji[1][0] = c01 / det;
  Ji[2][0] = c02 / det;
  Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
  Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
  Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
  Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
  Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
  Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
  return det;
}

}  // namespace

namespace fdp {

// Implementations behind the C ABI wrappers in abi.cpp (which set fdp_last_error).
fdp_status geometry_coeffs_impl(int kind, int D, int k, int nq, const double* x, double* c_out) {
  if (kind != FDP_GEOM_IDENTITY && kind != FDP_GEOM_ANNULUS) return FDP_ERR_INVALID_ARG;
  if (D != 3 && !(D == 2 && kind == FDP_GEOM_IDENTITY)) return FDP_ERR_UNSUPPORTED;
  if (k < 0 || k >= D || nq < 1 || !x || !c_out) return FDP_ERR_INVALID_ARG;
  long long NQ = 1;
  for (int d = 0; d < D; ++d) NQ *= nq;
  std::vector<int> idx(D, 0);
  for (long long i = 0; i < NQ; ++i) {
    long long t = i;
    double e[3] = {0.0, 0.0, 0.0};
    for (int d = 0; d < D; ++d) {
      e[d] = x[t % nq];
      t /= nq;
    }
    double J[3][3], Ji[3][3];
    jacobian(kind, e, J);
    const double det = std::fabs(inverse3(J, Ji));
    for (int d = 0; d < D; ++d) {
      double g = 0.0;  // (J^{-1} J^{-T})_dd
      for (int m = 0; m < 3; ++m) g += Ji[d][m] * Ji[d][m];
      const double dk = Ji[d][k];  // (D_k)_d
      c_out[(long long)d * NQ + i] = (g + dk * dk) * det;
    }
  }
  return FDP_OK;
}

fdp_status separable_fit_impl(int D, const int32_t* nq, const double* const* c, int max_sweeps,
                              double tol, double* tau, double* mu, int* sweeps) {
  if (D < 2 || D > 3 || !nq || !c || !tau || !mu || max_sweeps < 0) return FDP_ERR_INVALID_ARG;
  long long NQ = 1;
  int off[4] = {0, 0, 0, 0};
  for (int d = 0; d < D; ++d) {
    if (nq[d] < 1 || !c[d]) return FDP_ERR_INVALID_ARG;
    NQ *= nq[d];
    off[d + 1] = off[d] + nq[d];
  }
  std::vector<double> L((size_t)D * NQ);
  for (int d = 0; d < D; ++d)
    for (long long i = 0; i < NQ; ++i) {
      if (!(c[d][i] > 0.0)) return FDP_ERR_INVALID_ARG;
      L[(size_t)d * NQ + i] = std::log(c[d][i]);
    }
  // grid index of point i (i1 fastest)
  std::vector<int> gi((size_t)D * NQ);
  for (long long i = 0; i < NQ; ++i) {
    long long t = i;
    for (int d = 0; d < D; ++d) {
      gi[(size_t)d * NQ + i] = (int)(t % nq[d]);
      t /= nq[d];
    }
  }
  std::vector<double> lt(off[D], 0.0), lm(off[D], 0.0);  // log tau_d, log mu_m (concatenated)
  auto at = [&](int d, long long i) { return gi[(size_t)d * NQ + i]; };
  // model_d(i) without direction `skip` (skip = -1: full model)
  auto model = [&](int d, long long i, int skip) {
    double v = lt[off[d] + at(d, i)];
    for (int m = 0; m < D; ++m)
      if (m != d && m != skip) v += lm[off[m] + at(m, i)];
    return v;
  };
  auto objective = [&]() {
    double s = 0.0;
    for (int d = 0; d < D; ++d)
      for (long long i = 0; i < NQ; ++i) {
        const double r = L[(size_t)d * NQ + i] - model(d, i, -1);
        s += r * r;
      }
    return s;
  };
  std::vector<double> acc;
  // init: mu = 1, log tau_d = slice means of log c_d
  for (int d = 0; d < D; ++d) {
    acc.assign(nq[d], 0.0);
    for (long long i = 0; i < NQ; ++i) acc[at(d, i)] += L[(size_t)d * NQ + i];
    for (int j = 0; j < nq[d]; ++j) lt[off[d] + j] = acc[j] / (double)(NQ / nq[d]);
  }
  double prev = objective();
  int sw = 0;
  for (; sw < max_sweeps;) {
    for (int d = 0; d < D; ++d) {  // tau_d: slice mean of L_d - sum_{m != d} log mu_m
      acc.assign(nq[d], 0.0);
      for (long long i = 0; i < NQ; ++i)
        acc[at(d, i)] += L[(size_t)d * NQ + i] - (model(d, i, -1) - lt[off[d] + at(d, i)]);
      for (int j = 0; j < nq[d]; ++j) lt[off[d] + j] = acc[j] / (double)(NQ / nq[d]);
    }
    for (int m = 0; m < D; ++m) {  // mu_m: mean over d != m and the slice of the residual
      acc.assign(nq[m], 0.0);
      for (int d = 0; d < D; ++d) {
        if (d == m) continue;
        for (long long i = 0; i < NQ; ++i) acc[at(m, i)] += L[(size_t)d * NQ + i] - model(d, i, m);
      }
      for (int j = 0; j < nq[m]; ++j) lm[off[m] + j] = acc[j] / ((double)(NQ / nq[m]) * (D - 1));
    }
    for (int m = 0; m < D; ++m) {  // gauge: geometric mean of mu_m = 1
      double g = 0.0;
      for (int j = 0; j < nq[m]; ++j) g += lm[off[m] + j];
      g /= nq[m];
      for (int j = 0; j < nq[m]; ++j) lm[off[m] + j] -= g;
      for (int d = 0; d < D; ++d)
        if (d != m)
          for (int j = 0; j < nq[d]; ++j) lt[off[d] + j] += g;
    }
    ++sw;
    const double cur = objective();
    const bool done = std::fabs(prev - cur) <= tol * std::fmax(std::fabs(prev), 1e-300);
    prev = cur;
    if (done) break;
  }
  for (int j = 0; j < off[D]; ++j) {
    tau[j] = std::exp(lt[j]);
    mu[j] = std::exp(lm[j]);
  }
  if (sweeps) *sweeps = sw;
  return FDP_OK;
}

}  // namespace fdp
