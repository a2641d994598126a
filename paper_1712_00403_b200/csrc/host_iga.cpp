// Host builder of the univariate isogeometric factors (PAPER.md P:689-707 K, M, K~, M~ and
// P:734-737 pressure mass), used by iga_univariate / iga_greville.
//
// Own implementation, independent of the oracle: B-splines are evaluated span-locally with the
// triangular (knot-difference) table -- the non-zero degree-p functions on a span and their first
// derivatives from the degree-(p-1) row -- and Gauss-Legendre nodes come from Newton iteration on
// the three-term Legendre recurrence. (The oracle uses the full Cox-de Boor recursion of P:184-196
// over all functions and numpy's leggauss.)
#include <cmath>
#include <string>
#include <vector>

#include "fdp_internal.h"

namespace fdp {
namespace {

std::vector<double> knot_vector(int deg, int alpha, int n_el) {
  // open, uniform; interior breakpoints repeated deg - alpha times
  std::vector<double> xi;
  for (int i = 0; i <= deg; ++i) xi.push_back(0.0);
  for (int e = 1; e < n_el; ++e)
    for (int r = 0; r < deg - alpha; ++r) xi.push_back((double)e / n_el);
  for (int i = 0; i <= deg; ++i) xi.push_back(1.0);
  return xi;
}

// Span s (0-based) with xi[s] <= u < xi[s+1], deg <= s <= m-1; u == 1 -> last non-empty span.
int find_span(const std::vector<double>& xi, int deg, int m, double u) {
  if (u >= xi[m]) return m - 1;
  int lo = deg, hi = m;
  while (hi - lo > 1) {
    int mid = (lo + hi) / 2;
    if (u < xi[mid]) hi = mid; else lo = mid;
  }
  return lo;
}

// Non-zero functions N[r] = b_{s-deg+r}(u), r = 0..deg, and first derivatives dN[r].
void span_basis(const std::vector<double>& xi, int deg, int s, double u, double* N, double* dN) {
  // ndu[j][r] (j <= r): basis of degree r on the span; ndu[r][j] (r > j): knot differences
  std::vector<double> ndu((size_t)(deg + 1) * (deg + 1)), left(deg + 1), right(deg + 1);
  auto T = [&](int a, int b) -> double& { return ndu[(size_t)a * (deg + 1) + b]; };
  T(0, 0) = 1.0;
  for (int j = 1; j <= deg; ++j) {
    left[j] = u - xi[s + 1 - j];
    right[j] = xi[s + j] - u;
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      T(j, r) = right[r + 1] + left[j - r];
      const double tmp = T(r, j - 1) / T(j, r);
      T(r, j) = saved + right[r + 1] * tmp;
      saved = left[j - r] * tmp;
    }
    T(j, j) = saved;
  }
  for (int r = 0; r <= deg; ++r) {
    N[r] = T(r, deg);
    double d = 0.0;
    if (deg >= 1) {
      if (r >= 1) d += T(r - 1, deg - 1) / T(deg, r - 1);
      if (r <= deg - 1) d -= T(r, deg - 1) / T(deg, r);
      d *= deg;
    }
    dN[r] = d;
  }
}

void gauss_rule(int q, std::vector<double>* x, std::vector<double>* w) {
  // nodes/weights on [-1, 1]
  x->assign(q, 0.0);
  w->assign(q, 0.0);
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < (q + 1) / 2; ++i) {
    double z = std::cos(pi * (i + 0.75) / (q + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= q; ++k) {
        const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (q == 1) { p1 = z; p0 = 1.0; }
      dp = q * (z * p1 - p0) / (z * z - 1.0);
      const double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    // recompute derivative at the converged node
    double p0 = 1.0, p1 = z;
    for (int k = 2; k <= q; ++k) {
      const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    if (q == 1) { p1 = z; p0 = 1.0; }
    dp = q * (z * p1 - p0) / (z * z - 1.0);
    (*x)[i] = -z;
    (*x)[q - 1 - i] = z;
    const double wt = 2.0 / ((1.0 - z * z) * dp * dp);
    (*w)[i] = wt;
    (*w)[q - 1 - i] = wt;
  }
  if (q % 2 == 1) (*x)[q / 2] = 0.0;
}

}  // namespace

int iga_build(int deg, int alpha, int n_el, int flags, double c_pen, int q, double* K, double* M,
              int* n_out, std::string* err) {
  if (deg < 1 || alpha < -1 || alpha >= deg || n_el < 1) {
    if (err) *err = "iga_univariate: need deg >= 1, -1 <= alpha < deg, n_el >= 1";
    return FDP_ERR_SHAPE;
  }
  const std::vector<double> xi = knot_vector(deg, alpha, n_el);
  const int m = (int)xi.size() - deg - 1;
  const bool interior = flags & FDP_IGA_INTERIOR;
  const int off = interior ? 1 : 0;
  const int n = m - 2 * off;
  if (n < 1) {
    if (err) *err = "iga_univariate: empty space after interior restriction";
    return FDP_ERR_SHAPE;
  }
  *n_out = n;
  if (!K && !M) return FDP_OK;
  if (q <= 0) q = deg + 1;
  std::vector<double> Kf((size_t)m * m, 0.0), Mf((size_t)m * m, 0.0);
  std::vector<double> gx, gw;
  gauss_rule(q, &gx, &gw);
  std::vector<double> N(deg + 1), dN(deg + 1);
  for (int s = deg; s < m; ++s) {
    const double a = xi[s], b = xi[s + 1];
    if (!(b > a)) continue;  // empty span (repeated knot)
    for (int g = 0; g < q; ++g) {
      const double u = 0.5 * (a + b) + 0.5 * (b - a) * gx[g];
      const double wq = 0.5 * (b - a) * gw[g];
      span_basis(xi, deg, s, u, N.data(), dN.data());
      for (int r = 0; r <= deg; ++r)
        for (int c = 0; c <= deg; ++c) {
          const int i = s - deg + r, j = s - deg + c;
          Mf[i + (size_t)m * j] += wq * N[r] * N[c];
          Kf[i + (size_t)m * j] += wq * dN[r] * dN[c];
        }
    }
  }
  if (flags & FDP_IGA_NITSCHE) {
    // K~ = K - [ b_l'(1)b_s(1) - b_l'(0)b_s(0) + b_s'(1)b_l(1) - b_s'(0)b_l(0)
    //            - 2 (c_pen/h)(b_l(1)b_s(1) + b_l(0)b_s(0)) ],  h = 1/n_el
    const double h = 1.0 / n_el;
    std::vector<double> v0(m, 0.0), d0(m, 0.0), v1(m, 0.0), d1(m, 0.0);
    int s0 = find_span(xi, deg, m, 0.0), s1 = find_span(xi, deg, m, 1.0);
    span_basis(xi, deg, s0, 0.0, N.data(), dN.data());
    for (int r = 0; r <= deg; ++r) { v0[s0 - deg + r] = N[r]; d0[s0 - deg + r] = dN[r]; }
    span_basis(xi, deg, s1, 1.0, N.data(), dN.data());
    for (int r = 0; r <= deg; ++r) { v1[s1 - deg + r] = N[r]; d1[s1 - deg + r] = dN[r]; }
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < m; ++i) {
        const double br = d1[i] * v1[j] - d0[i] * v0[j] + d1[j] * v1[i] - d0[j] * v0[i] -
                          2.0 * (c_pen / h) * (v1[i] * v1[j] + v0[i] * v0[j]);
        Kf[i + (size_t)m * j] -= br;
      }
  }
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      if (K) K[i + (size_t)n * j] = Kf[(i + off) + (size_t)m * (j + off)];
      if (M) M[i + (size_t)n * j] = Mf[(i + off) + (size_t)m * (j + off)];
    }
  return FDP_OK;
}

int iga_greville_build(int deg, int alpha, int n_el, int flags, double* g, int* n_out,
                       std::string* err) {
  int n = 0;
  int st = iga_build(deg, alpha, n_el, flags & FDP_IGA_INTERIOR, 0.0, 0, nullptr, nullptr, &n, err);
  if (st) return st;
  *n_out = n;
  if (!g) return FDP_OK;
  const std::vector<double> xi = knot_vector(deg, alpha, n_el);
  const int off = (flags & FDP_IGA_INTERIOR) ? 1 : 0;
  for (int j = 0; j < n; ++j) {
    double s = 0.0;
    for (int r = 1; r <= deg; ++r) s += xi[j + off + r];
    g[j] = s / deg;
  }
  return FDP_OK;
}

int iga_quadrature_build(int n_el, int q, double* x, double* w) {
  std::vector<double> gx, gw;
  gauss_rule(q, &gx, &gw);
  for (int e = 0; e < n_el; ++e) {
    const double a = (double)e / n_el, b = (double)(e + 1) / n_el;
    for (int g = 0; g < q; ++g) {
      if (x) x[e * q + g] = 0.5 * (a + b) + 0.5 * (b - a) * gx[g];
      if (w) w[e * q + g] = 0.5 * (b - a) * gw[g];
    }
  }
  return FDP_OK;
}

// out[i, j] = int wt b_test_i^(dtest) b_trial_j^(dtrial) over the uniform mesh (both spaces live
// on the same n_el elements; each element has exactly one non-empty span in each knot vector).
int iga_mass_diag_factor_build(int deg, int alpha, int n_el, int flags, int q, double* out,
                               int* n_out, std::string* err) {
  int n = 0;
  int st = iga_build(deg, alpha, n_el, flags & FDP_IGA_INTERIOR, 0.0, 0, nullptr, nullptr, &n, err);
  if (st) return st;
  *n_out = n;
  if (!out) return FDP_OK;
  if (q < 1) {
    if (err) *err = "q must be >= 1";
    return FDP_ERR_SHAPE;
  }
  const std::vector<double> xi = knot_vector(deg, alpha, n_el);
  const int m = (int)xi.size() - deg - 1;
  const int off = (flags & FDP_IGA_INTERIOR) ? 1 : 0;
  std::vector<double> gx, gw;
  gauss_rule(q, &gx, &gw);
  std::vector<double> N(deg + 1), dN(deg + 1);
  const long long npts = (long long)n_el * q;
  for (long long i = 0; i < (long long)n * npts; ++i) out[i] = 0.0;
  for (int e = 0; e < n_el; ++e) {
    const double a = (double)e / n_el, b = (double)(e + 1) / n_el;
    const double mid = 0.5 * (a + b);
    const int s = find_span(xi, deg, m, mid);
    for (int g = 0; g < q; ++g) {
      const double u = mid + 0.5 * (b - a) * gx[g];
      const double wt = 0.5 * (b - a) * gw[g];
      span_basis(xi, deg, s, u, N.data(), dN.data());
      for (int r = 0; r <= deg; ++r) {
        const int i = s - deg + r - off;  // basis index within the (restricted) space
        if (i < 0 || i >= n) continue;
        out[i + (size_t)n * (e * q + g)] = wt * N[r] * N[r];
      }
    }
  }
  return FDP_OK;
}

int iga_mixed_build(int deg_t, int alpha_t, int flags_t, int deg_r, int alpha_r, int flags_r,
                    int n_el, int dtest, int dtrial, int q, const double* wq, double* out,
                    int* n_test, int* n_trial, std::string* err) {
  int nt = 0, nr = 0;
  int st = iga_build(deg_t, alpha_t, n_el, flags_t & FDP_IGA_INTERIOR, 0.0, 0, nullptr, nullptr, &nt, err);
  if (st) return st;
  st = iga_build(deg_r, alpha_r, n_el, flags_r & FDP_IGA_INTERIOR, 0.0, 0, nullptr, nullptr, &nr, err);
  if (st) return st;
  *n_test = nt;
  *n_trial = nr;
  if (!out) return FDP_OK;
  if (q <= 0) q = (deg_t + deg_r) / 2 + 2;
  const std::vector<double> xt = knot_vector(deg_t, alpha_t, n_el), xr = knot_vector(deg_r, alpha_r, n_el);
  const int mt = (int)xt.size() - deg_t - 1, mr = (int)xr.size() - deg_r - 1;
  const int ot = (flags_t & FDP_IGA_INTERIOR) ? 1 : 0, orr = (flags_r & FDP_IGA_INTERIOR) ? 1 : 0;
  std::vector<double> full((size_t)mt * mr, 0.0);
  std::vector<double> gx, gw;
  gauss_rule(q, &gx, &gw);
  std::vector<double> Nt(deg_t + 1), dNt(deg_t + 1), Nr(deg_r + 1), dNr(deg_r + 1);
  for (int e = 0; e < n_el; ++e) {
    const double a = (double)e / n_el, b = (double)(e + 1) / n_el;
    const double mid = 0.5 * (a + b);
    const int st_ = find_span(xt, deg_t, mt, mid), sr = find_span(xr, deg_r, mr, mid);
    for (int g = 0; g < q; ++g) {
      const double u = mid + 0.5 * (b - a) * gx[g];
      double wt = 0.5 * (b - a) * gw[g];
      if (wq) wt *= wq[e * q + g];
      span_basis(xt, deg_t, st_, u, Nt.data(), dNt.data());
      span_basis(xr, deg_r, sr, u, Nr.data(), dNr.data());
      for (int i = 0; i <= deg_t; ++i)
        for (int j = 0; j <= deg_r; ++j) {
          const double vt = dtest ? dNt[i] : Nt[i], vr = dtrial ? dNr[j] : Nr[j];
          full[(st_ - deg_t + i) + (size_t)mt * (sr - deg_r + j)] += wt * vt * vr;
        }
    }
  }
  for (int j = 0; j < nr; ++j)
    for (int i = 0; i < nt; ++i) out[i + (size_t)nt * j] = full[(i + ot) + (size_t)mt * (j + orr)];
  return FDP_OK;
}

}  // namespace fdp
