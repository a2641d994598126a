// Host numerics for fd_setup / kron_mass_setup (Algorithm 1 step 1, PAPER.md P:990-996, 1006;
// banded factorisation of the pressure factors). Own implementations, no LAPACK:
//   gen_eig: Cholesky M = L L^T, C = L^{-1} K L^{-T}, Householder tridiagonalisation of C with
//            accumulated reflectors, implicit QL with Wilkinson shifts, U = L^{-T} V.
// (The oracle uses LAPACK's dsygvd through scipy; the two share no code.)
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "fdp_internal.h"

namespace fdp {

// In-place lower Cholesky of a column-major n x n SPD matrix (upper part ignored).
static bool cholesky_lower(int n, std::vector<double>& A) {
  for (int j = 0; j < n; ++j) {
    double d = A[j + (size_t)n * j];
    for (int k = 0; k < j; ++k) d -= A[j + (size_t)n * k] * A[j + (size_t)n * k];
    if (!(d > 0.0)) return false;
    d = std::sqrt(d);
    A[j + (size_t)n * j] = d;
    for (int i = j + 1; i < n; ++i) {
      double s = A[i + (size_t)n * j];
      for (int k = 0; k < j; ++k) s -= A[i + (size_t)n * k] * A[j + (size_t)n * k];
      A[i + (size_t)n * j] = s / d;
    }
    for (int i = 0; i < j; ++i) A[i + (size_t)n * j] = 0.0;
  }
  return true;
}

// Householder reduction of symmetric T (row-major, n x n) to tridiagonal form; Z (column-major)
// accumulates the orthogonal transformation so that Z^T T_orig Z = tridiag(d, e).
static void tridiagonalize(int n, std::vector<double>& T, std::vector<double>& Z,
                           std::vector<double>& d, std::vector<double>& e) {
  Z.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) Z[i + (size_t)n * i] = 1.0;
  std::vector<double> v(n), p(n), w(n), zs(n);
  for (int k = 0; k + 2 < n; ++k) {
    const int m = n - k - 1;  // length of x = T[k+1.., k]
    double nrm = 0.0;
    for (int i = 0; i < m; ++i) nrm += T[(size_t)(k + 1 + i) * n + k] * T[(size_t)(k + 1 + i) * n + k];
    nrm = std::sqrt(nrm);
    const double x0 = T[(size_t)(k + 1) * n + k];
    double tail = nrm * nrm - x0 * x0;
    if (nrm == 0.0 || tail <= 0.0 * nrm) continue;
    const double alpha = x0 > 0 ? -nrm : nrm;
    for (int i = 0; i < m; ++i) v[i] = T[(size_t)(k + 1 + i) * n + k];
    v[0] -= alpha;
    double vn = 0.0;
    for (int i = 0; i < m; ++i) vn += v[i] * v[i];
    vn = std::sqrt(vn);
    if (vn == 0.0) continue;
    for (int i = 0; i < m; ++i) v[i] /= vn;
    // p = A22 v  (A22 = T[k+1.., k+1..])
    for (int i = 0; i < m; ++i) {
      const double* row = &T[(size_t)(k + 1 + i) * n + (k + 1)];
      double s = 0.0;
      for (int j = 0; j < m; ++j) s += row[j] * v[j];
      p[i] = s;
    }
    double vp = 0.0;
    for (int i = 0; i < m; ++i) vp += v[i] * p[i];
    // A22 <- A22 - v w^T - w v^T with w = 2p - 2(v^T p) v
    for (int i = 0; i < m; ++i) w[i] = 2.0 * p[i] - 2.0 * vp * v[i];
    for (int i = 0; i < m; ++i) {
      double* row = &T[(size_t)(k + 1 + i) * n + (k + 1)];
      for (int j = 0; j < m; ++j) row[j] -= v[i] * w[j] + w[i] * v[j];
    }
    T[(size_t)(k + 1) * n + k] = alpha;
    T[(size_t)k * n + (k + 1)] = alpha;
    for (int i = 1; i < m; ++i) {
      T[(size_t)(k + 1 + i) * n + k] = 0.0;
      T[(size_t)k * n + (k + 1 + i)] = 0.0;
    }
    // Z <- Z H, H = I - 2 v v^T on columns k+1..n-1 (column-major: inner loops contiguous)
    std::fill(zs.begin(), zs.end(), 0.0);
    for (int j = 0; j < m; ++j) {
      const double* zc = &Z[(size_t)n * (k + 1 + j)];
      for (int r = 0; r < n; ++r) zs[r] += zc[r] * v[j];
    }
    for (int j = 0; j < m; ++j) {
      double* zc = &Z[(size_t)n * (k + 1 + j)];
      const double f = 2.0 * v[j];
      for (int r = 0; r < n; ++r) zc[r] -= zs[r] * f;
    }
  }
  d.resize(n);
  e.assign(n, 0.0);
  for (int i = 0; i < n; ++i) d[i] = T[(size_t)i * n + i];
  for (int i = 0; i + 1 < n; ++i) e[i] = T[(size_t)(i + 1) * n + i];
}

// Implicit QL with Wilkinson shifts on tridiag(d, e) (e[i] couples i and i+1), rotating the
// columns of Z (column-major). Returns false on non-convergence.
static bool tridiag_ql(int n, std::vector<double>& d, std::vector<double>& e, std::vector<double>& Z) {
  const double eps = 2.220446049250313e-16;
  for (int l = 0; l < n; ++l) {
    int iter = 0;
    int m;
    do {
      for (m = l; m < n - 1; ++m) {
        const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
        if (std::fabs(e[m]) <= eps * dd) break;
      }
      if (m != l) {
        if (iter++ == 100) return false;
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = d[m] - d[l] + e[l] / (g + (g >= 0 ? std::fabs(r) : -std::fabs(r)));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = std::hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[m] = 0.0;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          double* zi = &Z[(size_t)n * i];
          double* zi1 = &Z[(size_t)n * (i + 1)];
          for (int k = 0; k < n; ++k) {
            f = zi1[k];
            zi1[k] = s * zi[k] + c * f;
            zi[k] = c * zi[k] - s * f;
          }
        }
        if (r == 0.0 && i >= l) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
  return true;
}

int gen_eig(int n, const double* K, const double* M, double* U, double* lam, std::string* err) {
  std::vector<double> L(M, M + (size_t)n * n);
  if (!cholesky_lower(n, L)) {
    if (err) *err = "mass matrix is not symmetric positive definite (Cholesky failed)";
    return FDP_ERR_NOT_SPD;
  }
  // Lr: row-major copy of L so that L(i, k) for k < i is contiguous
  std::vector<double> Lr((size_t)n * n);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) Lr[(size_t)i * n + k] = L[i + (size_t)n * k];
  // Y = L^{-1} K (column-major), column by column forward substitution
  std::vector<double> Y(K, K + (size_t)n * n);
  for (int c = 0; c < n; ++c) {
    double* y = &Y[(size_t)n * c];
    for (int i = 0; i < n; ++i) {
      double s = y[i];
      const double* li = &Lr[(size_t)i * n];
      for (int k = 0; k < i; ++k) s -= li[k] * y[k];
      y[i] = s / li[i];
    }
  }
  // C = L^{-1} Y^T: column c of C solves L x = (row c of Y)
  std::vector<double> C((size_t)n * n);
  std::vector<double> x(n);
  for (int c = 0; c < n; ++c) {
    for (int i = 0; i < n; ++i) x[i] = Y[c + (size_t)n * i];
    for (int i = 0; i < n; ++i) {
      double s = x[i];
      const double* li = &Lr[(size_t)i * n];
      for (int k = 0; k < i; ++k) s -= li[k] * x[k];
      x[i] = s / li[i];
    }
    for (int i = 0; i < n; ++i) C[i + (size_t)n * c] = x[i];
  }
  // symmetrise, store row-major (symmetric, so same array)
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      const double a = 0.5 * (C[i + (size_t)n * j] + C[j + (size_t)n * i]);
      C[i + (size_t)n * j] = C[j + (size_t)n * i] = a;
    }
  std::vector<double> Z, d, e;
  tridiagonalize(n, C, Z, d, e);
  if (!tridiag_ql(n, d, e, Z)) {
    if (err) *err = "tridiagonal QL iteration did not converge";
    return FDP_ERR_SINGULAR;
  }
  // sort ascending
  std::vector<int> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](int a, int b) { return d[a] < d[b]; });
  // U = L^{-T} V (back substitution with L^T per column)
  for (int jj = 0; jj < n; ++jj) {
    const int j = ord[jj];
    lam[jj] = d[j];
    for (int i = 0; i < n; ++i) x[i] = Z[i + (size_t)n * j];
    for (int i = n - 1; i >= 0; --i) {
      double s = x[i];
      for (int k = i + 1; k < n; ++k) s -= L[k + (size_t)n * i] * x[k];
      x[i] = s / L[i + (size_t)n * i];
    }
    // sign: largest-magnitude entry positive (cosmetic)
    int im = 0;
    for (int i = 1; i < n; ++i)
      if (std::fabs(x[i]) > std::fabs(x[im])) im = i;
    const double sg = x[im] < 0 ? -1.0 : 1.0;
    for (int i = 0; i < n; ++i) U[i + (size_t)n * jj] = sg * x[i];
  }
  return FDP_OK;
}

int detect_bandwidth(int n, const double* M) {
  int b = 0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      if (M[i + (size_t)n * j] != 0.0) b = std::max(b, std::abs(i - j));
  return b;
}

int band_cholesky(int n, int b, const double* M, std::vector<double>* Lb, std::vector<double>* invd,
                  std::string* err) {
  // Dense Cholesky restricted to the band (no fill outside the band for SPD banded matrices).
  Lb->assign((size_t)n * (b + 1), 0.0);
  invd->assign(n, 0.0);
  auto L = [&](int i, int j) -> double& { return (*Lb)[(size_t)i * (b + 1) + (j - i + b)]; };
  for (int j = 0; j < n; ++j) {
    double dsum = M[j + (size_t)n * j];
    for (int k = std::max(0, j - b); k < j; ++k) dsum -= L(j, k) * L(j, k);
    if (!(dsum > 0.0)) {
      if (err) *err = "pressure mass factor is not positive definite";
      return FDP_ERR_NOT_SPD;
    }
    const double djj = std::sqrt(dsum);
    L(j, j) = djj;
    (*invd)[j] = 1.0 / djj;
    for (int i = j + 1; i <= std::min(n - 1, j + b); ++i) {
      double s = M[i + (size_t)n * j];
      for (int k = std::max(0, i - b); k < j; ++k) s -= L(i, k) * L(j, k);
      L(i, j) = s / djj;
    }
  }
  return FDP_OK;
}

// Dense inverse of an SPD banded matrix from its band Cholesky factor: solve L L^T X = I column
// by column (X symmetric). Used for the dense-inverse variant of the P_Q solve (C-9).
int spd_inverse_from_band(int n, int b, const std::vector<double>& Lb, std::vector<double>* X) {
  X->assign((size_t)n * n, 0.0);
  auto L = [&](int i, int j) -> double { return Lb[(size_t)i * (b + 1) + (j - i + b)]; };
  std::vector<double> y(n);
  for (int c = 0; c < n; ++c) {
    for (int i = 0; i < n; ++i) {
      double v = (i == c) ? 1.0 : 0.0;
      for (int k = std::max(0, i - b); k < i; ++k) v -= L(i, k) * y[k];
      y[i] = v / L(i, i);
    }
    for (int i = n - 1; i >= 0; --i) {
      double v = y[i];
      for (int k = i + 1; k <= std::min(n - 1, i + b); ++k) v -= L(k, i) * y[k];
      y[i] = v / L(i, i);
    }
    for (int i = 0; i < n; ++i) (*X)[i + (size_t)n * c] = y[i];
  }
  return FDP_OK;
}

}  // namespace fdp
