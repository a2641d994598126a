// C ABI of libfdp (include/fdp.h): handle lifetime, argument validation, error reporting and the
// launch orchestration of the preconditioner application (§4-§5: P_D of P:591-598,
// Algorithm 1 of P:1003-1011, P_Q solve of P:975-976, diagonal scaling of P:1038-1059).
#include <algorithm>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "fdp_internal.h"

using namespace fdp;

// ------------------------------------------------------------------------------------------------
// errors
// ------------------------------------------------------------------------------------------------
static thread_local std::string g_last_error;

static fdp_status fail(fdp_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}
// No C++ exception crosses the C ABI: every entry point catches and reports (mostly
// std::bad_alloc from host-side containers). Called from inside a catch handler.
static fdp_status abi_exception(const char* fn) {
  try {
    throw;
  } catch (const std::bad_alloc&) {
    return fail(FDP_ERR_OOM, std::string(fn) + ": host allocation failed");
  } catch (const std::exception& e) {
    return fail(FDP_ERR_INVALID_ARG, std::string(fn) + ": " + e.what());
  } catch (...) {
    return fail(FDP_ERR_INVALID_ARG, std::string(fn) + ": unexpected exception");
  }
}

static fdp_status cuda_fail(cudaError_t e, const char* where) {
  cudaGetLastError();  // clear sticky-free errors
  return fail(FDP_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define FDP_CUDA(call, where)                                  \
  do {                                                         \
    cudaError_t e_ = (call);                                   \
    if (e_ != cudaSuccess) return cuda_fail(e_, where);        \
  } while (0)

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

// A pointer is acceptable as a device operand if the runtime knows it as device or managed memory.
static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static int num_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess &&
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
    return n;
  cudaGetLastError();
  return 148;
}

struct DeviceGuard {  // select the handle's device for the duration of a call, then restore
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) { cudaGetLastError(); prev = -1; }
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    int cur;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

template <class T>
static fdp_status dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) return FDP_OK;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(FDP_ERR_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  return FDP_OK;
}

static bool symmetric(int n, const double* A) {
  double mx = 0.0;
  for (size_t i = 0; i < (size_t)n * n; ++i) mx = std::max(mx, std::fabs(A[i]));
  for (int j = 0; j < n; ++j)
    for (int i = j + 1; i < n; ++i)
      if (std::fabs(A[i + (size_t)n * j] - A[j + (size_t)n * i]) > 1e-12 * mx) return false;
  return true;
}

// ------------------------------------------------------------------------------------------------
// per-launch profiling (events recorded on the launching stream, optionally into a graph)
// ------------------------------------------------------------------------------------------------
struct LaunchInfo {
  int kind;      // 0 K1 mode contraction, 1 K2 scaling, 2 K3 mass
  double flops;  // algorithmic
  double bytes;  // algorithmic DRAM bytes
};
struct Recorder {
  std::vector<cudaEvent_t>* ev = nullptr;
  std::vector<LaunchInfo>* info = nullptr;
  cudaStream_t s = nullptr;
  cudaError_t before(int kind, double flops, double bytes) {
    if (!ev) return cudaSuccess;
    size_t i = info->size();
    if (i >= ev->size()) return cudaErrorInvalidValue;
    info->push_back({kind, flops, bytes});
    return cudaEventRecordWithFlags((*ev)[i], s, cudaEventRecordExternal);
  }
  cudaError_t finish() {
    if (!ev) return cudaSuccess;
    size_t i = info->size();
    if (i >= ev->size()) return cudaErrorInvalidValue;
    return cudaEventRecordWithFlags((*ev)[i], s, cudaEventRecordExternal);
  }
};

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
// FD handle
// ------------------------------------------------------------------------------------------------
struct fdp_fd_s {
  int D = 0;
  int n[3] = {1, 1, 1};
  long long N = 0;
  double coef[3] = {0, 0, 0};
  int device = 0;
  TileCfg cfg[3];
  std::vector<double> U_host[3], lam_host[3];
  std::vector<double> dK[3], dM[3];  // diagonals of the pencils (fd_operator_diagonal)
  double* Wf[3] = {nullptr, nullptr, nullptr};  // forward  W[k][a] = U[k][a]
  double* Wb[3] = {nullptr, nullptr, nullptr};  // backward W[k][a] = U[a][k]
  double* lamc[3] = {nullptr, nullptr, nullptr};  // coef[d] * lambda_d
  double* ws = nullptr;
  int64_t ws_batch = 0;
  int* sync = nullptr;        // plane-pipeline counters (zeroed, self-resetting)
  long long sync_cap = 0;
  int64_t sync_batch = 0;
};

// Intermediate tensors between passes use an even leading dimension n1p (16-byte aligned rows
// and row pairs for vector memory operations); the C-ABI input/output stay unpadded.
static int n1pad(const fdp_fd_s* h) { return h->n[0] + (h->n[0] & 1); }
static long long Npad(const fdp_fd_s* h) { return h->N / h->n[0] * n1pad(h); }

static void free_fd(fdp_fd h) {
  if (!h) return;
  for (int d = 0; d < 3; ++d) {
    cudaFree(h->Wf[d]);
    cudaFree(h->Wb[d]);
    cudaFree(h->lamc[d]);
  }
  cudaFree(h->ws);
  cudaFree(h->sync);
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
      cudaError_t e;
      if ((e = cudaMemcpy(raw->Wf[d], wf.data(), wf.size() * 8, cudaMemcpyHostToDevice)) ||
          (e = cudaMemcpy(raw->Wb[d], wb.data(), wb.size() * 8, cudaMemcpyHostToDevice)) ||
          (e = cudaMemcpy(raw->lamc[d], lc.data(), lc.size() * 8, cudaMemcpyHostToDevice)) ||
          (e = prepare_mode_kernels(c)) || (e = prepare_mode_small(c.NT))) {
        free_fd(raw);
        return cuda_fail(e, "fd_setup: upload");
      }
    }
    {
      const int64_t sb = std::max<int64_t>(1, max_batch);
      const long long cap = 2 * ((long long)raw->n[2] * sb + 1);
      fdp_status st = dalloc(&raw->sync, (size_t)cap);
      if (st) {
        free_fd(raw);
        return st;
      }
      cudaError_t e = cudaMemset(raw->sync, 0, cap * sizeof(int));
      if (e != cudaSuccess) {
        free_fd(raw);
        return cuda_fail(e, "fd_setup: sync init");
      }
      raw->sync_cap = cap;
      raw->sync_batch = sb;
    }
    if (max_batch > 0) {
      fdp_status st = dalloc(&raw->ws, (size_t)(2 * max_batch * Npad(raw)));
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
static void kron_diag_accumulate(int D, const int* n, const std::vector<const double*>& f, double c,
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
    return h && batch > 0 ? (size_t)(2 * batch * Npad(h)) * sizeof(double) : 0;
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
  if (epi == EPI_LAMBDA || epi == EPI_FUSED) {
    p.lam0 = h->lamc[0];
    p.lam1 = h->D == 3 ? h->lamc[1] : nullptr;
    p.lamcol = h->lamc[h->D - 1];
  }
  const int BM = kK1Warps * 8 * h->cfg[d].MT;
  const long long M = P * Q * batch;
  p.tiles_m = (int)((M + BM - 1) / BM);
  p.tiles_n = h->cfg[d].tiles_n;
  p.fd_work = 1;
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
  const double elems = (double)p.P * p.Q * p.batch * p.n;
  // dense-inverse pressure passes ride along but are not FD work: count their bytes only
  return p.fd_work ? (p.epi == EPI_FUSED ? 4.0 : 2.0) * elems * p.n : 0.0;
}
static double recorded_bytes(const ModeProb& p) {
  const double elems = (double)p.P * p.Q * p.batch * p.n;
  return 16.0 * elems + (p.epi == EPI_SCALE ? 8.0 * p.N : 0.0);
}

// diagnostics (fdp_debug_trace): per-warp phase timestamps of small-path launches
static unsigned long long* g_trace = nullptr;
static size_t g_trace_cap = 0, g_trace_used = 0;

static cudaError_t launch_stage(std::vector<ModeProb>& probs_in, const std::vector<TileCfg>& cfgs_in,
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
      if (done[j] || cfgs[j].NT != cfgs[i].NT || cfgs[j].MT != cfgs[i].MT) continue;
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
        w[j] = (double)p.tiles_m * ((p.n + 3) / 4) * (p.epi == EPI_FUSED ? 2 : 1);
      }
      alloc_small_ctas(g, w);
    } else {
      for (int j = 0; j < g.count; ++j)
        if (g.prob[j].epi == EPI_FUSED) return cudaErrorInvalidValue;  // fused needs small path
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
    cudaError_t e = small ? launch_mode_small(g, cfgs[i].NT, kmaj, s)
                          : launch_mode_group(g, cfgs[i], kmaj, s);
    if (e != cudaSuccess) return e;
    if (nlaunch) ++*nlaunch;
  }
  return cudaSuccess;
}

// Plane pipeline: phase-1 problems probs1 (mode 0 fwd or mode 1 bwd) and phase-2 problems probs2
// (mode 1 fwd or mode 0 bwd) of the same tensors in one launch (D = 3, small path, NT <= 10).
// sync: zero-initialised ints (self-resetting), capacity sync_cap.
static cudaError_t launch_pp_stage(std::vector<ModeProb>& probs1, std::vector<ModeProb>& probs2,
                                   int NT, bool kmaj1, int* sync, long long sync_cap,
                                   cudaStream_t s, int* nlaunch, Recorder* rec) {
  if (probs1.size() > (size_t)kSmallGroup || probs2.size() != probs1.size()) return cudaErrorInvalidValue;
  ModeGroup g1{}, g2{};
  g1.count = g2.count = (int)probs1.size();
  std::vector<double> w(g1.count);
  PlaneSync ps{};
  long long off = 0;
  for (int j = 0; j < g1.count; ++j) {
    ModeProb a = probs1[j], b = probs2[j];
    a.tiles_m = (int)(((long long)a.P * a.Q * a.batch + 7) / 8);
    b.tiles_m = (int)(((long long)b.P * b.Q * b.batch + 7) / 8);
    w[j] = (double)a.tiles_m * ((a.n + 3) / 4) + (double)b.tiles_m * ((b.n + 3) / 4);
    g1.prob[j] = a;
    g2.prob[j] = b;
    // planes = the (i3, item) slices; rows per plane of each phase
    const int rpp1 = kmaj1 ? b.n : a.P, rpp2 = kmaj1 ? b.P : a.n, planes = kmaj1 ? b.Q : a.Q;
    ps.cnt_off[j] = (int)off;
    ps.rows_per_plane1[j] = rpp1;
    ps.rows_per_plane2[j] = rpp2;
    off += (long long)planes * a.batch;
  }
  if (off + 1 > sync_cap) return cudaErrorInvalidValue;
  alloc_small_ctas(g1, w);
  for (int j = 0; j < g1.count; ++j) {
    g2.prob[j].ctas = g1.prob[j].ctas;
    g2.prob[j].cta_begin = g1.prob[j].cta_begin;
  }
  g2.total_ctas = g1.total_ctas;
  ps.cnt = sync;
  ps.done = sync + off;
  ps.cnt_total = (int)off;
  if (rec) {
    double fl = 0.0, by = 0.0;
    for (int j = 0; j < g1.count; ++j) {
      fl += recorded_flops(g1.prob[j]) + recorded_flops(g2.prob[j]);
      by += recorded_bytes(g1.prob[j]) + recorded_bytes(g2.prob[j]);
    }
    cudaError_t e0 = rec->before(0, fl, by);
    if (e0 != cudaSuccess) return e0;
  }
  cudaError_t e = launch_mode_pp(g1, g2, ps, NT, kmaj1, s);
  if (e != cudaSuccess) return e;
  if (nlaunch) ++*nlaunch;
  return cudaSuccess;
}

static long long pp_sync_ints(const std::vector<const fdp_fd_s*>& hs, int64_t batch, int extra_n3) {
  long long n = 0;
  for (const fdp_fd_s* h : hs) n += (long long)h->n[2] * batch;
  n += (long long)extra_n3 * batch;
  return n + 1;  // + done counter
}

// Enqueue FD solves for several handles (block components) on stream s.
// in[k], out[k] with batch strides ibs/obs; T[k] workspace with stride N_k. dscale[k] may be NULL.
// Pre-scaling (if any) must already have been applied by the caller (into out[k]) and `in` point
// at it.
using StageHook = std::function<void(int pass, bool fwd, int d, std::vector<ModeProb>&,
                                     std::vector<TileCfg>&)>;
static cudaError_t enqueue_fd(const std::vector<const fdp_fd_s*>& hs,
                              const std::vector<const double*>& in, long long ibs,
                              const std::vector<double*>& out, long long obs,
                              const std::vector<double*>& T,
                              const std::vector<const double*>& dscale, int64_t batch,
                              cudaStream_t s, int* nlaunch, Recorder* rec = nullptr,
                              const StageHook& hook = nullptr, int* sync = nullptr,
                              long long sync_cap = 0) {
  const int D = hs[0]->D;
  const size_t K = hs.size();
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
  // plane pipeline (D = 3): passes (0, 1) and (3, 4) each become one launch
  // (opt-in, FDP_PP=1: with about one 8-row tile per warp per pass at batch 1 the two passes
  // cannot overlap, so the separate launches are as fast)
  bool pp = fuse && D == 3 && sync != nullptr && std::getenv("FDP_PP") != nullptr;
  for (size_t k = 0; k < K; ++k)
    for (int d = 0; d < 2; ++d)
      pp = pp && hs[k]->cfg[d].NT <= kPPMaxNT && hs[k]->cfg[d].NT == hs[0]->cfg[0].NT;
  std::vector<ModeProb> held;  // phase-1 problems waiting for their phase-2 partners
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
      cfgs.push_back(hs[k]->cfg[d]);
    }
    if (hook) hook(pass, st.fwd, d, probs, cfgs);
    if (pp && (pass == 0 || pass == 3)) {
      bool ok = probs.size() <= (size_t)kSmallGroup;
      for (const ModeProb& p : probs) ok = ok && small_ok(p);
      if (ok) {
        held = probs;
        continue;
      }
      pp = false;  // fall back to one launch per pass
    }
    if (pp && (pass == 1 || pass == 4)) {
      bool ok = probs.size() == held.size();
      for (const ModeProb& p : probs) ok = ok && small_ok(p);
      if (ok) {
        const int sync_half = (int)(sync_cap / 2);
        int* sy = pass == 1 ? sync : sync + sync_half;
        cudaError_t e = launch_pp_stage(held, probs, cfgs[0].NT, pass == 1, sy, sync_half, s,
                                        nlaunch, rec);
        if (e == cudaSuccess) {
          held.clear();
          continue;
        }
        if (e != cudaErrorInvalidValue) return e;
      }
      // could not pipeline: launch the held pass, then this one
      std::vector<TileCfg> hc(held.size(), cfgs[0]);
      cudaError_t e = launch_stage(held, hc, pass == 1, s, nlaunch, rec);
      if (e != cudaSuccess) return e;
      held.clear();
    }
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
    if (dscale) {  // x <- D^{-1/2} b, then the transforms read x
      FDP_CUDA(launch_scale(b, x, dscale, h->N, batch, h->N, h->N, s), "fd_apply: prescale");
      src = x;
    }
    const bool sy = batch <= h->sync_batch;
    FDP_CUDA(enqueue_fd({h}, {src}, h->N, {x}, h->N, {T}, {dscale}, batch, s, nullptr, nullptr,
                        nullptr, sy ? h->sync : nullptr, sy ? h->sync_cap : 0),
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

// ------------------------------------------------------------------------------------------------
// Kronecker mass handle
// ------------------------------------------------------------------------------------------------
struct fdp_mass_s {
  int D = 0;
  int n[3] = {1, 1, 1};
  int band[3] = {0, 0, 0};
  long long N = 0;
  int device = 0;
  double* Lb[3] = {nullptr, nullptr, nullptr};
  double* invd[3] = {nullptr, nullptr, nullptr};
  double* Mb[3] = {nullptr, nullptr, nullptr};
  std::vector<double> Lb_host[3];
};

static void free_mass(fdp_mass h) {
  if (!h) return;
  for (int d = 0; d < 3; ++d) {
    cudaFree(h->Lb[d]);
    cudaFree(h->invd[d]);
    cudaFree(h->Mb[d]);
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
      if ((st = dalloc(&raw->Lb[d], Lb[d].size())) || (st = dalloc(&raw->invd[d], invd[d].size())) ||
          (st = dalloc(&raw->Mb[d], Mb[d].size()))) {
        free_mass(raw);
        return st;
      }
      cudaError_t e;
      if ((e = cudaMemcpy(raw->Lb[d], Lb[d].data(), Lb[d].size() * 8, cudaMemcpyHostToDevice)) ||
          (e = cudaMemcpy(raw->invd[d], invd[d].data(), invd[d].size() * 8, cudaMemcpyHostToDevice)) ||
          (e = cudaMemcpy(raw->Mb[d], Mb[d].data(), Mb[d].size() * 8, cudaMemcpyHostToDevice))) {
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
static cudaError_t enqueue_mass(const fdp_mass_s* h, int mode, const double* in, double* out,
                                long long bs, const double* dscale, int64_t batch, cudaStream_t s,
                                int* nlaunch, Recorder* rec = nullptr) {
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

// ------------------------------------------------------------------------------------------------
// block preconditioner
// ------------------------------------------------------------------------------------------------
struct fdp_block_s {
  int D = 0;
  int device = 0;
  std::vector<const fdp_fd_s*> vel;
  const fdp_mass_s* pres = nullptr;
  std::vector<long long> off;  // offsets of u_1..u_D, p within one item; off[D+1] = size
  long long size = 0;
  long long nvel = 0;
  double* dv = nullptr;        // D_V^{-1/2} (sum N_k) or NULL
  double* dq = nullptr;        // D_Q^{-1/2} (n_Q) or NULL
  double* dall = nullptr;      // [D_V^{-1/2} | D_Q^{-1/2}] (ones where absent), dense-P_Q path
  // dense-inverse P_Q path: M_d^{-1} padded to the velocity tile config of mode d, so the
  // pressure passes join the velocity launches of stages 0..D-1 (C-9)
  bool pres_dense = false;
  double* Wq[3] = {nullptr, nullptr, nullptr};
  int q_tiles_n[3] = {0, 0, 0};
  int q_ldw[3] = {0, 0, 0};
  cudaStream_t cap = nullptr;  // private capture stream
  // graph cache
  std::mutex mu;
  struct GraphEntry {
    const double* r;
    double* s;
    void* ws;
    int64_t batch;
    cudaGraphExec_t exec;
    unsigned long long used;
  };
  std::vector<GraphEntry> graphs;  // small LRU cache keyed by (r, s, workspace, batch)
  unsigned long long tick = 0;
  // plane-pipeline counters (zeroed at allocation, self-resetting)
  int* sync = nullptr;
  long long sync_cap = 0;
  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> ev;
  std::vector<LaunchInfo> info;
  // host e2e buffers
  double* e2e_r = nullptr;
  double* e2e_s = nullptr;
  void* e2e_ws = nullptr;
  int64_t e2e_batch = 0;
  // host-buffer pipeline: copy-in / copy-out streams and per-unit events
  cudaStream_t cin = nullptr, cout = nullptr;
  cudaStream_t cs[3] = {nullptr, nullptr, nullptr};  // per-component compute streams (batch 1)
  std::vector<cudaEvent_t> ev_in, ev_done;
  cudaEvent_t ev_start = nullptr;
  // batch-1 pipeline over pinned buffers, captured once per (r_host, s_host) and replayed
  const double* e2e_gr = nullptr;
  double* e2e_gs = nullptr;
  cudaGraphExec_t e2e_graph = nullptr;
};

static void free_block(fdp_block h) {
  if (!h) return;
  for (cudaEvent_t e : h->ev) cudaEventDestroy(e);
  cudaFree(h->sync);
  for (auto& g : h->graphs) cudaGraphExecDestroy(g.exec);
  if (h->cap) cudaStreamDestroy(h->cap);
  cudaFree(h->dv);
  cudaFree(h->dq);
  cudaFree(h->dall);
  for (int d = 0; d < 3; ++d) cudaFree(h->Wq[d]);
  cudaFree(h->e2e_r);
  cudaFree(h->e2e_s);
  cudaFree(h->e2e_ws);
  for (cudaEvent_t e : h->ev_in) cudaEventDestroy(e);
  for (cudaEvent_t e : h->ev_done) cudaEventDestroy(e);
  if (h->e2e_graph) cudaGraphExecDestroy(h->e2e_graph);
  for (cudaStream_t c : h->cs)
    if (c) cudaStreamDestroy(c);
  if (h->ev_start) cudaEventDestroy(h->ev_start);
  if (h->cin) cudaStreamDestroy(h->cin);
  if (h->cout) cudaStreamDestroy(h->cout);
  delete h;
}

extern "C" fdp_status block_precond_setup(int D, const fdp_fd* vel, fdp_mass pres,
                                          const double* dscale_vel, const double* dscale_pres,
                                          fdp_block* out) {
  try {
    if (!out) return fail(FDP_ERR_INVALID_ARG, "block_precond_setup: out is NULL");
    *out = nullptr;
    if (D < 2 || D > 3) return fail(FDP_ERR_UNSUPPORTED, "block_precond_setup: D must be 2 or 3");
    if (!vel || !pres) return fail(FDP_ERR_INVALID_ARG, "block_precond_setup: NULL handle");
    std::unique_ptr<fdp_block_s> h(new (std::nothrow) fdp_block_s);
    if (!h) return fail(FDP_ERR_OOM, "block_precond_setup: host allocation");
    h->D = D;
    h->device = pres->device;
    h->pres = pres;
    long long o = 0;
    for (int k = 0; k < D; ++k) {
      if (!vel[k]) return fail(FDP_ERR_INVALID_ARG, "block_precond_setup: NULL velocity handle");
      if (vel[k]->D != D) return fail(FDP_ERR_SHAPE, "block_precond_setup: velocity handle dimension != D");
      if (vel[k]->device != h->device) return fail(FDP_ERR_INVALID_ARG, "block_precond_setup: handles on different devices");
      h->vel.push_back(vel[k]);
      h->off.push_back(o);
      o += vel[k]->N;
    }
    if (pres->D != D) return fail(FDP_ERR_SHAPE, "block_precond_setup: pressure handle dimension != D");
    h->nvel = o;
    h->off.push_back(o);
    o += pres->N;
    h->off.push_back(o);
    h->size = o;
    if ((dscale_vel && is_device_ptr(dscale_vel)) || (dscale_pres && is_device_ptr(dscale_pres)))
      return fail(FDP_ERR_INVALID_ARG, "block_precond_setup: dscale vectors must be host arrays");
    DeviceGuard dg(h->device);
    fdp_block raw = h.release();
    auto upload_isqrt = [&](const double* src, long long n, double** dst) -> fdp_status {
      std::vector<double> v(n);
      for (long long i = 0; i < n; ++i) {
        if (!(src[i] > 0.0)) return fail(FDP_ERR_INVALID_ARG, "block_precond_setup: dscale entries must be > 0");
        v[i] = 1.0 / std::sqrt(src[i]);
      }
      fdp_status st = dalloc(dst, (size_t)n);
      if (st) return st;
      cudaError_t e = cudaMemcpy(*dst, v.data(), n * 8, cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return cuda_fail(e, "block_precond_setup: upload");
      return FDP_OK;
    };
    fdp_status st = FDP_OK;
    if (dscale_vel) st = upload_isqrt(dscale_vel, raw->nvel, &raw->dv);
    if (!st && dscale_pres) st = upload_isqrt(dscale_pres, pres->N, &raw->dq);
    // P_Q by dense per-mode inverses when every factor is small (2 n flops/entry/mode beat the
    // banded recurrences' latency and ride in the velocity launches); banded otherwise.
    const char* env = std::getenv("FDP_PRESSURE");
    bool dense = true;
    for (int d = 0; d < D; ++d) dense = dense && pres->n[d] <= 160;
    if (env && std::string(env) == "banded") dense = false;
    if (env && std::string(env) == "dense") dense = true;
    for (int d = 0; d < D && dense; ++d)
      for (int k = 1; k < D; ++k) dense = dense && raw->vel[k]->cfg[d].NT == raw->vel[0]->cfg[d].NT;
    if (!st && dense) {
      raw->pres_dense = true;
      for (int d = 0; d < D && !st; ++d) {
        const int nq = pres->n[d];
        const TileCfg& vc = raw->vel[0]->cfg[d];
        const int BN = 8 * vc.NT;
        raw->q_tiles_n[d] = (nq + BN - 1) / BN;
        raw->q_ldw[d] = raw->q_tiles_n[d] * BN;
        const int kpad = ((nq + 15) / 16) * 16;
        std::vector<double> X;
        spd_inverse_from_band(nq, pres->band[d], pres->Lb_host[d], &X);
        std::vector<double> w((size_t)kpad * raw->q_ldw[d], 0.0);
        for (int k = 0; k < nq; ++k)
          for (int a = 0; a < nq; ++a) w[(size_t)k * raw->q_ldw[d] + a] = X[a + (size_t)nq * k];
        st = dalloc(&raw->Wq[d], w.size());
        if (!st) {
          cudaError_t e = cudaMemcpy(raw->Wq[d], w.data(), w.size() * 8, cudaMemcpyHostToDevice);
          if (e != cudaSuccess) st = cuda_fail(e, "block_precond_setup: upload");
        }
      }
      if (!st && (dscale_vel || dscale_pres)) {
        std::vector<double> v(raw->size, 1.0);
        for (long long i = 0; i < raw->nvel && dscale_vel; ++i) v[i] = 1.0 / std::sqrt(dscale_vel[i]);
        for (long long i = 0; i < pres->N && dscale_pres; ++i) v[raw->nvel + i] = 1.0 / std::sqrt(dscale_pres[i]);
        st = dalloc(&raw->dall, v.size());
        if (!st) {
          cudaError_t e = cudaMemcpy(raw->dall, v.data(), v.size() * 8, cudaMemcpyHostToDevice);
          if (e != cudaSuccess) st = cuda_fail(e, "block_precond_setup: upload");
        }
      }
    }
    if (!st) {
      cudaError_t e = cudaStreamCreateWithFlags(&raw->cap, cudaStreamNonBlocking);
      if (e != cudaSuccess) st = cuda_fail(e, "block_precond_setup: stream");
    }
    if (st) {
      free_block(raw);
      return st;
    }
    *out = raw;
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" int64_t block_precond_size(fdp_block h) { return h ? h->size : 0; }
static long long block_ws_elems(const fdp_block_s* h, int64_t batch) {
  long long v = 0;
  for (const fdp_fd_s* f : h->vel) v += 2 * Npad(f);
  return batch * (v + (h->pres_dense ? 2 * h->pres->N : 0));
}
extern "C" size_t block_precond_workspace_bytes(fdp_block h, int64_t batch) {
  try {
    return h && batch > 0 ? (size_t)block_ws_elems(h, batch) * sizeof(double) : 0;
  } catch (...) {
    return 0;
  }
}

static cudaError_t enqueue_block(fdp_block h, const double* r, double* s, int64_t batch, double* ws,
                                 cudaStream_t st, int* nlaunch) {
  Recorder recv;
  Recorder* rec = nullptr;
  if (h->prof) {
    h->info.clear();
    recv.ev = &h->ev;
    recv.info = &h->info;
    recv.s = st;
    rec = &recv;
  }
  const int D = h->D;
  const long long sz = h->size;
  std::vector<const double*> in(D), dsc(D);
  std::vector<double*> out(D), T(D);
  long long toff = 0;
  for (int k = 0; k < D; ++k) {
    in[k] = r + h->off[k];
    out[k] = s + h->off[k];
    T[k] = ws + toff;  // component k workspace: two padded intermediates, 2 x batch x Np_k
    toff += 2 * Npad(h->vel[k]) * batch;
    dsc[k] = h->dv ? h->dv + h->off[k] : nullptr;
  }
  const long long nq = h->pres->N;
  double* Tq1 = ws + toff;
  double* Tq2 = Tq1 + nq * batch;
  const double* rq = r + h->off[D];
  if (h->pres_dense && h->dall) {
    // s <- [D_V^{-1/2} | D_Q^{-1/2}] o r over the whole item (one streaming launch)
    if (rec) {
      cudaError_t e0 = rec->before(1, (double)sz * batch, 16.0 * sz * batch + 8.0 * sz);
      if (e0 != cudaSuccess) return e0;
    }
    cudaError_t e = launch_scale(r, s, h->dall, sz, batch, sz, sz, st);
    if (e != cudaSuccess) return e;
    if (nlaunch) ++*nlaunch;
    for (int k = 0; k < D; ++k) in[k] = s + h->off[k];
    rq = s + h->off[D];
  } else if (h->dv) {
    // s_vel <- D_V^{-1/2} r_vel (one streaming launch over all velocity components)
    if (rec) {
      cudaError_t e0 = rec->before(1, (double)h->nvel * batch, 16.0 * h->nvel * batch + 8.0 * h->nvel);
      if (e0 != cudaSuccess) return e0;
    }
    cudaError_t e = launch_scale(r, s, h->dv, h->nvel, batch, sz, sz, st);
    if (e != cudaSuccess) return e;
    if (nlaunch) ++*nlaunch;
    for (int k = 0; k < D; ++k) in[k] = s + h->off[k];
  }
  StageHook hook = nullptr;
  if (h->pres_dense) {
    // pressure pass d joins forward stage d: rq -> Tq1 -> Tq2 -> s_p (x_d M_d^{-1})
    hook = [&](int pass, bool fwd, int d, std::vector<ModeProb>& probs, std::vector<TileCfg>& cfgs) {
      if (!fwd) return;
      ModeProb p{};
      long long P = 1, Q = 1;
      for (int e = 0; e < d; ++e) P *= h->pres->n[e];
      for (int e = d + 1; e < D; ++e) Q *= h->pres->n[e];
      p.X = d == 0 ? rq : (d % 2 == 1 ? Tq1 : Tq2);
      p.xbs = d == 0 ? sz : nq;
      const bool last = d == D - 1;
      p.Y = last ? s + h->off[D] : (d % 2 == 0 ? Tq1 : Tq2);
      p.ybs = last ? sz : nq;
      p.W = h->Wq[d];
      p.N = nq;
      p.P = (int)P;
      p.n = p.nout = h->pres->n[d];
      p.Q = (int)Q;
      p.batch = (int)batch;
      p.ldw = h->q_ldw[d];
      p.n1 = p.n1v = h->pres->n[0];
      p.xld = p.yld = h->pres->n[0];
      p.vx = p.vy = 0;
      p.epi = (last && h->dall) ? EPI_SCALE : EPI_NONE;
      p.scale = (last && h->dall) ? h->dall + h->off[D] : nullptr;
      const int BM = kK1Warps * 8 * cfgs[0].MT;
      p.tiles_m = (int)((P * Q * batch + BM - 1) / BM);
      p.tiles_n = h->q_tiles_n[d];
      p.fd_work = 0;
      probs.push_back(p);
      cfgs.push_back(cfgs[0]);
      (void)pass;
    };
  }
  const long long need = 2 * pp_sync_ints(h->vel, batch, h->pres_dense && D == 3 ? h->pres->n[2] : 0);
  const bool sy = h->sync && h->sync_cap >= need;
  cudaError_t e = enqueue_fd(h->vel, in, sz, out, sz, T, dsc, batch, st, nlaunch, rec, hook,
                             sy ? h->sync : nullptr, sy ? need : 0);
  if (e != cudaSuccess) return e;
  if (!h->pres_dense) {
    // pressure block by banded per-mode solves: r_p -> s_p
    e = enqueue_mass(h->pres, FDP_MASS_INVERSE, r + h->off[D], s + h->off[D], sz, h->dq, batch, st,
                     nlaunch, rec);
    if (e != cudaSuccess) return e;
  }
  return rec ? rec->finish() : cudaSuccess;
}

extern "C" fdp_status block_precond_profile(fdp_block h, int enable) {
  try {
    if (!h) return fail(FDP_ERR_INVALID_ARG, "block_precond_profile: NULL handle");
    std::lock_guard<std::mutex> lk(h->mu);
    DeviceGuard dg(h->device);
    if (enable && h->ev.empty()) {
      h->ev.resize(64);
      for (auto& e : h->ev) FDP_CUDA(cudaEventCreate(&e), "block_precond_profile: event");
    }
    if ((enable != 0) != h->prof) {
      h->prof = enable != 0;
      for (auto& g : h->graphs) cudaGraphExecDestroy(g.exec);  // re-capture with / without events
      h->graphs.clear();
    }
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" int block_precond_profile_read(fdp_block h, int max, int32_t* kind, float* ms,
                                          double* flops, double* bytes) {
  try {
    if (!h || !h->prof) return -1;
    std::lock_guard<std::mutex> lk(h->mu);
    DeviceGuard dg(h->device);
    const int n = (int)h->info.size();
    for (int i = 0; i < n && i < max; ++i) {
      if (kind) kind[i] = h->info[i].kind;
      if (flops) flops[i] = h->info[i].flops;
      if (bytes) bytes[i] = h->info[i].bytes;
      if (ms) {
        float t = 0.f;
        if (cudaEventElapsedTime(&t, h->ev[i], h->ev[i + 1]) != cudaSuccess) {
          cudaGetLastError();
          return -1;
        }
        ms[i] = t;
      }
    }
    return n;
  } catch (...) {
    return -1;
  }
}

extern "C" int fdp_block_launch_count(fdp_block h, int64_t batch) {
  try {
    if (!h || batch <= 0) return 0;
    int n = 0;
    int D = h->D;
    n += h->dv ? 1 : 0;
    for (int d = 0; d < D; ++d) {
      // components with equal tile config share a launch
      std::vector<int> nts;
      for (int k = 0; k < D; ++k) nts.push_back(h->vel[k]->cfg[d].NT);
      std::sort(nts.begin(), nts.end());
      int groups = (int)(std::unique(nts.begin(), nts.end()) - nts.begin());
      n += 2 * groups;
    }
    bool fuse = std::getenv("FDP_NO_FUSE") == nullptr && std::getenv("FDP_NO_SMALL") == nullptr;
    for (int k = 0; k < D; ++k)
      for (int d = 0; d < D; ++d) fuse = fuse && h->vel[k]->n[d] <= kSmallMaxN && h->vel[k]->cfg[d].tiles_n == 1;
    if (fuse) n -= 1;
    bool pp = fuse && D == 3 && std::getenv("FDP_PP") != nullptr;
    for (int k = 0; k < D; ++k)
      for (int d = 0; d < 2; ++d)
        pp = pp && h->vel[k]->cfg[d].NT <= kPPMaxNT && h->vel[k]->cfg[d].NT == h->vel[0]->cfg[0].NT;
    if (pp) n -= 2;
    if (!h->pres_dense) n += h->pres->D;
    else if (h->dall) n += h->dv ? 0 : 1;
    return n;
  } catch (...) {
    return -1;
  }
}

extern "C" fdp_status block_precond_apply(fdp_block h, const double* r, double* s, int64_t batch,
                                          void* workspace, void* stream) {
  try {
    if (!h) return fail(FDP_ERR_INVALID_ARG, "block_precond_apply: NULL handle");
    if (batch < 0) return fail(FDP_ERR_SHAPE, "block_precond_apply: batch < 0");
    if (batch == 0) return FDP_OK;
    std::lock_guard<std::mutex> lk(h->mu);
    fdp_block_s::GraphEntry* hit = nullptr;
    for (auto& g : h->graphs)
      if (g.r == r && g.s == s && g.ws == workspace && g.batch == batch) hit = &g;
    const bool same = hit != nullptr;
    if (!same) {
      if (!is_device_ptr(r) || !is_device_ptr(s))
        return fail(FDP_ERR_INVALID_ARG, "block_precond_apply: r and s must be device pointers");
      if (!workspace || !is_device_ptr(workspace))
        return fail(FDP_ERR_INVALID_ARG, "block_precond_apply: workspace must be device memory");
    }
    DeviceGuard dg(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    FDP_CUDA(cudaStreamIsCapturing(st, &cs), "block_precond_apply: capture query");
    if (!same && cs != cudaStreamCaptureStatusActive) {
      const long long need =
          2 * pp_sync_ints(h->vel, batch, h->pres_dense && h->D == 3 ? h->pres->n[2] : 0);
      if (h->sync_cap < need) {
        FDP_CUDA(cudaStreamSynchronize(st), "block_precond_apply: sync before realloc");
        cudaFree(h->sync);
        h->sync = nullptr;
        h->sync_cap = 0;
        fdp_status s2 = dalloc(&h->sync, (size_t)need);
        if (s2) return s2;
        FDP_CUDA(cudaMemset(h->sync, 0, need * sizeof(int)), "block_precond_apply: sync init");
        h->sync_cap = need;
      }
    }
    if (cs == cudaStreamCaptureStatusActive) {
      FDP_CUDA(enqueue_block(h, r, s, batch, static_cast<double*>(workspace), st, nullptr),
               "block_precond_apply");
      return FDP_OK;
    }
    if (!same) {
      constexpr size_t kMaxGraphs = 4;
      if (h->graphs.size() >= kMaxGraphs) {  // evict the least recently used
        size_t lru = 0;
        for (size_t i = 1; i < h->graphs.size(); ++i)
          if (h->graphs[i].used < h->graphs[lru].used) lru = i;
        FDP_CUDA(cudaStreamSynchronize(st), "block_precond_apply: evict sync");
        cudaGraphExecDestroy(h->graphs[lru].exec);
        h->graphs.erase(h->graphs.begin() + lru);
      }
      cudaGraph_t g = nullptr;
      FDP_CUDA(cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal), "capture begin");
      cudaError_t e = enqueue_block(h, r, s, batch, static_cast<double*>(workspace), h->cap, nullptr);
      cudaError_t e2 = cudaStreamEndCapture(h->cap, &g);
      if (e != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        return cuda_fail(e, "block_precond_apply: enqueue");
      }
      if (e2 != cudaSuccess) return cuda_fail(e2, "block_precond_apply: capture end");
      cudaGraphExec_t ex = nullptr;
      e = cudaGraphInstantiate(&ex, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) return cuda_fail(e, "block_precond_apply: instantiate");
      h->graphs.push_back({r, s, workspace, batch, ex, 0});
      hit = &h->graphs.back();
    }
    hit->used = ++h->tick;
    FDP_CUDA(cudaGraphLaunch(hit->exec, st), "block_precond_apply: graph launch");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

// One pipeline unit of the host-buffer path at batch 1: velocity component k (k < D) or the
// pressure block (k == D), r -> s on stream st (T: component workspace).
static cudaError_t enqueue_unit(fdp_block h, int k, const double* r, double* s, double* T,
                                cudaStream_t st) {
  if (k == h->D) {
    const double* rq = r + h->off[k];
    double* sq = s + h->off[k];
    if (!h->pres_dense)  // banded per-mode solves
      return enqueue_mass(h->pres, FDP_MASS_INVERSE, rq, sq, h->size, h->dq, 1, st, nullptr);
    // dense per-mode inverses (C-9): three small-path passes rq -> T -> T' -> sq, with the
    // D_Q^{-1/2} scalings as a pre-scale and the last pass's epilogue
    const long long nq = h->pres->N;
    double* T1 = T;
    double* T2 = T + nq;
    const double* dq = h->dall ? h->dall + h->off[k] : nullptr;
    if (dq) {
      cudaError_t e = launch_scale(rq, T2, dq, nq, 1, nq, nq, st);
      if (e != cudaSuccess) return e;
      rq = T2;
    }
    const TileCfg& vc = h->vel[0]->cfg[0];
    for (int d = 0; d < h->D; ++d) {
      long long P = 1, Q = 1;
      for (int e = 0; e < d; ++e) P *= h->pres->n[e];
      for (int e = d + 1; e < h->D; ++e) Q *= h->pres->n[e];
      const bool last = d == h->D - 1;
      ModeProb p{};
      p.X = d == 0 ? rq : (d % 2 == 1 ? T1 : T2);
      p.Y = last ? sq : (d % 2 == 0 ? T1 : T2);
      p.W = h->Wq[d];
      p.N = nq;
      p.P = (int)P;
      p.n = p.nout = h->pres->n[d];
      p.Q = (int)Q;
      p.batch = 1;
      p.ldw = h->q_ldw[d];
      p.n1 = p.n1v = h->pres->n[0];
      p.xld = p.yld = h->pres->n[0];
      p.epi = (last && dq) ? EPI_SCALE : EPI_NONE;
      p.scale = (last && dq) ? dq : nullptr;
      const int BM = kK1Warps * 8 * vc.MT;
      p.tiles_m = (int)((P * Q + BM - 1) / BM);
      p.tiles_n = h->q_tiles_n[d];
      std::vector<ModeProb> probs{p};
      std::vector<TileCfg> cfgs{h->vel[0]->cfg[d]};
      cudaError_t e = launch_stage(probs, cfgs, d == 0, st, nullptr, nullptr);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  const fdp_fd_s* f = h->vel[k];
  const double* in = r + h->off[k];
  const double* dsc = h->dv ? h->dv + h->off[k] : nullptr;
  if (dsc) {
    cudaError_t e = launch_scale(in, s + h->off[k], dsc, f->N, 1, f->N, f->N, st);
    if (e != cudaSuccess) return e;
    in = s + h->off[k];
  }
  return enqueue_fd({f}, {in}, f->N, {s + h->off[k]}, f->N, {T}, {dsc}, 1, st, nullptr);
}

extern "C" fdp_status block_precond_apply_host(fdp_block h, const double* r_host, double* s_host,
                                               int64_t batch, void* stream) {
  try {
    if (!h) return fail(FDP_ERR_INVALID_ARG, "block_precond_apply_host: NULL handle");
    if (!r_host || !s_host) return fail(FDP_ERR_INVALID_ARG, "block_precond_apply_host: NULL buffer");
    if (batch <= 0) return batch == 0 ? FDP_OK : fail(FDP_ERR_SHAPE, "block_precond_apply_host: batch < 0");
    std::lock_guard<std::mutex> lk(h->mu);
    DeviceGuard dg(h->device);
    if (batch > h->e2e_batch) {
      cudaFree(h->e2e_r);
      cudaFree(h->e2e_s);
      cudaFree(h->e2e_ws);
      h->e2e_r = h->e2e_s = nullptr;
      h->e2e_ws = nullptr;
      h->e2e_batch = 0;
      fdp_status st;
      if ((st = dalloc(&h->e2e_r, (size_t)(batch * h->size))) ||
          (st = dalloc(&h->e2e_s, (size_t)(batch * h->size))) ||
          (st = dalloc(reinterpret_cast<double**>(&h->e2e_ws), (size_t)block_ws_elems(h, batch))))
        return st;
      h->e2e_batch = batch;
      if (h->e2e_graph) {  // captured against the old device buffers
        cudaGraphExecDestroy(h->e2e_graph);
        h->e2e_graph = nullptr;
      }
    }
    if (!h->cin) {
      FDP_CUDA(cudaStreamCreateWithFlags(&h->cin, cudaStreamNonBlocking), "apply_host: stream");
      FDP_CUDA(cudaStreamCreateWithFlags(&h->cout, cudaStreamNonBlocking), "apply_host: stream");
      for (int k = 0; k < h->D; ++k)
        FDP_CUDA(cudaStreamCreateWithFlags(&h->cs[k], cudaStreamNonBlocking), "apply_host: stream");
      FDP_CUDA(cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming), "apply_host: event");
    }
    // Pipeline units: the D + 1 blocks of one item at batch 1, whole items at batch > 1. Copies in
    // run on cin, the applies on the caller's stream, copies out on cout, so unit j's compute
    // overlaps unit j+1's upload and unit j-1's download (PCIe is full duplex).
    // batch 1: D + 1 units (velocity components in order, then the pressure block), batch > 1:
    // the items
    const int units = batch == 1 ? h->D + 1 : (int)batch;
    while ((int)h->ev_in.size() < units) {
      cudaEvent_t a, b;
      FDP_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming), "apply_host: event");
      FDP_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming), "apply_host: event");
      h->ev_in.push_back(a);
      h->ev_done.push_back(b);
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto pinned = [](const void* p) {
      cudaPointerAttributes a{};
      if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
      return a.type == cudaMemoryTypeHost;
    };
    // batch 1 with page-locked buffers: replay the captured pipeline (copies, applies, events)
    const bool use_graph = batch == 1 && pinned(r_host) && pinned(s_host) &&
                           std::getenv("FDP_E2E_NO_GRAPH") == nullptr;
    if (use_graph && h->e2e_graph && h->e2e_gr == r_host && h->e2e_gs == s_host) {
      FDP_CUDA(cudaGraphLaunch(h->e2e_graph, st), "apply_host: graph launch");
      FDP_CUDA(cudaStreamSynchronize(st), "apply_host: sync");
      return FDP_OK;
    }
    cudaStream_t origin = st;
    if (use_graph) {
      if (h->e2e_graph) {
        cudaGraphExecDestroy(h->e2e_graph);
        h->e2e_graph = nullptr;
      }
      st = h->cap;  // capture on the handle's private stream, then launch on the caller's
      FDP_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "apply_host: capture");
    }
    // batch 1: velocity components in order on the caller's stream (each apply uses every SM),
    // the pressure block last, solved on its own stream (measured: pressure first or merged with
    // the last component's copies is slower)
    auto span = [&](int j, long long* off, long long* len) {
      if (batch == 1) {
        *off = h->off[j];
        *len = h->off[j + 1] - h->off[j];
      } else {
        *off = (long long)j * h->size;
        *len = h->size;
      }
    };
    // the copy-in stream must not overwrite device inputs still read by a previous call
    FDP_CUDA(cudaEventRecord(h->ev_done[0], st), "apply_host: order");
    FDP_CUDA(cudaStreamWaitEvent(h->cin, h->ev_done[0], 0), "apply_host: order");
    for (int j = 0; j < units; ++j) {
      long long off, len;
      span(j, &off, &len);
      FDP_CUDA(cudaMemcpyAsync(h->e2e_r + off, r_host + off, (size_t)len * sizeof(double),
                               cudaMemcpyHostToDevice, h->cin), "apply_host: H2D");
      FDP_CUDA(cudaEventRecord(h->ev_in[j], h->cin), "apply_host: event");
    }
    double* ws = static_cast<double*>(h->e2e_ws);
    for (int j = 0; j < units; ++j) {
      cudaStream_t us = (batch == 1 && j == h->D) ? h->cs[0] : st;
      FDP_CUDA(cudaStreamWaitEvent(us, h->ev_in[j], 0), "apply_host: wait");
      if (batch == 1) {
        long long toff = 0;
        for (int k = 0; k < j; ++k) toff += 2 * Npad(h->vel[k]);
        FDP_CUDA(enqueue_unit(h, j, h->e2e_r, h->e2e_s, ws + toff, us), "apply_host: apply");
      } else {
        FDP_CUDA(enqueue_block(h, h->e2e_r + (long long)j * h->size, h->e2e_s + (long long)j * h->size, 1,
                               ws, st, nullptr), "apply_host: apply");
      }
      FDP_CUDA(cudaEventRecord(h->ev_done[j], us), "apply_host: event");
      if (us != st) FDP_CUDA(cudaStreamWaitEvent(st, h->ev_done[j], 0), "apply_host: join");
      FDP_CUDA(cudaStreamWaitEvent(h->cout, h->ev_done[j], 0), "apply_host: wait");
      long long off, len;
      span(j, &off, &len);
      FDP_CUDA(cudaMemcpyAsync(s_host + off, h->e2e_s + off, (size_t)len * sizeof(double),
                               cudaMemcpyDeviceToHost, h->cout), "apply_host: D2H");
    }
    if (use_graph) {
      // join the copy-out branch back into the origin stream, end the capture, launch
      FDP_CUDA(cudaEventRecord(h->ev_in[0], h->cout), "apply_host: join");
      FDP_CUDA(cudaStreamWaitEvent(st, h->ev_in[0], 0), "apply_host: join");
      cudaGraph_t g = nullptr;
      FDP_CUDA(cudaStreamEndCapture(st, &g), "apply_host: capture end");
      cudaError_t e = cudaGraphInstantiate(&h->e2e_graph, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) {
        h->e2e_graph = nullptr;
        return cuda_fail(e, "apply_host: instantiate");
      }
      h->e2e_gr = r_host;
      h->e2e_gs = s_host;
      FDP_CUDA(cudaGraphLaunch(h->e2e_graph, origin), "apply_host: graph launch");
      FDP_CUDA(cudaStreamSynchronize(origin), "apply_host: sync");
      return FDP_OK;
    }
    FDP_CUDA(cudaStreamSynchronize(h->cout), "apply_host: sync");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" void* fdp_host_alloc(size_t bytes) {
  try {
    void* p = nullptr;
    cudaError_t e = cudaMallocHost(&p, bytes ? bytes : 1);
    if (e != cudaSuccess) {
      cuda_fail(e, "fdp_host_alloc");
      return nullptr;
    }
    return p;
  } catch (...) {
    return nullptr;
  }
}

extern "C" fdp_status fdp_host_free(void* p) {
  try {
    if (!p) return FDP_OK;
    FDP_CUDA(cudaFreeHost(p), "fdp_host_free");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status block_precond_destroy(fdp_block h) {
  try {
    if (!h) return FDP_OK;
    DeviceGuard dg(h->device);
    free_block(h);
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
// slab decomposition (multi-GPU phases)
// ------------------------------------------------------------------------------------------------
static void part_range(long long n, int G, int r, long long* lo, long long* len) {
  const long long q = n / G, rem = n % G;
  *lo = r * q + std::min<long long>(r, rem);
  *len = q + (r < rem ? 1 : 0);
}

extern "C" fdp_status fdp_slab_range(int64_t n, int nranks, int rank, int64_t* lo, int64_t* len) {
  try {
    if (nranks < 1 || rank < 0 || rank >= nranks || n < 0 || !lo || !len)
      return fail(FDP_ERR_INVALID_ARG, "fdp_slab_range: bad arguments");
    long long a, b;
    part_range(n, nranks, rank, &a, &b);
    *lo = a;
    *len = b;
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" size_t fd_slab_workspace_bytes(fdp_fd h, int nranks, int rank) {
  try {
    if (!h || h->D != 3 || nranks < 1 || rank < 0 || rank >= nranks) return 0;
    long long z0, nz, y0, ny;
    part_range(h->n[2], nranks, rank, &z0, &nz);
    part_range(h->n[1], nranks, rank, &y0, &ny);
    const long long zs = (long long)h->n[0] * h->n[1] * nz, ys = (long long)h->n[0] * ny * h->n[2];
    return (size_t)std::max(2 * zs, ys) * sizeof(double);
  } catch (...) {
    return 0;
  }
}

// Mode contraction of a (P, n, Q) view with the handle's direction-d matrices (batch 1).
static ModeProb slab_prob(const fdp_fd_s* h, int d, bool fwd, const double* X, double* Y,
                          long long P, long long Q, int epi, const double* scale,
                          const double* lam1) {
  ModeProb p{};
  p.X = X;
  p.Y = Y;
  p.W = fwd ? h->Wf[d] : h->Wb[d];
  p.P = (int)P;
  p.n = p.nout = h->n[d];
  p.Q = (int)Q;
  p.N = P * h->n[d] * Q;
  p.xbs = p.ybs = 0;
  p.batch = 1;
  p.ldw = h->cfg[d].ldw;
  p.n1 = p.n1v = h->n[0];
  p.xld = p.yld = h->n[0];
  p.vx = p.vy = 0;
  p.epi = epi;
  p.scale = scale;
  if (epi == EPI_LAMBDA || epi == EPI_FUSED) {
    p.lam0 = h->lamc[0];
    p.lam1 = lam1;
    p.lamcol = h->lamc[2];
  }
  const int BM = kK1Warps * 8 * h->cfg[d].MT;
  p.tiles_m = (int)((P * Q + BM - 1) / BM);
  p.tiles_n = h->cfg[d].tiles_n;
  p.fd_work = 1;
  return p;
}

static cudaError_t run1(ModeProb p, const TileCfg& c, bool kmaj, cudaStream_t s) {
  std::vector<ModeProb> v{p};
  std::vector<TileCfg> cv{c};
  return launch_stage(v, cv, kmaj, s, nullptr, nullptr);
}

extern "C" fdp_status fd_apply_slab(fdp_fd h, int phase, int nranks, int rank, const double* in,
                                    double* out, const double* dscale, void* workspace,
                                    void* stream) {
  try {
    if (!h) return fail(FDP_ERR_INVALID_ARG, "fd_apply_slab: NULL handle");
    if (h->D != 3) return fail(FDP_ERR_UNSUPPORTED, "fd_apply_slab: D must be 3");
    if (nranks < 1 || rank < 0 || rank >= nranks || phase < 0 || phase > 2)
      return fail(FDP_ERR_INVALID_ARG, "fd_apply_slab: bad phase / rank");
    const long long n1 = h->n[0], n2 = h->n[1], n3 = h->n[2];
    long long z0, nz, y0, ny;
    part_range(n3, nranks, rank, &z0, &nz);
    part_range(n2, nranks, rank, &y0, &ny);
    if ((phase == 1 ? ny : nz) == 0) return FDP_OK;  // this rank owns nothing of that axis
    if (!is_device_ptr(in) || !is_device_ptr(out) || !is_device_ptr(workspace) ||
        (dscale && !is_device_ptr(dscale)))
      return fail(FDP_ERR_INVALID_ARG, "fd_apply_slab: device pointers required");
    DeviceGuard dg(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    double* T1 = static_cast<double*>(workspace);
    double* T2 = T1 + n1 * n2 * nz;
    if (phase == 0) {
      const double* src = in;
      if (dscale) {
        FDP_CUDA(launch_scale(in, T2, dscale, n1 * n2 * nz, 1, 0, 0, s), "fd_apply_slab: prescale");
        src = T2;
      }
      FDP_CUDA(run1(slab_prob(h, 0, true, src, T1, 1, n2 * nz, EPI_NONE, nullptr, nullptr), h->cfg[0], true, s),
               "fd_apply_slab: mode 1");
      FDP_CUDA(run1(slab_prob(h, 1, true, T1, T2, n1, nz, EPI_NONE, nullptr, nullptr), h->cfg[1], false, s),
               "fd_apply_slab: mode 2");
      FDP_CUDA(launch_slab_copy(T2, out, (int)n1, (int)n2, (int)nz, nranks, 0, nullptr, s), "fd_apply_slab: pack");
    } else if (phase == 1) {
      const double* lam1 = h->lamc[1] + y0;
      const bool fuse = std::getenv("FDP_NO_FUSE") == nullptr && std::getenv("FDP_NO_SMALL") == nullptr &&
                        n3 <= kSmallMaxN && h->cfg[2].tiles_n == 1;
      if (fuse) {  // in place: each 8-row tile is read whole before it is written
        FDP_CUDA(run1(slab_prob(h, 2, true, in, out, n1 * ny, 1, EPI_FUSED, nullptr, lam1), h->cfg[2], false, s),
                 "fd_apply_slab: fused mode 3");
      } else {
        FDP_CUDA(run1(slab_prob(h, 2, true, in, T1, n1 * ny, 1, EPI_LAMBDA, nullptr, lam1), h->cfg[2], false, s),
                 "fd_apply_slab: mode 3 fwd");
        FDP_CUDA(run1(slab_prob(h, 2, false, T1, out, n1 * ny, 1, EPI_NONE, nullptr, nullptr), h->cfg[2], false, s),
                 "fd_apply_slab: mode 3 bwd");
      }
    } else {
      FDP_CUDA(launch_slab_copy(in, T1, (int)n1, (int)n2, (int)nz, nranks, 1, nullptr, s), "fd_apply_slab: unpack");
      FDP_CUDA(run1(slab_prob(h, 1, false, T1, T2, n1, nz, EPI_NONE, nullptr, nullptr), h->cfg[1], false, s),
               "fd_apply_slab: mode 2 bwd");
      FDP_CUDA(run1(slab_prob(h, 0, false, T2, out, 1, n2 * nz, dscale ? EPI_SCALE : EPI_NONE, dscale, nullptr),
                    h->cfg[0], true, s),
               "fd_apply_slab: mode 1 bwd");
    }
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

// ---- peer-store slab exchange: the exchanges are fused into the epilogues of
// the contraction that precedes them; data crosses NVLink as the kernels' own stores ----
static void set_scatter(ModeProb& p, double* const* peers, int G, int na, int n1, int qoff, int a0,
                        int a1, int q0, int q1) {
  p.peers = peers;
  p.sc_G = G;
  p.sc_na = na;
  p.sc_n1 = n1;
  p.sc_qoff = qoff;
  p.sc_a0 = a0;
  p.sc_a1 = a1;
  p.sc_q0 = q0;
  p.sc_q1 = q1;
}

extern "C" fdp_status fd_apply_slab_peer(fdp_fd h, int phase, int nranks, int rank, const double* in,
                                         double* out, double* const* peers, const double* dscale,
                                         void* workspace, void* stream) {
  try {
    if (!h) return fail(FDP_ERR_INVALID_ARG, "fd_apply_slab_peer: NULL handle");
    if (h->D != 3) return fail(FDP_ERR_UNSUPPORTED, "fd_apply_slab_peer: D must be 3");
    if (nranks < 1 || nranks > 32 || rank < 0 || rank >= nranks || phase < 0 || phase > 2)
      return fail(FDP_ERR_INVALID_ARG, "fd_apply_slab_peer: bad phase / rank");
    const long long n1 = h->n[0], n2 = h->n[1], n3 = h->n[2];
    long long z0, nz, y0, ny;
    part_range(n3, nranks, rank, &z0, &nz);
    part_range(n2, nranks, rank, &y0, &ny);
    if ((phase == 1 ? ny : nz) == 0) return FDP_OK;
    if (!is_device_ptr(in) || !is_device_ptr(workspace) || (phase == 2 && !is_device_ptr(out)) ||
        (phase < 2 && !is_device_ptr(peers)) || (dscale && !is_device_ptr(dscale)))
      return fail(FDP_ERR_INVALID_ARG, "fd_apply_slab_peer: device pointers required");
    DeviceGuard dg(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    double* T1 = static_cast<double*>(workspace);
    double* T2 = T1 + n1 * n2 * nz;
    if (phase == 0) {
      // modes 1, 2 on the z-slab; mode 2 stores element (i1, i2, i3) straight into the y-slab
      // buffer (n1, ny_h, n3) of the rank h owning i2, at (i1, i2 - y0_h, z0 + i3)
      const double* src = in;
      if (dscale) {
        FDP_CUDA(launch_scale(in, T2, dscale, n1 * n2 * nz, 1, 0, 0, s), "fd_apply_slab_peer: prescale");
        src = T2;
      }
      FDP_CUDA(run1(slab_prob(h, 0, true, src, T1, 1, n2 * nz, EPI_NONE, nullptr, nullptr), h->cfg[0], true, s),
               "fd_apply_slab_peer: mode 1");
      ModeProb p = slab_prob(h, 1, true, T1, nullptr, n1, nz, EPI_NONE, nullptr, nullptr);
      set_scatter(p, peers, nranks, (int)n2, (int)n1, (int)z0, 1, 0, 0, 1);
      FDP_CUDA(run1(p, h->cfg[1], false, s), "fd_apply_slab_peer: mode 2 + exchange");
    } else if (phase == 1) {
      // the mode-3 triple on the y-slab; the last contraction stores element (i1, i2, i3) straight
      // into the z-slab buffer (n1, n2, nz_g) of the rank g owning i3, at (i1, y0 + i2, i3 - z0_g)
      const double* lam1 = h->lamc[1] + y0;
      const bool fuse = std::getenv("FDP_NO_FUSE") == nullptr && std::getenv("FDP_NO_SMALL") == nullptr &&
                        n3 <= kSmallMaxN && h->cfg[2].tiles_n == 1;
      if (fuse) {
        ModeProb p = slab_prob(h, 2, true, in, nullptr, n1 * ny, 1, EPI_FUSED, nullptr, lam1);
        set_scatter(p, peers, nranks, (int)n3, (int)n1, (int)y0, (int)n2, 0, 1, 0);
        FDP_CUDA(run1(p, h->cfg[2], false, s), "fd_apply_slab_peer: fused mode 3 + exchange");
      } else {
        FDP_CUDA(run1(slab_prob(h, 2, true, in, T1, n1 * ny, 1, EPI_LAMBDA, nullptr, lam1), h->cfg[2], false, s),
                 "fd_apply_slab_peer: mode 3 fwd");
        ModeProb p = slab_prob(h, 2, false, T1, nullptr, n1 * ny, 1, EPI_NONE, nullptr, nullptr);
        set_scatter(p, peers, nranks, (int)n3, (int)n1, (int)y0, (int)n2, 0, 1, 0);
        FDP_CUDA(run1(p, h->cfg[2], false, s), "fd_apply_slab_peer: mode 3 bwd + exchange");
      }
    } else {
      FDP_CUDA(run1(slab_prob(h, 1, false, in, T2, n1, nz, EPI_NONE, nullptr, nullptr), h->cfg[1], false, s),
               "fd_apply_slab_peer: mode 2 bwd");
      FDP_CUDA(run1(slab_prob(h, 0, false, T2, out, 1, n2 * nz, dscale ? EPI_SCALE : EPI_NONE, dscale, nullptr),
                    h->cfg[0], true, s),
               "fd_apply_slab_peer: mode 1 bwd");
    }
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status kron_mass_apply_slab_peer(fdp_mass h, int phase, int nranks, int rank,
                                                const double* in, double* out, double* const* peers,
                                                const double* dscale, void* workspace, void* stream) {
  try {
    if (!h) return fail(FDP_ERR_INVALID_ARG, "kron_mass_apply_slab_peer: NULL handle");
    if (h->D != 3) return fail(FDP_ERR_UNSUPPORTED, "kron_mass_apply_slab_peer: D must be 3");
    if (nranks < 1 || nranks > 32 || rank < 0 || rank >= nranks || phase < 0 || phase > 2)
      return fail(FDP_ERR_INVALID_ARG, "kron_mass_apply_slab_peer: bad phase / rank");
    const long long n1 = h->n[0], n2 = h->n[1], n3 = h->n[2];
    long long z0, nz, y0, ny;
    part_range(n3, nranks, rank, &z0, &nz);
    part_range(n2, nranks, rank, &y0, &ny);
    if ((phase == 1 ? ny : nz) == 0) return FDP_OK;
    if (!is_device_ptr(in) || (phase < 2 && (!is_device_ptr(workspace) || !is_device_ptr(peers))) ||
        (phase == 2 && !is_device_ptr(out)) || (dscale && !is_device_ptr(dscale)))
      return fail(FDP_ERR_INVALID_ARG, "kron_mass_apply_slab_peer: device pointers required");
    DeviceGuard dg(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto mode = [&](int d, const double* src, double* dst, long long P, long long Q, const double* pre) {
      MassMode m{};
      m.in = src;
      m.out = dst;
      m.Lb = h->Lb[d];
      m.invd = h->invd[d];
      m.Mb = h->Mb[d];
      m.pre = pre;
      m.N = P * h->n[d] * Q;
      m.bs = 0;
      m.P = (int)P;
      m.n = h->n[d];
      m.Q = (int)Q;
      m.batch = 1;
      m.band = h->band[d];
      return launch_mass_mode(m, s);
    };
    double* T = static_cast<double*>(workspace);
    if (phase == 0) {
      FDP_CUDA(mode(0, in, T, 1, n2 * nz, dscale), "kron_mass_apply_slab_peer: mode 1");
      FDP_CUDA(mode(1, T, T, n1, nz, nullptr), "kron_mass_apply_slab_peer: mode 2");
      ScatterDesc sd{peers, nranks, (int)n2, (int)n1, (int)z0, 1, 0, 0, 1};
      FDP_CUDA(launch_slab_scatter(T, sd, (int)nz, 0, s), "kron_mass_apply_slab_peer: exchange");
    } else if (phase == 1) {
      FDP_CUDA(mode(2, in, T, n1 * ny, 1, nullptr), "kron_mass_apply_slab_peer: mode 3");
      ScatterDesc sd{peers, nranks, (int)n3, (int)n1, (int)y0, (int)n2, 0, 1, 0};
      FDP_CUDA(launch_slab_scatter(T, sd, (int)ny, 1, s), "kron_mass_apply_slab_peer: exchange");
    } else if (dscale) {
      FDP_CUDA(launch_scale(in, out, dscale, n1 * n2 * nz, 1, 0, 0, s), "kron_mass_apply_slab_peer: postscale");
    } else if (in != out) {
      FDP_CUDA(cudaMemcpyAsync(out, in, (size_t)(n1 * n2 * nz) * sizeof(double), cudaMemcpyDeviceToDevice, s),
               "kron_mass_apply_slab_peer: copy");
    }
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_peer_barrier(unsigned long long* const* flags, unsigned long long* counter,
                                       int nranks, int rank, void* stream) {
  try {
    if (nranks < 1 || nranks > 32 || rank < 0 || rank >= nranks)
      return fail(FDP_ERR_INVALID_ARG, "fdp_peer_barrier: bad rank");
    if (!is_device_ptr(flags) || !is_device_ptr(counter))
      return fail(FDP_ERR_INVALID_ARG, "fdp_peer_barrier: device pointers required");
    FDP_CUDA(launch_peer_barrier(flags, counter, nranks, rank, static_cast<cudaStream_t>(stream)),
             "fdp_peer_barrier");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_peer_alloc(size_t bytes, int device, void** dev_ptr, void* ipc_handle) {
  try {
    if (!dev_ptr || !ipc_handle) return fail(FDP_ERR_INVALID_ARG, "fdp_peer_alloc: NULL argument");
    *dev_ptr = nullptr;
    DeviceGuard dg(device);
    void* p = nullptr;
    FDP_CUDA(cudaMalloc(&p, bytes ? bytes : 8), "fdp_peer_alloc: cudaMalloc");
    cudaError_t e = cudaMemset(p, 0, bytes ? bytes : 8);
    cudaIpcMemHandle_t hd;
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&hd, p);
    if (e != cudaSuccess) {
      cudaFree(p);
      return cuda_fail(e, "fdp_peer_alloc: IPC handle");
    }
    std::memcpy(ipc_handle, &hd, sizeof(hd));
    *dev_ptr = p;
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_peer_open(const void* ipc_handle, int device, void** dev_ptr) {
  try {
    if (!ipc_handle || !dev_ptr) return fail(FDP_ERR_INVALID_ARG, "fdp_peer_open: NULL argument");
    *dev_ptr = nullptr;
    DeviceGuard dg(device);
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, ipc_handle, sizeof(hd));
    FDP_CUDA(cudaIpcOpenMemHandle(dev_ptr, hd, cudaIpcMemLazyEnablePeerAccess), "fdp_peer_open");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_peer_close(void* dev_ptr) {
  try {
    if (!dev_ptr) return FDP_OK;
    FDP_CUDA(cudaIpcCloseMemHandle(dev_ptr), "fdp_peer_close");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_peer_free(void* dev_ptr) {
  try {
    if (!dev_ptr) return FDP_OK;
    FDP_CUDA(cudaFree(dev_ptr), "fdp_peer_free");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

// ---- C-level communicator for the sharded block apply (SURVEY.md §8(b) "multi-GPU") ----
// Every rank owns, per block of the preconditioner, a y-slab receive buffer (exchange 1) and a
// z-slab return buffer (exchange 2), plus an nranks-slot barrier flag array; their CUDA IPC
// handles form the rank's blob, which the caller all-gathers (torch.distributed is plumbing).
struct fdp_comm_s {
  int nranks = 0, rank = 0, device = 0, nblocks = 0;
  std::vector<void*> own;             // y-slab, z-slab per block, then flags (device)
  std::vector<void*> opened;          // peer mappings to close
  double** peers_y = nullptr;         // device: [block][rank] pointer tables
  double** peers_z = nullptr;
  unsigned long long** flag_ptrs = nullptr;  // device: [rank]
  unsigned long long* counter = nullptr;
  bool connected = false;
};

static void free_comm(fdp_comm c) {
  if (!c) return;
  for (void* p : c->opened) cudaIpcCloseMemHandle(p);
  for (void* p : c->own) cudaFree(p);
  cudaFree(c->peers_y);
  cudaFree(c->peers_z);
  cudaFree(c->flag_ptrs);
  cudaFree(c->counter);
  delete c;
}

static void block_dims(const fdp_block_s* P, int b, long long* n1, long long* n2, long long* n3) {
  const int* n = b < P->D ? P->vel[b]->n : P->pres->n;
  *n1 = n[0];
  *n2 = n[1];
  *n3 = n[2];
}

extern "C" size_t fdp_comm_blob_bytes(fdp_block P, int nranks) {
  try {
    if (!P || P->D != 3 || nranks < 1) return 0;
    return (size_t)(2 * (P->D + 1) + 1) * sizeof(cudaIpcMemHandle_t);
  } catch (...) {
    return 0;
  }
}

extern "C" fdp_status fdp_comm_create(fdp_block P, int nranks, int rank, fdp_comm* out, void* blob) {
  try {
    if (!out || !blob) return fail(FDP_ERR_INVALID_ARG, "fdp_comm_create: NULL argument");
    *out = nullptr;
    if (!P) return fail(FDP_ERR_INVALID_ARG, "fdp_comm_create: NULL block");
    if (P->D != 3) return fail(FDP_ERR_UNSUPPORTED, "fdp_comm_create: D must be 3");
    if (nranks < 1 || nranks > 32 || rank < 0 || rank >= nranks)
      return fail(FDP_ERR_INVALID_ARG, "fdp_comm_create: bad rank");
    DeviceGuard dg(P->device);
    std::unique_ptr<fdp_comm_s> c(new (std::nothrow) fdp_comm_s);
    if (!c) return fail(FDP_ERR_OOM, "fdp_comm_create: host allocation");
    c->nranks = nranks;
    c->rank = rank;
    c->device = P->device;
    c->nblocks = P->D + 1;
    fdp_comm raw = c.release();
    auto alloc = [&](size_t bytes) -> fdp_status {
      void* p = nullptr;
      cudaIpcMemHandle_t hd;
      fdp_status st = fdp_peer_alloc(bytes, raw->device, &p, &hd);
      if (st) return st;
      std::memcpy(static_cast<char*>(blob) + raw->own.size() * sizeof(hd), &hd, sizeof(hd));
      raw->own.push_back(p);
      return FDP_OK;
    };
    fdp_status st = FDP_OK;
    for (int b = 0; b < raw->nblocks && !st; ++b) {
      long long n1, n2, n3, y0, ny, z0, nz;
      block_dims(P, b, &n1, &n2, &n3);
      part_range(n2, nranks, rank, &y0, &ny);
      part_range(n3, nranks, rank, &z0, &nz);
      st = alloc((size_t)std::max(1LL, n1 * ny * n3) * sizeof(double));
      if (!st) st = alloc((size_t)std::max(1LL, n1 * n2 * nz) * sizeof(double));
    }
    if (!st) st = alloc((size_t)nranks * sizeof(unsigned long long));
    if (!st) st = dalloc(&raw->counter, 1);
    if (!st) {
      cudaError_t e = cudaMemset(raw->counter, 0, sizeof(unsigned long long));
      if (e != cudaSuccess) st = cuda_fail(e, "fdp_comm_create: counter");
    }
    if (st) {
      free_comm(raw);
      return st;
    }
    *out = raw;
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_comm_connect(fdp_comm c, const void* all_blobs) {
  try {
    if (!c || !all_blobs) return fail(FDP_ERR_INVALID_ARG, "fdp_comm_connect: NULL argument");
    if (c->connected) return fail(FDP_ERR_INVALID_ARG, "fdp_comm_connect: already connected");
    DeviceGuard dg(c->device);
    const int G = c->nranks, nb = c->nblocks, per = 2 * nb + 1;
    std::vector<double*> py((size_t)nb * G), pz((size_t)nb * G);
    std::vector<unsigned long long*> pf(G);
    for (int r = 0; r < G; ++r) {
      for (int i = 0; i < per; ++i) {
        void* p = c->own[i];
        if (r != c->rank) {  // map the peer's buffer (P2P over NVLink)
          const char* hp = static_cast<const char*>(all_blobs) + ((size_t)r * per + i) * sizeof(cudaIpcMemHandle_t);
          fdp_status st = fdp_peer_open(hp, c->device, &p);
          if (st) return st;
          c->opened.push_back(p);
        }
        if (i < 2 * nb) {
          const int b = i / 2;
          (i % 2 == 0 ? py : pz)[(size_t)b * G + r] = static_cast<double*>(p);
        } else {
          pf[r] = static_cast<unsigned long long*>(p);
        }
      }
    }
    fdp_status st;
    if ((st = dalloc(&c->peers_y, py.size())) || (st = dalloc(&c->peers_z, pz.size())) ||
        (st = dalloc(&c->flag_ptrs, pf.size())))
      return st;
    FDP_CUDA(cudaMemcpy(c->peers_y, py.data(), py.size() * sizeof(double*), cudaMemcpyHostToDevice), "fdp_comm_connect");
    FDP_CUDA(cudaMemcpy(c->peers_z, pz.data(), pz.size() * sizeof(double*), cudaMemcpyHostToDevice), "fdp_comm_connect");
    FDP_CUDA(cudaMemcpy(c->flag_ptrs, pf.data(), pf.size() * sizeof(void*), cudaMemcpyHostToDevice), "fdp_comm_connect");
    c->connected = true;
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" int64_t block_precond_sharded_size(fdp_block P, int nranks, int rank) {
  try {
    if (!P || P->D != 3 || nranks < 1 || rank < 0 || rank >= nranks) return 0;
    long long tot = 0;
    for (int b = 0; b <= P->D; ++b) {
      long long n1, n2, n3, z0, nz;
      block_dims(P, b, &n1, &n2, &n3);
      part_range(n3, nranks, rank, &z0, &nz);
      tot += n1 * n2 * nz;
    }
    return tot;
  } catch (...) {
    return 0;
  }
}

extern "C" size_t block_precond_sharded_workspace_bytes(fdp_block P, fdp_comm c) {
  try {
    if (!P || !c || P->D != 3) return 0;
    size_t m = 0;
    for (int k = 0; k < P->D; ++k)
      m = std::max(m, fd_slab_workspace_bytes(const_cast<fdp_fd>(P->vel[k]), c->nranks, c->rank));
    m = std::max(m, kron_mass_slab_workspace_bytes(const_cast<fdp_mass>(P->pres), c->nranks, c->rank));
    return m;
  } catch (...) {
    return 0;
  }
}

extern "C" fdp_status block_precond_apply_sharded(fdp_block P, fdp_comm c, const double* r, double* s,
                                                  void* workspace, void* stream) {
  try {
    if (!P || !c) return fail(FDP_ERR_INVALID_ARG, "block_precond_apply_sharded: NULL handle");
    if (!c->connected) return fail(FDP_ERR_INVALID_ARG, "block_precond_apply_sharded: comm not connected");
    if (!is_device_ptr(r) || !is_device_ptr(s) || !is_device_ptr(workspace))
      return fail(FDP_ERR_INVALID_ARG, "block_precond_apply_sharded: device pointers required");
    DeviceGuard dg(P->device);
    const int G = c->nranks, g = c->rank, D = P->D;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // local layout [u_1 z-slab | .. | u_D z-slab | p z-slab]; D^{-1/2} slices of the P^G scalings
    std::vector<long long> loff(D + 2, 0), goff(D + 1, 0);
    for (int b = 0; b <= D; ++b) {
      long long n1, n2, n3, z0, nz;
      block_dims(P, b, &n1, &n2, &n3);
      part_range(n3, G, g, &z0, &nz);
      loff[b + 1] = loff[b] + n1 * n2 * nz;
      goff[b] = n1 * n2 * z0;
    }
    auto dsc = [&](int b) -> const double* {
      if (b < D) return P->dv ? P->dv + P->off[b] + goff[b] : nullptr;
      return P->dq ? P->dq + goff[b] : nullptr;
    };
    const int nb = c->nblocks;
    for (int phase = 0; phase < 3; ++phase) {
      for (int b = 0; b < nb; ++b) {
        double* const* peers = phase == 0 ? c->peers_y + (size_t)b * G : c->peers_z + (size_t)b * G;
        const double* in = phase == 0 ? r + loff[b] : static_cast<const double*>(c->own[2 * b + (phase == 1 ? 0 : 1)]);
        double* out = phase == 2 ? s + loff[b] : nullptr;
        const double* ds = phase == 1 ? nullptr : dsc(b);
        fdp_status e = b < D ? fd_apply_slab_peer(const_cast<fdp_fd>(P->vel[b]), phase, G, g, in, out,
                                                  phase == 2 ? nullptr : peers, ds, workspace, stream)
                             : kron_mass_apply_slab_peer(const_cast<fdp_mass>(P->pres), phase, G, g, in, out,
                                                         phase == 2 ? nullptr : peers, ds, workspace, stream);
        if (e) return e;
      }
      // exchanges complete on every rank before the next phase reads (and, after phase 2, before
      // the next apply's phase 0 overwrites y-slabs)
      FDP_CUDA(launch_peer_barrier(c->flag_ptrs, c->counter, G, g, st), "block_precond_apply_sharded: barrier");
    }
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_comm_destroy(fdp_comm c) {
  try {
    if (!c) return FDP_OK;
    DeviceGuard dg(c->device);
    free_comm(c);
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" size_t kron_mass_slab_workspace_bytes(fdp_mass h, int nranks, int rank) {
  try {
    if (!h || h->D != 3 || nranks < 1 || rank < 0 || rank >= nranks) return 0;
    long long z0, nz;
    part_range(h->n[2], nranks, rank, &z0, &nz);
    return (size_t)((long long)h->n[0] * h->n[1] * nz) * sizeof(double);
  } catch (...) {
    return 0;
  }
}

extern "C" fdp_status kron_mass_apply_slab(fdp_mass h, int phase, int nranks, int rank,
                                           const double* in, double* out, const double* dscale,
                                           void* workspace, void* stream) {
  try {
    if (!h) return fail(FDP_ERR_INVALID_ARG, "kron_mass_apply_slab: NULL handle");
    if (h->D != 3) return fail(FDP_ERR_UNSUPPORTED, "kron_mass_apply_slab: D must be 3");
    if (nranks < 1 || rank < 0 || rank >= nranks || phase < 0 || phase > 2)
      return fail(FDP_ERR_INVALID_ARG, "kron_mass_apply_slab: bad phase / rank");
    const long long n1 = h->n[0], n2 = h->n[1], n3 = h->n[2];
    long long z0, nz, y0, ny;
    part_range(n3, nranks, rank, &z0, &nz);
    part_range(n2, nranks, rank, &y0, &ny);
    if ((phase == 1 ? ny : nz) == 0) return FDP_OK;
    if (!is_device_ptr(in) || !is_device_ptr(out) || (phase == 0 && !is_device_ptr(workspace)) ||
        (dscale && !is_device_ptr(dscale)))
      return fail(FDP_ERR_INVALID_ARG, "kron_mass_apply_slab: device pointers required");
    DeviceGuard dg(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto mode = [&](int d, const double* src, double* dst, long long P, long long Q, const double* pre) {
      MassMode m{};
      m.in = src;
      m.out = dst;
      m.Lb = h->Lb[d];
      m.invd = h->invd[d];
      m.Mb = h->Mb[d];
      m.pre = pre;
      m.N = P * h->n[d] * Q;
      m.bs = 0;
      m.P = (int)P;
      m.n = h->n[d];
      m.Q = (int)Q;
      m.batch = 1;
      m.band = h->band[d];
      return launch_mass_mode(m, s);
    };
    double* T = static_cast<double*>(workspace);
    if (phase == 0) {
      FDP_CUDA(mode(0, in, T, 1, n2 * nz, dscale), "kron_mass_apply_slab: mode 1");
      FDP_CUDA(mode(1, T, T, n1, nz, nullptr), "kron_mass_apply_slab: mode 2");
      FDP_CUDA(launch_slab_copy(T, out, (int)n1, (int)n2, (int)nz, nranks, 0, nullptr, s),
               "kron_mass_apply_slab: pack");
    } else if (phase == 1) {
      FDP_CUDA(mode(2, in, out, n1 * ny, 1, nullptr), "kron_mass_apply_slab: mode 3");
    } else {
      FDP_CUDA(launch_slab_copy(in, out, (int)n1, (int)n2, (int)nz, nranks, 1, dscale, s),
               "kron_mass_apply_slab: unpack");
    }
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

// ------------------------------------------------------------------------------------------------
// vector kernels
// ------------------------------------------------------------------------------------------------
static double* dot_scratch(int dev) {
  static double* scratch[64] = {nullptr};
  if (dev < 0 || dev >= 64) return nullptr;
  if (!scratch[dev] && cudaMalloc(&scratch[dev], dot_scratch_doubles() * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    scratch[dev] = nullptr;
  }
  return scratch[dev];
}

extern "C" fdp_status fdp_vec_dot(const double* x, const double* y, int64_t n, double* result,
                                  void* stream) {
  try {
    if (n < 0) return fail(FDP_ERR_SHAPE, "fdp_vec_dot: n < 0");
    if (!is_device_ptr(result) || (n > 0 && (!is_device_ptr(x) || !is_device_ptr(y))))
      return fail(FDP_ERR_INVALID_ARG, "fdp_vec_dot: device pointers required");
    int dev = 0;
    cudaGetDevice(&dev);
    double* sc = dot_scratch(dev);
    if (!sc) return fail(FDP_ERR_OOM, "fdp_vec_dot: scratch");
    FDP_CUDA(launch_dot(x, y, n, result, sc, static_cast<cudaStream_t>(stream)), "fdp_vec_dot");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_vec_lincomb(double a, const double* x, double b, const double* y,
                                      double c, const double* z, double* out, int64_t n,
                                      void* stream) {
  try {
    if (n < 0) return fail(FDP_ERR_SHAPE, "fdp_vec_lincomb: n < 0");
    if (n == 0) return FDP_OK;
    if (!is_device_ptr(x) || !is_device_ptr(out) || (y && !is_device_ptr(y)) || (z && !is_device_ptr(z)))
      return fail(FDP_ERR_INVALID_ARG, "fdp_vec_lincomb: device pointers required");
    FDP_CUDA(launch_lincomb(a, x, b, y, c, z, out, n, static_cast<cudaStream_t>(stream)), "fdp_vec_lincomb");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

// ------------------------------------------------------------------------------------------------
// matrix-free sums of Kronecker products (NEXT-1 Stokes operator blocks)
// ------------------------------------------------------------------------------------------------
struct KronFactor {
  int nin = 0, nout = 0;
  TileCfg cfg{};
  std::vector<double> diag;  // F[i][i] for i < min(nin, nout) (kron_op_diagonal)
  double* W = nullptr;  // W[k][a] = F[a][k], kpad x ldw
};
struct fdp_kron_s {
  int D = 0, nterms = 0, device = 0;
  int nin[3] = {1, 1, 1}, nout[3] = {1, 1, 1};
  std::vector<double> coef;
  std::vector<KronFactor> f;  // nterms * D
};

static void free_kron(fdp_kron h) {
  if (!h) return;
  for (auto& k : h->f) cudaFree(k.W);
  delete h;
}

extern "C" fdp_status kron_op_setup(int D, int nterms, const int32_t* nin, const int32_t* nout,
                                    const double* const* factors, const double* coef, int device,
                                    fdp_kron* out) {
  try {
    if (!out) return fail(FDP_ERR_INVALID_ARG, "kron_op_setup: out is NULL");
    *out = nullptr;
    if (D < 2 || D > 3) return fail(FDP_ERR_UNSUPPORTED, "kron_op_setup: D must be 2 or 3");
    if (nterms < 1 || !nin || !nout || !factors || !coef)
      return fail(FDP_ERR_INVALID_ARG, "kron_op_setup: bad arguments");
    std::unique_ptr<fdp_kron_s> h(new (std::nothrow) fdp_kron_s);
    if (!h) return fail(FDP_ERR_OOM, "kron_op_setup: host allocation");
    h->D = D;
    h->nterms = nterms;
    h->device = device;
    for (int d = 0; d < D; ++d) {
      if (nin[d] < 1 || nin[d] > 2048 || nout[d] < 1 || nout[d] > 2048)
        return fail(FDP_ERR_SHAPE, "kron_op_setup: extents must be in [1, 2048]");
      h->nin[d] = nin[d];
      h->nout[d] = nout[d];
    }
    h->coef.assign(coef, coef + nterms);
    DeviceGuard dg(device);
    fdp_kron raw = h.release();
    raw->f.resize((size_t)nterms * D);
    for (int t = 0; t < nterms; ++t)
      for (int d = 0; d < D; ++d) {
        const double* F = factors[t * D + d];
        if (!F) {
          free_kron(raw);
          return fail(FDP_ERR_INVALID_ARG, "kron_op_setup: NULL factor");
        }
        KronFactor& kf = raw->f[t * D + d];
        kf.nin = nin[d];
        kf.nout = nout[d];
        for (int i = 0; i < std::min(nin[d], nout[d]); ++i) kf.diag.push_back(F[i + (size_t)nout[d] * i]);
        // columns tile over nout; the small path also needs BN >= nin (W rows staged in smem)
        TileCfg c = choose_tile(std::max(nin[d], nout[d]) <= kSmallMaxN ? std::max(nin[d], nout[d]) : nout[d]);
        c.kpad = ((nin[d] + 31) / 32) * 32;
        kf.cfg = c;
        const int rows = std::max(c.kpad, c.ldw);
        std::vector<double> w((size_t)rows * c.ldw, 0.0);
        for (int k = 0; k < nin[d]; ++k)
          for (int a = 0; a < nout[d]; ++a) w[(size_t)k * c.ldw + a] = F[a + (size_t)nout[d] * k];
        fdp_status st = dalloc(&kf.W, w.size());
        cudaError_t e = st ? cudaSuccess : cudaMemcpy(kf.W, w.data(), w.size() * 8, cudaMemcpyHostToDevice);
        if (!st && e == cudaSuccess) e = prepare_mode_kernels(c);
        if (!st && e == cudaSuccess) e = prepare_mode_small(c.NT);
        if (st || e != cudaSuccess) {
          free_kron(raw);
          return st ? st : cuda_fail(e, "kron_op_setup: upload");
        }
      }
    *out = raw;
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

static long long kron_max_inter(const fdp_kron_s* h) {
  long long mx = 1;
  for (int d = 0; d < h->D; ++d) {  // after contracting modes 0..d: nout for e <= d, nin after
    long long sz = 1;
    for (int e = 0; e < h->D; ++e) sz *= (e <= d ? h->nout[e] : h->nin[e]);
    mx = std::max(mx, sz);
  }
  return mx;
}

extern "C" size_t kron_op_workspace_bytes(fdp_kron h, int64_t batch) {
  try {
    return h && batch > 0 ? (size_t)(2 * kron_max_inter(h) * batch) * sizeof(double) : 0;
  } catch (...) {
    return 0;
  }
}

extern "C" fdp_status kron_op_apply(fdp_kron h, const double* x, int64_t xbs, double* y,
                                    int64_t ybs, double alpha, double beta, int64_t batch,
                                    void* workspace, void* stream) {
  try {
    if (!h) return fail(FDP_ERR_INVALID_ARG, "kron_op_apply: NULL handle");
    if (batch < 0) return fail(FDP_ERR_SHAPE, "kron_op_apply: batch < 0");
    if (batch == 0) return FDP_OK;
    if (!is_device_ptr(x) || !is_device_ptr(y) || !is_device_ptr(workspace))
      return fail(FDP_ERR_INVALID_ARG, "kron_op_apply: device pointers required");
    DeviceGuard dg(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int D = h->D;
    const long long inter = kron_max_inter(h);
    double* buf[2] = {static_cast<double*>(workspace), static_cast<double*>(workspace) + inter * batch};
    for (int t = 0; t < h->nterms; ++t) {
      const double* src = x;
      long long sbs = xbs;
      for (int d = 0; d < D; ++d) {
        const KronFactor& kf = h->f[t * D + d];
        long long P = 1, Q = 1;
        for (int e = 0; e < d; ++e) P *= h->nout[e];
        for (int e = d + 1; e < D; ++e) Q *= h->nin[e];
        const bool last = d == D - 1;
        double* dst = last ? y : buf[d % 2];
        const long long dbs = last ? ybs : P * kf.nout * Q;
        ModeProb p{};
        p.X = src;
        p.Y = dst;
        p.W = kf.W;
        p.P = (int)P;
        p.n = kf.nin;
        p.nout = kf.nout;
        p.Q = (int)Q;
        p.N = P * kf.nout * Q;
        p.xbs = sbs;
        p.ybs = dbs;
        p.batch = (int)batch;
        p.ldw = kf.cfg.ldw;
        p.n1 = p.n1v = 1;
        p.xld = kf.nin;
        p.yld = kf.nout;
        p.vx = p.vy = 0;
        p.epi = last ? EPI_AXPBY : EPI_NONE;
        p.alpha = alpha * h->coef[t];
        p.beta = t == 0 ? beta : 1.0;
        const int BM = kK1Warps * 8 * kf.cfg.MT;
        p.tiles_m = (int)((P * Q * batch + BM - 1) / BM);
        p.tiles_n = kf.cfg.tiles_n;
        p.fd_work = 0;
        FDP_CUDA(run1(p, kf.cfg, d == 0, s), "kron_op_apply");
        src = dst;
        sbs = dbs;
      }
    }
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status kron_op_diagonal(fdp_kron h, double* out) {
  try {
    if (!h || !out) return fail(FDP_ERR_INVALID_ARG, "kron_op_diagonal: NULL argument");
    for (int d = 0; d < h->D; ++d)
      if (h->nin[d] != h->nout[d]) return fail(FDP_ERR_SHAPE, "kron_op_diagonal: operator is not square");
    long long N = 1;
    for (int d = 0; d < h->D; ++d) N *= h->nin[d];
    std::fill(out, out + N, 0.0);
    for (int t = 0; t < h->nterms; ++t) {
      std::vector<const double*> f(h->D);
      for (int d = 0; d < h->D; ++d) f[d] = h->f[t * h->D + d].diag.data();
      kron_diag_accumulate(h->D, h->nin, f, h->coef[t], out);
    }
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status kron_op_destroy(fdp_kron h) {
  try {
    if (!h) return FDP_OK;
    DeviceGuard dg(h->device);
    free_kron(h);
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

static long long kron_prod(const int* v, int D) {
  long long p = 1;
  for (int d = 0; d < D; ++d) p *= v[d];
  return p;
}

// One Kronecker operator application y (+)= alpha op x, batch 1 (grouped multi-operator path).
struct KronTask {
  const fdp_kron_s* op;
  const double* x;
  double* y;
  double alpha;
};
// An extra vector added (times coef) to output y in the combine pass.
struct ExtraPart {
  double* y;
  const double* part;
  double coef;
};

static long long kron_tasks_ws_elems(const std::vector<KronTask>& tasks) {
  long long tot = 0;
  for (const KronTask& t : tasks)
    tot += (long long)t.op->nterms * (2 * kron_max_inter(t.op) + kron_prod(t.op->nout, t.op->D));
  return tot;
}

// For every distinct output Y: Y = beta Y + sum_{tasks into Y} alpha op x + sum_{extras into Y}
// coef part. All terms of all tasks run as one grouped launch per mode (independent problems,
// each writing a private partial), then one summation pass per output.
static cudaError_t enqueue_kron_tasks(const std::vector<KronTask>& tasks, double beta,
                                      const std::vector<ExtraPart>& extra, double* ws,
                                      cudaStream_t s) {
  if (tasks.empty()) return cudaSuccess;
  const int D = tasks[0].op->D;
  struct Term { const fdp_kron_s* op; int t; const double* x; double* T[2]; double* part; double scale; double* y; };
  std::vector<Term> terms;
  for (const KronTask& tk : tasks) {
    const fdp_kron_s* op = tk.op;
    const long long inter = kron_max_inter(op), outn = kron_prod(op->nout, D);
    for (int t = 0; t < op->nterms; ++t) {
      terms.push_back({op, t, tk.x, {ws, ws + inter}, ws + 2 * inter, tk.alpha * op->coef[t], tk.y});
      ws += 2 * inter + outn;
    }
  }
  for (int d = 0; d < D; ++d) {
    std::vector<ModeProb> probs;
    std::vector<TileCfg> cfgs;
    for (const Term& tm : terms) {
      const fdp_kron_s* op = tm.op;
      const KronFactor& kf = op->f[tm.t * D + d];
      long long P = 1, Q = 1;
      for (int e = 0; e < d; ++e) P *= op->nout[e];
      for (int e = d + 1; e < D; ++e) Q *= op->nin[e];
      const bool last = d == D - 1;
      ModeProb p{};
      p.X = d == 0 ? tm.x : tm.T[(d - 1) % 2];
      p.Y = last ? tm.part : tm.T[d % 2];
      p.W = kf.W;
      p.P = (int)P;
      p.n = kf.nin;
      p.nout = kf.nout;
      p.Q = (int)Q;
      p.N = P * kf.nout * Q;
      p.xbs = p.ybs = 0;
      p.batch = 1;
      p.ldw = kf.cfg.ldw;
      p.n1 = p.n1v = 1;
      p.xld = kf.nin;
      p.yld = kf.nout;
      p.vx = p.vy = 0;
      p.epi = last ? EPI_AXPBY : EPI_NONE;
      p.alpha = tm.scale;
      p.beta = 0.0;
      const int BM = kK1Warps * 8 * kf.cfg.MT;
      p.tiles_m = (int)((P * Q + BM - 1) / BM);
      p.tiles_n = kf.cfg.tiles_n;
      p.fd_work = 0;
      probs.push_back(p);
      cfgs.push_back(kf.cfg);
    }
    cudaError_t e = launch_stage(probs, cfgs, d == 0, s, nullptr, nullptr);
    if (e != cudaSuccess) return e;
  }
  std::vector<std::pair<double*, long long>> outs;
  auto add_out = [&](double* y, long long n) {
    for (auto& o : outs)
      if (o.first == y) return;
    outs.push_back({y, n});
  };
  for (const Term& tm : terms) add_out(tm.y, kron_prod(tm.op->nout, D));
  for (const ExtraPart& ex : extra) add_out(ex.y, -1);
  for (auto& o : outs) {
    std::vector<std::pair<const double*, double>> parts;
    for (const Term& tm : terms)
      if (tm.y == o.first) parts.push_back({tm.part, 1.0});
    for (const ExtraPart& ex : extra)
      if (ex.y == o.first) parts.push_back({ex.part, ex.coef});
    double b = beta;
    for (size_t c = 0; c < parts.size(); c += kMaxParts) {
      PartSum ps{};
      ps.nparts = (int)std::min<size_t>(kMaxParts, parts.size() - c);
      for (int j = 0; j < ps.nparts; ++j) {
        ps.parts[j] = parts[c + j].first;
        ps.coef[j] = parts[c + j].second;
      }
      cudaError_t e = launch_partsum(ps, o.first, b, o.second, s);
      if (e != cudaSuccess) return e;
      b = 1.0;
    }
  }
  return cudaSuccess;
}

extern "C" size_t kron_ops_workspace_bytes(int nops, const fdp_kron* ops) {
  try {
    if (nops < 1 || !ops) return 0;
    std::vector<KronTask> tasks;
    for (int i = 0; i < nops; ++i) {
      if (!ops[i]) return 0;
      tasks.push_back({ops[i], nullptr, nullptr, 1.0});
    }
    return (size_t)kron_tasks_ws_elems(tasks) * sizeof(double);
  } catch (...) {
    return 0;
  }
}

extern "C" fdp_status kron_ops_apply(int nops, const fdp_kron* ops, const double* const* x,
                                     double* const* y, const double* alpha, double beta,
                                     void* workspace, void* stream) {
  try {
    if (nops < 1 || !ops || !x || !y || !alpha) return fail(FDP_ERR_INVALID_ARG, "kron_ops_apply: bad arguments");
    const int D = ops[0] ? ops[0]->D : 0;
    std::vector<KronTask> tasks;
    for (int i = 0; i < nops; ++i) {
      if (!ops[i] || ops[i]->D != D) return fail(FDP_ERR_INVALID_ARG, "kron_ops_apply: NULL or mixed-D operator");
      if (!is_device_ptr(x[i]) || !is_device_ptr(y[i])) return fail(FDP_ERR_INVALID_ARG, "kron_ops_apply: device pointers required");
      tasks.push_back({ops[i], x[i], y[i], alpha[i]});
    }
    if (!is_device_ptr(workspace)) return fail(FDP_ERR_INVALID_ARG, "kron_ops_apply: workspace must be device memory");
    DeviceGuard dg(ops[0]->device);
    FDP_CUDA(enqueue_kron_tasks(tasks, beta, {}, static_cast<double*>(workspace), static_cast<cudaStream_t>(stream)),
             "kron_ops_apply");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

// ------------------------------------------------------------------------------------------------
// block-triangular P_T and constrained P_C (§4)
// ------------------------------------------------------------------------------------------------
static long long vel_ws_elems(const fdp_block_s* h) {
  long long v = 0;
  for (const fdp_fd_s* f : h->vel) v += 2 * Npad(f);
  return v;
}

// s_u = P_V^{-1} r_u on the contiguous velocity part [u_1 | .. | u_D] (batch 1); s_u may not alias r_u
static cudaError_t enqueue_vel(const fdp_block_s* h, const double* ru, double* su, double* T,
                               cudaStream_t st) {
  const int D = h->D;
  std::vector<const double*> in(D), dsc(D);
  std::vector<double*> out(D), Tk(D);
  long long toff = 0;
  if (h->dv) {
    cudaError_t e = launch_scale(ru, su, h->dv, h->nvel, 1, h->nvel, h->nvel, st);
    if (e != cudaSuccess) return e;
  }
  for (int k = 0; k < D; ++k) {
    in[k] = (h->dv ? su : ru) + h->off[k];
    out[k] = su + h->off[k];
    Tk[k] = T + toff;
    toff += 2 * Npad(h->vel[k]);
    dsc[k] = h->dv ? h->dv + h->off[k] : nullptr;
  }
  return enqueue_fd(h->vel, in, h->nvel, out, h->nvel, Tk, dsc, 1, st, nullptr);
}

static fdp_status check_tri_args(fdp_block h, int variant, const fdp_kron* B, const fdp_kron* BT,
                                 const char* who) {
  if (!h || !B || !BT) return fail(FDP_ERR_INVALID_ARG, std::string(who) + ": NULL argument");
  if (variant != FDP_PREC_TRIANGULAR && variant != FDP_PREC_CONSTRAINED)
    return fail(FDP_ERR_INVALID_ARG, std::string(who) + ": unknown variant");
  const int D = h->D;
  for (int k = 0; k < D; ++k) {
    if (!B[k] || !BT[k] || B[k]->D != D || BT[k]->D != D)
      return fail(FDP_ERR_INVALID_ARG, std::string(who) + ": NULL or mismatched B / B^T handle");
    for (int d = 0; d < D; ++d)
      if (B[k]->nin[d] != h->vel[k]->n[d] || B[k]->nout[d] != h->pres->n[d] ||
          BT[k]->nin[d] != h->pres->n[d] || BT[k]->nout[d] != h->vel[k]->n[d])
        return fail(FDP_ERR_SHAPE, std::string(who) + ": B_k / B_k^T extents do not match the blocks");
  }
  return FDP_OK;
}

static long long tri_ws_elems(const fdp_block_s* h, int variant, const fdp_kron* B, const fdp_kron* BT) {
  std::vector<KronTask> tb, tbt;
  for (int k = 0; k < h->D; ++k) {
    tb.push_back({B[k], nullptr, nullptr, 1.0});
    tbt.push_back({BT[k], nullptr, nullptr, 1.0});
  }
  const long long kr = std::max(kron_tasks_ws_elems(tbt), variant == FDP_PREC_CONSTRAINED ? kron_tasks_ws_elems(tb) : 0LL);
  return vel_ws_elems(h) + kr + 2 * h->nvel + h->pres->N;
}

extern "C" size_t block_tri_workspace_bytes(fdp_block h, int variant, const fdp_kron* B,
                                            const fdp_kron* BT) {
  try {
    if (check_tri_args(h, variant, B, BT, "block_tri_workspace_bytes")) return 0;
    return (size_t)tri_ws_elems(h, variant, B, BT) * sizeof(double);
  } catch (...) {
    return 0;
  }
}

extern "C" fdp_status block_tri_apply(fdp_block h, int variant, const fdp_kron* B, const fdp_kron* BT,
                                      const double* r, double* s, void* workspace, void* stream) {
  try {
    fdp_status cs = check_tri_args(h, variant, B, BT, "block_tri_apply");
    if (cs) return cs;
    if (!is_device_ptr(r) || !is_device_ptr(s) || !is_device_ptr(workspace))
      return fail(FDP_ERR_INVALID_ARG, "block_tri_apply: r, s and workspace must be device memory");
    if (r == s) return fail(FDP_ERR_INVALID_ARG, "block_tri_apply: r and s must not alias");
    DeviceGuard dg(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int D = h->D;
    const long long nv = h->nvel;
    double* T = static_cast<double*>(workspace);        // velocity FD intermediates
    double* K = T + vel_ws_elems(h);                    // Kronecker partials
    std::vector<KronTask> tb, tbt;
    for (int k = 0; k < D; ++k) {
      tb.push_back({B[k], nullptr, nullptr, 1.0});
      tbt.push_back({BT[k], nullptr, nullptr, 1.0});
    }
    const long long kr = std::max(kron_tasks_ws_elems(tbt), variant == FDP_PREC_CONSTRAINED ? kron_tasks_ws_elems(tb) : 0LL);
    double* tu = K + kr;                                // velocity temporaries
    double* zu = tu + nv;
    double* tp = zu + nv;                               // pressure temporary
    const double* ru = r;
    const double* rp = r + nv;
    double* su = s;
    double* sp = s + nv;
    auto negate = [&](const double* a, double* y, long long n) {
      PartSum ps{};
      ps.nparts = 1;
      ps.parts[0] = a;
      ps.coef[0] = -1.0;
      return launch_partsum(ps, y, 0.0, n, st);
    };
    if (variant == FDP_PREC_TRIANGULAR) {
      // [[P_V, B^T], [0, -P_Q]] s = r: t_p = P_Q^{-1} r_p, s_p = -t_p, s_u = P_V^{-1}(r_u + B^T t_p)
      FDP_CUDA(enqueue_mass(h->pres, FDP_MASS_INVERSE, rp, tp, h->pres->N, h->dq, 1, st, nullptr), "block_tri_apply: P_Q");
      for (int k = 0; k < D; ++k) {
        tbt[k].x = tp;
        tbt[k].y = tu + h->off[k];
      }
      std::vector<ExtraPart> ex;
      for (int k = 0; k < D; ++k) ex.push_back({tu + h->off[k], ru + h->off[k], 1.0});
      FDP_CUDA(enqueue_kron_tasks(tbt, 0.0, ex, K, st), "block_tri_apply: B^T");
      FDP_CUDA(enqueue_vel(h, tu, su, T, st), "block_tri_apply: P_V");
      FDP_CUDA(negate(tp, sp, h->pres->N), "block_tri_apply: negate");
      return FDP_OK;
    }
    // P_C^{-1} = [[I, -P_V^{-1}B^T], [0, I]] diag(I, -P_Q^{-1}) [[I, 0], [-B, I]] diag(P_V^{-1}, I)
    FDP_CUDA(enqueue_vel(h, ru, su, T, st), "block_tri_apply: P_V");                 // w_u
    for (int k = 0; k < D; ++k) {
      tb[k].x = su + h->off[k];
      tb[k].y = zu;  // g_p = r_p - B w_u (zu reused as the pressure temporary g_p)
      tb[k].alpha = -1.0;
    }
    FDP_CUDA(enqueue_kron_tasks(tb, 0.0, {{zu, rp, 1.0}}, K, st), "block_tri_apply: B");
    FDP_CUDA(enqueue_mass(h->pres, FDP_MASS_INVERSE, zu, tp, h->pres->N, h->dq, 1, st, nullptr), "block_tri_apply: P_Q");
    FDP_CUDA(negate(tp, sp, h->pres->N), "block_tri_apply: negate");                 // s_p = -t_p
    for (int k = 0; k < D; ++k) {
      tbt[k].x = tp;
      tbt[k].y = tu + h->off[k];
    }
    FDP_CUDA(enqueue_kron_tasks(tbt, 0.0, {}, K, st), "block_tri_apply: B^T");        // B^T t_p
    FDP_CUDA(enqueue_vel(h, tu, zu, T, st), "block_tri_apply: P_V");                 // P_V^{-1} B^T t_p
    PartSum ps{};
    ps.nparts = 1;
    ps.parts[0] = zu;
    ps.coef[0] = 1.0;
    FDP_CUDA(launch_partsum(ps, su, 1.0, nv, st), "block_tri_apply: update");        // s_u = w_u - P_V^{-1} B^T s_p
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_vec_lincomb_dev(const double* coef, const double* x, const double* y,
                                          const double* z, double* out, int64_t n, void* stream) {
  try {
    if (n < 0) return fail(FDP_ERR_SHAPE, "fdp_vec_lincomb_dev: n < 0");
    if (n == 0) return FDP_OK;
    if (!is_device_ptr(coef) || !is_device_ptr(x) || !is_device_ptr(out) || (y && !is_device_ptr(y)) ||
        (z && !is_device_ptr(z)))
      return fail(FDP_ERR_INVALID_ARG, "fdp_vec_lincomb_dev: device pointers required");
    FDP_CUDA(launch_lincomb_dev(coef, x, y, z, out, n, static_cast<cudaStream_t>(stream)), "fdp_vec_lincomb_dev");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_minres_scalars(int phase, double* state, double* hist, int hist_cap,
                                         void* stream) {
  try {
    if (phase < 0 || phase > 3 || hist_cap < 0) return fail(FDP_ERR_INVALID_ARG, "fdp_minres_scalars: bad phase");
    if (!is_device_ptr(state) || (hist && !is_device_ptr(hist)))
      return fail(FDP_ERR_INVALID_ARG, "fdp_minres_scalars: device pointers required");
    FDP_CUDA(launch_minres_scalars(phase, state, hist, hist_cap, static_cast<cudaStream_t>(stream)),
             "fdp_minres_scalars");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_vec_copy_indexed(const double* V, int64_t ldv, const int* idx, double* out,
                                           int64_t n, void* stream) {
  try {
    if (n < 0 || ldv < n) return fail(FDP_ERR_SHAPE, "fdp_vec_copy_indexed: bad extents");
    if (!is_device_ptr(V) || !is_device_ptr(idx) || !is_device_ptr(out))
      return fail(FDP_ERR_INVALID_ARG, "fdp_vec_copy_indexed: device pointers required");
    FDP_CUDA(launch_copy_indexed(V, ldv, idx, out, n, static_cast<cudaStream_t>(stream)), "fdp_vec_copy_indexed");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_vec_store_indexed(double* V, int64_t ldv, const int* idx, const double* w,
                                            const double* coef, int64_t n, void* stream) {
  try {
    if (n < 0 || ldv < n) return fail(FDP_ERR_SHAPE, "fdp_vec_store_indexed: bad extents");
    if (!is_device_ptr(V) || !is_device_ptr(idx) || !is_device_ptr(w) || !is_device_ptr(coef))
      return fail(FDP_ERR_INVALID_ARG, "fdp_vec_store_indexed: device pointers required");
    FDP_CUDA(launch_store_indexed(V, ldv, idx, w, coef, n, static_cast<cudaStream_t>(stream)), "fdp_vec_store_indexed");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_vec_multidot_dev(const double* V, int64_t ldv, const int* m, int m_max,
                                           const double* w, int64_t n, double* h, void* workspace,
                                           void* stream) {
  try {
    if (m_max < 0 || n < 0 || (m_max > 0 && ldv < n)) return fail(FDP_ERR_SHAPE, "fdp_vec_multidot_dev: bad extents");
    if (m_max == 0) return FDP_OK;
    if (!is_device_ptr(V) || !is_device_ptr(m) || !is_device_ptr(w) || !is_device_ptr(h) || !is_device_ptr(workspace))
      return fail(FDP_ERR_INVALID_ARG, "fdp_vec_multidot_dev: device pointers required");
    FDP_CUDA(launch_multidot_dev(V, ldv, m, m_max, w, n, h, static_cast<double*>(workspace),
                                 static_cast<cudaStream_t>(stream)), "fdp_vec_multidot_dev");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_vec_gemv_dev(const double* V, int64_t ldv, const int* m, int m_max,
                                       const double* h, double alpha, double* w, double beta,
                                       int64_t n, void* stream) {
  try {
    if (m_max < 0 || m_max > 6144 || n < 0 || ldv < n) return fail(FDP_ERR_SHAPE, "fdp_vec_gemv_dev: bad extents");
    if (n == 0) return FDP_OK;
    if (!is_device_ptr(V) || !is_device_ptr(m) || !is_device_ptr(h) || !is_device_ptr(w))
      return fail(FDP_ERR_INVALID_ARG, "fdp_vec_gemv_dev: device pointers required");
    FDP_CUDA(launch_gemv_dev(V, ldv, m, m_max, h, alpha, w, beta, n, static_cast<cudaStream_t>(stream)),
             "fdp_vec_gemv_dev");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_gmres_scalars(int phase, int* istate, double* dstate, double* H, int ldh,
                                        const double* h1, const double* h2, double* hist, int m_max,
                                        void* stream) {
  try {
    if ((phase != 0 && phase != 1) || m_max < 1 || ldh < m_max + 1)
      return fail(FDP_ERR_INVALID_ARG, "fdp_gmres_scalars: bad phase or extents");
    if (!is_device_ptr(istate) || !is_device_ptr(dstate) || !is_device_ptr(H) || !is_device_ptr(h1) ||
        !is_device_ptr(h2) || (hist && !is_device_ptr(hist)))
      return fail(FDP_ERR_INVALID_ARG, "fdp_gmres_scalars: device pointers required");
    FDP_CUDA(launch_gmres_scalars(phase, istate, dstate, H, ldh, h1, h2, hist, m_max,
                                  static_cast<cudaStream_t>(stream)), "fdp_gmres_scalars");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

// ------------------------------------------------------------------------------------------------
// Arnoldi helpers (GMRES orthogonalization, NEXT-2)
// ------------------------------------------------------------------------------------------------
extern "C" size_t fdp_vec_multidot_workspace_bytes(int m) {
  try {
    return m > 0 ? multidot_scratch_elems(m) * sizeof(double) : 0;
  } catch (...) {
    return 0;
  }
}

extern "C" fdp_status fdp_vec_multidot(const double* V, int64_t ldv, int m, const double* w,
                                       int64_t n, double* h, void* workspace, void* stream) {
  try {
    if (m < 0 || n < 0 || (m > 0 && ldv < n)) return fail(FDP_ERR_SHAPE, "fdp_vec_multidot: bad extents");
    if (m == 0) return FDP_OK;
    if (!is_device_ptr(V) || !is_device_ptr(w) || !is_device_ptr(h) || !is_device_ptr(workspace))
      return fail(FDP_ERR_INVALID_ARG, "fdp_vec_multidot: device pointers required");
    FDP_CUDA(launch_multidot(V, ldv, m, w, n, h, static_cast<double*>(workspace), static_cast<cudaStream_t>(stream)),
             "fdp_vec_multidot");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_vec_gemv(const double* V, int64_t ldv, int m, const double* h, double alpha,
                                   double* w, double beta, int64_t n, void* stream) {
  try {
    if (m < 0 || m > 6144 || n < 0 || (m > 0 && ldv < n)) return fail(FDP_ERR_SHAPE, "fdp_vec_gemv: bad extents (m <= 6144)");
    if (n == 0) return FDP_OK;
    if (!is_device_ptr(w) || (m > 0 && (!is_device_ptr(V) || !is_device_ptr(h))))
      return fail(FDP_ERR_INVALID_ARG, "fdp_vec_gemv: device pointers required");
    FDP_CUDA(launch_gemv(V, ldv, m, h, alpha, w, beta, n, static_cast<cudaStream_t>(stream)), "fdp_vec_gemv");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}
