// C ABI of libfdp (include/fdp.h): handle lifetime, argument validation, error reporting and the
// launch orchestration of the preconditioner application (§4-§5: P_D of P:591-598,
// Algorithm 1 of P:1003-1011, P_Q solve of P:975-976, diagonal scaling of P:1038-1059).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
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
  if (!n_out) return fail(FDP_ERR_INVALID_ARG, "iga_univariate: n_out is NULL");
  std::string err;
  int n = 0;
  int st = iga_build(deg, alpha, n_el, flags, c_pen, q, K, M, &n, &err);
  if (st) return fail((fdp_status)st, err);
  *n_out = n;
  return FDP_OK;
}

extern "C" fdp_status iga_greville(int deg, int alpha, int n_el, int flags, double* g,
                                   int32_t* n_out) {
  if (!n_out) return fail(FDP_ERR_INVALID_ARG, "iga_greville: n_out is NULL");
  std::string err;
  int n = 0;
  int st = iga_greville_build(deg, alpha, n_el, flags, g, &n, &err);
  if (st) return fail((fdp_status)st, err);
  *n_out = n;
  return FDP_OK;
}

extern "C" fdp_status fdp_gen_eig(int n, const double* K, const double* M, double* U,
                                  double* lambda) {
  if (n < 1) return fail(FDP_ERR_SHAPE, "fdp_gen_eig: n < 1");
  if (!K || !M || !U || !lambda) return fail(FDP_ERR_INVALID_ARG, "fdp_gen_eig: NULL argument");
  std::string err;
  int st = gen_eig(n, K, M, U, lambda, &err);
  if (st) return fail((fdp_status)st, "fdp_gen_eig: " + err);
  return FDP_OK;
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
  double* Wf[3] = {nullptr, nullptr, nullptr};  // forward  W[k][a] = U[k][a]
  double* Wb[3] = {nullptr, nullptr, nullptr};  // backward W[k][a] = U[a][k]
  double* lamc[3] = {nullptr, nullptr, nullptr};  // coef[d] * lambda_d
  double* ws = nullptr;
  int64_t ws_batch = 0;
};

static void free_fd(fdp_fd h) {
  if (!h) return;
  for (int d = 0; d < 3; ++d) {
    cudaFree(h->Wf[d]);
    cudaFree(h->Wb[d]);
    cudaFree(h->lamc[d]);
  }
  cudaFree(h->ws);
  delete h;
}

extern "C" fdp_status fd_setup(int D, const int32_t* n, const double* const* K,
                               const double* const* M, const double* coef, int device,
                               int64_t max_batch, fdp_fd* out) {
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
    std::vector<double> wf((size_t)c.kpad * c.ldw, 0.0), wb((size_t)c.kpad * c.ldw, 0.0);
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
        (e = prepare_mode_kernels(c))) {
      free_fd(raw);
      return cuda_fail(e, "fd_setup: upload");
    }
  }
  if (max_batch > 0) {
    fdp_status st = dalloc(&raw->ws, (size_t)(max_batch * N));
    if (st) {
      free_fd(raw);
      return st;
    }
    raw->ws_batch = max_batch;
  }
  *out = raw;
  return FDP_OK;
}

extern "C" fdp_status fd_get_eigs(fdp_fd h, int d, double* U_out, double* lambda_out) {
  if (!h) return fail(FDP_ERR_INVALID_ARG, "fd_get_eigs: NULL handle");
  if (d < 0 || d >= h->D) return fail(FDP_ERR_SHAPE, "fd_get_eigs: d out of range");
  if (U_out) std::memcpy(U_out, h->U_host[d].data(), h->U_host[d].size() * 8);
  if (lambda_out) std::memcpy(lambda_out, h->lam_host[d].data(), h->lam_host[d].size() * 8);
  return FDP_OK;
}

extern "C" int64_t fd_size(fdp_fd h) { return h ? h->N : 0; }
extern "C" size_t fd_workspace_bytes(fdp_fd h, int64_t batch) {
  return h && batch > 0 ? (size_t)(batch * h->N) * sizeof(double) : 0;
}

// One FD problem inside a grouped stage: mode d (0-based), direction fwd/bwd.
static ModeProb make_mode_prob(const fdp_fd_s* h, int d, bool fwd, const double* X, long long xbs,
                               double* Y, long long ybs, int64_t batch, int epi, const double* scale) {
  ModeProb p{};
  long long P = 1, Q = 1;
  for (int e = 0; e < d; ++e) P *= h->n[e];
  for (int e = d + 1; e < h->D; ++e) Q *= h->n[e];
  p.X = X;
  p.Y = Y;
  p.W = fwd ? h->Wf[d] : h->Wb[d];
  p.N = h->N;
  p.xbs = xbs;
  p.ybs = ybs;
  p.P = (int)P;
  p.n = h->n[d];
  p.Q = (int)Q;
  p.batch = (int)batch;
  p.ldw = h->cfg[d].ldw;
  p.n1 = h->n[0];
  p.epi = epi;
  p.scale = scale;
  if (epi == EPI_LAMBDA) {
    p.lam0 = h->lamc[0];
    p.lam1 = h->D == 3 ? h->lamc[1] : nullptr;
    p.lamcol = h->lamc[h->D - 1];
  }
  const int BM = 4 * 8 * h->cfg[d].MT;
  const long long M = P * Q * batch;
  p.tiles_m = (int)((M + BM - 1) / BM);
  p.tiles_n = h->cfg[d].tiles_n;
  return p;
}

// Stage = one mode/direction for a set of FD problems. Problems with the same tile config share a
// launch (up to kMaxGroup); others get their own.
static cudaError_t launch_stage(std::vector<ModeProb>& probs, const std::vector<TileCfg>& cfgs,
                                bool kmaj, cudaStream_t s, int* nlaunch, Recorder* rec) {
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
    if (rec) {
      double fl = 0.0, by = 0.0;
      for (int j = 0; j < g.count; ++j) {
        const ModeProb& p = g.prob[j];
        const double elems = (double)p.P * p.Q * p.batch * p.n;
        fl += 2.0 * elems * p.n;
        by += 16.0 * elems + (p.epi == EPI_SCALE ? 8.0 * p.N : 0.0);
      }
      cudaError_t e0 = rec->before(0, fl, by);
      if (e0 != cudaSuccess) return e0;
    }
    cudaError_t e = launch_mode_group(g, cfgs[i], kmaj, s);
    if (e != cudaSuccess) return e;
    if (nlaunch) ++*nlaunch;
  }
  return cudaSuccess;
}

// Enqueue FD solves for several handles (block components) on stream s.
// in[k], out[k] with batch strides ibs/obs; T[k] workspace with stride N_k. dscale[k] may be NULL.
// Pre-scaling (if any) must already have been applied by the caller (into out[k]) and `in` point
// at it.
static cudaError_t enqueue_fd(const std::vector<const fdp_fd_s*>& hs,
                              const std::vector<const double*>& in, long long ibs,
                              const std::vector<double*>& out, long long obs,
                              const std::vector<double*>& T,
                              const std::vector<const double*>& dscale, int64_t batch,
                              cudaStream_t s, int* nlaunch, Recorder* rec = nullptr) {
  const int D = hs[0]->D;
  const size_t K = hs.size();
  // pass sequence: forward d = 0..D-1, backward d = D-1..0; 2D passes alternate T <- src, out <- T
  int pass = 0;
  for (int dir = 0; dir < 2; ++dir) {
    for (int step = 0; step < D; ++step) {
      const int d = dir == 0 ? step : D - 1 - step;
      const bool fwd = dir == 0;
      std::vector<ModeProb> probs;
      std::vector<TileCfg> cfgs;
      for (size_t k = 0; k < K; ++k) {
        const double* src;
        long long sbs;
        double* dst;
        long long dbs;
        if (pass == 0) { src = in[k]; sbs = ibs; } else if (pass % 2 == 1) { src = T[k]; sbs = hs[k]->N; } else { src = out[k]; sbs = obs; }
        if (pass % 2 == 0) { dst = T[k]; dbs = hs[k]->N; } else { dst = out[k]; dbs = obs; }
        int epi = EPI_NONE;
        const double* sc = nullptr;
        if (fwd && d == D - 1) epi = EPI_LAMBDA;
        if (!fwd && d == 0 && dscale[k]) { epi = EPI_SCALE; sc = dscale[k]; }
        probs.push_back(make_mode_prob(hs[k], d, fwd, src, sbs, dst, dbs, batch, epi, sc));
        cfgs.push_back(hs[k]->cfg[d]);
      }
      cudaError_t e = launch_stage(probs, cfgs, d == 0, s, nlaunch, rec);
      if (e != cudaSuccess) return e;
      ++pass;
    }
  }
  return cudaSuccess;
}

extern "C" fdp_status fd_apply(fdp_fd h, const double* b, double* x, const double* dscale,
                               int64_t batch, void* workspace, void* stream) {
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
  FDP_CUDA(enqueue_fd({h}, {src}, h->N, {x}, h->N, {T}, {dscale}, batch, s, nullptr), "fd_apply");
  return FDP_OK;
}

extern "C" fdp_status fd_destroy(fdp_fd h) {
  if (!h) return FDP_OK;
  DeviceGuard dg(h->device);
  free_fd(h);
  return FDP_OK;
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
}

extern "C" fdp_status kron_mass_destroy(fdp_mass h) {
  if (!h) return FDP_OK;
  DeviceGuard dg(h->device);
  free_mass(h);
  return FDP_OK;
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
  cudaStream_t cap = nullptr;  // private capture stream
  // graph cache
  std::mutex mu;
  const double* g_r = nullptr;
  double* g_s = nullptr;
  void* g_ws = nullptr;
  int64_t g_batch = -1;
  cudaGraphExec_t exec = nullptr;
  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> ev;
  std::vector<LaunchInfo> info;
  // host e2e buffers
  double* e2e_r = nullptr;
  double* e2e_s = nullptr;
  void* e2e_ws = nullptr;
  int64_t e2e_batch = 0;
};

static void free_block(fdp_block h) {
  if (!h) return;
  for (cudaEvent_t e : h->ev) cudaEventDestroy(e);
  if (h->exec) cudaGraphExecDestroy(h->exec);
  if (h->cap) cudaStreamDestroy(h->cap);
  cudaFree(h->dv);
  cudaFree(h->dq);
  cudaFree(h->e2e_r);
  cudaFree(h->e2e_s);
  cudaFree(h->e2e_ws);
  delete h;
}

extern "C" fdp_status block_precond_setup(int D, const fdp_fd* vel, fdp_mass pres,
                                          const double* dscale_vel, const double* dscale_pres,
                                          fdp_block* out) {
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
}

extern "C" int64_t block_precond_size(fdp_block h) { return h ? h->size : 0; }
extern "C" size_t block_precond_workspace_bytes(fdp_block h, int64_t batch) {
  return h && batch > 0 ? (size_t)(batch * h->nvel) * sizeof(double) : 0;
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
    T[k] = ws + toff;  // component k workspace: batch x N_k, compact
    toff += h->vel[k]->N * batch;
    dsc[k] = h->dv ? h->dv + h->off[k] : nullptr;
  }
  if (h->dv) {
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
  cudaError_t e = enqueue_fd(h->vel, in, sz, out, sz, T, dsc, batch, st, nlaunch, rec);
  if (e != cudaSuccess) return e;
  // pressure block: r_p -> s_p
  e = enqueue_mass(h->pres, FDP_MASS_INVERSE, r + h->off[D], s + h->off[D], sz, h->dq, batch, st,
                   nlaunch, rec);
  if (e != cudaSuccess) return e;
  return rec ? rec->finish() : cudaSuccess;
}

extern "C" fdp_status block_precond_profile(fdp_block h, int enable) {
  if (!h) return fail(FDP_ERR_INVALID_ARG, "block_precond_profile: NULL handle");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard dg(h->device);
  if (enable && h->ev.empty()) {
    h->ev.resize(64);
    for (auto& e : h->ev) FDP_CUDA(cudaEventCreate(&e), "block_precond_profile: event");
  }
  if ((enable != 0) != h->prof) {
    h->prof = enable != 0;
    if (h->exec) {  // force re-capture with / without event nodes
      cudaGraphExecDestroy(h->exec);
      h->exec = nullptr;
    }
  }
  return FDP_OK;
}

extern "C" int block_precond_profile_read(fdp_block h, int max, int32_t* kind, float* ms,
                                          double* flops, double* bytes) {
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
}

extern "C" int fdp_block_launch_count(fdp_block h, int64_t batch) {
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
  n += h->pres->D;
  return n;
}

extern "C" fdp_status block_precond_apply(fdp_block h, const double* r, double* s, int64_t batch,
                                          void* workspace, void* stream) {
  if (!h) return fail(FDP_ERR_INVALID_ARG, "block_precond_apply: NULL handle");
  if (batch < 0) return fail(FDP_ERR_SHAPE, "block_precond_apply: batch < 0");
  if (batch == 0) return FDP_OK;
  std::lock_guard<std::mutex> lk(h->mu);
  const bool same = h->exec && r == h->g_r && s == h->g_s && workspace == h->g_ws && batch == h->g_batch;
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
  if (cs == cudaStreamCaptureStatusActive) {
    FDP_CUDA(enqueue_block(h, r, s, batch, static_cast<double*>(workspace), st, nullptr),
             "block_precond_apply");
    return FDP_OK;
  }
  if (!same) {
    if (h->exec) {
      cudaGraphExecDestroy(h->exec);
      h->exec = nullptr;
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
    e = cudaGraphInstantiate(&h->exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      h->exec = nullptr;
      return cuda_fail(e, "block_precond_apply: instantiate");
    }
    h->g_r = r;
    h->g_s = s;
    h->g_ws = workspace;
    h->g_batch = batch;
  }
  FDP_CUDA(cudaGraphLaunch(h->exec, st), "block_precond_apply: graph launch");
  return FDP_OK;
}

extern "C" fdp_status block_precond_apply_host(fdp_block h, const double* r_host, double* s_host,
                                               int64_t batch, void* stream) {
  if (!h) return fail(FDP_ERR_INVALID_ARG, "block_precond_apply_host: NULL handle");
  if (!r_host || !s_host) return fail(FDP_ERR_INVALID_ARG, "block_precond_apply_host: NULL buffer");
  if (batch <= 0) return batch == 0 ? FDP_OK : fail(FDP_ERR_SHAPE, "block_precond_apply_host: batch < 0");
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
        (st = dalloc(reinterpret_cast<double**>(&h->e2e_ws), (size_t)(batch * h->nvel))))
      return st;
    h->e2e_batch = batch;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t bytes = (size_t)(batch * h->size) * sizeof(double);
  FDP_CUDA(cudaMemcpyAsync(h->e2e_r, r_host, bytes, cudaMemcpyHostToDevice, st), "apply_host: H2D");
  fdp_status s = block_precond_apply(h, h->e2e_r, h->e2e_s, batch, h->e2e_ws, stream);
  if (s) return s;
  FDP_CUDA(cudaMemcpyAsync(s_host, h->e2e_s, bytes, cudaMemcpyDeviceToHost, st), "apply_host: D2H");
  FDP_CUDA(cudaStreamSynchronize(st), "apply_host: sync");
  return FDP_OK;
}

extern "C" fdp_status block_precond_destroy(fdp_block h) {
  if (!h) return FDP_OK;
  DeviceGuard dg(h->device);
  free_block(h);
  return FDP_OK;
}
