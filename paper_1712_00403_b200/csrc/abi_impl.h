// Internal header of the C ABI implementation (abi_*.cpp): shared helpers, error reporting,
// handle structs and the launch orchestration entry points used across the ABI files.
#pragma once
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
#include "mode_tma.h"


// ------------------------------------------------------------------------------------------------
// errors
// ------------------------------------------------------------------------------------------------
inline thread_local std::string g_last_error;

inline fdp_status fail(fdp_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}
// No C++ exception crosses the C ABI: every entry point catches and reports (mostly
// std::bad_alloc from host-side containers). Called from inside a catch handler.
inline fdp_status abi_exception(const char* fn) {
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

inline fdp_status cuda_fail(cudaError_t e, const char* where) {
  cudaGetLastError();  // clear sticky-free errors
  return fail(FDP_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define FDP_CUDA(call, where)                                  \
  do {                                                         \
    cudaError_t e_ = (call);                                   \
    if (e_ != cudaSuccess) return cuda_fail(e_, where);        \
  } while (0)

// A pointer is acceptable as a device operand if the runtime knows it as device or managed memory.
inline bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

inline int num_sms() {
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
inline fdp_status dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) return FDP_OK;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(FDP_ERR_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  return FDP_OK;
}

inline bool symmetric(int n, const double* A) {
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

using namespace fdp;

// ------------------------------------------------------------------------------------------------
// handle structs
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
  // even-odd folded transforms: modes with a persymmetric pencil and a small-path
  // extent. WfF / WbF: blocks E (rows [0, foldh)) and O (rows [foldh, 2 foldh)), ldwF columns;
  // lamcF: coef[d] * lambda_d in the folded spectral order [E | O] (= lamc for unfolded modes).
  // The dense Wf / Wb / lamc stay for the slab-sharded paths.
  int fold[3] = {0, 0, 0};
  int fold_nt[3] = {0, 0, 0};  // small-kernel NT of a folded mode: 2 * ceil(ceil(n/2) / 8)
  int foldh[3] = {0, 0, 0};
  int ldwF[3] = {0, 0, 0};     // forward matrix columns (small-path fold: both matrices)
  int ldwFb[3] = {0, 0, 0};    // backward matrix columns
  // fold[d] == 2: K1-path fold (n > 96), tile configs of the forward / backward transforms
  TileCfg cfgFf[3], cfgFb[3];
  int tiles_ne[3] = {0, 0, 0};
  double* WfF[3] = {nullptr, nullptr, nullptr};
  double* WbF[3] = {nullptr, nullptr, nullptr};
  double* lamcF[3] = {nullptr, nullptr, nullptr};
  // K1t fragment-native chunks of the folded forward / backward matrices (fold[d] == 2)
  double* WtF[3] = {nullptr, nullptr, nullptr};
  double* WtB[3] = {nullptr, nullptr, nullptr};
  // 1 / Lambda in the output layout of the Lambda pass (padded rows n1p, last mode's folded
  // spectral order; 0 at pad rows), when that pass runs on K1t (fold[D-1] == 2)
  double* rlam = nullptr;
  double* ws = nullptr;
  int64_t ws_batch = 0;
};

// Intermediate tensors between passes use an even leading dimension n1p (16-byte aligned rows
// and row pairs for vector memory operations); the C-ABI input/output stay unpadded.
static int n1pad(const fdp_fd_s* h) { return h->n[0] + (h->n[0] & 1); }
static long long Npad(const fdp_fd_s* h) { return h->N / h->n[0] * n1pad(h); }

struct fdp_mass_s {
  int D = 0;
  int n[3] = {1, 1, 1};
  int band[3] = {0, 0, 0};
  long long N = 0;
  int device = 0;
  double* Lb[3] = {nullptr, nullptr, nullptr};
  double* invd[3] = {nullptr, nullptr, nullptr};
  double* Mb[3] = {nullptr, nullptr, nullptr};
  double* cf[3] = {nullptr, nullptr, nullptr};  // K3t coefficients (MassMode::cf / cb)
  double* cb[3] = {nullptr, nullptr, nullptr};
  std::vector<double> Lb_host[3];
};

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
  int q_fold[3] = {0, 0, 0};   // M_d^{-1} is centrosymmetric: folded (FOLD_SYM) pass, Wq = E | O
                               // (1: small path, riding in the velocity launch; 2: folded K1)
  TileCfg q_cfgF[3];           // q_fold == 2: tile shape of the folded K1 pass
  int q_foldh[3] = {0, 0, 0};
  cudaStream_t cap = nullptr;  // private capture stream
  // banded pressure solve on its own branch of a captured apply (enqueue_block): the pressure
  // block is independent of the velocity blocks, and the velocity path's memory-bound first
  // launch (the row-padding pass) fits under the issue-bound pressure kernels
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // graph cache
  std::mutex mu;
  struct GraphEntry {
    const double* r;
    double* s;
    void* ws;
    int64_t batch;
    cudaGraphExec_t exec;
    unsigned long long used;
    int kernels;  // kernel nodes of the captured apply (fdp_block_launch_count)
  };
  std::vector<GraphEntry> graphs;  // small LRU cache keyed by (r, s, workspace, batch)
  std::vector<std::pair<int64_t, int>> launch_counts;  // (batch, kernels) of captured applies
  unsigned long long tick = 0;
  // plane-pipeline counters (zeroed at allocation, self-resetting)
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

struct KronFactor {
  int nin = 0, nout = 0;
  TileCfg cfg{};
  std::vector<double> diag;  // F[i][i] for i < min(nin, nout) (kron_op_diagonal)
  double* W = nullptr;  // W[k][a] = F[a][k], kpad x ldw
  // banded copy (bw > 0): row a's nonzeros F[a][lo[a] .. lo[a] + bw) (K4, kernels/kron_band.cu)
  int bw = 0;
  int* lo = nullptr;
  double* Wb = nullptr;
};

struct fdp_kron_s {
  int D = 0, nterms = 0, device = 0;
  int nin[3] = {1, 1, 1}, nout[3] = {1, 1, 1};
  std::vector<double> coef;
  std::vector<KronFactor> f;  // nterms * D
};

// ------------------------------------------------------------------------------------------------
// launch orchestration shared by the ABI files (abi_fd.cpp)
// ------------------------------------------------------------------------------------------------
// K1t host side (abi_tma.cpp)
#include <atomic>
namespace fdp {
extern std::atomic<long long> g_k1_launches[2];  // [0] K1f folded launches, [1] K1t
int tma_ctiles(int ne);
std::vector<double> tma_wt_build(int n, int foldh, int ldw, const std::vector<double>& w, bool kmaj);
bool tma_eligible(const ModeProb& p, bool kmaj);
bool tma_input_ok(const ModeProb& p, bool kmaj);
cudaError_t launch_tma_stage(const ModeProb* probs, int count, bool kmaj, cudaStream_t s);
// rlam[p + P a] = 1 / (lam0[p % n1p] + lam1[p / n1p] + lamcol[a]) (lam1 NULL: no middle term), 0 for
// p % n1p >= n1v; P = n1p * n_mid
cudaError_t launch_rlam(double* rlam, const double* lam0, const double* lam1, const double* lamcol, int n1p,
                        int n1v, int n_mid, int n_last, cudaStream_t s);
cudaError_t launch_pad_rows(const double* x, long long xbs, double* y, long long ybs, int n1,
                            int n1p, long long rows, long long batch, cudaStream_t s);
}  // namespace fdp
// Workspace slack (doubles): K1t's non-KMAJ tensor maps read up to 15 elements past the end of a
// tensor in the last (partial) p-group (computed, never stored); every workspace size adds this.
constexpr long long kWsSlack = 32;
// Even-odd folding helpers (abi.cpp). fold_nt: the small-kernel NT of a folded extent n.
bool persymmetric(int n, const double* A, double rtol);
inline int fold_nt(int n) { return 2 * (((n + 1) / 2 + 7) / 8); }
// Centrosymmetric A (n x n, column-major): folded single-pass matrix (FOLD_SYM) in the global
// layout of the folded kernels: rows [0, foldh) = E block, [foldh, 2 foldh) = O block, ldw cols.
void fold_sym_matrix(int n, const double* A, int foldh, int ldw, std::vector<double>* w);
using StageHook = std::function<void(int pass, bool fwd, int d, std::vector<ModeProb>&,
                                     std::vector<TileCfg>&)>;
cudaError_t launch_stage(std::vector<ModeProb>& probs_in, const std::vector<TileCfg>& cfgs_in,
                         bool kmaj, cudaStream_t s, int* nlaunch, Recorder* rec);
// Dense P_Q riding in the plane path (D = 3, every M_d^{-1} folded): mode 1 (FOLD_SYM, plane-major
// output into Tq) joins the velocity mode-1 forward launch, modes 2 and 3 are planes of kind 1
// in the plane launch, which stores s_p (optionally scaled) at out.
struct PresPlane {
  const int* n;                   // pressure extents n[0..2]
  const double* rq;
  long long rbs;
  double* Tq;
  long long tqbs;
  double* out;
  long long obs;
  const double* scale;
  double* const* Wq;
  const int* q_ldw;
  const int* q_foldh;
  const int* q_fold;
  const double* pre;              // D_Q^{-1/2} fused into the mode-1 pass (when the block's
                                  // pre-scaling launch is skipped), else NULL
};
// True when enqueue_fd will take the plane path for these handles (and pressure).
bool plane_path(const std::vector<const fdp_fd_s*>& hs, const PresPlane* pq, int64_t batch);
cudaError_t enqueue_fd(const std::vector<const fdp_fd_s*>& hs,
                       const std::vector<const double*>& in, long long ibs,
                       const std::vector<double*>& out, long long obs,
                       const std::vector<double*>& T,
                       const std::vector<const double*>& dscale, int64_t batch,
                       cudaStream_t s, int* nlaunch, Recorder* rec = nullptr,
                       const StageHook& hook = nullptr, const PresPlane* pq = nullptr,
                       bool fuse_prescale = false);
cudaError_t enqueue_mass(const fdp_mass_s* h, int mode, const double* in, double* out,
                         long long bs, const double* dscale, int64_t batch, cudaStream_t s,
                         int* nlaunch, Recorder* rec = nullptr);
void kron_diag_accumulate(int D, const int* n, const std::vector<const double*>& f, double c,
                          double* out);
cudaError_t run1(ModeProb p, const TileCfg& c, bool kmaj, cudaStream_t s);
// NCCL loaded at run time (nccl_dl.cpp): the exchanges of the NCCL-communicator sharded applies.
namespace fdp {
struct NcclXfer {
  const double* buf;  // send: source; recv: destination
  long long count;    // doubles (0: skipped)
  int peer;
  bool send;
};
fdp_status nccl_unique_id(void* id);
fdp_status nccl_comm_init(void** comm, int nranks, int rank, const void* id);
void nccl_comm_destroy(void* comm);
// one grouped set of point-to-point transfers (ncclGroupStart .. ncclGroupEnd) on stream s
fdp_status nccl_exchange(void* comm, const std::vector<NcclXfer>& xs, cudaStream_t s, const char* where);
}  // namespace fdp
