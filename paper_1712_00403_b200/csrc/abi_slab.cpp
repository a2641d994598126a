// C ABI: slab decomposition over ranks: the phase functions with the
// NCCL-exchange layout, the peer-store variants, the barrier, CUDA IPC buffers and the communicator.
#include <functional>

#include "abi_impl.h"

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

// Even-odd folding in the slab phases: a mode is folded in every pass of a
// slab apply or in none (its spectral order must agree between the forward pass, the eigenvalue
// vector and the backward pass). The peer-store variant scatters from the folded K1 kernels
// (n > 96) but not from the small-path ones, so there modes 2 and 3 fold only on the K1 path.
static bool slab_fold(const fdp_fd_s* h, int d, bool peer) {
  return h->fold[d] == 2 || (h->fold[d] == 1 && (!peer || d == 0));
}
static const double* slab_lam(const fdp_fd_s* h, int d, bool peer) {
  return slab_fold(h, d, peer) ? h->lamcF[d] : h->lamc[d];
}
static TileCfg slab_cfg(const fdp_fd_s* h, int d, bool fwd, bool peer) {
  TileCfg c = h->cfg[d];
  if (slab_fold(h, d, peer)) {
    if (h->fold[d] == 1) c.NT = h->fold_nt[d];
    else c = fwd ? h->cfgFf[d] : h->cfgFb[d];
  }
  return c;
}

// Mode contraction of a (P, n, Q) view with the handle's direction-d matrices (batch 1).
static ModeProb slab_prob(const fdp_fd_s* h, int d, bool fwd, const double* X, double* Y,
                          long long P, long long Q, int epi, const double* scale,
                          const double* lam1, bool peer = false) {
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
    p.lam0 = slab_lam(h, 0, peer);
    p.lam1 = lam1;
    p.lamcol = slab_lam(h, 2, peer);
  }
  const int BM = kK1Warps * 8 * h->cfg[d].MT;
  p.tiles_m = (int)((P * Q + BM - 1) / BM);
  p.tiles_n = h->cfg[d].tiles_n;
  p.fd_work = 1;
  if (slab_fold(h, d, peer)) {
    p.fold = epi == EPI_FUSED ? FOLD_FUSED : (fwd ? FOLD_FWD : FOLD_BWD);
    p.W = fwd ? h->WfF[d] : h->WbF[d];
    p.ldw = fwd ? h->ldwF[d] : h->ldwFb[d];
    p.foldh = h->foldh[d];
    if (h->fold[d] == 2) {
      p.fold_k1 = 1;
      p.tiles_n = fwd ? h->cfgFf[d].tiles_n : h->cfgFb[d].tiles_n;
      p.tiles_ne = h->tiles_ne[d];
      p.Wt = fwd ? h->WtF[d] : h->WtB[d];  // K1t where a tensor map can read the operand
    }
  }
  return p;
}


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

// ---- the phases as step lists ----
// A slab phase of one block is a short list of steps: mode contractions (K1 family) and streaming
// auxiliary launches (scalings, pack / unpack, banded mass solves, scatter copies). The single-block
// entry points run their list step by step; the sharded block apply runs the lists of all blocks
// side by side, so step i of every velocity block is ONE grouped launch (launch_stage), the
// auxiliary steps one launch each. A block's own steps keep their order; blocks are independent.
namespace {

struct SlabOp {
  bool k1 = false;
  ModeProb p{};
  TileCfg c{};
  bool kmaj = false;
  std::function<cudaError_t(cudaStream_t)> aux;
  const char* what = "";
};
using SlabOps = std::vector<SlabOp>;

SlabOp k1_op(const ModeProb& p, const TileCfg& c, bool kmaj, const char* what) {
  SlabOp o;
  o.k1 = true;
  o.p = p;
  o.c = c;
  o.kmaj = kmaj;
  o.what = what;
  return o;
}
SlabOp aux_op(std::function<cudaError_t(cudaStream_t)> f, const char* what) {
  SlabOp o;
  o.aux = std::move(f);
  o.what = what;
  return o;
}

fdp_status run_ops(const std::vector<SlabOps>& blocks, cudaStream_t s) {
  size_t steps = 0;
  for (const SlabOps& b : blocks) steps = std::max(steps, b.size());
  for (size_t i = 0; i < steps; ++i) {
    for (int km = 0; km < 2; ++km) {
      std::vector<ModeProb> probs;
      std::vector<TileCfg> cfgs;
      const char* what = "";
      for (const SlabOps& b : blocks)
        if (i < b.size() && b[i].k1 && b[i].kmaj == (km == 1)) {
          probs.push_back(b[i].p);
          cfgs.push_back(b[i].c);
          what = b[i].what;
        }
      if (!probs.empty()) FDP_CUDA(launch_stage(probs, cfgs, km == 1, s, nullptr, nullptr), what);
    }
    for (const SlabOps& b : blocks)
      if (i < b.size() && !b[i].k1) FDP_CUDA(b[i].aux(s), b[i].what);
  }
  return FDP_OK;
}

// Steps of phase `phase` of velocity block h on rank g of G. peer: the peer-store variant (the
// exchange fused into the last contraction of phases 0 and 1, `peers` = the owners' buffers);
// otherwise the NCCL layout (phase 0 packs into `out`, phase 2 unpacks from `in`). T1, T2: this
// block's workspace halves (n1 n2 nz doubles each, T1 also >= the y-slab).
SlabOps fd_slab_ops(const fdp_fd_s* h, int phase, int G, int g, const double* in, double* out,
                    double* const* peers, const double* dscale, double* T1, double* T2, bool peer) {
  const long long n1 = h->n[0], n2 = h->n[1], n3 = h->n[2];
  long long z0, nz, y0, ny;
  part_range(n3, G, g, &z0, &nz);
  part_range(n2, G, g, &y0, &ny);
  SlabOps ops;
  if ((phase == 1 ? ny : nz) == 0) return ops;  // this rank owns nothing of that axis
  if (phase == 0) {
    const double* src = in;
    if (dscale) {  // x <- D^{-1/2} x on the z-slab
      ops.push_back(aux_op([=](cudaStream_t s) { return launch_scale(in, T2, dscale, n1 * n2 * nz, 1, 0, 0, s); },
                           "slab phase 0: prescale"));
      src = T2;
    }
    ops.push_back(k1_op(slab_prob(h, 0, true, src, T1, 1, n2 * nz, EPI_NONE, nullptr, nullptr, peer),
                        slab_cfg(h, 0, true, peer), true, "slab phase 0: mode 1"));
    if (peer) {
      // mode 2 stores element (i1, i2, i3) straight into the y-slab buffer (n1, ny_h, n3) of the
      // rank h owning i2, at (i1, i2 - y0_h, z0 + i3)
      ModeProb p = slab_prob(h, 1, true, T1, nullptr, n1, nz, EPI_NONE, nullptr, nullptr, true);
      set_scatter(p, peers, G, (int)n2, (int)n1, (int)z0, 1, 0, 0, 1);
      ops.push_back(k1_op(p, slab_cfg(h, 1, true, true), false, "slab phase 0: mode 2 + exchange"));
    } else {
      ops.push_back(k1_op(slab_prob(h, 1, true, T1, T2, n1, nz, EPI_NONE, nullptr, nullptr, false),
                          slab_cfg(h, 1, true, false), false, "slab phase 0: mode 2"));
      ops.push_back(aux_op([=](cudaStream_t s) { return launch_slab_copy(T2, out, (int)n1, (int)n2, (int)nz, G, 0, nullptr, s); },
                           "slab phase 0: pack"));
    }
  } else if (phase == 1) {
    // the mode-3 triple on the y-slab (in place for the NCCL layout); the peer variant's last
    // contraction stores (i1, i2, i3) into the z-slab buffer (n1, n2, nz_g) of the rank g owning
    // i3, at (i1, y0 + i2, i3 - z0_g)
    const double* lam1 = slab_lam(h, 1, peer) + y0;
    const bool fuse = std::getenv("FDP_NO_FUSE") == nullptr && std::getenv("FDP_NO_SMALL") == nullptr &&
                      n3 <= kSmallMaxN && h->cfg[2].tiles_n == 1;
    auto scatter = [&](ModeProb& p) { set_scatter(p, peers, G, (int)n3, (int)n1, (int)y0, (int)n2, 0, 1, 0); };
    if (fuse) {  // in place: each 8-row tile is read whole before it is written
      ModeProb p = slab_prob(h, 2, true, in, peer ? nullptr : out, n1 * ny, 1, EPI_FUSED, nullptr, lam1, peer);
      if (peer) scatter(p);
      ops.push_back(k1_op(p, slab_cfg(h, 2, true, peer), false, "slab phase 1: fused mode 3"));
    } else {
      ops.push_back(k1_op(slab_prob(h, 2, true, in, T1, n1 * ny, 1, EPI_LAMBDA, nullptr, lam1, peer),
                          slab_cfg(h, 2, true, peer), false, "slab phase 1: mode 3 fwd"));
      ModeProb p = slab_prob(h, 2, false, T1, peer ? nullptr : out, n1 * ny, 1, EPI_NONE, nullptr, nullptr, peer);
      if (peer) scatter(p);
      ops.push_back(k1_op(p, slab_cfg(h, 2, false, peer), false, "slab phase 1: mode 3 bwd"));
    }
  } else {
    const double* src = in;
    if (!peer) {
      ops.push_back(aux_op([=](cudaStream_t s) { return launch_slab_copy(in, T1, (int)n1, (int)n2, (int)nz, G, 1, nullptr, s); },
                           "slab phase 2: unpack"));
      src = T1;
    }
    ops.push_back(k1_op(slab_prob(h, 1, false, src, T2, n1, nz, EPI_NONE, nullptr, nullptr, peer),
                        slab_cfg(h, 1, false, peer), false, "slab phase 2: mode 2 bwd"));
    ops.push_back(k1_op(slab_prob(h, 0, false, T2, out, 1, n2 * nz, dscale ? EPI_SCALE : EPI_NONE, dscale, nullptr, peer),
                        slab_cfg(h, 0, false, peer), true, "slab phase 2: mode 1 bwd"));
  }
  return ops;
}

// Steps of phase `phase` of the pressure block (banded solves K3); T: n1 max(n2 nz,
// ny n3) doubles.
SlabOps mass_slab_ops(const fdp_mass_s* h, int phase, int G, int g, const double* in, double* out,
                      double* const* peers, const double* dscale, double* T, bool peer) {
  const long long n1 = h->n[0], n2 = h->n[1], n3 = h->n[2];
  long long z0, nz, y0, ny;
  part_range(n3, G, g, &z0, &nz);
  part_range(n2, G, g, &y0, &ny);
  SlabOps ops;
  if ((phase == 1 ? ny : nz) == 0) return ops;
  auto mode = [=](int d, const double* src, double* dst, long long P, long long Q, const double* pre) {
    MassMode m{};
    m.in = src;
    m.out = dst;
    m.Lb = h->Lb[d];
    m.invd = h->invd[d];
    m.Mb = h->Mb[d];
    m.cf = h->cf[d];
    m.cb = h->cb[d];
    m.pre = pre;
    m.N = P * h->n[d] * Q;
    m.bs = 0;
    m.P = (int)P;
    m.n = h->n[d];
    m.Q = (int)Q;
    m.batch = 1;
    m.band = h->band[d];
    return [m](cudaStream_t s) { return launch_mass_mode(m, s); };
  };
  if (phase == 0) {
    ops.push_back(aux_op(mode(0, in, T, 1, n2 * nz, dscale), "pressure slab phase 0: mode 1"));
    ops.push_back(aux_op(mode(1, T, T, n1, nz, nullptr), "pressure slab phase 0: mode 2"));
    if (peer) {
      const ScatterDesc sd{peers, G, (int)n2, (int)n1, (int)z0, 1, 0, 0, 1};
      ops.push_back(aux_op([=](cudaStream_t s) { return launch_slab_scatter(T, sd, (int)nz, 0, s); },
                           "pressure slab phase 0: exchange"));
    } else {
      ops.push_back(aux_op([=](cudaStream_t s) { return launch_slab_copy(T, out, (int)n1, (int)n2, (int)nz, G, 0, nullptr, s); },
                           "pressure slab phase 0: pack"));
    }
  } else if (phase == 1) {
    if (peer) {
      ops.push_back(aux_op(mode(2, in, T, n1 * ny, 1, nullptr), "pressure slab phase 1: mode 3"));
      const ScatterDesc sd{peers, G, (int)n3, (int)n1, (int)y0, (int)n2, 0, 1, 0};
      ops.push_back(aux_op([=](cudaStream_t s) { return launch_slab_scatter(T, sd, (int)ny, 1, s); },
                           "pressure slab phase 1: exchange"));
    } else {
      ops.push_back(aux_op(mode(2, in, out, n1 * ny, 1, nullptr), "pressure slab phase 1: mode 3"));
    }
  } else if (peer) {
    if (dscale)
      ops.push_back(aux_op([=](cudaStream_t s) { return launch_scale(in, out, dscale, n1 * n2 * nz, 1, 0, 0, s); },
                           "pressure slab phase 2: postscale"));
    else if (in != out)
      ops.push_back(aux_op([=](cudaStream_t s) {
        return cudaMemcpyAsync(out, in, (size_t)(n1 * n2 * nz) * sizeof(double), cudaMemcpyDeviceToDevice, s);
      }, "pressure slab phase 2: copy"));
  } else {
    ops.push_back(aux_op([=](cudaStream_t s) { return launch_slab_copy(in, out, (int)n1, (int)n2, (int)nz, G, 1, dscale, s); },
                         "pressure slab phase 2: unpack"));
  }
  return ops;
}

// argument checks shared by the single-block phase entry points
fdp_status check_phase(const char* fn, int D, int phase, int nranks, int rank, int maxranks) {
  if (D != 3) return fail(FDP_ERR_UNSUPPORTED, std::string(fn) + ": D must be 3");
  if (nranks < 1 || nranks > maxranks || rank < 0 || rank >= nranks || phase < 0 || phase > 2)
    return fail(FDP_ERR_INVALID_ARG, std::string(fn) + ": bad phase / rank");
  return FDP_OK;
}

}  // namespace

extern "C" fdp_status fd_apply_slab(fdp_fd h, int phase, int nranks, int rank, const double* in,
                                    double* out, const double* dscale, void* workspace,
                                    void* stream) {
  try {
    if (!h) return fail(FDP_ERR_INVALID_ARG, "fd_apply_slab: NULL handle");
    if (fdp_status st = check_phase("fd_apply_slab", h->D, phase, nranks, rank, 1 << 20)) return st;
    const long long n1 = h->n[0], n2 = h->n[1];
    long long z0, nz, y0, ny;
    part_range(h->n[2], nranks, rank, &z0, &nz);
    part_range(n2, nranks, rank, &y0, &ny);
    if ((phase == 1 ? ny : nz) == 0) return FDP_OK;  // this rank owns nothing of that axis
    if (!is_device_ptr(in) || !is_device_ptr(out) || !is_device_ptr(workspace) ||
        (dscale && !is_device_ptr(dscale)))
      return fail(FDP_ERR_INVALID_ARG, "fd_apply_slab: device pointers required");
    DeviceGuard dg(h->device);
    double* T1 = static_cast<double*>(workspace);
    return run_ops({fd_slab_ops(h, phase, nranks, rank, in, out, nullptr, dscale, T1, T1 + n1 * n2 * nz, false)},
                   static_cast<cudaStream_t>(stream));
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fd_apply_slab_peer(fdp_fd h, int phase, int nranks, int rank, const double* in,
                                         double* out, double* const* peers, const double* dscale,
                                         void* workspace, void* stream) {
  try {
    if (!h) return fail(FDP_ERR_INVALID_ARG, "fd_apply_slab_peer: NULL handle");
    if (fdp_status st = check_phase("fd_apply_slab_peer", h->D, phase, nranks, rank, 32)) return st;
    const long long n1 = h->n[0], n2 = h->n[1];
    long long z0, nz, y0, ny;
    part_range(h->n[2], nranks, rank, &z0, &nz);
    part_range(n2, nranks, rank, &y0, &ny);
    if ((phase == 1 ? ny : nz) == 0) return FDP_OK;
    if (!is_device_ptr(in) || !is_device_ptr(workspace) || (phase == 2 && !is_device_ptr(out)) ||
        (phase < 2 && !is_device_ptr(peers)) || (dscale && !is_device_ptr(dscale)))
      return fail(FDP_ERR_INVALID_ARG, "fd_apply_slab_peer: device pointers required");
    DeviceGuard dg(h->device);
    double* T1 = static_cast<double*>(workspace);
    return run_ops({fd_slab_ops(h, phase, nranks, rank, in, out, peers, dscale, T1, T1 + n1 * n2 * nz, true)},
                   static_cast<cudaStream_t>(stream));
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status kron_mass_apply_slab_peer(fdp_mass h, int phase, int nranks, int rank,
                                                const double* in, double* out, double* const* peers,
                                                const double* dscale, void* workspace, void* stream) {
  try {
    if (!h) return fail(FDP_ERR_INVALID_ARG, "kron_mass_apply_slab_peer: NULL handle");
    if (fdp_status st = check_phase("kron_mass_apply_slab_peer", h->D, phase, nranks, rank, 32)) return st;
    long long z0, nz, y0, ny;
    part_range(h->n[2], nranks, rank, &z0, &nz);
    part_range(h->n[1], nranks, rank, &y0, &ny);
    if ((phase == 1 ? ny : nz) == 0) return FDP_OK;
    if (!is_device_ptr(in) || (phase < 2 && (!is_device_ptr(workspace) || !is_device_ptr(peers))) ||
        (phase == 2 && !is_device_ptr(out)) || (dscale && !is_device_ptr(dscale)))
      return fail(FDP_ERR_INVALID_ARG, "kron_mass_apply_slab_peer: device pointers required");
    DeviceGuard dg(h->device);
    return run_ops({mass_slab_ops(h, phase, nranks, rank, in, out, peers, dscale, static_cast<double*>(workspace), true)},
                   static_cast<cudaStream_t>(stream));
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

// ---- C-level communicators for the sharded applies (SURVEY.md §8(b) "multi-GPU") ----
// Two kinds:
//  * NCCL (fdp_comm_init from an ncclUniqueId): the exchanges are grouped ncclSend / ncclRecv
//    all-to-alls of the packed slab pieces (one NCCL group per exchange for all blocks); every
//    buffer lives in the caller's workspace, so one communicator serves any handle.
//  * peer-store (fdp_comm_create / fdp_comm_connect for one block preconditioner): every rank
//    owns, per block, a y-slab receive buffer (exchange 1) and a z-slab return buffer (exchange
//    2), plus an nranks-slot barrier flag array; their CUDA IPC handles form the rank's blob,
//    which the caller all-gathers (torch.distributed is plumbing).
struct fdp_comm_s {
  int nranks = 0, rank = 0, device = 0, nblocks = 0;
  void* nccl = nullptr;               // ncclComm_t of an NCCL communicator
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
  if (c->nccl) nccl_comm_destroy(c->nccl);
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
    if (c->nccl) return fail(FDP_ERR_INVALID_ARG, "fdp_comm_connect: an NCCL communicator needs no connect");
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

// Workspace of the sharded applies: per block b (regions of 32-double multiples) the block's
// phase workspace T_b (fd_slab_workspace_bytes / kron_mass_slab_workspace_bytes), and for an NCCL
// communicator also S_b (z-slab: packed pieces out, returned pieces in) and Y_b (y-slab). Every
// block has its own regions, so the blocks' phases run side by side in grouped launches.
struct ShardLayout {
  std::vector<double*> T, S, Y;
  size_t doubles = 0;
};

static size_t round32(size_t n) { return (n + 31) / 32 * 32; }

static ShardLayout shard_layout(int nb, int nvel, const std::vector<const void*>& hs, const int* const* dims,
                                bool nccl, int G, int g, double* base) {
  ShardLayout L;
  size_t off = 0;
  for (int b = 0; b < nb; ++b) {
    const long long n1 = dims[b][0], n2 = dims[b][1], n3 = dims[b][2];
    long long z0, nz, y0, ny;
    part_range(n3, G, g, &z0, &nz);
    part_range(n2, G, g, &y0, &ny);
    const size_t tb = b < nvel
                          ? fd_slab_workspace_bytes(static_cast<fdp_fd>(const_cast<void*>(hs[b])), G, g)
                          : kron_mass_slab_workspace_bytes(static_cast<fdp_mass>(const_cast<void*>(hs[b])), G, g);
    L.T.push_back(base ? base + off : nullptr);
    off += round32(tb / sizeof(double) + 1);
    if (nccl) {
      L.S.push_back(base ? base + off : nullptr);
      off += round32((size_t)std::max(1LL, n1 * n2 * nz));
      L.Y.push_back(base ? base + off : nullptr);
      off += round32((size_t)std::max(1LL, n1 * ny * n3));
    }
  }
  L.doubles = off;
  return L;
}

// Per-peer element counts of the slab exchanges of one block (host only; also the plan of the
// NCCL exchange below): exchange 1 sends rank h the i2-planes [y0_h, y0_h + ny_h) of my z-slab
// (n1 ny_h nz, packed in rank order) and receives from h its z-planes of my y-range (n1 ny nz_h);
// exchange 2 is the reverse.
extern "C" fdp_status fdp_slab_exchange_counts(const int32_t* dims, int nranks, int rank, int exchange,
                                               int64_t* send_counts, int64_t* recv_counts) {
  try {
    if (!dims || !send_counts || !recv_counts || nranks < 1 || rank < 0 || rank >= nranks ||
        (exchange != 1 && exchange != 2) || dims[0] < 0 || dims[1] < 0 || dims[2] < 0)
      return fail(FDP_ERR_INVALID_ARG, "fdp_slab_exchange_counts: bad arguments");
    const long long n1 = dims[0], n2 = dims[1], n3 = dims[2];
    long long z0, nz, y0, ny;
    part_range(n3, nranks, rank, &z0, &nz);
    part_range(n2, nranks, rank, &y0, &ny);
    for (int h = 0; h < nranks; ++h) {
      long long zh0, nzh, yh0, nyh;
      part_range(n3, nranks, h, &zh0, &nzh);
      part_range(n2, nranks, h, &yh0, &nyh);
      const long long piece = n1 * nyh * nz, slab = n1 * ny * nzh;
      send_counts[h] = exchange == 1 ? piece : slab;
      recv_counts[h] = exchange == 1 ? slab : piece;
    }
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

// The NCCL all-to-all of exchange 1 (S_b pieces -> Y_b) or 2 (Y_b -> S_b pieces) of every block,
// one NCCL group.
static fdp_status nccl_slab_exchange(fdp_comm c, int nb, const int* const* dims, const ShardLayout& L, int ex,
                                     cudaStream_t st) {
  const int G = c->nranks, g = c->rank;
  std::vector<NcclXfer> xs;
  std::vector<int64_t> sc(G), rc(G);
  for (int b = 0; b < nb; ++b) {
    if (fdp_status e = fdp_slab_exchange_counts(dims[b], G, g, ex, sc.data(), rc.data())) return e;
    const double* sbuf = ex == 1 ? L.S[b] : L.Y[b];
    const double* rbuf = ex == 1 ? L.Y[b] : L.S[b];
    long long so = 0, ro = 0;
    for (int h = 0; h < G; ++h) {
      xs.push_back({sbuf + so, sc[h], h, true});
      xs.push_back({rbuf + ro, rc[h], h, false});
      so += sc[h];
      ro += rc[h];
    }
  }
  return nccl_exchange(c->nccl, xs, st, ex == 1 ? "sharded apply: exchange 1" : "sharded apply: exchange 2");
}

extern "C" size_t block_precond_sharded_workspace_bytes(fdp_block P, fdp_comm c) {
  try {
    if (!P || !c || P->D != 3) return 0;
    std::vector<const void*> hs;
    std::vector<const int*> dims;
    for (int k = 0; k < P->D; ++k) {
      hs.push_back(P->vel[k]);
      dims.push_back(P->vel[k]->n);
    }
    hs.push_back(P->pres);
    dims.push_back(P->pres->n);
    return shard_layout(P->D + 1, P->D, hs, dims.data(), c->nccl != nullptr, c->nranks, c->rank, nullptr).doubles *
           sizeof(double);
  } catch (...) {
    return 0;
  }
}

extern "C" fdp_status block_precond_apply_sharded(fdp_block P, fdp_comm c, const double* r, double* s,
                                                  void* workspace, void* stream) {
  try {
    if (!P || !c) return fail(FDP_ERR_INVALID_ARG, "block_precond_apply_sharded: NULL handle");
    if (!c->nccl && !c->connected)
      return fail(FDP_ERR_INVALID_ARG, "block_precond_apply_sharded: comm not connected");
    if (P->D != 3) return fail(FDP_ERR_UNSUPPORTED, "block_precond_apply_sharded: D must be 3");
    if (!c->nccl && c->nblocks != P->D + 1)
      return fail(FDP_ERR_INVALID_ARG, "block_precond_apply_sharded: comm created for another block");
    if (!is_device_ptr(r) || !is_device_ptr(s) || !is_device_ptr(workspace))
      return fail(FDP_ERR_INVALID_ARG, "block_precond_apply_sharded: device pointers required");
    DeviceGuard dg(P->device);
    const int G = c->nranks, g = c->rank, D = P->D, nb = D + 1;
    const bool peer = c->nccl == nullptr;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // local layout [u_1 z-slab | .. | u_D z-slab | p z-slab]; D^{-1/2} slices of the P^G scalings
    std::vector<long long> loff(nb + 1, 0), goff(nb, 0);
    std::vector<const void*> hs;
    std::vector<const int*> dims;
    for (int b = 0; b < nb; ++b) {
      long long n1, n2, n3, z0, nz;
      block_dims(P, b, &n1, &n2, &n3);
      part_range(n3, G, g, &z0, &nz);
      loff[b + 1] = loff[b] + n1 * n2 * nz;
      goff[b] = n1 * n2 * z0;
      hs.push_back(b < D ? static_cast<const void*>(P->vel[b]) : static_cast<const void*>(P->pres));
      dims.push_back(b < D ? P->vel[b]->n : P->pres->n);
    }
    auto dsc = [&](int b) -> const double* {
      if (b < D) return P->dv ? P->dv + P->off[b] + goff[b] : nullptr;
      return P->dq ? P->dq + goff[b] : nullptr;
    };
    const ShardLayout L = shard_layout(nb, D, hs, dims.data(), !peer, G, g, static_cast<double*>(workspace));
    for (int phase = 0; phase < 3; ++phase) {
      // every block's steps of this phase side by side: step i of the velocity blocks is one
      // grouped launch
      std::vector<SlabOps> ops;
      for (int b = 0; b < nb; ++b) {
        const double* in;
        double* out = nullptr;
        double* const* peers = nullptr;
        if (peer) {
          peers = phase == 0 ? c->peers_y + (size_t)b * G : phase == 1 ? c->peers_z + (size_t)b * G : nullptr;
          in = phase == 0 ? r + loff[b] : static_cast<const double*>(c->own[2 * b + (phase == 1 ? 0 : 1)]);
          if (phase == 2) out = s + loff[b];
        } else {
          in = phase == 0 ? r + loff[b] : phase == 1 ? L.Y[b] : L.S[b];
          out = phase == 0 ? L.S[b] : phase == 1 ? L.Y[b] : s + loff[b];
        }
        const double* ds = phase == 1 ? nullptr : dsc(b);
        if (b < D) {
          const fdp_fd_s* h = P->vel[b];
          long long z0, nz;
          part_range(h->n[2], G, g, &z0, &nz);
          ops.push_back(fd_slab_ops(h, phase, G, g, in, out, peers, ds, L.T[b],
                                    L.T[b] + (long long)h->n[0] * h->n[1] * nz, peer));
        } else {
          ops.push_back(mass_slab_ops(P->pres, phase, G, g, in, out, peers, ds, L.T[b], peer));
        }
      }
      if (fdp_status e = run_ops(ops, st)) return e;
      if (peer) {
        // exchanges complete on every rank before the next phase reads (and, after phase 2,
        // before the next apply's phase 0 overwrites y-slabs)
        FDP_CUDA(launch_peer_barrier(c->flag_ptrs, c->counter, G, g, st), "block_precond_apply_sharded: barrier");
      } else if (phase < 2) {
        if (fdp_status e = nccl_slab_exchange(c, nb, dims.data(), L, phase + 1, st)) return e;
      }
    }
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

// ---- NCCL communicator ----
extern "C" fdp_status fdp_nccl_unique_id(void* id) {
  try {
    if (!id) return fail(FDP_ERR_INVALID_ARG, "fdp_nccl_unique_id: NULL id");
    return nccl_unique_id(id);
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_comm_init(int nranks, int rank, const void* nccl_unique_id, int device,
                                    fdp_comm* out) {
  try {
    if (!out || !nccl_unique_id) return fail(FDP_ERR_INVALID_ARG, "fdp_comm_init: NULL argument");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(FDP_ERR_INVALID_ARG, "fdp_comm_init: bad rank");
    int ndev = 0;
    FDP_CUDA(cudaGetDeviceCount(&ndev), "fdp_comm_init");
    if (device < 0 || device >= ndev) return fail(FDP_ERR_INVALID_ARG, "fdp_comm_init: bad device");
    DeviceGuard dg(device);
    std::unique_ptr<fdp_comm_s> c(new (std::nothrow) fdp_comm_s);
    if (!c) return fail(FDP_ERR_OOM, "fdp_comm_init: host allocation");
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    if (fdp_status st = nccl_comm_init(&c->nccl, nranks, rank, nccl_unique_id)) return st;
    *out = c.release();
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" size_t fd_sharded_workspace_bytes(fdp_fd h, fdp_comm c) {
  try {
    if (!h || !c || !c->nccl || h->D != 3) return 0;
    std::vector<const void*> hs{h};
    const int* dims[1] = {h->n};
    return shard_layout(1, 1, hs, dims, true, c->nranks, c->rank, nullptr).doubles * sizeof(double);
  } catch (...) {
    return 0;
  }
}

extern "C" fdp_status fd_apply_sharded(fdp_fd h, fdp_comm c, const double* b, double* x,
                                       const double* dscale, void* workspace, void* stream) {
  try {
    if (!h || !c) return fail(FDP_ERR_INVALID_ARG, "fd_apply_sharded: NULL handle");
    if (!c->nccl) return fail(FDP_ERR_UNSUPPORTED, "fd_apply_sharded: needs an NCCL communicator (fdp_comm_init)");
    if (h->D != 3) return fail(FDP_ERR_UNSUPPORTED, "fd_apply_sharded: D must be 3");
    if (!is_device_ptr(b) || !is_device_ptr(x) || !is_device_ptr(workspace) || (dscale && !is_device_ptr(dscale)))
      return fail(FDP_ERR_INVALID_ARG, "fd_apply_sharded: device pointers required");
    DeviceGuard dg(h->device);
    const int G = c->nranks, g = c->rank;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::vector<const void*> hs{h};
    const int* dims[1] = {h->n};
    const ShardLayout L = shard_layout(1, 1, hs, dims, true, G, g, static_cast<double*>(workspace));
    long long z0, nz;
    part_range(h->n[2], G, g, &z0, &nz);
    double* T2 = L.T[0] + (long long)h->n[0] * h->n[1] * nz;
    if (fdp_status e = run_ops({fd_slab_ops(h, 0, G, g, b, L.S[0], nullptr, dscale, L.T[0], T2, false)}, st)) return e;
    if (fdp_status e = nccl_slab_exchange(c, 1, dims, L, 1, st)) return e;
    if (fdp_status e = run_ops({fd_slab_ops(h, 1, G, g, L.Y[0], L.Y[0], nullptr, nullptr, L.T[0], T2, false)}, st)) return e;
    if (fdp_status e = nccl_slab_exchange(c, 1, dims, L, 2, st)) return e;
    return run_ops({fd_slab_ops(h, 2, G, g, L.S[0], x, nullptr, dscale, L.T[0], T2, false)}, st);
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
    long long y0, ny;
    part_range(h->n[1], nranks, rank, &y0, &ny);
    // phase 0 stages the z-slab (n1 n2 nz), phase 1 the y-slab (n1 ny n3): the larger of the two
    return (size_t)std::max((long long)h->n[0] * h->n[1] * nz, (long long)h->n[0] * ny * h->n[2]) *
           sizeof(double);
  } catch (...) {
    return 0;
  }
}

extern "C" fdp_status kron_mass_apply_slab(fdp_mass h, int phase, int nranks, int rank,
                                           const double* in, double* out, const double* dscale,
                                           void* workspace, void* stream) {
  try {
    if (!h) return fail(FDP_ERR_INVALID_ARG, "kron_mass_apply_slab: NULL handle");
    if (fdp_status st = check_phase("kron_mass_apply_slab", h->D, phase, nranks, rank, 1 << 20)) return st;
    long long z0, nz, y0, ny;
    part_range(h->n[2], nranks, rank, &z0, &nz);
    part_range(h->n[1], nranks, rank, &y0, &ny);
    if ((phase == 1 ? ny : nz) == 0) return FDP_OK;
    if (!is_device_ptr(in) || !is_device_ptr(out) || (phase == 0 && !is_device_ptr(workspace)) ||
        (dscale && !is_device_ptr(dscale)))
      return fail(FDP_ERR_INVALID_ARG, "kron_mass_apply_slab: device pointers required");
    DeviceGuard dg(h->device);
    return run_ops({mass_slab_ops(h, phase, nranks, rank, in, out, nullptr, dscale, static_cast<double*>(workspace), false)},
                   static_cast<cudaStream_t>(stream));
  } catch (...) {
    return abi_exception(__func__);
  }
}
