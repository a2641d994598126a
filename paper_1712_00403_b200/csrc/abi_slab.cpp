// C ABI: slab decomposition over ranks: the phase functions with the
// NCCL-exchange layout, the peer-store variants, the barrier, CUDA IPC buffers and the communicator.
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
    }
  }
  return p;
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
      FDP_CUDA(run1(slab_prob(h, 0, true, src, T1, 1, n2 * nz, EPI_NONE, nullptr, nullptr, false), slab_cfg(h, 0, true, false), true, s),
               "fd_apply_slab: mode 1");
      FDP_CUDA(run1(slab_prob(h, 1, true, T1, T2, n1, nz, EPI_NONE, nullptr, nullptr, false), slab_cfg(h, 1, true, false), false, s),
               "fd_apply_slab: mode 2");
      FDP_CUDA(launch_slab_copy(T2, out, (int)n1, (int)n2, (int)nz, nranks, 0, nullptr, s), "fd_apply_slab: pack");
    } else if (phase == 1) {
      const double* lam1 = slab_lam(h, 1, false) + y0;
      const bool fuse = std::getenv("FDP_NO_FUSE") == nullptr && std::getenv("FDP_NO_SMALL") == nullptr &&
                        n3 <= kSmallMaxN && h->cfg[2].tiles_n == 1;
      if (fuse) {  // in place: each 8-row tile is read whole before it is written
        FDP_CUDA(run1(slab_prob(h, 2, true, in, out, n1 * ny, 1, EPI_FUSED, nullptr, lam1, false), slab_cfg(h, 2, true, false), false, s),
                 "fd_apply_slab: fused mode 3");
      } else {
        FDP_CUDA(run1(slab_prob(h, 2, true, in, T1, n1 * ny, 1, EPI_LAMBDA, nullptr, lam1, false), slab_cfg(h, 2, true, false), false, s),
                 "fd_apply_slab: mode 3 fwd");
        FDP_CUDA(run1(slab_prob(h, 2, false, T1, out, n1 * ny, 1, EPI_NONE, nullptr, nullptr, false), slab_cfg(h, 2, false, false), false, s),
                 "fd_apply_slab: mode 3 bwd");
      }
    } else {
      FDP_CUDA(launch_slab_copy(in, T1, (int)n1, (int)n2, (int)nz, nranks, 1, nullptr, s), "fd_apply_slab: unpack");
      FDP_CUDA(run1(slab_prob(h, 1, false, T1, T2, n1, nz, EPI_NONE, nullptr, nullptr, false), slab_cfg(h, 1, false, false), false, s),
               "fd_apply_slab: mode 2 bwd");
      FDP_CUDA(run1(slab_prob(h, 0, false, T2, out, 1, n2 * nz, dscale ? EPI_SCALE : EPI_NONE, dscale, nullptr, false),
                    slab_cfg(h, 0, false, false), true, s),
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
      FDP_CUDA(run1(slab_prob(h, 0, true, src, T1, 1, n2 * nz, EPI_NONE, nullptr, nullptr, true), slab_cfg(h, 0, true, true), true, s),
               "fd_apply_slab_peer: mode 1");
      ModeProb p = slab_prob(h, 1, true, T1, nullptr, n1, nz, EPI_NONE, nullptr, nullptr, true);
      set_scatter(p, peers, nranks, (int)n2, (int)n1, (int)z0, 1, 0, 0, 1);
      FDP_CUDA(run1(p, slab_cfg(h, 1, true, true), false, s), "fd_apply_slab_peer: mode 2 + exchange");
    } else if (phase == 1) {
      // the mode-3 triple on the y-slab; the last contraction stores element (i1, i2, i3) straight
      // into the z-slab buffer (n1, n2, nz_g) of the rank g owning i3, at (i1, y0 + i2, i3 - z0_g)
      const double* lam1 = slab_lam(h, 1, true) + y0;
      const bool fuse = std::getenv("FDP_NO_FUSE") == nullptr && std::getenv("FDP_NO_SMALL") == nullptr &&
                        n3 <= kSmallMaxN && h->cfg[2].tiles_n == 1;
      if (fuse) {
        ModeProb p = slab_prob(h, 2, true, in, nullptr, n1 * ny, 1, EPI_FUSED, nullptr, lam1, true);
        set_scatter(p, peers, nranks, (int)n3, (int)n1, (int)y0, (int)n2, 0, 1, 0);
        FDP_CUDA(run1(p, slab_cfg(h, 2, true, true), false, s), "fd_apply_slab_peer: fused mode 3 + exchange");
      } else {
        FDP_CUDA(run1(slab_prob(h, 2, true, in, T1, n1 * ny, 1, EPI_LAMBDA, nullptr, lam1, true), slab_cfg(h, 2, true, true), false, s),
                 "fd_apply_slab_peer: mode 3 fwd");
        ModeProb p = slab_prob(h, 2, false, T1, nullptr, n1 * ny, 1, EPI_NONE, nullptr, nullptr, true);
        set_scatter(p, peers, nranks, (int)n3, (int)n1, (int)y0, (int)n2, 0, 1, 0);
        FDP_CUDA(run1(p, slab_cfg(h, 2, false, true), false, s), "fd_apply_slab_peer: mode 3 bwd + exchange");
      }
    } else {
      FDP_CUDA(run1(slab_prob(h, 1, false, in, T2, n1, nz, EPI_NONE, nullptr, nullptr, true), slab_cfg(h, 1, false, true), false, s),
               "fd_apply_slab_peer: mode 2 bwd");
      FDP_CUDA(run1(slab_prob(h, 0, false, T2, out, 1, n2 * nz, dscale ? EPI_SCALE : EPI_NONE, dscale, nullptr, true),
                    slab_cfg(h, 0, false, true), true, s),
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
