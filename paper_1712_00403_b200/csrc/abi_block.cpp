// C ABI: the block preconditioner P_D / P_D^G: setup, the
// graph-cached device apply, per-launch profiling and the pipelined host-buffer path.
#include "abi_impl.h"

// ------------------------------------------------------------------------------------------------
// block preconditioner
// ------------------------------------------------------------------------------------------------

static void free_block(fdp_block h) {
  if (!h) return;
  for (cudaEvent_t e : h->ev) cudaEventDestroy(e);
  for (auto& g : h->graphs) cudaGraphExecDestroy(g.exec);
  if (h->cap) cudaStreamDestroy(h->cap);
  if (h->side) cudaStreamDestroy(h->side);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
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
        // the velocity launch of stage d is folded: a centrosymmetric M_d^{-1} joins it as a
        // FOLD_SYM pass (about half the DMMAs); otherwise its own dense launch
        bool vfold = true;
        for (int k = 0; k < D; ++k)
          vfold = vfold && raw->vel[k]->fold[d] == 1 && raw->vel[k]->fold_nt[d] == raw->vel[0]->fold_nt[d];
        std::vector<double> w;
        if (vfold && nq >= 8 && fold_nt(nq) <= raw->vel[0]->fold_nt[d] && persymmetric(nq, X.data(), 1e-10)) {
          const int nt = raw->vel[0]->fold_nt[d];
          raw->q_fold[d] = 1;
          raw->q_foldh[d] = 4 * nt;
          raw->q_ldw[d] = 4 * nt;
          raw->q_tiles_n[d] = 1;
          fold_sym_matrix(nq, X.data(), 4 * nt, 4 * nt, &w);
        } else if (nq > kSmallMaxN && std::getenv("FDP_NO_FOLD") == nullptr &&
                   persymmetric(nq, X.data(), 1e-10)) {
          // a K1-sized factor: the folded K1 kernel's FOLD_SYM pass (own launch, two
          // accumulator sets, column tiles of <= 6 n8-tiles over the ceil(n/2) outputs)
          const int ne = (nq + 1) / 2, n8e = (ne + 7) / 8;
          TileCfg c{};
          c.MT = 2;
          c.NT = (n8e + (n8e + 5) / 6 - 1) / ((n8e + 5) / 6);
          c.tiles_n = (n8e + c.NT - 1) / c.NT;
          c.ldw = c.tiles_n * 8 * c.NT;
          c.kpad = kpad;
          const int foldh = ((ne + 31) / 32) * 32;
          raw->q_fold[d] = 2;
          raw->q_foldh[d] = foldh;
          raw->q_ldw[d] = c.ldw;
          raw->q_tiles_n[d] = c.tiles_n;
          raw->q_cfgF[d] = c;
          fold_sym_matrix(nq, X.data(), foldh, c.ldw, &w);
          if (cudaError_t e = prepare_mode_kernels(c); e != cudaSuccess)
            st = cuda_fail(e, "block_precond_setup: prepare");
        } else {
          w.assign((size_t)kpad * raw->q_ldw[d], 0.0);
          for (int k = 0; k < nq; ++k)
            for (int a = 0; a < nq; ++a) w[(size_t)k * raw->q_ldw[d] + a] = X[a + (size_t)nq * k];
        }
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
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&raw->side, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&raw->ev_fork, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&raw->ev_join, cudaEventDisableTiming);
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
  return batch * (v + (h->pres_dense ? 2 * h->pres->N : 0)) + kWsSlack;
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
  // plane path with P^G: the D^{-1/2} pre-scaling rides in the mode-1 pass's loads
  PresPlane pq{};
  const bool pplane = h->pres_dense && (D == 3 || D == 2);
  if (pplane) {
    pq.n = h->pres->n;
    pq.Tq = Tq1;
    pq.tqbs = nq;
    pq.out = s + h->off[D];
    pq.obs = sz;
    pq.scale = h->dall ? h->dall + h->off[D] : nullptr;
    pq.Wq = h->Wq;
    pq.q_ldw = h->q_ldw;
    pq.q_foldh = h->q_foldh;
    pq.q_fold = h->q_fold;
  }
  const bool fuse_pre = pplane && h->dall && plane_path(h->vel, &pq, batch);
  if (fuse_pre) pq.pre = h->dall + h->off[D];
  if (h->pres_dense && h->dall && !fuse_pre) {
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
  } else if (h->dv && !fuse_pre) {
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
      TileCfg qc = h->vel[0]->cfg[d];
      if (h->q_fold[d]) {
        p.fold = FOLD_SYM;
        p.foldh = h->q_foldh[d];
        if (h->q_fold[d] == 2) {
          p.fold_k1 = 1;
          qc = h->q_cfgF[d];
        } else {
          qc.NT = h->vel[0]->fold_nt[d];
        }
      }
      probs.push_back(p);
      cfgs.push_back(qc);
      (void)pass;
    };
  }
  if (pplane) {
    pq.rq = rq;
    pq.rbs = sz;
  }
  // pressure block by banded per-mode solves: r_p -> s_p. Inside a stream capture
  // (every apply but the profiled one) it goes first and on a forked branch, so that the graph
  // may run it next to the velocity path's launches; the profiled apply keeps one stream, where
  // per-launch events mean what they say.
  cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
  static const bool nofork = std::getenv("FDP_NO_FORK") != nullptr;
  const bool fork = !h->pres_dense && !rec && !nofork && h->side &&
                    cudaStreamIsCapturing(st, &cst) == cudaSuccess && cst == cudaStreamCaptureStatusActive;
  cudaError_t e;
  if (fork) {
    if ((e = cudaEventRecord(h->ev_fork, st)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(h->side, h->ev_fork, 0)) != cudaSuccess) return e;
    e = enqueue_mass(h->pres, FDP_MASS_INVERSE, r + h->off[D], s + h->off[D], sz, h->dq, batch, h->side,
                     nlaunch, nullptr);
    if (e != cudaSuccess) return e;
    if ((e = cudaEventRecord(h->ev_join, h->side)) != cudaSuccess) return e;
  }
  e = enqueue_fd(h->vel, in, sz, out, sz, T, dsc, batch, st, nlaunch, rec, hook,
                 pplane ? &pq : nullptr, fuse_pre);
  if (e != cudaSuccess) return e;
  if (fork) {
    if ((e = cudaStreamWaitEvent(st, h->ev_join, 0)) != cudaSuccess) return e;
  } else if (!h->pres_dense) {
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
    {  // exact: the kernel nodes of a captured apply of this batch size
      std::lock_guard<std::mutex> lk(h->mu);
      for (const auto& lc : h->launch_counts)
        if (lc.first == batch && lc.second > 0) return lc.second;
    }
    // no apply of this batch captured yet: the static estimate of the pass structure
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
      int kernels = 0;  // the launches one apply makes, counted from the captured graph
      {
        size_t nn = 0;
        if (cudaGraphGetNodes(g, nullptr, &nn) == cudaSuccess && nn > 0) {
          std::vector<cudaGraphNode_t> nodes(nn);
          if (cudaGraphGetNodes(g, nodes.data(), &nn) == cudaSuccess)
            for (size_t i = 0; i < nn; ++i) {
              cudaGraphNodeType t;
              if (cudaGraphNodeGetType(nodes[i], &t) == cudaSuccess && t == cudaGraphNodeTypeKernel)
                ++kernels;
            }
        }
      }
      cudaGraphExec_t ex = nullptr;
      e = cudaGraphInstantiate(&ex, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) return cuda_fail(e, "block_precond_apply: instantiate");
      h->graphs.push_back({r, s, workspace, batch, ex, 0, kernels});
      bool known = false;
      for (auto& lc : h->launch_counts)
        if (lc.first == batch) { lc.second = kernels; known = true; }
      if (!known) h->launch_counts.push_back({batch, kernels});
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
      TileCfg qc = h->vel[0]->cfg[d];
      if (h->q_fold[d]) {
        p.fold = FOLD_SYM;
        p.foldh = h->q_foldh[d];
        if (h->q_fold[d] == 2) {
          p.fold_k1 = 1;
          qc = h->q_cfgF[d];
        } else {
          qc.NT = h->vel[0]->fold_nt[d];
        }
      }
      std::vector<ModeProb> probs{p};
      std::vector<TileCfg> cfgs{qc};
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
