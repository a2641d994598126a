// C ABI: matrix-free sums of Kronecker products (Stokes operator blocks, NEXT-1) and the
// block-triangular / constrained preconditioners (NEXT-2).
#include "abi_impl.h"

// ------------------------------------------------------------------------------------------------
// matrix-free sums of Kronecker products (NEXT-1 Stokes operator blocks)
// ------------------------------------------------------------------------------------------------

static void free_kron(fdp_kron h) {
  if (!h) return;
  for (auto& k : h->f) {
    cudaFree(k.W);
    cudaFree(k.lo);
    cudaFree(k.Wb);
  }
  delete h;
}

// Banded copy of a factor (column-major nout x nin): per output row the contiguous range that
// holds its nonzeros, widened to the widest row (bw) and shifted to stay inside [0, nin). Used
// for large extents (the dense contraction's 2 n_in flops per output exceed the band's by n/bw);
// FDP_KRON_BAND=0 / 1 disables / forces it.
static fdp_status kron_band_setup(KronFactor& kf, const double* F) {
  const char* env = std::getenv("FDP_KRON_BAND");
  if (env && env[0] == '0') return FDP_OK;
  const int nin = kf.nin, nout = kf.nout;
  std::vector<int> lo(nout, 0);
  int bw = 0;
  for (int a = 0; a < nout; ++a) {
    int l = -1, h = -1;
    for (int k = 0; k < nin; ++k)
      if (F[a + (size_t)nout * k] != 0.0) {
        if (l < 0) l = k;
        h = k;
      }
    lo[a] = l < 0 ? 0 : l;
    bw = std::max(bw, l < 0 ? 1 : h - l + 1);
  }
  const bool force = env && env[0] == '1';
  if (!(bw <= 32 && (force || (nin >= 128 && 4 * bw <= nin)))) return FDP_OK;
  std::vector<double> wb((size_t)nout * bw, 0.0);
  for (int a = 0; a < nout; ++a) {
    lo[a] = std::min(lo[a], nin - bw);
    for (int j = 0; j < bw; ++j) wb[(size_t)a * bw + j] = F[a + (size_t)nout * (lo[a] + j)];
  }
  fdp_status st;
  if ((st = dalloc(&kf.Wb, wb.size()))) return st;
  int* dlo = nullptr;
  if (cudaMalloc(&dlo, (size_t)nout * sizeof(int)) != cudaSuccess) return fail(FDP_ERR_OOM, "kron_op_setup: band");
  kf.lo = dlo;
  cudaError_t e = cudaMemcpy(kf.Wb, wb.data(), wb.size() * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(kf.lo, lo.data(), lo.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "kron_op_setup: band upload");
  kf.bw = bw;
  return FDP_OK;
}

// Launch the banded problems of a stage, grouped kBandMax per launch.
static cudaError_t launch_band_probs(std::vector<BandProb>& bp, cudaStream_t s) {
  for (size_t i = 0; i < bp.size(); i += kBandMax) {
    BandGroup g{};
    g.count = (int)std::min<size_t>(kBandMax, bp.size() - i);
    int blk = 0;
    for (int j = 0; j < g.count; ++j) {
      g.prob[j] = bp[i + j];
      g.prob[j].blk_begin = blk;
      blk += kron_band_blocks((long long)g.prob[j].P * g.prob[j].nout * g.prob[j].Q);
    }
    g.total_blocks = blk;
    cudaError_t e = launch_kron_band(g, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
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
        if ((st = kron_band_setup(kf, F))) {
          free_kron(raw);
          return st;
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
        if (kf.bw > 0 && batch == 1) {
          std::vector<BandProb> bp(1);
          BandProb& b = bp[0];
          b.X = src;
          b.Y = dst;
          b.Wb = kf.Wb;
          b.lo = kf.lo;
          b.bw = kf.bw;
          b.P = (int)P;
          b.nin = kf.nin;
          b.nout = kf.nout;
          b.Q = (int)Q;
          b.alpha = last ? alpha * h->coef[t] : 1.0;
          b.beta = last ? (t == 0 ? beta : 1.0) : 0.0;
          FDP_CUDA(launch_band_probs(bp, s), "kron_op_apply: band");
          src = dst;
          sbs = dbs;
          continue;
        }
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
    std::vector<BandProb> bands;
    for (const Term& tm : terms) {
      const fdp_kron_s* op = tm.op;
      const KronFactor& kf = op->f[tm.t * D + d];
      long long P = 1, Q = 1;
      for (int e = 0; e < d; ++e) P *= op->nout[e];
      for (int e = d + 1; e < D; ++e) Q *= op->nin[e];
      const bool last = d == D - 1;
      if (kf.bw > 0) {
        BandProb b{};
        b.X = d == 0 ? tm.x : tm.T[(d - 1) % 2];
        b.Y = last ? tm.part : tm.T[d % 2];
        b.Wb = kf.Wb;
        b.lo = kf.lo;
        b.bw = kf.bw;
        b.P = (int)P;
        b.nin = kf.nin;
        b.nout = kf.nout;
        b.Q = (int)Q;
        b.alpha = last ? tm.scale : 1.0;
        b.beta = 0.0;
        bands.push_back(b);
        continue;
      }
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
    cudaError_t e = probs.empty() ? cudaSuccess : launch_stage(probs, cfgs, d == 0, s, nullptr, nullptr);
    if (e == cudaSuccess && !bands.empty()) e = launch_band_probs(bands, s);
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
