// K1t: the even-odd folded FD transform as a warp-specialised, TMA-fed,
// mbarrier-pipelined FP64 tensor-core kernel for sm_100a -- Algorithm 1 steps 2 and 4 (PAPER.md
// one m-mode product, against the folded eigenvector blocks), with the
// step-3 division by Lambda and the P^G post-scaling D^{-1/2} in the epilogue.
//
// FP64 tensor cores on sm_100a are the warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4; tcgen05
// has no f64 kind), so accumulators live in registers. Everything around them is Blackwell-native:
//   * one persistent CTA per SM, warp-specialised: 8 consumer warps (4 row slices x the E / O
//     roles), 1 producer warp, 3 store warps (12 warps, <= 168 registers each);
//   * the producer's lane 0 streams every K stage of the CTA's tile sequence through a 3-deep
//     ring: the two A tiles of a stage are cp.async.bulk.tensor loads through a tensor map with
//     the 128-byte swizzle (SASS UTMALDG), the E and O eigenvector chunks cp.async.bulk copies of
//     a host-prepared fragment-native layout (UBLKCP); completion is counted in bytes on the
//     stage's "full" mbarrier, and each consumer warp releases the slot on its "empty" mbarrier;
//   * a CTA tile is 64 rows x (up to 72 E + 72 O) folded columns; the CTAs of a column-tile group
//     work on the same row block at the same time (its A rows come from DRAM once);
//   * the consumers hand each finished tile to the store warps through a shared-memory staging
//     buffer (one mbarrier pair) and go straight on with the next tile's K loop; the store warps
//     drain it to HBM with 16-byte stores (an in-register epilogue stalled every consumer for
//     6-10k cycles per tile: all CTAs finish together and the store burst backs up the memory
//     system -- 13-21% of the kernel, measured with clock64 per phase);
//   * Lambda^{-1} (the last forward mode) is applied by the store warps on the way out, with the
//     Lambda factors staged in shared memory at kernel start (in the consumers its MUFU / FP64
//     work idled the DMMA pipe ~5k cycles per tile: 11-20% of that pass, measured).
//
// Folded algebra (persymmetric pencil, n = ne + no, ne = ceil(n/2)):
//   FOLD_FWD: y_E = W_E^T s, y_O = W_O^T d, s_k = x_k + x_{n-1-k}, d_k = x_k - x_{n-1-k}:
//     a stage holds the direct A tile (k0 .. k0+15) and the mirrored one (n-k0-16 .. n-k0-1);
//     E warps form s and O warps d per fragment; spectral output order [E | O].
//   FOLD_BWD: e = W_E y_E, o = W_O y_O, x_c = e_c + o_c, x_{n-1-c} = e_c - o_c (c < ne):
//     a stage holds the E part (k0 ..) and the O part (ne + k0 ..) of the spectral row; E warps
//     contract the first with W_E, O warps the second with W_O; the O warps hand their tile to
//     the E warps through shared memory, which store both mirrored outputs.
// The K loop runs over ne for both roles (W rows past ne / no are zero, so the extra terms add 0).
//
// Shared-memory fragment loads are bank-conflict free under the swizzle by the choice of the
// k order inside a stage (all operands use the same order, so the sum is unchanged):
//   non-KMAJ A ([k][p], p contiguous): the k4 step j covers k = 8(j>>1) + (j&1) + {0,2,4,6};
//   KMAJ A     ([row][k], k contiguous): k = 4j + {0..3}, and DMMA tile t of a warp takes the
//              rows 2r + t (r = 0..7) of its 16-row slice;
// the W chunks are laid out per (k4 step, n8 pair, lane) in that same k order.
#include <cuda.h>

#include <type_traits>

#include "../fdp_internal.h"
#include "../mode_tma.h"

namespace fdp {
namespace {

constexpr int kWM = 4;                              // row slices (x 2 roles = 8 warps)
constexpr int kMT = kTmaBM / (8 * kWM);             // 8-row DMMA tiles per warp (2)
constexpr int kConsumerWarps = 2 * kWM;
constexpr int kStoreWarps = 3;
constexpr int kThreads = (kConsumerWarps + 1 + kStoreWarps) * 32;  // + producer + store warps
// output-tile staging buffer: non-KMAJ [col 0..143][row] with a column stride == 16 B (mod 128),
// KMAJ [row 0..63][col] with a row stride == 32 B (mod 128): conflict-free fragment stores
constexpr int kCLdN = 66;
constexpr int kCLdK = 148;
constexpr int kCBytes = (144 * kCLdN > kTmaBM * kCLdK ? 144 * kCLdN : kTmaBM * kCLdK) * 8;
constexpr int kLamMax = 4800;
  // doubles of staged Lambda factors (all problems of a launch)
constexpr int kABytes = kTmaBM * kTmaBK * 8;        // one A tile (8 KB)
constexpr int kBBytes = kTmaWChunk * 8;             // one role's W chunk (10 KB)
constexpr int kMiniBytes = kTmaBM * 2 * 8;          // odd-start fix-up column pair (1 KB)
constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes + kMiniBytes;  // 37 KB
static_assert(kMT == 2, "fragment offsets below assume two 8-row tiles per warp");

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(unsigned dst, const CUtensorMap* map, unsigned bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(unsigned dst, const CUtensorMap* map, unsigned bar, int c0,
                                            int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
      "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_load(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ double lds64(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void lds128(unsigned a, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}
__device__ __forceinline__ void sts64(unsigned a, double x) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(x) : "memory");
}
__device__ __forceinline__ void sts128(unsigned a, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Diagnostic build only (-DFDP_K1T_PROF, `make prof` -> libfdp_prof.so): clock64 totals per
// warp role, summed over CTAs: [0] consumer wait on "full", [1] consumer wait on the staging
// buffer, [2] consumer total, [3] store wait on a staged tile, [4] store total, [5] producer wait
// on "empty", [6] producer total, [7] tiles (consumer warp 0), [8] consumer wait on the first
// stage of a tile, [9] producer time issuing (tile decode + copies).
#ifdef FDP_K1T_PROF
__device__ unsigned long long g_k1t_prof[8 * 16];
#define FDP_PT(v) long long v = clock64()
#define FDP_PACC(acc, t0) acc += clock64() - (t0)
#define FDP_PEND(v) v = clock64() - v
#define FDP_PFLUSH(slot, v) if (lane == 0) atomicAdd(&g_k1t_prof[16 * g.prof_slot + (slot)], (unsigned long long)(v))
#else
#define FDP_PT(v)
#define FDP_PACC(acc, t0)
#define FDP_PEND(v)
#define FDP_PFLUSH(slot, v)
#endif

struct Tile {
  int pi, ct, tp, tq, b;
};

// peer-store scatter target of output (GEMM row m, column a) of a batch-1 problem: the rank o
// owning a under the even split of sc_na over sc_G ranks, at its buffer offset (scatter_ptr's
// addressing, fdp_internal.h)
__device__ __forceinline__ double* tma_scatter_ptr(const TmaProb& p, long long m, int a) {
  const int G = p.sc_G, na = p.sc_na;
  const int q = na / G, rem = na % G;
  const int o = (q == 0 || a < rem * (q + 1)) ? a / (q + 1) : rem + (a - rem * (q + 1)) / q;
  const int lo = o * q + (o < rem ? o : rem);
  const int len = q + (o < rem ? 1 : 0);
  const long long r = m % p.sc_n1, qq = m / p.sc_n1;
  return p.peers[o] + r +
         (long long)p.sc_n1 * ((long long)(a - lo) * (p.sc_a0 + p.sc_a1 * len) + (qq + p.sc_qoff) * (p.sc_q0 + p.sc_q1 * len));
}

// Tile of this CTA's it-th iteration (-1: done). With a uniform column-tile count CT (grid a
// multiple of CT) the CT CTAs of a group work on the column tiles of the same row block at the
// same time -- its A rows are fetched from DRAM once and hit L2 for the others -- and rotate
// through the column tiles (which differ by one n8 tile of work), so no group member drifts ahead.
__device__ __forceinline__ int tile_of(const TmaGroup& g, int it) {
  if (g.ct_uniform > 0) {
    const int CT = g.ct_uniform, groups = gridDim.x / CT;
    const int rb = blockIdx.x / CT + groups * it;
    return rb * CT < g.total_tiles ? rb * CT + (blockIdx.x % CT + it) % CT : -1;
  }
  const int tau = blockIdx.x + gridDim.x * it;
  return tau < g.total_tiles ? tau : -1;
}

__device__ __forceinline__ Tile decode(const TmaGroup& g, int tau, bool kmaj) {
  Tile t;
  t.pi = 0;
#pragma unroll
  for (int i = 1; i < kTmaMaxProbs; ++i)
    if (i < g.count && tau >= g.prob[i].tile_begin) t.pi = i;
  const TmaProb& p = g.prob[t.pi];
  int local = tau - p.tile_begin;
  t.ct = local % p.ctiles;
  int rt = local / p.ctiles;
  if (kmaj) {
    t.tp = 0;
  } else {
    t.tp = rt % p.tiles_p;
    rt /= p.tiles_p;
  }
  t.tq = rt % p.tiles_q;
  t.b = rt / p.tiles_q;
  return t;
}

// ---------------------------------------------------------------------------------------------
// producer: issue stage s of the CTA's it-th tile into `slot` (out of line: the consumers'
// instruction stream only holds the call)
// ---------------------------------------------------------------------------------------------
// Per-tile constants of the producer (decoded once per tile: the tile decode's integer divisions
// cost ~1.7 k cycles per stage when they were redone for every stage -- the producer then spent
// 70% of its time issuing and the consumers waited on the ring)
struct TileIssue {
  const CUtensorMap* map;
  const CUtensorMap* map2;
  const double* w0;   // W chunks of stage 0: E role, O role
  const double* w1;
  int c2, c3, c4;     // tensor-map coordinates after k (KMAJ: row, batch; else p-group, q, batch)
  int n, ne, a1odd, kst;
};

template <bool KMAJ>
__device__ __forceinline__ TileIssue tile_issue(const TmaGroup& g, int tau) {
  const Tile t = decode(g, tau, KMAJ);
  const TmaProb& p = g.prob[t.pi];
  TileIssue ti;
  ti.map = &g.map[t.pi];
  ti.map2 = &g.map2[t.pi];
  ti.w0 = p.Wt + (size_t)((0 * p.ctiles + t.ct) * p.kst) * kTmaWChunk;
  ti.w1 = p.Wt + (size_t)((1 * p.ctiles + t.ct) * p.kst) * kTmaWChunk;
  if (KMAJ) {
    ti.c2 = t.tq * kTmaBM;
    ti.c3 = t.b;
    ti.c4 = 0;
  } else {
    ti.c2 = t.tp * p.bp;
    ti.c3 = t.tq * p.bq;
    ti.c4 = t.b;
  }
  ti.n = p.n;
  ti.ne = p.ne;
  ti.a1odd = p.a1odd;
  ti.kst = p.kst;
  return ti;
}

// producer: issue stage s of a tile into `slot`
template <bool KMAJ, int FOLD>
__device__ __forceinline__ void issue_stage(const TileIssue& ti, unsigned sbase, unsigned bar_full, int slot, int s) {
  const unsigned full = bar_full + 8 * slot;
  const unsigned dA0 = sbase + slot * kStageBytes;
  const unsigned dA1 = dA0 + kABytes;
  const unsigned dB = dA1 + kABytes;
  const int k0 = s * kTmaBK;
  const int k1 = FOLD == FOLD_FWD ? ti.n - k0 - kTmaBK : ti.ne + k0;
  if (KMAJ) {
    // a TMA box must start on a 16-byte boundary: an odd k1 (odd n forward, odd ne backward)
    // loads the 16 columns from k1 - 1 and the last one (k1 + 15) through a 2-column box
    mbar_expect_tx(full, 2 * kABytes + 2 * kBBytes + (ti.a1odd ? kMiniBytes : 0));
    tma_load_3d(dA0, ti.map, full, k0, ti.c2, ti.c3);
    tma_load_3d(dA1, ti.map, full, k1 - ti.a1odd, ti.c2, ti.c3);
    if (ti.a1odd) tma_load_3d(dB + 2 * kBBytes, ti.map2, full, k1 + 15, ti.c2, ti.c3);
  } else {
    mbar_expect_tx(full, 2 * kABytes + 2 * kBBytes);
    tma_load_5d(dA0, ti.map, full, 0, k0, ti.c2, ti.c3, ti.c4);
    tma_load_5d(dA1, ti.map, full, 0, k1, ti.c2, ti.c3, ti.c4);
  }
  bulk_load(dB, ti.w0 + (size_t)s * kTmaWChunk, kBBytes, full);
  bulk_load(dB + kBBytes, ti.w1 + (size_t)s * kTmaWChunk, kBBytes, full);
}

// the producer warp's loop (lane 0): every stage of the CTA's tile sequence, in order, into the
// ring slot the consumers released (the slot's "empty" mbarrier completes when all 8 consumer
// warps arrived on it); the next tile is decoded while the current one's stages are in flight
template <bool KMAJ, int FOLD, int STAGES>
__device__ __noinline__ void producer_loop(const TmaGroup& g, unsigned sbase, unsigned bar_full,
                                           unsigned bar_empty) {
  for (int i = 0; i < g.count; ++i)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&g.map[i]))
                 : "memory");
  int slot = 0;
  unsigned phase = 0;
  const int lane = 0;
  long long pw = 0, pis = 0;
  FDP_PT(ptot);
  int tau = tile_of(g, 0);
  if (tau < 0) return;
  TileIssue cur = tile_issue<KMAJ>(g, tau);
  for (int it = 0;; ++it) {
    const int tau_next = tile_of(g, it + 1);
    for (int s = 0; s < cur.kst; ++s) {
      FDP_PT(t0);
      mbar_wait(bar_empty + 8 * slot, phase ^ 1);
      FDP_PACC(pw, t0);
      FDP_PT(t2);
      issue_stage<KMAJ, FOLD>(cur, sbase, bar_full, slot, s);
      FDP_PACC(pis, t2);
      if (++slot == STAGES) {
        slot = 0;
        phase ^= 1;
      }
    }
    if (tau_next < 0) break;
    cur = tile_issue<KMAJ>(g, tau_next);
  }
  FDP_PFLUSH(5, pw);
  FDP_PFLUSH(9, pis);
  (void)pis;
  FDP_PEND(ptot);
  FDP_PFLUSH(6, ptot);
  (void)pw;
  (void)lane;
}

// ---------------------------------------------------------------------------------------------
// one stage of the consumer K loop: J k4 steps (4, or fewer in a partial last stage),
// NTV = n8 tiles per role (9 or 8; 0 = any nt <= 9, masked), ODD = KMAJ second A tile loaded
// from one column earlier (see issue_stage). Fragment offsets (bytes within an A tile):
//   off[ti][jj]: non-KMAJ: A0 and A1 rows k = 8(j>>1) + 2 fc + jj (j & 1 = jj) of 16-row group
//                wm; KMAJ: row base + in-row part for k = 4j + fc (see kmaj_col)
// ---------------------------------------------------------------------------------------------
struct Frag {
  unsigned a0[kMT][2];   // non-KMAJ: direct / E-part offsets per (tile, j & 1); KMAJ: row bases
  unsigned a1[kMT][2];   // non-KMAJ: mirror offsets (FWD) ; KMAJ: xor term y per tile in [ti][0]
};

// KMAJ: byte of column lam in row R of a swizzled [row][16] tile
__device__ __forceinline__ unsigned kmaj_col(unsigned rowbase, int x, int lam) {
  return rowbase + ((((lam >> 1) ^ x) << 4) | ((lam & 1) << 3));
}

// NAT: the natural k order k = 4 j + c in a non-KMAJ last stage (tma_last_nat; offsets computed
// here, the same bank-conflicted order in the host's W chunk of that stage)
__device__ __forceinline__ unsigned swz(int plo, int k) {
  return (unsigned)((((plo >> 1) ^ (k & 7)) << 4) | ((plo & 1) << 3));
}

template <bool KMAJ, int FOLD, int NTV, int ODD, int J, bool NAT = false>
__device__ __forceinline__ void stage_mma(double (&acc)[kMT][9][2], int nt, unsigned A0, unsigned A1,
                                          unsigned B, unsigned Mini, const Frag& f, double sgn,
                                          int role, int wm, int fr, int fc, int lane, int jmax) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (j < J && (J == 4 || j < jmax)) {
      double a[kMT];
#pragma unroll
      for (int ti = 0; ti < kMT; ++ti) {
        if (KMAJ) {
          const unsigned rb = f.a0[ti][0];
          const int x = (int)f.a1[ti][0];
          const int k = 4 * j + fc;
          const int l1 = (FOLD == FOLD_FWD ? kTmaBK - 1 - k : k) + ODD;
          const unsigned a1 = (ODD && l1 == kTmaBK) ? Mini + f.a1[ti][1] : A1 + kmaj_col(rb, x, l1);
          if (FOLD == FOLD_FWD) {
            const double v = lds64(A0 + kmaj_col(rb, x, k)), w = lds64(a1);
            a[ti] = fma(sgn, w, v);
          } else {
            a[ti] = lds64(role ? a1 : A0 + kmaj_col(rb, x, k));
          }
        } else if (NAT) {
          const int k = 4 * j + fc, km = kTmaBK - 1 - k, plo = 8 * ti + fr;
          const unsigned o0 = (unsigned)((k + 16 * wm) * 128) + swz(plo, k);
          if (FOLD == FOLD_FWD) {
            const unsigned o1 = (unsigned)((km + 16 * wm) * 128) + swz(plo, km);
            const double v = lds64(A0 + o0), w = lds64(A1 + o1);
            a[ti] = fma(sgn, w, v);
          } else {
            a[ti] = lds64((role ? A1 : A0) + o0);
          }
        } else {
          const unsigned o0 = f.a0[ti][j & 1] + (j >> 1) * 8 * 128;
          if (FOLD == FOLD_FWD) {
            const unsigned o1 = f.a1[ti][j & 1] - (j >> 1) * 8 * 128;
            const double v = lds64(A0 + o0), w = lds64(A1 + o1);
            a[ti] = fma(sgn, w, v);
          } else {
            a[ti] = lds64((role ? A1 : A0) + o0);
          }
        }
      }
      double b[10];
#pragma unroll
      for (int tp = 0; tp < 5; ++tp) lds128(B + ((j * 5 + tp) * 32 + lane) * 16, b[2 * tp], b[2 * tp + 1]);
#pragma unroll
      for (int ti = 0; ti < kMT; ++ti)
#pragma unroll
        for (int u = 0; u < 9; ++u) {
          if (NTV ? (u < NTV) : (u < nt)) dmma(acc[ti][u], a[ti], b[u]);
        }
    }
  }
}

template <bool KMAJ, int FOLD, int STAGES, int NTV, int ODD>
__device__ __forceinline__ void kloop(const TmaGroup& g, double (&acc)[kMT][9][2], int nt, int kst, int ne,
                                      unsigned sbase, unsigned bar_full, unsigned bar_empty, int& stage,
                                      unsigned& phase, const Frag& f, int role, int wm, int fr, int fc, int lane,
                                      long long& wfull, long long& wfirst) {
  const double sgn = role ? -1.0 : 1.0;  // FWD: E warps form s = x + Jx, O warps d = x - Jx
  const int rem = ne - (kst - 1) * kTmaBK;  // valid k of the last stage (1 .. 16)
  const bool nat = tma_last_nat(ne, KMAJ);
  const int jlast = KMAJ || nat ? (rem + 3) >> 2 : (rem <= 8 ? 2 : 4);
  for (int s = 0; s < kst; ++s) {
    FDP_PT(t0);
    mbar_wait(bar_full + 8 * stage, phase);
    FDP_PACC(wfull, t0);
    if (s == 0) FDP_PACC(wfirst, t0);
    const unsigned A0 = sbase + stage * kStageBytes;
    const unsigned A1 = A0 + kABytes;
    const unsigned B = A1 + kABytes + role * kBBytes;
    const unsigned Mini = A1 + kABytes + 2 * kBBytes;
    if (s + 1 < kst || jlast == 4)
      stage_mma<KMAJ, FOLD, NTV, ODD, 4>(acc, nt, A0, A1, B, Mini, f, sgn, role, wm, fr, fc, lane, 4);
    else if (!KMAJ && nat)
      stage_mma<KMAJ, FOLD, NTV, ODD, 3, true>(acc, nt, A0, A1, B, Mini, f, sgn, role, wm, fr, fc, lane, jlast);
    else
      stage_mma<KMAJ, FOLD, NTV, ODD, 3>(acc, nt, A0, A1, B, Mini, f, sgn, role, wm, fr, fc, lane, jlast);
    __syncwarp();
    if (lane == 0) mbar_arrive(bar_empty + 8 * stage);  // this warp is done with the slot
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// the store warp: drains each finished output tile from the shared-memory staging buffer to HBM
// while the consumers already run the next tile's K loop (an in-register epilogue stalled every
// consumer for 6-10k cycles per tile: all CTAs finish their tiles together and the store burst
// backs up the memory system). Staged columns: E at 0, O at 72 (FWD) / e at 0, o at 72 (BWD).
//   non-KMAJ: [col][row] (kCLdN), lane l owns rows 2l, 2l+1 (consecutive p: 16-byte stores);
//   KMAJ    : [row][col] (kCLdK), lanes walk column pairs of a row.
//   FWD: E column c -> spectral column 8 nt0 + c (< ne), O column c -> ne + 8 nt0 + c (< n);
//        EPI_LAMBDA divides by lrow(p) + lamcol[col]; a KMAJ output row's pad column gets 0.
//   BWD: x_c = e_c + o_c, x_{n-1-c} = e_c - o_c for c = 8 nt0 + col < ne; EPI_SCALE multiplies.
// Rows: KMAJ row R is q = 64 tq + R; otherwise R = 16 g + p_lo of p-group g (see decode).
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ double lds_f64(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}

template <bool KMAJ, int FOLD>
__device__ __noinline__ void store_loop(const TmaGroup& g, unsigned cbuf, unsigned bar_cfull,
                                        unsigned bar_cempty, double* lsm, int lane, int sw) {
  const unsigned lsa = smem_u32(lsm);
  long long sw_wait = 0;
  FDP_PT(stot);
  if (FOLD == FOLD_FWD && !KMAJ && g.lam_elems > 0) {
    // stage the Lambda factors of every EPI_LAMBDA problem: [lam0 (n1v of n1) | lam1 | lamcol]
    for (int pi = 0; pi < g.count; ++pi) {
      const TmaProb& q = g.prob[pi];
      if (q.epi != EPI_LAMBDA) continue;
      double* d = lsm + q.lam_off;
      const int tid = lane + 32 * sw;
      for (int i = tid; i < q.n1v; i += kStoreWarps * 32) d[i] = q.lam0[i];
      if (q.lam1)
        for (int i = tid; i < q.lam1_n; i += kStoreWarps * 32) d[q.n1 + i] = q.lam1[i];
      for (int i = tid; i < q.n; i += kStoreWarps * 32) d[q.n1 + q.lam1_n + i] = q.lamcol[i];
    }
    named_bar(14, kStoreWarps * 32);
  }
  unsigned phase = 0;
  for (int it = 0;; ++it) {
    const int tau = tile_of(g, it);
    if (tau < 0) break;
    const Tile t = decode(g, tau, KMAJ);
    const TmaProb& p = g.prob[t.pi];
    const int nbase = p.n8h / p.ctiles, nrem = p.n8h % p.ctiles;
    const int nt = nbase + (t.ct < nrem ? 1 : 0);
    const int c0 = 8 * (t.ct * nbase + min(t.ct, nrem));
    const int ncol = 8 * nt;
    double* __restrict__ Y = p.Y;
    const int ne = p.ne, no = p.no, n = p.n;
    FDP_PT(t0);
    mbar_wait(bar_cfull, phase);
    FDP_PACC(sw_wait, t0);
    // Every path gathers a chunk of U columns / elements from shared (and global, for D^{-1/2})
    // memory first, then does the arithmetic, then stores: the store warps' FP64 work queues
    // behind the consumers' DMMAs on the shared FP64 datapath, so a dependent load -> divide ->
    // store chain per column (~600 cycles) made them the bottleneck of the short-K passes;
    // independent chains across the chunk hide that latency. Out-of-range entries read a clamped
    // (valid) address and are not stored.
    if (!KMAJ) {
      // lane l: rows R = 2l, 2l + 1 (same p-group, consecutive p; P is even so both exist or not)
      const long long P = p.P;
      const int R = 2 * lane, gq = R >> 4, plo = R & 15;
      const long long q = (long long)t.tq * p.bq + gq / p.bp;
      const int pp = 16 * (t.tp * p.bp + gq % p.bp) + plo;
      const bool valid = pp < p.P && q < p.Q;
      const long long sidx = pp + P * n * q;
      double* yrow = Y + sidx + p.ybs * t.b;
      if (valid && FOLD == FOLD_FWD) {
        // Algorithm 1 step 3 on the way out (EPI_LAMBDA): q~ = t~ / (lrow(p) +
        // lamcol(a)), Lambda formed from its factors; the padding rows i1 >= n1v of a padded
        // intermediate stay exactly 0
        // with a stored 1 / Lambda table (rlam, the block / FD path): one DMUL per element, its
        // loads coalesced like the stores; otherwise (slab phases) the on-the-fly division
        const bool tab = p.epi == EPI_LAMBDA && p.rlam != nullptr;
        const bool lam = p.epi == EPI_LAMBDA && !tab;
        const double* rl = tab ? p.rlam + sidx : nullptr;
        double lr0 = 0.0, lr1 = 0.0;
        bool zr0 = false, zr1 = false;
        if (lam) {
          const unsigned L = lsa + 8u * (unsigned)p.lam_off;
          const int i10 = pp % p.n1, i11 = (pp + 1) % p.n1;
          zr0 = i10 >= p.n1v;
          zr1 = i11 >= p.n1v;
          if (p.lam1) {
            lr0 = lds_f64(L + 8u * (zr0 ? 0 : i10)) + lds_f64(L + 8u * (p.n1 + pp / p.n1));
            lr1 = lds_f64(L + 8u * (zr1 ? 0 : i11)) + lds_f64(L + 8u * (p.n1 + (pp + 1) / p.n1));
          } else {
            lr0 = lds_f64(L + 8u * (zr0 ? 0 : pp));
            lr1 = lds_f64(L + 8u * (zr1 ? 0 : pp + 1));
          }
        }
        const unsigned Lc = lsa + 8u * (unsigned)(p.lam_off + p.n1 + p.lam1_n);
        constexpr int U = 6;
        const int total = 2 * ncol;  // (half, column) pairs dealt over the store warps: h = 0 E, 1 O
        for (int w0 = sw; w0 < total; w0 += U * kStoreWarps) {
          double v[U][2], lc[U], rv[U][2];
          int oc[U];
          bool ok[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int w = w0 + u * kStoreWarps;
            const int h = w >= ncol, c = w - h * ncol, a = c0 + c;
            ok[u] = w < total && a < (h ? no : ne);
            oc[u] = ok[u] ? (h ? ne : 0) + a : 0;
            lds128(cbuf + (unsigned)((ok[u] ? 72 * h + c : 0) * kCLdN + R) * 8u, v[u][0], v[u][1]);
            lc[u] = lam ? lds_f64(Lc + 8u * oc[u]) : 0.0;
            if (tab) {
              const double2 r2 = __ldg(reinterpret_cast<const double2*>(rl + P * oc[u]));
              rv[u][0] = r2.x;
              rv[u][1] = r2.y;
            }
          }
          if (tab) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
              v[u][0] *= rv[u][0];
              v[u][1] *= rv[u][1];
            }
          } else if (lam) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
              v[u][0] = zr0 ? 0.0 : fdp_div(v[u][0], lr0 + lc[u]);
              v[u][1] = zr1 ? 0.0 : fdp_div(v[u][1], lr1 + lc[u]);
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (!ok[u]) continue;
            // the peer-store exchange: rows pp, pp + 1 of the same i1-row land contiguously
            double* dst = p.peers ? tma_scatter_ptr(p, pp + P * q, oc[u]) : yrow + P * oc[u];
            *reinterpret_cast<double2*>(dst) = make_double2(v[u][0], v[u][1]);
          }
        }
      } else if (valid) {
        const bool scl = p.epi == EPI_SCALE;
        constexpr int U = 4;
        for (int w0 = sw; w0 < ncol; w0 += U * kStoreWarps) {
          double e[U][2], o[U][2], s0[U][2], s1[U][2];
          int cc[U];
          bool ok[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int w = w0 + u * kStoreWarps;
            ok[u] = w < ncol && c0 + w < ne;
            const int c = ok[u] ? w : 0;
            cc[u] = c0 + c;
            lds128(cbuf + (unsigned)(c * kCLdN + R) * 8u, e[u][0], e[u][1]);
            lds128(cbuf + (unsigned)((72 + c) * kCLdN + R) * 8u, o[u][0], o[u][1]);
            if (scl) {
              const double2 a0 = __ldg(reinterpret_cast<const double2*>(p.scale + sidx + P * cc[u]));
              const double2 a1 = __ldg(reinterpret_cast<const double2*>(p.scale + sidx + P * (n - 1 - cc[u])));
              s0[u][0] = a0.x; s0[u][1] = a0.y; s1[u][0] = a1.x; s1[u][1] = a1.y;
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            double x0 = e[u][0] + o[u][0], x1 = e[u][1] + o[u][1];
            double y0 = e[u][0] - o[u][0], y1 = e[u][1] - o[u][1];
            if (scl) {
              x0 *= s0[u][0]; x1 *= s0[u][1]; y0 *= s1[u][0]; y1 *= s1[u][1];
            }
            const int cm = n - 1 - cc[u];
            if (ok[u]) {
              double* dx = p.peers ? tma_scatter_ptr(p, pp + P * q, cc[u]) : yrow + P * cc[u];
              *reinterpret_cast<double2*>(dx) = make_double2(x0, x1);
              if (cm != cc[u]) {
                double* dy = p.peers ? tma_scatter_ptr(p, pp + P * q, cm) : yrow + P * cm;
                *reinterpret_cast<double2*>(dy) = make_double2(y0, y1);
              }
            }
          }
        }
      }
    } else if (FOLD == FOLD_FWD) {
      // KMAJ FWD (mode 1 forward into a padded intermediate: 16-byte aligned rows): (row, column
      // pair) elements flattened over the lanes of the store warps, 16-byte stores; the pad
      // column of a padded row (past the O part) gets 0
      const int pairs = ncol / 2;  // column pairs per half (ncol = 8 nt)
      const int per_row = 2 * pairs;
      const int total = kTmaBM * per_row;
      constexpr int U = 4;
      for (int e0 = lane + 32 * sw; e0 < total; e0 += U * 32 * kStoreWarps) {
        double va[U][2];
        int Rr[U], ww[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + u * 32 * kStoreWarps;
          const int ee = e < total ? e : 0;
          const int R = ee / per_row, w = ee - R * per_row;
          Rr[u] = R;
          ww[u] = w;
          ok[u] = e < total && (long long)t.tq * kTmaBM + R < p.Q;
          const int h = w >= pairs, c = 2 * (w - h * pairs);
          lds128(cbuf + (unsigned)(R * kCLdK + 72 * h + c) * 8u, va[u][0], va[u][1]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (!ok[u]) continue;
          double* yrow = Y + (long long)p.yld * ((long long)t.tq * kTmaBM + Rr[u]) + p.ybs * t.b;
          const int w = ww[u];
          const int h = w >= pairs, c = 2 * (w - h * pairs);
          const int a = c0 + c, oc = (h ? ne : 0) + a;
          const int lim = h ? no : ne;
          const double v0 = va[u][0], v1 = va[u][1];
          if (a + 1 < lim && ((reinterpret_cast<unsigned long long>(yrow + oc) & 15) == 0)) {
            *reinterpret_cast<double2*>(yrow + oc) = make_double2(v0, v1);
          } else {
#pragma unroll
            for (int d = 0; d < 2; ++d) {
              const double v = d ? v1 : v0;
              if (a + d < lim) yrow[oc + d] = v;
              else if (h && oc + d < p.yld) yrow[oc + d] = 0.0;  // the pad column of a padded row
            }
          }
        }
      }
    } else {
      // KMAJ BWD (mode 1 backward, usually into the C-ABI layout, whose rows need not be 16-byte
      // aligned): (row, column pair) elements flattened over the store warps' lanes, the butterfly
      // x_c = e_c + o_c, x_{n-1-c} = e_c - o_c, 16-byte stores where the pair is aligned. (Chunked
      // gather / compute / store variants and row-aligned segment copies of this loop measured
      // 1.2-2.3x slower on configs 4-5.)
      const int pairs = ncol / 2;
      for (int e = lane + 32 * sw; e < kTmaBM * pairs; e += 32 * kStoreWarps) {
        const int R = e / pairs, w = e - R * pairs;
        const long long q = (long long)t.tq * kTmaBM + R;
        if (q >= p.Q) continue;
        const long long sidx = (long long)p.yld * q;
        double* yrow = Y + sidx + p.ybs * t.b;
        const int c = 2 * w, cc = c0 + c;
        double e0, e1, o0, o1;
        lds128(cbuf + (unsigned)(R * kCLdK + c) * 8u, e0, e1);
        lds128(cbuf + (unsigned)(R * kCLdK + 72 + c) * 8u, o0, o1);
        double x0 = e0 + o0, x1 = e1 + o1, y0 = e0 - o0, y1 = e1 - o1;
        const int cm = n - 1 - cc;  // y_d goes to column cm - d
        if (p.epi == EPI_SCALE) {
          x0 *= p.scale[sidx + cc];
          y0 *= p.scale[sidx + cm];
          if (cc + 1 < ne) {
            x1 *= p.scale[sidx + cc + 1];
            y1 *= p.scale[sidx + cm - 1];
          }
        }
        if (cc + 1 < ne && (reinterpret_cast<unsigned long long>(yrow + cc) & 15) == 0)
          *reinterpret_cast<double2*>(yrow + cc) = make_double2(x0, x1);
        else {
          if (cc < ne) yrow[cc] = x0;
          if (cc + 1 < ne) yrow[cc + 1] = x1;
        }
        // mirrored pair (cm - 1, cm) = (y1, y0); the middle column of an odd n (cm == cc) is x
        if (cc + 1 < ne && cm - 1 > cc + 1 && (reinterpret_cast<unsigned long long>(yrow + cm - 1) & 15) == 0)
          *reinterpret_cast<double2*>(yrow + cm - 1) = make_double2(y1, y0);
        else {
          if (cc < ne && cm != cc) yrow[cm] = y0;
          if (cc + 1 < ne && cm - 1 != cc + 1) yrow[cm - 1] = y1;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(bar_cempty);  // the buffer may take the next tile
    phase ^= 1;
  }
  FDP_PFLUSH(3, sw_wait);
  FDP_PEND(stot);
  FDP_PFLUSH(4, stot);
  (void)sw_wait;
}

// ---------------------------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------------------------
template <bool KMAJ, int FOLD, int STAGES>
__global__ void __launch_bounds__(kThreads, 1) mode_tma_kernel(const __grid_constant__ TmaGroup g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment (shared-window address) for the 128-byte swizzle atoms
  const unsigned sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const unsigned cbuf = sbase + STAGES * kStageBytes;
  const unsigned bar_full = cbuf + kCBytes;
  const unsigned bar_empty = bar_full + 8 * STAGES;
  const unsigned bar_cfull = bar_empty + 8 * STAGES;
  const unsigned bar_cempty = bar_cfull + 8;
  // Lambda factors of every problem (EPI_LAMBDA launches): [lam0 | lam1 | lamcol] per problem
  double* lsm = reinterpret_cast<double*>(smem_raw + (bar_cempty + 64 - smem_u32(smem_raw)));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, kConsumerWarps);
    }
    mbar_init(bar_cfull, kConsumerWarps);
    mbar_init(bar_cempty, kStoreWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kConsumerWarps) {  // the producer warp
    if (lane == 0) producer_loop<KMAJ, FOLD, STAGES>(g, sbase, bar_full, bar_empty);
    return;
  }
  if (warp > kConsumerWarps) {  // the store warps
    store_loop<KMAJ, FOLD>(g, cbuf, bar_cfull, bar_cempty, lsm, lane, warp - kConsumerWarps - 1);
    return;
  }

  const int wm = warp % kWM, role = warp / kWM;  // role 0: E, 1: O
  const int fr = lane >> 2, fc = lane & 3;
  int stage = 0;
  unsigned phase = 0, cphase = 0;
  long long wfull = 0, wcempty = 0, ntiles = 0, wfirst = 0;
  FDP_PT(ctot);
  // per-thread fragment offsets (see Frag)
  Frag f;
#pragma unroll
  for (int ti = 0; ti < kMT; ++ti) {
    if (KMAJ) {
      const int R = 16 * wm + 2 * fr + ti;       // rows 2r + t of the 16-row slice
      f.a0[ti][0] = f.a0[ti][1] = (unsigned)(R * 128);
      f.a1[ti][0] = (unsigned)(R & 7);
      f.a1[ti][1] = (unsigned)(R * 16);          // fix-up box row (2 doubles per row)
    } else {
      const int plo = 8 * ti + fr;               // 16-row group wm, rows p_lo
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const int k = 2 * fc + jj, km = kTmaBK - 1 - k;   // j < 2 rows; j >= 2 add / sub 8 rows
        f.a0[ti][jj] = (unsigned)((k + 16 * wm) * 128) + swz(plo, k);
        f.a1[ti][jj] = (unsigned)((km + 16 * wm) * 128) + swz(plo, km);
      }
    }
  }

  for (int it = 0;; ++it) {
    const int tau = tile_of(g, it);
    if (tau < 0) break;
    const Tile t = decode(g, tau, KMAJ);
    const TmaProb& p = g.prob[t.pi];
    // n8 tiles of this column tile (same count for both roles; the O half's extra column, if
    // any, multiplies zero W columns)
    const int nbase = p.n8h / p.ctiles, nrem = p.n8h % p.ctiles;
    const int nt = nbase + (t.ct < nrem ? 1 : 0);

    double acc[kMT][9][2];
#pragma unroll
    for (int i = 0; i < kMT; ++i)
#pragma unroll
      for (int u = 0; u < 9; ++u) acc[i][u][0] = acc[i][u][1] = 0.0;

    // the K loop, specialised on the column tile's n8 count (no per-DMMA predicate: a predicated
    // mma.sync costs a WARPSYNC + NOP pair) and, for KMAJ, on the odd-start second A tile
    const int odd = KMAJ ? p.a1odd : 0;
#define FDP_K1T_RUN(NTV_, ODD_) \
  kloop<KMAJ, FOLD, STAGES, NTV_, ODD_>(g, acc, nt, p.kst, p.ne, sbase, bar_full, bar_empty, stage, phase, f, role, wm, fr, fc, lane, wfull, wfirst)
    if (nt == 9) {
      if (odd) FDP_K1T_RUN(9, 1); else FDP_K1T_RUN(9, 0);
    } else if (nt == 8) {
      if (odd) FDP_K1T_RUN(8, 1); else FDP_K1T_RUN(8, 0);
    } else {
      if (odd) FDP_K1T_RUN(0, 1); else FDP_K1T_RUN(0, 0);
    }
#undef FDP_K1T_RUN
    // ------------------------------ epilogue ------------------------------
    // stage the accumulators (E columns at 0, O at 72) for the store warps, once they have
    // drained the previous tile; rows as in the fragment layout (KMAJ: 2r + t of the slice; else
    // p_lo). The epilogue arithmetic (Lambda^{-1}, the backward butterfly, D^{-1/2}) is the store
    // warps' (measured: forming the butterfly here instead cost the consumers ~4% on config 5).
    FDP_PT(t1);
    mbar_wait(bar_cempty, cphase ^ 1);
    FDP_PACC(wcempty, t1);
    ++ntiles;
#pragma unroll
    for (int ti = 0; ti < kMT; ++ti) {
      if (KMAJ) {
        const int R = 16 * wm + 2 * fr + ti;
#pragma unroll
        for (int u = 0; u < 9; ++u)
          if (u < nt) sts128(cbuf + (unsigned)(R * kCLdK + 72 * role + 8 * u + 2 * fc) * 8u, acc[ti][u][0], acc[ti][u][1]);
      } else {
        const int R = 16 * wm + 8 * ti + fr;
#pragma unroll
        for (int u = 0; u < 9; ++u)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (u < nt) sts64(cbuf + (unsigned)((72 * role + 8 * u + 2 * fc + h) * kCLdN + R) * 8u, acc[ti][u][h]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(bar_cfull);
    cphase ^= 1;
  }
  FDP_PFLUSH(0, wfull);
  FDP_PFLUSH(1, wcempty);
  FDP_PFLUSH(8, wfirst);
  (void)wfirst;
  FDP_PEND(ctot);
  FDP_PFLUSH(2, ctot);
  if (warp == 0) FDP_PFLUSH(7, ntiles);
  (void)wfull;
  (void)wcempty;
  (void)ntiles;
}

// Shared memory: the A / W ring, the output staging buffer, the barriers, and (LAM: launches with
// an EPI_LAMBDA problem) the staged Lambda factors. Launches without Lambda factors afford a
// 4-deep ring (229,760 B of the 232,448 B opt-in limit); the Lambda pass keeps 3 stages.
template <int STAGES, bool LAM>
constexpr size_t smem_bytes() {
  return 1024 + (size_t)STAGES * kStageBytes + kCBytes + 16 * STAGES + 64 + (LAM ? (size_t)kLamMax * 8 : 0);
}
static_assert(smem_bytes<4, false>() <= 232448 && smem_bytes<3, true>() <= 232448, "K1t shared memory");

template <bool KMAJ, int FOLD, int STAGES, bool LAM>
cudaError_t launch_t(const TmaGroup& g, int grid, cudaStream_t s) {
  constexpr size_t sm = smem_bytes<STAGES, LAM>();
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(mode_tma_kernel<KMAJ, FOLD, STAGES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  mode_tma_kernel<KMAJ, FOLD, STAGES><<<grid, kThreads, sm, s>>>(g);
  return cudaGetLastError();
}

template <bool KMAJ, int FOLD, int STAGES, bool LAM>
cudaError_t set_smem_attr() {
  return cudaFuncSetAttribute(mode_tma_kernel<KMAJ, FOLD, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem_bytes<STAGES, LAM>());
}

}  // namespace

cudaError_t prepare_mode_tma() {
  // set the shared-memory attributes outside any stream capture
  cudaError_t e;
  if ((e = set_smem_attr<true, FOLD_FWD, 4, false>()) || (e = set_smem_attr<false, FOLD_FWD, 4, false>()) ||
      (e = set_smem_attr<false, FOLD_FWD, 3, true>()) || (e = set_smem_attr<true, FOLD_BWD, 4, false>()) ||
      (e = set_smem_attr<false, FOLD_BWD, 4, false>()))
    return e;
  return cudaSuccess;
}

cudaError_t launch_mode_tma(const TmaGroup& g, bool kmaj, int fold, int grid, cudaStream_t s) {
  if (g.total_tiles <= 0) return cudaSuccess;
  if (fold == FOLD_FWD) {
    if (kmaj) return g.lam_elems > 0 ? cudaErrorInvalidValue : launch_t<true, FOLD_FWD, 4, false>(g, grid, s);
    return g.lam_elems > 0 ? launch_t<false, FOLD_FWD, 3, true>(g, grid, s) : launch_t<false, FOLD_FWD, 4, false>(g, grid, s);
  }
  if (fold == FOLD_BWD)
    return kmaj ? launch_t<true, FOLD_BWD, 4, false>(g, grid, s) : launch_t<false, FOLD_BWD, 4, false>(g, grid, s);
  return cudaErrorInvalidValue;
}

// 1 / Lambda of the Lambda pass's output layout (setup time; Algorithm 1 step 3, with
// Lambda = sum_d c_d lambda_d formed from its factors; IEEE division)
namespace {
__global__ void rlam_kernel(double* __restrict__ rlam, const double* __restrict__ lam0,
                            const double* __restrict__ lam1, const double* __restrict__ lamcol, int n1p,
                            int n1v, int n_mid, long long total) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long P = (long long)n1p * n_mid;
    const long long a = i / P, p = i - a * P;
    const int i1 = (int)(p % n1p), im = (int)(p / n1p);
    rlam[i] = i1 >= n1v ? 0.0 : 1.0 / (lam0[i1] + (lam1 ? lam1[im] : 0.0) + lamcol[a]);
  }
}
}  // namespace

cudaError_t launch_rlam(double* rlam, const double* lam0, const double* lam1, const double* lamcol, int n1p,
                        int n1v, int n_mid, int n_last, cudaStream_t s) {
  const long long total = (long long)n1p * n_mid * n_last;
  if (total == 0) return cudaSuccess;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  rlam_kernel<<<blocks, 256, 0, s>>>(rlam, lam0, lam1, lamcol, n1p, n1v, n_mid, total);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Row padding for K1t's first pass: y (rows of n1p = n1 + 1, pad entry zero) <- x (rows of odd
// n1), batch items at strides xbs / ybs (even). Used only when the C-ABI input cannot be read
// through a tensor map (odd row length or a base not 16-byte aligned: a TMA box starts on a
// 16-byte boundary and strides are multiples of 16 B). HBM streaming, 16 B per element: each
// thread writes output pairs with 16-byte stores, four independent pairs in flight.
// ---------------------------------------------------------------------------------------------
namespace {
__global__ void pad_rows_kernel(const double* __restrict__ x, long long xbs, double* __restrict__ y,
                                long long ybs, int n1, int n1p, long long rows, long long batch) {
  const long long pairs_item = rows * n1p / 2, total = pairs_item * batch;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < total; i0 += 4 * stride) {
    double v[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = i0 + u * stride;
      v[u][0] = v[u][1] = 0.0;
      if (i < total) {
        const long long b = i / pairs_item, j = 2 * (i - b * pairs_item);
        const long long r = j / n1p;
        const int c = (int)(j - r * n1p);
        const double* src = x + b * xbs + r * n1 + c;
        v[u][0] = c < n1 ? __ldg(src) : 0.0;
        v[u][1] = c + 1 < n1 ? __ldg(src + 1) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = i0 + u * stride;
      if (i < total) {
        const long long b = i / pairs_item, j = 2 * (i - b * pairs_item);
        *reinterpret_cast<double2*>(y + b * ybs + j) = make_double2(v[u][0], v[u][1]);
      }
    }
  }
}
}  // namespace

cudaError_t launch_pad_rows(const double* x, long long xbs, double* y, long long ybs, int n1,
                            int n1p, long long rows, long long batch, cudaStream_t s) {
  const long long total = rows * n1p / 2 * batch;
  if (total == 0) return cudaSuccess;
  if ((n1p & 1) || (ybs & 1) || (reinterpret_cast<uintptr_t>(y) & 15)) return cudaErrorInvalidValue;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = (int)std::min<long long>((total + 1023) / 1024, (long long)sms * 8);
  pad_rows_kernel<<<blocks, 256, 0, s>>>(x, xbs, y, ybs, n1, n1p, rows, batch);
  return cudaGetLastError();
}

}  // namespace fdp

#ifdef FDP_K1T_PROF
// diagnostic build: copy out and reset the K1t per-role clock totals ([launch ordinal mod 8][8])
extern "C" int fdp_k1t_prof_read(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, fdp::g_k1t_prof, sizeof(unsigned long long) * 128) != cudaSuccess) return -1;
  unsigned long long z[128] = {};
  return cudaMemcpyToSymbol(fdp::g_k1t_prof, z, sizeof(z)) == cudaSuccess ? 0 : -1;
}
#endif
