// K1t: the even-odd folded FD transform as a warp-specialised, TMA-fed,
// mbarrier-pipelined FP64 tensor-core kernel for sm_100a -- Algorithm 1 steps 2 and 4 (PAPER.md
// one m-mode product, against the folded eigenvector blocks), with the
// step-3 division by Lambda and the P^G post-scaling D^{-1/2} in the epilogue.
//
// FP64 tensor cores on sm_100a are the warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4; tcgen05
// has no f64 kind), so accumulators live in registers. Everything around them is Blackwell-native:
//   * one persistent CTA per SM: 8 warps (4 along M x the E / O roles; two per SM sub-partition,
//     so each may hold up to 255 registers -- a ninth, producer-only warp would put three warps on
//     one sub-partition and cap every thread at 168 registers);
//   * lane 0 of warp 0 is the producer: it streams every K stage with TMA, STAGES deep ahead of
//     the consumers and across tile boundaries: the two A tiles of a stage are
//     cp.async.bulk.tensor loads through a tensor map with the 128-byte swizzle (SASS UTMALDG),
//     the E and O eigenvector chunks are cp.async.bulk copies of a host-prepared fragment-native
//     layout (UBLKCP); completion is counted in bytes on the stage's "full" mbarrier, and the
//     consumer warps release a stage on its "empty" mbarrier -- no CTA-wide barrier in the loop;
//   * a CTA tile is 128 rows x (up to 72 E + 72 O) folded columns: every A element fetched from
//     L2 feeds 144 outputs (the round-1 cp.async K1f fed 88), which halves the L2 traffic per DMMA;
//   * the loads of the next tile's first stages are in flight while the consumers run the epilogue.
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
//              rows 16(t>>1) + 2r + (t&1) (r = 0..7) of its 32-row slice;
// the W chunks are laid out per (k4 step, n8 pair, lane) in that same k order.
#include <cuda.h>

#include <type_traits>

#include "../fdp_internal.h"
#include "../mode_tma.h"

namespace fdp {
#ifdef FDP_K1T_PROF
__device__ unsigned long long g_k1t_prof[8][4];
__device__ unsigned long long g_k1t_prof2[8][4];
__device__ unsigned long long g_k1t_wwait[8][32];  // per-warp wait cycles  // wait at stage 0, issue->need slack, issue->ready, count
__shared__ long long t_issue[8];  // [kmaj*4 + fold-1 + 2*(epi!=0)]: wait, kloop, epilogue, tiles
#endif
namespace {

// kWM row slices of 8 kMT rows (kWM * 8 * kMT = kTmaBM) times the two roles
#ifndef FDP_K1T_WM
#define FDP_K1T_WM 4
#endif
constexpr int kWM = FDP_K1T_WM;
constexpr int kMT = kTmaBM / (8 * kWM);
constexpr int kConsumerWarps = 2 * kWM;
constexpr int kThreads = kConsumerWarps * 32;
constexpr int kXR = kMT / 2;  // 8-row tiles per BWD exchange round (two rounds)
constexpr int kABytes = kTmaBM * kTmaBK * 8;             // one A tile (8 KB)
constexpr int kBBytes = kTmaWChunk * 8;                  // one role's W chunk (10 KB)
constexpr int kMiniBytes = kTmaBM * 2 * 8;               // odd-start fix-up column pair (1 KB)
constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes + kMiniBytes;  // 54 KB
constexpr int kEpiBytes = kWM * kXR * 8 * 72 * 8;        // BWD o-exchange, half a tile (36 KB)

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

struct Tile {
  int pi, ct, tp, tq, b;
};

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
// consumer K loop of one tile: NTV = n8 tiles per role (9 or 8; 0 = any nt <= 9, masked),
// ODD = KMAJ second A tile loaded from one column earlier (see the producer)
// ---------------------------------------------------------------------------------------------
template <bool KMAJ, int FOLD, int STAGES, int NTV, int ODD, class Release>
__device__ __forceinline__ void kloop(double (&acc)[kMT][9][2], int nt, int kst, int ne, unsigned sbase,
                                      unsigned bar_full, int& stage, unsigned& phase, int wm,
                                      int role, int fr, int fc, int lane, int it, Release& release,
                                      int pslot = 0) {
  const double sgn = role ? -1.0 : 1.0;  // FWD: E warps form s = x + Jx, O warps d = x - Jx
  for (int s = 0; s < kst; ++s) {
#ifdef FDP_K1T_PROF
    const long long w0 = clock64();
    mbar_wait(bar_full + 8 * stage, phase);
    if (lane == 0) {
      const long long w1 = clock64();
      atomicAdd(&g_k1t_prof[pslot][0], (unsigned long long)(w1 - w0));
      atomicAdd(&g_k1t_wwait[pslot][threadIdx.x >> 5], (unsigned long long)(w1 - w0));

      if (threadIdx.x == 0) {
        atomicAdd(&g_k1t_prof2[pslot][1], (unsigned long long)(w0 - t_issue[stage]));
        atomicAdd(&g_k1t_prof2[pslot][2], (unsigned long long)(w1 - t_issue[stage]));
        atomicAdd(&g_k1t_prof2[pslot][3], 1ULL);
      }
    }
#else
    mbar_wait(bar_full + 8 * stage, phase);
#endif
    const unsigned A0 = sbase + stage * kStageBytes;
    const unsigned A1 = A0 + kABytes;
    const unsigned B = A1 + kABytes + role * kBBytes;
    const unsigned Mini = A1 + kABytes + 2 * kBBytes;
    const int rem = ne - s * kTmaBK;  // valid k of this stage (>= 1)
    const int jmax = KMAJ ? min(4, (rem + 3) >> 2) : (rem <= 8 ? 2 : 4);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j < jmax) {
        double a[kMT];
#pragma unroll
        for (int ti = 0; ti < kMT; ++ti) {
          if (KMAJ) {
            const int R = 8 * kMT * wm + 16 * (ti >> 1) + 2 * fr + (ti & 1);
            const int x = R & 7;
            const int k = 4 * j + fc;
            // column lam of the swizzled [row][16] tile
            auto sw = [&](int lam) { return (unsigned)(R * 128 + ((((lam >> 1) ^ x) << 4) | ((lam & 1) << 3))); };
            // A1 column: FWD the mirror 15 - k, BWD k; shifted by one for an odd-start tile,
            // whose 16th column sits in the 2-column fix-up box
            const int l1 = (FOLD == FOLD_FWD ? kTmaBK - 1 - k : k) + ODD;
            const unsigned a1 = (ODD && l1 == kTmaBK) ? Mini + R * 16 : A1 + sw(l1);
            if (FOLD == FOLD_FWD) {
              const double v = lds64(A0 + sw(k)), w = lds64(a1);
              a[ti] = fma(sgn, w, v);
            } else {
              a[ti] = lds64(role ? a1 : A0 + sw(k));
            }
          } else {
            const int gq = kXR * wm + (ti >> 1), plo = 8 * (ti & 1) + fr;
            const int k = 8 * (j >> 1) + 2 * fc + (j & 1), km = kTmaBK - 1 - k;
            const unsigned off0 = (k + 16 * gq) * 128 + ((((plo >> 1) ^ (k & 7)) << 4) | ((plo & 1) << 3));
            const unsigned off1 = (km + 16 * gq) * 128 + ((((plo >> 1) ^ (km & 7)) << 4) | ((plo & 1) << 3));
            if (FOLD == FOLD_FWD) {
              const double v = lds64(A0 + off0), w = lds64(A1 + off1);
              a[ti] = fma(sgn, w, v);
            } else {
              a[ti] = lds64((role ? A1 : A0) + off0);
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
    release(stage, it, s);
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------------------------
template <bool KMAJ, int FOLD, int STAGES>
__global__ void __launch_bounds__(kThreads, kTmaCtasPerSM) mode_tma_kernel(const __grid_constant__ TmaGroup g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment (shared-window address) for the 128-byte swizzle atoms
  const unsigned sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const unsigned bar_full = sbase + STAGES * kStageBytes + (FOLD == FOLD_BWD ? kEpiBytes : 0);
  const unsigned epi_base = sbase + STAGES * kStageBytes;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // per-slot release counters (see release), after the mbarriers
  int* cnt = reinterpret_cast<int*>(smem_raw + (bar_full + 8 * STAGES - smem_u32(smem_raw)));
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      cnt[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // ------------------------------ producer ------------------------------
  // There is no producer warp: the last consumer warp to release a slot (a per-slot arrival
  // counter in shared memory) issues that slot's refill, STAGES stages ahead in the CTA's tile
  // sequence -- at the earliest moment the slot is free, with no thread waiting for it.
  // issue(it, s): stage s of this CTA's it-th tile into slot `slot`.
  auto issue = [&](int slot, int it, int s) {
    const int tau = tile_of(g, it);
    if (tau < 0) return;
#ifdef FDP_K1T_PROF
    t_issue[slot] = clock64();
#endif
    const Tile t = decode(g, tau, KMAJ);
    const TmaProb& p = g.prob[t.pi];
    const unsigned full = bar_full + 8 * slot;
    const unsigned dA0 = sbase + slot * kStageBytes;
    const unsigned dA1 = dA0 + kABytes;
    const unsigned dB = dA1 + kABytes;
    const int k0 = s * kTmaBK;
    const int k1 = FOLD == FOLD_FWD ? p.n - k0 - kTmaBK : p.ne + k0;
    const CUtensorMap* map = &g.map[t.pi];
    if (KMAJ) {
      // a TMA box must start on a 16-byte boundary: an odd k1 (odd n forward, odd ne backward)
      // loads the 16 columns from k1 - 1 and the last one (k1 + 15) through a 2-column box
      mbar_expect_tx(full, 2 * kABytes + 2 * kBBytes + (p.a1odd ? kMiniBytes : 0));
      tma_load_3d(dA0, map, full, k0, t.tq * kTmaBM, t.b);
      tma_load_3d(dA1, map, full, k1 - p.a1odd, t.tq * kTmaBM, t.b);
      if (p.a1odd) tma_load_3d(dB + 2 * kBBytes, &g.map2[t.pi], full, k1 + 15, t.tq * kTmaBM, t.b);
    } else {
      mbar_expect_tx(full, 2 * kABytes + 2 * kBBytes);
#ifdef FDP_K1T_PROF
      if (g.dbg & 2) {  // timing experiment: A tiles of row tile 0 only (wrong results)
        tma_load_5d(dA0, map, full, 0, k0, 0, 0, 0);
        tma_load_5d(dA1, map, full, 0, k1, 0, 0, 0);
      } else
#endif
      {
      tma_load_5d(dA0, map, full, 0, k0, t.tp * p.bp, t.tq * p.bq, t.b);
      tma_load_5d(dA1, map, full, 0, k1, t.tp * p.bp, t.tq * p.bq, t.b);
      }
    }
    const double* wE = p.Wt + (size_t)((0 * p.ctiles + t.ct) * p.kst + s) * kTmaWChunk;
    const double* wO = p.Wt + (size_t)((1 * p.ctiles + t.ct) * p.kst + s) * kTmaWChunk;
#ifdef FDP_K1T_PROF
    if (g.dbg & 1) {  // timing experiment: W chunks of stage 0 only (wrong results)
      wE = p.Wt;
      wO = p.Wt + kTmaWChunk;
    }
#endif
    bulk_load(dB, wE, kBBytes, full);
    bulk_load(dB + kBBytes, wO, kBBytes, full);
  };
  // release(slot, it, s): this warp is done with stage s of tile `it` (held in `slot`)
  auto release = [&](int slot, int it, int s) {
#ifndef FDP_K1T_ASYNC
    // every warp finishes the stage together (measured faster than letting warps run ahead
    // through the ring: the sub-partition arbiter favours high warp ids, the leaders then stall
    // on refills gated by the slowest warp while the laggards run alone)
#ifdef FDP_K1T_PROF
    const long long b0 = clock64();
    named_bar(15, kThreads);
    if (lane == 0) atomicAdd(&g_k1t_prof2[0][0], (unsigned long long)(clock64() - b0));
#else
    named_bar(15, kThreads);
#endif
    if (threadIdx.x == 0) {
      {
#else
    __syncwarp();
    if (lane == 0) {
      if (atomicAdd(&cnt[slot], 1) == kConsumerWarps - 1) {
#endif
        cnt[slot] = 0;
        // advance STAGES stages through the tile sequence
        int it2 = it, s2 = s + STAGES;
        for (int tau = tile_of(g, it2); tau >= 0; tau = tile_of(g, it2)) {
          const int kst = g.prob[decode(g, tau, KMAJ).pi].kst;
          if (s2 < kst) break;
          s2 -= kst;
          ++it2;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // reads before TMA writes
        issue(slot, it2, s2);
      }
    }
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < g.count; ++i)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&g.map[i]))
                   : "memory");
    // prologue: the first STAGES stages
    int it = 0, s = 0;
    for (int i = 0; i < STAGES; ++i) {
      const int tau = tile_of(g, it);
      if (tau < 0) break;
      issue(i, it, s);
      if (++s == g.prob[decode(g, tau, KMAJ).pi].kst) {
        s = 0;
        ++it;
      }
    }
  }

  // ------------------------------ consumers ------------------------------
  const int wm = warp % kWM, role = warp / kWM;  // role 0: E, 1: O
  const int fr = lane >> 2, fc = lane & 3;
  int stage = 0;
  unsigned phase = 0;

  // per-thread fragment offsets within an A tile (bytes, before the j-dependent part)
  //   non-KMAJ: rows of DMMA tile t are p_lo = 8(t&1) + fr of the 16-row group g = 2 wm + (t>>1);
  //             byte = (k + 16 g) * 128 + swz(p_lo, k)
  //   KMAJ:     rows R = 32 wm + 16 (t>>1) + 2 fr + (t&1); byte = R * 128 + swz(k, R)
  for (int it = 0;; ++it) {
    const int tau = tile_of(g, it);
    if (tau < 0) break;
    const Tile t = decode(g, tau, KMAJ);
    const TmaProb& p = g.prob[t.pi];
    // n8 tiles of this column tile (same count for both roles; the O half's extra column, if
    // any, multiplies zero W columns)
    const int nbase = p.n8h / p.ctiles, nrem = p.n8h % p.ctiles;
    const int nt = nbase + (t.ct < nrem ? 1 : 0);
    const int nt0 = t.ct * nbase + min(t.ct, nrem);

    double acc[kMT][9][2];
#pragma unroll
    for (int i = 0; i < kMT; ++i)
#pragma unroll
      for (int u = 0; u < 9; ++u) acc[i][u][0] = acc[i][u][1] = 0.0;

#ifdef FDP_K1T_PROF
    const long long tk0 = clock64();
#endif
    // the K loop, specialised on the column tile's n8 count (no per-DMMA predicate: a predicated
    // mma.sync costs a WARPSYNC + NOP pair) and, for KMAJ, on the odd-start second A tile
    const int odd = KMAJ ? p.a1odd : 0;
    auto run = [&](auto ntv, auto oddv) {
      kloop<KMAJ, FOLD, STAGES, decltype(ntv)::value, decltype(oddv)::value>(
          acc, nt, p.kst, p.ne, sbase, bar_full, stage, phase, wm, role, fr, fc, lane, it, release,
          KMAJ * 4 + (FOLD - 1) + 2 * (p.epi != 0));
    };
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    if (nt == 9) {
      if (odd) run(std::integral_constant<int, 9>{}, I1{}); else run(std::integral_constant<int, 9>{}, I0{});
    } else if (nt == 8) {
      if (odd) run(std::integral_constant<int, 8>{}, I1{}); else run(std::integral_constant<int, 8>{}, I0{});
    } else {
      if (odd) run(I0{}, I1{}); else run(I0{}, I0{});
    }

#ifdef FDP_K1T_PROF
    const long long e0 = clock64();
    if (lane == 0) atomicAdd(&g_k1t_prof[KMAJ * 4 + (FOLD - 1) + 2 * (p.epi != 0)][1], (unsigned long long)(e0 - tk0));
#endif
    // ------------------------------ epilogue ------------------------------
    // row r (0..31 of this warp's slice) of DMMA tile ti: see the fragment-offset comment above
    auto row_of = [&](int ti, long long& yoff, long long& sidx, int& pp, bool& valid) {
      if (KMAJ) {
        const int R = 8 * kMT * wm + 16 * (ti >> 1) + 2 * fr + (ti & 1);
        const long long q = (long long)t.tq * kTmaBM + R;
        valid = q < p.Q;
        sidx = (long long)p.yld * q;
        yoff = sidx + p.ybs * t.b;
        pp = 0;
      } else {
        const int gq = kXR * wm + (ti >> 1);
        const int plo = 8 * (ti & 1) + fr;
        const int ph = t.tp * p.bp + gq % p.bp;
        const long long q = (long long)t.tq * p.bq + gq / p.bp;
        pp = 16 * ph + plo;
        valid = pp < p.P && q < p.Q;
        sidx = pp + (long long)p.P * p.n * q;
        yoff = sidx + p.ybs * t.b;
      }
    };
    const long long cs = KMAJ ? 1 : p.P;  // column stride of the output
    if (FOLD == FOLD_FWD) {
      const int cval = role ? p.no : p.ne;
      const int coff = role ? p.ne : 0;
#pragma unroll
      for (int ti = 0; ti < kMT; ++ti) {
        long long yoff, sidx;
        int pp;
        bool valid;
        row_of(ti, yoff, sidx, pp, valid);
        if (!valid) continue;
        double lrow = 0.0;
        bool pad_row = false;
        if (p.epi == EPI_LAMBDA) {  // non-KMAJ (the last mode): p = i1 + n1p * i2
          const int i1 = pp % p.n1;
          pad_row = i1 >= p.n1v;
          if (!pad_row) lrow = p.lam1 ? p.lam0[i1] + p.lam1[pp / p.n1] : p.lam0[pp];
        }
#pragma unroll
        for (int u = 0; u < 9; ++u) {
          if (u < nt) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int a = 8 * (nt0 + u) + 2 * fc + h;
              const int oc = coff + a;
              if (a < cval) {
                double v = acc[ti][u][h];
                if (p.epi == EPI_LAMBDA) v = pad_row ? 0.0 : fdp_div(v, lrow + p.lamcol[oc]);
                p.Y[yoff + cs * oc] = v;
              } else if (KMAJ && role && oc < p.yld) {
                p.Y[yoff + oc] = 0.0;  // the zero pad column of a padded KMAJ output row
              }
            }
          }
        }
      }
    } else {
      // FOLD_BWD: O warps pass o through shared memory (two halves of 16 rows), E warps store
      // x_c = e + o and x_{n-1-c} = e - o
      const unsigned ex = epi_base + wm * (kXR * 8 * 72 * 8);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        if (role) {
#pragma unroll
          for (int tt = 0; tt < kXR; ++tt) {
            const int ti = kXR * half + tt;
#pragma unroll
            for (int u = 0; u < 9; ++u)
              if (u < nt) sts128(ex + ((8 * tt + fr) * 72 + 8 * u + 2 * fc) * 8, acc[ti][u][0], acc[ti][u][1]);
          }
        }
        named_bar(1 + wm, 64);
        if (!role) {
#pragma unroll
          for (int tt = 0; tt < kXR; ++tt) {
            const int ti = kXR * half + tt;
            long long yoff, sidx;
            int pp;
            bool valid;
            row_of(ti, yoff, sidx, pp, valid);
            if (!valid) continue;
#pragma unroll
            for (int u = 0; u < 9; ++u) {
              if (u < nt) {
                double o0, o1;
                lds128(ex + ((8 * tt + fr) * 72 + 8 * u + 2 * fc) * 8, o0, o1);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  const int c = 8 * (nt0 + u) + 2 * fc + h;
                  if (c < p.ne) {
                    const double e = acc[ti][u][h], o = h ? o1 : o0;
                    double v0 = e + o, v1 = e - o;
                    const int cm = p.n - 1 - c;
                    if (p.epi == EPI_SCALE) {
                      v0 *= p.scale[sidx + cs * c];
                      v1 *= p.scale[sidx + cs * cm];
                    }
                    p.Y[yoff + cs * c] = v0;
                    if (cm != c) p.Y[yoff + cs * cm] = v1;
                  }
                }
              }
            }
          }
        }
        named_bar(1 + wm, 64);
      }
    }
#ifdef FDP_K1T_PROF
    if (lane == 0) {
      atomicAdd(&g_k1t_prof[KMAJ * 4 + (FOLD - 1) + 2 * (p.epi != 0)][2], (unsigned long long)(clock64() - e0));
      atomicAdd(&g_k1t_prof[KMAJ * 4 + (FOLD - 1) + 2 * (p.epi != 0)][3], 1ULL);
    }
#endif
  }
}

template <bool KMAJ, int FOLD, int STAGES>
constexpr size_t smem_bytes() {
  return 1024 + (size_t)STAGES * kStageBytes + (FOLD == FOLD_BWD ? kEpiBytes : 0) + 16 * STAGES + 16;
}

#ifndef FDP_K1T_SF
#define FDP_K1T_SF 3
#endif
#ifndef FDP_K1T_SB
#define FDP_K1T_SB 2
#endif
constexpr int kStagesFwd = FDP_K1T_SF;
constexpr int kStagesBwd = FDP_K1T_SB;

template <bool KMAJ, int FOLD, int STAGES>
cudaError_t launch_t(const TmaGroup& g, int grid, cudaStream_t s) {
  constexpr size_t sm = smem_bytes<KMAJ, FOLD, STAGES>();
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

}  // namespace

cudaError_t prepare_mode_tma() {
  // set the shared-memory attributes outside any stream capture
  const int fwd = (int)smem_bytes<true, FOLD_FWD, kStagesFwd>();
  const int bwd = (int)smem_bytes<true, FOLD_BWD, kStagesBwd>();
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(mode_tma_kernel<true, FOLD_FWD, kStagesFwd>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, fwd)) ||
      (e = cudaFuncSetAttribute(mode_tma_kernel<false, FOLD_FWD, kStagesFwd>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, fwd)) ||
      (e = cudaFuncSetAttribute(mode_tma_kernel<true, FOLD_BWD, kStagesBwd>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, bwd)) ||
      (e = cudaFuncSetAttribute(mode_tma_kernel<false, FOLD_BWD, kStagesBwd>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, bwd)))
    return e;
  return cudaSuccess;
}

cudaError_t launch_mode_tma(const TmaGroup& g, bool kmaj, int fold, int grid, cudaStream_t s) {
  if (g.total_tiles <= 0) return cudaSuccess;
  if (fold == FOLD_FWD)
    return kmaj ? launch_t<true, FOLD_FWD, kStagesFwd>(g, grid, s)
                : launch_t<false, FOLD_FWD, kStagesFwd>(g, grid, s);
  if (fold == FOLD_BWD)
    return kmaj ? launch_t<true, FOLD_BWD, kStagesBwd>(g, grid, s)
                : launch_t<false, FOLD_BWD, kStagesBwd>(g, grid, s);
  return cudaErrorInvalidValue;
}

}  // namespace fdp

// ---------------------------------------------------------------------------------------------
// Row padding for K1t's first pass: y (rows of n1p, pad entries zero) <- x (rows of n1), batch
// items at strides xbs / ybs. HBM streaming (16 B per element); used only when the C-ABI input
// cannot be read through a tensor map (odd row length or a base not 16-byte aligned).
// ---------------------------------------------------------------------------------------------
namespace fdp {
namespace {
__global__ void pad_rows_kernel(const double* __restrict__ x, long long xbs, double* __restrict__ y,
                                long long ybs, int n1, int n1p, long long rows, long long batch) {
  const long long per = rows * n1p, total = per * batch;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / per, j = i - b * per;
    const long long r = j / n1p;
    const int c = (int)(j - r * n1p);
    y[b * ybs + j] = c < n1 ? x[b * xbs + r * n1 + c] : 0.0;
  }
}
}  // namespace

cudaError_t launch_pad_rows(const double* x, long long xbs, double* y, long long ybs, int n1,
                            int n1p, long long rows, long long batch, cudaStream_t s) {
  const long long total = rows * n1p * batch;
  if (total == 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = (int)std::min<long long>((total + 255) / 256, (long long)sms * 8);
  pad_rows_kernel<<<blocks, 256, 0, s>>>(x, xbs, y, ybs, n1, n1p, rows, batch);
  return cudaGetLastError();
}
}  // namespace fdp

#ifdef FDP_K1T_PROF
extern "C" void fdp_k1t_prof(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, fdp::g_k1t_prof, sizeof(unsigned long long) * 32);
  cudaMemcpyFromSymbol(out + 32, fdp::g_k1t_prof2, sizeof(unsigned long long) * 32);
  cudaMemcpyFromSymbol(out + 64, fdp::g_k1t_wwait, sizeof(unsigned long long) * 256);
  if (reset) {
    unsigned long long z[32] = {0};
    cudaMemcpyToSymbol(fdp::g_k1t_prof2, z, sizeof(z));
    unsigned long long z2[256] = {0};
    cudaMemcpyToSymbol(fdp::g_k1t_wwait, z2, sizeof(z2));
    cudaMemcpyToSymbol(fdp::g_k1t_prof, z, sizeof(z));
  }
}
#endif
