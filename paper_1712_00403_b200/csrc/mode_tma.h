// K1t (kernels/mode_tma.cu): the TMA-fed, warp-specialised even-odd folded FD transform.
// Shared by the kernel and the host orchestration (abi.cpp); nothing here crosses the C ABI.
#pragma once

#include <cuda.h>

#include "fdp_internal.h"

namespace fdp {

constexpr int kTmaBM = 64;             // rows of a CTA tile
constexpr int kTmaCtasPerSM = 1;       // one persistent CTA per SM (DESIGN.md §5 "K1t")
constexpr int kTmaBK = 16;             // k per pipeline stage
constexpr int kTmaMaxNT = 9;           // n8 tiles per role and column tile
constexpr int kTmaWChunk = 4 * 5 * 32 * 2;  // doubles of one role's W chunk per stage
constexpr int kTmaMaxProbs = 4;

// The last (partial) K stage of a non-KMAJ problem takes the natural k order k = 4 j + c (one k4
// step per 4 valid k) instead of the bank-conflict-free order k = 8 (j >> 1) + 2 c + (j & 1)
// (one k4 step pair per 8) when that saves a k4 step: valid k in the stage (rem = ne - 16 (KS - 1))
// of 1-4 or 9-12. KMAJ stages always use the natural order.
inline __host__ __device__ bool tma_last_nat(int ne, bool kmaj) {
  const int rem = ne - kTmaBK * ((ne + kTmaBK - 1) / kTmaBK - 1);
  return !kmaj && ((rem - 1) & 7) < 4;
}

// One folded transform problem of a grouped launch.
//   A operand (read by TMA through map[i]):
//     KMAJ (mode 1): 3-D map {n (k, contiguous), Q (rows, stride xld), batch (stride xbs)},
//       box {16, kTmaBM, 1}; a row tile = kTmaBM consecutive rows of one batch item.
//     otherwise: 5-D map {16 (p_lo), n (k, stride P), ceil(P/16) (p_hi, stride 16), Q (stride
//       P n), batch (stride xbs)}, box {16, 16, bp, bq, 1} with bp * bq = kTmaBM / 16; a row tile = bp
//       16-row p-groups times bq q-lines. Rows p >= P of the last p-group alias the next k line
//       (read, computed, never stored).
//   Wt: fragment-native folded eigenvector chunks, [role E/O][ctile][stage][j 4][n8 pair 5]
//       [lane 32][2] (tmat_build in abi.cpp).
//   Output Y as ModeProb (KMAJ row stride yld; otherwise column stride P), epilogues EPI_NONE,
//   EPI_LAMBDA (forward) or EPI_SCALE (backward).
struct TmaProb {
  const double* Wt;
  double* Y;
  const double* scale;
  const double* lam0;
  const double* lam1;
  const double* lamcol;
  const double* rlam;   // EPI_LAMBDA: 1 / Lambda in the output layout (NULL: divide on the fly)
  long long ybs;
  int n, ne, no, n8h, ctiles, kst;
  int P, Q, bp, bq, tiles_p, tiles_q;
  int yld, n1, n1v, epi;
  int a1odd;      // KMAJ: the second A tile starts at an odd column (odd n FWD / odd ne BWD)
  int lam_off, lam1_n;  // EPI_LAMBDA: offset of this problem's staged factors, length of lam1
  int tile_begin;
  // peer-store scatter of a non-KMAJ, batch-1 problem (the slab exchange fused into the store,
  // DESIGN.md §9; same addressing as ModeProb / scatter_ptr); peers == NULL: store into Y
  double* const* peers;
  int sc_G, sc_na, sc_n1, sc_qoff, sc_a0, sc_a1, sc_q0, sc_q1;
};

struct TmaGroup {
  CUtensorMap map[kTmaMaxProbs];
  CUtensorMap map2[kTmaMaxProbs];  // KMAJ: the same tensor, box {2, kTmaBM, 1}, no swizzle
  TmaProb prob[kTmaMaxProbs];
  int count;
  int total_tiles;
  int ct_uniform;  // column tiles of every problem when equal (grid a multiple of it), else 0
  int lam_elems;   // doubles of staged Lambda factors (0: none)
  int prof_slot;   // diagnostic build (FDP_K1T_PROF): K1t launch ordinal mod 8
};

cudaError_t launch_mode_tma(const TmaGroup& g, bool kmaj, int fold, int grid, cudaStream_t s);
cudaError_t prepare_mode_tma();

}  // namespace fdp
