// Host side of K1t (kernels/mode_tma.cu): the fragment-native eigenvector chunks built at setup,
// the tensor maps encoded per launch, and the grouping of folded K1 problems into one persistent
// TMA launch. DESIGN.md §5 "K1t".
#include <atomic>

#include "abi_impl.h"

namespace fdp {

std::atomic<long long> g_k1_launches[2];

int tma_ctiles(int ne) {
  const int n8h = (ne + 7) / 8;
  return (n8h + kTmaMaxNT - 1) / kTmaMaxNT;
}

// Fragment-native chunks of a folded transform (FOLD_FWD: wf of fold_eig, FOLD_BWD: wb), rows E
// [0, foldh) and O [foldh, 2 foldh), ldw columns. Layout [role][ctile][stage][j][pair][lane][2]:
// lane (r, c) = (lane >> 2, lane & 3) of k4 step j holds W_role[k][a] with
//   k = 16 stage + (kmaj ? 4 j + c : 8 (j >> 1) + 2 c + (j & 1)),
//   a = 8 (nt0(ctile) + 2 pair + h) + r,
// zero outside k < (E: ne, O: no), a < (E: ne, O: no) and the column tile's n8 count.
std::vector<double> tma_wt_build(int n, int foldh, int ldw, const std::vector<double>& w, bool kmaj) {
  const int ne = (n + 1) / 2, no = n / 2;
  const int n8h = (ne + 7) / 8, CT = tma_ctiles(ne), KS = (ne + kTmaBK - 1) / kTmaBK;
  const int nbase = n8h / CT, nrem = n8h % CT;
  std::vector<double> out((size_t)2 * CT * KS * kTmaWChunk, 0.0);
  for (int role = 0; role < 2; ++role) {
    const int kv = role ? no : ne, av = role ? no : ne, r0 = role ? foldh : 0;
    for (int ct = 0; ct < CT; ++ct) {
      const int nt = nbase + (ct < nrem ? 1 : 0), nt0 = ct * nbase + std::min(ct, nrem);
      for (int s = 0; s < KS; ++s) {
        double* o = out.data() + (size_t)((role * CT + ct) * KS + s) * kTmaWChunk;
        for (int j = 0; j < 4; ++j)
          for (int pr = 0; pr < 5; ++pr)
            for (int lane = 0; lane < 32; ++lane)
              for (int h = 0; h < 2; ++h) {
                const int u = 2 * pr + h, r = lane >> 2, c = lane & 3;
                const bool nat = kmaj || (s == KS - 1 && tma_last_nat(ne, false));
                const int k = kTmaBK * s + (nat ? 4 * j + c : 8 * (j >> 1) + 2 * c + (j & 1));
                const int a = 8 * (nt0 + u) + r;
                double v = 0.0;
                if (u < nt && k < kv && a < av) v = w[(size_t)(r0 + k) * ldw + a];
                o[((j * 5 + pr) * 32 + lane) * 2 + h] = v;
              }
      }
    }
  }
  return out;
}

namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return (EncodeFn) nullptr;
    }
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

CUtensorMapL2promotion promotion() { return CU_TENSOR_MAP_L2_PROMOTION_L2_256B; }

}  // namespace

// A tensor map can describe the A operand (else: the first pass's input is row-padded first).
bool tma_input_ok(const ModeProb& p, bool kmaj) {
  if (!aligned16(p.X)) return false;
  if (p.batch > 1 && (p.xbs & 1)) return false;
  return kmaj ? (p.xld % 2 == 0) : (p.P % 2 == 0);
}

// The folded K1 problems of one grouped stage can run on K1t.
bool tma_eligible(const ModeProb& p, bool kmaj) {
  if (std::getenv("FDP_NO_TMA")) return false;
  if (!p.Wt || !p.fold_k1 || p.tio) return false;
  // K1t scatters from non-KMAJ batch-1 stores, a lane's row pair contiguous and 16-byte aligned in
  // the owner's buffer (sc_n1 even)
  if (p.peers && (kmaj || p.batch != 1 || (p.sc_n1 & 1))) return false;
  if (p.fold != FOLD_FWD && p.fold != FOLD_BWD) return false;
  if (p.fold == FOLD_FWD && p.epi != EPI_NONE && p.epi != EPI_LAMBDA) return false;
  if (kmaj && p.epi == EPI_LAMBDA) return false;  // Lambda^{-1} is applied on the non-KMAJ store path
  if (p.fold == FOLD_BWD && p.epi != EPI_NONE && p.epi != EPI_SCALE) return false;
  if (p.nout != p.n || p.n < 8) return false;
  if (kmaj && p.P != 1) return false;
  if ((long long)p.Q * p.batch >= (1LL << 31)) return false;
  return encoder() != nullptr;
}

bool mass_tile_map(CUtensorMap* map, const double* X, int P, int n, long long Q, long long batch, long long bs,
                   int F, int boxn) {
  EncodeFn enc = encoder();
  if (!enc || !aligned16(X) || (P & 1) || (F & 1) || boxn < 1 || boxn > 256) return false;
  const unsigned long long qstride = (unsigned long long)P * n * 8;
  const unsigned long long bstride = batch > 1 ? (unsigned long long)bs * 8 : qstride * Q + 16;
  if (bstride & 15) return false;
  cuuint64_t dims[4] = {(cuuint64_t)P, (cuuint64_t)n, (cuuint64_t)Q, (cuuint64_t)batch};
  cuuint64_t strides[3] = {(cuuint64_t)P * 8, qstride, (cuuint64_t)(bstride & ~15ULL)};
  cuuint32_t box[4] = {(cuuint32_t)F, (cuuint32_t)boxn, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(X), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promotion(),
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_tma_stage(const ModeProb* probs, int count, bool kmaj, cudaStream_t s) {
  if (count < 1 || count > kTmaMaxProbs) return cudaErrorInvalidValue;
  EncodeFn enc = encoder();
  if (!enc) return cudaErrorNotSupported;
  TmaGroup g;
  std::memset(&g, 0, sizeof(g));
  g.count = count;
  int tiles = 0;
  const int fold = probs[0].fold;

  for (int i = 0; i < count; ++i) {
    const ModeProb& m = probs[i];
    if (m.fold != fold) return cudaErrorInvalidValue;
    TmaProb& t = g.prob[i];
    t.Wt = m.Wt;
    t.Y = m.Y;
    t.scale = m.scale;
    t.lam0 = m.lam0;
    t.lam1 = m.lam1;
    t.lamcol = m.lamcol;
    t.peers = m.peers;
    t.sc_G = m.sc_G;
    t.sc_na = m.sc_na;
    t.sc_n1 = m.sc_n1;
    t.sc_qoff = m.sc_qoff;
    t.sc_a0 = m.sc_a0;
    t.sc_a1 = m.sc_a1;
    t.sc_q0 = m.sc_q0;
    t.sc_q1 = m.sc_q1;
    t.rlam = m.rlam;
    t.ybs = m.ybs;
    t.n = m.n;
    t.ne = (m.n + 1) / 2;
    t.no = m.n / 2;
    t.n8h = (t.ne + 7) / 8;
    t.ctiles = tma_ctiles(t.ne);
    t.kst = (t.ne + kTmaBK - 1) / kTmaBK;
    t.P = m.P;
    t.Q = m.Q;
    t.yld = m.yld;
    t.n1 = m.n1;
    t.n1v = m.n1v;
    t.epi = m.epi;
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r;
    if (kmaj) {
      t.bp = t.bq = 1;
      t.tiles_p = 1;
      t.tiles_q = (m.Q + kTmaBM - 1) / kTmaBM;
      const unsigned long long bstride =
          m.batch > 1 ? (unsigned long long)m.xbs * 8 : (unsigned long long)m.xld * m.Q * 8 + 16;
      cuuint64_t dims[3] = {(cuuint64_t)m.n, (cuuint64_t)m.Q, (cuuint64_t)m.batch};
      cuuint64_t strides[2] = {(cuuint64_t)m.xld * 8, (cuuint64_t)(bstride & ~15ULL)};
      cuuint32_t box[3] = {(cuuint32_t)kTmaBK, (cuuint32_t)kTmaBM, 1};
      r = enc(&g.map[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(m.X), dims, strides,
              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      // a box starts on a 16-byte boundary: an odd first column of the second A tile (mirror of
      // an odd n, O part after an odd ne) is read from one column earlier plus a 2-column box
      t.a1odd = (m.fold == FOLD_FWD ? (m.n & 1) : (t.ne & 1));
      cuuint32_t box2[3] = {2, (cuuint32_t)kTmaBM, 1};
      if (r == CUDA_SUCCESS)
        r = enc(&g.map2[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(m.X), dims, strides,
                box2, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      const int PH = (m.P + 15) / 16;
      // row-tile shape: bp 16-row p-groups x bq q-lines (bp bq = kTmaBM / 16), the fewest tiles
      long long best = -1;
      for (int bp = kTmaBM / 16; bp >= 1; bp /= 2) {
        const int bq = kTmaBM / 16 / bp;
        const long long nt = (long long)((PH + bp - 1) / bp) * ((m.Q + bq - 1) / bq);
        if (best < 0 || nt < best) {
          best = nt;
          t.bp = bp;
          t.bq = bq;
        }
      }
      t.tiles_p = (PH + t.bp - 1) / t.bp;
      t.tiles_q = (m.Q + t.bq - 1) / t.bq;
      const unsigned long long qstride = (unsigned long long)m.P * m.n * 8;
      const unsigned long long bstride = m.batch > 1 ? (unsigned long long)m.xbs * 8 : qstride * m.Q + 16;
      cuuint64_t dims[5] = {16, (cuuint64_t)m.n, (cuuint64_t)PH, (cuuint64_t)m.Q, (cuuint64_t)m.batch};
      cuuint64_t strides[4] = {(cuuint64_t)m.P * 8, 128, qstride, (cuuint64_t)(bstride & ~15ULL)};
      cuuint32_t box[5] = {16, (cuuint32_t)kTmaBK, (cuuint32_t)t.bp, (cuuint32_t)t.bq, 1};
      r = enc(&g.map[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double*>(m.X), dims, strides,
              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    if (m.epi == EPI_LAMBDA && !m.rlam) {  // Lambda factors staged in shared memory: lam0 (n1), lam1 (P / n1), lamcol (n)
      t.lam_off = g.lam_elems;
      t.lam1_n = m.lam1 ? m.P / m.n1 : 0;
      g.lam_elems += m.n1 + t.lam1_n + m.n;
    }
    t.tile_begin = tiles;
    tiles += t.ctiles * t.tiles_p * t.tiles_q * m.batch;
  }
  if (g.lam_elems > 4800) return cudaErrorInvalidValue;  // kLamMax of mode_tma.cu
  g.total_tiles = tiles;
  g.ct_uniform = g.prob[0].ctiles;
  for (int i = 1; i < count; ++i)
    if (g.prob[i].ctiles != g.ct_uniform) g.ct_uniform = 0;
  int grid = std::min(tiles, kTmaCtasPerSM * num_sms());
  if (g.ct_uniform > 0) grid = std::max(g.ct_uniform, grid / g.ct_uniform * g.ct_uniform);
  g.prof_slot = (int)(g_k1_launches[1].load() & 7);
  ++g_k1_launches[1];
  return launch_mode_tma(g, kmaj, fold, grid, s);
}

}  // namespace fdp

extern "C" int64_t fdp_debug_k1_launches(int tma) { return fdp::g_k1_launches[tma ? 1 : 0].load(); }
