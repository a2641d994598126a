// Probe: may a tiled TMA box (cp.async.bulk.tensor) start at an arbitrary (odd) element
// coordinate, with and without the 128-byte swizzle, and with a tensor map whose base is offset
// by one element from a 16-byte boundary? Loads boxes {16, 8} of an FP64 [rows][cols] array at
// several start columns and compares shared memory with the expected (un)swizzled contents.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void load_box(const __grid_constant__ CUtensorMap map, int c0, int c1, double* out) {
  __shared__ __align__(1024) double sm[16 * 8];
  __shared__ __align__(8) unsigned long long bar;
  const unsigned sb = (unsigned)__cvta_generic_to_shared(sm), bb = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(16 * 8 * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(sb),
        "l"(reinterpret_cast<unsigned long long>(&map)), "r"(c0), "r"(c1), "r"(bb)
        : "memory");
  }
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(bb)
      : "memory");
  for (int i = threadIdx.x; i < 128; i += blockDim.x) out[i] = sm[i];
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(p);
  const int rows = 64, cols = 518;  // row stride 4144 B (a multiple of 16)
  std::vector<double> h((size_t)rows * cols + 2);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, 128 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  int bad_total = 0;
  for (int base_off = 0; base_off < 2; ++base_off) {
    for (int sw = 0; sw < 2; ++sw) {
      CUtensorMap map;
      // base_off = 1: the map's base is d + 0 (aligned) and element (r, c) of the array starting
      // at d + 1 is read at column c + 1 (the coordinate shift of an unaligned C-ABI input)
      cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
      cuuint64_t str[1] = {(cuuint64_t)cols * 8};
      cuuint32_t box[2] = {16, 8}, es[2] = {1, 1};
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", (int)r);
        return 1;
      }
      const int starts[] = {0, 1, 3, 259, 260, 503, 510};
      for (int c0 : starts) {
        const int r0 = 5;
        const int c = c0 + base_off;
        load_box<<<1, 128>>>(map, c, r0, o);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("launch error %s\n", cudaGetErrorString(e));
          return 1;
        }
        double got[128];
        cudaMemcpy(got, o, sizeof(got), cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int rr = 0; rr < 8; ++rr)
          for (int cc = 0; cc < 16; ++cc) {
            // 128B swizzle: 16-byte chunk index (cc / 2) xor (row & 7) within the 128-byte row
            const int chunk = sw ? ((cc >> 1) ^ (rr & 7)) : (cc >> 1);
            const double v = got[rr * 16 + chunk * 2 + (cc & 1)];
            const int col = c + cc;
            const double want = col < cols ? h[(size_t)(r0 + rr) * cols + col] : 0.0;
            if (v != want) ++bad;
          }
        printf("base_off %d swizzle %d start col %d: %s (%d wrong)\n", base_off, sw, c, bad ? "MISMATCH" : "ok", bad);
        bad_total += bad;
      }
    }
  }
  printf("tma_odd %s\n", bad_total ? "FAIL" : "PASS");
  return 0;
}
