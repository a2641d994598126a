// Launch-latency probe: per-kernel time of back-to-back dependent launches (stream and CUDA
// graph), for an empty kernel and for kernels with large dynamic shared memory, with and without
// programmatic dependent launch. Diagnostic only.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

__global__ void empty_k(int* p) { if (p && threadIdx.x == 1234567) p[0] = 1; }
__global__ void smem_k(int* p) {
  extern __shared__ double sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (p && sm[threadIdx.x] == -1.0) p[0] = 1;
}
__global__ void pdl_k(int* p) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  extern __shared__ double sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (p && sm[threadIdx.x] == -1.0) p[0] = 1;
}

template <class F>
float time_graph(cudaStream_t s, F enqueue, int n) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) { printf("begin fail\n"); return -1; }
  for (int i = 0; i < n; ++i) enqueue();
  cudaError_t e = cudaStreamEndCapture(s, &g);
  if (e != cudaSuccess) { printf("end capture fail %s\n", cudaGetErrorString(e)); fflush(stdout); return -1; }
  e = cudaGraphInstantiate(&ge, g, 0);
  if (e != cudaSuccess) { printf("inst fail %s\n", cudaGetErrorString(e)); fflush(stdout); return -1; }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEventRecord(a, s);
  for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  fflush(stdout);
  return ms * 1e3f / (10 * n);
}

int main() {
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  int* d;
  CK(cudaMalloc(&d, 4));
  const int N = 100;
  for (int smem : {4096, 48 * 1024, 180 * 1024}) {
    CK(cudaFuncSetAttribute(smem_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(pdl_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (int grid : {1, 148, 444}) {
      float t1 = time_graph(s, [&] { smem_k<<<grid, 256, smem, s>>>(d); }, N);
      float t2 = time_graph(s, [&] {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, pdl_k, d);
      }, N);
      fflush(stdout);
      printf("{\"smem\": %d, \"grid\": %d, \"graph_us_per_kernel\": %.2f, \"graph_pdl_us_per_kernel\": %.2f}\n", smem, grid, t1, t2);
    }
  }
  float t0 = time_graph(s, [&] { empty_k<<<1, 32, 0, s>>>(d); }, N);
  printf("{\"empty_graph_us_per_kernel\": %.2f}\n", t0);
  CK(cudaGetLastError());
  return 0;
}
