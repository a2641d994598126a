// C ABI: vector kernels of the GPU-resident Krylov drivers (MINRES / GMRES, NEXT-1 / NEXT-2).
#include "abi_impl.h"

// ------------------------------------------------------------------------------------------------
// vector kernels
// ------------------------------------------------------------------------------------------------
static double* dot_scratch(int dev) {
  static double* scratch[64] = {nullptr};
  if (dev < 0 || dev >= 64) return nullptr;
  if (!scratch[dev] && cudaMalloc(&scratch[dev], dot_scratch_doubles() * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    scratch[dev] = nullptr;
  }
  return scratch[dev];
}

extern "C" fdp_status fdp_vec_dot(const double* x, const double* y, int64_t n, double* result,
                                  void* stream) {
  try {
    if (n < 0) return fail(FDP_ERR_SHAPE, "fdp_vec_dot: n < 0");
    if (!is_device_ptr(result) || (n > 0 && (!is_device_ptr(x) || !is_device_ptr(y))))
      return fail(FDP_ERR_INVALID_ARG, "fdp_vec_dot: device pointers required");
    int dev = 0;
    cudaGetDevice(&dev);
    double* sc = dot_scratch(dev);
    if (!sc) return fail(FDP_ERR_OOM, "fdp_vec_dot: scratch");
    FDP_CUDA(launch_dot(x, y, n, result, sc, static_cast<cudaStream_t>(stream)), "fdp_vec_dot");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_vec_lincomb(double a, const double* x, double b, const double* y,
                                      double c, const double* z, double* out, int64_t n,
                                      void* stream) {
  try {
    if (n < 0) return fail(FDP_ERR_SHAPE, "fdp_vec_lincomb: n < 0");
    if (n == 0) return FDP_OK;
    if (!is_device_ptr(x) || !is_device_ptr(out) || (y && !is_device_ptr(y)) || (z && !is_device_ptr(z)))
      return fail(FDP_ERR_INVALID_ARG, "fdp_vec_lincomb: device pointers required");
    FDP_CUDA(launch_lincomb(a, x, b, y, c, z, out, n, static_cast<cudaStream_t>(stream)), "fdp_vec_lincomb");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_vec_lincomb_dev(const double* coef, const double* x, const double* y,
                                          const double* z, double* out, int64_t n, void* stream) {
  try {
    if (n < 0) return fail(FDP_ERR_SHAPE, "fdp_vec_lincomb_dev: n < 0");
    if (n == 0) return FDP_OK;
    if (!is_device_ptr(coef) || !is_device_ptr(x) || !is_device_ptr(out) || (y && !is_device_ptr(y)) ||
        (z && !is_device_ptr(z)))
      return fail(FDP_ERR_INVALID_ARG, "fdp_vec_lincomb_dev: device pointers required");
    FDP_CUDA(launch_lincomb_dev(coef, x, y, z, out, n, static_cast<cudaStream_t>(stream)), "fdp_vec_lincomb_dev");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_minres_scalars(int phase, double* state, double* hist, int hist_cap,
                                         void* stream) {
  try {
    if (phase < 0 || phase > 3 || hist_cap < 0) return fail(FDP_ERR_INVALID_ARG, "fdp_minres_scalars: bad phase");
    if (!is_device_ptr(state) || (hist && !is_device_ptr(hist)))
      return fail(FDP_ERR_INVALID_ARG, "fdp_minres_scalars: device pointers required");
    FDP_CUDA(launch_minres_scalars(phase, state, hist, hist_cap, static_cast<cudaStream_t>(stream)),
             "fdp_minres_scalars");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_vec_copy_indexed(const double* V, int64_t ldv, const int* idx, double* out,
                                           int64_t n, void* stream) {
  try {
    if (n < 0 || ldv < n) return fail(FDP_ERR_SHAPE, "fdp_vec_copy_indexed: bad extents");
    if (!is_device_ptr(V) || !is_device_ptr(idx) || !is_device_ptr(out))
      return fail(FDP_ERR_INVALID_ARG, "fdp_vec_copy_indexed: device pointers required");
    FDP_CUDA(launch_copy_indexed(V, ldv, idx, out, n, static_cast<cudaStream_t>(stream)), "fdp_vec_copy_indexed");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_vec_store_indexed(double* V, int64_t ldv, const int* idx, const double* w,
                                            const double* coef, int64_t n, void* stream) {
  try {
    if (n < 0 || ldv < n) return fail(FDP_ERR_SHAPE, "fdp_vec_store_indexed: bad extents");
    if (!is_device_ptr(V) || !is_device_ptr(idx) || !is_device_ptr(w) || !is_device_ptr(coef))
      return fail(FDP_ERR_INVALID_ARG, "fdp_vec_store_indexed: device pointers required");
    FDP_CUDA(launch_store_indexed(V, ldv, idx, w, coef, n, static_cast<cudaStream_t>(stream)), "fdp_vec_store_indexed");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_vec_multidot_dev(const double* V, int64_t ldv, const int* m, int m_max,
                                           const double* w, int64_t n, double* h, void* workspace,
                                           void* stream) {
  try {
    if (m_max < 0 || n < 0 || (m_max > 0 && ldv < n)) return fail(FDP_ERR_SHAPE, "fdp_vec_multidot_dev: bad extents");
    if (m_max == 0) return FDP_OK;
    if (!is_device_ptr(V) || !is_device_ptr(m) || !is_device_ptr(w) || !is_device_ptr(h) || !is_device_ptr(workspace))
      return fail(FDP_ERR_INVALID_ARG, "fdp_vec_multidot_dev: device pointers required");
    FDP_CUDA(launch_multidot_dev(V, ldv, m, m_max, w, n, h, static_cast<double*>(workspace),
                                 static_cast<cudaStream_t>(stream)), "fdp_vec_multidot_dev");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_vec_gemv_dev(const double* V, int64_t ldv, const int* m, int m_max,
                                       const double* h, double alpha, double* w, double beta,
                                       int64_t n, void* stream) {
  try {
    if (m_max < 0 || m_max > 6144 || n < 0 || ldv < n) return fail(FDP_ERR_SHAPE, "fdp_vec_gemv_dev: bad extents");
    if (n == 0) return FDP_OK;
    if (!is_device_ptr(V) || !is_device_ptr(m) || !is_device_ptr(h) || !is_device_ptr(w))
      return fail(FDP_ERR_INVALID_ARG, "fdp_vec_gemv_dev: device pointers required");
    FDP_CUDA(launch_gemv_dev(V, ldv, m, m_max, h, alpha, w, beta, n, static_cast<cudaStream_t>(stream)),
             "fdp_vec_gemv_dev");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_gmres_scalars(int phase, int* istate, double* dstate, double* H, int ldh,
                                        const double* h1, const double* h2, double* hist, int m_max,
                                        void* stream) {
  try {
    if ((phase != 0 && phase != 1) || m_max < 1 || ldh < m_max + 1)
      return fail(FDP_ERR_INVALID_ARG, "fdp_gmres_scalars: bad phase or extents");
    if (!is_device_ptr(istate) || !is_device_ptr(dstate) || !is_device_ptr(H) || !is_device_ptr(h1) ||
        !is_device_ptr(h2) || (hist && !is_device_ptr(hist)))
      return fail(FDP_ERR_INVALID_ARG, "fdp_gmres_scalars: device pointers required");
    FDP_CUDA(launch_gmres_scalars(phase, istate, dstate, H, ldh, h1, h2, hist, m_max,
                                  static_cast<cudaStream_t>(stream)), "fdp_gmres_scalars");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

// ------------------------------------------------------------------------------------------------
// Arnoldi helpers (GMRES orthogonalization, NEXT-2)
// ------------------------------------------------------------------------------------------------
extern "C" size_t fdp_vec_multidot_workspace_bytes(int m) {
  try {
    return m > 0 ? multidot_scratch_elems(m) * sizeof(double) : 0;
  } catch (...) {
    return 0;
  }
}

extern "C" fdp_status fdp_vec_multidot(const double* V, int64_t ldv, int m, const double* w,
                                       int64_t n, double* h, void* workspace, void* stream) {
  try {
    if (m < 0 || n < 0 || (m > 0 && ldv < n)) return fail(FDP_ERR_SHAPE, "fdp_vec_multidot: bad extents");
    if (m == 0) return FDP_OK;
    if (!is_device_ptr(V) || !is_device_ptr(w) || !is_device_ptr(h) || !is_device_ptr(workspace))
      return fail(FDP_ERR_INVALID_ARG, "fdp_vec_multidot: device pointers required");
    FDP_CUDA(launch_multidot(V, ldv, m, w, n, h, static_cast<double*>(workspace), static_cast<cudaStream_t>(stream)),
             "fdp_vec_multidot");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}

extern "C" fdp_status fdp_vec_gemv(const double* V, int64_t ldv, int m, const double* h, double alpha,
                                   double* w, double beta, int64_t n, void* stream) {
  try {
    if (m < 0 || m > 6144 || n < 0 || (m > 0 && ldv < n)) return fail(FDP_ERR_SHAPE, "fdp_vec_gemv: bad extents (m <= 6144)");
    if (n == 0) return FDP_OK;
    if (!is_device_ptr(w) || (m > 0 && (!is_device_ptr(V) || !is_device_ptr(h))))
      return fail(FDP_ERR_INVALID_ARG, "fdp_vec_gemv: device pointers required");
    FDP_CUDA(launch_gemv(V, ldv, m, h, alpha, w, beta, n, static_cast<cudaStream_t>(stream)), "fdp_vec_gemv");
    return FDP_OK;
  } catch (...) {
    return abi_exception(__func__);
  }
}
