// Shared helpers for libtoepcuda: complex arithmetic on double2/float2,
// error plumbing (thread-local message + status codes of include/toepcuda.h).
#pragma once

#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cmath>
#include <cstdio>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "../../include/toepcuda.h"

namespace toep {

template <typename T> struct cplx_t;
template <> struct cplx_t<double> { using type = double2; };
template <> struct cplx_t<float> { using type = float2; };
template <typename T> using C = typename cplx_t<T>::type;

template <typename T> __host__ __device__ __forceinline__ C<T> mk(T re, T im) { C<T> z; z.x = re; z.y = im; return z; }
template <typename Z> __host__ __device__ __forceinline__ Z cadd(Z a, Z b) { a.x += b.x; a.y += b.y; return a; }
template <typename Z> __host__ __device__ __forceinline__ Z csub(Z a, Z b) { a.x -= b.x; a.y -= b.y; return a; }
template <typename Z> __host__ __device__ __forceinline__ Z cmul(Z a, Z b) {
  Z r; r.x = a.x * b.x - a.y * b.y; r.y = a.x * b.y + a.y * b.x; return r;
}
// conj(a) * b
template <typename Z> __host__ __device__ __forceinline__ Z cmulc(Z a, Z b) {
  Z r; r.x = a.x * b.x + a.y * b.y; r.y = a.x * b.y - a.y * b.x; return r;
}
// acc += a * b (FMA form)
template <typename Z> __device__ __forceinline__ void cfma(Z& acc, Z a, Z b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
template <typename Z> __device__ __forceinline__ void cfmac(Z& acc, Z a, Z b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(-a.y, b.x, acc.y);
}
template <typename Z, typename S> __host__ __device__ __forceinline__ Z cscale(Z a, S s) { a.x *= s; a.y *= s; return a; }

// ---------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
const char* last_error();

// cudaFuncAttributeMaxDynamicSharedMemorySize >= bytes for `func` on the CURRENT device.
// Function attributes belong to a device context, so the cache is keyed by (device, function);
// thread-safe.  Cheap on the hit path (one lock + map lookup).
cudaError_t ensure_smem_attr(const void* func, size_t bytes);
template <typename F> inline cudaError_t ensure_smem(F* func, size_t bytes) {
  return ensure_smem_attr(reinterpret_cast<const void*>(func), bytes);
}

struct Status {
  int code = TOEP_OK;
};

// NVTX range over a C-ABI entry point (header-only NVTX v3: a no-op unless a tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace toep

#define TOEP_CUDA(call)                                                                  \
  do {                                                                                   \
    cudaError_t _e = (call);                                                             \
    if (_e != cudaSuccess) {                                                             \
      ::toep::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(_e)); \
      return TOEP_ERR_CUDA;                                                              \
    }                                                                                    \
  } while (0)

#define TOEP_LAUNCHED()                                                                  \
  do {                                                                                   \
    cudaError_t _e = cudaGetLastError();                                                 \
    if (_e != cudaSuccess) {                                                             \
      ::toep::set_error("%s:%d kernel launch: %s", __FILE__, __LINE__, cudaGetErrorString(_e)); \
      return TOEP_ERR_CUDA;                                                              \
    }                                                                                    \
  } while (0)

#define TOEP_TRY(expr)                 \
  do {                                 \
    int _s = (expr);                   \
    if (_s != TOEP_OK) return _s;      \
  } while (0)

#define TOEP_NVTX(name) ::toep::NvtxRange _toep_nvtx_range(name)

#define TOEP_REQUIRE(cond, code, ...)         \
  do {                                        \
    if (!(cond)) {                            \
      ::toep::set_error(__VA_ARGS__);         \
      return (code);                          \
    }                                         \
  } while (0)
