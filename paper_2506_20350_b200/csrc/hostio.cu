// Host-side helpers of the problem-file path (TBZ1, problems.py:219-322 of the reference).
#include "common.cuh"

extern "C" int toep_fnv1a64(const void* data, uint64_t bytes, uint64_t* out) {
  TOEP_REQUIRE(out != nullptr && (data != nullptr || bytes == 0), TOEP_ERR_ARG, "bad fnv1a64 arguments");
  const unsigned char* p = static_cast<const unsigned char*>(data);
  uint64_t h = 0xCBF29CE484222325ull;  // offset basis
  for (uint64_t i = 0; i < bytes; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ull;  // FNV prime (wraps mod 2^64)
  }
  *out = h;
  return TOEP_OK;
}

// Page-locked host buffers for the host-in / host-out calls (toep_matvec_host).  cudaHostAlloc
// memory is read by the copy engines at the PCIe rate (1.84 MB H2D: 37 us = 50 GB/s on the B200
// boxes); torch's caching host allocator's blocks measured 17-19 GB/s in the same direction
// (tools/hostbuf_probe.py), so the Python layer stages host vectors in these.
extern "C" int toep_host_alloc(uint64_t bytes, void** out) {
  TOEP_REQUIRE(out != nullptr, TOEP_ERR_ARG, "null output pointer");
  *out = nullptr;
  if (bytes == 0) return TOEP_OK;
  const cudaError_t e = cudaHostAlloc(out, bytes, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *out = nullptr;
    toep::set_error("cudaHostAlloc of %llu bytes failed: %s", static_cast<unsigned long long>(bytes),
                    cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? TOEP_ERR_OOM : TOEP_ERR_CUDA;
  }
  return TOEP_OK;
}

extern "C" int toep_host_free(void* p) {
  if (p == nullptr) return TOEP_OK;
  TOEP_CUDA(cudaFreeHost(p));
  return TOEP_OK;
}
