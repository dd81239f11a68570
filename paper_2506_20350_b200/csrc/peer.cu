// Peer-memory plumbing of the slab-decomposed matvec (multi-GPU).
//
// The two all-to-all exchanges of a distributed matvec are fused into the DFT passes that
// produce them (toep_matvec_stage_peer, fft.cu: the last pass stores every output row straight
// into the owning rank's receive buffer over NVLink and then bumps that rank's arrival counter).
// What is left here: the stream-side wait on an arrival counter, and cudaMalloc'd exchange
// memory with its CUDA IPC handle / mapping (the process group exchanges the 64-byte handles).
#include "kernels.cuh"
#include "launch.cuh"

namespace toep {
namespace {

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One thread spins (acquire, system scope) until the counter reaches the target.  Launched without
// griddepcontrol.wait, so it may start while the stream's previous kernel (this rank's own scatter)
// drains; it completes only when every producer has signalled.  A peer that never arrives (a rank
// that died or diverged) traps after 30 s rather than hanging the device.
__global__ void peer_wait_kernel(const unsigned long long* counter, unsigned long long target) {
  if (threadIdx.x != 0) return;
  const uint64_t t0 = global_ns();
  for (;;) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(counter) : "memory");
    if (v >= target) return;
    if (global_ns() - t0 > 30ull * 1000000000ull) __trap();
    __nanosleep(128);
  }
}

}  // namespace
}  // namespace toep

extern "C" {

int toep_peer_wait(const uint64_t* counter, uint64_t target, void* stream) {
  TOEP_REQUIRE(counter != nullptr, TOEP_ERR_ARG, "null counter");
  return toep::launch_k(toep::peer_wait_kernel, dim3(1), dim3(32), 0, static_cast<cudaStream_t>(stream),
                        reinterpret_cast<const unsigned long long*>(counter),
                        static_cast<unsigned long long>(target));
}

int toep_peer_alloc(uint64_t bytes, void** out) {
  TOEP_REQUIRE(out != nullptr && bytes > 0, TOEP_ERR_ARG, "bad peer_alloc arguments");
  void* p = nullptr;
  const cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    toep::set_error("peer_alloc of %llu bytes failed: %s", static_cast<unsigned long long>(bytes),
                    cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? TOEP_ERR_OOM : TOEP_ERR_CUDA;
  }
  TOEP_CUDA(cudaMemset(p, 0, bytes));
  *out = p;
  return TOEP_OK;
}

int toep_peer_free(void* ptr) {
  if (ptr == nullptr) return TOEP_OK;
  TOEP_CUDA(cudaFree(ptr));
  return TOEP_OK;
}

int toep_ipc_handle(const void* ptr, void* handle64) {
  TOEP_REQUIRE(ptr != nullptr && handle64 != nullptr, TOEP_ERR_ARG, "null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t h;
  TOEP_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(ptr)));
  std::memcpy(handle64, &h, sizeof(h));
  return TOEP_OK;
}

int toep_ipc_open(const void* handle64, void** out) {
  TOEP_REQUIRE(handle64 != nullptr && out != nullptr, TOEP_ERR_ARG, "null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  void* p = nullptr;
  TOEP_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *out = p;
  return TOEP_OK;
}

int toep_ipc_close(void* ptr) {
  TOEP_REQUIRE(ptr != nullptr, TOEP_ERR_ARG, "null pointer");
  TOEP_CUDA(cudaIpcCloseMemHandle(ptr));
  return TOEP_OK;
}

}  // extern "C"
