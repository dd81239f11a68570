// Kernel launch helper with Programmatic Dependent Launch (PDL).
//
// Every kernel of the matvec / GMRES chains is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization: the next kernel's CTAs
// are scheduled while the previous grid drains, run their prologue, and block
// in griddepcontrol.wait until the predecessor's memory is visible.  This
// hides the ~2-4 us launch/ramp gap at each of the many kernel boundaries of
// a 170 us matvec and of the short Arnoldi kernels.
#pragma once

#include <cstdlib>
#include <cstring>
#include <utility>

#include "common.cuh"

namespace toep {

inline bool pdl_enabled() { return true; }

// Wait until the predecessor grid (PDL) has completed and its writes are visible.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Allow the dependent grid to start launching (its CTAs still pdl_wait for us).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
int launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(std::forward<Args>(args))...);
  if (e != cudaSuccess) {
    set_error("kernel launch failed: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return TOEP_ERR_CUDA;
  }
  return TOEP_OK;
}

// Grid-barrier kernels launched WITHOUT the cooperative attribute (one CTA per SM, the caller has
// checked that every CTA fits): the next such grid's CTAs start on the SMs the previous grid
// vacates first instead of waiting for the whole grid plus the cooperative dispatch.  What the
// cooperative attribute guarded against — two grid-barrier grids on different streams each holding
// part of the SMs — is excluded by serialising these launches across streams: a launch on another
// stream than the previous one waits for the previous one (per-device event, recorded after every
// launch because a stream may be destroyed later).  Other kernels holding SMs only delay CTAs; the
// grid barriers trap after 10 s.
int gridsync_order(cudaStream_t s);     // wait for the previous grid-barrier launch if on another stream
void gridsync_launched(cudaStream_t s, bool ok);  // record this launch (if it went out); releases the order lock

template <typename... KArgs, typename... Args>
int launch_gridsync(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  const int o = gridsync_order(s);
  if (o != TOEP_OK) return o;
  const int rc = launch_k(kern, grid, block, smem, s, std::forward<Args>(args)...);
  gridsync_launched(s, rc == TOEP_OK);
  return rc;
}

// Cooperative (all CTAs co-resident, grid barriers allowed) + PDL launch.
template <typename... KArgs, typename... Args>
int launch_coop(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(std::forward<Args>(args))...);
  if (e != cudaSuccess) {
    set_error("cooperative launch failed: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return TOEP_ERR_CUDA;
  }
  return TOEP_OK;
}

}  // namespace toep
