// Internal definition of the resident spectral operator (toep_op_t).
#pragma once

#include <map>
#include <mutex>

#include "kernels.cuh"

struct toep_op_s {
  int n2 = 0, n1 = 0, n0 = 0, l2 = 0, l1 = 0, dtype = TOEP_C128;
  int64_t K = 0;
  void* DT = nullptr;  // [K][n0][n0], DT[k][j][m] = D_k[m][j]
  double* DTp = nullptr;  // multi-RHS 3M: (re, im, re+im) planes of DT, K*n0*n0 doubles apart
  int device = 0;
  struct Workspace {
    int64_t w_cap = 0;    // x1
    int64_t hat_cap = 0;  // hat / hat2
    void* x1 = nullptr;    // [n2][l1][n0*w]
    void* hat = nullptr;   // [K][n0][w]
    void* hat2 = nullptr;  // [K][n0][w]
    double* hatp = nullptr;   // multi-RHS 3M: planes of u_hat (3 x K*n0*w)
    double* hat2p = nullptr;  // multi-RHS 3M: product planes T1, T2, T3
    size_t p_bytes = 0;       // capacity of hatp / hat2p in bytes (the chunking depends on w)
    void* io = nullptr;  // toep_matvec_host: device copies of u and v
    size_t io_cap = 0;
    void* pin_in = nullptr;  // toep_matvec_host + TOEP_MV_STAGE_INPUT: page-locked staging of u
    size_t pin_cap = 0;
    unsigned* bar = nullptr;  // fused single-RHS matvec: [0] grid-barrier counter, [1] bin hand-out counter
    int8_t* oz_b = nullptr;     // Ozaki path: int8 slices of one chunk's U planes
    int32_t* oz_bexp = nullptr; // and their column exponents
    size_t oz_b_bytes = 0, oz_bexp_bytes = 0;  // capacities in bytes
  };
  int8_t* oz_a = nullptr;       // Ozaki path: int8 slices of [Dr -Di; Di Dr] per bin (kx-major)
  int32_t* oz_aexp = nullptr;   // row exponents
  // operator-wide buffers built lazily (oz_a / oz_aexp, DTp) on the first caller's stream: an
  // event recorded after the build orders every other stream's first use after it
  cudaEvent_t lazy_ev = nullptr;
  cudaStream_t lazy_stream = nullptr;
  // kx-slab operator of the multi-GPU row/slab decomposition (toep_op_slab): bins
  // k' = ky*slab_kxs + (kx - slab_k0); 0 = full operator
  int slab_k0 = 0, slab_kxs = 0;
  std::mutex mu;
  std::map<cudaStream_t, Workspace> ws;
};

namespace toep {

size_t elt_size(int dtype);
int64_t op_dim(const toep_op_s* op);
int op_workspace(toep_op_s* op, int64_t w, cudaStream_t s, toep_op_s::Workspace** out, bool need_hat = true);

// matvec with optional device-side stop flag (GMRES speculative steps).
// io_c128: u / v are complex128 while the operator computes in its own dtype.
// in_scale: optional device scalar s, computes A (s u)
int matvec_impl(toep_op_s* op, const void* u, void* v, int64_t w, bool transpose, bool io_c128,
                const int* stop, cudaStream_t s, const double* in_scale = nullptr);

void keep_pool();

// hostio.cu: copy `bytes` from pageable `src` to page-locked `dst` with the library's copy threads
// in chunks, enqueueing each chunk's H2D copy (dst -> dev) on `s` as soon as it is staged
int staged_h2d(const void* src, void* dst_pinned, void* dev, size_t bytes, cudaStream_t s);
// large pageable host -> device copy, staged through double-buffered page-locked chunks
int pipelined_h2d(const void* src, void* dst, size_t bytes, cudaStream_t s);


// the local stages of the slab-decomposed matvec (toep_matvec_stage / toep_matvec_stage_peer)
int matvec_stage_impl(toep_op_s* op, int stage, const void* in, void* out, int64_t w, int count,
                      const toep_peer_scatter* scatter, cudaStream_t s);

int block_apply_impl(const void* m, int n0, const void* in, void* out, int64_t segments, int64_t w, int dtype,
                     cudaStream_t s, const int* stop);

}  // namespace toep
