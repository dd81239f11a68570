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
    void* parts = nullptr; // fused path: [l1][maxp][n2][n0] inverse level-2 partial slabs
    int* cnt = nullptr;    // fused path: [l1] slab arrival counters
    double* hatp = nullptr;   // multi-RHS 3M: planes of u_hat (3 x K*n0*w)
    double* hat2p = nullptr;  // multi-RHS 3M: product planes T1, T2, T3
    int64_t p_cap = 0;
    void* io = nullptr;  // toep_matvec_host: device copies of u and v
    size_t io_cap = 0;
    int8_t* oz_b = nullptr;     // Ozaki path: int8 slices of one chunk's U planes
    int32_t* oz_bexp = nullptr; // and their column exponents
    int64_t oz_cap = 0;         // w the buffers were sized for
  };
  int8_t* oz_a = nullptr;       // Ozaki path: int8 slices of [Dr -Di; Di Dr] per bin (kx-major)
  int32_t* oz_aexp = nullptr;   // row exponents
  // kx-slab operator of the multi-GPU row/slab decomposition (toep_op_slab): bins
  // k' = ky*slab_kxs + (kx - slab_k0); 0 = full operator
  int slab_k0 = 0, slab_kxs = 0;
  // fused single-RHS path (fused.cu): kx-major persistent partition
  int fused_grid = 0;
  int fused_maxp = 0;
  int* part_count = nullptr;  // device [l1]
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

// the local stages of the slab-decomposed matvec (toep_matvec_stage / toep_matvec_stage_peer)
int matvec_stage_impl(toep_op_s* op, int stage, const void* in, void* out, int64_t w, int count,
                      const toep_peer_scatter* scatter, cudaStream_t s);

// fused.cu
bool fused_eligible(const toep_op_s* op, int64_t w, bool transpose);
int fused_prepare(toep_op_s* op, cudaStream_t s);
int fused_spectral(toep_op_s* op, const void* x1, void* parts, void* x2, int* cnt, const int* stop, cudaStream_t s);

int block_apply_impl(const void* m, int n0, const void* in, void* out, int64_t segments, int64_t w, int dtype,
                     cudaStream_t s, const int* stop);

}  // namespace toep
