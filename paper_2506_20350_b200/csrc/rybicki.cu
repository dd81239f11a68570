// Block Rybicki (bordering) direct solver on the device: rybicki.py:63-144 + numerics.lu_factor /
// lu_solve (numerics.py:67-96).
//
// Every block product of the recursion (the block sums d1, d2, the numerators, the generator
// cross-updates) is a dense complex GEMM on the FP64 tensor cores (zgemm_tc); the two
// denominators per step are LU-factored on the device with partial pivoting (right-looking
// blocked LU: single-CTA panel + TRSM + tensor-core GEMM trailing update) and applied through
// blocked triangular solves whose off-diagonal work is again GEMM.  All matrices are row-major
// complex128; row swaps are contiguous.  Singular pivots (|p| < 1e-300, numerics.py:27) raise
// SingularBlock for R_0 and SingularDenominator(step) for D1 / D2, as the reference.
#include <vector>

#include "op.h"

namespace toep {
namespace {

constexpr int kNB = 32;         // LU / TRSM block size
constexpr int kPanelThreads = 1024;
constexpr double kPivotTiny = 1e-300;

__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double den = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / den, (a.y * b.x - a.x * b.y) / den);
}

// Factor panel columns [j0, j0+nb) of the n x n row-major matrix A (rows j0..n-1) with partial
// pivoting; rows are swapped across all n columns immediately.  One CTA.
__global__ void __launch_bounds__(kPanelThreads) lu_panel(double2* A, int n, int lda, int j0, int nb, int* ipiv,
                                                          int* info) {
  __shared__ double sval[kPanelThreads / 32];
  __shared__ int sidx[kPanelThreads / 32];
  __shared__ int piv_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = j0; j < j0 + nb; ++j) {
    // argmax_i |A[i][j]| (first max on ties, like LAPACK's izamax)
    double best = -1.0;
    int bi = n;
    for (int i = j + tid; i < n; i += kPanelThreads) {
      const double v = cabs2(A[static_cast<int64_t>(i) * lda + j]);
      if (v > best) { best = v; bi = i; }
    }
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) { sval[warp] = best; sidx[warp] = bi; }
    __syncthreads();
    if (tid == 0) {
      double b = sval[0];
      int id = sidx[0];
      for (int w2 = 1; w2 < kPanelThreads / 32; ++w2)
        if (sval[w2] > b || (sval[w2] == b && sidx[w2] < id)) { b = sval[w2]; id = sidx[w2]; }
      piv_s = id;
      ipiv[j] = id;
      if (!(sqrt(b) >= kPivotTiny) && *info == 0) *info = j + 1;
    }
    __syncthreads();
    const int p = piv_s;
    if (p != j) {
      for (int c = tid; c < n; c += kPanelThreads) {
        const double2 t = A[static_cast<int64_t>(j) * lda + c];
        A[static_cast<int64_t>(j) * lda + c] = A[static_cast<int64_t>(p) * lda + c];
        A[static_cast<int64_t>(p) * lda + c] = t;
      }
    }
    __syncthreads();
    const double2 d = A[static_cast<int64_t>(j) * lda + j];
    const bool ok = cabs2(d) > 0.0;
    // scale the column below the pivot and update the rest of the panel (rank 1)
    const int rows = n - j - 1, cols = j0 + nb - j - 1;
    for (int i = tid; i < rows; i += kPanelThreads) {
      double2* a = A + static_cast<int64_t>(j + 1 + i) * lda;
      const double2 l = ok ? cdiv(a[j], d) : a[j];
      a[j] = l;
      for (int c = 0; c < cols; ++c) cfma(a[j + 1 + c], make_double2(-l.x, -l.y), A[static_cast<int64_t>(j) * lda + j + 1 + c]);
    }
    __syncthreads();
  }
}

// U12 = L11^-1 A12: unit-lower forward substitution on rows [j0, j0+nb), columns [c0, n)
__global__ void trsm_lower_unit_rows(double2* A, int lda, int j0, int nb, int c0, int ncols) {
  const int c = c0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= c0 + ncols) return;
  for (int i = 1; i < nb; ++i) {
    double2 acc = A[static_cast<int64_t>(j0 + i) * lda + c];
    for (int k = 0; k < i; ++k)
      cfma(acc, make_double2(-A[static_cast<int64_t>(j0 + i) * lda + j0 + k].x, -A[static_cast<int64_t>(j0 + i) * lda + j0 + k].y),
           A[static_cast<int64_t>(j0 + k) * lda + c]);
    A[static_cast<int64_t>(j0 + i) * lda + c] = acc;
  }
}

// B[j] <-> B[ipiv[j]] for j = 0..n-1 (sequential in j, parallel over the nrhs columns)
__global__ void laswp_rows(double2* B, int ldb, int nrhs, const int* ipiv, int n) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nrhs) return;
  for (int j = 0; j < n; ++j) {
    const int p = ipiv[j];
    if (p != j) {
      const double2 t = B[static_cast<int64_t>(j) * ldb + c];
      B[static_cast<int64_t>(j) * ldb + c] = B[static_cast<int64_t>(p) * ldb + c];
      B[static_cast<int64_t>(p) * ldb + c] = t;
    }
  }
}

// diagonal-block triangular solve on rows [r0, r0+nb) of B (nrhs columns):
// lower (unit): forward;  upper: backward with the diagonal of LU
__global__ void trsm_diag_block(const double2* LU, int lda, double2* B, int ldb, int nrhs, int r0, int nb, int upper) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nrhs) return;
  if (!upper) {
    for (int i = 1; i < nb; ++i) {
      double2 acc = B[static_cast<int64_t>(r0 + i) * ldb + c];
      for (int k = 0; k < i; ++k) {
        const double2 l = LU[static_cast<int64_t>(r0 + i) * lda + r0 + k];
        cfma(acc, make_double2(-l.x, -l.y), B[static_cast<int64_t>(r0 + k) * ldb + c]);
      }
      B[static_cast<int64_t>(r0 + i) * ldb + c] = acc;
    }
  } else {
    for (int i = nb - 1; i >= 0; --i) {
      double2 acc = B[static_cast<int64_t>(r0 + i) * ldb + c];
      for (int k = i + 1; k < nb; ++k) {
        const double2 u = LU[static_cast<int64_t>(r0 + i) * lda + r0 + k];
        cfma(acc, make_double2(-u.x, -u.y), B[static_cast<int64_t>(r0 + k) * ldb + c]);
      }
      B[static_cast<int64_t>(r0 + i) * ldb + c] = cdiv(acc, LU[static_cast<int64_t>(r0 + i) * lda + r0 + i]);
    }
  }
}

__global__ void copy_scaled(const double2* __restrict__ src, double2* __restrict__ dst, int64_t count, double s) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = cscale(src[i], s);
}

int copy_neg(const double2* src, double2* dst, int64_t count, double s, cudaStream_t st) {
  const int grid = static_cast<int>(std::min<int64_t>((count + 255) / 256, 148 * 8));
  copy_scaled<<<grid, 256, 0, st>>>(src, dst, count, s);
  TOEP_LAUNCHED();
  return TOEP_OK;
}

// C (+)= alpha A B, all row-major, A: m x k (lda), B: k x nn (ldb), C: m x nn (ldc)
int gemm_rm(int64_t m, int64_t nn, int64_t k, double2 alpha, const double2* A, int64_t lda, const double2* B,
            int64_t ldb, double2 beta, double2* C, int64_t ldc, cudaStream_t s) {
  return gemm(TOEP_C128, m, nn, k, alpha, A, lda, 1, 0, B, ldb, 1, 0, beta, C, ldc, 1, 0, 1, s);
}

// in-place LU with partial pivoting of the n x n row-major A; info (device) > 0: singular
int getrf(double2* A, int n, int* ipiv, int* info, cudaStream_t s) {
  for (int j0 = 0; j0 < n; j0 += kNB) {
    const int nb = std::min(kNB, n - j0);
    lu_panel<<<1, kPanelThreads, 0, s>>>(A, n, n, j0, nb, ipiv, info);
    TOEP_LAUNCHED();
    const int c0 = j0 + nb, rest = n - c0;
    if (rest > 0) {
      trsm_lower_unit_rows<<<(rest + 127) / 128, 128, 0, s>>>(A, n, j0, nb, c0, rest);
      TOEP_LAUNCHED();
      // A22 -= L21 U12
      TOEP_TRY(gemm_rm(rest, rest, nb, make_double2(-1, 0), A + static_cast<int64_t>(c0) * n + j0, n,
                       A + static_cast<int64_t>(j0) * n + c0, n, make_double2(1, 0), A + static_cast<int64_t>(c0) * n + c0,
                       n, s));
    }
  }
  return TOEP_OK;
}

// B <- A^-1 B with A = P L U from getrf; B: n x nrhs row-major (ldb)
int getrs(const double2* LU, int n, const int* ipiv, double2* B, int ldb, int nrhs, cudaStream_t s) {
  const int gr = (nrhs + 127) / 128;
  laswp_rows<<<gr, 128, 0, s>>>(B, ldb, nrhs, ipiv, n);
  TOEP_LAUNCHED();
  for (int r0 = 0; r0 < n; r0 += kNB) {  // L y = P b (unit lower)
    const int nb = std::min(kNB, n - r0);
    trsm_diag_block<<<gr, 128, 0, s>>>(LU, n, B, ldb, nrhs, r0, nb, 0);
    TOEP_LAUNCHED();
    const int rest = n - r0 - nb;
    if (rest > 0)
      TOEP_TRY(gemm_rm(rest, nrhs, nb, make_double2(-1, 0), LU + static_cast<int64_t>(r0 + nb) * n + r0, n,
                       B + static_cast<int64_t>(r0) * ldb, ldb, make_double2(1, 0), B + static_cast<int64_t>(r0 + nb) * ldb,
                       ldb, s));
  }
  for (int r1 = n; r1 > 0; r1 -= kNB) {  // U x = y
    const int r0 = std::max(0, r1 - kNB);
    const int nb = r1 - r0;
    trsm_diag_block<<<gr, 128, 0, s>>>(LU, n, B, ldb, nrhs, r0, nb, 1);
    TOEP_LAUNCHED();
    if (r0 > 0)
      TOEP_TRY(gemm_rm(r0, nrhs, nb, make_double2(-1, 0), LU + r0, n, B + static_cast<int64_t>(r0) * ldb, ldb,
                       make_double2(1, 0), B, ldb, s));
  }
  return TOEP_OK;
}

}  // namespace
}  // namespace toep

using namespace toep;

extern "C" int toep_lu_factor(void* a, int n, int* ipiv, int* info, void* stream) {
  TOEP_REQUIRE(a != nullptr && ipiv != nullptr && info != nullptr && n >= 1, TOEP_ERR_ARG, "bad lu_factor args");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  TOEP_CUDA(cudaMemsetAsync(info, 0, sizeof(int), s));
  return getrf(static_cast<double2*>(a), n, ipiv, info, s);
}

extern "C" int toep_lu_solve(const void* lu, int n, const int* ipiv, void* b, int64_t nrhs, void* stream) {
  TOEP_REQUIRE(lu != nullptr && ipiv != nullptr && b != nullptr && n >= 1, TOEP_ERR_ARG, "bad lu_solve args");
  return getrs(static_cast<const double2*>(lu), n, ipiv, static_cast<double2*>(b), static_cast<int>(nrhs),
               static_cast<int>(nrhs), static_cast<cudaStream_t>(stream));
}

extern "C" int toep_rybicki(const void* blocks_v, int N, int s, const void* y_v, void* x_v, int64_t w,
                            int* fail_step, toep_stage_fn hook, void* hook_ctx, void* stream) {
  TOEP_REQUIRE(blocks_v != nullptr && y_v != nullptr && x_v != nullptr && N >= 1 && s >= 1 && w >= 1, TOEP_ERR_ARG,
               "bad rybicki arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  keep_pool();
  const double2* blocks = static_cast<const double2*>(blocks_v);
  const double2* y = static_cast<const double2*>(y_v);
  double2* x = static_cast<double2*>(x_v);  // (N, s, w): x_j at x + j*s*w
  const int64_t ss = static_cast<int64_t>(s) * s, sw = static_cast<int64_t>(s) * w;
  const int nb2 = 2 * N - 1;
  auto rb = [&](int o) { return blocks + static_cast<int64_t>(((o % nb2) + nb2) % nb2) * ss; };
  if (fail_step) *fail_step = -1;

  double2 *g = nullptr, *h = nullptr, *gtmp = nullptr, *lu0 = nullptr, *lu1 = nullptr, *lu2 = nullptr;
  double2 *gnew = nullptr, *hnew = nullptr, *num = nullptr;
  int *piv0 = nullptr, *piv1 = nullptr, *piv2 = nullptr, *info = nullptr;
  auto cleanup = [&]() {
    for (void* q : {(void*)g, (void*)h, (void*)gtmp, (void*)lu0, (void*)lu1, (void*)lu2, (void*)gnew, (void*)hnew,
                    (void*)num, (void*)piv0, (void*)piv1, (void*)piv2, (void*)info})
      if (q) cudaFreeAsync(q, st);
    cudaStreamSynchronize(st);
  };
  int rc = TOEP_OK;
#define R_ALLOC(ptr, count)                                                                                      \
  do {                                                                                                           \
    if (cudaMallocAsync(reinterpret_cast<void**>(&(ptr)), sizeof(*(ptr)) * (size_t)(count), st) != cudaSuccess) { \
      cudaGetLastError();                                                                                        \
      set_error("out of device memory in rybicki");                                                              \
      cleanup();                                                                                                 \
      return TOEP_ERR_OOM;                                                                                       \
    }                                                                                                            \
  } while (0)
#define R_TRY(expr)      \
  do {                   \
    rc = (expr);         \
    if (rc != TOEP_OK) { \
      cleanup();         \
      return rc;         \
    }                    \
  } while (0)
  const int nm1 = std::max(N - 1, 1);
  R_ALLOC(g, nm1 * ss);
  R_ALLOC(h, nm1 * ss);
  R_ALLOC(gtmp, nm1 * ss);
  R_ALLOC(lu0, ss);
  R_ALLOC(lu1, ss);
  R_ALLOC(lu2, ss);
  R_ALLOC(gnew, ss);
  R_ALLOC(hnew, ss);
  R_ALLOC(num, std::max<int64_t>(sw, 1));
  R_ALLOC(piv0, s);
  R_ALLOC(piv1, s);
  R_ALLOC(piv2, s);
  R_ALLOC(info, 1);
  const double2 one = make_double2(1, 0), mone = make_double2(-1, 0);
  auto check_info = [&](int code, int step) -> int {
    int hinfo = 0;
    TOEP_CUDA(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, st));
    TOEP_CUDA(cudaStreamSynchronize(st));
    if (hinfo != 0) {
      if (fail_step) *fail_step = step;
      set_error(code == TOEP_ERR_SINGULAR_BLOCK ? "self block R_0 is singular"
                                                : "singular denominator at bordering step %d", step);
      return code;
    }
    return TOEP_OK;
  };
  auto stage_hook = [&](int stage) -> int {
    if (hook == nullptr) return TOEP_OK;
    TOEP_REQUIRE(hook(hook_ctx, stage, x, g, h, stream) == 0, TOEP_ERR_ARG, "rybicki step hook failed");
    return TOEP_OK;
  };

  // base stage (rybicki.py:94-108)
  TOEP_CUDA(cudaMemcpyAsync(lu0, rb(0), ss * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  R_TRY(toep_lu_factor(lu0, s, piv0, info, stream));
  R_TRY(check_info(TOEP_ERR_SINGULAR_BLOCK, 0));
  TOEP_CUDA(cudaMemcpyAsync(x, y, sw * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  R_TRY(getrs(lu0, s, piv0, x, static_cast<int>(w), static_cast<int>(w), st));
  if (N > 1) {
    TOEP_CUDA(cudaMemcpyAsync(g, rb(-1), ss * sizeof(double2), cudaMemcpyDeviceToDevice, st));
    R_TRY(getrs(lu0, s, piv0, g, s, s, st));
    TOEP_CUDA(cudaMemcpyAsync(h, rb(1), ss * sizeof(double2), cudaMemcpyDeviceToDevice, st));
    R_TRY(getrs(lu0, s, piv0, h, s, s, st));
  }
  R_TRY(stage_hook(1));

  for (int m = 1; m < N; ++m) {
    // d1 = sum_{k=1..m} R_k G_k - R_0  (G_k = g[k-1])
    R_TRY(copy_neg(rb(0), lu1, ss, -1.0, st));
    for (int k = 1; k <= m; ++k)
      R_TRY(gemm_rm(s, s, s, one, rb(k), s, g + (k - 1) * ss, s, one, lu1, s, st));
    R_TRY(toep_lu_factor(lu1, s, piv1, info, stream));
    R_TRY(check_info(TOEP_ERR_SINGULAR_DENOM, m));
    // x_{m+1} = D1^-1 (sum_j R_{m+1-j} x_j - y_{m+1})
    R_TRY(copy_neg(y + m * sw, num, sw, -1.0, st));
    for (int jj = 1; jj <= m; ++jj)
      R_TRY(gemm_rm(s, w, s, one, rb(m + 1 - jj), s, x + (jj - 1) * sw, w, one, num, w, st));
    R_TRY(getrs(lu1, s, piv1, num, static_cast<int>(w), static_cast<int>(w), st));
    TOEP_CUDA(cudaMemcpyAsync(x + m * sw, num, sw * sizeof(double2), cudaMemcpyDeviceToDevice, st));
    // x_j -= G_{m+1-j} x_{m+1}
    for (int jj = 1; jj <= m; ++jj)
      R_TRY(gemm_rm(s, w, s, mone, g + (m - jj) * ss, s, x + m * sw, w, one, x + (jj - 1) * sw, w, st));
    if (m < N - 1) {
      // d2 = sum_{k=1..m} R_{-k} H_k - R_0
      R_TRY(copy_neg(rb(0), lu2, ss, -1.0, st));
      for (int k = 1; k <= m; ++k)
        R_TRY(gemm_rm(s, s, s, one, rb(-k), s, h + (k - 1) * ss, s, one, lu2, s, st));
      R_TRY(toep_lu_factor(lu2, s, piv2, info, stream));
      R_TRY(check_info(TOEP_ERR_SINGULAR_DENOM, m));
      // G_new = D2^-1 (sum_j R_{j-m-1} G_j - R_{-(m+1)})
      R_TRY(copy_neg(rb(-(m + 1)), gnew, ss, -1.0, st));
      for (int jj = 1; jj <= m; ++jj)
        R_TRY(gemm_rm(s, s, s, one, rb(jj - m - 1), s, g + (jj - 1) * ss, s, one, gnew, s, st));
      R_TRY(getrs(lu2, s, piv2, gnew, s, s, st));
      // H_new = D1^-1 (sum_j R_{m+1-j} H_j - R_{m+1})
      R_TRY(copy_neg(rb(m + 1), hnew, ss, -1.0, st));
      for (int jj = 1; jj <= m; ++jj)
        R_TRY(gemm_rm(s, s, s, one, rb(m + 1 - jj), s, h + (jj - 1) * ss, s, one, hnew, s, st));
      R_TRY(getrs(lu1, s, piv1, hnew, s, s, st));
      // G_j -= H_{m+1-j} G_new (into gtmp, old H);  H_j -= G_{m+1-j} H_new (old G)
      for (int jj = 1; jj <= m; ++jj) {
        TOEP_CUDA(cudaMemcpyAsync(gtmp + (jj - 1) * ss, g + (jj - 1) * ss, ss * sizeof(double2),
                                  cudaMemcpyDeviceToDevice, st));
        R_TRY(gemm_rm(s, s, s, mone, h + (m - jj) * ss, s, gnew, s, one, gtmp + (jj - 1) * ss, s, st));
      }
      for (int jj = 1; jj <= m; ++jj)
        R_TRY(gemm_rm(s, s, s, mone, g + (m - jj) * ss, s, hnew, s, one, h + (jj - 1) * ss, s, st));
      TOEP_CUDA(cudaMemcpyAsync(g, gtmp, m * ss * sizeof(double2), cudaMemcpyDeviceToDevice, st));
      TOEP_CUDA(cudaMemcpyAsync(g + m * ss, gnew, ss * sizeof(double2), cudaMemcpyDeviceToDevice, st));
      TOEP_CUDA(cudaMemcpyAsync(h + m * ss, hnew, ss * sizeof(double2), cudaMemcpyDeviceToDevice, st));
    }
    R_TRY(stage_hook(m + 1));
  }
  cleanup();
#undef R_ALLOC
#undef R_TRY
  return TOEP_OK;
}
