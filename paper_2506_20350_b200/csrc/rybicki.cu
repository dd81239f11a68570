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

constexpr int kOB = 32;           // outer LU block (trailing-update GEMM depth), TRSM block
constexpr int kPB = 8;            // sub-panel factored in shared memory
constexpr int kPanelThreads = 1024;
constexpr double kPivotTiny = 1e-300;

__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double den = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / den, (a.y * b.x - a.x * b.y) / den);
}

// Factor the kPB columns [j0, j0+kPB) over rows [j0, n) with partial pivoting, the sub-panel
// resident in shared memory (row-major (n-j0) x kPB).  Interchanges are applied inside the
// sub-panel only (laswp_cols applies them to the other columns); ipiv[j] = absolute pivot row.
__global__ void __launch_bounds__(kPanelThreads) lu_subpanel(double2* A, int n, int lda, int j0, int* ipiv, int* info) {
  extern __shared__ double2 P[];
  __shared__ double sval[kPanelThreads / 32];
  __shared__ int sidx[kPanelThreads / 32];
  __shared__ int piv_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rows = n - j0;
  const int pb = min(kPB, n - j0);
  for (int e = tid; e < rows * kPB; e += kPanelThreads) {
    const int r = e / kPB, c = e - r * kPB;
    P[e] = (c < pb) ? A[static_cast<int64_t>(j0 + r) * lda + j0 + c] : make_double2(0, 0);
  }
  __syncthreads();
  for (int jj = 0; jj < pb; ++jj) {
    double best = -1.0;
    int bi = rows;
    for (int r = jj + tid; r < rows; r += kPanelThreads) {
      const double v = cabs2(P[r * kPB + jj]);
      if (v > best) { best = v; bi = r; }
    }
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) { sval[warp] = best; sidx[warp] = bi; }
    __syncthreads();
    if (tid == 0) {
      double bb = sval[0];
      int id = sidx[0];
      for (int w2 = 1; w2 < kPanelThreads / 32; ++w2)
        if (sval[w2] > bb || (sval[w2] == bb && sidx[w2] < id)) { bb = sval[w2]; id = sidx[w2]; }
      piv_s = id;
      ipiv[j0 + jj] = j0 + id;
      if (!(sqrt(bb) >= kPivotTiny) && *info == 0) *info = j0 + jj + 1;
    }
    __syncthreads();
    const int p = piv_s;
    if (p != jj && tid < kPB) {
      const double2 t = P[jj * kPB + tid];
      P[jj * kPB + tid] = P[p * kPB + tid];
      P[p * kPB + tid] = t;
    }
    __syncthreads();
    const double2 d = P[jj * kPB + jj];
    const bool ok = cabs2(d) > 0.0;
    for (int r = jj + 1 + tid; r < rows; r += kPanelThreads) {
      const double2 l = ok ? cdiv(P[r * kPB + jj], d) : P[r * kPB + jj];
      P[r * kPB + jj] = l;
#pragma unroll
      for (int c = 0; c < kPB; ++c)
        if (c > jj) cfma(P[r * kPB + c], make_double2(-l.x, -l.y), P[jj * kPB + c]);
    }
    __syncthreads();
  }
  for (int e = tid; e < rows * kPB; e += kPanelThreads) {
    const int r = e / kPB, c = e - r * kPB;
    if (c < pb) A[static_cast<int64_t>(j0 + r) * lda + j0 + c] = P[e];
  }
}

// apply the interchanges ipiv[j0 .. j0+cnt) to every column outside [j0, j0+cnt)
__global__ void laswp_cols(double2* A, int n, int lda, int j0, int cnt, const int* ipiv) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n || (c >= j0 && c < j0 + cnt)) return;
  for (int jj = 0; jj < cnt; ++jj) {
    const int r = j0 + jj, p = ipiv[r];
    if (p != r) {
      const double2 t = A[static_cast<int64_t>(r) * lda + c];
      A[static_cast<int64_t>(r) * lda + c] = A[static_cast<int64_t>(p) * lda + c];
      A[static_cast<int64_t>(p) * lda + c] = t;
    }
  }
}

constexpr int kTrsmWarps = 8;

// X = T^-1 X on the nb (<= NB) rows [r0, r0+nb) of X (row stride ldx), T = the diagonal block
// LU[r0.., r0..] (unit lower, or upper), staged in shared memory.  One warp per column of X
// (columns [c0, c0+ncols)): lane l holds rows l, l+32, ...; the substitution broadcasts the
// solved entry with a shuffle and updates the remaining rows in parallel.
template <int NB>
__global__ void __launch_bounds__(kTrsmWarps * 32) trsm_block(const double2* LU, int lda, double2* X, int64_t ldx,
                                                               int r0, int nb, int c0, int ncols, int upper) {
  extern __shared__ double2 trsm_smem[];
  double2 (*T)[NB + 1] = reinterpret_cast<double2 (*)[NB + 1]>(trsm_smem);
  for (int e = threadIdx.x; e < nb * nb; e += kTrsmWarps * 32) {
    const int i = e / nb, k = e - i * nb;
    T[i][k] = LU[static_cast<int64_t>(r0 + i) * lda + r0 + k];
  }
  __syncthreads();
  constexpr int R = NB / 32;
  const int lane = threadIdx.x & 31;
  const int c = c0 + blockIdx.x * kTrsmWarps + (threadIdx.x >> 5);
  if (c >= c0 + ncols) return;
  double2 x[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int i = lane + 32 * q;
    x[q] = (i < nb) ? X[static_cast<int64_t>(r0 + i) * ldx + c] : make_double2(0, 0);
  }
  if (!upper) {
    for (int k = 0; k < nb - 1; ++k) {
      const int qk = k >> 5;
      double2 xk;
#pragma unroll
      for (int q = 0; q < R; ++q)
        if (q == qk) {
          xk.x = __shfl_sync(0xffffffffu, x[q].x, k & 31);
          xk.y = __shfl_sync(0xffffffffu, x[q].y, k & 31);
        }
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int i = lane + 32 * q;
        if (i > k && i < nb) cfma(x[q], make_double2(-T[i][k].x, -T[i][k].y), xk);
      }
    }
  } else {
    for (int k = nb - 1; k >= 0; --k) {
      const int qk = k >> 5;
      double2 xk;
#pragma unroll
      for (int q = 0; q < R; ++q)
        if (q == qk) {
          if (lane == (k & 31)) x[q] = cdiv(x[q], T[k][k]);
          xk.x = __shfl_sync(0xffffffffu, x[q].x, k & 31);
          xk.y = __shfl_sync(0xffffffffu, x[q].y, k & 31);
        }
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int i = lane + 32 * q;
        if (i < k) cfma(x[q], make_double2(-T[i][k].x, -T[i][k].y), xk);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int i = lane + 32 * q;
    if (i < nb) X[static_cast<int64_t>(r0 + i) * ldx + c] = x[q];
  }
}

template <int NB>
void trsm(const double2* LU, int lda, double2* X, int64_t ldx, int r0, int nb, int c0, int ncols, int upper,
          cudaStream_t s) {
  constexpr int smem = NB * (NB + 1) * static_cast<int>(sizeof(double2));
  static bool configured = false;  // opt-in above 48 KB, once per process
  if (!configured) {
    cudaFuncSetAttribute(trsm_block<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    configured = true;
  }
  trsm_block<NB><<<(ncols + kTrsmWarps - 1) / kTrsmWarps, kTrsmWarps * 32, smem, s>>>(LU, lda, X, ldx, r0, nb, c0, ncols,
                                                                                  upper);
}

// perm[i] = source row of position i after the interchanges ipiv[0..n) (one thread; n <= 8192)
__global__ void build_perm(const int* ipiv, int n, int* perm) {
  extern __shared__ int pm[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) pm[i] = i;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 0; j < n; ++j) {
      const int p = ipiv[j];
      const int t = pm[j];
      pm[j] = pm[p];
      pm[p] = t;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = pm[i];
}

__global__ void gather_rows(const double2* __restrict__ B, double2* __restrict__ out, const int* __restrict__ perm,
                            int n, int nrhs, int64_t ldb) {
  const int64_t total = static_cast<int64_t>(n) * nrhs;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = t / nrhs, c = t - i * nrhs;
    out[i * ldb + c] = B[static_cast<int64_t>(perm[i]) * ldb + c];
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

// in-place LU with partial pivoting of the n x n row-major A; info (device) > 0: singular.
// Blocked right-looking: outer blocks of kOB columns; inside, kPB-column sub-panels factored in
// shared memory (lu_subpanel), their interchanges applied to all other columns, the sub-panel's
// U rows solved and the rest of the outer block updated; then the outer block's U12 = L11^-1 A12
// (trsm_block) and the trailing update A22 -= L21 U12 on the tensor cores (K = kOB).
int getrf(double2* A, int n, int* ipiv, int* info, cudaStream_t s) {
  const size_t psmem = sizeof(double2) * static_cast<size_t>(n) * kPB;
  TOEP_REQUIRE(psmem <= 227 * 1024, TOEP_ERR_ARG, "lu_factor: n = %d exceeds the shared-memory sub-panel (<= 1816)", n);
  static size_t attr = 0;
  if (psmem > 48 * 1024 && attr < psmem) {
    TOEP_CUDA(cudaFuncSetAttribute(lu_subpanel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem));
    attr = psmem;
  }
  for (int j0 = 0; j0 < n; j0 += kOB) {
    const int ob = std::min(kOB, n - j0);
    for (int jj = j0; jj < j0 + ob; jj += kPB) {
      const int pb = std::min(kPB, j0 + ob - jj);
      lu_subpanel<<<1, kPanelThreads, sizeof(double2) * static_cast<size_t>(n - jj) * kPB, s>>>(A, n, n, jj, ipiv, info);
      TOEP_LAUNCHED();
      laswp_cols<<<(n + 255) / 256, 256, 0, s>>>(A, n, n, jj, pb, ipiv);
      TOEP_LAUNCHED();
      const int c0 = jj + pb, ncol = j0 + ob - c0;  // rest of the outer block
      if (ncol > 0) {
        trsm<32>(A, n, A, n, jj, pb, c0, ncol, 0, s);
        TOEP_LAUNCHED();
        const int rows = n - c0;
        if (rows > 0)
          TOEP_TRY(gemm_rm(rows, ncol, pb, make_double2(-1, 0), A + static_cast<int64_t>(c0) * n + jj, n,
                           A + static_cast<int64_t>(jj) * n + c0, n, make_double2(1, 0),
                           A + static_cast<int64_t>(c0) * n + c0, n, s));
      }
    }
    const int c0 = j0 + ob, rest = n - c0;
    if (rest > 0) {
      trsm<32>(A, n, A, n, j0, ob, c0, rest, 0, s);
      TOEP_LAUNCHED();
      TOEP_TRY(gemm_rm(rest, rest, ob, make_double2(-1, 0), A + static_cast<int64_t>(c0) * n + j0, n,
                       A + static_cast<int64_t>(j0) * n + c0, n, make_double2(1, 0),
                       A + static_cast<int64_t>(c0) * n + c0, n, s));
    }
  }
  return TOEP_OK;
}

// B <- A^-1 B with A = P L U from getrf; B: n x nrhs row-major (ldb)
int getrs(const double2* LU, int n, const int* ipiv, double2* B, int ldb, int nrhs, cudaStream_t s) {
  int* perm = nullptr;
  double2* tmp = nullptr;
  TOEP_REQUIRE(cudaMallocAsync(reinterpret_cast<void**>(&perm), sizeof(int) * n, s) == cudaSuccess &&
                   cudaMallocAsync(reinterpret_cast<void**>(&tmp), sizeof(double2) * static_cast<size_t>(n) * ldb, s) ==
                       cudaSuccess,
               TOEP_ERR_OOM, "out of device memory in lu_solve");
  build_perm<<<1, 256, sizeof(int) * n, s>>>(ipiv, n, perm);
  TOEP_LAUNCHED();
  const int64_t total = static_cast<int64_t>(n) * nrhs;
  const int gg = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  gather_rows<<<gg, 256, 0, s>>>(B, tmp, perm, n, nrhs, ldb);
  TOEP_LAUNCHED();
  TOEP_CUDA(cudaMemcpyAsync(B, tmp, sizeof(double2) * static_cast<size_t>(n) * ldb, cudaMemcpyDeviceToDevice, s));
  cudaFreeAsync(tmp, s);
  cudaFreeAsync(perm, s);
  constexpr int kSB = 64;  // solve block: halves the GEMM count of the 32-row LU block
  for (int r0 = 0; r0 < n; r0 += kSB) {  // L y = P b (unit lower)
    const int nb = std::min(kSB, n - r0);
    trsm<kSB>(LU, n, B, ldb, r0, nb, 0, nrhs, 0, s);
    TOEP_LAUNCHED();
    const int rest = n - r0 - nb;
    if (rest > 0)
      TOEP_TRY(gemm_rm(rest, nrhs, nb, make_double2(-1, 0), LU + static_cast<int64_t>(r0 + nb) * n + r0, n,
                       B + static_cast<int64_t>(r0) * ldb, ldb, make_double2(1, 0), B + static_cast<int64_t>(r0 + nb) * ldb,
                       ldb, s));
  }
  for (int r1 = n; r1 > 0; r1 -= kSB) {  // U x = y
    const int r0 = std::max(0, r1 - kSB);
    const int nb = r1 - r0;
    trsm<kSB>(LU, n, B, ldb, r0, nb, 0, nrhs, 1, s);
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
