// Block Rybicki (bordering) direct solver on the device: rybicki.py:63-144 + numerics.lu_factor /
// lu_solve (numerics.py:67-96).
//
// Every block sum of the recursion (d1, d2, the numerators) is ONE complex GEMM of depth m*s on
// the FP64 tensor cores (three real DMMA GEMMs of dmma.cu, 3M) against "wide" copies of the generator blocks, and the
// generator cross-updates are single batched GEMMs (negative batch stride walks the reversed
// block order).  The two denominators per step are LU-factored together on the device with
// partial pivoting (LAPACK zgetrf semantics, |re|+|im| pivots): kPW-column panels factored by an
// 8-CTA cluster with the panel resident in distributed shared memory, the row permutation and
// U12 solve in one warp-per-column kernel, the trailing update on the tensor cores.  Solves are
// blocked triangular solves whose off-diagonal work is again GEMM.  All matrices are row-major
// complex128.  Singular pivots (|p| < 1e-300, numerics.py:27) raise SingularBlock for R_0 and
// SingularDenominator(step) for D1 / D2, as the reference.
#include <climits>
#include <vector>

#include <cooperative_groups.h>

#include "op.h"

namespace toep {
namespace {

namespace cg = cooperative_groups;

constexpr double kPivotTiny = 1e-300;


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
  __shared__ double2 rdiag[NB];
  constexpr int R = NB / 32;
  constexpr int kRowsPerWarp = NB / kTrsmWarps;
  const int lane = threadIdx.x & 31, wrp = threadIdx.x >> 5;
  {  // stage the diagonal block: all loads issued before any store (one latency, not NB*NB/256)
    double2 v[kRowsPerWarp][R];
#pragma unroll
    for (int t = 0; t < kRowsPerWarp; ++t)
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int i = wrp + t * kTrsmWarps, k = lane + 32 * q;
        v[t][q] = (i < nb && k < nb) ? LU[static_cast<int64_t>(r0 + i) * lda + r0 + k] : make_double2(0, 0);
      }
#pragma unroll
    for (int t = 0; t < kRowsPerWarp; ++t)
#pragma unroll
      for (int q = 0; q < R; ++q) T[wrp + t * kTrsmWarps][lane + 32 * q] = v[t][q];
  }
  __syncthreads();
  if (upper && threadIdx.x < nb) {  // reciprocal pivots: the substitution chain multiplies
    const double2 d = T[threadIdx.x][threadIdx.x];
    const double r = 1.0 / (d.x * d.x + d.y * d.y);
    rdiag[threadIdx.x] = make_double2(d.x * r, -d.y * r);
  }
  __syncthreads();
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
          if (lane == (k & 31)) x[q] = cmul(x[q], rdiag[k]);
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
  static_assert(NB % kTrsmWarps == 0 && NB % 32 == 0, "trsm block");
  constexpr int smem = NB * (NB + 1) * static_cast<int>(sizeof(double2));
  ensure_smem(trsm_block<NB>, smem);
  trsm_block<NB><<<(ncols + kTrsmWarps - 1) / kTrsmWarps, kTrsmWarps * 32, smem, s>>>(LU, lda, X, ldx, r0, nb, c0, ncols,
                                                                                  upper);
}

// ----------------------------------------------------------------------------- cluster panel LU
// The kPW-column panel [j0, j0+kPW) over all rows [j0, n) is factored by one 8-CTA thread-block
// cluster, the panel resident in the cluster's distributed shared memory (CTA r owns physical rows
// [r*rpc, (r+1)*rpc)).  Rows never move during the panel: per column, every CTA proposes its
// local pivot candidate (max |re|+|im|, LAPACK izamax's measure), one cluster barrier publishes
// the candidates, every warp reads the winner and the pivot row straight from the owner's shared
// memory (DSMEM) and each thread eliminates the rows it owns.  The row interchanges are tracked as
// a permutation (LAPACK ipiv semantics) and applied once, at write-back; `moves` receives the
// (destination, source) row pairs so the other columns can be permuted by swap_trsm.
#ifndef TOEP_PANEL_CL
#define TOEP_PANEL_CL 8
#endif
constexpr int kCL = TOEP_PANEL_CL;
constexpr int kPW = 32;
constexpr int kMovesStride = 1 + 4 * kPW;  // count + up to 2*kPW (dst, src) pairs

__device__ __forceinline__ double cabs1(double2 a) { return fabs(a.x) + fabs(a.y); }

__device__ __forceinline__ void argmax_merge(double& v, int& i, double ov, int oi) {
  if (ov > v || (ov == v && oi < i)) { v = ov; i = oi; }
}

__device__ __forceinline__ void warp_argmax(double& v, int& i) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, off);
    const int oi = __shfl_xor_sync(0xffffffffu, i, off);
    argmax_merge(v, i, ov, oi);
  }
}

// explicit distributed-shared-memory stores (st.shared::cluster on a mapa'd address)
__device__ __forceinline__ uint32_t dsmem_addr(const void* local, uint32_t rank) {
  uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(local)), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void dsmem_st_c128(uint32_t a, double2 v) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void dsmem_st_f64(uint32_t a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void dsmem_st_s32(uint32_t a, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
size_t panel_smem(int n, int j0) { return 2 * sizeof(int) * static_cast<size_t>(n - j0); }

// Panel rows live in registers, each row split over kTPR adjacent lanes (kCPT columns each):
// thread t of CTA r owns columns (t % kTPR)*kCPT .. +kCPT of physical rows
// r*rpc + t / kTPR + q*kRowsPass, q < RPT.
#ifndef TOEP_PANEL_TPR
#define TOEP_PANEL_TPR 2  // lanes per panel row (measured: 2 -> 105 us, 4 -> 121 us, 8 -> 134 us per 1024-row panel)
#endif
constexpr int kTPR = TOEP_PANEL_TPR;
constexpr int kPanelThr2 = 128 * kTPR;
constexpr int kCPT = kPW / kTPR;                 // 8 columns per thread
constexpr int kRowsPass = kPanelThr2 / kTPR;     // 128 rows per pass

template <int RPT>
__device__ __forceinline__ double2 pick(const double2 (&a)[RPT][kCPT], int q, int k) {
  double2 v = make_double2(0, 0);
#pragma unroll
  for (int qq = 0; qq < RPT; ++qq)
#pragma unroll
    for (int kk = 0; kk < kCPT; ++kk)
      if (qq == q && kk == k) v = a[qq][kk];
  return v;
}

#ifdef TOEP_PANEL_PROBE
__device__ long long g_probe[kCL][8];
#endif

template <int RPT>
__global__ void __cluster_dims__(kCL, 1, 1) __launch_bounds__(kPanelThr2, 1)
    lu_panel_cluster(double2* A0, int64_t mstride, int n, int j0, int* ipiv0, int* info0, int* moves0) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  double2* A = A0 + blockIdx.y * mstride;
  int* ipiv = ipiv0 + static_cast<int64_t>(blockIdx.y) * n;
  int* info = info0 + blockIdx.y;
  int* moves = moves0 + blockIdx.y * kMovesStride;
  const int R = n - j0, pw = min(kPW, R);
  const int rpc = (R + kCL - 1) / kCL;
  const int row0 = rank * rpc, nrow = max(0, min(R, row0 + rpc) - row0);
  extern __shared__ int panel_sm[];
  int* pos_of = panel_sm;     // [R]
  int* phys_at = pos_of + R;  // [R]
  // inbox: every CTA pushes its candidate (|pivot|, row index, row) into every CTA's inbox slot
  // [column parity][source rank] with remote stores before the cluster barrier, so that after
  // the barrier all pivot decisions read local shared memory only
  __shared__ double2 ib_row[2][kCL][kPW];
  __shared__ double ib_v[2][kCL];
  __shared__ int ib_i[2][kCL];
  __shared__ double wv[2][kPanelThr2 / 32];
  __shared__ int wi[2][kPanelThr2 / 32];
  __shared__ int nmoves;
  __shared__ int spiv[kPW];  // ipiv of the panel, written to global memory once at the end
  __shared__ int sinfo;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sub = tid % kTPR, rl = tid / kTPR, cbase = sub * kCPT;

  double2 a[RPT][kCPT];
  bool used[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int i = rl + q * kRowsPass;
    used[q] = !(i < nrow);
    const double2* src = A + static_cast<int64_t>(j0 + row0 + (used[q] ? 0 : i)) * n + j0 + cbase;
#pragma unroll
    for (int k = 0; k < kCPT; ++k) a[q][k] = (!used[q] && cbase + k < pw) ? src[k] : make_double2(0, 0);
  }
  for (int i = tid; i < R; i += kPanelThr2) {
    pos_of[i] = i;
    phys_at[i] = i;
  }
  if (tid == 0) {
    nmoves = 0;
    sinfo = 0;
  }
  __syncthreads();

#ifdef TOEP_PANEL_PROBE
#define PROBE(k)                        \
  do {                                  \
    const long long t1 = clock64();     \
    acc[k] += t1 - tp;                  \
    tp = t1;                            \
  } while (0)
  long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tp = clock64();
#else
#define PROBE(k)
#endif
  for (int jj = 0; jj < pw; ++jj) {
    const int par = jj & 1, jc = jj / kCPT, jk = jj % kCPT;
    const bool mine = (sub == jc);  // this thread holds column jj of its rows
    double best = -1.0;
    int bi = INT_MAX;
#pragma unroll
    for (int q = 0; q < RPT; ++q)
      if (mine && !used[q]) argmax_merge(best, bi, cabs1(pick<RPT>(a, q, jk)), row0 + rl + q * kRowsPass);
    warp_argmax(best, bi);
    PROBE(0);
    if (lane == 0) {
      wv[par][warp] = best;
      wi[par][warp] = bi;
    }
    __syncthreads();
    PROBE(1);
    double cb = lane < kPanelThr2 / 32 ? wv[par][lane] : -1.0;
    int cix = lane < kPanelThr2 / 32 ? wi[par][lane] : INT_MAX;
    warp_argmax(cb, cix);
#pragma unroll
    for (int q = 0; q < RPT; ++q)  // the CTA's candidate row is pushed by its kTPR owners
      if (!used[q] && row0 + rl + q * kRowsPass == cix) {
#pragma unroll
        for (int d = 0; d < kCL; ++d) {
          const uint32_t dst = dsmem_addr(&ib_row[par][rank][cbase], d);
#pragma unroll
          for (int k = 0; k < kCPT; ++k) dsmem_st_c128(dst + k * 16, a[q][k]);
        }
      }
    if (tid < kCL) {
      dsmem_st_f64(dsmem_addr(&ib_v[par][rank], tid), cb);
      dsmem_st_s32(dsmem_addr(&ib_i[par][rank], tid), cix);
    }
    PROBE(2);
    cluster.sync();
    PROBE(3);
    double gpv = lane < kCL ? ib_v[par][lane] : -1.0;
    int p = lane < kCL ? ib_i[par][lane] : INT_MAX;
    warp_argmax(gpv, p);
    const int owner = p / rpc;
    if (tid == 0) {  // interchange bookkeeping (redundantly in every CTA)
      const int ppos = pos_of[p], phj = phys_at[jj];
      phys_at[jj] = p;
      phys_at[ppos] = phj;
      pos_of[p] = jj;
      pos_of[phj] = ppos;
      spiv[jj] = j0 + ppos;
      if (!(gpv >= kPivotTiny) && sinfo == 0) sinfo = j0 + jj + 1;
    }
    PROBE(4);
    const bool zero = !(gpv >= kPivotTiny);
    const double2 piv = ib_row[par][owner][jj];
    // multiplier = a / piv as a * (1 / piv): one reciprocal per column, as LAPACK's zgetf2 scales
    const double rden = zero ? 0.0 : 1.0 / (piv.x * piv.x + piv.y * piv.y);
    const double2 rpiv = make_double2(piv.x * rden, -piv.y * rden);
    double2 u[kCPT];
#pragma unroll
    for (int k = 0; k < kCPT; ++k) u[k] = ib_row[par][owner][cbase + k];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      bool act = !used[q];
      if (act && row0 + rl + q * kRowsPass == p) {
        used[q] = true;
        act = false;
      }
      double2 l = pick<RPT>(a, q, jk);
      if (!zero) l = cmul(l, rpiv);
      // the multiplier lives with the column-jj owner of the row; share it across the row's lanes
      const int src = (lane & ~(kTPR - 1)) | jc;
      l.x = __shfl_sync(0xffffffffu, l.x, src);
      l.y = __shfl_sync(0xffffffffu, l.y, src);
      const double2 nl = make_double2(-l.x, -l.y);
#pragma unroll
      for (int k = 0; k < kCPT; ++k) {
        const int c = cbase + k;
        if (act && c > jj) cfma(a[q][k], nl, u[k]);
        if (act && c == jj) a[q][k] = l;
      }
    }
  }
#ifdef TOEP_PANEL_PROBE
  if (tid == 0)
    for (int k = 0; k < 8; ++k) g_probe[rank][k] = acc[k];
#endif
  cluster.sync();  // remote reads done; pos_of final
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int i = rl + q * kRowsPass;
    if (i < nrow) {
      double2* dst = A + static_cast<int64_t>(j0 + pos_of[row0 + i]) * n + j0 + cbase;
#pragma unroll
      for (int k = 0; k < kCPT; ++k)
        if (cbase + k < pw) dst[k] = a[q][k];
    }
  }
  if (rank == 0) {
    if (tid < pw) ipiv[j0 + tid] = spiv[tid];
    if (tid == 0 && sinfo != 0 && *info == 0) *info = sinfo;
    for (int q = tid; q < R; q += kPanelThr2)
      if (phys_at[q] != q) {
        const int k = atomicAdd(&nmoves, 1);
        moves[1 + 2 * k] = q;
        moves[2 + 2 * k] = phys_at[q];
      }
    __syncthreads();
    if (tid == 0) moves[0] = nmoves;
  }
}

// Columns outside the panel: apply the panel's row permutation (moves), then, right of the
// panel, U12 = L11^-1 A12 (unit lower, L11 in shared memory).  One warp per column; lane = row.
__global__ void __launch_bounds__(256) swap_trsm(double2* A0, int64_t mstride, int n, int j0, int pw,
                                                 const int* moves0) {
  double2* A = A0 + blockIdx.y * mstride;
  const int* moves = moves0 + blockIdx.y * kMovesStride;
  __shared__ double2 L[kPW][kPW + 1];
  __shared__ int mv[kMovesStride];
  const int tid = threadIdx.x, lane = tid & 31;
  const int cnt = moves[0];
  for (int e = tid; e < 2 * cnt; e += 256) mv[e] = moves[1 + e];
  {
    double2 v[kPW / 8];
#pragma unroll
    for (int t = 0; t < kPW / 8; ++t) {
      const int i = (tid >> 5) + 8 * t;
      v[t] = (i < pw && lane < pw) ? A[static_cast<int64_t>(j0 + i) * n + j0 + lane] : make_double2(0, 0);
    }
#pragma unroll
    for (int t = 0; t < kPW / 8; ++t) L[(tid >> 5) + 8 * t][lane] = v[t];
  }
  __syncthreads();
  const int t = blockIdx.x * 8 + (tid >> 5);
  if (t >= n - pw) return;
  const int c = t < j0 ? t : t + pw;
  double2 v0 = make_double2(0, 0), v1 = make_double2(0, 0);
  if (lane < cnt) v0 = A[static_cast<int64_t>(j0 + mv[2 * lane + 1]) * n + c];
  if (lane + 32 < cnt) v1 = A[static_cast<int64_t>(j0 + mv[2 * lane + 65]) * n + c];
  __syncwarp();
  if (lane < cnt) A[static_cast<int64_t>(j0 + mv[2 * lane]) * n + c] = v0;
  if (lane + 32 < cnt) A[static_cast<int64_t>(j0 + mv[2 * lane + 64]) * n + c] = v1;
  __syncwarp();
  if (c < j0 + pw) return;
  double2 x = lane < pw ? A[static_cast<int64_t>(j0 + lane) * n + c] : make_double2(0, 0);
  for (int k = 0; k < pw - 1; ++k) {
    double2 xk;
    xk.x = __shfl_sync(0xffffffffu, x.x, k);
    xk.y = __shfl_sync(0xffffffffu, x.y, k);
    if (lane > k && lane < pw) cfma(x, make_double2(-L[lane][k].x, -L[lane][k].y), xk);
  }
  if (lane < pw) A[static_cast<int64_t>(j0 + lane) * n + c] = x;
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

// 3M complex products (Gauss): A B = (Ar Br - Ai Bi) + i ((Ar + Ai)(Br + Bi) - Ar Br - Ai Bi), three
// real FP64 tensor-core GEMMs instead of the four real products of a complex GEMM.  Operands are
// split into planes (re, im, re + im) with a common leading dimension.
struct Planes {
  double* re = nullptr;
  double* im = nullptr;
  double* sm = nullptr;
  int64_t ld = 0;
  Planes at(int64_t off) const { return Planes{re + off, im + off, sm + off, ld}; }
};

__global__ void k_split3(const double2* __restrict__ src, int64_t rows, int64_t cols, int64_t lds, Planes d) {
  const int64_t total = rows * cols;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / cols, c = t - r * cols;
    const double2 v = src[r * lds + c];
    const int64_t o = r * d.ld + c;
    d.re[o] = v.x;
    d.im[o] = v.y;
    d.sm[o] = v.x + v.y;
  }
}

// C += sign * ((T1 - T2) + i (T3 - T1 - T2)),  C and T: rows x cols with leading dims ldc / ldt
__global__ void k_combine3(Planes t, int64_t rows, int64_t cols, double2* __restrict__ c, int64_t ldc, double sign) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, q = i - r * cols;
    const int64_t o = r * t.ld + q;
    const double t1 = t.re[o], t2 = t.im[o], t3 = t.sm[o];
    double2 v = c[r * ldc + q];
    v.x += sign * (t1 - t2);
    v.y += sign * (t3 - t1 - t2);
    c[r * ldc + q] = v;
  }
}

int split3(const double2* src, int64_t rows, int64_t cols, int64_t lds, const Planes& d, cudaStream_t st) {
  const int grid = static_cast<int>(std::min<int64_t>((rows * cols + 255) / 256, 148 * 16));
  k_split3<<<grid, 256, 0, st>>>(src, rows, cols, lds, d);
  TOEP_LAUNCHED();
  return TOEP_OK;
}

int combine3(const Planes& t, int64_t rows, int64_t cols, double2* c, int64_t ldc, double sign, cudaStream_t st) {
  const int grid = static_cast<int>(std::min<int64_t>((rows * cols + 255) / 256, 148 * 16));
  k_combine3<<<grid, 256, 0, st>>>(t, rows, cols, c, ldc, sign);
  TOEP_LAUNCHED();
  return TOEP_OK;
}

// T_p = A_p B_p for p in (re, im, sm), batched (row-major planes, batch strides in doubles)
int gemm3(int64_t m, int64_t n, int64_t k, const Planes& a, int64_t a_bs, const Planes& b, int64_t b_bs,
          const Planes& t, int64_t t_bs, int64_t batch, cudaStream_t st) {
  // the three plane products in one launch (3x the CTAs of one product: fewer partial waves)
  const double* ap[3] = {a.re, a.im, a.sm};
  const double* bp[3] = {b.re, b.im, b.sm};
  double* tp[3] = {t.re, t.im, t.sm};
  const int rc = dgemm_dmma_planes(m, n, k, 1.0, ap, a.ld, 1, a_bs, bp, b.ld, 1, b_bs, 0.0, tp, t.ld, 1, t_bs, batch, 3,
                                   st, nullptr);
  if (rc < 0) {
    set_error("gemm3: unsupported operand layout");
    return TOEP_ERR_ARG;
  }
  return rc;
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

// In-place LU with partial pivoting of `batch` n x n row-major matrices spaced mstride apart
// (LAPACK getrf semantics: ipiv 0-based absolute rows, info > 0 = first zero pivot, 1-based).
// Right-looking, kPW-column panels: cluster panel factorisation (lu_panel_cluster), the row
// permutation + U12 solve for the other columns (swap_trsm), then the trailing update
// A22 -= L21 U12 on the tensor cores (K = kPW), batched over the matrices.
int getrf_batched(double2* A, int64_t mstride, int batch, int n, int* ipiv, int* info, cudaStream_t s) {
  const size_t psmem = panel_smem(n, 0);
  const int rpc = (n + kCL - 1) / kCL;
  TOEP_REQUIRE(rpc <= 4 * kRowsPass, TOEP_ERR_ARG, "lu_factor: n = %d exceeds the cluster-resident panel (n <= 4096)",
               n);
  TOEP_CUDA(ensure_smem(lu_panel_cluster<1>, psmem));
  TOEP_CUDA(ensure_smem(lu_panel_cluster<2>, psmem));
  TOEP_CUDA(ensure_smem(lu_panel_cluster<4>, psmem));
  int* moves = nullptr;
  TOEP_REQUIRE(cudaMallocAsync(reinterpret_cast<void**>(&moves), sizeof(int) * kMovesStride * batch, s) == cudaSuccess,
               TOEP_ERR_OOM, "out of device memory in lu_factor");
  TOEP_CUDA(cudaMemsetAsync(info, 0, sizeof(int) * batch, s));
  int rc = TOEP_OK;
  for (int j0 = 0; j0 < n && rc == TOEP_OK; j0 += kPW) {
    const int pw = std::min(kPW, n - j0);
    const int rows_cta = (n - j0 + kCL - 1) / kCL;
    const dim3 pg(kCL, batch);
    const size_t ps = panel_smem(n, j0);
    if (rows_cta <= kRowsPass)
      lu_panel_cluster<1><<<pg, kPanelThr2, ps, s>>>(A, mstride, n, j0, ipiv, info, moves);
    else if (rows_cta <= 2 * kRowsPass)
      lu_panel_cluster<2><<<pg, kPanelThr2, ps, s>>>(A, mstride, n, j0, ipiv, info, moves);
    else
      lu_panel_cluster<4><<<pg, kPanelThr2, ps, s>>>(A, mstride, n, j0, ipiv, info, moves);
    if (cudaGetLastError() != cudaSuccess) {
      set_error("lu_panel_cluster launch failed");
      rc = TOEP_ERR_CUDA;
      break;
    }
    if (n - pw > 0) {
      swap_trsm<<<dim3((n - pw + 7) / 8, batch), 256, 0, s>>>(A, mstride, n, j0, pw, moves);
      if (cudaGetLastError() != cudaSuccess) {
        set_error("swap_trsm launch failed");
        rc = TOEP_ERR_CUDA;
        break;
      }
    }
    const int c0 = j0 + pw, rest = n - c0;
    if (rest > 0)
      rc = gemm(TOEP_C128, rest, rest, pw, make_double2(-1, 0), A + static_cast<int64_t>(c0) * n + j0, n, 1, mstride,
                A + static_cast<int64_t>(j0) * n + c0, n, 1, mstride, make_double2(1, 0),
                A + static_cast<int64_t>(c0) * n + c0, n, 1, mstride, batch, s);
  }
  cudaFreeAsync(moves, s);
  return rc;
}

int getrf(double2* A, int n, int* ipiv, int* info, cudaStream_t s) { return getrf_batched(A, 0, 1, n, ipiv, info, s); }

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

namespace toep {
namespace {

// assemble_level1 (rybicki.py:53-60): out[p][i*n0 + a][j*n0 + b] = s4[p][(i - j) mod k1][a][b].
// One CTA per output row (p, i, a): n1 runs of n0 contiguous elements, each a contiguous run of the
// generator row (L2-resident: every generator row feeds n1 output rows), stores fully coalesced.
__global__ void __launch_bounds__(256) k_assemble_level1(const double2* __restrict__ s4, int n1, int n0,
                                                         double2* __restrict__ out) {
  const int k1 = 2 * n1 - 1;
  const int64_t row = blockIdx.x;  // (p * n1 + i) * n0 + a
  const int a = static_cast<int>(row % n0);
  const int64_t pi = row / n0;
  const int i = static_cast<int>(pi % n1);
  const int64_t p = pi / n1;
  const int64_t side = static_cast<int64_t>(n1) * n0;
  double2* dst = out + row * side;
  const double2* src = s4 + p * k1 * static_cast<int64_t>(n0) * n0 + static_cast<int64_t>(a) * n0;
  for (int64_t e = threadIdx.x; e < side; e += blockDim.x) {
    const int j = static_cast<int>(e / n0), b = static_cast<int>(e - static_cast<int64_t>(j) * n0);
    int q = i - j;
    if (q < 0) q += k1;
    dst[e] = __ldg(src + static_cast<int64_t>(q) * n0 * n0 + b);
  }
}

}  // namespace
}  // namespace toep

extern "C" int toep_assemble_level1(const void* stacked4, int n2, int n1, int n0, void* out, void* stream) {
  TOEP_NVTX("toep_assemble_level1");
  TOEP_REQUIRE(stacked4 != nullptr && out != nullptr && stacked4 != out, TOEP_ERR_ARG, "bad assemble_level1 buffers");
  TOEP_REQUIRE(n2 >= 1 && n1 >= 1 && n0 >= 1, TOEP_ERR_SHAPE, "n2, n1, n0 must be positive");
  const int64_t rows = static_cast<int64_t>(2 * n2 - 1) * n1 * n0;
  TOEP_REQUIRE(rows <= 0x7fffffff, TOEP_ERR_SHAPE, "assemble_level1: too many rows");
  toep::k_assemble_level1<<<static_cast<unsigned>(rows), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const double2*>(stacked4), n1, n0, static_cast<double2*>(out));
  TOEP_LAUNCHED();
  return TOEP_OK;
}

extern "C" int toep_lu_factor(void* a, int n, int* ipiv, int* info, void* stream) {
  TOEP_NVTX("toep_lu_factor");
  TOEP_REQUIRE(a != nullptr && ipiv != nullptr && info != nullptr && n >= 1, TOEP_ERR_ARG, "bad lu_factor args");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return getrf(static_cast<double2*>(a), n, ipiv, info, s);
}

extern "C" int toep_lu_solve(const void* lu, int n, const int* ipiv, void* b, int64_t nrhs, void* stream) {
  TOEP_REQUIRE(lu != nullptr && ipiv != nullptr && b != nullptr && n >= 1, TOEP_ERR_ARG, "bad lu_solve args");
  return getrs(static_cast<const double2*>(lu), n, ipiv, static_cast<double2*>(b), static_cast<int>(nrhs),
               static_cast<int>(nrhs), static_cast<cudaStream_t>(stream));
}

extern "C" int toep_rybicki(const void* blocks_v, int N, int s, const void* y_v, void* x_v, int64_t w,
                            int* fail_step, toep_stage_fn hook, void* hook_ctx, void* stream) {
  TOEP_NVTX("toep_rybicki");
  TOEP_REQUIRE(blocks_v != nullptr && y_v != nullptr && x_v != nullptr && N >= 1 && s >= 1 && w >= 1, TOEP_ERR_ARG,
               "bad rybicki arguments");
  // The recursion runs on two library streams: `st` (highest priority) carries the latency-bound
  // chain — the cluster LU of the denominators, the triangular solves, the denominator updates — and
  // `s2` (lowest priority) the tensor-core block sums and cross-updates.  With equal priorities the
  // GEMM CTAs held every SM and each LU panel launch waited for SMs to drain: the LU of a step grew
  // from 3.7 to 12 ms as the block sums deepened.  The caller's stream `sc` is ordered before and after.
  const cudaStream_t sc = static_cast<cudaStream_t>(stream);
  cudaStream_t st = nullptr;
  keep_pool();
  const double2* blocks = static_cast<const double2*>(blocks_v);
  const double2* y = static_cast<const double2*>(y_v);
  double2* x = static_cast<double2*>(x_v);  // (N, s, w): x_j at x + j*s*w
  const int64_t ss = static_cast<int64_t>(s) * s, sw = static_cast<int64_t>(s) * w;
  const int nb2 = 2 * N - 1;
  auto rb = [&](int o) { return blocks + static_cast<int64_t>(((o % nb2) + nb2) % nb2) * ss; };
  if (fail_step) *fail_step = -1;

  double2 *g = nullptr, *h = nullptr, *gtmp = nullptr, *lu0 = nullptr, *lu12 = nullptr, *wide = nullptr;
  double2 *d12 = nullptr, *num_save = nullptr;  // unfactored D1 / D2; copies of the step's H / G numerators
  int *piv0 = nullptr, *piv12 = nullptr, *info = nullptr;
  double *wplanes = nullptr, *scr = nullptr;  // 3M: planes of the wide blocks; per-stream B / T scratch
  int8_t *oz_a = nullptr, *oz_b = nullptr;    // Ozaki digits: wide planes (once), per-stream G / H stack planes
  int32_t *oz_aexp = nullptr, *oz_bexp = nullptr;
  // side stream: the block sums that do not depend on the step's LU factors run on it while the
  // (latency-bound, few-SM) cluster LU of D1/D2 runs on `st`
  cudaStream_t s2 = nullptr;
  cudaEvent_t ev_step = nullptr, ev_sums = nullptr, ev_solved = nullptr;
  constexpr bool overlap = true;  // side stream (cfg5: 184 ms vs 217 ms with every kernel on one stream)
  auto cleanup = [&]() {
    if (s2 != nullptr) {
      cudaStreamSynchronize(s2);
      cudaStreamDestroy(s2);
    }
    if (st == nullptr) return;
    if (ev_step != nullptr) cudaEventDestroy(ev_step);
    if (ev_sums != nullptr) cudaEventDestroy(ev_sums);
    if (ev_solved != nullptr) cudaEventDestroy(ev_solved);
    for (void* q : {(void*)g, (void*)h, (void*)gtmp, (void*)lu0, (void*)lu12, (void*)wide, (void*)piv0, (void*)piv12,
                    (void*)info, (void*)wplanes, (void*)scr, (void*)d12, (void*)num_save, (void*)oz_a, (void*)oz_b,
                    (void*)oz_aexp, (void*)oz_bexp})
      if (q) cudaFreeAsync(q, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  };
  int rc = TOEP_OK;
  {
    int lo = 0, hi = 0;
    TOEP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    TOEP_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, hi));
    cudaEvent_t e0 = nullptr;
    TOEP_CUDA(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
    cudaEventRecord(e0, sc);  // inputs were produced on the caller's stream
    cudaStreamWaitEvent(st, e0, 0);
    cudaEventDestroy(e0);
  }
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
  R_ALLOC(g, N * ss);  // G_1..G_m stacked (+1 slot for G_new)
  R_ALLOC(h, N * ss);
  R_ALLOC(gtmp, N * ss);
  R_ALLOC(lu0, ss);
  R_ALLOC(lu12, 4 * ss);  // D1, D2 factored together; two sets by step parity (the side stream still
                          // solves with step m's factors while step m+1 is factored)
  R_ALLOC(d12, 2 * ss);
  R_ALLOC(num_save, 4 * ss);  // two sets by step parity (the side stream fills the next while st reads this)
  R_ALLOC(piv0, s);
  R_ALLOC(piv12, 4 * s);
  R_ALLOC(info, 2 * (N + 1));  // per step: checked at the end unless a step hook needs them at once
  // Block sums over k become single GEMMs of depth m*s against "wide" copies of the generator
  // blocks, s x (N-1)s row-major each:  Wp = [R_1 .. R_{N-1}],  Wpr = [R_{N-1} .. R_1],
  // Wn = [R_-1 .. R_-(N-1)],  Wnr = [R_-(N-1) .. R_-1].
  const int64_t wld = static_cast<int64_t>(nm1) * s, wsz = static_cast<int64_t>(s) * wld;
  if (N > 1) {
    R_ALLOC(wide, 4 * wsz);
    for (int t = 0; t < N - 1; ++t) {
      const double2* src[4] = {rb(t + 1), rb(N - 1 - t), rb(-(t + 1)), rb(-(N - 1 - t))};
      for (int q = 0; q < 4; ++q)
        TOEP_CUDA(cudaMemcpy2DAsync(wide + q * wsz + static_cast<int64_t>(t) * s, wld * sizeof(double2), src[q],
                                    s * sizeof(double2), s * sizeof(double2), s, cudaMemcpyDeviceToDevice, st));
    }
  }
  double2 *Wp = wide, *Wpr = wide + wsz, *Wn = wide + 2 * wsz, *Wnr = wide + 3 * wsz;
  // 3M products for the s x s block products (TOEP_RYB_3M=0: complex GEMMs)
  // 3M (Gauss) products for the s x s block products: 3 real DMMA GEMMs instead of a complex one
  constexpr bool use3m = true;
  Planes wp[4];
  // Block sums of depth >= kOzMinK on the int8 tensor cores (Ozaki, ozaki.cu): 1.8x the DMMA rate at
  // depth 15 360, break-even near 4 096 (tools/ozaki_gemm_time.py); depth <= 19 000 keeps the digit
  // sums exact in int32
#ifndef TOEP_RYB_OZAKI
#define TOEP_RYB_OZAKI 1
#endif
  constexpr int64_t kOzMinK = 4096;
  const bool use_oz = TOEP_RYB_OZAKI != 0 && use3m && N > 1 && s % 128 == 0 && static_cast<int64_t>(N - 1) * s >= kOzMinK &&
                      static_cast<int64_t>(N - 1) * s <= 19000;
  Planes bsc[2], tsc[2];  // per stream (st, s2): B planes (N s x s) and T planes (N s x s)
  if (use3m && N > 1) {
    R_ALLOC(wplanes, 12 * wsz);
    for (int q = 0; q < 4; ++q) {
      wp[q] = Planes{wplanes + (3 * q) * wsz, wplanes + (3 * q + 1) * wsz, wplanes + (3 * q + 2) * wsz, wld};
      R_TRY(split3(wide + q * wsz, s, wld, wld, wp[q], st));
    }
    const int64_t pl = static_cast<int64_t>(N) * ss;  // one plane
    R_ALLOC(scr, 2 * 2 * 3 * pl);
    for (int k = 0; k < 2; ++k) {
      double* base = scr + static_cast<int64_t>(k) * 6 * pl;
      bsc[k] = Planes{base, base + pl, base + 2 * pl, s};
      tsc[k] = Planes{base + 3 * pl, base + 4 * pl, base + 5 * pl, s};
    }
    if (use_oz) {  // row digits of the 12 wide planes, cut once per solve (exponents over whole rows)
      R_ALLOC(oz_a, 12 * ozaki_rows_bytes(s, wld));
      R_ALLOC(oz_aexp, 12 * static_cast<int64_t>(s));
      R_ALLOC(oz_b, 2 * 3 * ozaki_cols_bytes(s, wld));
      R_ALLOC(oz_bexp, 2 * 3 * ozaki_cols_exps(s));
      for (int q = 0; q < 4; ++q)
        R_TRY(ozaki_slice_rows(wp[q].re, wld, wsz, 3, s, wld, oz_a + 3 * q * ozaki_rows_bytes(s, wld),
                               oz_aexp + 3 * q * static_cast<int64_t>(s), st));
    }
  }
  double2 *lu1 = lu12, *lu2 = lu12 + ss;
  int *piv1 = piv12, *piv2 = piv12 + s;
  auto use_factor_set = [&](int par) {
    lu1 = lu12 + par * 2 * ss;
    lu2 = lu1 + ss;
    piv1 = piv12 + par * 2 * s;
    piv2 = piv1 + s;
  };
  const double2 one = make_double2(1, 0), mone = make_double2(-1, 0);
  auto check_info = [&](int code, int step, int count) -> int {
    int hinfo[2] = {0, 0};
    TOEP_CUDA(cudaMemcpyAsync(hinfo, info + 2 * step, sizeof(int) * count, cudaMemcpyDeviceToHost, st));
    TOEP_CUDA(cudaStreamSynchronize(st));
    if (hinfo[0] != 0 || (count > 1 && hinfo[1] != 0)) {
      if (fail_step) *fail_step = step;
      set_error(code == TOEP_ERR_SINGULAR_BLOCK ? "self block R_0 is singular"
                                                : "singular denominator at bordering step %d", step);
      return code;
    }
    return TOEP_OK;
  };
  auto stage_hook = [&](int stage) -> int {
    if (hook == nullptr) return TOEP_OK;
    TOEP_CUDA(cudaStreamSynchronize(st));  // (the caller synchronised s2 into st first)
    TOEP_REQUIRE(hook(hook_ctx, stage, x, g, h, stream) == 0, TOEP_ERR_ARG, "rybicki step hook failed");
    return TOEP_OK;
  };
  // C (+)= alpha * W[:, t0*s : (t0+m)*s] @ stack(m blocks of s x ncol), one GEMM of depth m*s
  auto wide_gemm = [&](const double2* W, int t0, int m, const double2* B, int64_t ncol, double2* C,
                       cudaStream_t sx) {
    if (use3m && ncol == s) {  // G / H stacks: 3 real tensor-core GEMMs of depth m*s
      const int k = sx == st ? 0 : 1;
      const int64_t q = (W - wide) / wsz;
      const Planes& a = wp[q];
      TOEP_TRY(split3(B, static_cast<int64_t>(m) * s, s, s, bsc[k], sx));
      const int64_t depth = static_cast<int64_t>(m) * s;
      if (use_oz && depth >= kOzMinK) {
        const int64_t pl = static_cast<int64_t>(N) * ss;
        int8_t* bdig = oz_b + static_cast<int64_t>(k) * 3 * ozaki_cols_bytes(s, wld);
        int32_t* bexp = oz_bexp + static_cast<int64_t>(k) * 3 * ozaki_cols_exps(s);
        TOEP_TRY(ozaki_slice_cols(bsc[k].re, s, pl, 3, s, depth, bdig, bexp, sx));
        OzGemm og{};
        og.asl = oz_a + 3 * q * ozaki_rows_bytes(s, wld);
        og.aexp = oz_aexp + 3 * q * static_cast<int64_t>(s);
        og.a_kcs = wld / 32; og.a_k0 = static_cast<int64_t>(t0) * s; og.a_z0 = 0; og.a_zo = 0; og.a_zp = 1;
        og.bsl = bdig; og.bexp = bexp; og.b_z0 = 0; og.b_zo = 0; og.b_zp = 1;
        og.c = tsc[k].re; og.ldc = s; og.c_zo = 0; og.c_zp = pl;
        og.alpha = 1.0; og.beta = 0.0;
        og.M = s; og.N = s; og.K = depth; og.planes = 3; og.zcount = 3;
        TOEP_TRY(ozaki_gemm(og, sx));
        return combine3(tsc[k], s, s, C, s, 1.0, sx);
      }
      TOEP_TRY(gemm3(s, s, static_cast<int64_t>(m) * s, a.at(static_cast<int64_t>(t0) * s), 0, bsc[k], 0, tsc[k], 0, 1,
                     sx));
      return combine3(tsc[k], s, s, C, s, 1.0, sx);
    }
    return gemm_rm(s, ncol, static_cast<int64_t>(m) * s, one, W + static_cast<int64_t>(t0) * s, wld, B, ncol, one, C,
                   ncol, sx);
  };
  if (overlap && N > 1) {
    {
      int lo = 0, hi = 0;
      TOEP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      TOEP_CUDA(cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, lo));
    }
    TOEP_CUDA(cudaEventCreateWithFlags(&ev_step, cudaEventDisableTiming));
    TOEP_CUDA(cudaEventCreateWithFlags(&ev_sums, cudaEventDisableTiming));
    TOEP_CUDA(cudaEventCreateWithFlags(&ev_solved, cudaEventDisableTiming));
  }
  cudaStream_t ss2 = s2 != nullptr ? s2 : st;
  // C_b (+)= alpha * A_{m-1-b} @ B for b = 0..m-1 (A blocks s x s stacked, reversed), one batched GEMM
  auto rev_batched = [&](const double2* Astack, int m, const double2* B, int64_t ncol, double2* C, int64_t c_bs,
                         cudaStream_t sx) {
    if (use3m && ncol == s && c_bs == ss) {  // C stack -= reversed A stack x B, as 3 batched real GEMMs
      const int k = sx == st ? 0 : 1;  // the stream's own scratch planes
      TOEP_TRY(split3(Astack, static_cast<int64_t>(m) * s, s, s, bsc[k], sx));       // A stack planes
      const Planes bb = tsc[k].at(static_cast<int64_t>(m) * ss);                       // B planes after T
      TOEP_TRY(split3(B, s, s, s, bb, sx));
      TOEP_TRY(gemm3(s, s, s, bsc[k].at(static_cast<int64_t>(m - 1) * ss), -ss, bb, 0, tsc[k], ss, m, sx));
      return combine3(tsc[k], static_cast<int64_t>(m) * s, s, C, s, -1.0, sx);
    }
    return gemm(TOEP_C128, s, ncol, s, mone, Astack + static_cast<int64_t>(m - 1) * ss, s, 1, -ss, B, ncol, 1, 0, one,
                C, ncol, 1, c_bs, m, sx);
  };

  // base stage (rybicki.py:94-108)
  TOEP_CUDA(cudaMemcpyAsync(lu0, rb(0), ss * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  R_TRY(getrf(lu0, s, piv0, info, st));
  R_TRY(check_info(TOEP_ERR_SINGULAR_BLOCK, 0, 1));
  TOEP_CUDA(cudaMemcpyAsync(x, y, sw * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  R_TRY(getrs(lu0, s, piv0, x, static_cast<int>(w), static_cast<int>(w), st));
  if (N > 1) {
    TOEP_CUDA(cudaMemcpyAsync(g, rb(-1), ss * sizeof(double2), cudaMemcpyDeviceToDevice, st));
    TOEP_CUDA(cudaMemcpyAsync(h, rb(1), ss * sizeof(double2), cudaMemcpyDeviceToDevice, st));
    // G_1 and H_1 share the factor: one solve with 2s right-hand sides would need them side by
    // side; two solves keep the stacked layout.
    R_TRY(getrs(lu0, s, piv0, g, s, s, st));
    R_TRY(getrs(lu0, s, piv0, h, s, s, st));
  }
  R_TRY(stage_hook(1));

  // Denominators.  The reference forms d1 = sum_{k<=m} R_k G_k - R_0 and d2 = sum_{k<=m} R_-k H_k - R_0
  // afresh every step (rybicki.py:114,125), two block sums of depth m*s.  Substituting the step's
  // cross-updates G_k' = G_k - H_{m+1-k} G_new, G_{m+1}' = G_new (and H_k' likewise) into the next
  // step's sums gives, exactly in exact arithmetic,
  //     d1(m+1) = d1(m) - hnum(m) G_new(m),    d2(m+1) = d2(m) - gnum(m) H_new(m),
  // with hnum = sum_j R_{m+1-j} H_j - R_{m+1} and gnum = sum_j R_{j-m-1} G_j - R_-(m+1) the
  // numerators this step already forms (rybicki.py:126-127): one s x s product each instead of a
  // depth-m*s sum, a third fewer tensor-core flops over the solve.  It also takes the next LU off
  // the cross-updates' path: D1 / D2 are ready as soon as the step's solves are, so the (few-SM,
  // latency-bound) cluster LU of step m+1 runs on `st` while the side stream does step m's x and
  // G / H cross-updates and step m+1's block sums.
  double2 *D1 = d12, *D2 = d12 + ss;
  if (N > 1) {
    R_TRY(copy_neg(rb(0), D1, ss, -1.0, st));
    R_TRY(wide_gemm(Wp, 0, 1, g, s, D1, st));
    if (N > 2) {
      R_TRY(copy_neg(rb(0), D2, ss, -1.0, st));
      R_TRY(wide_gemm(Wn, 0, 1, h, s, D2, st));
    }
  }
  for (int m = 1; m < N; ++m) {
    const bool more = m < N - 1;
    double2* xn = x + m * sw;
    double2* gnew = gtmp + m * ss;  // slot m of the next G stack
    double2* hnew = h + m * ss;     // slot m of H
    double2* hsave = num_save + (m & 1) * 2 * ss;  // this step's numerators, kept for the D updates
    double2* gsave = hsave + ss;
    if (m == 1 && s2 != nullptr) {  // the side stream starts after the base stage
      TOEP_CUDA(cudaEventRecord(ev_step, st));
      TOEP_CUDA(cudaStreamWaitEvent(s2, ev_step, 0));
    }
    // side stream (after the previous step's cross-updates, queued there): the right-hand sides of
    // this step's three solves, independent of the D1 / D2 factors —
    //   x_{m+1} <- sum_j R_{m+1-j} x_j - y_{m+1},  G_new <- gnum,  H_new <- hnum
    R_TRY(copy_neg(y + m * sw, xn, sw, -1.0, ss2));
    R_TRY(wide_gemm(Wpr, N - 1 - m, m, x, w, xn, ss2));
    if (more) {
      R_TRY(copy_neg(rb(-(m + 1)), gnew, ss, -1.0, ss2));
      R_TRY(wide_gemm(Wnr, N - 1 - m, m, g, s, gnew, ss2));
      R_TRY(copy_neg(rb(m + 1), hnew, ss, -1.0, ss2));
      R_TRY(wide_gemm(Wpr, N - 1 - m, m, h, s, hnew, ss2));
      if (m + 1 < N - 1)  // the numerators for the next step's D2 / D1 update
        TOEP_CUDA(cudaMemcpyAsync(gsave, gnew, ss * sizeof(double2), cudaMemcpyDeviceToDevice, ss2));
      TOEP_CUDA(cudaMemcpyAsync(hsave, hnew, ss * sizeof(double2), cudaMemcpyDeviceToDevice, ss2));
    }
    if (s2 != nullptr) TOEP_CUDA(cudaEventRecord(ev_sums, s2));
    // D1, D2 of this step, factored together (copies: the unfactored matrices take the next update)
    use_factor_set(m & 1);
    TOEP_CUDA(cudaMemcpyAsync(lu1, d12, (more ? 2 : 1) * ss * sizeof(double2), cudaMemcpyDeviceToDevice, st));
    R_TRY(getrf_batched(lu1, ss, more ? 2 : 1, s, piv1, info + 2 * m, st));
    // With a step hook the failure must surface before the next stage runs (rybicki.py raises
    // SingularDenominator(m) at once); otherwise the host does not wait for each LU — every step's
    // info is read back once at the end and the first failing step reported (a singular step's
    // later results are discarded with x).
    if (hook != nullptr) R_TRY(check_info(TOEP_ERR_SINGULAR_DENOM, m, more ? 2 : 1));
    if (s2 != nullptr) TOEP_CUDA(cudaStreamWaitEvent(st, ev_sums, 0));
    // G_new = D2^-1 gnum on the side stream (latency-bound blocked TRSM chain), concurrently with
    // x_{m+1} = D1^-1 (...) and H_new = D1^-1 hnum here
    if (more && s2 != nullptr) {
      TOEP_CUDA(cudaEventRecord(ev_step, st));
      TOEP_CUDA(cudaStreamWaitEvent(s2, ev_step, 0));
      R_TRY(getrs(lu2, s, piv2, gnew, s, s, s2));
      TOEP_CUDA(cudaEventRecord(ev_sums, s2));
      // x_{m+1} = D1^-1 (...) also here: nothing on the main stream's chain (the next LU) needs it
      R_TRY(getrs(lu1, s, piv1, xn, static_cast<int>(w), static_cast<int>(w), s2));
    } else {
      R_TRY(getrs(lu1, s, piv1, xn, static_cast<int>(w), static_cast<int>(w), st));
    }
    if (more) {
      if (s2 == nullptr) R_TRY(getrs(lu2, s, piv2, gnew, s, s, st));
      R_TRY(getrs(lu1, s, piv1, hnew, s, s, st));
      if (s2 != nullptr) {
        TOEP_CUDA(cudaEventRecord(ev_solved, st));  // H_new
        TOEP_CUDA(cudaStreamWaitEvent(st, ev_sums, 0));  // G_new
      }
      // next step's denominators (on st, ahead of its LU): D1 -= hnum G_new, D2 -= gnum H_new
      if (m + 1 < N) {
        R_TRY(gemm(TOEP_C128, s, s, s, mone, hsave, s, 1, 0, gnew, s, 1, 0, one, D1, s, 1, 0, 1, st, nullptr));
        if (m + 1 < N - 1)
          R_TRY(gemm(TOEP_C128, s, s, s, mone, gsave, s, 1, 0, hnew, s, 1, 0, one, D2, s, 1, 0, 1, st, nullptr));
      }
      // side stream: x_j -= G_{m+1-j} x_{m+1};  G_j' = G_j - H_{m+1-j} G_new (old H, into the next
      // stack);  H_j -= G_{m+1-j} H_new (old G)
      if (s2 != nullptr) TOEP_CUDA(cudaStreamWaitEvent(s2, ev_solved, 0));
      R_TRY(rev_batched(g, m, xn, w, x, sw, ss2));
      TOEP_CUDA(cudaMemcpyAsync(gtmp, g, m * ss * sizeof(double2), cudaMemcpyDeviceToDevice, ss2));
      R_TRY(rev_batched(h, m, gnew, s, gtmp, ss, ss2));
      R_TRY(rev_batched(g, m, hnew, s, h, ss, ss2));
      std::swap(g, gtmp);
    } else {
      R_TRY(rev_batched(g, m, xn, w, x, sw, st));  // last step: x_j -= G_{m+1-j} x_{m+1}
    }
    if (hook != nullptr && s2 != nullptr) {  // the hook sees the finished stage
      TOEP_CUDA(cudaEventRecord(ev_step, s2));
      TOEP_CUDA(cudaStreamWaitEvent(st, ev_step, 0));
    }
    R_TRY(stage_hook(m + 1));
  }
  if (s2 != nullptr) {  // everything queued on the side stream is ordered before the return
    TOEP_CUDA(cudaEventRecord(ev_step, s2));
    TOEP_CUDA(cudaStreamWaitEvent(st, ev_step, 0));
  }
  TOEP_CUDA(cudaStreamSynchronize(st));  // x is complete before the caller's stream uses it
  if (hook == nullptr && N > 1) {  // deferred denominator checks, first failing step
    std::vector<int> hinfo(2 * N, 0);
    TOEP_CUDA(cudaMemcpy(hinfo.data(), info, sizeof(int) * 2 * N, cudaMemcpyDeviceToHost));
    for (int m = 1; m < N; ++m)
      if (hinfo[2 * m] != 0 || (m < N - 1 && hinfo[2 * m + 1] != 0)) {
        if (fail_step) *fail_step = m;
        set_error("singular denominator at bordering step %d", m);
        cleanup();
        return TOEP_ERR_SINGULAR_DENOM;
      }
  }
  cleanup();
#undef R_ALLOC
#undef R_TRY
  return TOEP_OK;
}
