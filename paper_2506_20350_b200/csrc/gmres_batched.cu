// Batched per-column GMRES: solve_multi_rhs_sequential (solvers/gmres.py:304-336) for all
// columns at once.
//
// The reference solves each right-hand-side column with its own _gmres_block (n x 1).  Here
// every column keeps its own Krylov basis, Hessenberg columns, Givens rotations, residual
// history and stop flag, but all columns advance in lock step so that each Arnoldi step is
// ONE multi-RHS matvec over the (n, W) block: the per-bin product becomes a complex GEMM
// on the FP64 tensor cores (zgemm_tc, 256x256 x 256xW per bin at cfg3).  Columns that have
// stopped (converged, breakdown or iteration cap) are frozen: their Gram-Schmidt, Givens
// and solution updates are masked, so each column's iterate and report are those of an
// independent solve.  Cycle boundaries coincide for all columns (same restart length).
//
// Per-column reductions run over row chunks: thread = column (coalesced over the W
// contiguous columns of a row), partials [l][chunk][column] are reduced in fixed order.
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "launch.cuh"
#include "op.h"

namespace toep {
namespace {

constexpr int kCols = 64;   // columns per CTA in the row-chunked kernels
constexpr int kLG = 8;      // basis vectors per accumulation group

struct BCol {               // per-column state (arrays of length W)
  double* beta0;
  int* stop;                // 0 running, 1 converged/breakdown, 2 cycle exhausted / cap
  int* conv;
  int* brk;
  int* m;                   // completed steps in the current cycle
  int* total;
  int* nhist;
};

__device__ __forceinline__ int64_t rows_begin(int chunk, int nchunks, int64_t n) {
  return n * chunk / nchunks;
}

// One-sweep CGS2 (Gram-matrix form), per column: partial[l] = V_l^H w and partial2[l] =
// V_l^H V_{m-1} (the newest basis vector's Gram column) in the same basis sweep
constexpr int kLGG = 4;
// The groups of kLGG basis vectors of one (row chunk, column tile) run side by side on threadIdx.y
// (up to kGramGroups per CTA), so the rows of w and v_{m-1} that every group needs come from HBM
// once and from L1 for the other groups (one group after the other re-read them from HBM).
constexpr int kGramGroups = 4;
__global__ void __launch_bounds__(kCols * kGramGroups) kb_dots_gram(const double2* const* __restrict__ Vp, int m,
                                                      const double2* __restrict__ w, int64_t n, int W, int nchunks,
                                                      double2* __restrict__ partial, double2* __restrict__ partial2) {
  pdl_wait();
  pdl_trigger();
  const int c = blockIdx.y * kCols + threadIdx.x;
  if (c >= W) return;
  const int chunk = blockIdx.x;
  const int64_t r0 = rows_begin(chunk, nchunks, n), r1 = rows_begin(chunk + 1, nchunks, n);
  const double2* vl = Vp[m - 1];
  for (int l0 = threadIdx.y * kLGG; l0 < m; l0 += blockDim.y * kLGG) {
    double2 acc[kLGG], acg[kLGG];
    const double2* vp[kLGG];
#pragma unroll
    for (int g = 0; g < kLGG; ++g) {
      acc[g] = acg[g] = make_double2(0, 0);
      vp[g] = Vp[l0 + g < m ? l0 + g : m - 1];
    }
    int64_t i = r0;
    // two rows per iteration, every load issued before the first use (the sweep is latency-bound:
    // ncu long-scoreboard stalls at 32 resident warps per SM); same accumulation order as one row
    for (; i + 1 < r1; i += 2) {
      const int64_t o0 = i * W + c, o1 = o0 + W;
      const double2 w0 = w[o0], w1 = w[o1], a0 = vl[o0], a1 = vl[o1];
      double2 x0[kLGG], x1[kLGG];
#pragma unroll
      for (int g = 0; g < kLGG; ++g) {
        x0[g] = l0 + g < m ? __ldg(vp[g] + o0) : make_double2(0, 0);
        x1[g] = l0 + g < m ? __ldg(vp[g] + o1) : make_double2(0, 0);
      }
#pragma unroll
      for (int g = 0; g < kLGG; ++g)
        if (l0 + g < m) {
          cfmac(acc[g], x0[g], w0);
          cfmac(acg[g], x0[g], a0);
          cfmac(acc[g], x1[g], w1);
          cfmac(acg[g], x1[g], a1);
        }
    }
    for (; i < r1; ++i) {
      const double2 wi = w[i * W + c], li = vl[i * W + c];
#pragma unroll
      for (int g = 0; g < kLGG; ++g)
        if (l0 + g < m) {
          const double2 v = vp[g][i * W + c];
          cfmac(acc[g], v, wi);
          cfmac(acg[g], v, li);
        }
    }
#pragma unroll
    for (int g = 0; g < kLGG; ++g)
      if (l0 + g < m) {
        partial[(static_cast<int64_t>(l0 + g) * nchunks + chunk) * W + c] = acc[g];
        partial2[(static_cast<int64_t>(l0 + g) * nchunks + chunk) * W + c] = acg[g];
      }
  }
}

// h1[l][c] = sum_chunk partial; Gram column G[l][m-1] = sum_chunk partial2 (stored with its conjugate
// row; gram[(k*ldr + l)*W + c] = G[l][k]).  CTA (column tile of 32, l): warp g sums chunks g, g+32, ...
// in two interleaved chains, then warp 0 adds the 32 group sums in order (fixed, run-to-run
// identical).  A thread per (l, c) walking all row chunks serially was latency-bound: 1.5 ms per
// step at cfg3; 8 warps with one chain each still were (one dependent 7 KB-strided load per ~1.2 us:
// 450 us per Gram reduction, 755 us per norm reduction of the 4 736 x 900 partials).
constexpr int kRedGroups = 32;
__global__ void __launch_bounds__(kRedGroups * 32) kb_reduce_gram(const double2* __restrict__ partial,
                                                                  const double2* __restrict__ partial2, int m,
                                                                  int nchunks, int W, double2* __restrict__ h1,
                                                                  double2* __restrict__ gram, int ldr,
                                                                  const int* __restrict__ stop) {
  pdl_wait();
  pdl_trigger();
  __shared__ double2 r1[kRedGroups][32], r2[kRedGroups][32];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane, l = blockIdx.y;
  double2 s1 = make_double2(0, 0), s2 = make_double2(0, 0);
  if (c < W && !stop[c]) {
    const double2* p1 = partial + static_cast<int64_t>(l) * nchunks * W + c;
    const double2* p2 = partial2 + static_cast<int64_t>(l) * nchunks * W + c;
    double2 t1 = make_double2(0, 0), t2 = make_double2(0, 0);
    int ch = grp;
    for (; ch + kRedGroups < nchunks; ch += 2 * kRedGroups) {
      const double2 a1 = p1[static_cast<int64_t>(ch) * W], b1 = p1[static_cast<int64_t>(ch + kRedGroups) * W];
      const double2 a2 = p2[static_cast<int64_t>(ch) * W], b2 = p2[static_cast<int64_t>(ch + kRedGroups) * W];
      s1 = cadd(s1, a1);
      t1 = cadd(t1, b1);
      s2 = cadd(s2, a2);
      t2 = cadd(t2, b2);
    }
    if (ch < nchunks) {
      s1 = cadd(s1, p1[static_cast<int64_t>(ch) * W]);
      s2 = cadd(s2, p2[static_cast<int64_t>(ch) * W]);
    }
    s1 = cadd(s1, t1);
    s2 = cadd(s2, t2);
  }
  r1[grp][lane] = s1;
  r2[grp][lane] = s2;
  __syncthreads();
  if (grp != 0 || c >= W || stop[c]) return;
#pragma unroll
  for (int g = 1; g < kRedGroups; ++g) {
    s1 = cadd(s1, r1[g][lane]);
    s2 = cadd(s2, r2[g][lane]);
  }
  h1[static_cast<int64_t>(l) * W + c] = s1;
  gram[(static_cast<int64_t>(m - 1) * ldr + l) * W + c] = s2;
  gram[(static_cast<int64_t>(l) * ldr + (m - 1)) * W + c] = make_double2(s2.x, -s2.y);
}

// nsum[c] = sum_chunk part[chunk][c] (squared-norm partials), same fixed-order two-level reduction;
// the per-column kernels (init, cycle start, Givens) then read one value per column
__global__ void __launch_bounds__(kRedGroups * 32) kb_norm_reduce(const double* __restrict__ part, int nchunks, int W,
                                                                  double* __restrict__ nsum) {
  pdl_wait();
  pdl_trigger();
  __shared__ double r[kRedGroups][32];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  double sacc = 0.0;
  if (c < W) {
    double tacc = 0.0;
    int ch = grp;
    for (; ch + kRedGroups < nchunks; ch += 2 * kRedGroups) {
      const double a = part[static_cast<int64_t>(ch) * W + c], b = part[static_cast<int64_t>(ch + kRedGroups) * W + c];
      sacc += a;
      tacc += b;
    }
    if (ch < nchunks) sacc += part[static_cast<int64_t>(ch) * W + c];
    sacc += tacc;
  }
  r[grp][lane] = sacc;
  __syncthreads();
  if (grp != 0 || c >= W) return;
#pragma unroll
  for (int g = 1; g < kRedGroups; ++g) sacc += r[g][lane];
  nsum[c] = sacc;
}

// per column: h = h1 + (h1 - G h1) (the second CGS pass from the Gram matrix) -> h, Hessenberg column;
// one thread per (column, l)
__global__ void kb_coef_gram(const double2* __restrict__ h1, const double2* __restrict__ gram, int m, int ldr, int W,
                             double2* __restrict__ h, double2* __restrict__ hcol, const int* __restrict__ stop) {
  pdl_wait();
  pdl_trigger();
  const int c = blockIdx.x * blockDim.x + threadIdx.x, l = blockIdx.y;
  if (c >= W || stop[c]) return;
  double2 t = make_double2(0, 0);
  for (int k = 0; k < m; ++k)
    cfma(t, gram[(static_cast<int64_t>(k) * ldr + l) * W + c], h1[static_cast<int64_t>(k) * W + c]);
  const double2 a = h1[static_cast<int64_t>(l) * W + c];
  const double2 hv = make_double2(2.0 * a.x - t.x, 2.0 * a.y - t.y);
  h[static_cast<int64_t>(l) * W + c] = hv;
  hcol[static_cast<int64_t>(l) * W + c] = hv;
}

// w[:, c] -= sum_l V_l[:, c] h[l][c]  (active columns); mode 1: partial dots of the result,
// mode 2: ||w[:, c]||^2 partials
__global__ void __launch_bounds__(kCols) kb_upd(const double2* const* __restrict__ Vp, int m,
                                                const double2* __restrict__ h, double2* __restrict__ w, int64_t n,
                                                int W, int nchunks, int mode, double2* __restrict__ partial,
                                                double* __restrict__ norm_part, const int* __restrict__ stop) {
  pdl_wait();
  pdl_trigger();
  const int c = blockIdx.y * kCols + threadIdx.x;
  if (c >= W || stop[c]) return;
  const int chunk = blockIdx.x;
  const int64_t r0 = rows_begin(chunk, nchunks, n), r1 = rows_begin(chunk + 1, nchunks, n);
  double nrm = 0.0;
  // coefficients in register blocks of kLG (each thread owns one column): w is swept
  // ceil(m / kLG) times, the basis once
  for (int l0 = 0; l0 < m; l0 += kLG) {
    double2 cl[kLG];
#pragma unroll
    for (int g = 0; g < kLG; ++g) {
      const double2 hv = (l0 + g < m) ? h[static_cast<int64_t>(l0 + g) * W + c] : make_double2(0, 0);
      cl[g] = make_double2(-hv.x, -hv.y);
    }
    const bool last = (l0 + kLG >= m);
    const double2* vp[kLG];
#pragma unroll
    for (int g = 0; g < kLG; ++g) vp[g] = Vp[l0 + g < m ? l0 + g : m - 1];
    int64_t i = r0;
    for (; i + 1 < r1; i += 2) {  // two rows per iteration, loads first (as kb_dots_gram)
      const int64_t o0 = i * W + c, o1 = o0 + W;
      double2 acc0 = w[o0], acc1 = w[o1];
      double2 x0[kLG], x1[kLG];
#pragma unroll
      for (int g = 0; g < kLG; ++g) {
        x0[g] = l0 + g < m ? __ldg(vp[g] + o0) : make_double2(0, 0);
        x1[g] = l0 + g < m ? __ldg(vp[g] + o1) : make_double2(0, 0);
      }
#pragma unroll
      for (int g = 0; g < kLG; ++g)
        if (l0 + g < m) {
          cfma(acc0, x0[g], cl[g]);
          cfma(acc1, x1[g], cl[g]);
        }
      w[o0] = acc0;
      w[o1] = acc1;
      if (last) {
        nrm = fma(acc0.x, acc0.x, fma(acc0.y, acc0.y, nrm));
        nrm = fma(acc1.x, acc1.x, fma(acc1.y, acc1.y, nrm));
      }
    }
    for (; i < r1; ++i) {
      double2 acc = w[i * W + c];
#pragma unroll
      for (int g = 0; g < kLG; ++g)
        if (l0 + g < m) cfma(acc, vp[g][i * W + c], cl[g]);
      w[i * W + c] = acc;
      if (last) nrm = fma(acc.x, acc.x, fma(acc.y, acc.y, nrm));
    }
  }
  if (mode == 2) {
    norm_part[static_cast<int64_t>(chunk) * W + c] = nrm;
    return;
  }
  for (int l0 = 0; l0 < m; l0 += kLG) {
    double2 a[kLG];
#pragma unroll
    for (int g = 0; g < kLG; ++g) a[g] = make_double2(0, 0);
    for (int64_t i = r0; i < r1; ++i) {
      const double2 wi = w[i * W + c];
#pragma unroll
      for (int g = 0; g < kLG; ++g)
        if (l0 + g < m) cfmac(a[g], Vp[l0 + g][i * W + c], wi);
    }
#pragma unroll
    for (int g = 0; g < kLG; ++g)
      if (l0 + g < m) partial[(static_cast<int64_t>(l0 + g) * nchunks + chunk) * W + c] = a[g];
  }
}

// ||x[:, c]||^2 partials over row chunks (all columns)
__global__ void __launch_bounds__(kCols) kb_norm(const double2* __restrict__ x, int64_t n, int W, int nchunks,
                                                 double* __restrict__ norm_part) {
  pdl_wait();
  pdl_trigger();
  const int c = blockIdx.y * kCols + threadIdx.x;
  if (c >= W) return;
  const int chunk = blockIdx.x;
  const int64_t r0 = rows_begin(chunk, nchunks, n), r1 = rows_begin(chunk + 1, nchunks, n);
  double nrm = 0.0;
  for (int64_t i = r0; i < r1; ++i) {
    const double2 v = x[i * W + c];
    nrm = fma(v.x, v.x, fma(v.y, v.y, nrm));
  }
  norm_part[static_cast<int64_t>(chunk) * W + c] = nrm;
}

__device__ __forceinline__ double colnorm(const double* part, int nchunks, int W, int c) {
  double s = 0.0;
  for (int ch = 0; ch < nchunks; ++ch) s += part[static_cast<int64_t>(ch) * W + c];
  return sqrt(s);
}

__global__ void kb_init(BCol st, const double* norm_part, int nchunks, int W, double* hist) {
  pdl_wait();
  pdl_trigger();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= W) return;
  const double b0 = colnorm(norm_part, nchunks, W, c);
  st.beta0[c] = b0;
  st.stop[c] = (b0 == 0.0) ? 1 : 0;
  st.conv[c] = 1;  // provisional; cleared at the first cycle start of a non-trivial column
  st.brk[c] = 0;
  st.m[c] = 0;
  st.total[c] = 0;
  st.nhist[c] = 1;
  hist[c] = (b0 == 0.0) ? 0.0 : 1.0;
}

// cycle start: beta = ||z[:, c]||, test, g[0] = beta, inv for V[0] scaling
__global__ void kb_cycle_start(BCol st, const double* norm_part, int nchunks, int W, double tol, double2* g,
                               double* inv, int first, int* active) {
  pdl_wait();
  pdl_trigger();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= W) return;
  if (first) {
    if (st.beta0[c] == 0.0) { inv[c] = 0.0; return; }
    st.conv[c] = 0;
  } else if (st.conv[c] || st.brk[c] || st.stop[c] == 3) {
    inv[c] = 0.0;
    return;
  }
  const double beta = colnorm(norm_part, nchunks, W, c);
  st.m[c] = 0;
  if (beta / st.beta0[c] <= tol) {
    st.conv[c] = 1;
    st.stop[c] = 1;
    inv[c] = 0.0;
  } else {
    st.stop[c] = 0;
    g[c] = make_double2(beta, 0.0);
    inv[c] = 1.0 / beta;
    atomicAdd(active, 1);
  }
}

// per-column Givens step (gmres.py:160-189); hcol layout [i][c] with row stride ldh
__global__ void kb_givens(BCol st, const double* norm_part, int nchunks, int W, double2* rcols, int ldr, double* cs,
                          double2* sn, double2* g, double* hist, double* inv, double tol, int max_total, int cycle_len,
                          int* active) {
  pdl_wait();
  pdl_trigger();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= W) return;
  if (st.stop[c]) {  // frozen column: its next basis vector is exactly zero (no NaN can leak)
    inv[c] = 0.0;
    return;
  }
  const double hnext = colnorm(norm_part, nchunks, W, c);
  const int j = st.m[c];
  double2* hcol = rcols + static_cast<int64_t>(j) * ldr * W;  // element i at hcol[i*W + c]
  for (int i = 0; i < j; ++i) {
    const double2 a0 = hcol[i * W + c], a1 = hcol[(i + 1) * W + c];
    const double cc = cs[i * W + c];
    const double2 s = sn[i * W + c];
    hcol[i * W + c] = cadd(cscale(a0, cc), cmul(s, a1));
    hcol[(i + 1) * W + c] = cadd(cscale(cmulc(s, a0), -1.0), cscale(a1, cc));
  }
  const double2 a = hcol[j * W + c];
  const double absa = hypot(a.x, a.y);
  const double t = hypot(absa, hnext);
  double cr;
  double2 s, r;
  if (t == 0.0) {
    cr = 1.0; s = make_double2(0, 0); r = make_double2(0, 0);
  } else if (a.x == 0.0 && a.y == 0.0) {
    cr = 0.0; s = make_double2(1, 0); r = make_double2(hnext, 0);
  } else {
    const double2 alpha = make_double2(a.x / absa, a.y / absa);
    cr = absa / t;
    s = cscale(alpha, hnext / t);
    r = cscale(alpha, t);
  }
  hcol[j * W + c] = r;
  cs[j * W + c] = cr;
  sn[j * W + c] = s;
  const double2 gj = g[j * W + c];
  g[(j + 1) * W + c] = cscale(cmulc(s, gj), -1.0);
  g[j * W + c] = cscale(gj, cr);
  st.m[c] = j + 1;
  st.total[c] += 1;
  const double2 gn = g[(j + 1) * W + c];
  const double est = hypot(gn.x, gn.y) / st.beta0[c];
  hist[static_cast<int64_t>(st.nhist[c]) * W + c] = est;
  st.nhist[c] += 1;
  inv[c] = 0.0;
  if (est <= tol) {
    st.conv[c] = 1;
    st.stop[c] = 1;
  } else if (hnext == 0.0) {
    st.conv[c] = 1;
    st.brk[c] = 1;
    st.stop[c] = 1;
  } else {
    inv[c] = 1.0 / hnext;
    if (st.total[c] >= max_total) st.stop[c] = 3;
    else if (st.m[c] >= cycle_len) st.stop[c] = 2;
  }
  if (st.stop[c]) atomicSub(active, 1);
}

// V_next[:, c] = w[:, c] * inv[c]  (in place), all columns (inv = 0 for frozen columns is harmless)
__global__ void kb_scale(double2* __restrict__ x, const double* __restrict__ inv, int64_t n, int W,
                         const double2* __restrict__ src) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = n * W;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int cstep = static_cast<int>(stride % W);  // column advances by a constant: no 64-bit % per element
  int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  int c = static_cast<int>(t % W);
  for (; t < total; t += stride) {
    x[t] = cscale(src[t], inv[c]);
    c += cstep;
    if (c >= W) c -= W;
  }
}

// y = R^-1 g per column (gmres.py:193-204) for columns that ran steps this cycle
__global__ void kb_backsub(BCol st, const double2* rcols, int ldr, const double2* g, double2* y, int W,
                           const int* ran) {
  pdl_wait();
  pdl_trigger();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= W) return;
  const int m = ran[c] ? st.m[c] : 0;
  for (int i = m - 1; i >= 0; --i) {
    const double2 d = rcols[(static_cast<int64_t>(i) * ldr + i) * W + c];
    if (d.x == 0.0 && d.y == 0.0) {
      y[i * W + c] = make_double2(0, 0);
      continue;
    }
    double2 acc = g[i * W + c];
    for (int k = i + 1; k < m; ++k) acc = csub(acc, cmul(rcols[(static_cast<int64_t>(k) * ldr + i) * W + c], y[k * W + c]));
    const double den = d.x * d.x + d.y * d.y;
    y[i * W + c] = make_double2((acc.x * d.x + acc.y * d.y) / den, (acc.y * d.x - acc.x * d.y) / den);
  }
  for (int i = m; i < ldr; ++i) y[i * W + c] = make_double2(0, 0);
}

// x[:, c] += sum_l V_l[:, c] y[l][c]
__global__ void kb_axpy(const double2* const* __restrict__ Vp, int m, const double2* __restrict__ y,
                        double2* __restrict__ x, int64_t n, int W) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = n * W;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(t % W);
    double2 acc = x[t];
    for (int l = 0; l < m; ++l) cfma(acc, Vp[l][t], y[static_cast<int64_t>(l) * W + c]);
    x[t] = acc;
  }
}

// mark which columns run Arnoldi steps this cycle (stop == 0 after the cycle start)
__global__ void kb_mark_running(const BCol st, int* ran, int W) {
  pdl_wait();
  pdl_trigger();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < W) ran[c] = (st.stop[c] == 0);
}

__global__ void k_sub_b(const double2* __restrict__ a, const double2* __restrict__ b, double2* __restrict__ out,
                        int64_t N) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = csub(a[i], b[i]);
}

}  // namespace

// Batched independent-column GMRES.  rep_iters / rep_conv / rep_final: per column (host arrays,
// length w); hist: host array (max_iter + 2) x w, column c's history at hist[t*w + c];
// nhist per column in rep_nhist.
int gmres_batched_run(const toep_gmres_problem_t* p, const toep_gmres_cfg_t* cfg, const double2* b, double2* x,
                      cudaStream_t s, int32_t* rep_iters, int32_t* rep_conv, double* rep_final, int32_t* rep_nhist,
                      double* hist_host, int64_t hist_cap_rows) {
  keep_pool();
  TOEP_REQUIRE(p->op != nullptr, TOEP_ERR_ARG, "batched GMRES needs a resident operator");
  TOEP_REQUIRE(p->precond == TOEP_PC_NONE || p->precond == TOEP_PC_FOLDED || p->precond == TOEP_PC_BLOCK,
               TOEP_ERR_ARG, "batched GMRES supports none / folded / block preconditioners");
  TOEP_REQUIRE(op_dim(p->op) == p->n, TOEP_ERR_SHAPE, "rhs rows != operator dim");
  TOEP_REQUIRE(cfg->tol > 0 && cfg->max_iter >= 1 && cfg->restart >= 0, TOEP_ERR_ARG, "bad GMRES config");
  const int64_t n = p->n;
  const int W = static_cast<int>(p->w);
  const int64_t N = n * W;
  const int64_t max_total = std::min<int64_t>(cfg->max_iter, n);
  const int cycle_len = static_cast<int>(cfg->restart == 0 ? max_total : std::min<int64_t>(cfg->restart, max_total));
  const int ldr = cycle_len + 1;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int ctiles = (W + kCols - 1) / kCols;
  // row chunks: enough CTAs of kCols threads for ~32 resident warps per SM (the sweeps are
  // latency-bound per thread; occupancy is what keeps HBM busy)
  constexpr int chunk_mult = 32;
  const int nchunks = static_cast<int>(
      std::max<int64_t>(1, std::min<int64_t>(n / 16, (chunk_mult * sms + ctiles - 1) / ctiles)));
  const int g1 = static_cast<int>(std::min<int64_t>((N + 255) / 256, 8 * sms));
  const int gc = (W + 127) / 128;
  const int gr = (W + 31) / 32;  // column tiles of the partial reductions
  const bool per_step_pc = p->precond == TOEP_PC_BLOCK;
  const bool io64 = p->op->dtype == TOEP_C64;

  std::vector<double2*> Vh;  // basis vectors, allocated as the cycle grows
  double2 *w = nullptr, *tmp = nullptr, *pb = nullptr, *h1 = nullptr, *h2 = nullptr, *rcols = nullptr;
  double2 *sn = nullptr, *g = nullptr, *y = nullptr, *part = nullptr;
  double2 *part2 = nullptr, *gram = nullptr;  // one-sweep CGS2: Gram-column partials, per-column Gram matrices
  double *cs = nullptr, *hist = nullptr, *inv = nullptr, *npart = nullptr, *nsum = nullptr;
  double2** Vp = nullptr;
  int *ran = nullptr, *active = nullptr;
  BCol st{};
  int* active_host = nullptr;
  int rc = TOEP_OK;
  auto cleanup = [&]() {
    for (auto v : Vh) cudaFreeAsync(v, s);
    for (void* q : {(void*)w, (void*)tmp, (void*)pb, (void*)h1, (void*)h2, (void*)rcols, (void*)sn, (void*)g, (void*)y,
                    (void*)part, (void*)cs, (void*)hist, (void*)inv, (void*)npart, (void*)nsum, (void*)Vp, (void*)ran,
                    (void*)part2, (void*)gram, (void*)active, (void*)st.beta0, (void*)st.stop, (void*)st.conv, (void*)st.brk, (void*)st.m,
                    (void*)st.total, (void*)st.nhist})
      if (q) cudaFreeAsync(q, s);
    cudaStreamSynchronize(s);
  };
#define B_ALLOC(ptr, count)                                                                                       \
  do {                                                                                                            \
    if (cudaMallocAsync(reinterpret_cast<void**>(&(ptr)), sizeof(*(ptr)) * (size_t)(count), s) != cudaSuccess) { \
      cudaGetLastError();                                                                                         \
      set_error("out of device memory in batched gmres");                                                         \
      cleanup();                                                                                                  \
      return TOEP_ERR_OOM;                                                                                        \
    }                                                                                                             \
  } while (0)
#define B_TRY(expr)      \
  do {                   \
    rc = (expr);         \
    if (rc != TOEP_OK) { \
      cleanup();         \
      return rc;         \
    }                    \
  } while (0)
  B_ALLOC(w, N);
  B_ALLOC(tmp, N);
  B_ALLOC(pb, N);
  B_ALLOC(h1, static_cast<int64_t>(ldr) * W);
  B_ALLOC(h2, static_cast<int64_t>(ldr) * W);
  // one-sweep CGS2 in Gram-matrix form per column (the explicit two-pass variant measured slower)
  B_ALLOC(part2, static_cast<int64_t>(ldr) * nchunks * W);
  B_ALLOC(gram, static_cast<int64_t>(ldr) * ldr * W);
  B_ALLOC(rcols, static_cast<int64_t>(cycle_len) * ldr * W);
  B_ALLOC(sn, static_cast<int64_t>(ldr) * W);
  B_ALLOC(cs, static_cast<int64_t>(ldr) * W);
  B_ALLOC(g, static_cast<int64_t>(ldr + 1) * W);
  B_ALLOC(y, static_cast<int64_t>(ldr) * W);
  B_ALLOC(part, static_cast<int64_t>(ldr) * nchunks * W);
  B_ALLOC(npart, static_cast<int64_t>(nchunks) * W);
  B_ALLOC(nsum, W);
  B_ALLOC(hist, (max_total + 2) * W);
  B_ALLOC(inv, W);
  B_ALLOC(ran, W);
  B_ALLOC(active, 1);
  B_ALLOC(Vp, ldr + 1);
  B_ALLOC(st.beta0, W);
  B_ALLOC(st.stop, W);
  B_ALLOC(st.conv, W);
  B_ALLOC(st.brk, W);
  B_ALLOC(st.m, W);
  B_ALLOC(st.total, W);
  B_ALLOC(st.nhist, W);
  if (cudaHostAlloc(reinterpret_cast<void**>(&active_host), sizeof(int), cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    cleanup();
    set_error("pinned allocation failed");
    return TOEP_ERR_OOM;
  }
  struct PinFree {
    int* p;
    ~PinFree() { cudaFreeHost(p); }
  } pin_guard{active_host};
  auto ensure_basis = [&](int count) -> int {
    while (static_cast<int>(Vh.size()) < count) {
      double2* v = nullptr;
      if (cudaMallocAsync(reinterpret_cast<void**>(&v), sizeof(double2) * N, s) != cudaSuccess) {
        cudaGetLastError();
        set_error("out of device memory for the Krylov basis (%d vectors of %lld complex)", count, (long long)N);
        return TOEP_ERR_OOM;
      }
      Vh.push_back(v);
      TOEP_CUDA(cudaMemcpyAsync(Vp + Vh.size() - 1, &Vh.back(), sizeof(double2*), cudaMemcpyHostToDevice, s));
      TOEP_CUDA(cudaStreamSynchronize(s));  // the pageable source must outlive the copy
    }
    return TOEP_OK;
  };
  const dim3 gridc(nchunks, ctiles);

  // ---- P^-1 b and beta0 per column
  const double2* zb = b;
  if (p->precond != TOEP_PC_NONE) {
    B_TRY(block_apply_impl(p->pinv, p->pside, b, pb, n / p->pside, W, TOEP_C128, s, nullptr));
    zb = pb;
  }
  B_TRY(launch_k(kb_norm, gridc, dim3(kCols), 0, s, zb, n, W, nchunks, npart));
  B_TRY(launch_k(kb_norm_reduce, dim3(gr), dim3(kRedGroups * 32), 0, s, (const double*)npart, nchunks, W, nsum));
  B_TRY(launch_k(kb_init, dim3(gc), dim3(128), 0, s, st, (const double*)nsum, 1, W, hist));
  TOEP_CUDA(cudaMemsetAsync(x, 0, N * sizeof(double2), s));
  B_TRY(ensure_basis(1));

  bool first = true;
  while (true) {
    // ---- cycle start: V[0] = (P^-1 (b - A x)) / beta per column
    TOEP_CUDA(cudaMemsetAsync(active, 0, sizeof(int), s));
    const double2* z = zb;
    if (!first) {
      B_TRY(matvec_impl(p->op, x, tmp, W, false, io64, nullptr, s));
      if (p->precond == TOEP_PC_FOLDED) {
        B_TRY(launch_k(k_sub_b, dim3(g1), dim3(256), 0, s, (const double2*)pb, (const double2*)tmp, w, N));
      } else if (per_step_pc) {
        B_TRY(launch_k(k_sub_b, dim3(g1), dim3(256), 0, s, b, (const double2*)tmp, tmp, N));
        B_TRY(block_apply_impl(p->pinv, p->pside, tmp, w, n / p->pside, W, TOEP_C128, s, nullptr));
      } else {
        B_TRY(launch_k(k_sub_b, dim3(g1), dim3(256), 0, s, b, (const double2*)tmp, w, N));
      }
      z = w;
    }
    B_TRY(launch_k(kb_norm, gridc, dim3(kCols), 0, s, z, n, W, nchunks, npart));
    B_TRY(launch_k(kb_norm_reduce, dim3(gr), dim3(kRedGroups * 32), 0, s, (const double*)npart, nchunks, W, nsum));
    B_TRY(launch_k(kb_cycle_start, dim3(gc), dim3(128), 0, s, st, (const double*)nsum, 1, W, cfg->tol, g, inv,
                   first ? 1 : 0, active));
    B_TRY(launch_k(kb_mark_running, dim3(gc), dim3(128), 0, s, (const BCol)st, ran, W));
    B_TRY(launch_k(kb_scale, dim3(g1), dim3(256), 0, s, Vh[0], (const double*)inv, n, W, z));
    first = false;
    TOEP_CUDA(cudaMemcpyAsync(active_host, active, sizeof(int), cudaMemcpyDeviceToHost, s));
    TOEP_CUDA(cudaStreamSynchronize(s));
    int j = 0;
    int lagged_active = *active_host;
    while (lagged_active > 0 && j < cycle_len) {
      B_TRY(ensure_basis(j + 2));
      const int m = j + 1;
      if (per_step_pc) {
        B_TRY(matvec_impl(p->op, Vh[j], tmp, W, false, io64, nullptr, s));
        B_TRY(block_apply_impl(p->pinv, p->pside, tmp, w, n / p->pside, W, TOEP_C128, s, nullptr));
      } else {
        B_TRY(matvec_impl(p->op, Vh[j], w, W, false, io64, nullptr, s));
      }
      B_TRY(launch_k(kb_dots_gram, gridc, dim3(kCols, std::min(kGramGroups, (m + kLGG - 1) / kLGG)), 0, s,
                     (const double2* const*)Vp, m, (const double2*)w, n, W, nchunks, part, part2));
      B_TRY(launch_k(kb_reduce_gram, dim3(gr, m), dim3(kRedGroups * 32), 0, s, (const double2*)part,
                     (const double2*)part2, m, nchunks, W, h1, gram, ldr, (const int*)st.stop));
      B_TRY(launch_k(kb_coef_gram, dim3(gc, m), dim3(128), 0, s, (const double2*)h1, (const double2*)gram, m, ldr, W,
                     h2, rcols + static_cast<int64_t>(j) * ldr * W, (const int*)st.stop));
      B_TRY(launch_k(kb_upd, gridc, dim3(kCols), 0, s, (const double2* const*)Vp, m, (const double2*)h2, w, n,
                     W, nchunks, 2, (double2*)nullptr, npart, (const int*)st.stop));
      B_TRY(launch_k(kb_norm_reduce, dim3(gr), dim3(kRedGroups * 32), 0, s, (const double*)npart, nchunks, W, nsum));
      B_TRY(launch_k(kb_givens, dim3(gc), dim3(128), 0, s, st, (const double*)nsum, 1, W, rcols, ldr, cs, sn, g,
                     hist, inv, cfg->tol, static_cast<int>(max_total), cycle_len, active));
      B_TRY(launch_k(kb_scale, dim3(g1), dim3(256), 0, s, Vh[j + 1], (const double*)inv, n, W, (const double2*)w));
      TOEP_CUDA(cudaMemcpyAsync(active_host, active, sizeof(int), cudaMemcpyDeviceToHost, s));
      TOEP_CUDA(cudaStreamSynchronize(s));  // one multi-RHS step is tens of ms: a sync per step is free
      lagged_active = *active_host;
      ++j;
    }
    // ---- x += V y per column
    B_TRY(launch_k(kb_backsub, dim3(gc), dim3(128), 0, s, st, (const double2*)rcols, ldr, (const double2*)g, y, W,
                   (const int*)ran));
    B_TRY(launch_k(kb_axpy, dim3(g1), dim3(256), 0, s, (const double2* const*)Vp, j, (const double2*)y, x, n, W));
    // columns still needing a cycle: stop == 2 (cycle exhausted, not capped)
    std::vector<int> hstop(W);
    TOEP_CUDA(cudaMemcpyAsync(hstop.data(), st.stop, sizeof(int) * W, cudaMemcpyDeviceToHost, s));
    TOEP_CUDA(cudaStreamSynchronize(s));
    bool more = false;
    for (int c = 0; c < W; ++c) more |= (hstop[c] == 2);
    if (!more) break;
  }
  // ---- exit residuals per column: ||b - A x|| / ||b||
  B_TRY(matvec_impl(p->op, x, tmp, W, false, io64, nullptr, s));
  double2* ax = tmp;
  if (p->precond == TOEP_PC_FOLDED) {
    B_TRY(block_apply_impl(p->pmat, p->pside, tmp, pb, n / p->pside, W, TOEP_C128, s, nullptr));
    ax = pb;
  }
  B_TRY(launch_k(k_sub_b, dim3(g1), dim3(256), 0, s, b, (const double2*)ax, w, N));
  // per-column sums on the device (the same fixed-order reduction as the in-cycle norms): two
  // W-long read-backs instead of the nchunks x W partials (2 x 34 MB pageable at cfg3, ~20 ms)
  std::vector<double> nr(W), nb(W);
  B_TRY(launch_k(kb_norm, gridc, dim3(kCols), 0, s, (const double2*)w, n, W, nchunks, npart));
  B_TRY(launch_k(kb_norm_reduce, dim3(gr), dim3(kRedGroups * 32), 0, s, (const double*)npart, nchunks, W, nsum));
  TOEP_CUDA(cudaMemcpyAsync(nr.data(), nsum, sizeof(double) * W, cudaMemcpyDeviceToHost, s));
  TOEP_CUDA(cudaStreamSynchronize(s));
  B_TRY(launch_k(kb_norm, gridc, dim3(kCols), 0, s, b, n, W, nchunks, npart));
  B_TRY(launch_k(kb_norm_reduce, dim3(gr), dim3(kRedGroups * 32), 0, s, (const double*)npart, nchunks, W, nsum));
  TOEP_CUDA(cudaMemcpyAsync(nb.data(), nsum, sizeof(double) * W, cudaMemcpyDeviceToHost, s));
  std::vector<int> it(W), cv(W), nh(W);
  TOEP_CUDA(cudaMemcpyAsync(it.data(), st.total, sizeof(int) * W, cudaMemcpyDeviceToHost, s));
  TOEP_CUDA(cudaMemcpyAsync(cv.data(), st.conv, sizeof(int) * W, cudaMemcpyDeviceToHost, s));
  TOEP_CUDA(cudaMemcpyAsync(nh.data(), st.nhist, sizeof(int) * W, cudaMemcpyDeviceToHost, s));
  const int64_t rows = std::min<int64_t>(hist_cap_rows, max_total + 2);
  if (hist_host != nullptr && rows > 0)
    TOEP_CUDA(cudaMemcpyAsync(hist_host, hist, sizeof(double) * rows * W, cudaMemcpyDeviceToHost, s));
  TOEP_CUDA(cudaStreamSynchronize(s));
  for (int c = 0; c < W; ++c) {
    const double sr = nr[c], sb = nb[c];
    rep_final[c] = sb > 0 ? std::sqrt(sr) / std::sqrt(sb) : 0.0;
    rep_iters[c] = it[c];
    rep_conv[c] = cv[c];
    rep_nhist[c] = nh[c];
  }
  cleanup();
#undef B_ALLOC
#undef B_TRY
  return TOEP_OK;
}

}  // namespace toep

extern "C" int toep_gmres_batched(const toep_gmres_problem_t* prob, const toep_gmres_cfg_t* cfg, const void* b,
                                  void* x, void* stream, int32_t* iterations, int32_t* converged,
                                  double* final_residual, int32_t* n_history, double* history, int64_t history_rows) {
  TOEP_NVTX("toep_gmres_batched");
  TOEP_REQUIRE(prob != nullptr && cfg != nullptr && b != nullptr && x != nullptr && iterations != nullptr &&
                   converged != nullptr && final_residual != nullptr && n_history != nullptr,
               TOEP_ERR_ARG, "null argument");
  return toep::gmres_batched_run(prob, cfg, static_cast<const double2*>(b), static_cast<double2*>(x),
                                 static_cast<cudaStream_t>(stream), iterations, converged, final_residual, n_history,
                                 history, history_rows);
}
