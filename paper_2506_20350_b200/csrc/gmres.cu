// Device-resident left-preconditioned GMRES (solvers/gmres.py:98-219).
//
// Semantics follow _gmres_block exactly: beta0 = ||P^-1 b||_F, a zero rhs
// returns 0, max_total = min(max_iter, n*w), cycles restart from the true
// residual, the per-step estimate is |g_{j+1}| / beta0 from the Givens
// recurrence (gmres.py:164-183), a lucky breakdown h_{j+1,j} == 0 stops the
// cycle, back substitution skips zero diagonals (gmres.py:193-204), and the
// exit residual is the unpreconditioned ||b - A x|| / ||b||.
//
// Orthogonalisation is classical Gram-Schmidt with one re-orthogonalisation
// (CGS2) instead of the reference's j sequential vdot/axpy pairs
// (gmres.py:155-159); CGS2 keeps the basis orthogonal to working precision
// like MGS, so Hessenberg entries and residual histories agree to rounding.
//
// Kernel chain of one Arnoldi step (all PDL-launched, all no-ops once the
// device stop flag is set):
//   matvec(v_j) -> V[j+1]                       (4-5 kernels, matvec_impl)
//   k_dots      : partials of V_{0..j}^H w       (pass 1)
//   k_upd       : h1 = reduce(partials) [every CTA, fixed order], w -= V h1,
//                 partials of V^H w'             (pass 2)
//   k_upd       : h2, w -= V h2, ||w||^2 partials, H[:, j] = h1 + h2
//   k_givens    : ||w||, rotations, g, estimate, stop flags, scale of V[j+1]
// The basis is stored unnormalised: v_l = vs[l] * V[l].  The 1/h_{j+1,j}
// normalisation is a device scalar consumed by the next matvec's first DFT
// pass and by the Gram-Schmidt kernels, so no kernel rescales the vector.
//
// Host/device split: every scalar (Hessenberg column, rotations, g, the
// residual history, the stop flags) lives on the device.  The host only
// launches; after launching step j it waits for step j-1 and reads the stop
// flag from mapped pinned memory, so the launch queue stays one step ahead
// and no step waits on a host round trip.
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "launch.cuh"
#include "op.h"

namespace toep {
namespace {

constexpr int kThreads = 256;

struct GState {
  int stop;       // 0 running, 1 converged / breakdown, 2 cycle exhausted
  int converged;
  int breakdown;
  int m;          // completed steps in the current cycle
  int total;      // completed steps overall
  int nhist;
  double beta0, beta, hnext;
};

__device__ __forceinline__ long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct HostFlags {
  volatile int stop;
  volatile int total;
  volatile int converged;
  volatile int breakdown;
};

__device__ __forceinline__ double2 warp_sum(double2 v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, off);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, off);
  }
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

template <typename Z>
__device__ __forceinline__ Z block_sum(Z v, Z* red /* [kThreads/32] */) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  Z t = red[0];
#pragma unroll
  for (int ww = 1; ww < kThreads / 32; ++ww) t = t + red[ww];
  __syncthreads();
  return t;
}

// CTA b of nblk owns the contiguous element range [c0, c1) (32-aligned starts, coalesced)
__device__ __forceinline__ void chunk_of(int64_t N, int64_t* c0, int64_t* c1) {
  const int64_t b = blockIdx.x, nb = gridDim.x;
  *c0 = ((N * b / nb) / 32) * 32;
  *c1 = (b + 1 == nb) ? N : ((N * (b + 1) / nb) / 32) * 32;
}

constexpr int kDG = 4;  // basis vectors per warp in the dot kernels

// partial[l*nblk + cta] = sum_{i in chunk} conj(V_l[i]) w[i], l < m.  Each warp takes groups of
// kDG basis vectors over the whole chunk (independent loads in flight, no block barrier).
__device__ __forceinline__ void dots_into(const double2* __restrict__ V, int64_t ld, int m,
                                          const double2* __restrict__ w, int64_t N, double2* __restrict__ partial) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nblk = gridDim.x;
  int64_t c0, c1;
  chunk_of(N, &c0, &c1);
  for (int l0 = warp * kDG; l0 < m; l0 += (kThreads / 32) * kDG) {
    double2 acc[kDG];
#pragma unroll
    for (int g = 0; g < kDG; ++g) acc[g] = make_double2(0, 0);
#pragma unroll 2
    for (int64_t i = c0 + lane; i < c1; i += 32) {
      const double2 wi = w[i];
#pragma unroll
      for (int g = 0; g < kDG; ++g)
        if (l0 + g < m) cfmac(acc[g], V[(l0 + g) * ld + i], wi);
    }
#pragma unroll
    for (int g = 0; g < kDG; ++g) {
      const double2 s = warp_sum(acc[g]);
      if (lane == 0 && l0 + g < m) partial[(l0 + g) * nblk + blockIdx.x] = s;
    }
  }
}

__global__ void __launch_bounds__(kThreads)
k_dots(const double2* __restrict__ V, int64_t ld, int m, const double2* __restrict__ w, int64_t N,
       double2* __restrict__ partial, const int* stop) {
  pdl_wait();
  pdl_trigger();
  if (stop != nullptr && *stop) return;
  dots_into(V, ld, m, w, N, partial);
}

// Gram-Schmidt update:  h_l = vs_l * sum_b partial[l][b]  (reduced redundantly, same order, in every CTA)
//   w -= sum_l V_l (vs_l h_l)
// mode 1: partials of V^H w (next pass); hout[l] = h_l (CTA 0)
// mode 2: ||w||^2 partials; hcol[l] = hprev[l] + h_l (CTA 0)
__global__ void __launch_bounds__(kThreads)
k_upd(const double2* __restrict__ V, int64_t ld, int m, const double* __restrict__ vs,
      const double2* __restrict__ partial_in, int nblk_in, double2* __restrict__ w, int64_t N, int mode,
      double2* __restrict__ hout, const double2* __restrict__ hprev, double2* __restrict__ partial_out,
      double* __restrict__ norm_out, const int* stop) {
  pdl_wait();
  pdl_trigger();
  if (stop != nullptr && *stop) return;
  extern __shared__ double2 coef[];  // [m]
  __shared__ double red_n[kThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int l = warp; l < m; l += kThreads / 32) {
    double2 s = make_double2(0, 0);
    for (int b = lane; b < nblk_in; b += 32) s = cadd(s, partial_in[l * nblk_in + b]);
    s = warp_sum(s);
    if (lane == 0) {
      const double2 h = cscale(s, vs[l]);
      coef[l] = cscale(h, vs[l]);
      if (blockIdx.x == 0) {
        if (mode == 1) hout[l] = h;
        else hout[l] = cadd(hprev[l], h);
      }
    }
  }
  __syncthreads();
  double nrm = 0.0;
  int64_t c0, c1;
  chunk_of(N, &c0, &c1);
  for (int64_t i = c0 + threadIdx.x; i < c1; i += kThreads) {
    double2 acc = w[i];
    int l = 0;
    for (; l + 3 < m; l += 4) {
      const double2 v0 = V[l * ld + i], v1 = V[(l + 1) * ld + i], v2 = V[(l + 2) * ld + i], v3 = V[(l + 3) * ld + i];
      cfma(acc, v0, make_double2(-coef[l].x, -coef[l].y));
      cfma(acc, v1, make_double2(-coef[l + 1].x, -coef[l + 1].y));
      cfma(acc, v2, make_double2(-coef[l + 2].x, -coef[l + 2].y));
      cfma(acc, v3, make_double2(-coef[l + 3].x, -coef[l + 3].y));
    }
    for (; l < m; ++l) cfma(acc, V[l * ld + i], make_double2(-coef[l].x, -coef[l].y));
    w[i] = acc;
    nrm = fma(acc.x, acc.x, fma(acc.y, acc.y, nrm));
  }
  if (mode == 1) {
    __syncthreads();  // this CTA's w updates are its own elements: visible to itself after the barrier
    dots_into(V, ld, m, w, N, partial_out);
  } else {
    nrm = warp_sum(nrm);
    if (lane == 0) red_n[warp] = nrm;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = red_n[0];
      for (int ww = 1; ww < kThreads / 32; ++ww) t += red_n[ww];
      norm_out[blockIdx.x] = t;
    }
  }
}

// x += sum_{l < m} V_l (vs_l y_l),  m = min(m_max, *m_dev)   (gmres.py:203-204)
__global__ void __launch_bounds__(kThreads)
k_axpy_basis(const double2* __restrict__ V, int64_t ld, int m_max, const int* m_dev, const double* __restrict__ vs,
             const double2* __restrict__ y, double2* __restrict__ x, int64_t N) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ double2 coef[];
  const int m = min(m_max, *m_dev);
  for (int l = threadIdx.x; l < m; l += kThreads) coef[l] = cscale(y[l], vs[l]);
  __syncthreads();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; i < N;
       i += static_cast<int64_t>(gridDim.x) * kThreads) {
    double2 acc = x[i];
    int l = 0;
    for (; l + 7 < m; l += 8) {  // 8 independent basis loads in flight
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = V[(l + u) * ld + i];
#pragma unroll
      for (int u = 0; u < 8; ++u) cfma(acc, v[u], coef[l + u]);
    }
    for (; l < m; ++l) cfma(acc, V[l * ld + i], coef[l]);
    x[i] = acc;
  }
}

__global__ void __launch_bounds__(kThreads)
k_norm2(const double2* __restrict__ x, int64_t N, double* __restrict__ partial) {
  pdl_wait();
  pdl_trigger();
  __shared__ double red[kThreads / 32];
  double nrm = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; i < N;
       i += static_cast<int64_t>(gridDim.x) * kThreads) {
    const double2 v = x[i];
    nrm = fma(v.x, v.x, fma(v.y, v.y, nrm));
  }
  const double t = block_sum(nrm, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// out[0] = sum_b part[b] (one warp, fixed order per lane + butterfly)
__global__ void k_collapse_d(const double* __restrict__ part, int nblk, double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += 32) s += part[b];
  s = warp_sum(s);
  if (threadIdx.x == 0) out[0] = s;
}

// out[l] = sum_b part[l*nblk + b], l < m (warp per l)
__global__ void k_collapse_c(const double2* __restrict__ part, int m, int nblk, double2* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int l = warp; l < m; l += blockDim.x / 32) {
    double2 s = make_double2(0, 0);
    for (int b = lane; b < nblk; b += 32) s = cadd(s, part[l * nblk + b]);
    s = warp_sum(s);
    if (lane == 0) out[l] = s;
  }
}

__device__ double sum_partials_warp(const double* p, int n) {
  double s = 0.0;
  for (int b = threadIdx.x; b < n; b += 32) s += p[b];
  return warp_sum(s);
}

// out = a - b
__global__ void k_sub(const double2* __restrict__ a, const double2* __restrict__ b, double2* __restrict__ out,
                      int64_t N) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = csub(a[i], b[i]);
}

// out = x * (*scal), unless *stop  (normalised copy for callback operators)
__global__ void k_scale(const double2* __restrict__ x, double2* __restrict__ out, const double* scal, int64_t N,
                        const int* stop) {
  pdl_wait();
  pdl_trigger();
  if (stop != nullptr && *stop) return;
  const double s = *scal;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = cscale(x[i], s);
}

// beta0 = ||P^-1 b||; history[0]
__global__ void k_init(GState* st, const double* partial, int nblk, double* hist) {
  pdl_wait();
  pdl_trigger();
  const double s = sum_partials_warp(partial, nblk);
  if (threadIdx.x == 0) {
    const double beta0 = sqrt(s);
    st->beta0 = beta0;
    st->stop = 0;
    st->converged = 0;
    st->breakdown = 0;
    st->m = 0;
    st->total = 0;
    st->nhist = 1;
    hist[0] = (beta0 == 0.0) ? 0.0 : 1.0;
  }
}

// cycle start (gmres.py:130-144): beta = ||z||, convergence test, g[0] = beta, vs[0] = 1/beta
__global__ void k_cycle_start(GState* st, const double* partial, int nblk, double tol, double2* g, double* vs,
                              HostFlags* hf, long long* ts) {
  pdl_wait();
  pdl_trigger();
  const double s = sum_partials_warp(partial, nblk);
  if (threadIdx.x == 0) {
    if (ts != nullptr) ts[2 * st->total + 1] = global_ns();  // "previous step end" of the cycle's first step
    const double beta = sqrt(s);
    st->beta = beta;
    st->m = 0;
    if (st->beta0 == 0.0 || beta / st->beta0 <= tol) {  // b = 0: x = 0 is the solution
      st->converged = 1;
      st->stop = 1;
    } else {
      st->stop = 0;
      g[0] = make_double2(beta, 0.0);
      vs[0] = 1.0 / beta;
    }
    hf->stop = st->stop;
    hf->converged = st->converged;
    hf->total = st->total;
  }
}

// end-of-cycle report straight into mapped page-locked host memory: the solver state, the exit
// residual's partials, the history written so far and (timed solves) the step stamps, then the
// sequence word the host spins on (written last, after a system-scope fence).  Replaces the
// device-to-host copies and the stream synchronisation of each cycle end.
struct ReportLayout {
  size_t st, r, b, h, t, bytes;
};
__global__ void k_report(const GState* st, const double* rpart, int rcnt, const double* hist, int hist_cap,
                         const long long* ts, unsigned char* out, ReportLayout lay, unsigned seq) {
  pdl_wait();
  pdl_trigger();
  const int nh = min(st->nhist, hist_cap);
  double* orp = reinterpret_cast<double*>(out + lay.r);
  double* oh = reinterpret_cast<double*>(out + lay.h);
  for (int i = threadIdx.x; i < rcnt; i += blockDim.x) orp[i] = __ldcg(rpart + i);
  for (int i = threadIdx.x; i < nh; i += blockDim.x) oh[i] = __ldcg(hist + i);
  if (ts != nullptr) {
    long long* ot = reinterpret_cast<long long*>(out + lay.t);
    const int nt = 2 * st->total + 2;
    for (int i = threadIdx.x; i < nt; i += blockDim.x) ot[i] = __ldcg(ts + i);
  }
  if (threadIdx.x == 0) *reinterpret_cast<GState*>(out + lay.st) = *st;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    *reinterpret_cast<volatile unsigned*>(out) = seq;
  }
}

// one Givens step on column j = st->m (gmres.py:160-189), executed by one warp;
// hn2 = ||w||^2, gsm: shared scratch of (2*16 + 8)*(j+1) bytes
__device__ void givens_warp(GState* st, double hn2, double2* rcols, int ldr, double* cs, double2* sn, double2* g,
                            double* hist, double* vs, double tol, int max_total, int cycle_len, HostFlags* hf,
                            double2* gsm) {
  const int j = st->m;
  double2* hcol_g = rcols + static_cast<int64_t>(j) * ldr;  // hcol[0..j] = h1 + h2
  // stage the column and the previous rotations in shared memory (one parallel load instead of
  // a chain of dependent global accesses), rotate on lane 0, write the column back
  double2* hcol = gsm;                                      // [j+1]
  double2* snl = gsm + (j + 1);                             // [j]
  double* csl = reinterpret_cast<double*>(snl + j);         // [j]
  for (int i = threadIdx.x; i <= j; i += 32) hcol[i] = hcol_g[i];
  for (int i = threadIdx.x; i < j; i += 32) {
    snl[i] = sn[i];
    csl[i] = cs[i];
  }
  __syncwarp();
  if (threadIdx.x == 0) {
    for (int i = 0; i < j; ++i) {
      const double2 a0 = hcol[i], a1 = hcol[i + 1];
      const double c = csl[i];
      const double2 s = snl[i];
      hcol[i] = cadd(cscale(a0, c), cmul(s, a1));
      hcol[i + 1] = cadd(cscale(cmulc(s, a0), -1.0), cscale(a1, c));
    }
  }
  __syncwarp();
  for (int i = threadIdx.x; i < j; i += 32) hcol_g[i] = hcol[i];
  __syncwarp();
  if (threadIdx.x != 0) return;
  const double hnext = sqrt(hn2);
  // _givens(hcol[j], hnext) (gmres.py:87-95)
  const double2 a = hcol[j];
  const double absa = hypot(a.x, a.y);
  const double t = hypot(absa, hnext);
  double c;
  double2 s, r;
  if (t == 0.0) {
    c = 1.0; s = make_double2(0, 0); r = make_double2(0, 0);
  } else if (a.x == 0.0 && a.y == 0.0) {
    c = 0.0; s = make_double2(1, 0); r = make_double2(hnext, 0);
  } else {
    const double2 alpha = make_double2(a.x / absa, a.y / absa);
    c = absa / t;
    s = cscale(alpha, hnext / t);
    r = cscale(alpha, t);
  }
  hcol_g[j] = r;
  cs[j] = c;
  sn[j] = s;
  const double2 gj = g[j];
  g[j + 1] = cscale(cmulc(s, gj), -1.0);
  g[j] = cscale(gj, c);
  st->m = j + 1;
  st->total += 1;
  const double2 gn = g[j + 1];
  const double est = hypot(gn.x, gn.y) / st->beta0;
  hist[st->nhist++] = est;
  st->hnext = hnext;
  if (est <= tol) {
    st->converged = 1;
    st->stop = 1;
  } else if (hnext == 0.0) {
    st->converged = 1;
    st->breakdown = 1;
    st->stop = 1;
  } else {
    vs[j + 1] = 1.0 / hnext;  // v_{j+1} = w / h_{j+1,j}, applied lazily
    if (st->m >= cycle_len || st->total >= max_total) st->stop = 2;
  }
  hf->stop = st->stop;
  hf->total = st->total;
  hf->converged = st->converged;
  hf->breakdown = st->breakdown;
}

__global__ void k_givens(GState* st, const double* norm_partial, int nblk, double2* rcols, int ldr, double* cs,
                         double2* sn, double2* g, double* hist, double* vs, double tol, int max_total, int cycle_len,
                         HostFlags* hf) {
  pdl_wait();
  pdl_trigger();
  if (st->stop) return;
  extern __shared__ double2 gsm[];
  const double hn2 = sum_partials_warp(norm_partial, nblk);
  givens_warp(st, hn2, rcols, ldr, cs, sn, g, hist, vs, tol, max_total, cycle_len, hf, gsm);
}

// ------------------------------------------------------------------------------------------
// The whole CGS2 orthogonalisation + Givens step of one Arnoldi step as ONE cooperative kernel
// (all CTAs co-resident, one per SM, 1024 threads): dots -> grid barrier -> coefficients
// (every CTA reduces the per-CTA partials in the same order) -> update + dots -> barrier ->
// update + norm -> barrier -> Givens on CTA 0.  Replaces 4 launches and their drain / ramp
// gaps; 32 warps per SM keep enough L2 requests in flight for the basis sweeps.
#ifndef TOEP_COOP_THREADS
#define TOEP_COOP_THREADS 512
#endif
constexpr int kCoopThreads = TOEP_COOP_THREADS;

struct OrthArgs {
  const double2* V;
  int64_t N;        // vector length = basis stride
  int m;            // basis vectors v_0..v_{m-1}
  const double* vs; // lazy scales
  double2* w;       // = V_m, updated in place
  double2* part;    // [ldr][nblk] dot partials
  double* npart;    // [nblk]
  double2* h1;      // [ldr]
  GState* st;
  double2* rcols;
  int ldr;
  double* cs;
  double2* sn;
  double2* g;
  double* hist;
  double* vsw;      // vs (written by Givens)
  double tol;
  int max_total, cycle_len;
  HostFlags* hf;
  unsigned* bar;    // [2] grid barrier: arrival count, generation
  long long* ts;    // optional phase stamps: [2k+2] = step k orth start, [2k+3] = step k end
  L2Prefetch pf;    // operator stream prefetched into L2 for the next matvec (HBM is idle here)
  double2* gram;    // one-sweep CGS2: Gram matrix of the cycle's basis [ldr][ldr] (col-major)
  double2* part2;   // [ldr][nblk] partials of V^H v_{m-1}
  int gram_smem;    // 1: the Gram block is staged in shared memory (small cycles, see coop_smem)
};
constexpr int kMaxOrthM = 1024;  // basis vectors per cycle handled by the cooperative kernel
constexpr int kOrthGroupedMinChunk = 2048;  // elements per CTA from which the grouped dot sweep is used

// Grid barrier on a monotonic arrival counter (zeroed once per solve): every CTA adds 1 and
// waits until the counter reaches the next multiple of gridDim.x (one atomic per CTA, no reset).
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
    const unsigned target = (old / gridDim.x + 1) * gridDim.x;
    // a CTA that never arrives (a fault elsewhere in the grid) must not hang the device forever:
    // trap after 10 s, which surfaces as a CUDA error on the host
    long long t0 = 0;
    for (unsigned spins = 1; static_cast<int>(ld_acquire_gpu(bar) - target) < 0; ++spins) {
      if ((spins & 1023u) == 0) {
        const long long t = global_ns();
        if (t0 == 0) t0 = t;
        else if (t - t0 > 10000000000ll) __trap();
      }
    }
  }
  __syncthreads();
}

// coef[l] = vs_l * (vs_l * sum_b part[l][b]); CTA 0 stores h (mode 1) or hprev + h (mode 2)

__device__ __forceinline__ double orth_update(const OrthArgs& a, const double2* coef, int64_t c0, int64_t c1) {
  constexpr int U = 8;  // basis loads issued together (latency-bound sweep over L2-resident vectors)
  double nrm = 0.0;
  // back to front: the dots sweep before it (and the next step's) run front to back, so when the
  // basis outgrows L2 (cfg4 beyond ~13 vectors) each sweep starts on the lines the previous one
  // touched last instead of the ones LRU has just evicted
  const int64_t first = c0 + threadIdx.x;
  const int64_t iters = first < c1 ? (c1 - first + kCoopThreads - 1) / kCoopThreads : 0;
  for (int64_t i = first + (iters - 1) * kCoopThreads; i >= first; i -= kCoopThreads) {
    double2 acc = a.w[i];
    int l = 0;
    for (; l + U - 1 < a.m; l += U) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = a.V[(l + u) * a.N + i];
#pragma unroll
      for (int u = 0; u < U; ++u) cfma(acc, v[u], make_double2(-coef[l + u].x, -coef[l + u].y));
    }
    for (; l < a.m; ++l) cfma(acc, a.V[l * a.N + i], make_double2(-coef[l].x, -coef[l].y));
    a.w[i] = acc;
    nrm = fma(acc.x, acc.x, fma(acc.y, acc.y, nrm));
  }
  return nrm;
}

// One-sweep CGS2 dots for short chunks: V_l^H w and V_l^H V_{m-1} (the last basis vector's Gram
// column) over the CTA's chunk, reading V_l once.  Work item = (basis vector l, sub-chunk): with m
// basis vectors and NW warps, S = NW / m warps split each vector's chunk so that every warp has
// loads in flight (all of a lane's U iterations issued before any use); the items of vector 0
// also accumulate ||w||^2 from the w values they load anyway.  Sub-chunk partials are combined in
// shared memory in a fixed order (deterministic).
__device__ __forceinline__ void orth_dots_gram_pv(const OrthArgs& a, int64_t c0, int64_t c1) {
  constexpr int NW = kCoopThreads / 32, U = 4;
  __shared__ double2 sp1[NW], sp2[NW];
  __shared__ double spn[NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nblk = gridDim.x, m = a.m;
  const double2* vl = a.V + static_cast<int64_t>(m - 1) * a.N;
  const int S = m >= NW ? 1 : NW / m;  // warps per basis vector
  const int per_round = NW / S;        // vectors per round
  const int64_t len = c1 - c0;
  for (int l0 = 0; l0 < m; l0 += per_round) {
    const int l = l0 + warp / S, sc = warp - (warp / S) * S;
    double2 acc[U], acg[U];
    double wn = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = acg[u] = make_double2(0, 0);
    if (l < m && warp / S < per_round) {
      const int64_t s0 = c0 + ((len * sc / S) / 32) * 32;
      const int64_t s1 = (sc + 1 == S) ? c1 : c0 + ((len * (sc + 1) / S) / 32) * 32;
      const double2* v = a.V + static_cast<int64_t>(l) * a.N;
      int64_t i = s0 + lane;
      for (; i + 32 * (U - 1) < s1; i += 32 * U) {
        double2 vv[U], ww[U], ll[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          vv[u] = v[i + 32 * u];
          ww[u] = a.w[i + 32 * u];
          ll[u] = vl[i + 32 * u];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          cfmac(acc[u], vv[u], ww[u]);
          cfmac(acg[u], vv[u], ll[u]);
          if (l == 0) wn = fma(ww[u].x, ww[u].x, fma(ww[u].y, ww[u].y, wn));
        }
      }
      for (; i < s1; i += 32) {
        const double2 vi = v[i], wi = a.w[i];
        cfmac(acc[0], vi, wi);
        cfmac(acg[0], vi, vl[i]);
        if (l == 0) wn = fma(wi.x, wi.x, fma(wi.y, wi.y, wn));
      }
#pragma unroll
      for (int u = 1; u < U; ++u) {
        acc[0] = cadd(acc[0], acc[u]);
        acg[0] = cadd(acg[0], acg[u]);
      }
    }
    const double2 t1 = warp_sum(acc[0]);
    const double2 t2 = warp_sum(acg[0]);
    if (l0 == 0) wn = warp_sum(wn);
    if (lane == 0) {
      sp1[warp] = t1;
      sp2[warp] = t2;
      if (l0 == 0) spn[warp] = wn;
    }
    __syncthreads();
    if (threadIdx.x < per_round) {
      const int lv = l0 + static_cast<int>(threadIdx.x);
      if (lv < m) {
        double2 u1 = sp1[threadIdx.x * S], u2 = sp2[threadIdx.x * S];
        for (int q = 1; q < S; ++q) {
          u1 = cadd(u1, sp1[threadIdx.x * S + q]);
          u2 = cadd(u2, sp2[threadIdx.x * S + q]);
        }
        a.part[static_cast<int64_t>(lv) * nblk + blockIdx.x] = u1;
        a.part2[static_cast<int64_t>(lv) * nblk + blockIdx.x] = u2;
      }
      if (l0 == 0 && threadIdx.x == 0) {
        double t = spn[0];
        for (int q = 1; q < S; ++q) t += spn[q];
        a.npart[blockIdx.x] = t;
      }
    }
    __syncthreads();
  }
}

// One-sweep CGS2 dots over the CTA's chunk: V_l^H w and V_l^H V_{m-1} (the last basis vector's
// Gram column) for every l, plus ||w||^2.  Work items are (group of G basis vectors) x (sub-chunk):
// a warp reads w and V_{m-1} once per group instead of once per vector, and with few basis vectors
// (early steps) the chunk is split over several warps per group so that all 32 warps keep loads
// in flight.  Sub-chunk partials are combined in shared memory in a fixed order (deterministic).
__device__ __forceinline__ void orth_dots_gram(const OrthArgs& a, int64_t c0, int64_t c1) {
  constexpr int NW = kCoopThreads / 32, G = 4;
  __shared__ double2 dpart[2][NW * G];
  __shared__ double nsub[NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nblk = gridDim.x, m = a.m;
  const double2* vl = a.V + static_cast<int64_t>(m - 1) * a.N;
  const int ngroups = (m + G - 1) / G;
  const int64_t len = c1 - c0;
  const int S = ngroups >= NW ? 1 : NW / ngroups;  // warps (sub-chunks) per group; S * m <= NW * G
  for (int item = warp; item < ngroups * S; item += NW) {
    const int g = item / S, sc = item - g * S;
    const int64_t s0 = c0 + ((len * sc / S) / 32) * 32;
    const int64_t s1 = (sc + 1 == S) ? c1 : c0 + ((len * (sc + 1) / S) / 32) * 32;
    const int l0 = g * G;
    const int nl = min(G, m - l0);
    const double2* v0 = a.V + static_cast<int64_t>(l0) * a.N;
    double2 acc[G], acg[G];
#pragma unroll
    for (int u = 0; u < G; ++u) acc[u] = acg[u] = make_double2(0, 0);
    double wn = 0.0;
    for (int64_t i = s0 + lane; i < s1; i += 32) {
      const double2 wi = a.w[i], li = vl[i];
      double2 vv[G];
#pragma unroll
      for (int u = 0; u < G; ++u) vv[u] = u < nl ? v0[u * a.N + i] : make_double2(0, 0);
#pragma unroll
      for (int u = 0; u < G; ++u) {
        cfmac(acc[u], vv[u], wi);
        cfmac(acg[u], vv[u], li);
      }
      wn = fma(wi.x, wi.x, fma(wi.y, wi.y, wn));
    }
#pragma unroll
    for (int u = 0; u < G; ++u) {
      if (u >= nl) break;
      const double2 d1 = warp_sum(acc[u]);
      const double2 d2 = warp_sum(acg[u]);
      if (lane == 0) {
        if (S == 1) {
          a.part[static_cast<int64_t>(l0 + u) * nblk + blockIdx.x] = d1;
          a.part2[static_cast<int64_t>(l0 + u) * nblk + blockIdx.x] = d2;
        } else {
          dpart[0][sc * m + l0 + u] = d1;
          dpart[1][sc * m + l0 + u] = d2;
        }
      }
    }
    if (g == 0) {
      wn = warp_sum(wn);
      if (lane == 0) nsub[sc] = wn;
    }
  }
  __syncthreads();
  if (S > 1) {
    for (int l = threadIdx.x; l < m; l += kCoopThreads) {
      double2 d1 = dpart[0][l], d2 = dpart[1][l];
      for (int sc = 1; sc < S; ++sc) {
        d1 = cadd(d1, dpart[0][sc * m + l]);
        d2 = cadd(d2, dpart[1][sc * m + l]);
      }
      a.part[static_cast<int64_t>(l) * nblk + blockIdx.x] = d1;
      a.part2[static_cast<int64_t>(l) * nblk + blockIdx.x] = d2;
    }
  }
  if (threadIdx.x == 0) {
    double t = nsub[0];
    for (int sc = 1; sc < S; ++sc) t += nsub[sc];
    a.npart[blockIdx.x] = t;
  }
}

// one warp per basis vector: warp l sweeps the CTA's chunk of V_l and w with 8 independent
// loads in flight per lane and ends with a single warp reduction; lane 0 stores the CTA partial

// the new rotation from the rotated column's diagonal entry and h_{j+1,j} = ||w|| (gmres.py:
// 87-95, 171-190); same arithmetic as givens_warp's tail, with the scalars prefetched
__device__ void givens_finish(const OrthArgs& a, int j, double2 hj, double hn2, double2 gj, double beta0, int nhist) {
  GState* st = a.st;
  double2* hcol_g = a.rcols + static_cast<int64_t>(j) * a.ldr;
  const double hnext = sqrt(hn2);
  const double absa = hypot(hj.x, hj.y);
  const double t = hypot(absa, hnext);
  double c;
  double2 s, r;
  if (t == 0.0) {
    c = 1.0; s = make_double2(0, 0); r = make_double2(0, 0);
  } else if (hj.x == 0.0 && hj.y == 0.0) {
    c = 0.0; s = make_double2(1, 0); r = make_double2(hnext, 0);
  } else {
    const double2 alpha = make_double2(hj.x / absa, hj.y / absa);
    c = absa / t;
    s = cscale(alpha, hnext / t);
    r = cscale(alpha, t);
  }
  hcol_g[j] = r;
  a.cs[j] = c;
  a.sn[j] = s;
  const double2 gn = cscale(cmulc(s, gj), -1.0);
  a.g[j + 1] = gn;
  a.g[j] = cscale(gj, c);
  const int m = j + 1, total = st->total + 1;
  st->m = m;
  st->total = total;
  const double est = hypot(gn.x, gn.y) / beta0;
  a.hist[nhist] = est;
  st->nhist = nhist + 1;
  st->hnext = hnext;
  int stop = 0, conv = st->converged, brk = st->breakdown;
  if (est <= a.tol) {
    conv = 1;
    stop = 1;
  } else if (hnext == 0.0) {
    conv = 1;
    brk = 1;
    stop = 1;
  } else {
    a.vsw[j + 1] = 1.0 / hnext;  // v_{j+1} = w / h_{j+1,j}, applied lazily
    if (m >= a.cycle_len || total >= a.max_total) stop = 2;
  }
  st->converged = conv;
  st->breakdown = brk;
  st->stop = stop;
  a.hf->stop = stop;
  a.hf->total = total;
  a.hf->converged = conv;
  a.hf->breakdown = brk;
}

// CTA 0: apply the cycle's previous rotations to the new Hessenberg column held in hsm
// (gmres.py:165-170) and write rows 0..j-1 back; row j is written by givens_finish
__device__ void orth_prepare_givens(const OrthArgs& a, int jcol, double2* hsm, double2* snl, double* csl,
                                    double2* hcol) {
  for (int i = threadIdx.x; i < jcol; i += kCoopThreads) {
    snl[i] = a.sn[i];
    csl[i] = a.cs[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < jcol; ++i) {
      const double2 a0 = hsm[i], a1 = hsm[i + 1];
      const double c = csl[i];
      const double2 sv = snl[i];
      hsm[i] = cadd(cscale(a0, c), cmul(sv, a1));
      hsm[i + 1] = cadd(cscale(cmulc(sv, a0), -1.0), cscale(a1, c));
      hcol[i] = hsm[i];
    }
  }
}

__global__ void __launch_bounds__(kCoopThreads, 1) k_orth_coop(OrthArgs a, const int* stop) {
  pdl_wait();
  pdl_trigger();
  if (*stop) return;  // uniform across the grid (written by the previous step, read-only here)
  if (a.ts != nullptr && blockIdx.x == 0 && threadIdx.x == 0) a.ts[2 * a.st->total + 2] = global_ns();
  if (threadIdx.x >= kCoopThreads - 32) l2_prefetch_heads(a.pf, blockIdx.x, gridDim.x, threadIdx.x & 31);
#ifdef TOEP_ORTH_PROBE
  long long pt[12];
  int np = 0;
#define OPROBE() \
  if (blockIdx.x == (gridDim.x > 1 ? 1 : 0) && threadIdx.x == 0) pt[np++] = global_ns()
#else
#define OPROBE()
#endif
  OPROBE();
  extern __shared__ double2 osm[];  // coef [ldr] | dot partials [32][ldr]; Givens scratch reuses it
  __shared__ double red[kCoopThreads / 32];
  double2* coef = osm;
  double2* hsm = osm + a.ldr;        // CTA 0: the new Hessenberg column
  double2* snl = hsm + a.ldr;        // CTA 0: previous rotations
  double* csl = reinterpret_cast<double*>(snl + a.ldr);
  // CTA 0 owns no elements (unless it is alone): it prepares the Givens step while the others
  // sweep the basis
  int64_t c0 = 0, c1 = gridDim.x == 1 ? a.N : 0;
  if (blockIdx.x > 0) {
    const int64_t nb = gridDim.x - 1, b = blockIdx.x - 1;
    c0 = ((a.N * b / nb) / 32) * 32;
    c1 = (b + 1 == nb) ? a.N : ((a.N * (b + 1) / nb) / 32) * 32;
  }
  const int jcol = a.m - 1;  // this step's column index in the cycle (st->m)
  double2 g_j = make_double2(0, 0);
  double beta0 = 1.0;
  int k_step = 0, nhist = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // scalars for the final rotation, fetched early
    g_j = a.g[jcol];
    beta0 = a.st->beta0;
    k_step = a.st->total;
    nhist = a.st->nhist;
  }
  {
    // ---- one-sweep CGS2 (Gram-matrix form): the second pass coefficients V^H w' = h1 - G h1 with
    // G = V^H V, the basis Gram matrix, whose new column comes out of the same sweep as h1; then
    // one update w'' = w - V (h1 + h2) and ||w''||^2 = ||w||^2 - 2 Re(h^H h1) + h^H G h.
    // One grid barrier and two basis sweeps per step instead of three barriers and four sweeps.
    // grouped sweep for long chunks (cfg4: 3 567 elements per CTA, GMRES 23.4 -> 22.8 ms); per-vector
    // warps for short ones (cfg1 / cfg2 chunks of 32 / 784 elements measured slower grouped)
    // the previous steps' Gram block G[0..m-2][0..m-2] (written by earlier launches, complete at
    // pdl_wait) is staged into shared memory with cp.async while the dots sweep runs
    // (and the basis scale factors vs[0..m-1], read by every coefficient below)
    const int mp = a.m - 1;
    double2* gs = osm + 7 * a.ldr;  // column-major [mp][mp] when a.gram_smem
    double* vss = reinterpret_cast<double*>(osm + 7 * a.ldr + (a.gram_smem ? a.ldr * a.ldr : 0));
    if (a.gram_smem) {
      for (int e = threadIdx.x; e < mp * mp; e += kCoopThreads) {
        const int k = e / mp, l = e - k * mp;
        const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(gs + e));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(a.gram + static_cast<int64_t>(k) * a.ldr + l)
                     : "memory");
      }
    }
    for (int l = threadIdx.x; l < a.m; l += kCoopThreads) {
      const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(vss + l));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(a.vs + l) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (a.N >= static_cast<int64_t>(kOrthGroupedMinChunk) * (gridDim.x - 1)) orth_dots_gram(a, c0, c1);
    else orth_dots_gram_pv(a, c0, c1);
    OPROBE();
    grid_barrier(a.bar);
    OPROBE();
    const int m = a.m, nblk = gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double2* h1s = osm + 4 * a.ldr;
    double2* gcol = osm + 5 * a.ldr;
    double2* gh = osm + 6 * a.ldr;
    // ||w||^2 partials: the last warp sums them now (their L2 round trip overlaps the partials'
    // loads of the other warps); the norm below reads the total from shared memory
    __shared__ double wn_s, hn2_g;
    if (warp == kCoopThreads / 32 - 1) {
      double wn = 0.0;
      if (nblk <= 160) {
        double q[5];
#pragma unroll
        for (int j = 0; j < 5; ++j) q[j] = lane + 32 * j < nblk ? __ldcg(a.npart + lane + 32 * j) : 0.0;
#pragma unroll
        for (int j = 0; j < 5; ++j) wn += q[j];
      } else {
        for (int b = lane; b < nblk; b += 32) wn += __ldcg(a.npart + b);
      }
      wn = warp_sum(wn);
      if (lane == 0) wn_s = wn;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    const double vlast = vss[m - 1];
    // cross-CTA partials: one warp per (vector, sum) item, up to 4 items per warp with all of their
    // loads issued before any is summed (one L2 round trip); each item is summed in a fixed order,
    // identical in every CTA (the decisions below are uniform across the grid)
    {
      constexpr int NWc = kCoopThreads / 32, IT = 4, Q = 5;
      const int items = 2 * m;
      auto item_ptr = [&](int it) {
        return ((it & 1) ? a.part2 : a.part) + static_cast<int64_t>(it >> 1) * nblk;
      };
      auto finish = [&](int it, double2 sacc) {
        sacc = warp_sum(sacc);
        if (lane == 0) {
          const int l = it >> 1;
          if (it & 1) gcol[l] = cscale(sacc, vss[l] * vlast);  // G[l][m-1]
          else h1s[l] = cscale(sacc, vss[l]);
        }
      };
      if (nblk <= 32 * Q && items <= IT * NWc) {
        double2 q[IT][Q];
#pragma unroll
        for (int r = 0; r < IT; ++r) {
          const int it = warp + r * NWc;
#pragma unroll
          for (int j = 0; j < Q; ++j)
            q[r][j] = (it < items && lane + 32 * j < nblk) ? __ldcg(item_ptr(it) + lane + 32 * j) : make_double2(0, 0);
        }
#pragma unroll
        for (int r = 0; r < IT; ++r) {
          const int it = warp + r * NWc;
          double2 sacc = make_double2(0, 0);
#pragma unroll
          for (int j = 0; j < Q; ++j) sacc = cadd(sacc, q[r][j]);
          if (it < items) finish(it, sacc);
        }
      } else {
        for (int it = warp; it < items; it += NWc) {
          double2 sacc = make_double2(0, 0);
          for (int b = lane; b < nblk; b += 32) sacc = cadd(sacc, __ldcg(item_ptr(it) + b));
          finish(it, sacc);
        }
      }
    }
    __syncthreads();
    OPROBE();
    auto G = [&](int l, int k) -> double2 {  // G[l][k], Hermitian; column m-1 from this step
      if (k == m - 1) return gcol[l];
      if (l == m - 1) return make_double2(gcol[k].x, -gcol[k].y);
      return a.gram_smem ? gs[k * mp + l] : a.gram[static_cast<int64_t>(k) * a.ldr + l];
    };
    // h2 = h1 - G h1, h = h1 + h2; gh = G h (for the norm)
    for (int l = warp; l < m; l += kCoopThreads / 32) {
      double2 t = make_double2(0, 0);
      for (int k = lane; k < m; k += 32) t = cadd(t, cmul(G(l, k), h1s[k]));
      t = warp_sum(t);
      if (lane == 0) {
        const double2 h = csub(cscale(h1s[l], 2.0), t);
        coef[l] = cscale(h, vss[l]);
        hsm[l] = h;
      }
    }
    __syncthreads();
    OPROBE();
    // (G h)_l, then ||w''||^2 = ||w||^2 - 2 Re(h^H h1) + h^H G h -- every CTA evaluates it (same
    // data, same order), so the precision test below is uniform across the grid
    for (int l = warp; l < m; l += kCoopThreads / 32) {
      double2 t = make_double2(0, 0);
      for (int k = lane; k < m; k += 32) t = cadd(t, cmul(G(l, k), hsm[k]));
      t = warp_sum(t);
      if (lane == 0) gh[l] = t;
    }
    __syncthreads();
    OPROBE();
    if (threadIdx.x < 32) {
      double t = 0.0;
      for (int l = threadIdx.x; l < m; l += 32)
        t += -2.0 * (hsm[l].x * h1s[l].x + hsm[l].y * h1s[l].y) + (hsm[l].x * gh[l].x + hsm[l].y * gh[l].y);
      t = warp_sum(t);
      if (threadIdx.x == 0) hn2_g = wn_s + t;
    }
    __syncthreads();
    OPROBE();
    // below ~1e-13 of ||w||^2 the formula is cancellation noise (e.g. a lucky breakdown): measure
    // ||w''|| directly instead (third sweep + barrier)
    const bool direct = !(hn2_g > 1e-13 * wn_s);
    double2* hcol = a.rcols + static_cast<int64_t>(jcol) * a.ldr;
    if (blockIdx.x == 0) {
      for (int l = threadIdx.x; l < m; l += kCoopThreads) {  // keep the Gram matrix for later steps
        a.gram[static_cast<int64_t>(m - 1) * a.ldr + l] = gcol[l];
        a.gram[static_cast<int64_t>(l) * a.ldr + (m - 1)] = make_double2(gcol[l].x, -gcol[l].y);
      }
      orth_prepare_givens(a, jcol, hsm, snl, csl, hcol);
      if (!direct && threadIdx.x == 0) {
        givens_finish(a, jcol, hsm[jcol], hn2_g, g_j, beta0, nhist);
        if (a.ts != nullptr) a.ts[2 * k_step + 3] = global_ns();
      }
    }
    if (!direct) {
      OPROBE();
      orth_update(a, coef, c0, c1);
#ifdef TOEP_ORTH_PROBE
      __syncthreads();
      OPROBE();
      if (blockIdx.x == 1 && threadIdx.x == 0 && (a.m == 8 || a.m == 16 || a.m == 24 || a.m == 31))
        printf("orth-gram m=%d: dots %lld bar %lld partials %lld Gh1 %lld Gh %lld norm %lld ->upd %lld upd %lld ns\n",
               a.m, pt[1] - pt[0], pt[2] - pt[1], pt[3] - pt[2], pt[4] - pt[3], pt[5] - pt[4], pt[6] - pt[5],
               pt[7] - pt[6], pt[8] - pt[7]);
#endif
      return;
    }
    double nrm = orth_update(a, coef, c0, c1);
    nrm = warp_sum(nrm);
    if (lane == 0) red[warp] = nrm;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = red[0];
      for (int ww = 1; ww < kCoopThreads / 32; ++ww) t += red[ww];
      a.npart[blockIdx.x] = t;
    }
    grid_barrier(a.bar);
    if (blockIdx.x == 0 && threadIdx.x < 32) {
      double hn2 = 0.0;
      for (int b = threadIdx.x; b < nblk; b += 32) hn2 += __ldcg(a.npart + b);
      hn2 = warp_sum(hn2);
      if (threadIdx.x == 0) {
        givens_finish(a, jcol, hsm[jcol], hn2, g_j, beta0, nhist);
        if (a.ts != nullptr) a.ts[2 * k_step + 3] = global_ns();
      }
    }
    return;
  }
}

// y = R^-1 g (gmres.py:193-204), R upper triangular from the rotated columns (rcols[j][0..j]).
// One warp, column-oriented substitution: lane l owns rows l, l+32, ...; the pivots' reciprocals
// are formed for all rows at once up front (the divisions leave the serial chain), then each solved
// y_i is broadcast with a shuffle and subtracted from the remaining rows.  A zero pivot gives
// y_i = 0.  rs: column i of R at rs[i * rld + 0..i]; out[i] = y_i * (scale ? scale[i] : 1).
template <int ROWS>
__device__ __forceinline__ void tri_solve_warp(const double2* rs, int rld, const double2* g, int m, const double* scale,
                                               double2* out) {
  const int lane = threadIdx.x & 31;
  double2 acc[ROWS], pinv[ROWS];
#pragma unroll
  for (int q = 0; q < ROWS; ++q) {
    const int r = lane + 32 * q;
    acc[q] = make_double2(0, 0);
    pinv[q] = make_double2(0, 0);
    if (r < m) {
      acc[q] = g[r];
      const double2 d = rs[static_cast<int64_t>(r) * rld + r];
      if (!(d.x == 0.0 && d.y == 0.0)) {
        const double inv = 1.0 / (d.x * d.x + d.y * d.y);
        pinv[q] = make_double2(d.x * inv, -d.y * inv);  // 1 / d = conj(d) / |d|^2
      }
    }
  }
  for (int i = m - 1; i >= 0; --i) {
    const int qi = i >> 5;
    double2 yi = make_double2(0, 0);
#pragma unroll
    for (int q = 0; q < ROWS; ++q)
      if (q == qi) yi = cmul(acc[q], pinv[q]);
    yi.x = __shfl_sync(0xffffffffu, yi.x, i & 31);
    yi.y = __shfl_sync(0xffffffffu, yi.y, i & 31);
    if (lane == (i & 31)) out[i] = scale != nullptr ? cscale(yi, scale[i]) : yi;
    const double2 ny = make_double2(-yi.x, -yi.y);
#pragma unroll
    for (int q = 0; q < ROWS; ++q) {
      const int r = lane + 32 * q;
      if (r < i) cfma(acc[q], rs[static_cast<int64_t>(i) * rld + r], ny);
    }
  }
}

// every thread of the block stages the m x m upper triangle of R into shared memory (column-major,
// leading dimension m) with its loads batched: one L2 round trip per batch of 8
template <int NT>
__device__ __forceinline__ void stage_triangle(const double2* rcols, int ldr, int m, double2* rsm) {
  constexpr int B = 8;
  const int tot = m * m;
  for (int e0 = threadIdx.x; e0 < tot; e0 += B * NT) {
    double2 v[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int e = e0 + u * NT, i = e / max(m, 1), r = e - i * m;
      v[u] = (e < tot && r <= i) ? rcols[static_cast<int64_t>(i) * ldr + r] : make_double2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int e = e0 + u * NT;
      if (e < tot) rsm[e] = v[u];
    }
  }
}

constexpr int kBsRows = 8;  // rows per lane: cycles up to 256 steps
constexpr int kBsThreads = 256;  // k_backsub block: all stage the triangle, warp 0 solves
__global__ void k_backsub(const GState* st, const double2* rcols, int ldr, const double2* g, double2* y, int staged) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ double2 rsm[];  // staged: [m][m] column-major upper triangle
  const int m = st->m;
  const double2* rs = rcols;
  int rld = ldr;
  if (staged) {
    stage_triangle<kBsThreads>(rcols, ldr, m, rsm);
    __syncthreads();
    rs = rsm;
    rld = m;
  }
  if (threadIdx.x >= 32) return;  // one warp solves
  tri_solve_warp<kBsRows>(rs, rld, g, m, nullptr, y);
}

// cycles up to kSolveAxpyMax steps: the triangular solve and x += V (vs y) in one kernel -- every
// CTA stages R (L2-resident, m^2 * 16 bytes) and solves it redundantly, then updates its elements
constexpr int kSolveAxpyMax = 64;
__global__ void __launch_bounds__(kThreads)
k_solve_axpy(const GState* st, const double2* __restrict__ rcols, int ldr, const double2* __restrict__ g,
             const double* __restrict__ vs, const double2* __restrict__ V, int64_t ld, int m_max,
             double2* __restrict__ x, int64_t N) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ double2 ssm[];  // [m_max][m_max] triangle | coef [m_max]
  const int m = min(m_max, st->m);
  double2* rsm = ssm;
  double2* coef = ssm + static_cast<int64_t>(m_max) * m_max;
  stage_triangle<kThreads>(rcols, ldr, m, rsm);
  __syncthreads();
  if (threadIdx.x < 32) tri_solve_warp<(kSolveAxpyMax + 31) / 32>(rsm, m, g, m, vs, coef);
  __syncthreads();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; i < N;
       i += static_cast<int64_t>(gridDim.x) * kThreads) {
    double2 acc = x[i];
    int l = 0;
    for (; l + 7 < m; l += 8) {  // 8 independent basis loads in flight
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = V[(l + u) * ld + i];
#pragma unroll
      for (int u = 0; u < 8; ++u) cfma(acc, v[u], coef[l + u]);
    }
    for (; l < m; ++l) cfma(acc, V[l * ld + i], coef[l]);
    x[i] = acc;
  }
}

// long cycles (> 256 steps): the same substitution on one thread, row-oriented
__global__ void k_backsub_serial(const GState* st, const double2* rcols, int ldr, const double2* g, double2* y) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x != 0) return;
  const int m = st->m;
  for (int i = m - 1; i >= 0; --i) {
    const double2 d = rcols[static_cast<int64_t>(i) * ldr + i];
    if (d.x == 0.0 && d.y == 0.0) {
      y[i] = make_double2(0, 0);
      continue;
    }
    double2 acc = g[i];
    for (int k = i + 1; k < m; ++k) acc = csub(acc, cmul(rcols[static_cast<int64_t>(k) * ldr + i], y[k]));
    const double den = d.x * d.x + d.y * d.y;
    y[i] = make_double2((acc.x * d.x + acc.y * d.y) / den, (acc.y * d.x - acc.x * d.y) / den);
  }
}

// Per-thread host resources reused across solves: the mapped pinned flag word
// the device writes and a pool of CUDA events (creating / freeing these per
// solve costs milliseconds of host time).
struct HostRes {
  HostFlags* hf = nullptr;
  HostFlags* hf_dev = nullptr;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  // mapped page-locked block the device writes each cycle's report into (k_report)
  unsigned char* stage = nullptr;
  unsigned char* stage_dev = nullptr;
  size_t stage_cap = 0;
  unsigned seq = 0;
  unsigned char* stage_bytes(size_t bytes) {
    if (bytes > stage_cap) {
      if (stage != nullptr) cudaFreeHost(stage);
      stage = stage_dev = nullptr;
      stage_cap = 0;
      if (cudaHostAlloc(reinterpret_cast<void**>(&stage), bytes, cudaHostAllocMapped) != cudaSuccess ||
          cudaHostGetDevicePointer(reinterpret_cast<void**>(&stage_dev), stage, 0) != cudaSuccess) {
        cudaGetLastError();
        if (stage != nullptr) cudaFreeHost(stage);
        stage = stage_dev = nullptr;
        return nullptr;
      }
      std::memset(stage, 0, bytes);
      stage_cap = bytes;
    }
    return stage;
  }
  cudaEvent_t event() {
    if (used == pool.size()) {
      cudaEvent_t ev;
      cudaEventCreate(&ev);
      pool.push_back(ev);
    }
    return pool[used++];
  }
};

HostRes& host_res() {
  static thread_local HostRes r;
  if (r.hf == nullptr) {
    if (cudaHostAlloc(reinterpret_cast<void**>(&r.hf), sizeof(HostFlags), cudaHostAllocMapped) != cudaSuccess) {
      cudaGetLastError();
      r.hf = nullptr;
    } else {
      cudaHostGetDevicePointer(reinterpret_cast<void**>(&r.hf_dev), r.hf, 0);
    }
  }
  return r;
}

// TOEP_TRACE=1: host-side timeline of a solve on stderr (launch / wait split)
struct Trace {
  using clk = std::chrono::steady_clock;
  bool on = std::getenv("TOEP_TRACE") != nullptr;
  clk::time_point t0 = clk::now(), last = t0;
  double wait = 0.0;
  double launch_us_sum = 0.0, launch_us_max = 0.0;
  int steps = 0;
  void mark(const char* what) {
    if (!on) return;
    const auto now = clk::now();
    std::fprintf(stderr, "[toep_gmres] %-28s +%9.3f ms (t=%9.3f ms, waited %8.3f ms, step launch mean %.1f max %.1f us)\n",
                 what, std::chrono::duration<double, std::milli>(now - last).count(),
                 std::chrono::duration<double, std::milli>(now - t0).count(), wait,
                 steps ? launch_us_sum / steps : 0.0, launch_us_max);
    last = now;
  }
  // spin on the event: cudaEventSynchronize may yield the thread and wake it up
  // hundreds of microseconds late, which starves the launch queue
  // spin until the device has completed `target` steps overall (or stopped)
  // Every 4096 spins the stream is queried: a device fault returns TOEP_ERR_CUDA instead of
  // spinning forever, and a drained stream (nothing left that could advance the word) ends the wait.
  int wait_total(const HostFlags* hf, int target, cudaStream_t s) {
    const auto a = clk::now();
    for (unsigned spins = 1; hf->total < target && !hf->stop; ++spins) {
      if ((spins & 4095u) != 0) continue;
      const cudaError_t e = cudaStreamQuery(s);
      if (e == cudaSuccess) break;
      if (e != cudaErrorNotReady) {
        set_error("gmres: device error while waiting for step %d: %s", target, cudaGetErrorString(e));
        return TOEP_ERR_CUDA;
      }
    }
    if (on) wait += std::chrono::duration<double, std::milli>(clk::now() - a).count();
    return TOEP_OK;
  }
};

struct Engine {
  const toep_gmres_problem_t* p;
  cudaStream_t s;
  int64_t N;
  int nblk;
  double* norm_partial = nullptr;
  double2* tmp2 = nullptr;  // normalised copy for callback operators

  // y = A (scale * x); scale: optional device scalar
  int apply_a(const double2* x, const double* scale, double2* y, const int* stop) {
    if (p->op != nullptr) {
      const bool io = p->op->dtype == TOEP_C64;
      return matvec_impl(p->op, x, y, p->w, false, io, stop, s, scale);
    }
    const double2* xin = x;
    if (scale != nullptr) {
      TOEP_TRY(launch_k(k_scale, dim3(grid1()), dim3(kThreads), 0, s, x, tmp2, scale, N, stop));
      xin = tmp2;
    }
    const int rc = p->apply(p->apply_ctx, xin, y, p->w, s);
    TOEP_REQUIRE(rc == 0, TOEP_ERR_ARG, "operator callback failed (%d)", rc);
    return TOEP_OK;
  }
  bool precond_per_step() const { return p->precond == TOEP_PC_BLOCK || p->precond == TOEP_PC_CALLBACK; }
  // z = P^-1 x (BLOCK / CALLBACK)
  int apply_p(const double2* x, double2* z, const int* stop) {
    if (p->precond == TOEP_PC_BLOCK)
      return block_apply_impl(p->pinv, p->pside, x, z, p->n / p->pside, p->w, TOEP_C128, s, stop);
    if (p->precond == TOEP_PC_CALLBACK) {
      const int rc = p->papply(p->papply_ctx, x, z, p->w, s);
      TOEP_REQUIRE(rc == 0, TOEP_ERR_ARG, "preconditioner callback failed (%d)", rc);
      return TOEP_OK;
    }
    set_error("no per-step preconditioner");
    return TOEP_ERR_ARG;
  }
  int grid1() const { return static_cast<int>(std::min<int64_t>((N + kThreads - 1) / kThreads, 4 * 148)); }
  int norm2_partials(const double2* x) {
    return launch_k(k_norm2, dim3(nblk), dim3(kThreads), 0, s, x, N, norm_partial);
  }

  // ---- distributed reductions (rows split over ranks): collapse the per-CTA partials to one
  // value per quantity, all-reduce it over ranks, hand (buffer, 1) to the consumer kernel
  double* nred = nullptr;    // [1]
  double2* hred = nullptr;   // [ldr]
  bool distributed() const { return p->allreduce != nullptr; }
  int allreduce(void* buf, int64_t ndoubles) {
    const int rc = p->allreduce(p->allreduce_ctx, buf, ndoubles, s);
    TOEP_REQUIRE(rc == 0, TOEP_ERR_CUDA, "allreduce callback failed (%d)", rc);
    return TOEP_OK;
  }
  // norm partials -> (ptr, count) for k_init / k_cycle_start / k_givens
  int finish_norm(const double** ptr, int* count) {
    if (!distributed()) {
      *ptr = norm_partial;
      *count = nblk;
      return TOEP_OK;
    }
    TOEP_TRY(launch_k(k_collapse_d, dim3(1), dim3(32), 0, s, (const double*)norm_partial, nblk, nred));
    TOEP_TRY(allreduce(nred, 1));
    *ptr = nred;
    *count = 1;
    return TOEP_OK;
  }
  int finish_dots(const double2* part, int m, const double2** ptr, int* count) {
    if (!distributed()) {
      *ptr = part;
      *count = nblk;
      return TOEP_OK;
    }
    TOEP_TRY(launch_k(k_collapse_c, dim3(1), dim3(256), 0, s, part, m, nblk, hred));
    TOEP_TRY(allreduce(hred, 2 * static_cast<int64_t>(m)));
    *ptr = hred;
    *count = 1;
    return TOEP_OK;
  }
};

int gmres_run(const toep_gmres_problem_t* p, const toep_gmres_cfg_t* cfg, const double2* b, double2* x,
              cudaStream_t s, toep_gmres_report_t* rep) {
  using clk = std::chrono::steady_clock;
  const auto t_start = clk::now();
  Trace tr;
  keep_pool();
  TOEP_REQUIRE(cfg->tol > 0, TOEP_ERR_ARG, "tol must be > 0");
  TOEP_REQUIRE(cfg->max_iter >= 1, TOEP_ERR_ARG, "max_iter must be >= 1");
  TOEP_REQUIRE(cfg->restart >= 0, TOEP_ERR_ARG, "restart must be >= 1 or 0 (none)");
  TOEP_REQUIRE(p->op != nullptr || p->apply != nullptr, TOEP_ERR_ARG, "no operator");
  TOEP_REQUIRE(p->n >= 1 && p->w >= 1, TOEP_ERR_SHAPE, "empty system");
  if (p->op != nullptr)
    TOEP_REQUIRE(op_dim(p->op) == p->n, TOEP_ERR_SHAPE, "rhs rows %lld != operator dim %lld", (long long)p->n,
                 (long long)op_dim(p->op));
  if (p->precond == TOEP_PC_BLOCK || p->precond == TOEP_PC_FOLDED)
    TOEP_REQUIRE(p->pinv != nullptr && p->pside >= 1 && (p->n % p->pside) == 0, TOEP_ERR_SHAPE,
                 "preconditioner side does not divide n");
  if (p->precond == TOEP_PC_FOLDED)
    TOEP_REQUIRE(p->pmat != nullptr && p->op != nullptr, TOEP_ERR_ARG, "folded preconditioner needs op and pmat");
  if (p->precond == TOEP_PC_CALLBACK) TOEP_REQUIRE(p->papply != nullptr, TOEP_ERR_ARG, "no preconditioner callback");

  Engine e{p, s, p->n * p->w, 0};
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  e.nblk = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((e.N + kThreads - 1) / kThreads, sms)));
  const int64_t N = e.N;
  const int64_t max_total = std::min<int64_t>(cfg->max_iter, N);
  const int cycle_len = static_cast<int>(cfg->restart == 0 ? max_total : std::min<int64_t>(cfg->restart, max_total));
  const int ldr = cycle_len + 1;
  const int nblk = e.nblk;
  const int grid1 = e.grid1();

  double2 *V = nullptr, *tmp = nullptr, *tmp2 = nullptr, *pb = nullptr, *h1 = nullptr, *rres = nullptr;
  double2 *rcols = nullptr, *sn = nullptr, *g = nullptr, *y = nullptr, *part1 = nullptr, *part2 = nullptr;
  double *cs = nullptr, *hist = nullptr, *vs = nullptr;
  GState* st = nullptr;
  unsigned* bar = nullptr;  // grid barrier of k_orth_coop
  long long* ts = nullptr;  // device phase stamps (replace per-step events on the cooperative path)
  double2* gram = nullptr;  // Gram matrix of the cycle's basis (one-sweep CGS2)
  HostRes& res = host_res();
  res.used = 0;
  HostFlags* hf = res.hf;
  HostFlags* hf_dev = res.hf_dev;
  int rc = TOEP_OK;
  // stream-ordered frees; error paths also drain the stream (success: the last report already
  // proved every kernel done)
  // every device buffer of the solve is carved from ONE stream-ordered allocation (two pool calls
  // per solve instead of ~40)
  unsigned char* arena = nullptr;
  // error paths also drain the stream (success: the last report already proved every kernel done)
  auto cleanup = [&](bool sync = true) {
    if (arena != nullptr) cudaFreeAsync(arena, s);
    arena = nullptr;
    if (sync) cudaStreamSynchronize(s);
    res.used = 0;
  };
  TOEP_REQUIRE(hf != nullptr, TOEP_ERR_OOM, "pinned allocation failed");
  std::vector<std::pair<void**, size_t>> plan;
#define G_ALLOC(ptr, count) plan.emplace_back(reinterpret_cast<void**>(&(ptr)), sizeof(*(ptr)) * (size_t)(count))
#define G_TRY(expr)      \
  do {                   \
    rc = (expr);         \
    if (rc != TOEP_OK) { \
      cleanup();         \
      return rc;         \
    }                    \
  } while (0)
#define G_CUDA(call)                                                                 \
  do {                                                                               \
    const cudaError_t _ge = (call);                                                  \
    if (_ge != cudaSuccess) {                                                        \
      set_error("gmres: %s: %s", #call, cudaGetErrorString(_ge));                    \
      cleanup();                                                                     \
      return TOEP_ERR_CUDA;                                                          \
    }                                                                                \
  } while (0)
  G_ALLOC(V, (int64_t)(cycle_len + 1) * N);
  G_ALLOC(tmp, N);
  G_ALLOC(pb, N);
  G_ALLOC(tmp2, N);
  G_ALLOC(rres, N);
  G_ALLOC(h1, ldr);
  G_ALLOC(rcols, (int64_t)cycle_len * ldr);
  G_ALLOC(sn, cycle_len + 1);
  G_ALLOC(g, cycle_len + 2);
  G_ALLOC(y, cycle_len + 1);
  G_ALLOC(cs, cycle_len + 1);
  G_ALLOC(vs, cycle_len + 2);
  G_ALLOC(hist, max_total + 2);
  G_ALLOC(st, 1);
  G_ALLOC(e.norm_partial, nblk);
  G_ALLOC(part1, (int64_t)nblk * ldr);
  G_ALLOC(part2, (int64_t)nblk * ldr);
  if (e.distributed()) {
    G_ALLOC(e.nred, 1);
    G_ALLOC(e.hred, ldr);
  }
  G_ALLOC(bar, 2);  // grid barrier of the cooperative orthogonalisation kernel
  G_ALLOC(ts, 2 * max_total + 4);
  G_ALLOC(gram, (int64_t)ldr * ldr);
  {
    size_t bytes = 0;
    for (auto& pp : plan) bytes += (pp.second + 255) & ~size_t(255);
    if (cudaMallocAsync(reinterpret_cast<void**>(&arena), bytes, s) != cudaSuccess) {
      cudaGetLastError();
      arena = nullptr;
      set_error("out of device memory in gmres (%zu bytes)", bytes);
      cleanup();
      return TOEP_ERR_OOM;
    }
    size_t off = 0;
    for (auto& pp : plan) {
      *pp.first = arena + off;
      off += (pp.second + 255) & ~size_t(255);
    }
  }
  e.tmp2 = tmp2;
  TOEP_CUDA(cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), s));
  // Gram block staged in shared memory for cycles up to 64 vectors (64 KB); larger cycles read it from L2
  const bool gram_smem = ldr <= 64;
  const size_t coop_smem = std::max({sizeof(double2) * ldr * (1 + kCoopThreads / 32),
                                     (2 * sizeof(double2) + sizeof(double)) * ldr,
                                     sizeof(double2) * (7 * ldr + (gram_smem ? ldr * ldr : 0)) +
                                         sizeof(double) * ldr});
  const int coop_grid = nblk;
  // the cooperative orthogonalisation kernel (grid barrier): single process, cycles up to
  // kMaxOrthM vectors, and every CTA co-resident; otherwise the per-phase kernel chain
  bool use_coop = !e.distributed() && cycle_len <= kMaxOrthM;
  if (use_coop) {
    ensure_smem(k_orth_coop, coop_smem + 8 * 1024);  // + headroom: the kernel's static shared memory
    // same (maximal) shared-memory carveout as the 2-D DFT kernels, so the next forward DFT can
    // become resident next to this kernel without an SM reconfiguration
    cudaFuncSetAttribute(k_orth_coop, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_orth_coop, kCoopThreads, coop_smem) != cudaSuccess ||
        per_sm * sms < coop_grid)
      use_coop = false;
    cudaGetLastError();
  }
  hf->stop = 0;
  hf->total = 0;
  hf->converged = 0;
  hf->breakdown = 0;
  tr.mark("allocations");

  const bool timed = cfg->timings != 0;
  // orthogonalisation: one-sweep CGS2 in Gram-matrix form (histories track the reference's MGS to
  // 1e-6; the measured alternatives -- explicit two-pass CGS2, selective re-orthogonalisation --
  // are recorded in DESIGN.md)
  const L2Prefetch orth_pf = (p->op != nullptr && p->w == 1) ? binprod_prefetch_plan(p->op->dtype, p->op->DT,
                                                                                    p->op->K, p->op->n0, 2)
                                                            : L2Prefetch{};
  // per-step matvec / orthogonalisation split from device timestamps: events between the
  // kernels of a step would break their programmatic-dependent-launch overlap
  bool stamped = timed && use_coop && !e.precond_per_step();
  long long* ts_dev = stamped ? ts : nullptr;
  struct Phase { cudaEvent_t a, b; int kind; };
  std::vector<Phase> phases;
  auto mark = [&](int kind, cudaEvent_t a) {
    cudaEvent_t bb = res.event();
    cudaEventRecord(bb, s);
    phases.push_back({a, bb, kind});
    return bb;
  };
  auto start_mark = [&]() {
    cudaEvent_t a = res.event();
    cudaEventRecord(a, s);
    return a;
  };
  const size_t coef_smem = sizeof(double2) * ldr;
  const bool solve_axpy = cycle_len <= kSolveAxpyMax;  // else backsub kernel + axpy kernel
  const size_t solve_axpy_smem = sizeof(double2) * static_cast<size_t>(cycle_len) * (cycle_len + 1);
  if (solve_axpy) ensure_smem(k_solve_axpy, solve_axpy_smem);
  const bool backsub_warp = cycle_len <= 32 * kBsRows;  // else the serial kernel
  const int backsub_staged = sizeof(double2) * static_cast<size_t>(cycle_len) * cycle_len <= 200 * 1024 ? 1 : 0;
  const size_t backsub_smem = backsub_staged ? sizeof(double2) * static_cast<size_t>(cycle_len) * cycle_len : 0;
  if (backsub_smem > 48 * 1024)
    cudaFuncSetAttribute(k_backsub, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)backsub_smem);
  const size_t givens_smem = (2 * sizeof(double2) + sizeof(double)) * ldr;
  if (givens_smem > 48 * 1024)
    cudaFuncSetAttribute(k_givens, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)givens_smem);
  if (coef_smem > 48 * 1024) {
    cudaFuncSetAttribute(k_upd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)coef_smem);
    cudaFuncSetAttribute(k_axpy_basis, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)coef_smem);
  }

  // ---- P^-1 b, beta0 (gmres.py:104-113)
  const double2* zb = b;
  {
    cudaEvent_t t0 = timed ? start_mark() : nullptr;
    if (p->precond == TOEP_PC_BLOCK || p->precond == TOEP_PC_FOLDED) {
      G_TRY(block_apply_impl(p->pinv, p->pside, b, pb, p->n / p->pside, p->w, TOEP_C128, s, nullptr));
      zb = pb;
    } else if (p->precond == TOEP_PC_CALLBACK) {
      G_TRY(e.apply_p(b, pb, nullptr));
      zb = pb;
    }
    if (timed) mark(1, t0);
  }
  // every value the host needs back (state, exit-residual and ||b|| partials, history) lands in
  // one page-locked block read back by ONE copy + sync at the end of each cycle; the start of the
  // solve does not wait for the device at all (b = 0 is caught by k_cycle_start)
  const int hist_copy = static_cast<int>(std::min<int64_t>(rep->history != nullptr ? rep->history_cap : 0,
                                                           max_total + 2));
  ReportLayout lay{};
  lay.st = 16;
  lay.r = (lay.st + sizeof(GState) + 15) & ~size_t(15);
  lay.b = lay.r + sizeof(double) * nblk;
  lay.h = lay.b + sizeof(double) * nblk;
  lay.t = lay.h + sizeof(double) * (hist_copy + 1);
  lay.bytes = lay.t + sizeof(long long) * (2 * max_total + 4);
  unsigned char* stage = res.stage_bytes(lay.bytes);
  if (stage == nullptr) {
    set_error("pinned allocation failed");
    cleanup();
    return TOEP_ERR_OOM;
  }
  const GState& hst = *reinterpret_cast<const GState*>(stage + lay.st);
  const double* h_rpart = reinterpret_cast<const double*>(stage + lay.r);
  double* h_bpart = reinterpret_cast<double*>(stage + lay.b);
  const double* h_hist = reinterpret_cast<const double*>(stage + lay.h);
  const long long* h_ts = reinterpret_cast<const long long*>(stage + lay.t);
  // wait for report `want` (spin on the mapped sequence word; a device fault or a stream that
  // drained without writing it ends the wait with an error)
  auto wait_report = [&](unsigned want) -> int {
    volatile const unsigned* sq = reinterpret_cast<volatile const unsigned*>(stage);
    for (unsigned spins = 1; *sq != want; ++spins) {
      if ((spins & 4095u) != 0) continue;
      const cudaError_t ce = cudaStreamQuery(s);
      if (ce == cudaSuccess) {
        if (*sq == want) break;
        set_error("gmres: cycle report missing");
        return TOEP_ERR_CUDA;
      }
      if (ce != cudaErrorNotReady) {
        set_error("gmres cycle failed: %s", cudaGetErrorString(ce));
        return TOEP_ERR_CUDA;
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    return TOEP_OK;
  };
  int rcnt = 0, bcnt = 0;
  const double* nptr = nullptr;
  int ncnt = 0;
  G_TRY(e.norm2_partials(zb));
  G_TRY(e.finish_norm(&nptr, &ncnt));
  G_TRY(launch_k(k_init, dim3(1), dim3(32), 0, s, st, nptr, ncnt, hist));
  if (zb != b) {  // ||b|| for the exit residual (unpreconditioned)
    G_TRY(e.norm2_partials(b));
    G_TRY(e.finish_norm(&nptr, &ncnt));
  }
  bcnt = ncnt;
  G_CUDA(cudaMemcpyAsync(h_bpart, nptr, sizeof(double) * ncnt, cudaMemcpyDeviceToHost, s));
  tr.mark("init (P^-1 b, beta0) queued");
  rep->iterations = 0;
  rep->converged = 1;
  rep->breakdown = 0;
  rep->t_matvec = rep->t_precond = rep->t_orth = 0.0;
  cudaMemsetAsync(x, 0, N * sizeof(double2), s);

  int* stop_dev = &st->stop;
  int* m_dev = &st->m;
  int total = 0;
  bool first = true;
  while (true) {
    // ---- cycle start (gmres.py:123-144): V[0] = P^-1 (b - A x), vs[0] = 1 / ||.||
    double2* v0 = V;
    if (!first) {  // tmp = A x (P^-1 A x when folded) from the previous cycle's exit block
      cudaEvent_t t0 = timed ? start_mark() : nullptr;
      if (p->precond == TOEP_PC_FOLDED) {
        G_TRY(launch_k(k_sub, dim3(grid1), dim3(kThreads), 0, s, (const double2*)pb, (const double2*)tmp, v0, N));
      } else if (e.precond_per_step()) {
        G_TRY(e.apply_p(rres, v0, nullptr));  // rres = b - A x
      } else {
        G_TRY(launch_k(k_sub, dim3(grid1), dim3(kThreads), 0, s, b, (const double2*)tmp, v0, N));
      }
      if (timed) mark(1, t0);
    } else {
      cudaMemcpyAsync(v0, zb, N * sizeof(double2), cudaMemcpyDeviceToDevice, s);
    }
    first = false;
    G_TRY(e.norm2_partials(v0));
    G_TRY(e.finish_norm(&nptr, &ncnt));
    G_TRY(launch_k(k_cycle_start, dim3(1), dim3(32), 0, s, st, nptr, ncnt, cfg->tol, g, vs, hf_dev, ts_dev));

    // ---- Arnoldi steps (gmres.py:146-190)
    int j = 0;
    while (j < cycle_len && total + j < max_total) {
      const auto t_launch0 = clk::now();
      const double2* vj = V + static_cast<int64_t>(j) * N;
      double2* w = V + static_cast<int64_t>(j + 1) * N;  // unnormalised v_{j+1} is built in place
      const bool ev_timed = timed && !(stamped && use_coop);
      cudaEvent_t t0 = ev_timed ? start_mark() : nullptr;
      if (e.precond_per_step()) {
        G_TRY(e.apply_a(vj, vs + j, tmp, stop_dev));
        if (ev_timed) t0 = mark(0, t0);
        G_TRY(e.apply_p(tmp, w, stop_dev));
        if (ev_timed) t0 = mark(1, t0);
      } else {
        G_TRY(e.apply_a(vj, vs + j, w, stop_dev));
        if (ev_timed) t0 = mark(0, t0);
      }
      const int m = j + 1;
      if (use_coop) {
        OrthArgs oa{V, N, m, vs, w, part1, e.norm_partial, h1, st, rcols, ldr, cs, sn, g, hist, vs, cfg->tol,
                    static_cast<int>(max_total), cycle_len, hf_dev, bar, ts_dev, orth_pf, gram, part2,
                    gram_smem ? 1 : 0};
        rc = launch_gridsync(k_orth_coop, dim3(coop_grid), dim3(kCoopThreads), coop_smem, s, oa, (const int*)stop_dev);
        if (rc != TOEP_OK) {  // cooperative launch unavailable: permanent fallback to the 4-kernel chain
          use_coop = false;
          rc = TOEP_OK;
          if (stamped) {  // this step's matvec went unmeasured; events from here on
            stamped = false;
            ts_dev = nullptr;
          }
        }
      }
      if (use_coop) {
        // orthogonalisation + Givens done by k_orth_coop
      } else {
      const double2* dptr = nullptr;
      int dcnt = 0;
      G_TRY(launch_k(k_dots, dim3(nblk), dim3(kThreads), 0, s, (const double2*)V, N, m, (const double2*)w, N, part1,
                     (const int*)stop_dev));
      G_TRY(e.finish_dots(part1, m, &dptr, &dcnt));
      G_TRY(launch_k(k_upd, dim3(nblk), dim3(kThreads), coef_smem, s, (const double2*)V, N, m, (const double*)vs,
                     dptr, dcnt, w, N, 1, h1, (const double2*)nullptr, part2, (double*)nullptr, (const int*)stop_dev));
      G_TRY(e.finish_dots(part2, m, &dptr, &dcnt));
      G_TRY(launch_k(k_upd, dim3(nblk), dim3(kThreads), coef_smem, s, (const double2*)V, N, m, (const double*)vs,
                     dptr, dcnt, w, N, 2, rcols + (int64_t)j * ldr, (const double2*)h1, (double2*)nullptr,
                     e.norm_partial, (const int*)stop_dev));
      G_TRY(e.finish_norm(&nptr, &ncnt));
      G_TRY(launch_k(k_givens, dim3(1), dim3(32), givens_smem, s, st, nptr, ncnt, rcols, ldr, cs, sn, g, hist, vs, cfg->tol,
                     static_cast<int>(max_total), cycle_len, hf_dev));
      }
      if (ev_timed) mark(2, t0);
      if (tr.on) {
        const double us = std::chrono::duration<double, std::micro>(clk::now() - t_launch0).count();
        tr.launch_us_sum += us;
        tr.launch_us_max = std::max(tr.launch_us_max, us);
        tr.steps++;
      }
      ++j;
      // keep up to kLag steps queued ahead of the one the host last saw finish.  Progress is read
      // from the mapped flag word the Givens step writes (no events between the kernels: an event
      // record would break their programmatic-dependent-launch chain)
      constexpr int kLag = 1;
      if (j > kLag) {
        G_TRY(tr.wait_total(hf, total + (j - kLag), s));
        if (hf->stop) break;
      }
    }
    tr.mark("arnoldi steps launched");
    // ---- assemble x += V y (gmres.py:192-204)
    if (solve_axpy)
      G_TRY(launch_k(k_solve_axpy, dim3(grid1), dim3(kThreads), solve_axpy_smem, s, (const GState*)st,
                     (const double2*)rcols, ldr, (const double2*)g, (const double*)vs, (const double2*)V, N, cycle_len,
                     x, N));
    else if (backsub_warp)
      G_TRY(launch_k(k_backsub, dim3(1), dim3(kBsThreads), backsub_smem, s, (const GState*)st, (const double2*)rcols, ldr,
                     (const double2*)g, y, backsub_staged));
    else
      G_TRY(launch_k(k_backsub_serial, dim3(1), dim3(32), 0, s, (const GState*)st, (const double2*)rcols, ldr,
                     (const double2*)g, y));
    if (!solve_axpy)
      G_TRY(launch_k(k_axpy_basis, dim3(grid1), dim3(kThreads), coef_smem, s, (const double2*)V, N, cycle_len,
                     (const int*)m_dev, (const double*)vs, (const double2*)y, x, N));
    // ---- exit residual ||b - A x|| (gmres.py:209-216), unpreconditioned, queued before the host
    // learns whether the solve ends here: A x is also the next cycle's start on a restart
    {
      cudaEvent_t t0 = timed ? start_mark() : nullptr;
      G_TRY(e.apply_a(x, nullptr, tmp, nullptr));
      const double2* ax = tmp;
      if (p->precond == TOEP_PC_FOLDED) {  // A x = P (P^-1 A x)
        G_TRY(block_apply_impl(p->pmat, p->pside, tmp, rres, p->n / p->pside, p->w, TOEP_C128, s, nullptr));
        ax = rres;
      }
      if (timed) mark(0, t0);
      G_TRY(launch_k(k_sub, dim3(grid1), dim3(kThreads), 0, s, b, ax, rres, N));
      G_TRY(e.norm2_partials(rres));
      G_TRY(e.finish_norm(&nptr, &ncnt));
      rcnt = ncnt;
    }
    const unsigned want = ++res.seq;
    G_TRY(launch_k(k_report, dim3(1), dim3(256), 0, s, (const GState*)st, nptr, rcnt, (const double*)hist, hist_copy,
                   (const long long*)ts_dev, res.stage_dev, lay, want));
    G_TRY(wait_report(want));
    total = hst.total;
    tr.mark("cycle synced");
    if (hst.converged || hst.breakdown || total >= max_total) break;
  }

  auto host_sum = [](const double* v, int n) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += v[i];
    return std::sqrt(t);
  };
  tr.mark("exit residual synced");
  if (hst.beta0 == 0.0) {  // b = 0 (P^-1 b = 0): x = 0, residual 0
    rep->final_residual = 0.0;
    rep->iterations = 0;
    rep->converged = 1;
    rep->breakdown = 0;
  } else {
    rep->final_residual = host_sum(h_rpart, rcnt) / host_sum(h_bpart, bcnt);
    rep->iterations = hst.total;
    rep->converged = hst.converged;
    rep->breakdown = hst.breakdown;
  }
  const int nh = std::min(hst.nhist, hist_copy);
  if (nh > 0) std::memcpy(rep->history, h_hist, nh * sizeof(double));
  rep->n_history = hst.nhist;
  if (timed && stamped) {
    for (int k = 0; k < hst.total; ++k) {
      rep->t_matvec += 1e-9 * static_cast<double>(h_ts[2 * k + 2] - h_ts[2 * k + 1]);
      rep->t_orth += 1e-9 * static_cast<double>(h_ts[2 * k + 3] - h_ts[2 * k + 2]);
    }
  }
  if (timed && !phases.empty()) {
    cudaStreamSynchronize(s);
    for (auto& ph : phases) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, ph.a, ph.b) == cudaSuccess) {
        if (ph.kind == 0) rep->t_matvec += ms * 1e-3;
        else if (ph.kind == 1) rep->t_precond += ms * 1e-3;
        else rep->t_orth += ms * 1e-3;
      }
    }
    cudaGetLastError();
  }
  cleanup(false);
  tr.mark("cleanup");
  rep->t_total = std::chrono::duration<double>(clk::now() - t_start).count();
#undef G_ALLOC
#undef G_TRY
#undef G_CUDA
  return TOEP_OK;
}

}  // namespace
}  // namespace toep

extern "C" int toep_gmres(const toep_gmres_problem_t* prob, const toep_gmres_cfg_t* cfg, const void* b, void* x,
                          void* stream, toep_gmres_report_t* rep) {
  TOEP_NVTX("toep_gmres");
  TOEP_REQUIRE(prob != nullptr && cfg != nullptr && b != nullptr && x != nullptr && rep != nullptr, TOEP_ERR_ARG,
               "null argument");
  return toep::gmres_run(prob, cfg, static_cast<const double2*>(b), static_cast<double2*>(x),
                         static_cast<cudaStream_t>(stream), rep);
}
