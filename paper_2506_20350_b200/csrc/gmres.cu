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
// (CGS2): two passes of (V^H w, w -= V h), each a single coalesced sweep of the
// resident basis instead of the reference's j sequential vdot/axpy pairs
// (gmres.py:155-159); CGS2 keeps the basis orthogonal to working precision
// like MGS does, so the Hessenberg entries agree to rounding.
//
// Host/device split: every scalar (Hessenberg column, rotations, g, the
// residual history, the stop flags) lives on the device.  The host only
// launches; after launching step j it waits for step j-1 and reads the stop
// flag from mapped pinned memory, so the launch queue stays one step ahead
// and no step waits on a host round trip.  Steps launched past a stop are
// no-ops (every step kernel checks the device stop flag).
#include <chrono>
#include <cstdlib>
#include <vector>

#include "launch.cuh"
#include "op.h"

namespace toep {
namespace {

constexpr int kThreads = 256;
constexpr int kLG = 8;  // basis vectors per accumulation group

struct GState {
  int stop;       // no further Arnoldi steps in this cycle
  int converged;
  int breakdown;
  int m;          // completed steps in the current cycle
  int total;      // completed steps overall
  int nhist;
  double beta0, beta, hnext, inv;
};

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

// partial[l * nblk + cta] = sum_{i in cta} conj(V[l][i]) w[i]   for l < m
__global__ void __launch_bounds__(kThreads)
dots_partial_kernel(const double2* __restrict__ V, int64_t ld, int m, const double2* __restrict__ w, int64_t N,
                    double2* __restrict__ partial, const int* stop) {
  pdl_wait();
  pdl_trigger();
  if (stop != nullptr && *stop) return;
  __shared__ double2 red[kThreads / 32][kLG];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nblk = gridDim.x;
  for (int l0 = 0; l0 < m; l0 += kLG) {
    double2 acc[kLG];
#pragma unroll
    for (int g = 0; g < kLG; ++g) acc[g] = make_double2(0, 0);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; i < N;
         i += static_cast<int64_t>(nblk) * kThreads) {
      const double2 wi = w[i];
#pragma unroll
      for (int g = 0; g < kLG; ++g)
        if (l0 + g < m) cfmac(acc[g], V[(l0 + g) * ld + i], wi);
    }
#pragma unroll
    for (int g = 0; g < kLG; ++g) {
      const double2 s = warp_sum(acc[g]);
      if (lane == 0) red[warp][g] = s;
    }
    __syncthreads();
    if (threadIdx.x < kLG && l0 + threadIdx.x < m) {
      double2 s = red[0][threadIdx.x];
      for (int ww = 1; ww < kThreads / 32; ++ww) s = cadd(s, red[ww][threadIdx.x]);
      partial[(l0 + threadIdx.x) * nblk + blockIdx.x] = s;
    }
    __syncthreads();
  }
}

// h[l] = sum_b partial[l*nblk + b]; pass 2 also writes hcol[l] = h1[l] + h[l]
__global__ void __launch_bounds__(kThreads)
dots_final_kernel(const double2* __restrict__ partial, int nblk, double2* __restrict__ h,
                  const double2* __restrict__ h1, double2* __restrict__ hcol, const int* stop) {
  pdl_wait();
  pdl_trigger();
  if (stop != nullptr && *stop) return;
  __shared__ double2 red[kThreads / 32];
  const int l = blockIdx.x;
  double2 s = make_double2(0, 0);
  for (int b = threadIdx.x; b < nblk; b += kThreads) s = cadd(s, partial[l * nblk + b]);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 t = red[0];
    for (int ww = 1; ww < kThreads / 32; ++ww) t = cadd(t, red[ww]);
    h[l] = t;
    if (hcol != nullptr) hcol[l] = cadd(h1[l], t);
  }
}

// w[i] -= sum_l V[l][i] h[l]  (l < m, m = min(m_max, *m_dev) when m_dev != null)
// optionally norm2 partials of the result.  neg_h: use -h (x += V y with h = y).
__global__ void __launch_bounds__(kThreads)
update_kernel(const double2* __restrict__ V, int64_t ld, int m_max, const int* m_dev, const double2* __restrict__ h,
              bool neg_h, double2* __restrict__ w, int64_t N, double* __restrict__ norm_partial, const int* stop) {
  pdl_wait();
  pdl_trigger();
  if (stop != nullptr && *stop) return;
  extern __shared__ double2 hs[];
  __shared__ double red[kThreads / 32];
  const int m = (m_dev != nullptr) ? min(m_max, *m_dev) : m_max;
  for (int l = threadIdx.x; l < m; l += kThreads) hs[l] = neg_h ? make_double2(-h[l].x, -h[l].y) : h[l];
  __syncthreads();
  double nrm = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; i < N;
       i += static_cast<int64_t>(gridDim.x) * kThreads) {
    double2 acc = w[i];
    int l = 0;
    for (; l + 3 < m; l += 4) {
      const double2 v0 = V[l * ld + i], v1 = V[(l + 1) * ld + i], v2 = V[(l + 2) * ld + i], v3 = V[(l + 3) * ld + i];
      cfma(acc, v0, make_double2(-hs[l].x, -hs[l].y));
      cfma(acc, v1, make_double2(-hs[l + 1].x, -hs[l + 1].y));
      cfma(acc, v2, make_double2(-hs[l + 2].x, -hs[l + 2].y));
      cfma(acc, v3, make_double2(-hs[l + 3].x, -hs[l + 3].y));
    }
    for (; l < m; ++l) cfma(acc, V[l * ld + i], make_double2(-hs[l].x, -hs[l].y));
    w[i] = acc;
    nrm = fma(acc.x, acc.x, fma(acc.y, acc.y, nrm));
  }
  if (norm_partial != nullptr) {
    nrm = warp_sum(nrm);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = red[0];
      for (int ww = 1; ww < kThreads / 32; ++ww) t += red[ww];
      norm_partial[blockIdx.x] = t;
    }
  }
}

__global__ void __launch_bounds__(kThreads)
norm2_partial_kernel(const double2* __restrict__ x, int64_t N, double* __restrict__ partial) {
  pdl_wait();
  pdl_trigger();
  __shared__ double red[kThreads / 32];
  double nrm = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; i < N;
       i += static_cast<int64_t>(gridDim.x) * kThreads) {
    const double2 v = x[i];
    nrm = fma(v.x, v.x, fma(v.y, v.y, nrm));
  }
  nrm = warp_sum(nrm);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = red[0];
    for (int ww = 1; ww < kThreads / 32; ++ww) t += red[ww];
    partial[blockIdx.x] = t;
  }
}

__device__ double sum_partials_warp(const double* p, int n) {
  double s = 0.0;
  for (int b = threadIdx.x; b < n; b += 32) s += p[b];
  return warp_sum(s);
}

// out = a - b   (elementwise)
__global__ void sub_kernel(const double2* __restrict__ a, const double2* __restrict__ b, double2* __restrict__ out,
                           int64_t N) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = csub(a[i], b[i]);
}

// out = x * (*scal)  unless *stop
__global__ void scale_kernel(const double2* __restrict__ x, double2* __restrict__ out, const double* scal, int64_t N,
                             const int* stop) {
  pdl_wait();
  pdl_trigger();
  if (stop != nullptr && *stop) return;
  const double s = *scal;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = cscale(x[i], s);
}

// beta0 = ||pb||; history[0]
__global__ void init_kernel(GState* st, const double* partial, int nblk, double* hist) {
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

// cycle start (gmres.py:130-144): beta = ||z||, convergence test, g[0] = beta, inv = 1/beta
__global__ void cycle_start_kernel(GState* st, const double* partial, int nblk, double tol, double2* g,
                                   HostFlags* hf) {
  pdl_wait();
  pdl_trigger();
  const double s = sum_partials_warp(partial, nblk);
  if (threadIdx.x == 0) {
    const double beta = sqrt(s);
    st->beta = beta;
    st->m = 0;
    if (beta / st->beta0 <= tol) {
      st->converged = 1;
      st->stop = 1;
    } else {
      st->stop = 0;
      g[0] = make_double2(beta, 0.0);
      st->inv = 1.0 / beta;
    }
    hf->stop = st->stop;
    hf->converged = st->converged;
    hf->total = st->total;
  }
}

// one Givens step on column j = st->m (gmres.py:160-189)
__global__ void givens_kernel(GState* st, const double* norm_partial, int nblk, double2* rcols, int ldr, double* cs,
                              double2* sn, double2* g, double* hist, double tol, int max_total, int cycle_len,
                              HostFlags* hf) {
  pdl_wait();
  pdl_trigger();
  if (st->stop) return;
  const double hn2 = sum_partials_warp(norm_partial, nblk);
  if (threadIdx.x != 0) return;
  const int j = st->m;
  const double hnext = sqrt(hn2);
  double2* hcol = rcols + static_cast<int64_t>(j) * ldr;  // hcol[0..j] written by dots_final pass 2
  for (int i = 0; i < j; ++i) {
    const double2 a0 = hcol[i], a1 = hcol[i + 1];
    const double c = cs[i];
    const double2 s = sn[i];
    const double2 t0 = cadd(cscale(a0, c), cmul(s, a1));
    const double2 t1 = cadd(cscale(cmulc(s, a0), -1.0), cscale(a1, c));
    hcol[i] = t0;
    hcol[i + 1] = t1;
  }
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
  hcol[j] = r;
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
    st->inv = 1.0 / hnext;
    if (st->m >= cycle_len || st->total >= max_total) st->stop = 2;  // cycle exhausted, basis not needed
  }
  hf->stop = st->stop;
  hf->total = st->total;
  hf->converged = st->converged;
  hf->breakdown = st->breakdown;
}

// y = R^-1 g (gmres.py:193-204), R upper triangular from the rotated columns
__global__ void backsub_kernel(const GState* st, const double2* rcols, int ldr, const double2* g, double2* y) {
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
    // acc / d
    const double den = d.x * d.x + d.y * d.y;
    y[i] = make_double2((acc.x * d.x + acc.y * d.y) / den, (acc.y * d.x - acc.x * d.y) / den);
  }
}

// Per-thread host resources reused across solves: the mapped pinned flag word
// the device writes and a pool of CUDA events (creating / freeing these per
// solve cost milliseconds of host time).
struct HostRes {
  HostFlags* hf = nullptr;
  HostFlags* hf_dev = nullptr;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
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

struct Engine {
  const toep_gmres_problem_t* p;
  cudaStream_t s;
  int64_t N;
  int nblk;
  double* norm_partial = nullptr;
  double2* dot_partial = nullptr;

  int apply_a(const void* x, void* y, const int* stop) {
    if (p->op != nullptr) {
      const bool io = p->op->dtype == TOEP_C64;
      return matvec_impl(p->op, x, y, p->w, false, io, stop, s);
    }
    const int rc = p->apply(p->apply_ctx, x, y, p->w, s);
    TOEP_REQUIRE(rc == 0, TOEP_ERR_ARG, "operator callback failed (%d)", rc);
    return TOEP_OK;
  }
  // z = P^-1 x for the per-step preconditioner (BLOCK / CALLBACK); NONE/FOLDED: no-op
  int apply_p(const void* x, void* z, bool* applied, const int* stop) {
    *applied = false;
    if (p->precond == TOEP_PC_BLOCK) {
      *applied = true;
      return block_apply_impl(p->pinv, p->pside, x, z, p->n / p->pside, p->w, TOEP_C128, s, stop);
    }
    if (p->precond == TOEP_PC_CALLBACK) {
      *applied = true;
      const int rc = p->papply(p->papply_ctx, x, z, p->w, s);
      TOEP_REQUIRE(rc == 0, TOEP_ERR_ARG, "preconditioner callback failed (%d)", rc);
    }
    return TOEP_OK;
  }
  int norm2_partials(const void* x) {
    TOEP_TRY(launch_k(norm2_partial_kernel, dim3(nblk), dim3(kThreads), 0, s, static_cast<const double2*>(x), N,
                      norm_partial));
    TOEP_LAUNCHED();
    return TOEP_OK;
  }
  double host_norm(const void* x) {
    std::vector<double> h(nblk);
    if (norm2_partials(x) != TOEP_OK) return -1.0;
    cudaMemcpyAsync(h.data(), norm_partial, nblk * sizeof(double), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double t = 0.0;
    for (double v : h) t += v;
    return std::sqrt(t);
  }
};

// TOEP_TRACE=1: host-side timeline of a solve on stderr (launch / wait split)
struct Trace {
  using clk = std::chrono::steady_clock;
  bool on = std::getenv("TOEP_TRACE") != nullptr;
  clk::time_point t0 = clk::now(), last = t0;
  double wait = 0.0;
  void mark(const char* what) {
    if (!on) return;
    const auto now = clk::now();
    std::fprintf(stderr, "[toep_gmres] %-28s +%9.3f ms (t=%9.3f ms, waited %8.3f ms)\n", what,
                 std::chrono::duration<double, std::milli>(now - last).count(),
                 std::chrono::duration<double, std::milli>(now - t0).count(), wait);
    last = now;
  }
  void sync_event(cudaEvent_t ev) {
    const auto a = clk::now();
    cudaEventSynchronize(ev);
    wait += std::chrono::duration<double, std::milli>(clk::now() - a).count();
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
  if (p->op != nullptr) TOEP_REQUIRE(op_dim(p->op) == p->n, TOEP_ERR_SHAPE, "rhs rows %lld != operator dim %lld",
                                     (long long)p->n, (long long)op_dim(p->op));
  if (p->precond == TOEP_PC_BLOCK || p->precond == TOEP_PC_FOLDED)
    TOEP_REQUIRE(p->pinv != nullptr && p->pside >= 1 && (p->n % p->pside) == 0, TOEP_ERR_SHAPE,
                 "preconditioner side does not divide n");
  if (p->precond == TOEP_PC_FOLDED) TOEP_REQUIRE(p->pmat != nullptr && p->op != nullptr, TOEP_ERR_ARG,
                                                 "folded preconditioner needs op and pmat");

  Engine e{p, s, p->n * p->w, 0};
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  e.nblk = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((e.N + kThreads - 1) / kThreads, 2 * sms)));
  const int64_t N = e.N;
  const int64_t max_total = std::min<int64_t>(cfg->max_iter, N);
  const int cycle_len = static_cast<int>(cfg->restart == 0 ? max_total : std::min<int64_t>(cfg->restart, max_total));
  const int ldr = cycle_len + 1;
  const int nblk = e.nblk;

  // device allocations (stream ordered)
  double2 *V = nullptr, *w = nullptr, *tmp = nullptr, *pb = nullptr, *dots1 = nullptr, *dots2 = nullptr;
  double2 *rcols = nullptr, *sn = nullptr, *g = nullptr, *y = nullptr;
  double *cs = nullptr, *hist = nullptr;
  GState* st = nullptr;
  HostRes& res = host_res();
  res.used = 0;
  HostFlags* hf = res.hf;
  HostFlags* hf_dev = res.hf_dev;
  int rc = TOEP_OK;
  auto cleanup = [&]() {
    for (void* q : {(void*)V, (void*)w, (void*)tmp, (void*)pb, (void*)dots1, (void*)dots2, (void*)rcols, (void*)sn,
                    (void*)g, (void*)y, (void*)cs, (void*)hist, (void*)st, (void*)e.norm_partial,
                    (void*)e.dot_partial})
      if (q) cudaFreeAsync(q, s);
    cudaStreamSynchronize(s);
    res.used = 0;
  };
  TOEP_REQUIRE(hf != nullptr, TOEP_ERR_OOM, "pinned allocation failed");
#define G_ALLOC(ptr, count)                                                                   \
  do {                                                                                        \
    if (cudaMallocAsync(reinterpret_cast<void**>(&(ptr)), sizeof(*(ptr)) * (size_t)(count), s) != cudaSuccess) { \
      cudaGetLastError();                                                                     \
      set_error("out of device memory in gmres");                                             \
      cleanup();                                                                              \
      return TOEP_ERR_OOM;                                                                    \
    }                                                                                         \
  } while (0)
#define G_TRY(expr)          \
  do {                       \
    rc = (expr);             \
    if (rc != TOEP_OK) {     \
      cleanup();             \
      return rc;             \
    }                        \
  } while (0)
  G_ALLOC(V, (int64_t)(cycle_len + 1) * N);
  G_ALLOC(w, N);
  G_ALLOC(tmp, N);
  G_ALLOC(pb, N);
  G_ALLOC(dots1, ldr);
  G_ALLOC(dots2, ldr);
  G_ALLOC(rcols, (int64_t)cycle_len * ldr);
  G_ALLOC(sn, cycle_len + 1);
  G_ALLOC(g, cycle_len + 2);
  G_ALLOC(y, cycle_len + 1);
  G_ALLOC(cs, cycle_len + 1);
  G_ALLOC(hist, max_total + 2);
  G_ALLOC(st, 1);
  G_ALLOC(e.norm_partial, nblk);
  G_ALLOC(e.dot_partial, (int64_t)nblk * ldr);
  hf->stop = 0;
  hf->total = 0;
  hf->converged = 0;
  hf->breakdown = 0;
  tr.mark("allocations");

  const bool timed = cfg->timings != 0;
  auto new_event = [&](cudaEvent_t* ev) { *ev = res.event(); };
  struct Phase { cudaEvent_t a, b; int kind; };
  std::vector<Phase> phases;
  auto mark = [&](int kind, cudaEvent_t a) {
    cudaEvent_t bb;
    new_event(&bb);
    cudaEventRecord(bb, s);
    phases.push_back({a, bb, kind});
    return bb;
  };
  auto start_mark = [&]() {
    cudaEvent_t a;
    new_event(&a);
    cudaEventRecord(a, s);
    return a;
  };

  const int grid1 = std::min<int64_t>((N + kThreads - 1) / kThreads, 4 * sms);
  const size_t upd_smem = sizeof(double2) * ldr;
  if (upd_smem > 48 * 1024)
    cudaFuncSetAttribute(update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_smem);

  // ---- P^-1 b, beta0 (gmres.py:104-113)
  const double2* zb = b;
  {
    cudaEvent_t t0 = timed ? start_mark() : nullptr;
    if (p->precond == TOEP_PC_BLOCK || p->precond == TOEP_PC_FOLDED) {
      G_TRY(block_apply_impl(p->pinv, p->pside, b, pb, p->n / p->pside, p->w, TOEP_C128, s, nullptr));
      zb = pb;
    } else if (p->precond == TOEP_PC_CALLBACK) {
      if (p->papply(p->papply_ctx, b, pb, p->w, s) != 0) {
        set_error("preconditioner callback failed");
        cleanup();
        return TOEP_ERR_ARG;
      }
      zb = pb;
    }
    if (timed) mark(1, t0);
  }
  G_TRY(e.norm2_partials(zb));
  G_TRY(launch_k(init_kernel, dim3(1), dim3(32), 0, s, st, e.norm_partial, nblk, hist));
  GState hst{};
  if (cudaMemcpyAsync(&hst, st, sizeof(GState), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess) {
    set_error("gmres init failed: %s", cudaGetErrorString(cudaGetLastError()));
    cleanup();
    return TOEP_ERR_CUDA;
  }
  tr.mark("init (P^-1 b, beta0) synced");
  rep->iterations = 0;
  rep->converged = 1;
  rep->breakdown = 0;
  rep->t_matvec = rep->t_precond = rep->t_orth = 0.0;
  if (hst.beta0 == 0.0) {
    cudaMemsetAsync(x, 0, N * sizeof(double2), s);
    cudaStreamSynchronize(s);
    if (rep->history != nullptr && rep->history_cap >= 1) rep->history[0] = 0.0;
    rep->n_history = 1;
    rep->final_residual = 0.0;
    cleanup();
    rep->t_total = std::chrono::duration<double>(clk::now() - t_start).count();
    return TOEP_OK;
  }
  cudaMemsetAsync(x, 0, N * sizeof(double2), s);

  int* stop_dev = &st->stop;
  int* m_dev = &st->m;
  int total = 0;
  bool first = true;
  std::vector<cudaEvent_t> step_ev;
  while (true) {
    // ---- cycle start (gmres.py:123-144)
    const double2* z = zb;
    if (!first) {
      cudaEvent_t t0 = timed ? start_mark() : nullptr;
      G_TRY(e.apply_a(x, tmp, nullptr));
      if (timed) t0 = mark(0, t0);
      if (p->precond == TOEP_PC_FOLDED) {
        G_TRY(launch_k(sub_kernel, dim3(grid1), dim3(kThreads), 0, s, pb, tmp, w, N));  // P^-1 b - (P^-1 A) x
      } else {
        G_TRY(launch_k(sub_kernel, dim3(grid1), dim3(kThreads), 0, s, b, tmp, w, N));
        bool applied = false;
        G_TRY(e.apply_p(w, tmp, &applied, nullptr));
        if (applied) cudaMemcpyAsync(w, tmp, N * sizeof(double2), cudaMemcpyDeviceToDevice, s);
      }
      if (timed) mark(1, t0);
      z = w;
    }
    first = false;
    G_TRY(e.norm2_partials(z));
    G_TRY(launch_k(cycle_start_kernel, dim3(1), dim3(32), 0, s, st, e.norm_partial, nblk, cfg->tol, g, hf_dev));
    G_TRY(launch_k(scale_kernel, dim3(grid1), dim3(kThreads), 0, s, z, V, &st->inv, N, stop_dev));
    TOEP_LAUNCHED();

    // ---- Arnoldi steps (gmres.py:146-190)
    int j = 0;
    step_ev.clear();
    while (j < cycle_len && total + j < max_total) {
      const double2* vj = V + static_cast<int64_t>(j) * N;
      cudaEvent_t t0 = timed ? start_mark() : nullptr;
      G_TRY(e.apply_a(vj, w, stop_dev));
      if (timed) t0 = mark(0, t0);
      bool applied = false;
      G_TRY(e.apply_p(w, tmp, &applied, stop_dev));
      double2* wv = applied ? tmp : w;
      if (timed) t0 = mark(1, t0);
      const int m = j + 1;
      // CGS2 pass 1
      G_TRY(launch_k(dots_partial_kernel, dim3(nblk), dim3(kThreads), 0, s, V, N, m, wv, N, e.dot_partial, stop_dev));
      G_TRY(launch_k(dots_final_kernel, dim3(m), dim3(kThreads), 0, s, e.dot_partial, nblk, dots1, nullptr, nullptr, stop_dev));
      G_TRY(launch_k(update_kernel, dim3(grid1), dim3(kThreads), upd_smem, s, V, N, m, nullptr, dots1, false, wv, N, nullptr, stop_dev));
      // CGS2 pass 2 (re-orthogonalisation), Hessenberg column = h1 + h2
      G_TRY(launch_k(dots_partial_kernel, dim3(nblk), dim3(kThreads), 0, s, V, N, m, wv, N, e.dot_partial, stop_dev));
      G_TRY(launch_k(dots_final_kernel, dim3(m), dim3(kThreads), 0, s, e.dot_partial, nblk, dots2, dots1, rcols + (int64_t)j * ldr, stop_dev));
      G_TRY(launch_k(update_kernel, dim3(nblk), dim3(kThreads), upd_smem, s, V, N, m, nullptr, dots2, false, wv, N, e.norm_partial, stop_dev));
      G_TRY(launch_k(givens_kernel, dim3(1), dim3(32), 0, s, st, e.norm_partial, nblk, rcols, ldr, cs, sn, g, hist, cfg->tol,
                                     static_cast<int>(max_total), cycle_len, hf_dev));
      G_TRY(launch_k(scale_kernel, dim3(grid1), dim3(kThreads), 0, s, wv, V + static_cast<int64_t>(j + 1) * N, &st->inv, N, stop_dev));
      TOEP_LAUNCHED();
      if (timed) mark(2, t0);
      cudaEvent_t ev = res.event();
      cudaEventRecord(ev, s);
      step_ev.push_back(ev);
      ++j;
      if (j >= 2) {
        tr.sync_event(step_ev[j - 2]);
        if (hf->stop) break;
      }
    }
    tr.mark("arnoldi steps launched");
    // ---- assemble x += V y (gmres.py:192-204)
    G_TRY(launch_k(backsub_kernel, dim3(1), dim3(32), 0, s, st, rcols, ldr, g, y));
    G_TRY(launch_k(update_kernel, dim3(grid1), dim3(kThreads), upd_smem, s, V, N, cycle_len, m_dev, y, true, x, N, nullptr, nullptr));
    TOEP_LAUNCHED();
    if (cudaMemcpyAsync(&hst, st, sizeof(GState), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
      set_error("gmres cycle failed: %s", cudaGetErrorString(cudaGetLastError()));
      cleanup();
      return TOEP_ERR_CUDA;
    }
    total = hst.total;
    tr.mark("cycle synced");
    if (hst.converged || hst.breakdown || total >= max_total) break;
  }
  // ---- exit residual ||b - A x|| / ||b|| (gmres.py:209-216), unpreconditioned
  {
    cudaEvent_t t0 = timed ? start_mark() : nullptr;
    G_TRY(e.apply_a(x, tmp, nullptr));
    if (p->precond == TOEP_PC_FOLDED) {  // A x = P (P^-1 A x)
      G_TRY(block_apply_impl(p->pmat, p->pside, tmp, w, p->n / p->pside, p->w, TOEP_C128, s, nullptr));
      cudaMemcpyAsync(tmp, w, N * sizeof(double2), cudaMemcpyDeviceToDevice, s);
    }
    if (timed) mark(0, t0);
    G_TRY(launch_k(sub_kernel, dim3(grid1), dim3(kThreads), 0, s, b, tmp, w, N));
  }
  const double rn = e.host_norm(w);
  const double bn = e.host_norm(b);
  tr.mark("exit residual synced");
  rep->final_residual = rn / bn;
  rep->iterations = hst.total;
  rep->converged = hst.converged;
  rep->breakdown = hst.breakdown;
  const int nh = std::min(hst.nhist, rep->history_cap);
  if (rep->history != nullptr && nh > 0)
    cudaMemcpyAsync(rep->history, hist, nh * sizeof(double), cudaMemcpyDeviceToHost, s);
  rep->n_history = hst.nhist;
  if (cudaStreamSynchronize(s) != cudaSuccess) {
    set_error("gmres exit failed: %s", cudaGetErrorString(cudaGetLastError()));
    cleanup();
    return TOEP_ERR_CUDA;
  }
  if (timed) {
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
  cleanup();
  tr.mark("cleanup");
  rep->t_total = std::chrono::duration<double>(clk::now() - t_start).count();
#undef G_ALLOC
#undef G_TRY
  return TOEP_OK;
}

}  // namespace
}  // namespace toep

extern "C" int toep_gmres(const toep_gmres_problem_t* prob, const toep_gmres_cfg_t* cfg, const void* b, void* x,
                          void* stream, toep_gmres_report_t* rep) {
  TOEP_REQUIRE(prob != nullptr && cfg != nullptr && b != nullptr && x != nullptr && rep != nullptr, TOEP_ERR_ARG,
               "null argument");
  return toep::gmres_run(prob, cfg, static_cast<const double2*>(b), static_cast<double2*>(x),
                         static_cast<cudaStream_t>(stream), rep);
}
