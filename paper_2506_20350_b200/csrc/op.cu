// Resident spectral operator: precompute (toeplitz.py:248-253), matvec
// (toeplitz.py:287-324), block preconditioner apply (precond.py:65-71) and the
// C-ABI entry points for them.
#include <cstdarg>
#include <cstring>
#include <new>

#include "op.h"

namespace toep {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
const char* last_error() { return g_err; }

cudaError_t ensure_smem_attr(const void* func, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  int dev = 0;
  cudaGetDevice(&dev);
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{dev, func}];
  if (have >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (e == cudaSuccess) have = bytes;
  return e;
}

size_t elt_size(int dtype) { return dtype == TOEP_C64 ? sizeof(float2) : sizeof(double2); }
int64_t op_dim(const toep_op_s* op) { return static_cast<int64_t>(op->n2) * op->n1 * op->n0; }

static int smooth7_at_least(int m) {
  for (int L = m;; ++L) {
    int r = L;
    for (int p : {2, 3, 5, 7})
      while (r % p == 0) r /= p;
    if (r == 1) return L;
  }
}

// Keep memory freed with cudaFreeAsync in the device pool: with the default
// release threshold (0) every stream synchronisation returns it to the driver
// and the next solve pays cudaMalloc again (milliseconds).
void keep_pool() {
  static thread_local int done_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (done_dev == dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  done_dev = dev;
}

// Register `s` as a stream with work reading the operator (toep_op_destroy synchronises it)
void note_stream(toep_op_s* op, cudaStream_t s) {
  std::lock_guard<std::mutex> lock(op->mu);
  op->ws[s];
}

int op_workspace(toep_op_s* op, int64_t w, cudaStream_t s, toep_op_s::Workspace** out, bool need_hat) {
  keep_pool();
  std::lock_guard<std::mutex> lock(op->mu);
  auto& ws = op->ws[s];
  const size_t es = elt_size(op->dtype);
  if (ws.w_cap < w) {
    if (ws.x1) TOEP_CUDA(cudaFreeAsync(ws.x1, s));
    ws.x1 = nullptr;
    ws.w_cap = 0;
    const size_t nx1 = static_cast<size_t>(op->n2) * op->l1 * op->n0 * w * es;
    if (cudaMallocAsync(&ws.x1, nx1, s) != cudaSuccess) {
      cudaGetLastError();
      set_error("out of device memory for matvec workspace (w=%lld)", static_cast<long long>(w));
      return TOEP_ERR_OOM;
    }
    ws.w_cap = w;
  }
  if (need_hat && ws.hat_cap < w) {  // complex spectral buffers (not used by the 3M multi-RHS path)
    if (ws.hat) TOEP_CUDA(cudaFreeAsync(ws.hat, s));
    if (ws.hat2) TOEP_CUDA(cudaFreeAsync(ws.hat2, s));
    ws.hat = ws.hat2 = nullptr;
    ws.hat_cap = 0;
    const size_t nhat = static_cast<size_t>(op->K) * op->n0 * w * es;
    if (cudaMallocAsync(&ws.hat, nhat, s) != cudaSuccess || cudaMallocAsync(&ws.hat2, nhat, s) != cudaSuccess) {
      cudaGetLastError();
      set_error("out of device memory for matvec workspace (w=%lld)", static_cast<long long>(w));
      return TOEP_ERR_OOM;
    }
    ws.hat_cap = w;
  }
  *out = &ws;
  return TOEP_OK;
}

// DT (bins ky-major, k = ky*l1 + kx) -> three planes with bins kx-major (kx*l2 + ky), so the bins
// of a kx-chunk are contiguous
__global__ void k_split_planes(const double2* __restrict__ src, int64_t count, int l2, int l1, int64_t bsz,
                               double* __restrict__ dst) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k = i / bsz, e = i - k * bsz;
    const int64_t ky = k / l1, kx = k - ky * l1;
    const int64_t o = (kx * l2 + ky) * bsz + e;
    const double2 v = src[i];
    dst[o] = v.x;
    dst[count + o] = v.y;
    dst[2 * count + o] = v.x + v.y;
  }
}

// kx columns per chunk of the 3M multi-RHS path: planes of one chunk stay under ~4 GB per buffer
int mrhs_chunk(const toep_op_s* op, int64_t w) {
  const int64_t per_kx = static_cast<int64_t>(op->l2) * op->n0 * w * 3 * static_cast<int64_t>(sizeof(double));
  const int64_t budget = int64_t{4} << 30;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(op->l1, budget / std::max<int64_t>(per_kx, 1))));
}

// Multi-RHS per-bin products as 3M (Gauss): V = D U with three real FP64 tensor-core GEMMs on split
// planes, T1 = Dr Ur, T2 = Di Ui, T3 = (Dr + Di)(Ur + Ui); the level-2 DFT passes write / read the
// planes directly, so the split and the recombination cost no extra pass.  Enabled for c128,
// W >= 16 and a compiled level-2 plan.
bool mrhs_3m(const toep_op_s* op, int64_t w, bool transpose) {
  return !transpose && w >= 16 && op->dtype == TOEP_C128 && op->slab_kxs == 0 &&
         fft_plan_has_planes(op->l2, static_cast<int64_t>(op->n0) * w);
}

// Ozaki scheme for the multi-RHS per-bin products (ozaki.cu: int8 tensor cores, FP64-accurate);
// TOEP_MRHS_OZAKI=0 keeps the 3M DMMA GEMMs
bool mrhs_ozaki(const toep_op_s* op) {
  static const bool on = [] {
    const char* e = std::getenv("TOEP_MRHS_OZAKI");
    return !(e != nullptr && e[0] == '0');
  }();
  return on && ozaki_supported(op->n0);
}

// Publish a lazily built operator-wide buffer: record an event on the building stream (op->mu held)
static int mark_lazy_build(toep_op_s* op, cudaStream_t s) {
  if (op->lazy_ev == nullptr) TOEP_CUDA(cudaEventCreateWithFlags(&op->lazy_ev, cudaEventDisableTiming));
  TOEP_CUDA(cudaEventRecord(op->lazy_ev, s));
  op->lazy_stream = s;
  return TOEP_OK;
}

// A stream other than the one that built the lazy buffers waits for that build (op->mu held)
static int order_after_lazy_build(toep_op_s* op, cudaStream_t s) {
  if (op->lazy_ev != nullptr && op->lazy_stream != s) TOEP_CUDA(cudaStreamWaitEvent(s, op->lazy_ev, 0));
  return TOEP_OK;
}

// (Re)size a per-stream device buffer to at least `need` bytes; capacity tracked in bytes because
// the per-call size depends on w through the chunking (mrhs_chunk), not monotonically
template <typename T>
static int ensure_bytes(T** buf, size_t* cap, size_t need, cudaStream_t s, const char* what) {
  if (*cap >= need && *buf != nullptr) return TOEP_OK;
  if (*buf) TOEP_CUDA(cudaFreeAsync(*buf, s));
  *buf = nullptr;
  *cap = 0;
  if (cudaMallocAsync(reinterpret_cast<void**>(buf), need, s) != cudaSuccess) {
    cudaGetLastError();
    *buf = nullptr;
    set_error("out of device memory for %s (%zu bytes)", what, need);
    return TOEP_ERR_OOM;
  }
  *cap = need;
  return TOEP_OK;
}

int ensure_ozaki(toep_op_s* op, toep_op_s::Workspace* ws, int64_t w, int kc, cudaStream_t s) {
  std::lock_guard<std::mutex> lock(op->mu);
  if (op->oz_a == nullptr) {
    const int64_t abytes = ozaki_a_bytes(op->n0, op->K);
    if (cudaMallocAsync(reinterpret_cast<void**>(&op->oz_a), abytes, s) != cudaSuccess ||
        cudaMallocAsync(reinterpret_cast<void**>(&op->oz_aexp), op->K * 2 * op->n0 * sizeof(int32_t), s) !=
            cudaSuccess) {
      cudaGetLastError();
      if (op->oz_a) cudaFreeAsync(op->oz_a, s);
      op->oz_a = nullptr;
      op->oz_aexp = nullptr;
      set_error("out of device memory for the operator's int8 slices");
      return TOEP_ERR_OOM;
    }
    TOEP_TRY(ozaki_slice_a(op->DT, op->n0, op->l2, op->l1, op->oz_a, op->oz_aexp, s));
    TOEP_TRY(mark_lazy_build(op, s));
  } else {
    TOEP_TRY(order_after_lazy_build(op, s));
  }
  const int64_t bins = static_cast<int64_t>(kc) * op->l2;
  TOEP_TRY(ensure_bytes(&ws->oz_b, &ws->oz_b_bytes, static_cast<size_t>(ozaki_b_bytes(op->n0, bins, w)), s,
                        "the int8 right-hand-side slices"));
  TOEP_TRY(ensure_bytes(&ws->oz_bexp, &ws->oz_bexp_bytes, static_cast<size_t>(ozaki_b_exps(bins, w)) * sizeof(int32_t),
                        s, "the int8 right-hand-side exponents"));
  return TOEP_OK;
}

int ensure_planes(toep_op_s* op, toep_op_s::Workspace* ws, int64_t w, cudaStream_t s, bool need_dtp) {
  std::lock_guard<std::mutex> lock(op->mu);
  const int64_t kn = op->K * op->n0;
  if (need_dtp && op->DTp == nullptr) {
    const int64_t cnt = kn * op->n0;
    if (cudaMallocAsync(reinterpret_cast<void**>(&op->DTp), 3 * cnt * sizeof(double), s) != cudaSuccess) {
      cudaGetLastError();
      op->DTp = nullptr;
      set_error("out of device memory for the 3M operator planes");
      return TOEP_ERR_OOM;
    }
    const int grid = static_cast<int>(std::min<int64_t>((cnt + 255) / 256, 148 * 16));
    k_split_planes<<<grid, 256, 0, s>>>(static_cast<const double2*>(op->DT), cnt, op->l2, op->l1,
                                        static_cast<int64_t>(op->n0) * op->n0, op->DTp);
    TOEP_LAUNCHED();
    TOEP_TRY(mark_lazy_build(op, s));
  } else if (need_dtp) {
    TOEP_TRY(order_after_lazy_build(op, s));
  }
  const size_t bytes = 3 * static_cast<size_t>(op->l2) * mrhs_chunk(op, w) * op->n0 * w * sizeof(double);
  if (ws->p_bytes < bytes || ws->hatp == nullptr || ws->hat2p == nullptr) {
    size_t c1 = 0, c2 = 0;
    if (ws->hatp) TOEP_CUDA(cudaFreeAsync(ws->hatp, s));
    if (ws->hat2p) TOEP_CUDA(cudaFreeAsync(ws->hat2p, s));
    ws->hatp = ws->hat2p = nullptr;
    ws->p_bytes = 0;
    TOEP_TRY(ensure_bytes(&ws->hatp, &c1, bytes, s, "the 3M workspace"));
    TOEP_TRY(ensure_bytes(&ws->hat2p, &c2, bytes, s, "the 3M workspace"));
    ws->p_bytes = bytes;
  }
  return TOEP_OK;
}

int matvec_impl(toep_op_s* op, const void* u, void* v, int64_t w, bool transpose, bool io_c128, const int* stop,
                cudaStream_t s, const double* in_scale) {
  if (w == 0) return TOEP_OK;
  toep_op_s::Workspace* ws = nullptr;
  const bool planar = mrhs_3m(op, w, transpose);
  TOEP_TRY(op_workspace(op, w, s, &ws, !planar));
  const int tc = op->dtype == TOEP_C64 ? 1 : 0;
  const int tio = io_c128 ? 0 : tc;
  const int64_t inner = static_cast<int64_t>(op->n0) * w;
  // forward transform of transpose() is the inverse DFT (toeplitz.py:318) and vice versa
  const int s1 = transpose ? +1 : -1;
  const double sc1y = transpose ? 1.0 / op->l2 : 1.0, sc1x = transpose ? 1.0 / op->l1 : 1.0;
  const double sc2y = transpose ? 1.0 : 1.0 / op->l2, sc2x = transpose ? 1.0 : 1.0 / op->l1;

  // one-CTA-per-column 2-D transforms when a compiled 2-D plan covers the grid
  if (w == 1) {
    const L2Prefetch pf = transpose ? L2Prefetch{} : binprod_prefetch_plan(op->dtype, op->DT, op->K, op->n0);
    if (!transpose && op->dtype == TOEP_C128 && tio == 0 && op->slab_kxs == 0 && op->n0 == 128) {
      // the three stages in one cooperative launch: the operator stream starts under the forward DFT
      {
        std::lock_guard<std::mutex> lock(op->mu);
        if (ws->bar == nullptr) {
          TOEP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws->bar), 2 * sizeof(unsigned), s));
          TOEP_CUDA(cudaMemsetAsync(ws->bar, 0, 2 * sizeof(unsigned), s));
        }
      }
      const int rc = matvec_fused(op->DT, op->K, op->n2, op->n1, op->l2, op->l1, op->n0, u, ws->hat, ws->hat2, v,
                                  ws->bar, in_scale, stop, pf, s);
      if (rc != -1) return rc;
    }
    const int rf =
        fft2d(false, u, ws->hat, op->n2, op->n1, op->l2, op->l1, inner, s1, tio, tc, tc, in_scale, stop, s, &pf);
    if (rf == TOEP_OK) {
      TOEP_TRY(bin_product(op->dtype, op->DT, ws->hat, ws->hat2, op->K, op->n0, w, transpose, stop, s));
      // the overall 1/(l1 l2) is applied by the second kernel (linear, so also right for transpose())
      const L2Prefetch pfi =
          transpose ? L2Prefetch{} : binprod_prefetch_plan(op->dtype, op->DT, op->K, op->n0, 1);
      const int ri =
          fft2d(true, ws->hat2, v, op->n2, op->n1, op->l2, op->l1, inner, -s1, tc, tc, tio, nullptr, stop, s, &pfi);
      return ri == -1 ? TOEP_ERR_ARG : ri;
    } else if (rf != -1) {
      return rf;
    }
  }

  PassArgs a;  // level-1 (x) pass: u [n2][n1][inner] -> x1 [n2][l1][inner]  (pad fused)
  a.in = u; a.out = ws->x1; a.L = op->l1; a.n_lo = op->n1; a.n_hi = 0; a.n_out = op->l1;
  a.inner = inner; a.outer = op->n2; a.in_sa = inner; a.in_so = op->n1 * inner; a.out_sa = inner;
  a.out_so = op->l1 * inner; a.sign = s1; a.scale = sc1x; a.stop = stop; a.in_scale = in_scale;
  TOEP_TRY(fft_pass(a, tio, tc, tc, s));

  if (planar) {
    // 3M in kx-chunks: level-2 DFT of the chunk's columns into split planes (bins kx-major within
    // the chunk), three real batched GEMMs against the operator planes, inverse level-2 DFT
    // recombining (T1 - T2) + i (T3 - T1 - T2) into x1
    const bool oz = mrhs_ozaki(op);
    TOEP_TRY(ensure_planes(op, ws, w, s, !oz));
    const int kc = mrhs_chunk(op, w);
    if (oz) TOEP_TRY(ensure_ozaki(op, ws, w, kc, s));
    const int64_t n0 = op->n0, nw = n0 * w, dn = op->K * n0 * n0;
    const int64_t plane = static_cast<int64_t>(op->l2) * kc * nw;  // doubles per plane (one chunk)
    for (int kx0 = 0; kx0 < op->l1; kx0 += kc) {
      const int cnt = std::min(kc, op->l1 - kx0);
      PassArgs b;  // level 2 over rows y < n2 of columns [kx0, kx0+cnt): out (kx_local, ky, inner)
      b.in = static_cast<const char*>(ws->x1) + kx0 * inner * elt_size(op->dtype);
      b.out = ws->hatp; b.L = op->l2; b.n_lo = op->n2; b.n_hi = 0; b.n_out = op->l2;
      b.inner = inner; b.outer = cnt; b.in_sa = op->l1 * inner; b.in_so = inner; b.out_sa = inner;
      b.out_so = op->l2 * inner; b.sign = s1; b.scale = sc1y; b.stop = stop;
      b.out_planes = ws->hatp; b.plane = plane; b.planes2 = oz;
      TOEP_TRY(fft_pass(b, tc, tc, tc, s));
      const int64_t bins = static_cast<int64_t>(cnt) * op->l2;
      const int64_t bin0 = static_cast<int64_t>(kx0) * op->l2;  // kx-major bin index of the chunk
      if (oz) {
        TOEP_TRY(ozaki_products(op->oz_a + bin0 * ozaki_a_bytes(op->n0, 1), op->oz_aexp + bin0 * 2 * n0, ws->hatp,
                                ws->hatp + plane, op->n0, bins, w, ws->oz_b, ws->oz_bexp, ws->hat2p,
                                ws->hat2p + plane, s));
      } else {
        const int64_t dofs = bin0 * n0 * n0;
        const double* ap[3] = {op->DTp + dofs, op->DTp + dn + dofs, op->DTp + 2 * dn + dofs};
        const double* bp[3] = {ws->hatp, ws->hatp + plane, ws->hatp + 2 * plane};
        double* cp[3] = {ws->hat2p, ws->hat2p + plane, ws->hat2p + 2 * plane};
        TOEP_TRY(dgemm_dmma_planes(n0, w, n0, 1.0, ap, 1, n0, n0 * n0, bp, w, 1, nw, 0.0, cp, w, 1, nw, bins, 3, s,
                                   nullptr));
      }
      PassArgs c;  // inverse level 2, keep rows y < n2 -> x1 columns [kx0, kx0+cnt)
      c.in = ws->hat2p; c.out = static_cast<char*>(ws->x1) + kx0 * inner * elt_size(op->dtype);
      c.L = op->l2; c.n_lo = op->l2; c.n_hi = 0; c.n_out = op->n2;
      c.inner = inner; c.outer = cnt; c.in_sa = inner; c.in_so = op->l2 * inner; c.out_sa = op->l1 * inner;
      c.out_so = inner; c.sign = -s1; c.scale = sc2y; c.stop = stop;
      c.in_planes = ws->hat2p; c.plane = plane; c.planes2 = oz;
      TOEP_TRY(fft_pass(c, tc, tc, tc, s));
    }
  } else {
    PassArgs b;  // level-2 (y) pass over the n2 non-zero rows: x1 -> hat [l2][l1][inner]
    b.in = ws->x1; b.out = ws->hat; b.L = op->l2; b.n_lo = op->n2; b.n_hi = 0; b.n_out = op->l2;
    b.inner = inner; b.outer = op->l1; b.in_sa = op->l1 * inner; b.in_so = inner; b.out_sa = op->l1 * inner;
    b.out_so = inner; b.sign = s1; b.scale = sc1y; b.stop = stop;
    TOEP_TRY(fft_pass(b, tc, tc, tc, s));

    TOEP_TRY(bin_product(op->dtype, op->DT, ws->hat, ws->hat2, op->K, op->n0, w, transpose, stop, s));

    PassArgs c;  // inverse level-2 pass, keep the n2 payload rows: hat2 -> x1 [n2][l1][inner]
    c.in = ws->hat2; c.out = ws->x1; c.L = op->l2; c.n_lo = op->l2; c.n_hi = 0; c.n_out = op->n2;
    c.inner = inner; c.outer = op->l1; c.in_sa = op->l1 * inner; c.in_so = inner; c.out_sa = op->l1 * inner;
    c.out_so = inner; c.sign = -s1; c.scale = sc2y; c.stop = stop;
    TOEP_TRY(fft_pass(c, tc, tc, tc, s));
  }

  PassArgs d;  // inverse level-1 pass + extract_result crop: x1 -> v [n2][n1][inner]
  d.in = ws->x1; d.out = v; d.L = op->l1; d.n_lo = op->l1; d.n_hi = 0; d.n_out = op->n1;
  d.inner = inner; d.outer = op->n2; d.in_sa = inner; d.in_so = op->l1 * inner; d.out_sa = inner;
  d.out_so = op->n1 * inner; d.sign = -s1; d.scale = sc2x; d.stop = stop;
  TOEP_TRY(fft_pass(d, tc, tc, tio, s));
  return TOEP_OK;
}

int block_apply_impl(const void* m, int n0, const void* in, void* out, int64_t segments, int64_t w, int dtype,
                     cudaStream_t s, const int* stop) {
  if (w == 1) {
    // one GEMM: out(:, seg) = M in(:, seg), segments as columns
    return gemm(dtype, n0, segments, n0, make_double2(1, 0), m, n0, 1, 0, in, 1, n0, 0, make_double2(0, 0), out, 1,
                n0, 0, 1, s, stop);
  }
  // batched over segments: (n0 x w) blocks
  int64_t done = 0;
  while (done < segments) {
    const int64_t nb = std::min<int64_t>(segments - done, 65535);
    const size_t es = elt_size(dtype);
    const char* pin = static_cast<const char*>(in) + done * n0 * w * es;
    char* pout = static_cast<char*>(out) + done * n0 * w * es;
    TOEP_TRY(gemm(dtype, n0, w, n0, make_double2(1, 0), m, n0, 1, 0, pin, w, 1, n0 * w, make_double2(0, 0), pout, w,
                  1, n0 * w, nb, s, stop));
    done += nb;
  }
  return TOEP_OK;
}

}  // namespace toep

using namespace toep;

extern "C" {

const char* toep_last_error(void) { return last_error(); }
int toep_version(void) { return 100; }

int toep_op_create(const void* stacked4, int on_device, int n2, int n1, int n0, int l2, int l1, int dtype,
                   void* stream, toep_op_t* out) {
  return toep_op_create_slab(stacked4, on_device, n2, n1, n0, l2, l1, dtype, 0, 0, stream, out);
}

// kx1 <= kx0 (e.g. 0, 0): the full operator; else only the bins of level-1 frequencies [kx0, kx1)
// are transformed and kept (the slab operator of the row / kx-slab decomposition)
int toep_op_create_slab(const void* stacked4, int on_device, int n2, int n1, int n0, int l2, int l1, int dtype,
                        int kx0, int kx1, void* stream, toep_op_t* out) {
  TOEP_NVTX("toep_op_create");
  TOEP_REQUIRE(out != nullptr && stacked4 != nullptr, TOEP_ERR_ARG, "null argument");
  TOEP_REQUIRE(n2 >= 1 && n1 >= 1 && n0 >= 1, TOEP_ERR_SHAPE, "n2, n1, n0 must be positive");
  TOEP_REQUIRE(dtype == TOEP_C128 || dtype == TOEP_C64, TOEP_ERR_ARG, "dtype must be TOEP_C128 or TOEP_C64");
  const int k2 = 2 * n2 - 1, k1 = 2 * n1 - 1;
  if (l2 <= 0) l2 = smooth7_at_least(k2);
  if (l1 <= 0) l1 = smooth7_at_least(k1);
  TOEP_REQUIRE(l2 >= k2 && l1 >= k1, TOEP_ERR_SHAPE, "embedding (%d,%d) shorter than 2n-1 (%d,%d)", l2, l1, k2, k1);
  cudaStream_t s = static_cast<cudaStream_t>(stream);

  const bool slab = kx1 > kx0;
  if (!slab) { kx0 = 0; kx1 = l1; }
  TOEP_REQUIRE(0 <= kx0 && kx1 <= l1, TOEP_ERR_SHAPE, "slab [%d,%d) outside [0,%d)", kx0, kx1, l1);
  const int kxs = kx1 - kx0;
  auto* op = new (std::nothrow) toep_op_s();
  TOEP_REQUIRE(op != nullptr, TOEP_ERR_OOM, "host allocation failed");
  op->n2 = n2; op->n1 = n1; op->n0 = n0; op->l2 = l2; op->l1 = l1; op->dtype = dtype;
  op->K = static_cast<int64_t>(l2) * kxs;
  if (slab) { op->slab_k0 = kx0; op->slab_kxs = kxs; }
  cudaGetDevice(&op->device);

  const int64_t nn = static_cast<int64_t>(n0) * n0;
  const size_t gen_bytes = static_cast<size_t>(k2) * k1 * nn * sizeof(double2);
  const size_t x_bytes = static_cast<size_t>(k2) * l1 * nn * sizeof(double2);
  const size_t d_bytes = static_cast<size_t>(op->K) * nn * sizeof(double2);
  void *gen = nullptr, *x = nullptr, *d = nullptr, *dt = nullptr;
  auto fail = [&](int code) {
    cudaGetLastError();
    if (gen && !on_device) cudaFreeAsync(gen, s);
    if (x) cudaFreeAsync(x, s);
    if (d) cudaFreeAsync(d, s);
    if (dt) cudaFreeAsync(dt, s);
    delete op;
    return code;
  };
#define TOEP_STEP(expr)                 \
  do {                                  \
    int _c = (expr);                    \
    if (_c != TOEP_OK) return fail(_c); \
  } while (0)
#define TOEP_ALLOC(ptr, bytes)                                                                   \
  do {                                                                                           \
    if (cudaMallocAsync(&(ptr), (bytes), s) != cudaSuccess) {                                    \
      set_error("out of device memory in precompute_spectral (%zu bytes)", (size_t)(bytes));    \
      return fail(TOEP_ERR_OOM);                                                                 \
    }                                                                                            \
  } while (0)

  if (on_device) {
    gen = const_cast<void*>(stacked4);
  } else {
    TOEP_ALLOC(gen, gen_bytes);
    const int up = pipelined_h2d(stacked4, gen, gen_bytes, s);
    if (up != TOEP_OK) return fail(up);
  }
  TOEP_ALLOC(x, x_bytes);
  // level-1 DFT of every (offset2) row of the generator, embedded at offset % l1
  PassArgs a;
  a.in = gen; a.out = x; a.L = l1; a.n_lo = n1; a.n_hi = n1 - 1; a.n_out = l1; a.inner = nn; a.outer = k2;
  a.in_sa = nn; a.in_so = k1 * nn; a.out_sa = nn; a.out_so = static_cast<int64_t>(l1) * nn; a.sign = -1;
  TOEP_STEP(fft_pass(a, 0, 0, 0, s));
  if (!on_device) { cudaFreeAsync(gen, s); }
  gen = nullptr;
  TOEP_ALLOC(d, d_bytes);
  PassArgs b;  // level-2 DFT of columns [kx0, kx1), embedded at offset % l2 -> D [l2][kxs][n0][n0]
  b.in = static_cast<const double2*>(x) + static_cast<int64_t>(kx0) * nn; b.out = d; b.L = l2; b.n_lo = n2;
  b.n_hi = n2 - 1; b.n_out = l2; b.inner = nn; b.outer = kxs;
  b.in_sa = static_cast<int64_t>(l1) * nn; b.in_so = nn; b.out_sa = static_cast<int64_t>(kxs) * nn; b.out_so = nn;
  b.sign = -1;
  TOEP_STEP(fft_pass(b, 0, 0, 0, s));
  cudaFreeAsync(x, s);
  x = nullptr;
  TOEP_ALLOC(dt, d_bytes);
  for (int64_t k0 = 0; k0 < op->K; k0 += 65535) {
    const int64_t nb = std::min<int64_t>(op->K - k0, 65535);
    TOEP_STEP(transpose_batched(TOEP_C128, static_cast<double2*>(d) + k0 * nn, static_cast<double2*>(dt) + k0 * nn,
                                nb, n0, n0, s));
  }
  cudaFreeAsync(d, s);
  d = nullptr;
  if (dtype == TOEP_C64) {
    void* dt32 = nullptr;
    TOEP_ALLOC(dt32, static_cast<size_t>(op->K) * nn * sizeof(float2));
    TOEP_STEP(cast_c128_to_c64(dt, dt32, op->K * nn, s));
    cudaFreeAsync(dt, s);
    dt = dt32;
  }
  op->DT = dt;
  op->ws[s];
  if (cudaStreamSynchronize(s) != cudaSuccess) {
    set_error("precompute_spectral failed: %s", cudaGetErrorString(cudaGetLastError()));
    dt = op->DT;
    return fail(TOEP_ERR_CUDA);
  }
#undef TOEP_STEP
#undef TOEP_ALLOC
  *out = op;
  return TOEP_OK;
}

int toep_op_destroy(toep_op_t op) {
  if (op == nullptr) return TOEP_OK;
  // Wait only for the streams this operator was used on (each entry point registers its stream in
  // op->ws), not the whole device; then return every buffer to the stream-ordered pool.
  cudaStream_t fs = cudaStreamPerThread;
  for (auto& kv : op->ws) cudaStreamSynchronize(kv.first);
  if (op->lazy_ev) cudaEventSynchronize(op->lazy_ev);
  cudaGetLastError();
  auto rel = [&](void* p) {
    if (p) cudaFreeAsync(p, fs);
  };
  for (auto& kv : op->ws) {
    auto& w = kv.second;
    if (w.pin_in) cudaFreeHost(w.pin_in);
    for (void* p : {w.x1, w.hat, w.hat2, static_cast<void*>(w.bar), static_cast<void*>(w.hatp),
                    static_cast<void*>(w.hat2p), w.io, static_cast<void*>(w.oz_b), static_cast<void*>(w.oz_bexp)})
      rel(p);
  }
  for (void* p : {static_cast<void*>(op->oz_a), static_cast<void*>(op->oz_aexp), op->DT, static_cast<void*>(op->DTp)})
    rel(p);
  if (op->lazy_ev) cudaEventDestroy(op->lazy_ev);
  delete op;
  TOEP_LAUNCHED();
  return TOEP_OK;
}

int toep_op_info(toep_op_t op, toep_op_info_t* info) {
  TOEP_REQUIRE(op != nullptr && info != nullptr, TOEP_ERR_ARG, "null argument");
  info->n2 = op->n2; info->n1 = op->n1; info->n0 = op->n0; info->l2 = op->l2; info->l1 = op->l1;
  info->dtype = op->dtype; info->bins = op->K; info->dim = op_dim(op);
  info->resident_bytes = static_cast<int64_t>(op->K) * op->n0 * op->n0 * static_cast<int64_t>(elt_size(op->dtype));
  return TOEP_OK;
}

int toep_op_diag_blocks(toep_op_t op, void* dst, void* stream) {
  TOEP_REQUIRE(op != nullptr && dst != nullptr, TOEP_ERR_ARG, "null argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  note_stream(op, s);
  const int64_t nn = static_cast<int64_t>(op->n0) * op->n0;
  const size_t es = elt_size(op->dtype);
  for (int64_t k0 = 0; k0 < op->K; k0 += 65535) {
    const int64_t nb = std::min<int64_t>(op->K - k0, 65535);
    TOEP_TRY(transpose_batched(op->dtype, static_cast<const char*>(op->DT) + k0 * nn * es,
                               static_cast<char*>(dst) + k0 * nn * es, nb, op->n0, op->n0, s));
  }
  return TOEP_OK;
}

int toep_op_fold_left(toep_op_t op, const void* m_dev, void* stream, toep_op_t* out) {
  TOEP_NVTX("toep_op_fold_left");
  TOEP_REQUIRE(op != nullptr && m_dev != nullptr && out != nullptr, TOEP_ERR_ARG, "null argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  note_stream(op, s);
  auto* f = new (std::nothrow) toep_op_s();
  TOEP_REQUIRE(f != nullptr, TOEP_ERR_OOM, "host allocation failed");
  f->n2 = op->n2; f->n1 = op->n1; f->n0 = op->n0; f->l2 = op->l2; f->l1 = op->l1; f->dtype = op->dtype;
  f->K = op->K; f->device = op->device;
  const int64_t n0 = op->n0;
  const size_t bytes = static_cast<size_t>(op->K) * n0 * n0 * elt_size(op->dtype);
  if (cudaMallocAsync(&f->DT, bytes, s) != cudaSuccess) {
    cudaGetLastError();
    delete f;
    set_error("out of device memory folding the preconditioner");
    return TOEP_ERR_OOM;
  }
  // DT'[k][j][:] = M DT[k][j][:]   ((M D_k)^T = D_k^T M^T, row j of D_k^T times M^T)
  const void* m = m_dev;
  void* m32 = nullptr;
  if (op->dtype == TOEP_C64) {
    TOEP_CUDA(cudaMallocAsync(&m32, n0 * n0 * sizeof(float2), s));
    TOEP_TRY(cast_c128_to_c64(m_dev, m32, n0 * n0, s));
    m = m32;
  }
  int rc = gemm(op->dtype, n0, op->K * n0, n0, make_double2(1, 0), m, n0, 1, 0, op->DT, 1, n0, 0,
                make_double2(0, 0), f->DT, 1, n0, 0, 1, s);
  if (m32) cudaFreeAsync(m32, s);
  if (rc != TOEP_OK) {
    cudaFreeAsync(f->DT, s);
    delete f;
    return rc;
  }
  f->ws[s];  // the build stream: toep_op_destroy(f) synchronises it
  *out = f;
  return TOEP_OK;
}

int toep_op_slab(toep_op_t op, int kx0, int kx1, void* stream, toep_op_t* out) {
  TOEP_REQUIRE(op != nullptr && out != nullptr && op->slab_kxs == 0, TOEP_ERR_ARG, "slab of a full operator only");
  TOEP_REQUIRE(0 <= kx0 && kx0 < kx1 && kx1 <= op->l1, TOEP_ERR_SHAPE, "slab [%d,%d) outside [0,%d)", kx0, kx1, op->l1);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  note_stream(op, s);
  auto* f = new (std::nothrow) toep_op_s();
  TOEP_REQUIRE(f != nullptr, TOEP_ERR_OOM, "host allocation failed");
  f->n2 = op->n2; f->n1 = op->n1; f->n0 = op->n0; f->l2 = op->l2; f->l1 = op->l1; f->dtype = op->dtype;
  f->device = op->device; f->slab_k0 = kx0; f->slab_kxs = kx1 - kx0;
  f->K = static_cast<int64_t>(op->l2) * f->slab_kxs;
  const size_t blk = static_cast<size_t>(op->n0) * op->n0 * elt_size(op->dtype);
  if (cudaMallocAsync(&f->DT, f->K * blk, s) != cudaSuccess) {
    cudaGetLastError();
    delete f;
    set_error("out of device memory for the spectral slab");
    return TOEP_ERR_OOM;
  }
  // one row of the (ky, kx) bin grid per ky: kxs contiguous bins
  const cudaError_t e = cudaMemcpy2DAsync(f->DT, f->slab_kxs * blk, static_cast<const char*>(op->DT) + kx0 * blk,
                                          op->l1 * blk, f->slab_kxs * blk, op->l2, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) {
    cudaFreeAsync(f->DT, s);
    delete f;
    set_error("slab copy failed: %s", cudaGetErrorString(e));
    return TOEP_ERR_CUDA;
  }
  f->ws[s];  // the build stream: toep_op_destroy(f) synchronises it
  *out = f;
  return TOEP_OK;
}

int toep_matvec_stage(toep_op_t op, int stage, const void* in, void* out, int64_t w, int count, void* stream) {
  TOEP_NVTX("toep_matvec_stage");
  TOEP_REQUIRE(op != nullptr && in != nullptr && out != nullptr && in != out && w >= 1 && count >= 0, TOEP_ERR_ARG,
               "bad matvec_stage arguments");
  return toep::matvec_stage_impl(op, stage, in, out, w, count, nullptr, static_cast<cudaStream_t>(stream));
}

int toep_matvec_stage_peer(toep_op_t op, int stage, const void* in, const toep_peer_scatter* scatter, int64_t w,
                           int count, void* stream) {
  TOEP_NVTX("toep_matvec_stage_peer");
  TOEP_REQUIRE(op != nullptr && in != nullptr && scatter != nullptr && w >= 1 && count >= 0, TOEP_ERR_ARG,
               "bad matvec_stage_peer arguments");
  TOEP_REQUIRE(stage == 0 || stage == 1, TOEP_ERR_ARG, "peer scatter is defined for stages 0 and 1, not %d", stage);
  return toep::matvec_stage_impl(op, stage, in, nullptr, w, count, scatter, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

namespace toep {

// stage 0 / 2: level-1 pass over `count` rows; stage 1: slab spectral step.  With `scatter` (device
// table, stages 0 and 1) the last pass stores into the destination ranks' buffers instead of `out`.
int matvec_stage_impl(toep_op_s* op, int stage, const void* in, void* out, int64_t w, int count,
                      const toep_peer_scatter* scatter, cudaStream_t s) {
  if (count == 0) return TOEP_OK;
  const int tc = op->dtype == TOEP_C64 ? 1 : 0;
  const int64_t inner = static_cast<int64_t>(op->n0) * w;
  if (stage == 0 || stage == 2) {  // level-1 forward / inverse pass over `count` array rows
    PassArgs a;
    a.in = in; a.out = out; a.L = op->l1; a.inner = inner; a.outer = count; a.scatter = scatter;
    if (stage == 0) {
      a.n_lo = op->n1; a.n_out = op->l1; a.in_sa = inner; a.in_so = op->n1 * inner; a.out_sa = inner;
      a.out_so = op->l1 * inner; a.sign = -1; a.scale = 1.0;
    } else {
      a.n_lo = op->l1; a.n_out = op->n1; a.in_sa = inner; a.in_so = op->l1 * inner; a.out_sa = inner;
      a.out_so = op->n1 * inner; a.sign = +1; a.scale = 1.0 / op->l1;
    }
    return fft_pass(a, tc, tc, tc, s);
  }
  TOEP_REQUIRE(stage == 1, TOEP_ERR_ARG, "unknown matvec stage %d", stage);
  const int kxs = op->slab_kxs ? op->slab_kxs : op->l1;
  TOEP_REQUIRE(count == kxs, TOEP_ERR_SHAPE, "slab width %d != operator slab %d", count, kxs);
  toep_op_s::Workspace* ws = nullptr;
  TOEP_TRY(op_workspace(op, w, s, &ws));
  PassArgs b;  // level-2 DFT of the slab columns: (n2, kxs, inner) -> (l2, kxs, inner) = bins ky*kxs + kx
  b.in = in; b.out = ws->hat; b.L = op->l2; b.n_lo = op->n2; b.n_out = op->l2; b.inner = inner; b.outer = kxs;
  b.in_sa = kxs * inner; b.in_so = inner; b.out_sa = kxs * inner; b.out_so = inner; b.sign = -1; b.scale = 1.0;
  TOEP_TRY(fft_pass(b, tc, tc, tc, s));
  TOEP_TRY(bin_product(op->dtype, op->DT, ws->hat, ws->hat2, op->K, op->n0, w, false, nullptr, s));
  PassArgs c;  // inverse level-2 DFT, kept rows only
  c.in = ws->hat2; c.out = out; c.L = op->l2; c.n_lo = op->l2; c.n_out = op->n2; c.inner = inner; c.outer = kxs;
  c.in_sa = kxs * inner; c.in_so = inner; c.out_sa = kxs * inner; c.out_so = inner; c.sign = +1;
  c.scale = 1.0 / op->l2;
  c.scatter = scatter;
  return fft_pass(c, tc, tc, tc, s);
}

}  // namespace toep

extern "C" {

int toep_matvec(toep_op_t op, const void* u, void* v, int64_t w, int flags, void* stream) {
  TOEP_NVTX("toep_matvec");
  TOEP_REQUIRE(op != nullptr && (w == 0 || (u != nullptr && v != nullptr)), TOEP_ERR_ARG, "null argument");
  TOEP_REQUIRE(op->slab_kxs == 0, TOEP_ERR_ARG, "a slab operator is applied through toep_matvec_stage");
  TOEP_REQUIRE(w >= 0, TOEP_ERR_SHAPE, "negative column count");
  TOEP_REQUIRE(w == 0 || u != v, TOEP_ERR_ARG, "matvec output must not alias its input");
  return matvec_impl(op, u, v, w, (flags & TOEP_MV_TRANSPOSE) != 0, (flags & TOEP_MV_IO_C128) != 0, nullptr,
                     static_cast<cudaStream_t>(stream));
}

int toep_matvec_host(toep_op_t op, const void* u_host, void* v_host, int64_t w, int flags, void* stream) {
  TOEP_NVTX("toep_matvec_host");
  TOEP_REQUIRE(op != nullptr && (w == 0 || (u_host != nullptr && v_host != nullptr)), TOEP_ERR_ARG, "null argument");
  TOEP_REQUIRE(op->slab_kxs == 0, TOEP_ERR_ARG, "a slab operator is applied through toep_matvec_stage");
  TOEP_REQUIRE(w >= 0, TOEP_ERR_SHAPE, "negative column count");
  TOEP_REQUIRE(w == 0 || u_host != v_host, TOEP_ERR_ARG, "matvec output must not alias its input");
  if (w == 0) return TOEP_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool io_c128 = (flags & TOEP_MV_IO_C128) != 0;
  const size_t bytes = static_cast<size_t>(toep::op_dim(op)) * w * (io_c128 ? 16 : toep::elt_size(op->dtype));
  toep_op_s::Workspace* ws = nullptr;
  {
    toep::keep_pool();
    std::lock_guard<std::mutex> lock(op->mu);
    ws = &op->ws[s];
    if (ws->io_cap < 2 * bytes) {
      if (ws->io) TOEP_CUDA(cudaFreeAsync(ws->io, s));
      ws->io = nullptr;
      ws->io_cap = 0;
      if (cudaMallocAsync(&ws->io, 2 * bytes, s) != cudaSuccess) {
        cudaGetLastError();
        toep::set_error("out of device memory for host matvec staging (w=%lld)", static_cast<long long>(w));
        return TOEP_ERR_OOM;
      }
      ws->io_cap = 2 * bytes;
    }
  }
  char* ud = static_cast<char*>(ws->io);
  char* vd = ud + bytes;
  if (flags & TOEP_MV_STAGE_INPUT) {
    void* pin = nullptr;
    {
      std::lock_guard<std::mutex> lock(op->mu);
      if (ws->pin_cap < bytes) {
        if (ws->pin_in) {
          cudaStreamSynchronize(s);  // an earlier call's DMA may still read the old buffer
          cudaFreeHost(ws->pin_in);
        }
        ws->pin_in = nullptr;
        ws->pin_cap = 0;
        if (cudaHostAlloc(&ws->pin_in, bytes, cudaHostAllocPortable) != cudaSuccess) {
          cudaGetLastError();
          toep::set_error("cudaHostAlloc of the input staging buffer (%zu bytes) failed", bytes);
          return TOEP_ERR_OOM;
        }
        ws->pin_cap = bytes;
      }
      pin = ws->pin_in;
    }
    TOEP_TRY(toep::staged_h2d(u_host, pin, ud, bytes, s));
  } else {
    TOEP_CUDA(cudaMemcpyAsync(ud, u_host, bytes, cudaMemcpyHostToDevice, s));
  }
  TOEP_TRY(toep::matvec_impl(op, ud, vd, w, (flags & TOEP_MV_TRANSPOSE) != 0, io_c128, nullptr, s));
  TOEP_CUDA(cudaMemcpyAsync(v_host, vd, bytes, cudaMemcpyDeviceToHost, s));
  // poll instead of cudaStreamSynchronize: the call is synchronous by contract and a sleeping
  // waiter's wake-up adds tens of microseconds to a ~240 us call (measured 244-299 us per call
  // box to box with the blocking wait)
  for (;;) {
    const cudaError_t e = cudaStreamQuery(s);
    if (e == cudaSuccess) break;
    if (e != cudaErrorNotReady) {
      toep::set_error("matvec_host: %s", cudaGetErrorString(e));
      return TOEP_ERR_CUDA;
    }
  }
  return TOEP_OK;
}

// host (pageable) -> device copy of `bytes`, staged through the library's page-locked buffers; the
// host source may be reused when the call returns, the device data is ordered on `stream`
int toep_h2d(const void* host, void* dev, uint64_t bytes, void* stream) {
  TOEP_REQUIRE(bytes == 0 || (host != nullptr && dev != nullptr), TOEP_ERR_ARG, "null argument");
  if (bytes == 0) return TOEP_OK;
  return toep::pipelined_h2d(host, dev, bytes, static_cast<cudaStream_t>(stream));
}

int toep_op_spectral_apply(toep_op_t op, const void* hat_in, void* hat_out, int64_t w, int flags, void* stream) {
  TOEP_REQUIRE(op != nullptr && hat_in != nullptr && hat_out != nullptr && hat_in != hat_out, TOEP_ERR_ARG,
               "bad spectral_apply arguments");
  note_stream(op, static_cast<cudaStream_t>(stream));
  return bin_product(op->dtype, op->DT, hat_in, hat_out, op->K, op->n0, w, (flags & TOEP_MV_TRANSPOSE) != 0, nullptr,
                     static_cast<cudaStream_t>(stream));
}

int toep_block_dft(const void* in, void* out, int n2, int n1, int64_t inner, int inverse, int dtype, void* stream) {
  TOEP_REQUIRE(in != nullptr && out != nullptr && in != out, TOEP_ERR_ARG, "bad block_dft buffers");
  TOEP_REQUIRE(n2 >= 1 && n1 >= 1 && inner >= 0, TOEP_ERR_SHAPE, "bad block_dft shape");
  if (inner == 0) return TOEP_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int t = dtype == TOEP_C64 ? 1 : 0;
  const int sign = inverse ? +1 : -1;
  void* mid = nullptr;
  const size_t bytes = static_cast<size_t>(n2) * n1 * inner * elt_size(dtype);
  TOEP_REQUIRE(cudaMallocAsync(&mid, bytes, s) == cudaSuccess, TOEP_ERR_OOM, "out of device memory in block_dft");
  PassArgs a;  // level 1 (axis of length n1) first, as block_fft_2l (toeplitz.py:241-243)
  a.in = in; a.out = mid; a.L = n1; a.n_lo = n1; a.n_out = n1; a.inner = inner; a.outer = n2; a.in_sa = inner;
  a.in_so = n1 * inner; a.out_sa = inner; a.out_so = n1 * inner; a.sign = sign; a.scale = inverse ? 1.0 / n1 : 1.0;
  int rc = fft_pass(a, t, t, t, s);
  if (rc == TOEP_OK) {
    PassArgs b;  // level 2
    b.in = mid; b.out = out; b.L = n2; b.n_lo = n2; b.n_out = n2; b.inner = inner; b.outer = n1;
    b.in_sa = static_cast<int64_t>(n1) * inner; b.in_so = inner; b.out_sa = static_cast<int64_t>(n1) * inner;
    b.out_so = inner; b.sign = sign; b.scale = inverse ? 1.0 / n2 : 1.0;
    rc = fft_pass(b, t, t, t, s);
  }
  cudaFreeAsync(mid, s);
  return rc;
}

int toep_block_apply(const void* m, int n0, const void* in, void* out, int64_t segments, int64_t w, int dtype,
                     void* stream) {
  TOEP_NVTX("toep_block_apply");
  TOEP_REQUIRE(m != nullptr && in != nullptr && out != nullptr, TOEP_ERR_ARG, "null argument");
  TOEP_REQUIRE(in != out, TOEP_ERR_ARG, "block_apply output must not alias its input");
  return block_apply_impl(m, n0, in, out, segments, w, dtype, static_cast<cudaStream_t>(stream), nullptr);
}

int toep_gemm(int dtype, int64_t m, int64_t n, int64_t k, const void* alpha, const void* a, int64_t a_rs,
              int64_t a_cs, int64_t a_bs, const void* b, int64_t b_rs, int64_t b_cs, int64_t b_bs, const void* beta,
              void* c, int64_t c_rs, int64_t c_cs, int64_t c_bs, int64_t batch, void* stream) {
  TOEP_NVTX("toep_gemm");
  TOEP_REQUIRE(alpha != nullptr && beta != nullptr, TOEP_ERR_ARG, "null alpha/beta");
  const double2 al = *static_cast<const double2*>(alpha);
  const double2 be = *static_cast<const double2*>(beta);
  int64_t done = 0;
  const size_t es = elt_size(dtype);
  while (done < batch) {
    const int64_t nb = std::min<int64_t>(batch - done, 65535);
    TOEP_TRY(gemm(dtype, m, n, k, al, static_cast<const char*>(a) + done * a_bs * es, a_rs, a_cs, a_bs,
                  static_cast<const char*>(b) + done * b_bs * es, b_rs, b_cs, b_bs, be,
                  static_cast<char*>(c) + done * c_bs * es, c_rs, c_cs, c_bs, nb, static_cast<cudaStream_t>(stream)));
    done += nb;
  }
  return TOEP_OK;
}

}  // extern "C"
