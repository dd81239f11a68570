// Native multi-GPU pieces of the row / kx-slab decomposition: an NCCL
// communicator owned by the library, the two all-to-all exchanges of the distributed matvec and the
// all-reduce of GMRES's inner products — all enqueued on the caller's stream, so the device GMRES
// engine (toep_gmres) drives a distributed solve through plain C function pointers
// (toep_slab_apply / toep_comm_allreduce) with no Python callback per Arnoldi step.
//
// NCCL is not linked: the library binds the libnccl.so.2 already loaded in the process (torch's,
// when torch.distributed runs the NCCL backend), else the system one, with dlopen / dlsym.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

#include "op.h"

namespace toep {
namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_get_async_error)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's own (torch's) first
    if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (h == nullptr) return;
    auto sym = [&](const char* name, auto* fn) {
      *fn = reinterpret_cast<std::remove_pointer_t<decltype(fn)>>(dlsym(h, name));
      return *fn != nullptr;
    };
    api.ok = sym("ncclGetUniqueId", &api.get_unique_id) && sym("ncclCommInitRank", &api.comm_init_rank) &&
             sym("ncclCommDestroy", &api.comm_destroy) && sym("ncclCommGetAsyncError", &api.comm_get_async_error) &&
             sym("ncclAllReduce", &api.all_reduce) && sym("ncclSend", &api.send) && sym("ncclRecv", &api.recv) &&
             sym("ncclGroupStart", &api.group_start) && sym("ncclGroupEnd", &api.group_end) &&
             sym("ncclGetErrorString", &api.error_string);
  });
  return api;
}

#define TOEP_NCCL(expr)                                                                          \
  do {                                                                                           \
    const ncclResult_t r_ = (expr);                                                              \
    if (r_ != ncclSuccess) {                                                                     \
      set_error("%s failed: %s", #expr, nccl().error_string ? nccl().error_string(r_) : "nccl"); \
      return TOEP_ERR_CUDA;                                                                      \
    }                                                                                            \
  } while (0)

// balanced contiguous split of n over `parts` (distributed.py column_range / row_range / slab_ranges)
inline void split_range(int n, int parts, int q, int* lo, int* hi) {
  const int per = n / parts, rem = n % parts;
  *lo = q * per + (q < rem ? q : rem);
  *hi = *lo + per + (q < rem ? 1 : 0);
}

}  // namespace
}  // namespace toep

struct toep_comm_s {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
};

struct toep_slab_ctx_s {
  toep_op_t op = nullptr;
  toep_comm_t comm = nullptr;
  int64_t w = 0;
  int ny = 0;                          // this rank's array rows
  std::vector<int> rows_lo, rows_hi;   // every rank's array rows
  std::vector<int> slab_lo, slab_hi;   // every rank's level-1 frequency slab
  void* buf[4] = {nullptr, nullptr, nullptr, nullptr};  // x1, pack / x1 slab, x2 slab, x2
  cudaStream_t alloc_stream = nullptr;
};

using namespace toep;

extern "C" {

int toep_comm_unique_id(void* id) {
  TOEP_REQUIRE(id != nullptr, TOEP_ERR_ARG, "null id buffer");
  TOEP_REQUIRE(nccl().ok, TOEP_ERR_CUDA, "libnccl.so.2 is not available");
  ncclUniqueId u;
  TOEP_NCCL(nccl().get_unique_id(&u));
  std::memcpy(id, &u, sizeof(u));
  return TOEP_OK;
}

int toep_comm_create(const void* id, int nranks, int rank, toep_comm_t* out) {
  TOEP_REQUIRE(id != nullptr && out != nullptr, TOEP_ERR_ARG, "null argument");
  TOEP_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, TOEP_ERR_ARG, "bad rank %d of %d", rank, nranks);
  TOEP_REQUIRE(nccl().ok, TOEP_ERR_CUDA, "libnccl.so.2 is not available");
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  auto* c = new toep_comm_s();
  c->nranks = nranks;
  c->rank = rank;
  const ncclResult_t r = nccl().comm_init_rank(&c->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    set_error("ncclCommInitRank failed: %s", nccl().error_string(r));
    delete c;
    return TOEP_ERR_CUDA;
  }
  *out = c;
  return TOEP_OK;
}

int toep_comm_destroy(toep_comm_t c) {
  if (c == nullptr) return TOEP_OK;
  if (c->comm != nullptr) nccl().comm_destroy(c->comm);
  delete c;
  return TOEP_OK;
}

// errors.py's contract for the collective path: an asynchronous NCCL failure (a peer died, a
// network error) surfaces as TOEP_ERR_CUDA with NCCL's message instead of a hang
int toep_comm_check(toep_comm_t c) {
  TOEP_REQUIRE(c != nullptr, TOEP_ERR_ARG, "null communicator");
  ncclResult_t ar = ncclSuccess;
  TOEP_NCCL(nccl().comm_get_async_error(c->comm, &ar));
  TOEP_REQUIRE(ar == ncclSuccess || ar == ncclInProgress, TOEP_ERR_CUDA, "NCCL asynchronous error: %s",
               nccl().error_string(ar));
  return TOEP_OK;
}

// in-place sum over the ranks of `n` doubles on the device; the signature of
// toep_gmres_problem_t.allreduce (ctx = the communicator)
int toep_comm_allreduce(void* ctx, void* buf, int64_t n, void* stream) {
  auto* c = static_cast<toep_comm_t>(ctx);
  TOEP_REQUIRE(c != nullptr && (n == 0 || buf != nullptr), TOEP_ERR_ARG, "bad allreduce arguments");
  if (c->nranks == 1 || n == 0) return TOEP_OK;
  TOEP_NCCL(nccl().all_reduce(buf, buf, static_cast<size_t>(n), ncclFloat64, ncclSum, c->comm,
                              static_cast<cudaStream_t>(stream)));
  return TOEP_OK;
}

// Distributed matvec context for a kx-slab operator (toep_op_slab / toep_op_create_slab) over the
// communicator's ranks: rank r owns array rows row_range(n2, P, r) of every vector and the bins of
// level-1 frequencies slab_ranges(l1, P, r) (distributed.py SlabOperator).  Scratch for w columns.
int toep_slab_ctx_create(toep_op_t op, toep_comm_t comm, int64_t w, void* stream, toep_slab_ctx_t* out) {
  TOEP_REQUIRE(op != nullptr && comm != nullptr && out != nullptr && w >= 1, TOEP_ERR_ARG, "bad slab ctx arguments");
  const int P = comm->nranks, r = comm->rank;
  auto* c = new toep_slab_ctx_s();
  c->op = op;
  c->comm = comm;
  c->w = w;
  c->rows_lo.resize(P);
  c->rows_hi.resize(P);
  c->slab_lo.resize(P);
  c->slab_hi.resize(P);
  for (int q = 0; q < P; ++q) {
    split_range(op->n2, P, q, &c->rows_lo[q], &c->rows_hi[q]);
    split_range(op->l1, P, q, &c->slab_lo[q], &c->slab_hi[q]);
  }
  const int kxs = op->slab_kxs ? op->slab_kxs : op->l1;
  const int k0 = op->slab_kxs ? op->slab_k0 : 0;
  if (k0 != c->slab_lo[r] || kxs != c->slab_hi[r] - c->slab_lo[r]) {
    set_error("slab operator holds kx [%d, %d), rank %d of %d owns [%d, %d)", k0, k0 + kxs, r, P, c->slab_lo[r],
              c->slab_hi[r]);
    delete c;
    return TOEP_ERR_ARG;
  }
  c->ny = c->rows_hi[r] - c->rows_lo[r];
  const size_t es = elt_size(op->dtype);
  const int64_t inner = static_cast<int64_t>(op->n0) * w;
  const size_t b_rows = static_cast<size_t>(c->ny) * op->l1 * inner * es;   // (ny, l1, inner)
  const size_t b_slab = static_cast<size_t>(op->n2) * kxs * inner * es;      // (n2, kxs, inner)
  const size_t sizes[4] = {b_rows, std::max(b_rows, b_slab), std::max(b_rows, b_slab), b_rows};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  c->alloc_stream = s;
  for (int i = 0; i < 4; ++i)
    if (sizes[i] && cudaMallocAsync(&c->buf[i], sizes[i], s) != cudaSuccess) {
      cudaGetLastError();
      for (int k = 0; k < i; ++k) cudaFreeAsync(c->buf[k], s);
      delete c;
      set_error("out of device memory for the slab matvec scratch");
      return TOEP_ERR_OOM;
    }
  *out = c;
  return TOEP_OK;
}

int toep_slab_ctx_destroy(toep_slab_ctx_t c) {
  if (c == nullptr) return TOEP_OK;
  for (void* p : c->buf)
    if (p) cudaFreeAsync(p, c->alloc_stream);
  cudaStreamSynchronize(c->alloc_stream);
  delete c;
  return TOEP_OK;
}

// y = A x for this rank's rows of x (ny*n1*n0, w): level-1 DFT of the local rows -> all-to-all
// (rows -> kx slabs) -> slab spectral step -> all-to-all back -> inverse level-1 DFT.  The
// toep_apply_fn signature of toep_gmres_problem_t.apply (ctx = the slab context).
int toep_slab_apply(void* ctx, const void* x, void* y, int64_t w, void* stream) {
  auto* c = static_cast<toep_slab_ctx_t>(ctx);
  TOEP_REQUIRE(c != nullptr && x != nullptr && y != nullptr && x != y, TOEP_ERR_ARG, "bad slab apply arguments");
  TOEP_REQUIRE(w == c->w, TOEP_ERR_SHAPE, "slab context built for %lld columns, got %lld", (long long)c->w,
               (long long)w);
  toep_op_s* op = c->op;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int P = c->comm->nranks, me = c->comm->rank;
  const size_t es = elt_size(op->dtype);
  const int64_t inner = static_cast<int64_t>(op->n0) * w;
  const size_t row_b = static_cast<size_t>(inner) * es;  // one (row, kx) line
  const int L1 = op->l1, kxs = c->slab_hi[me] - c->slab_lo[me];
  char* x1 = static_cast<char*>(c->buf[0]);    // (ny, L1, inner)
  char* pack = static_cast<char*>(c->buf[1]);  // [q](ny, kxs_q, inner) send blocks, later the slab output
  char* xs = static_cast<char*>(c->buf[2]);    // (n2, kxs, inner) slab input, later the [q](ny, kxs_q, inner) received
  char* x2 = static_cast<char*>(c->buf[3]);    // (ny, L1, inner)
  if (P == 1) {  // one rank: (ny, L1, inner) is already the (n2, kxs, inner) slab layout, no exchange
    TOEP_TRY(matvec_stage_impl(op, 0, x, x1, w, c->ny, nullptr, s));
    TOEP_TRY(matvec_stage_impl(op, 1, x1, x2, w, kxs, nullptr, s));
    return matvec_stage_impl(op, 2, x2, y, w, c->ny, nullptr, s);
  }
  TOEP_TRY(matvec_stage_impl(op, 0, x, x1, w, c->ny, nullptr, s));
  // exchange 1: rank q gets this rank's rows of its slab; the blocks from ranks 0..P-1 stacked in
  // rank order are its (n2, kxs, inner) slab input
  size_t off = 0;
  std::vector<size_t> pofs(P);
  for (int q = 0; q < P; ++q) {
    const int kq = c->slab_hi[q] - c->slab_lo[q];
    pofs[q] = off;
    if (c->ny > 0 && kq > 0)
      TOEP_CUDA(cudaMemcpy2DAsync(pack + off, kq * row_b, x1 + c->slab_lo[q] * row_b, L1 * row_b, kq * row_b, c->ny,
                                  cudaMemcpyDeviceToDevice, s));
    off += static_cast<size_t>(c->ny) * kq * row_b;
  }
  const size_t dw = es / sizeof(double);  // doubles per element
  TOEP_NCCL(nccl().group_start());
  for (int q = 0; q < P; ++q) {
    const int kq = c->slab_hi[q] - c->slab_lo[q];
    const size_t n_send = static_cast<size_t>(c->ny) * kq * inner * dw;
    const int nyq = c->rows_hi[q] - c->rows_lo[q];
    const size_t n_recv = static_cast<size_t>(nyq) * kxs * inner * dw;
    if (n_send) TOEP_NCCL(nccl().send(pack + pofs[q], n_send, ncclFloat64, q, c->comm->comm, s));
    if (n_recv)
      TOEP_NCCL(nccl().recv(xs + static_cast<size_t>(c->rows_lo[q]) * kxs * row_b, n_recv, ncclFloat64, q,
                            c->comm->comm, s));
  }
  TOEP_NCCL(nccl().group_end());
  TOEP_TRY(matvec_stage_impl(op, 1, xs, pack, w, kxs, nullptr, s));  // slab step -> pack
  // exchange 2: rank q gets its rows of this rank's slab; received blocks (ny, kxs_q, inner) land
  // at kx offset slab_lo[q] of (ny, L1, inner)
  char* ys = pack;  // (n2, kxs, inner) slab output
  char* recv2 = xs;  // reuse: [q](ny, kxs_q, inner)
  off = 0;
  for (int q = 0; q < P; ++q) {
    pofs[q] = off;
    off += static_cast<size_t>(c->ny) * (c->slab_hi[q] - c->slab_lo[q]) * row_b;
  }
  TOEP_NCCL(nccl().group_start());
  for (int q = 0; q < P; ++q) {
    const int nyq = c->rows_hi[q] - c->rows_lo[q];
    const int kq = c->slab_hi[q] - c->slab_lo[q];
    const size_t n_send = static_cast<size_t>(nyq) * kxs * inner * dw;
    const size_t n_recv = static_cast<size_t>(c->ny) * kq * inner * dw;
    if (n_send)
      TOEP_NCCL(nccl().send(ys + static_cast<size_t>(c->rows_lo[q]) * kxs * row_b, n_send, ncclFloat64, q,
                            c->comm->comm, s));
    if (n_recv) TOEP_NCCL(nccl().recv(recv2 + pofs[q], n_recv, ncclFloat64, q, c->comm->comm, s));
  }
  TOEP_NCCL(nccl().group_end());
  for (int q = 0; q < P; ++q) {
    const int kq = c->slab_hi[q] - c->slab_lo[q];
    if (c->ny > 0 && kq > 0)
      TOEP_CUDA(cudaMemcpy2DAsync(x2 + c->slab_lo[q] * row_b, L1 * row_b, recv2 + pofs[q], kq * row_b, kq * row_b,
                                  c->ny, cudaMemcpyDeviceToDevice, s));
  }
  return matvec_stage_impl(op, 2, x2, y, w, c->ny, nullptr, s);
}

}  // extern "C"
