/*
 * libtoepcuda — C ABI of the B200-native MLFFT block-Toeplitz hot path.
 *
 * This is the drop-in boundary: plain pointers and sizes, no torch types.
 * Each entry point replaces one function of the reference Python API
 * (toepsolve, /root/reference/pkg/src/toepsolve); the replaced function is
 * cited (file:line) above each declaration.  The Python host mirror
 * (paper_2506_20350_b200/) binds these with ctypes.
 *
 * Conventions
 *   - complex128 = interleaved {double re, im}; complex64 = {float re, im}.
 *   - A "stacked vector" / column block is (n, w) row-major, n = n2*n1*n0,
 *     row index (i2*n1 + i1)*n0 + b, exactly the reference layout
 *     (toeplitz.py:256-269).
 *   - All device pointers belong to the current CUDA device; `stream` is a
 *     cudaStream_t (NULL = legacy default stream).  Calls are asynchronous
 *     on `stream` unless stated otherwise.
 *   - Every function returns a status code; toep_last_error() gives the
 *     thread-local message of the last failure.
 */
#ifndef TOEPCUDA_H
#define TOEPCUDA_H

#include <stdint.h>

#if defined(__GNUC__)
#define TOEP_API __attribute__((visibility("default")))
#else
#define TOEP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes -> Python exceptions (paper_2506_20350_b200/_lib.py). */
#define TOEP_OK 0
#define TOEP_ERR_SHAPE 1          /* errors.ShapeError            (errors.py:8)  */
#define TOEP_ERR_ARG 2            /* ValueError                                  */
#define TOEP_ERR_SINGULAR 3       /* errors.SingularMatrix        (errors.py:24) */
#define TOEP_ERR_SINGULAR_BLOCK 4 /* errors.SingularBlock         (errors.py:28) */
#define TOEP_ERR_SINGULAR_DENOM 5 /* errors.SingularDenominator   (errors.py:32) */
#define TOEP_ERR_NOCONV 6         /* errors.NoConvergence         (errors.py:76) */
#define TOEP_ERR_CUDA 7           /* errors.CudaError (RuntimeError)             */
#define TOEP_ERR_OOM 8            /* MemoryError                                 */

/* Element types. */
#define TOEP_C128 0
#define TOEP_C64 1

/* toep_matvec flags. */
#define TOEP_MV_TRANSPOSE 1   /* matvec_transpose (toeplitz.py:306-324)                */
#define TOEP_MV_IO_C128 2     /* c64 operator, but u / v are complex128 (cast in the   */
                              /* first / last FFT pass; the GMRES Krylov space is c128) */
#define TOEP_MV_STAGE_INPUT 4 /* toep_matvec_host: u_host is pageable (e.g. a numpy      */
                              /* array): the library's copy threads stage it through a  */
                              /* page-locked buffer in chunks, each chunk's DMA issued  */
                              /* as soon as it is staged (copies overlap the transfer)  */

typedef struct toep_op_s* toep_op_t;

typedef struct {
  int32_t n2, n1, n0;     /* Ny (level 2), Nx (level 1), N_b (block side)          */
  int32_t l2, l1;         /* circulant embedding lengths (>= 2n-1; default 2n)     */
  int32_t dtype;          /* TOEP_C128 / TOEP_C64                                   */
  int64_t bins;           /* l2 * l1 frequency bins                                 */
  int64_t dim;            /* n2 * n1 * n0                                           */
  int64_t resident_bytes; /* spectral blocks resident in HBM                        */
} toep_op_info_t;

TOEP_API const char* toep_last_error(void);
TOEP_API int toep_version(void);

/* problems.py:219-226 fnv1a64: 64-bit FNV-1a of `bytes` host bytes (the TBZ1 payload checksum,
 * problems.py:236-322).  Host-only; the Python host code parses the container. */
TOEP_API int toep_fnv1a64(const void* data, uint64_t bytes, uint64_t* out);

/* toeplitz.py:248-253 precompute_spectral (+ SpectralOperator, :135-155).
 * stacked4: the generator, (2n2-1, 2n1-1, n0, n0) complex128 row-major in
 * circulant order (BlockGenerator2L.stacked4(), toeplitz.py:129-131), on the
 * host (on_device = 0) or on the device (on_device = 1).  The blocks are
 * embedded into an (l2, l1) circulant (l = 0 picks 2n), transformed on the
 * device by the batched FFT kernels and kept resident in HBM as one
 * n0 x n0 block per bin, stored transposed (column-major) for streaming. */
TOEP_API int toep_op_create(const void* stacked4, int on_device, int n2, int n1, int n0, int l2, int l1,
                   int dtype, void* stream, toep_op_t* out);
/* Releases the operator.  Waits for the streams the operator was used on (each entry point
 * registers its stream), not the whole device: those streams must still be valid here. */
TOEP_API int toep_op_destroy(toep_op_t op);
TOEP_API int toep_op_info(toep_op_t op, toep_op_info_t* info);
/* SpectralOperator.diag_blocks (toeplitz.py:153): copy the (bins, n0, n0) blocks, row-major. */
TOEP_API int toep_op_diag_blocks(toep_op_t op, void* dst_dev, void* stream);
/* New operator whose blocks are M * D_k (M: n0 x n0 complex128, device).
 * With M = R_00^-1 this folds the element preconditioner P_K (precond.py:124-131)
 * into the operator, valid because P_K = I (x) R_00 commutes with F (x) I_n0. */
TOEP_API int toep_op_fold_left(toep_op_t op, const void* m_dev, void* stream, toep_op_t* out);

/* toeplitz.py:287-303 matvec (flags & TOEP_MV_TRANSPOSE: :306-324 matvec_transpose).
 * u, v: (n, w) device column blocks.  pad_rhs / extract_result (:256-284) are
 * fused into the first / last FFT pass.  v must not alias u. */
TOEP_API int toep_matvec(toep_op_t op, const void* u, void* v, int64_t w, int flags, void* stream);
/* toep_matvec with HOST u / v (pinned for overlap-free DMA; pageable works): copy in, apply, copy
 * out and synchronise `stream` in one call (the numpy-in / numpy-out contract of toeplitz.py:287-303
 * without per-call device allocations); device staging is owned by the operator, per stream. */
TOEP_API int toep_matvec_host(toep_op_t op, const void* u_host, void* v_host, int64_t w, int flags, void* stream);

/* Page-locked host memory for the host vectors of toep_matvec_host (the numpy in/out buffers of
 * toeplitz.py:287-303 when the caller keeps them pinned).  cudaHostAlloc(Portable); `bytes` == 0
 * yields NULL.  No reference counterpart (the reference never leaves host memory). */
TOEP_API int toep_host_alloc(uint64_t bytes, void** out);
TOEP_API int toep_host_free(void* p);
/* Pageable host -> device copy of `bytes` staged through the library's double-buffered page-locked
 * chunks (the generator / level-1 block uploads behind precompute_spectral, toeplitz.py:248-253, and
 * assemble_level1, rybicki.py:53-60): near the DMA rate instead of the driver's pageable 8-9 GB/s.
 * The host source may be reused on return; the device data is ordered on `stream`. */
TOEP_API int toep_h2d(const void* host, void* dev, uint64_t bytes, void* stream);

/* Native multi-GPU plumbing for the slab decomposition (the reference is
 * single-process, so no counterpart): an NCCL communicator owned by the library (NCCL bound with
 * dlopen: the process's own libnccl.so.2 first), the distributed matvec of a slab operator with both
 * all-to-all exchanges enqueued on the stream, and the all-reduce of GMRES's inner products.
 * toep_slab_apply / toep_comm_allreduce have the toep_apply_fn / allreduce signatures of
 * toep_gmres_problem_t (ctx = the slab context / the communicator), so toep_gmres runs a
 * distributed solve with no host callback per Arnoldi step.  toep_comm_check reports an
 * asynchronous NCCL error (ncclCommGetAsyncError) as TOEP_ERR_CUDA. */
typedef struct toep_comm_s* toep_comm_t;
typedef struct toep_slab_ctx_s* toep_slab_ctx_t;
TOEP_API int toep_comm_unique_id(void* id /* 128 bytes */);
TOEP_API int toep_comm_create(const void* id, int nranks, int rank, toep_comm_t* out);
TOEP_API int toep_comm_destroy(toep_comm_t comm);
TOEP_API int toep_comm_check(toep_comm_t comm);
TOEP_API int toep_comm_allreduce(void* comm, void* buf, int64_t ndoubles, void* stream);
TOEP_API int toep_slab_ctx_create(toep_op_t slab_op, toep_comm_t comm, int64_t w, void* stream, toep_slab_ctx_t* out);
TOEP_API int toep_slab_ctx_destroy(toep_slab_ctx_t ctx);
TOEP_API int toep_slab_apply(void* ctx, const void* x, void* y, int64_t w, void* stream);

/* Multi-GPU row / kx-slab decomposition (no reference counterpart:
 * the reference is single-process).  toep_op_slab: operator holding only the bins with
 * level-1 frequency kx in [kx0, kx1).  toep_matvec_stage: the local steps of one distributed
 * matvec, the caller doing the two all-to-all exchanges in between:
 *   stage 0: level-1 forward DFT of `count` array rows, in (count, n1, n0*w) -> out (count, l1, n0*w)
 *   stage 1: slab spectral step (level-2 DFT, per-bin product, inverse level-2 DFT, kept rows),
 *            in/out (n2, count = slab width, n0*w)
 *   stage 2: level-1 inverse DFT + crop + 1/(l1*l2) of `count` rows, (count, l1, n0*w) -> (count, n1, n0*w) */
TOEP_API int toep_op_slab(toep_op_t op, int kx0, int kx1, void* stream, toep_op_t* out);
/* The slab operator built straight from the generator (toeplitz.py:248-253 restricted to the
 * rank's level-1 frequencies): level-1 DFT of all generator rows, level-2 DFT of columns
 * [kx0, kx1) only; the full spectral operator never exists on the rank (resident bytes = D * kxs / l1).
 * kx1 <= kx0 builds the full operator (= toep_op_create). */
TOEP_API int toep_op_create_slab(const void* stacked4, int on_device, int n2, int n1, int n0, int l2, int l1,
                                 int dtype, int kx0, int kx1, void* stream, toep_op_t* out);
TOEP_API int toep_matvec_stage(toep_op_t op, int stage, const void* in, void* out, int64_t w, int count,
                               void* stream);

/* Peer-memory exchange (NVLink P2P through CUDA IPC): stages 0 and 1 of toep_matvec_stage with
 * their output stored straight into the destination ranks' receive buffers, so the all-to-all
 * that follows each of them is fused into the DFT's final store.  Output index a of the pass
 * (stage 0: level-1 frequency kx; stage 1: array row y) in [lo[q], lo[q+1]) is written to
 *   base[q] + es * (off[q] + a*sa[q] + o*so[q] + i)     (o: the pass's outer index, i: n0*w index)
 * and after its last store every launch adds 1 to each destination's arrival counter
 * (release, system scope).  `scatter` is a DEVICE copy of the table; `done` must start at 0 and
 * is owned by the kernel.  toep_peer_wait blocks the stream until *counter >= target (acquire,
 * system scope; traps after 30 s so a missing peer fails loudly instead of hanging). */
#define TOEP_MAX_PEERS 8
typedef struct toep_peer_scatter {
  int64_t parts;                     /* destinations, 1..TOEP_MAX_PEERS */
  int64_t lo[TOEP_MAX_PEERS + 1];
  uint64_t base[TOEP_MAX_PEERS];     /* device (peer-mapped) address of destination q's buffer */
  int64_t off[TOEP_MAX_PEERS];
  int64_t sa[TOEP_MAX_PEERS];
  int64_t so[TOEP_MAX_PEERS];
  uint64_t signal[TOEP_MAX_PEERS];   /* device address of destination q's u64 arrival counter */
  uint64_t done;                     /* CTA completion count of the running launch */
} toep_peer_scatter;
TOEP_API int toep_matvec_stage_peer(toep_op_t op, int stage, const void* in, const toep_peer_scatter* scatter,
                                    int64_t w, int count, void* stream);
TOEP_API int toep_peer_wait(const uint64_t* counter, uint64_t target, void* stream);
/* cudaMalloc'd (not pool) memory for exchange buffers, and its IPC handle (64 bytes) / mapping */
TOEP_API int toep_peer_alloc(uint64_t bytes, void** out);
TOEP_API int toep_peer_free(void* ptr);
TOEP_API int toep_ipc_handle(const void* ptr, void* handle64);
TOEP_API int toep_ipc_open(const void* handle64, void** out);
TOEP_API int toep_ipc_close(void* ptr);

/* toeplitz.py:300 (flags & TOEP_MV_TRANSPOSE: :320): the per-bin product alone,
 * hat_out[k] = D_k @ hat_in[k] for every bin k, hat_* (bins, n0, w) in the
 * operator dtype.  This is the streaming kernel that carries >98% of the
 * matvec's HBM bytes; exposed separately for spectral-domain use and timing. */
TOEP_API int toep_op_spectral_apply(toep_op_t op, const void* hat_in, void* hat_out, int64_t w, int flags,
                                    void* stream);

/* toeplitz.py:229-245 block_fft_2l (n2 == 1: :215-226 block_fft_1l): F_{n2} (x) F_{n1} (x) I_inner
 * on (n2*n1*inner) contiguous values, level 1 first; inverse carries 1/(n1*n2) like
 * np.fft.ifft per axis.  Lengths must be 13-smooth. out must not alias in. */
TOEP_API int toep_block_dft(const void* in, void* out, int n2, int n1, int64_t inner, int inverse, int dtype, void* stream);

/* precond.py:65-71 Preconditioner._solve_segments as a product with the
 * precomputed inverse: out[s] = M @ in[s] for every (n0, w) segment s of an
 * (segments*n0, w) block; M: n0 x n0 device.  out must not alias in. */
TOEP_API int toep_block_apply(const void* m, int n0, const void* in, void* out, int64_t segments, int64_t w,
                     int dtype, void* stream);

/* Batched strided complex GEMM, the dense block product used by the solvers
 * (rybicki.py:114-133 block sums, bordered.py border products):
 * C_b = alpha * A_b @ B_b + beta * C_b, element (r, c) of X_b at
 * X + b*bs + r*rs + c*cs (strides in elements). */
TOEP_API int toep_gemm(int dtype, int64_t m, int64_t n, int64_t k, const void* alpha, const void* a, int64_t a_rs,
              int64_t a_cs, int64_t a_bs, const void* b, int64_t b_rs, int64_t b_cs, int64_t b_bs,
              const void* beta, void* c, int64_t c_rs, int64_t c_cs, int64_t c_bs, int64_t batch,
              void* stream);
/* Real FP64 C = alpha A B + beta C on the FP64 tensor cores (hand-written DMMA kernels, dmma.cu):
 * the real products of the 3M block products of rybicki.py:114-133.  Each operand needs a unit
 * stride in one dimension; batch strides may be negative. */
/* Real FP64 GEMM on the int8 tensor cores (Ozaki scheme: 7 signed base-128 digits per value, per-row
 * / per-column power-of-two scaling, exact int32 digit products in TMEM, FP64 recombination): the
 * engine of the Rybicki block sums (rybicki.py:114-131).  Row-major A (M x K, M % 128 == 0),
 * B (K x N), C (M x N); K % 32 == 0, K <= 19 000 (int32-exact digit sums).  ~1e-13 relative. */
TOEP_API int toep_ozaki_dgemm(int M, int N, int64_t K, double alpha, const double* A, int64_t lda, const double* B,
                              int64_t ldb, double beta, double* C, int64_t ldc, void* stream);
TOEP_API int toep_dgemm(int64_t m, int64_t n, int64_t k, double alpha, const double* a, int64_t a_rs, int64_t a_cs,
                        int64_t a_bs, const double* b, int64_t b_rs, int64_t b_cs, int64_t b_bs, double beta,
                        double* c, int64_t c_rs, int64_t c_cs, int64_t c_bs, int64_t batch, void* stream);

/* ------------------------------------------------------------------ GMRES
 * solvers/gmres.py:98-219 _gmres_block, device resident: the Krylov basis,
 * Hessenberg columns, Givens rotations and the residual recurrence live in
 * HBM; the host only polls a completion flag one Arnoldi step behind. */
typedef int (*toep_apply_fn)(void* ctx, const void* x, void* y, int64_t w, void* stream);

#define TOEP_PC_NONE 0     /* apply_precond(None, v) = v                            */
#define TOEP_PC_BLOCK 1    /* P_K^-1 applied every step: toep_block_apply(pinv)      */
#define TOEP_PC_FOLDED 2   /* op already holds P_K^-1 A (toep_op_fold_left);        */
                           /* pinv gives P^-1 b, pmat gives A x = P (P^-1 A) x      */
#define TOEP_PC_CALLBACK 3 /* papply(ctx, x, y, w, stream)                          */

typedef struct {
  toep_op_t op;               /* operator; NULL -> use apply/apply_ctx               */
  toep_apply_fn apply;
  void* apply_ctx;
  int32_t precond;            /* TOEP_PC_*                                           */
  int32_t pside;              /* n0 of pinv / pmat                                   */
  const void* pinv;           /* pside x pside complex128, device                    */
  const void* pmat;           /* pside x pside complex128, device (FOLDED only)      */
  toep_apply_fn papply;
  void* papply_ctx;
  int64_t n, w;               /* the Krylov vectors are (n, w) complex128 blocks     */
  /* distributed Krylov vectors (rows split over ranks, e.g. the slab-decomposed matvec):
   * every inner product / norm is summed over ranks by allreduce(ctx, buf, ndoubles, stream)
   * on a device buffer, enqueued on `stream` (NCCL all-reduce).  NULL: single process. */
  int (*allreduce)(void* ctx, void* buf, int64_t ndoubles, void* stream);
  void* allreduce_ctx;
} toep_gmres_problem_t;

typedef struct {
  double tol;                 /* GmresConfig.tol      (gmres.py:40)                  */
  int32_t max_iter;           /* GmresConfig.max_iter (gmres.py:41)                  */
  int32_t restart;            /* GmresConfig.restart, 0 = None (full GMRES)          */
  int32_t timings;            /* 1: fill per-phase timings with CUDA events          */
} toep_gmres_cfg_t;

typedef struct {
  int32_t iterations;         /* SolveReport.iterations                              */
  int32_t converged;          /* SolveReport.converged                               */
  int32_t breakdown;          /* Arnoldi breakdown (h_{j+1,j} == 0)                   */
  int32_t n_history;          /* entries written to history                          */
  double final_residual;      /* ||b - A x|| / ||b||, unpreconditioned               */
  double t_matvec, t_precond, t_orth, t_total;   /* phase_timings, seconds           */
  double* history;            /* caller-owned host buffer: residual_history          */
  int32_t history_cap;
} toep_gmres_report_t;

/* b, x: (n, w) complex128 device blocks; x is overwritten with the iterate.
 * Returns TOEP_OK even when not converged (report.converged = 0); the Python
 * layer raises NoConvergence with the iterate attached, as gmres.py:242-248. */
TOEP_API int toep_gmres(const toep_gmres_problem_t* prob, const toep_gmres_cfg_t* cfg, const void* b, void* x,
               void* stream, toep_gmres_report_t* rep);

/* solvers/gmres.py:304-336 solve_multi_rhs_sequential: an independent GMRES per column of
 * the (n, w) block b, all columns advanced in lock step so each Arnoldi step is one
 * multi-RHS matvec (per-bin complex GEMM on the FP64 tensor cores).  Requires prob->op;
 * precond NONE / FOLDED / BLOCK.  Per-column outputs (host arrays of length w): iterations,
 * converged, final_residual, n_history; history: host (history_rows, w) array, column c's
 * residual_history[t] at history[t*w + c]. */
TOEP_API int toep_gmres_batched(const toep_gmres_problem_t* prob, const toep_gmres_cfg_t* cfg, const void* b,
                                void* x, void* stream, int32_t* iterations, int32_t* converged,
                                double* final_residual, int32_t* n_history, double* history, int64_t history_rows);

/* ------------------------------------------------------------ direct solve
 * numerics.py:67-96 lu_factor / lu_solve: in-place LU with partial pivoting of an n x n
 * row-major complex128 device matrix (ipiv: device int[n], LAPACK-style row interchanges;
 * info: device int, > 0 when a pivot is below 1e-300), and the solve A X = B for an
 * (n, nrhs) row-major device block B (overwritten). */
TOEP_API int toep_lu_factor(void* a, int n, int* ipiv, int* info, void* stream);
TOEP_API int toep_lu_solve(const void* lu, int n, const int* ipiv, void* b, int64_t nrhs, void* stream);

/* rybicki.py:63-144 rybicki_solve: blocks (2N-1, s, s) complex128 device, circulant order
 * (block (i, j) of the system = blocks[(i - j) mod (2N-1)]); y, x: (N*s, w) device blocks.
 * Returns TOEP_ERR_SINGULAR_BLOCK (R_0) or TOEP_ERR_SINGULAR_DENOM with *fail_step = m.
 * hook (nullable): called after every stage with device views x (N,s,w), g, h (N-1,s,s)
 * whose first `stage` entries are valid (rybicki.py:107-108,139-141 step_hook). */
typedef int (*toep_stage_fn)(void* ctx, int stage, const void* x, const void* g, const void* h, void* stream);
TOEP_API int toep_rybicki(const void* blocks, int N, int s, const void* y, void* x, int64_t w, int* fail_step,
                          toep_stage_fn hook, void* hook_ctx, void* stream);
/* solvers/rybicki.py:53-60 assemble_level1: (2n2-1, n1*n0, n1*n0) dense level-1 blocks in circulant
 * order, gathered on the device from the stacked generator (2n2-1, 2n1-1, n0, n0) (device pointers). */
TOEP_API int toep_assemble_level1(const void* stacked4, int n2, int n1, int n0, void* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TOEPCUDA_H */
