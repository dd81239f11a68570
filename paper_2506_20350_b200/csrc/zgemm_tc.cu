// Complex FP64 GEMM on the FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64).
//
// sm_100a has no tcgen05 kind for f64 (ptxas rejects .kind::f64), so the FP64 tensor-core
// path on B200 is the warp-level DMMA instruction.  The tile machinery (3-stage cp.async
// pipeline, 64x64x16 CTA tile, 32x32x16 warp tile, complex accumulation as four real
// DMMA products per k-step) is CUTLASS's Sm80 tensor-op complex GEMM template,
// instantiated here for the three layouts the solvers use:
//   * per-bin product V_k = D_k U_k, many right-hand sides (toeplitz.py:300 at W >= 16):
//     A column-major (DT storage), B / C row-major, batched over the 3600 bins;
//   * P_K fold / block apply (precond.py:65-71): A row-major, B / C column-major;
//   * dense block products of the block-Rybicki recursion (rybicki.py:114-133): all row-major.
#include <cutlass/complex.h>
#include <cutlass/gemm/device/gemm_universal.h>
#include <cutlass/epilogue/thread/linear_combination.h>

#include "kernels.cuh"

namespace toep {

namespace {

using cd = cutlass::complex<double>;

template <typename LA, typename LB, typename LC>
using ZGemm = cutlass::gemm::device::GemmUniversal<
    cd, LA, cd, LB, cd, LC, cd, cutlass::arch::OpClassTensorOp, cutlass::arch::Sm80,
    cutlass::gemm::GemmShape<64, 64, 16>, cutlass::gemm::GemmShape<32, 32, 16>, cutlass::gemm::GemmShape<8, 8, 4>,
    cutlass::epilogue::thread::LinearCombination<cd, 1, cd, cd>,
    cutlass::gemm::threadblock::GemmIdentityThreadblockSwizzle<>, 3, 1, 1, cutlass::arch::OpMultiplyAddComplex>;

// real FP64 tensor-core GEMM (all row-major): the three products of the 3M complex method
using DGemmRM = cutlass::gemm::device::GemmUniversal<
    double, cutlass::layout::RowMajor, double, cutlass::layout::RowMajor, double, cutlass::layout::RowMajor, double,
    cutlass::arch::OpClassTensorOp, cutlass::arch::Sm80, cutlass::gemm::GemmShape<64, 64, 16>,
    cutlass::gemm::GemmShape<32, 32, 16>, cutlass::gemm::GemmShape<8, 8, 4>,
    cutlass::epilogue::thread::LinearCombination<double, 1, double, double>,
    cutlass::gemm::threadblock::GemmIdentityThreadblockSwizzle<>, 3>;

using DGemmCRR = cutlass::gemm::device::GemmUniversal<
    double, cutlass::layout::ColumnMajor, double, cutlass::layout::RowMajor, double, cutlass::layout::RowMajor,
    double, cutlass::arch::OpClassTensorOp, cutlass::arch::Sm80, cutlass::gemm::GemmShape<64, 64, 16>,
    cutlass::gemm::GemmShape<32, 32, 16>, cutlass::gemm::GemmShape<8, 8, 4>,
    cutlass::epilogue::thread::LinearCombination<double, 1, double, double>,
    cutlass::gemm::threadblock::GemmIdentityThreadblockSwizzle<>, 3>;

template <typename G>
int run(int64_t m, int64_t n, int64_t k, double2 alpha, const void* a, int64_t lda, int64_t a_bs, const void* b,
        int64_t ldb, int64_t b_bs, double2 beta, void* c, int64_t ldc, int64_t c_bs, int64_t batch, cudaStream_t s) {
  typename G::Arguments args(cutlass::gemm::GemmUniversalMode::kBatched,
                             {static_cast<int>(m), static_cast<int>(n), static_cast<int>(k)}, static_cast<int>(batch),
                             {cd(alpha.x, alpha.y), cd(beta.x, beta.y)}, a, b, c, c, a_bs, b_bs, c_bs, c_bs, lda, ldb,
                             ldc, ldc);
  G op;
  cutlass::Status st = op.can_implement(args);
  if (st != cutlass::Status::kSuccess) {
    set_error("zgemm_tc: cannot implement (%s)", cutlassGetStatusString(st));
    return TOEP_ERR_ARG;
  }
  st = op.initialize(args, nullptr, s);
  if (st == cutlass::Status::kSuccess) st = op.run(s);
  if (st != cutlass::Status::kSuccess) {
    set_error("zgemm_tc: %s", cutlassGetStatusString(st));
    return TOEP_ERR_CUDA;
  }
  TOEP_LAUNCHED();
  return TOEP_OK;
}

}  // namespace

int dgemm_tc_rm(int64_t m, int64_t n, int64_t k, double alpha, const double* a, int64_t lda, int64_t a_bs,
                const double* b, int64_t ldb, int64_t b_bs, double beta, double* c, int64_t ldc, int64_t c_bs,
                int64_t batch, cudaStream_t s) {
  if (m == 0 || n == 0 || batch == 0) return TOEP_OK;
  TOEP_REQUIRE(m <= INT32_MAX && n <= INT32_MAX && k <= INT32_MAX && batch <= INT32_MAX, TOEP_ERR_ARG,
               "dgemm_tc: size too large");
  typename DGemmRM::Arguments args(cutlass::gemm::GemmUniversalMode::kBatched,
                                   {static_cast<int>(m), static_cast<int>(n), static_cast<int>(k)},
                                   static_cast<int>(batch), {alpha, beta}, a, b, c, c, a_bs, b_bs, c_bs, c_bs, lda, ldb,
                                   ldc, ldc);
  DGemmRM op;
  cutlass::Status st = op.can_implement(args);
  if (st != cutlass::Status::kSuccess) {
    set_error("dgemm_tc: cannot implement (%s)", cutlassGetStatusString(st));
    return TOEP_ERR_ARG;
  }
  st = op.initialize(args, nullptr, s);
  if (st == cutlass::Status::kSuccess) st = op.run(s);
  if (st != cutlass::Status::kSuccess) {
    set_error("dgemm_tc: %s", cutlassGetStatusString(st));
    return TOEP_ERR_CUDA;
  }
  TOEP_LAUNCHED();
  return TOEP_OK;
}

int dgemm_tc_crr(int64_t m, int64_t n, int64_t k, const double* a, int64_t lda, int64_t a_bs, const double* b,
                 int64_t ldb, int64_t b_bs, double* c, int64_t ldc, int64_t c_bs, int64_t batch, cudaStream_t s) {
  if (m == 0 || n == 0 || batch == 0) return TOEP_OK;
  TOEP_REQUIRE(m <= INT32_MAX && n <= INT32_MAX && k <= INT32_MAX && batch <= INT32_MAX, TOEP_ERR_ARG,
               "dgemm_tc: size too large");
  typename DGemmCRR::Arguments args(cutlass::gemm::GemmUniversalMode::kBatched,
                                    {static_cast<int>(m), static_cast<int>(n), static_cast<int>(k)},
                                    static_cast<int>(batch), {1.0, 0.0}, a, b, c, c, a_bs, b_bs, c_bs, c_bs, lda, ldb,
                                    ldc, ldc);
  DGemmCRR op;
  cutlass::Status st = op.can_implement(args);
  if (st != cutlass::Status::kSuccess) {
    set_error("dgemm_tc: cannot implement (%s)", cutlassGetStatusString(st));
    return TOEP_ERR_ARG;
  }
  st = op.initialize(args, nullptr, s);
  if (st == cutlass::Status::kSuccess) st = op.run(s);
  if (st != cutlass::Status::kSuccess) {
    set_error("dgemm_tc: %s", cutlassGetStatusString(st));
    return TOEP_ERR_CUDA;
  }
  TOEP_LAUNCHED();
  return TOEP_OK;
}

// Tensor-core ZGEMM for a (row stride, column stride) pair per operand that is either
// row-major (cs == 1) or column-major (rs == 1).  Returns -1 if the layout is not covered.
int zgemm_tc(int64_t m, int64_t n, int64_t k, double2 alpha, const void* a, int64_t a_rs, int64_t a_cs, int64_t a_bs,
             const void* b, int64_t b_rs, int64_t b_cs, int64_t b_bs, double2 beta, void* c, int64_t c_rs,
             int64_t c_cs, int64_t c_bs, int64_t batch, cudaStream_t s) {
  using RM = cutlass::layout::RowMajor;
  using CM = cutlass::layout::ColumnMajor;
  const bool a_row = (a_cs == 1), a_col = (a_rs == 1);
  const bool b_row = (b_cs == 1), b_col = (b_rs == 1);
  const bool c_row = (c_cs == 1), c_col = (c_rs == 1);
  if (m > INT32_MAX || n > INT32_MAX || k > INT32_MAX || batch > INT32_MAX) return -1;
  if (a_col && b_row && c_row)
    return run<ZGemm<CM, RM, RM>>(m, n, k, alpha, a, a_cs, a_bs, b, b_rs, b_bs, beta, c, c_rs, c_bs, batch, s);
  if (a_row && b_col && c_col)
    return run<ZGemm<RM, CM, CM>>(m, n, k, alpha, a, a_rs, a_bs, b, b_cs, b_bs, beta, c, c_cs, c_bs, batch, s);
  if (a_row && b_row && c_row)
    return run<ZGemm<RM, RM, RM>>(m, n, k, alpha, a, a_rs, a_bs, b, b_rs, b_bs, beta, c, c_rs, c_bs, batch, s);
  return -1;
}

}  // namespace toep
