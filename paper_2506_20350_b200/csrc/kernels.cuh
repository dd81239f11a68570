// Internal kernel launchers of libtoepcuda (not part of the C ABI).
#pragma once

#include "common.cuh"

namespace toep {

// ------------------------------------------------------------------ FFT pass
// One batched 1-D DFT of length L along an "axis" of a strided array whose
// innermost ("batch") dimension of length `inner` is contiguous:
//   element (outer o, axis a, batch i) at base + o*so + a*sa + i.
// Input placement fuses the circulant embedding / pad_rhs (toeplitz.py:256-269):
//   slot s in [0, n_lo)        <- input row s
//   slot s in [L-n_hi, L)      <- input row n_lo + s - (L - n_hi)
//   all other slots            <- 0
// Only outputs 0..n_out-1 are stored (extract_result crop, toeplitz.py:272-284),
// each multiplied by `scale`.  sign = -1 forward (np.fft.fft), +1 inverse.
struct PassArgs {
  const void* in = nullptr;
  void* out = nullptr;
  int L = 1, n_lo = 0, n_hi = 0, n_out = 0;
  int64_t inner = 0;
  int64_t in_sa = 0, in_so = 0, out_sa = 0, out_so = 0;
  int outer = 1;
  int sign = -1;
  double scale = 1.0;
  // optional device-side offsets (GMRES basis indexing inside one launch sequence)
  const int* in_idx = nullptr;
  int64_t in_idx_stride = 0;
  const int* out_idx = nullptr;
  int64_t out_idx_stride = 0;
  const int* stop = nullptr;  // if non-null and *stop != 0 the launch is a no-op
  const double* in_scale = nullptr;  // optional device scalar multiplying the input
  // stride of the batch ("column") index; 1 = contiguous batch (all standalone passes)
  int64_t in_cs = 1, out_cs = 1;
  // optional split-plane I/O (3M products of the multi-RHS path): out_planes receives (re, im,
  // re+im) planes `plane` doubles apart instead of the complex output; in_planes supplies
  // (T1, T2, T3) planes combined into (T1 - T2) + i (T3 - T1 - T2).  Element indexing as for the
  // complex arrays (`in` / `out` must still be set: they anchor the element offsets).
  double* out_planes = nullptr;
  const double* in_planes = nullptr;
  int64_t plane = 0;
  int planes2 = 0;  // 1: (re, im) planes only — out: no re+im plane; in: (T1, T2) = (re, im) directly
  // optional peer scatter (toep_matvec_stage_peer): device table routing output index a to the
  // destination rank's receive buffer, plus the arrival signal after the launch's last store
  const toep_peer_scatter* scatter = nullptr;
};

// Whole 2-D transforms of the single-RHS matvec in one kernel each (one CTA per batch column,
// intermediate in shared memory): forward = pad + level-1 DFT + level-2 DFT -> u_hat (bin-major);
// inverse = inverse level-2 DFT (kept rows) + inverse level-1 DFT + crop + 1/(l1 l2).
// Returns -1 when no compiled 2-D plan covers (l2, l1, n2).
//
// `pf` (optional): while the transform runs, its CTAs prefetch into L2 the first `bytes` of each
// of the `ranges` contiguous bin ranges the streaming product kernel assigns to its CTAs, so the
// product's HBM stream effectively starts during the DFT.  The operator is constant, so the
// inverse transform of one matvec may prefetch for the next one.
struct L2Prefetch {
  const void* base = nullptr;
  int64_t bin_bytes = 0, K = 0, bytes = 0;
  int64_t skip = 0;  // start this many bytes into every range
  int ranges = 0;
};

// one warp of each of `ncta` CTAs issues the bulk L2 prefetches of its share of the ranges
__device__ __forceinline__ void l2_prefetch_heads(const L2Prefetch& pf, int cta, int ncta, int lane) {
  if (pf.bytes <= 0) return;
  const int64_t per = pf.K / pf.ranges, rem = pf.K % pf.ranges;
  constexpr int64_t kChunk = 32768;
  for (int c = cta; c < pf.ranges; c += ncta) {
    const int64_t b0 = c * per + (c < rem ? c : rem);
    const char* p0 = static_cast<const char*>(pf.base) + b0 * pf.bin_bytes + pf.skip;
    for (int64_t o = static_cast<int64_t>(lane) * kChunk; o < pf.bytes; o += 32 * kChunk) {
      const uint32_t n = static_cast<uint32_t>(pf.bytes - o < kChunk ? pf.bytes - o : kChunk);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p0 + o), "r"(n) : "memory");
    }
  }
}
// fused forward DFT -> per-bin product -> inverse DFT (one cooperative launch) for the cfg2 shape;
// -1 when it does not apply (fft.cu)
int matvec_fused(const void* DT, int64_t K, int n2, int n1, int l2, int l1, int n0, const void* u, void* hat,
                 void* hat2, void* v, unsigned* bar, const double* in_scale, const int* stop, const L2Prefetch& pf,
                 cudaStream_t s);
int fft2d(bool inverse, const void* in, void* out, int n2, int n1, int l2, int l1, int64_t inner, int sign,
          int tin, int tc, int tout, const double* in_scale, const int* stop, cudaStream_t s,
          const L2Prefetch* pf = nullptr);

// L2 prefetch plan for the streaming bin product that follows a forward transform (w == 1)
// side: 0 = forward DFT (range heads), 1 = inverse DFT, 2 = GMRES orthogonalisation (the bytes
// after the forward DFT's share)
L2Prefetch binprod_prefetch_plan(int dtype, const void* DT, int64_t K, int n0, int side = 0);

// type codes: 0 = complex128, 1 = complex64
int fft_pass(const PassArgs& a, int tin, int tcomp, int tout, cudaStream_t s);
int factorize(int L, int* rad, int* nrad);

// --------------------------------------------------------------- bin product
// V_k = D_k U_k for k < K, D_k stored transposed: DT[k][j][m] = D_k[m][j].
// U, V: [K][n0][w].  transpose: V_k = D_k^T U_k.
int bin_product(int dtype, const void* DT, const void* U, void* V, int64_t K, int n0, int64_t w,
                bool transpose, const int* stop, cudaStream_t s);

// ---------------------------------------------------------------- GEMM
int gemm(int dtype, int64_t m, int64_t n, int64_t k, double2 alpha, const void* a, int64_t a_rs,
         int64_t a_cs, int64_t a_bs, const void* b, int64_t b_rs, int64_t b_cs, int64_t b_bs,
         double2 beta, void* c, int64_t c_rs, int64_t c_cs, int64_t c_bs, int64_t batch,
         cudaStream_t s, const int* stop = nullptr);

// Hand-written FP64 tensor-core (DMMA) GEMMs, batched (batch <= 65535), any operand with a unit
// stride in one dimension (dmma.cu); return -1 when the stride pattern is not covered
int zgemm_dmma(int64_t m, int64_t n, int64_t k, double2 alpha, const void* a, int64_t a_rs, int64_t a_cs, int64_t a_bs,
               const void* b, int64_t b_rs, int64_t b_cs, int64_t b_bs, double2 beta, void* c, int64_t c_rs,
               int64_t c_cs, int64_t c_bs, int64_t batch, cudaStream_t s, const int* stop);
int dgemm_dmma(int64_t m, int64_t n, int64_t k, double alpha, const double* a, int64_t a_rs, int64_t a_cs,
               int64_t a_bs, const double* b, int64_t b_rs, int64_t b_cs, int64_t b_bs, double beta, double* c,
               int64_t c_rs, int64_t c_cs, int64_t c_bs, int64_t batch, cudaStream_t s, const int* stop);
// `planes` (<= 3) real products of one shape / stride set in ONE launch (the 3M planes)
int dgemm_dmma_planes(int64_t m, int64_t n, int64_t k, double alpha, const double* const* a, int64_t a_rs,
                      int64_t a_cs, int64_t a_bs, const double* const* b, int64_t b_rs, int64_t b_cs, int64_t b_bs,
                      double beta, double* const* c, int64_t c_rs, int64_t c_cs, int64_t c_bs, int64_t batch,
                      int planes, cudaStream_t s, const int* stop);
// true when the compiled pass plan for length L supports split-plane I/O
bool fft_plan_has_planes(int L, int64_t inner);


// Ozaki-scheme FP64 per-bin products on the int8 tensor cores (ozaki.cu): operator slices once,
// then per chunk of bins: slice the (re, im) planes of U and write the (re, im) planes of D U
bool ozaki_supported(int n0);
// generic real GEMMs C_z (alpha*)= A_z B_z (+ beta C_z) on the int8 tensor cores (Ozaki scheme, 7 digits):
// A row digits (M % 128 == 0, per-row exponents over the whole sliced row), B column digits
struct OzGemm {
  const int8_t* asl; const int32_t* aexp; int64_t a_kcs, a_k0, a_z0, a_zo, a_zp;
  const int8_t* bsl; const int32_t* bexp; int64_t b_z0, b_zo, b_zp;
  double* c; int64_t ldc, c_zo, c_zp;
  double alpha, beta;
  int M, N; int64_t K; int planes, zcount;
};
int64_t ozaki_rows_bytes(int64_t M, int64_t K);
int64_t ozaki_cols_bytes(int64_t N, int64_t K);
int64_t ozaki_cols_exps(int64_t N);
int ozaki_slice_rows(const double* a, int64_t lda, int64_t a_bs, int64_t batch, int M, int64_t K, int8_t* asl,
                     int32_t* aexp, cudaStream_t s);
int ozaki_slice_cols(const double* b, int64_t ldb, int64_t b_bs, int64_t batch, int N, int64_t K, int8_t* bsl,
                     int32_t* bexp, cudaStream_t s);
int ozaki_gemm(const OzGemm& g, cudaStream_t s);
int64_t ozaki_a_bytes(int n0, int64_t K);
int64_t ozaki_b_bytes(int n0, int64_t bins, int64_t w);
int64_t ozaki_b_exps(int64_t bins, int64_t w);
int ozaki_slice_a(const void* DT, int n0, int l2, int l1, int8_t* asl, int32_t* aexp, cudaStream_t s);
int ozaki_products(const int8_t* asl, const int32_t* aexp, const double* re, const double* im, int n0, int64_t bins,
                   int64_t w, int8_t* bsl, int32_t* bexp, double* out_re, double* out_im, cudaStream_t s);

// batched transpose of complex matrices: out[b][c][r] = in[b][r][c]  (rows x cols)
int transpose_batched(int dtype, const void* in, void* out, int64_t batch, int rows, int cols, cudaStream_t s);

// embed / cast helpers
int cast_c128_to_c64(const void* in, void* out, int64_t n, cudaStream_t s);

}  // namespace toep
