// FP64 per-bin products of the multi-RHS matvec on the INT8 tensor cores (Ozaki scheme).
//
// sm_100a has no FP64 kind of tcgen05.mma; the FP64 DMMA pipe (mma.sync) peaks near 32 TFLOP/s at
// the clocks the cfg3 products run at.  The int8 kind runs at ~4 POPS.  The Ozaki splitting makes
// an FP64 product exact-enough out of int8 products:
//   * every row i of A and column j of B is scaled by a power of two (exponents e_i, f_j) into
//     (-1, 1) and cut into S = 7 signed base-128 digits, x ~ sum_p a_p 2^(-7p) with |a_p| <= 127
//     (the digits of |round(x 2^49)|, sign applied to each);
//   * C_ij = 2^(e_i + f_j) sum_{t=2..S+1} 2^(-7t) G_t,  G_t = sum_{p+q=t} (A_p B_q)_ij  — the
//     28 slice products with p + q <= S + 1 (the dropped ones are below 2^-56 relative);
//   * every G_t is an exact int32 sum (|G_t| <= 7 * K * 127^2 < 2^31 for K <= 2048) accumulated in
//     TMEM; one epilogue per output tile combines the seven groups in FP64.
// The complex product D_k U_k is the real block product [Dr -Di; Di Dr] [Ur; Ui] (M = K = 2 n0).
//
// Kernel (ozaki_tile_kernel): one CTA per (bin, 128-row tile), walking the 64-column tiles of
// the right-hand sides; warp 0 lane 0 streams the A / B slice tiles of each 64-deep K chunk
// into a 2-stage shared-memory ring with bulk copies (TMA engine), warp 1 lane 0 issues the 56
// tcgen05.mma.kind::i8 (M=128, N=64, K=32) of a chunk into the seven TMEM accumulators (7 x 64 of
// the 512 columns), and all four warps run the epilogue (tcgen05.ld of the seven groups, FP64
// combination, 2^(e_i + f_j) scaling, stores into the Re / Im output planes).
//
// Slice layouts are the no-swizzle K-major "core matrix" layout of the UMMA descriptors (8 rows x
// 16 bytes per core matrix; adjacent K core matrices 128 B apart, adjacent 8-row groups
// (kBK / 16) * 128 B apart), stored in global memory exactly as one stage of shared memory wants them so that each
// stage is two contiguous bulk copies.
#include <cstdlib>

#include "kernels.cuh"
#include "launch.cuh"
#include "tma.cuh"

namespace toep {

namespace {

constexpr int kS = 7;            // slices per operand
constexpr int kBM = 128;         // rows per tile
constexpr int kBN = 128;         // columns per tile
constexpr int kBK = 32;          // K bytes per stage
constexpr int kATile = kS * kBM * kBK;  // 28 672 B
constexpr int kBTile = kS * kBN * kBK;  // 28 672 B
constexpr int kStages = 3;
constexpr int kOzThreads = 256;  // 8 warps: warp w reads TMEM lane quarter w % 4, column half w / 4

// element offset of (row, kk) inside one slice of a [g][c][r][16] tile (kk < kBK)
__device__ __forceinline__ int core_off(int row, int kk) {
  return (((row >> 3) * (kBK / 16) + (kk >> 4)) * 8 + (row & 7)) * 16 + (kk & 15);
}

__device__ __forceinline__ int row_exponent(double mx) {
  if (!(mx > 0.0)) return 0;
  return ilogb(mx) + 1;  // mx * 2^-e in [0.5, 1)
}

// 16 values (already scaled by 2^(49 - e)) -> kS int4 slices of signed base-128 digits.  The
// 49-bit magnitude is split into 32-bit halves (digits 0-2 from bits 28-48, 3-6 from bits 0-27) so
// every digit is one 32-bit shift-and (the kernel is ALU-bound on the 64-bit shifts otherwise);
// the sign is applied as (d ^ s) - s with s = 0 / -1.
__device__ __forceinline__ void digits16(const double* x, int4* out) {
  uint32_t hi[16], lo[16], sg[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    // round to nearest (unbiased truncation error, unlike chopping); |x| < 2^49 so |t| <= 2^49, and
    // the one value that can round up to 2^49 is clamped to the largest 7-digit magnitude
    const int64_t t = __double2ll_rn(x[i]);
    const int64_t a0 = t < 0 ? -t : t;
    const int64_t a = a0 < (int64_t{1} << (7 * kS)) ? a0 : (int64_t{1} << (7 * kS)) - 1;
    hi[i] = static_cast<uint32_t>(a >> 28);
    lo[i] = static_cast<uint32_t>(a) & ((1u << 28) - 1u);
    sg[i] = t < 0 ? 0xffffffffu : 0u;
  }
  static_assert(kS == 7, "digit split assumes 7 base-128 digits");
#pragma unroll
  for (int p = 0; p < kS; ++p) {
    uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint32_t d = p < 3 ? (hi[i] >> (7 * (2 - p))) & 127u : (lo[i] >> (7 * (6 - p))) & 127u;
      w[i >> 2] |= (((d ^ sg[i]) - sg[i]) & 0xffu) << (8 * (i & 3));
    }
    out[p] = make_int4(static_cast<int>(w[0]), static_cast<int>(w[1]), static_cast<int>(w[2]), static_cast<int>(w[3]));
  }
}

// ---- A side (operator, once): rows i of [Dr -Di; Di Dr] for every bin (kx-major bin order b =
// kx * l2 + ky), D_k[m][j] = DT[k][j][m].  One CTA per (bin, 128-row tile); thread = row.
__global__ void __launch_bounds__(kBM) ozaki_slice_a_kernel(const double2* __restrict__ DT, int n0, int l2, int l1,
                                                            int8_t* __restrict__ asl, int32_t* __restrict__ aexp) {
  const int b = blockIdx.x, mt = blockIdx.y;
  const int kx = b / l2, ky = b - kx * l2;
  const int64_t k = static_cast<int64_t>(ky) * l1 + kx;
  const double2* D = DT + k * n0 * n0;  // D[m][j] = D[j * n0 + m]
  const int i = mt * kBM + threadIdx.x;  // row of the 2 n0 block matrix
  const int m = i < n0 ? i : i - n0;
  const int kdim = 2 * n0;
  // row i: i < n0 -> [Dr[m][.], -Di[m][.]]; i >= n0 -> [Di[m][.], Dr[m][.]]
  auto val = [&](int kk) -> double {
    const double2 d = D[static_cast<int64_t>(kk < n0 ? kk : kk - n0) * n0 + m];
    if (i < n0) return kk < n0 ? d.x : -d.y;
    return kk < n0 ? d.y : d.x;
  };
  double mx = 0.0;
  for (int kk = 0; kk < kdim; ++kk) mx = fmax(mx, fabs(val(kk)));
  const int e = row_exponent(mx);
  aexp[static_cast<int64_t>(b) * kdim + i] = e;
  const int kcs = kdim / kBK;
  int8_t* base = asl + (static_cast<int64_t>(b) * (kdim / kBM) + mt) * kcs * kATile;
  const double sc = ldexp(1.0, 7 * kS - e);
  for (int kk0 = 0; kk0 < kdim; kk0 += 16) {
    double x[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) x[q] = val(kk0 + q) * sc;
    int4 sl[kS];
    digits16(x, sl);
    int8_t* t = base + static_cast<int64_t>(kk0 / kBK) * kATile;
#pragma unroll
    for (int p = 0; p < kS; ++p)
      *reinterpret_cast<int4*>(t + p * (kBM * kBK) + core_off(threadIdx.x, kk0 % kBK)) = sl[p];
  }
}

// ---- B side (per matvec chunk): column j of [Ur; Ui] for every bin of the chunk, read from the
// Re / Im planes (bin b: [e][j] row-major, w columns).  One CTA per (bin, 16-column group): the
// 2 n0 x 16 tile is staged in shared memory with cp.async (read once), column maxima are reduced
// there, and the slices are cut with integer arithmetic (digits16).
constexpr int kSliceCols = 16;
constexpr int kSliceThreads = 256;

__device__ __forceinline__ void cp_async8(void* smem, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(g) : "memory");
}

__global__ void __launch_bounds__(kSliceThreads) ozaki_slice_b_kernel(const double* __restrict__ re,
                                                                      const double* __restrict__ im, int n0, int64_t w,
                                                                      int ntiles, int8_t* __restrict__ bsl,
                                                                      int32_t* __restrict__ bexp) {
  extern __shared__ __align__(16) double tile[];  // [2 n0][kSliceCols]
  __shared__ double pmax[kSliceThreads / kSliceCols][kSliceCols];
  __shared__ double cscale[kSliceCols];
  const int b = blockIdx.y;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * kSliceCols;
  const int kdim = 2 * n0;
  const double* R = re + static_cast<int64_t>(b) * n0 * w;
  const double* I = im + static_cast<int64_t>(b) * n0 * w;
  const int tid = threadIdx.x, jl = tid % kSliceCols, part = tid / kSliceCols;
  if ((w & 1) == 0) {  // 16-byte copies: 8 threads per K row, two columns each
    const int jp = 2 * (tid & 7);
    const bool live2 = j0 + jp < w;  // w even: both columns live or both dead
    for (int kk = tid >> 3; kk < kdim; kk += kSliceThreads / 8) {
      double* dst = tile + kk * kSliceCols + jp;
      const double* src = (kk < n0 ? R + static_cast<int64_t>(kk) * w : I + static_cast<int64_t>(kk - n0) * w) + j0 + jp;
      if (live2) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
      } else {
        dst[0] = 0.0;
        dst[1] = 0.0;
      }
    }
  } else {
    const bool live = j0 + jl < w;
    for (int kk = part; kk < kdim; kk += kSliceThreads / kSliceCols) {
      double* dst = tile + kk * kSliceCols + jl;
      if (live) cp_async8(dst, (kk < n0 ? R + static_cast<int64_t>(kk) * w : I + static_cast<int64_t>(kk - n0) * w) + j0 + jl);
      else *dst = 0.0;
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  double mx = 0.0;
  for (int kk = part; kk < kdim; kk += kSliceThreads / kSliceCols) mx = fmax(mx, fabs(tile[kk * kSliceCols + jl]));
  pmax[part][jl] = mx;
  __syncthreads();
  if (tid < kSliceCols) {
    double m2 = 0.0;
    for (int p = 0; p < kSliceThreads / kSliceCols; ++p) m2 = fmax(m2, pmax[p][tid]);
    const int e = row_exponent(m2);
    const int64_t jg = j0 + tid;
    const int nt = static_cast<int>(jg / kBN);
    bexp[(static_cast<int64_t>(b) * ntiles + nt) * kBN + (jg % kBN)] = e;
    cscale[tid] = ldexp(1.0, 7 * kS - e);  // x 2^-e 2^49
  }
  __syncthreads();
  const int kcs = kdim / kBK;
  const double sc = cscale[jl];
  const int64_t jg = j0 + jl;
  const int nt = static_cast<int>(jg / kBN), jt = static_cast<int>(jg % kBN);
  int8_t* base = bsl + (static_cast<int64_t>(b) * ntiles + nt) * kcs * kBTile;
  for (int kk0 = part * 16; kk0 < kdim; kk0 += 16 * (kSliceThreads / kSliceCols)) {
    double x[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) x[q] = tile[(kk0 + q) * kSliceCols + jl] * sc;
    int4 sl[kS];
    digits16(x, sl);
    int8_t* t = base + static_cast<int64_t>(kk0 / kBK) * kBTile;
#pragma unroll
    for (int p = 0; p < kS; ++p) *reinterpret_cast<int4*>(t + p * (kBN * kBK) + core_off(jt, kk0 % kBK)) = sl[p];
  }
}

// ---- tcgen05 helpers
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  // no-swizzle K-major: LBO 128 B (next K core matrix), SBO (kBK / 16) * 128 B (next 8-row group),
  // descriptor version 1
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3fff);
  d |= static_cast<uint64_t>(128 >> 4) << 16;
  d |= static_cast<uint64_t>(((kBK / 16) * 128) >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  return d;
}
// kind::i8, D s32, A / B signed, K-major, N = 64, M = 128
constexpr uint32_t kIdescBase = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kBM >> 4) << 24);
__host__ __device__ constexpr uint32_t idesc_n(int n) { return kIdescBase | (static_cast<uint32_t>(n >> 3) << 17); }

__device__ __forceinline__ void mma_i8(uint32_t tmem, uint64_t da, uint64_t db, uint32_t acc, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

struct OzArgs {
  const int8_t* asl;   // A slices of the chunk's first bin
  const int32_t* aexp;
  const int8_t* bsl;
  const int32_t* bexp;
  double* out_re;      // [bin][n0][w]
  double* out_im;
  int n0;
  int64_t w;
  int ntiles;
};

// Groups t = 2..8 do not fit TMEM side by side at N = 128 (7 x 128 columns), so every column tile
// runs two phases over K: phase 0 accumulates t = 2..5 (4 x 128 columns, digits 1..4 only) into the
// exact integer G2 2^21 + G3 2^14 + G4 2^7 + G5, kept in registers; phase 1 accumulates t = 6..8,
// adds 2^-56 (G6 2^14 + G7 2^7 + G8) to 2^-35 times it, scales and stores.  N = 128 halves the shared-memory operand reads per MAC of the
// N = 64 single-phase tile (the tensor core's smem bandwidth is what bounds N = 64).
__device__ __forceinline__ int phase_slices(int ph) { return ph == 0 ? 4 : kS; }

__global__ void __launch_bounds__(kOzThreads, 1) ozaki_tile_kernel(OzArgs a) {
  extern __shared__ __align__(1024) unsigned char oz_smem[];
  int8_t* sA = reinterpret_cast<int8_t*>(oz_smem);              // [kStages][kATile]
  int8_t* sB = sA + kStages * kATile;                            // [kStages][kBTile]
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], tfull;
  __shared__ uint32_t tmem_base;
  __shared__ double scol[kBN];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = blockIdx.y, mt = blockIdx.x;  // the row tiles of one bin run together (B tiles reused from L2)
  const int kdim = 2 * a.n0, kcs = kdim / kBK, mtiles = kdim / kBM;
  const int nt_count = a.ntiles;
  const int total = nt_count * 2 * kcs;  // steps: (column tile, phase, K chunk)
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull, 1);
    mbar_init_fence();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const int8_t* Ab = a.asl + (static_cast<int64_t>(b) * mtiles + mt) * kcs * kATile;
  const int8_t* Bb = a.bsl + static_cast<int64_t>(b) * nt_count * kcs * kBTile;
  const int quarter = warp & 3, chalf = warp >> 2;
  const int row = mt * kBM + quarter * 32 + lane;  // this thread's output row (epilogue)
  const double srow = ldexp(1.0, a.aexp[static_cast<int64_t>(b) * kdim + row]);
  double* orow = (row < a.n0 ? a.out_re + (static_cast<int64_t>(b) * a.n0 + row) * a.w
                             : a.out_im + (static_cast<int64_t>(b) * a.n0 + row - a.n0) * a.w);
  const uint64_t pol = policy_evict_last();
  int issued = 0;  // producer: next step to load
  auto produce_until = [&](int limit) {
    for (; issued < limit && issued < total; ++issued) {
      const int st = issued % kStages;
      if (issued >= kStages) mbar_wait(&empty[st], ((issued / kStages) - 1) & 1);
      const int tp = issued / kcs, kc = issued - tp * kcs;  // tp = nt * 2 + phase
      const int nt = tp >> 1;
      const uint32_t bytes = static_cast<uint32_t>(phase_slices(tp & 1)) * (kBM * kBK);  // kBM == kBN
      mbar_expect_tx(&full[st], 2 * bytes);
      bulk_g2s(sA + st * kATile, Ab + static_cast<int64_t>(kc) * kATile, bytes, &full[st], pol);
      bulk_g2s(sB + st * kBTile, Bb + (static_cast<int64_t>(nt) * kcs + kc) * kBTile, bytes, &full[st], pol);
    }
  };
  const bool vec = (a.w & 1) == 0;
  double part[kBN / 2];  // per-thread partial sums of its 64 output columns (registers)
  for (int nt = 0; nt < nt_count; ++nt) {
    const int32_t* fe = a.bexp + (static_cast<int64_t>(b) * nt_count + nt) * kBN;
    if (tid < kBN) scol[tid] = ldexp(1.0, __ldg(fe + tid));  // read after the phase-0 barrier below
    for (int ph = 0; ph < 2; ++ph) {
      const int tp = nt * 2 + ph;
      if (warp == 0 && lane == 0) produce_until((tp + 1) * kcs);
      if (warp == 1 && lane == 0) {
        // the last column tile runs the narrowest N (multiple of 16 for M = 128) covering its live columns
        const int64_t live = a.w - static_cast<int64_t>(nt) * kBN;
        const uint32_t idesc = idesc_n(live >= kBN ? kBN : static_cast<int>((live + 15) / 16) * 16);
        for (int kc = 0; kc < kcs; ++kc) {
          const int step = tp * kcs + kc, st = step % kStages;
          mbar_wait(&full[st], (step / kStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a0 = smem_u32(sA + st * kATile), b0 = smem_u32(sB + st * kBTile);
          if (ph == 0) {
#pragma unroll
            for (int p = 1; p <= 4; ++p) {
#pragma unroll
              for (int q = 1; p + q <= 5; ++q)
                mma_i8(tmem + static_cast<uint32_t>((p + q - 2) * kBN),
                       umma_desc(a0 + (p - 1) * (kBM * kBK)), umma_desc(b0 + (q - 1) * (kBN * kBK)),
                       (kc > 0 || p > 1) ? 1u : 0u, idesc);
            }
          } else {
#pragma unroll
            for (int p = 1; p <= kS; ++p) {
#pragma unroll
              for (int q = (6 - p > 1 ? 6 - p : 1); p + q <= kS + 1; ++q)
                mma_i8(tmem + static_cast<uint32_t>((p + q - 6) * kBN),
                       umma_desc(a0 + (p - 1) * (kBM * kBK)), umma_desc(b0 + (q - 1) * (kBN * kBK)),
                       (kc > 0 || p > 1) ? 1u : 0u, idesc);
            }
          }
          umma_commit(&empty[st]);  // smem slot free once these MMAs have read it
        }
        umma_commit(&tfull);        // this phase's accumulators complete
      }
      // the producer runs ahead into the next phase before joining the epilogue
      if (warp == 0 && lane == 0) produce_until((tp + 1) * kcs + kStages);
      __syncwarp();
      mbar_wait(&tfull, tp & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      __syncthreads();  // scol visible
      const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
      {
        // this thread's 64 columns: the phase-0 partial stays in registers until phase 1 completes it
#pragma unroll
        for (int ci = 0; ci < kBN / 32; ++ci) {
          const int cc = chalf * (kBN / 32) + ci;
          if (static_cast<int64_t>(nt) * kBN + cc * 16 >= a.w) break;  // beyond the live columns (warp-uniform)
          uint32_t v[4][16];
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            if (ph == 1 && g == 3) break;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(v[g][0]), "=r"(v[g][1]), "=r"(v[g][2]), "=r"(v[g][3]), "=r"(v[g][4]), "=r"(v[g][5]),
                  "=r"(v[g][6]), "=r"(v[g][7]), "=r"(v[g][8]), "=r"(v[g][9]), "=r"(v[g][10]), "=r"(v[g][11]),
                  "=r"(v[g][12]), "=r"(v[g][13]), "=r"(v[g][14]), "=r"(v[g][15])
                : "r"(lane_base + static_cast<uint32_t>(g * kBN + cc * 16)));
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            auto G = [&](int g) { return static_cast<int64_t>(static_cast<int32_t>(v[g][jj])); };
            if (ph == 0) {
              part[ci * 16 + jj] = static_cast<double>((G(0) << 21) + (G(1) << 14) + (G(2) << 7) + G(3));
            } else {
              part[ci * 16 + jj] =
                  fma(part[ci * 16 + jj], 0x1p-35, static_cast<double>((G(0) << 14) + (G(1) << 7) + G(2)) * 0x1p-56);
            }
          }
        }
        if (ph == 1) {
#pragma unroll
          for (int ci = 0; ci < kBN / 32; ++ci) {
            const int cc = chalf * (kBN / 32) + ci;
            const int64_t j0 = static_cast<int64_t>(nt) * kBN + cc * 16;
            double o[16];
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) o[jj] = part[ci * 16 + jj] * srow * scol[cc * 16 + jj];
            if (vec && j0 + 16 <= a.w) {
#pragma unroll
              for (int jj = 0; jj < 16; jj += 2)
                *reinterpret_cast<double2*>(orow + j0 + jj) = make_double2(o[jj], o[jj + 1]);
            } else {
#pragma unroll
              for (int jj = 0; jj < 16; ++jj)
                if (j0 + jj < a.w) orow[j0 + jj] = o[jj];
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();  // TMEM free for the next phase
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace

bool ozaki_supported(int n0) { return n0 >= 64 && (2 * n0) % kBM == 0 && 2 * n0 <= 1024; }

int64_t ozaki_a_bytes(int n0, int64_t K) { return K * 4 * static_cast<int64_t>(n0) * n0 * kS; }
int64_t ozaki_b_bytes(int n0, int64_t bins, int64_t w) {
  return bins * ((w + kBN - 1) / kBN) * (2 * static_cast<int64_t>(n0) / kBK) * kBTile;
}
int64_t ozaki_b_exps(int64_t bins, int64_t w) { return bins * ((w + kBN - 1) / kBN) * kBN; }

int ozaki_slice_a(const void* DT, int n0, int l2, int l1, int8_t* asl, int32_t* aexp, cudaStream_t s) {
  TOEP_REQUIRE(ozaki_supported(n0), TOEP_ERR_ARG, "ozaki: unsupported block side %d", n0);
  dim3 grid(static_cast<unsigned>(static_cast<int64_t>(l2) * l1), static_cast<unsigned>(2 * n0 / kBM));
  ozaki_slice_a_kernel<<<grid, kBM, 0, s>>>(static_cast<const double2*>(DT), n0, l2, l1, asl, aexp);
  TOEP_LAUNCHED();
  return TOEP_OK;
}

int ozaki_products(const int8_t* asl, const int32_t* aexp, const double* re, const double* im, int n0, int64_t bins,
                   int64_t w, int8_t* bsl, int32_t* bexp, double* out_re, double* out_im, cudaStream_t s) {
  TOEP_REQUIRE(ozaki_supported(n0), TOEP_ERR_ARG, "ozaki: unsupported block side %d", n0);
  if (bins == 0 || w == 0) return TOEP_OK;
  const int ntiles = static_cast<int>((w + kBN - 1) / kBN);
  const size_t tsm = static_cast<size_t>(2 * n0) * kSliceCols * sizeof(double);
  TOEP_CUDA(ensure_smem(ozaki_slice_b_kernel, tsm));
  const size_t smem = kStages * (kATile + kBTile);
  TOEP_CUDA(ensure_smem(ozaki_tile_kernel, smem));
  const int64_t wpad = static_cast<int64_t>(ntiles) * kBN;
  const int64_t a_bin = ozaki_a_bytes(n0, 1), b_bin = ozaki_b_bytes(n0, 1, w), plane_bin = static_cast<int64_t>(n0) * w;
  for (int64_t b0 = 0; b0 < bins; b0 += 65535) {  // grid.y limit
    const unsigned nb = static_cast<unsigned>(std::min<int64_t>(65535, bins - b0));
    // digits of the right-hand sides (padded columns get zero digits / exponents every call)
    ozaki_slice_b_kernel<<<dim3(static_cast<unsigned>((wpad + kSliceCols - 1) / kSliceCols), nb), kSliceThreads, tsm,
                           s>>>(re + b0 * plane_bin, im + b0 * plane_bin, n0, w, ntiles, bsl + b0 * b_bin,
                                bexp + b0 * wpad);
    TOEP_LAUNCHED();
    OzArgs oa{asl + b0 * a_bin, aexp + b0 * 2 * n0, bsl + b0 * b_bin, bexp + b0 * wpad, out_re + b0 * plane_bin,
              out_im + b0 * plane_bin, n0, w, ntiles};
    ozaki_tile_kernel<<<dim3(static_cast<unsigned>(2 * n0 / kBM), nb), kOzThreads, smem, s>>>(oa);
    TOEP_LAUNCHED();
  }
  return TOEP_OK;
}

}  // namespace toep
