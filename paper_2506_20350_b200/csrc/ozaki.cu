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
// Kernel (ozaki_tile_kernel): one CTA per (bin, 128-row tile), walking the 128-column tiles of
// the right-hand sides in two K phases each (groups t = 2..5, then 6..8: seven groups of 128
// columns do not fit the 512 TMEM columns); warp 0 lane 0 streams the A / B digit tiles of each
// 32-deep K step into a 3-stage shared-memory ring with bulk copies (TMA engine), warp 1 lane 0
// issues the 10 / 18 tcgen05.mma.kind::i8 (M=128, N=128, K=32) of a step, and all 16 warps run
// the two epilogues (tcgen05.ld of the phase's groups, exact integer combination -> FP64,
// 2^(e_i + f_j) scaling, stores into the Re / Im output planes).
//
// Slice layouts are the no-swizzle K-major "core matrix" layout of the UMMA descriptors (8 rows x
// 16 bytes per core matrix; adjacent K core matrices 128 B apart, adjacent 8-row groups
// (kBK / 16) * 128 B apart), stored in global memory exactly as one stage of shared memory wants them so that each
// stage is two contiguous bulk copies.
#include <cstdlib>

#include "../../include/toepcuda.h"
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
constexpr int kTileSlot = 65536;  // ozaki_tile_kernel ring slot: 32 KB per operand
constexpr int kOzThreads = 256;  // generic GEMM: 8 warps, warp w reads TMEM lane quarter w % 4, column half w / 4
// per-bin tile kernel: 16 warps (lane quarter w % 4, column quarter w / 4).  Its two epilogues per
// column tile are not amortised over a deep K, and 8 warps left them latency-bound: cfg3 matvec
// 45.0 ms with 256 threads, 43.4 ms with 512, 44.2-45.7 ms with 1024 (64-register cap, spills)
constexpr int kOzTileThreads = 512;

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

// TMEM -> registers: 8 consecutive 32-bit columns of this warp's lane quarter
__device__ __forceinline__ void tmem_ld8(uint32_t addr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(addr));
}

__global__ void __launch_bounds__(kOzTileThreads, 1) ozaki_tile_kernel(OzArgs a) {
  constexpr int kCpt = kBN / (kOzTileThreads / 128);  // columns per thread (32)
  constexpr int CW = 8;                               // columns per TMEM load
  constexpr int kChunks = kCpt / CW;
  extern __shared__ __align__(1024) unsigned char oz_smem[];
  int8_t* sA = reinterpret_cast<int8_t*>(oz_smem);              // [kStages][kTileSlot]: A half, then B half
  int8_t* sB = sA + kTileSlot / 2;
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], tfull;
  __shared__ uint32_t tmem_base;
  __shared__ double scol[kBN];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = blockIdx.y, mt = blockIdx.x;  // the row tiles of one bin run together (B tiles reused from L2)
  const int kdim = 2 * a.n0, kcs = kdim / kBK, mtiles = kdim / kBM;
  const int nt_count = a.ntiles;
  // ring steps per column tile: phase 0 moves two K chunks per step (4 digits each: 2 x 16 KB per
  // operand, so a step carries 64 KB like a phase-1 step's 56 KB -- with one chunk per step only
  // 64 KB were in flight during phase 0 and its MMAs waited on L2), phase 1 one chunk per step
  const int steps0 = kcs / 2, steps_tile = steps0 + kcs;
  const int total = nt_count * steps_tile;
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
  const int quarter = warp & 3, cgrp = warp >> 2;
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
      const int nt = issued / steps_tile, r = issued - nt * steps_tile;
      int8_t* da = sA + st * kTileSlot;
      int8_t* db = sB + st * kTileSlot;
      const int8_t* gb = Bb + static_cast<int64_t>(nt) * kcs * kBTile;
      if (r < steps0) {
        constexpr uint32_t bytes = 4 * (kBM * kBK);  // digits 1..4 of one K chunk
        const int kc = 2 * r;
        mbar_expect_tx(&full[st], 4 * bytes);
        bulk_g2s(da, Ab + static_cast<int64_t>(kc) * kATile, bytes, &full[st], pol);
        bulk_g2s(da + bytes, Ab + static_cast<int64_t>(kc + 1) * kATile, bytes, &full[st], pol);
        bulk_g2s(db, gb + static_cast<int64_t>(kc) * kBTile, bytes, &full[st], pol);
        bulk_g2s(db + bytes, gb + static_cast<int64_t>(kc + 1) * kBTile, bytes, &full[st], pol);
      } else {
        const int kc = r - steps0;
        mbar_expect_tx(&full[st], kATile + kBTile);
        bulk_g2s(da, Ab + static_cast<int64_t>(kc) * kATile, kATile, &full[st], pol);
        bulk_g2s(db, gb + static_cast<int64_t>(kc) * kBTile, kBTile, &full[st], pol);
      }
    }
  };
  const bool vec = (a.w & 1) == 0;
  double part[kCpt];  // per-thread partial sums of its output columns (registers)
  for (int nt = 0; nt < nt_count; ++nt) {
    const int32_t* fe = a.bexp + (static_cast<int64_t>(b) * nt_count + nt) * kBN;
    if (tid < kBN) scol[tid] = ldexp(1.0, __ldg(fe + tid));  // read after the phase-0 barrier below
    for (int ph = 0; ph < 2; ++ph) {
      const int tp = nt * 2 + ph;
      const int step0 = nt * steps_tile + (ph ? steps0 : 0), nsteps = ph ? kcs : steps0;
      if (warp == 0 && lane == 0) produce_until(step0 + nsteps);
      if (warp == 1 && lane == 0) {
        // the last column tile runs the narrowest N (multiple of 16 for M = 128) covering its live columns
        const int64_t live = a.w - static_cast<int64_t>(nt) * kBN;
        const uint32_t idesc = idesc_n(live >= kBN ? kBN : static_cast<int>((live + 15) / 16) * 16);
        for (int i = 0; i < nsteps; ++i) {
          const int step = step0 + i, st = step % kStages;
          mbar_wait(&full[st], (step / kStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a0 = smem_u32(sA + st * kTileSlot), b0 = smem_u32(sB + st * kTileSlot);
          if (ph == 0) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t ah = a0 + h * 4 * (kBM * kBK), bh = b0 + h * 4 * (kBN * kBK);
#pragma unroll
              for (int p = 1; p <= 4; ++p) {
#pragma unroll
                for (int q = 1; p + q <= 5; ++q)
                  mma_i8(tmem + static_cast<uint32_t>((p + q - 2) * kBN), umma_desc(ah + (p - 1) * (kBM * kBK)),
                         umma_desc(bh + (q - 1) * (kBN * kBK)), (i > 0 || h > 0 || p > 1) ? 1u : 0u, idesc);
              }
            }
          } else {
#pragma unroll
            for (int p = 1; p <= kS; ++p) {
#pragma unroll
              for (int q = (6 - p > 1 ? 6 - p : 1); p + q <= kS + 1; ++q)
                mma_i8(tmem + static_cast<uint32_t>((p + q - 6) * kBN),
                       umma_desc(a0 + (p - 1) * (kBM * kBK)), umma_desc(b0 + (q - 1) * (kBN * kBK)),
                       (i > 0 || p > 1) ? 1u : 0u, idesc);
            }
          }
          umma_commit(&empty[st]);  // smem slot free once these MMAs have read it
        }
        umma_commit(&tfull);        // this phase's accumulators complete
      }
      // the producer runs ahead into the next phase before joining the epilogue
      if (warp == 0 && lane == 0) produce_until(step0 + nsteps + kStages);
      __syncwarp();
      mbar_wait(&tfull, tp & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      __syncthreads();  // scol visible
      const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
      {
        // this thread's columns: the phase-0 partial stays in registers until phase 1 completes it
#pragma unroll
        for (int ci = 0; ci < kChunks; ++ci) {
          const int c0 = cgrp * kCpt + ci * CW;  // first column of the chunk inside the tile
          if (static_cast<int64_t>(nt) * kBN + c0 >= a.w) break;  // beyond the live columns (warp-uniform)
          uint32_t v[4][CW];
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            if (ph == 1 && g == 3) break;
            tmem_ld8(lane_base + static_cast<uint32_t>(g * kBN + c0), v[g]);
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int jj = 0; jj < CW; ++jj) {
            auto G = [&](int g) { return static_cast<int64_t>(static_cast<int32_t>(v[g][jj])); };
            if (ph == 0) {
              part[ci * CW + jj] = static_cast<double>((G(0) << 21) + (G(1) << 14) + (G(2) << 7) + G(3));
            } else {
              part[ci * CW + jj] =
                  fma(part[ci * CW + jj], 0x1p-35, static_cast<double>((G(0) << 14) + (G(1) << 7) + G(2)) * 0x1p-56);
            }
          }
        }
        if (ph == 1) {
#pragma unroll
          for (int ci = 0; ci < kChunks; ++ci) {
            const int c0 = cgrp * kCpt + ci * CW;
            const int64_t j0 = static_cast<int64_t>(nt) * kBN + c0;
            double o[CW];
#pragma unroll
            for (int jj = 0; jj < CW; ++jj) o[jj] = part[ci * CW + jj] * srow * scol[c0 + jj];
            if (vec && j0 + CW <= a.w) {
#pragma unroll
              for (int jj = 0; jj < CW; jj += 2)
                *reinterpret_cast<double2*>(orow + j0 + jj) = make_double2(o[jj], o[jj + 1]);
            } else {
#pragma unroll
              for (int jj = 0; jj < CW; ++jj)
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

// ------------------------------------------------------------------------------------------
// Generic real GEMM on the int8 tensor cores (Ozaki scheme), for the Rybicki block sums:
// C_z (alpha *)= A_z B_z with A (M x K, row-major) cut into row digits [za][mt][kc] (per-row
// exponents over the whole row, so a GEMM may use any 32-aligned K sub-range of a sliced matrix),
// B (K x N, row-major) cut into column digits [zb][nt][kc] (per-column exponents over its K).
// One CTA per (128-row tile, 128-column tile, batch z x K split): the same two-phase MMA / epilogue
// as ozaki_tile_kernel.  Split partials go to `work` and are summed in a fixed order by
// ozaki_split_reduce.

// A digits: grid (M/128, kcs, batch); thread = row; 32 consecutive k of its row per CTA
__global__ void __launch_bounds__(kBM) ozaki_rows_slice_kernel(const double* __restrict__ a, int64_t lda,
                                                               int64_t a_bs, int M, int64_t kcs,
                                                               const int32_t* __restrict__ aexp, int8_t* __restrict__ asl) {
  const int mt = blockIdx.x, z = blockIdx.z;
  const int64_t kc = blockIdx.y;
  const int row = mt * kBM + threadIdx.x;
  const double* src = a + z * a_bs + static_cast<int64_t>(row) * lda + kc * kBK;
  const double sc = ldexp(1.0, 7 * kS - aexp[static_cast<int64_t>(z) * M + row]);
  int8_t* t = asl + ((static_cast<int64_t>(z) * (M / kBM) + mt) * kcs + kc) * kATile;
#pragma unroll
  for (int h = 0; h < kBK / 16; ++h) {
    double x[16];
    const double2* s2 = reinterpret_cast<const double2*>(src + h * 16);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double2 v = __ldg(s2 + q);
      x[2 * q] = v.x * sc;
      x[2 * q + 1] = v.y * sc;
    }
    int4 sl[kS];
    digits16(x, sl);
#pragma unroll
    for (int p = 0; p < kS; ++p)
      *reinterpret_cast<int4*>(t + p * (kBM * kBK) + core_off(threadIdx.x, h * 16)) = sl[p];
  }
}

// row exponents of A: one warp per row, max |a| over the row's K entries
__global__ void ozaki_rows_exp_kernel(const double* __restrict__ a, int64_t lda, int64_t a_bs, int M, int64_t K,
                                      int32_t* __restrict__ aexp) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int z = blockIdx.y;
  if (warp >= M) return;
  const double* src = a + z * a_bs + static_cast<int64_t>(warp) * lda;
  double mx = 0.0;
  for (int64_t k = lane; k < K; k += 32) mx = fmax(mx, fabs(__ldg(src + k)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) aexp[static_cast<int64_t>(z) * M + warp] = row_exponent(mx);
}

// column exponents of B (K x N row-major): grid (ntiles, kparts, batch), thread = column; the
// exponent of the max is the max of the exponents, so parts combine with atomicMax (bexp zeroed)
__global__ void __launch_bounds__(kBN) ozaki_cols_exp_kernel(const double* __restrict__ b, int64_t ldb, int64_t b_bs,
                                                            int N, int64_t K, int ntiles, int64_t rows_per_part,
                                                            int32_t* __restrict__ bexp) {
  const int nt = blockIdx.x, z = blockIdx.z;
  const int col = nt * kBN + threadIdx.x;
  if (col >= N) return;
  const int64_t k0 = blockIdx.y * rows_per_part, k1 = k0 + rows_per_part < K ? k0 + rows_per_part : K;
  const double* src = b + z * b_bs + col;
  double mx = 0.0;
  for (int64_t k = k0; k < k1; ++k) mx = fmax(mx, fabs(__ldg(src + k * ldb)));
  if (mx > 0.0) atomicMax(bexp + (static_cast<int64_t>(z) * ntiles + nt) * kBN + threadIdx.x, row_exponent(mx));
}

// B digits: grid (ntiles, kcs, batch); thread = column; 32 k of its column (coalesced across threads)
__global__ void __launch_bounds__(kBN) ozaki_cols_slice_kernel(const double* __restrict__ b, int64_t ldb, int64_t b_bs,
                                                              int N, int ntiles, int64_t kcs,
                                                              const int32_t* __restrict__ bexp,
                                                              int8_t* __restrict__ bsl) {
  const int nt = blockIdx.x, z = blockIdx.z;
  const int64_t kc = blockIdx.y;
  const int col = nt * kBN + threadIdx.x;
  const bool live = col < N;
  const int32_t e = bexp[(static_cast<int64_t>(z) * ntiles + nt) * kBN + threadIdx.x];
  const double sc = ldexp(1.0, 7 * kS - e);
  const double* src = b + z * b_bs + kc * kBK * ldb + (live ? col : 0);
  int8_t* t = bsl + ((static_cast<int64_t>(z) * ntiles + nt) * kcs + kc) * kBTile;
#pragma unroll
  for (int h = 0; h < kBK / 16; ++h) {
    double x[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) x[q] = live ? __ldg(src + (h * 16 + q) * ldb) * sc : 0.0;
    int4 sl[kS];
    digits16(x, sl);
#pragma unroll
    for (int p = 0; p < kS; ++p)
      *reinterpret_cast<int4*>(t + p * (kBN * kBK) + core_off(threadIdx.x, h * 16)) = sl[p];
  }
}

struct OzGemmArgs {
  const int8_t* asl;
  const int32_t* aexp;
  int64_t a_kcs, a_kc0;            // chunks per sliced A row; first chunk of this GEMM's K
  int64_t a_z0, a_zo, a_zp;        // A batch = a_z0 + (z / planes) * a_zo + (z % planes) * a_zp
  const int8_t* bsl;
  const int32_t* bexp;
  int64_t b_kcs, b_z0, b_zo, b_zp;
  double* c;
  int64_t ldc, c_zo, c_zp;         // C_z = c + (z / planes) * c_zo + (z % planes) * c_zp
  double alpha, beta;
  int M, N, mtiles, ntiles, planes, zcount;
  int kcs, ksplit, kcs_per_split;  // this GEMM's K chunks and their split
  double* work;                    // [split][z][M][N] partials when ksplit > 1
};

__global__ void __launch_bounds__(kOzThreads, 1) ozaki_gemm_kernel(OzGemmArgs a) {
  extern __shared__ __align__(1024) unsigned char oz_smem[];
  int8_t* sA = reinterpret_cast<int8_t*>(oz_smem);
  int8_t* sB = sA + kStages * kATile;
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], tfull;
  __shared__ uint32_t tmem_base;
  __shared__ double scol[kBN];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mt = blockIdx.x, nt = blockIdx.y;
  const int z = blockIdx.z / a.ksplit, split = blockIdx.z % a.ksplit;
  const int zo = z / a.planes, zp = z % a.planes;
  const int64_t za = a.a_z0 + zo * a.a_zo + zp * a.a_zp, zb = a.b_z0 + zo * a.b_zo + zp * a.b_zp;
  const int kc0 = split * a.kcs_per_split;
  const int nk = max(0, min(a.kcs, kc0 + a.kcs_per_split) - kc0);
  const int total = 2 * nk;  // steps: (phase, K chunk)
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
  const int8_t* Ab = a.asl + ((za * a.mtiles + mt) * a.a_kcs + a.a_kc0 + kc0) * kATile;
  const int8_t* Bb = a.bsl + ((zb * a.ntiles + nt) * a.b_kcs + kc0) * kBTile;
  const int quarter = warp & 3, chalf = warp >> 2;
  const int row = mt * kBM + quarter * 32 + lane;
  const double srow = ldexp(1.0, a.aexp[za * a.M + row]);
  if (tid < kBN) scol[tid] = ldexp(1.0, a.bexp[(zb * a.ntiles + nt) * kBN + tid]);
  const uint64_t pol = policy_evict_last();
  int issued = 0;
  auto produce_until = [&](int limit) {
    for (; issued < limit && issued < total; ++issued) {
      const int st = issued % kStages;
      if (issued >= kStages) mbar_wait(&empty[st], ((issued / kStages) - 1) & 1);
      const int ph = issued / nk, kc = issued - ph * nk;
      const uint32_t bytes = static_cast<uint32_t>(phase_slices(ph)) * (kBM * kBK);
      mbar_expect_tx(&full[st], 2 * bytes);
      bulk_g2s(sA + st * kATile, Ab + static_cast<int64_t>(kc) * kATile, bytes, &full[st], pol);
      bulk_g2s(sB + st * kBTile, Bb + static_cast<int64_t>(kc) * kBTile, bytes, &full[st], pol);
    }
  };
  const int64_t live = a.N - static_cast<int64_t>(nt) * kBN;
  double part[kBN / 2];
#pragma unroll
  for (int i = 0; i < kBN / 2; ++i) part[i] = 0.0;
  for (int ph = 0; ph < 2 && nk > 0; ++ph) {
    if (warp == 0 && lane == 0) produce_until((ph + 1) * nk);
    if (warp == 1 && lane == 0) {
      const uint32_t idesc = idesc_n(live >= kBN ? kBN : static_cast<int>((live + 15) / 16) * 16);
      for (int kc = 0; kc < nk; ++kc) {
        const int step = ph * nk + kc, st = step % kStages;
        mbar_wait(&full[st], (step / kStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a0 = smem_u32(sA + st * kATile), b0 = smem_u32(sB + st * kBTile);
        if (ph == 0) {
#pragma unroll
          for (int p = 1; p <= 4; ++p) {
#pragma unroll
            for (int q = 1; p + q <= 5; ++q)
              mma_i8(tmem + static_cast<uint32_t>((p + q - 2) * kBN), umma_desc(a0 + (p - 1) * (kBM * kBK)),
                     umma_desc(b0 + (q - 1) * (kBN * kBK)), (kc > 0 || p > 1) ? 1u : 0u, idesc);
          }
        } else {
#pragma unroll
          for (int p = 1; p <= kS; ++p) {
#pragma unroll
            for (int q = (6 - p > 1 ? 6 - p : 1); p + q <= kS + 1; ++q)
              mma_i8(tmem + static_cast<uint32_t>((p + q - 6) * kBN), umma_desc(a0 + (p - 1) * (kBM * kBK)),
                     umma_desc(b0 + (q - 1) * (kBN * kBK)), (kc > 0 || p > 1) ? 1u : 0u, idesc);
          }
        }
        umma_commit(&empty[st]);
      }
      umma_commit(&tfull);
    }
    if (warp == 0 && lane == 0) produce_until((ph + 1) * nk + kStages);
    __syncwarp();
    mbar_wait(&tfull, ph & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    __syncthreads();
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
#pragma unroll
    for (int ci = 0; ci < kBN / 32; ++ci) {
      const int cc = chalf * (kBN / 32) + ci;
      if (cc * 16 >= live) break;
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
        if (ph == 0)
          part[ci * 16 + jj] = static_cast<double>((G(0) << 21) + (G(1) << 14) + (G(2) << 7) + G(3));
        else
          part[ci * 16 + jj] =
              fma(part[ci * 16 + jj], 0x1p-35, static_cast<double>((G(0) << 14) + (G(1) << 7) + G(2)) * 0x1p-56);
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  // epilogue: this thread's row, its 64 columns (phase-1 values are complete in `part`)
  double* cz = a.c + zo * a.c_zo + zp * a.c_zp;
#pragma unroll
  for (int ci = 0; ci < kBN / 32; ++ci) {
    const int cc = chalf * (kBN / 32) + ci;
    const int64_t j0 = static_cast<int64_t>(nt) * kBN + cc * 16;
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      if (j0 + jj >= a.N) break;
      const double o = nk > 0 ? part[ci * 16 + jj] * srow * scol[cc * 16 + jj] : 0.0;
      if (a.work != nullptr) {
        a.work[((static_cast<int64_t>(split) * a.zcount + z) * a.M + row) * a.N + j0 + jj] = o;
      } else {
        double* cp = cz + static_cast<int64_t>(row) * a.ldc + j0 + jj;
        *cp = a.beta != 0.0 ? fma(a.beta, *cp, a.alpha * o) : a.alpha * o;
      }
    }
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

__global__ void ozaki_split_reduce(OzGemmArgs a) {
  const int64_t mn = static_cast<int64_t>(a.M) * a.N, total = a.zcount * mn;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t z = e / mn, rc = e - z * mn;
    double sum = 0.0;
    for (int sp = 0; sp < a.ksplit; ++sp) sum += a.work[(sp * a.zcount + z) * mn + rc];  // fixed order
    const int64_t r = rc / a.N, cidx = rc - r * a.N;
    double* cp = a.c + (z / a.planes) * a.c_zo + (z % a.planes) * a.c_zp + r * a.ldc + cidx;
    *cp = a.beta != 0.0 ? fma(a.beta, *cp, a.alpha * sum) : a.alpha * sum;
  }
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
  const size_t smem = kStages * kTileSlot;
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
    ozaki_tile_kernel<<<dim3(static_cast<unsigned>(2 * n0 / kBM), nb), kOzTileThreads, smem, s>>>(oa);
    TOEP_LAUNCHED();
  }
  return TOEP_OK;
}

void keep_pool();  // op.cu

// ---- generic GEMM host side
int64_t ozaki_rows_bytes(int64_t M, int64_t K) { return (M / kBM) * (K / kBK) * kATile; }
int64_t ozaki_cols_bytes(int64_t N, int64_t K) { return ((N + kBN - 1) / kBN) * (K / kBK) * kBTile; }
int64_t ozaki_cols_exps(int64_t N) { return ((N + kBN - 1) / kBN) * kBN; }

int ozaki_slice_rows(const double* a, int64_t lda, int64_t a_bs, int64_t batch, int M, int64_t K, int8_t* asl,
                     int32_t* aexp, cudaStream_t s) {
  TOEP_REQUIRE(M % kBM == 0 && K % kBK == 0 && batch <= 65535, TOEP_ERR_ARG, "ozaki rows: M %% 128, K %% 32 required");
  ozaki_rows_exp_kernel<<<dim3(static_cast<unsigned>((M * 32 + 255) / 256), static_cast<unsigned>(batch)), 256, 0, s>>>(
      a, lda, a_bs, M, K, aexp);
  TOEP_LAUNCHED();
  ozaki_rows_slice_kernel<<<dim3(static_cast<unsigned>(M / kBM), static_cast<unsigned>(K / kBK),
                                 static_cast<unsigned>(batch)),
                            kBM, 0, s>>>(a, lda, a_bs, M, K / kBK, aexp, asl);
  TOEP_LAUNCHED();
  return TOEP_OK;
}

int ozaki_slice_cols(const double* b, int64_t ldb, int64_t b_bs, int64_t batch, int N, int64_t K, int8_t* bsl,
                     int32_t* bexp, cudaStream_t s) {
  TOEP_REQUIRE(K % kBK == 0 && batch <= 65535, TOEP_ERR_ARG, "ozaki cols: K %% 32 required");
  const int ntiles = static_cast<int>((N + kBN - 1) / kBN);
  TOEP_CUDA(cudaMemsetAsync(bexp, 0, sizeof(int32_t) * ntiles * kBN * batch, s));
  const int64_t parts = std::max<int64_t>(1, std::min<int64_t>(K / 256, 64));
  const int64_t rpp = (K + parts - 1) / parts;
  ozaki_cols_exp_kernel<<<dim3(ntiles, static_cast<unsigned>(parts), static_cast<unsigned>(batch)), kBN, 0, s>>>(
      b, ldb, b_bs, N, K, ntiles, rpp, bexp);
  TOEP_LAUNCHED();
  ozaki_cols_slice_kernel<<<dim3(ntiles, static_cast<unsigned>(K / kBK), static_cast<unsigned>(batch)), kBN, 0, s>>>(
      b, ldb, b_bs, N, ntiles, K / kBK, bexp, bsl);
  TOEP_LAUNCHED();
  return TOEP_OK;
}

int ozaki_gemm(const OzGemm& g, cudaStream_t s) {
  TOEP_REQUIRE(g.M % kBM == 0 && g.K % kBK == 0 && g.K <= 19000, TOEP_ERR_ARG, "ozaki gemm: bad shape");
  OzGemmArgs a{};
  a.asl = g.asl; a.aexp = g.aexp; a.a_kcs = g.a_kcs; a.a_kc0 = g.a_k0 / kBK;
  a.a_z0 = g.a_z0; a.a_zo = g.a_zo; a.a_zp = g.a_zp;
  a.bsl = g.bsl; a.bexp = g.bexp; a.b_kcs = g.K / kBK; a.b_z0 = g.b_z0; a.b_zo = g.b_zo; a.b_zp = g.b_zp;
  a.c = g.c; a.ldc = g.ldc; a.c_zo = g.c_zo; a.c_zp = g.c_zp; a.alpha = g.alpha; a.beta = g.beta;
  a.M = g.M; a.N = g.N; a.mtiles = g.M / kBM; a.ntiles = static_cast<int>((g.N + kBN - 1) / kBN);
  a.planes = g.planes; a.zcount = g.zcount; a.kcs = static_cast<int>(g.K / kBK);
  // split K so the grid covers the SMs about twice (the partials cost one write + one read of C)
  const int64_t tiles = static_cast<int64_t>(a.mtiles) * a.ntiles * a.zcount;
  int ks = 1;
  while (tiles * ks < 2 * 148 && a.kcs / (ks * 2) >= 16) ks *= 2;
  a.ksplit = ks;
  a.kcs_per_split = (a.kcs + ks - 1) / ks;
  a.work = nullptr;
  const size_t smem = kStages * (kATile + kBTile);
  TOEP_CUDA(ensure_smem(ozaki_gemm_kernel, smem));
  if (ks > 1) {
    keep_pool();
    const size_t wbytes = static_cast<size_t>(ks) * a.zcount * a.M * a.N * sizeof(double);
    if (cudaMallocAsync(reinterpret_cast<void**>(&a.work), wbytes, s) != cudaSuccess) {
      cudaGetLastError();
      set_error("out of device memory for the ozaki split-K partials");
      return TOEP_ERR_OOM;
    }
  }
  ozaki_gemm_kernel<<<dim3(a.mtiles, a.ntiles, static_cast<unsigned>(a.zcount * ks)), kOzThreads, smem, s>>>(a);
  TOEP_LAUNCHED();
  if (ks > 1) {
    ozaki_split_reduce<<<148 * 8, 256, 0, s>>>(a);
    TOEP_LAUNCHED();
    cudaFreeAsync(a.work, s);
  }
  return TOEP_OK;
}

}  // namespace toep

// Standalone entry (tests, tools): C = alpha A B + beta C for row-major real FP64 matrices on the
// int8 tensor cores — A (M x K, M % 128 == 0), B (K x N), K % 32 == 0, K <= 19 000.
extern "C" int toep_ozaki_dgemm(int M, int N, int64_t K, double alpha, const double* A, int64_t lda, const double* B,
                                int64_t ldb, double beta, double* C, int64_t ldc, void* stream) {
  using namespace toep;
  TOEP_REQUIRE(A != nullptr && B != nullptr && C != nullptr && M > 0 && N > 0 && K > 0, TOEP_ERR_ARG,
               "bad ozaki_dgemm arguments");
  TOEP_REQUIRE(M % 128 == 0 && K % 32 == 0 && K <= 19000, TOEP_ERR_SHAPE, "ozaki_dgemm: M %% 128, K %% 32, K <= 19000");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  keep_pool();
  int8_t *asl = nullptr, *bsl = nullptr;
  int32_t *aexp = nullptr, *bexp = nullptr;
  const size_t ab = ozaki_rows_bytes(M, K), bb = ozaki_cols_bytes(N, K);
  if (cudaMallocAsync(reinterpret_cast<void**>(&asl), ab, s) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&bsl), bb, s) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&aexp), sizeof(int32_t) * M, s) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&bexp), sizeof(int32_t) * ozaki_cols_exps(N), s) != cudaSuccess) {
    cudaGetLastError();
    set_error("out of device memory in ozaki_dgemm");
    return TOEP_ERR_OOM;
  }
  int rc = ozaki_slice_rows(A, lda, 0, 1, M, K, asl, aexp, s);
  if (rc == TOEP_OK) rc = ozaki_slice_cols(B, ldb, 0, 1, N, K, bsl, bexp, s);
  if (rc == TOEP_OK) {
    OzGemm g{};
    g.asl = asl; g.aexp = aexp; g.a_kcs = K / 32; g.a_k0 = 0;
    g.bsl = bsl; g.bexp = bexp;
    g.c = C; g.ldc = ldc; g.alpha = alpha; g.beta = beta;
    g.M = M; g.N = N; g.K = K; g.planes = 1; g.zcount = 1;
    rc = ozaki_gemm(g, s);
  }
  for (void* p : {static_cast<void*>(asl), static_cast<void*>(bsl), static_cast<void*>(aexp), static_cast<void*>(bexp)})
    cudaFreeAsync(p, s);
  return rc;
}
