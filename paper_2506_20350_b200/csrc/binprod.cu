// Per-frequency-bin block products and the generic complex GEMM.
//
// bin_product replaces the stacked matmul of the reference matvec,
// `op.diag_blocks @ hat.reshape(k2*k1, n0, -1)` (toeplitz.py:300), and the
// transposed `np.swapaxes(op.diag_blocks, 1, 2) @ hat` (toeplitz.py:320).
//
// The spectral blocks are stored transposed, DT[k][j][m] = D_k[m][j], so that
// the dominant single-RHS product v_k[m] = sum_j D_k[m][j] u_k[j] streams D in
// contiguous rows of DT: lane l of a warp owns output rows m = m0 + l (+32 i),
// each warp walks a disjoint set of j, every 128-bit load is a coalesced
// complex128 and no cross-lane reduction is needed; the WARPS partial sums
// meet once in shared memory at the end of the bin.  D is read with the
// streaming (evict-first) hint so it does not wash the L2-resident spectral
// vectors and Krylov basis out of the 126 MB L2.
#include <cstdlib>
#include <cstring>

#include "kernels.cuh"
#include "launch.cuh"
#include "tma.cuh"

namespace toep {

namespace {

template <typename Z> __device__ __forceinline__ Z ld_stream(const Z* p);
template <> __device__ __forceinline__ double2 ld_stream<double2>(const double2* p) { return __ldcs(p); }
template <> __device__ __forceinline__ float2 ld_stream<float2>(const float2* p) { return __ldcs(p); }

template <typename T, int MPL, int WB, int WARPS, int UNR>
__global__ void __launch_bounds__(WARPS * 32)
binprod_cm_kernel(const C<T>* __restrict__ DT, const C<T>* __restrict__ U, C<T>* __restrict__ V, int64_t K,
                  int n0, int64_t w, int mtiles, const int* stop) {
  if (stop != nullptr && *stop != 0) return;
  using Z = C<T>;
  __shared__ Z red[WARPS][32 * MPL][WB];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nitems = K * mtiles;
  for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int64_t k = item / mtiles;
    const int m0 = static_cast<int>(item - k * mtiles) * 32 * MPL;
    const Z* Dk = DT + k * n0 * n0 + m0;
    const Z* Uk = U + k * n0 * w;
    Z* Vk = V + k * n0 * w;
    bool mok[MPL];
#pragma unroll
    for (int i = 0; i < MPL; ++i) mok[i] = (m0 + lane + 32 * i) < n0;
    for (int64_t w0 = 0; w0 < w; w0 += WB) {
      const int wc = static_cast<int>(std::min<int64_t>(WB, w - w0));
      Z acc[MPL][WB];
#pragma unroll
      for (int i = 0; i < MPL; ++i)
#pragma unroll
        for (int c = 0; c < WB; ++c) acc[i][c] = mk<T>(0, 0);
      int j = warp;
      for (; j + (UNR - 1) * WARPS < n0; j += UNR * WARPS) {
        Z d[UNR][MPL];
#pragma unroll
        for (int r = 0; r < UNR; ++r)
#pragma unroll
          for (int i = 0; i < MPL; ++i)
            d[r][i] = mok[i] ? ld_stream(Dk + static_cast<int64_t>(j + r * WARPS) * n0 + lane + 32 * i) : mk<T>(0, 0);
#pragma unroll
        for (int r = 0; r < UNR; ++r) {
          Z u[WB];
#pragma unroll
          for (int c = 0; c < WB; ++c)
            u[c] = (c < wc) ? Uk[static_cast<int64_t>(j + r * WARPS) * w + w0 + c] : mk<T>(0, 0);
#pragma unroll
          for (int i = 0; i < MPL; ++i)
#pragma unroll
            for (int c = 0; c < WB; ++c) cfma(acc[i][c], d[r][i], u[c]);
        }
      }
      for (; j < n0; j += WARPS) {
        Z d[MPL];
#pragma unroll
        for (int i = 0; i < MPL; ++i)
          d[i] = mok[i] ? ld_stream(Dk + static_cast<int64_t>(j) * n0 + lane + 32 * i) : mk<T>(0, 0);
#pragma unroll
        for (int c = 0; c < WB; ++c) {
          const Z u = (c < wc) ? Uk[static_cast<int64_t>(j) * w + w0 + c] : mk<T>(0, 0);
#pragma unroll
          for (int i = 0; i < MPL; ++i) cfma(acc[i][c], d[i], u);
        }
      }
#pragma unroll
      for (int i = 0; i < MPL; ++i)
#pragma unroll
        for (int c = 0; c < WB; ++c) red[warp][lane + 32 * i][c] = acc[i][c];
      __syncthreads();
      for (int t = threadIdx.x; t < 32 * MPL * WB; t += WARPS * 32) {
        const int mm = t / WB;
        const int c = t - mm * WB;
        Z s = red[0][mm][c];
#pragma unroll
        for (int ww = 1; ww < WARPS; ++ww) s = cadd(s, red[ww][mm][c]);
        const int m = m0 + mm;
        if (m < n0 && c < wc) Vk[static_cast<int64_t>(m) * w + w0 + c] = s;
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------------------------------
// TMA-bulk streaming version of the single-RHS product (the dominant kernel of the matvec).
//
// Persistent: one CTA per SM, a contiguous range of work items, item = (bin k, m-tile of MT
// output rows).  Warp 8 is the producer: one elected lane streams the item's DT rows
// (row j, columns m0..m0+MT: one contiguous MT*16 B run) into a STAGES-deep shared-memory
// ring with cp.async.bulk (evict-first L2 policy), completion signalled through per-stage
// mbarriers (complete_tx).  Warps 0-7 consume: lane l owns rows m0 + l + 32 i, each warp
// takes RB/8 rows j of every stage, no cross-lane reduction; the 8 warp partials meet in
// shared memory once per item.  The memory pipeline never waits for the math.
template <typename T, int MT, int RB, int STAGES>
struct TmaCfg {
  using Z = C<T>;
  static constexpr int kStageElems = RB * MT;
  static constexpr size_t kRing = sizeof(Z) * STAGES * kStageElems;
  static constexpr size_t kU = sizeof(Z) * 256;
  static constexpr size_t kRed = sizeof(Z) * kTmaConsumerWarps * MT;
  static constexpr size_t kSmem = kRing + kU + kRed + 2 * STAGES * sizeof(uint64_t);
};

template <typename T, int MT, int RB, int STAGES>
__global__ void __launch_bounds__(kTmaThreads, 1)
binprod_tma_kernel(const C<T>* __restrict__ DT, const C<T>* __restrict__ U, C<T>* __restrict__ V, int n0,
                   int mtiles, int64_t items, const int* stop) {
  // PDL: D is constant, so without a stop flag the producer starts streaming D
  // before the forward DFT kernel has drained; consumers wait for u_hat.
  if (stop != nullptr) {
    pdl_wait();
    if (*stop != 0) return;
  }
  pdl_trigger();
  using Z = C<T>;
  using Cfg = TmaCfg<T, MT, RB, STAGES>;
  constexpr int MPL = MT / 32;
  extern __shared__ __align__(128) unsigned char smem[];
  Z* ring = reinterpret_cast<Z*>(smem);
  Z* us = reinterpret_cast<Z*>(smem + Cfg::kRing);
  Z* red = reinterpret_cast<Z*>(smem + Cfg::kRing + Cfg::kU);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::kRing + Cfg::kU + Cfg::kRed);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t per = items / gridDim.x, rem = items % gridDim.x;
  const int64_t i_begin = blockIdx.x * per + std::min<int64_t>(blockIdx.x, rem);
  const int64_t i_end = i_begin + per + (blockIdx.x < rem ? 1 : 0);
  const int nrb = n0 / RB;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaConsumerWarps);
    }
    mbar_init_fence();
  }
  __syncthreads();

  if (warp == kTmaConsumerWarps) {  // ---------------- producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t it = i_begin; it < i_end; ++it) {
        const int64_t k = it / mtiles;
        const int m0 = static_cast<int>(it - k * mtiles) * MT;
        const Z* base = DT + k * n0 * n0 + m0;
        for (int rb = 0; rb < nrb; ++rb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], static_cast<uint32_t>(sizeof(Z) * Cfg::kStageElems));
          Z* dst = ring + stage * Cfg::kStageElems;
          if (MT == n0) {  // whole rows: the stage is one contiguous RB*n0 run
            bulk_g2s(dst, base + static_cast<int64_t>(rb * RB) * n0, sizeof(Z) * Cfg::kStageElems, &full[stage], pol);
          } else {
#pragma unroll 4
            for (int r = 0; r < RB; ++r)
              bulk_g2s(dst + r * MT, base + static_cast<int64_t>(rb * RB + r) * n0, sizeof(Z) * MT, &full[stage],
                       pol);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    return;
  }
  // ------------------------------------------------------ consumers
  pdl_wait();
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t it = i_begin; it < i_end; ++it) {
    const int64_t k = it / mtiles;
    const int m0 = static_cast<int>(it - k * mtiles) * MT;
    for (int t = threadIdx.x; t < n0; t += kTmaConsumerWarps * 32) us[t] = U[k * n0 + t];
    consumers_sync();
    Z acc[MPL];
#pragma unroll
    for (int i = 0; i < MPL; ++i) acc[i] = mk<T>(0, 0);
    for (int rb = 0; rb < nrb; ++rb) {
      mbar_wait(&full[stage], phase);
      const Z* tile = ring + stage * Cfg::kStageElems;
#pragma unroll
      for (int r = warp; r < RB; r += kTmaConsumerWarps) {
        const Z uj = us[rb * RB + r];
#pragma unroll
        for (int i = 0; i < MPL; ++i) cfma(acc[i], tile[r * MT + lane + 32 * i], uj);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
#pragma unroll
    for (int i = 0; i < MPL; ++i) red[warp * MT + lane + 32 * i] = acc[i];
    consumers_sync();
    for (int t = threadIdx.x; t < MT; t += kTmaConsumerWarps * 32) {
      Z s = red[t];
#pragma unroll
      for (int ww = 1; ww < kTmaConsumerWarps; ++ww) s = cadd(s, red[ww * MT + t]);
      V[k * n0 + m0 + t] = s;
    }
    consumers_sync();
  }
}

// transposed product: V_k[j][c] = sum_m DT[k][j][m] U_k[m][c]  (row dots of DT)
template <typename T, int MPL, int WB>
__global__ void __launch_bounds__(256)
binprod_rm_kernel(const C<T>* __restrict__ DT, const C<T>* __restrict__ U, C<T>* __restrict__ V, int64_t K,
                  int n0, int64_t w, const int* stop) {
  if (stop != nullptr && *stop != 0) return;
  using Z = C<T>;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t k = blockIdx.x; k < K; k += gridDim.x) {
    const Z* Dk = DT + k * n0 * n0;
    const Z* Uk = U + k * n0 * w;
    Z* Vk = V + k * n0 * w;
    for (int64_t w0 = 0; w0 < w; w0 += WB) {
      const int wc = static_cast<int>(std::min<int64_t>(WB, w - w0));
      for (int mb = 0; mb < n0; mb += 32 * MPL) {
        Z u[MPL][WB];
#pragma unroll
        for (int i = 0; i < MPL; ++i) {
          const int m = mb + lane + 32 * i;
#pragma unroll
          for (int c = 0; c < WB; ++c)
            u[i][c] = (m < n0 && c < wc) ? Uk[static_cast<int64_t>(m) * w + w0 + c] : mk<T>(0, 0);
        }
        for (int j = warp; j < n0; j += 8) {
          Z acc[WB];
#pragma unroll
          for (int c = 0; c < WB; ++c) acc[c] = mk<T>(0, 0);
#pragma unroll
          for (int i = 0; i < MPL; ++i) {
            const int m = mb + lane + 32 * i;
            const Z d = (m < n0) ? ld_stream(Dk + static_cast<int64_t>(j) * n0 + m) : mk<T>(0, 0);
#pragma unroll
            for (int c = 0; c < WB; ++c) cfma(acc[c], d, u[i][c]);
          }
#pragma unroll
          for (int c = 0; c < WB; ++c) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
              acc[c].x += __shfl_xor_sync(0xffffffffu, acc[c].x, off);
              acc[c].y += __shfl_xor_sync(0xffffffffu, acc[c].y, off);
            }
          }
          if (lane == 0) {
            for (int c = 0; c < wc; ++c) {
              Z* dst = Vk + static_cast<int64_t>(j) * w + w0 + c;
              *dst = (mb == 0) ? acc[c] : cadd(*dst, acc[c]);
            }
          }
        }
        __syncwarp();
      }
    }
  }
}

// --------------------------------------------------------------- GEMM (SIMT)
struct GemmArgs {
  int64_t m, n, k;
  double2 alpha, beta;
  const void* a;
  int64_t a_rs, a_cs, a_bs;
  const void* b;
  int64_t b_rs, b_cs, b_bs;
  void* c;
  int64_t c_rs, c_cs, c_bs;
  const int* stop;
};

constexpr int BM = 64, BN = 64, BK = 8;

template <typename T>
__global__ void __launch_bounds__(256) gemm_kernel(GemmArgs g) {
  if (g.stop != nullptr && *g.stop != 0) return;
  using Z = C<T>;
  __shared__ Z As[BK][BM + 1];
  __shared__ Z Bs[BK][BN + 1];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t bz = blockIdx.z;
  const int64_t row0 = static_cast<int64_t>(blockIdx.y) * BM;
  const int64_t col0 = static_cast<int64_t>(blockIdx.x) * BN;
  const Z* A = static_cast<const Z*>(g.a) + bz * g.a_bs;
  const Z* B = static_cast<const Z*>(g.b) + bz * g.b_bs;
  Z* Cm = static_cast<Z*>(g.c) + bz * g.c_bs;
  Z acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = mk<T>(0, 0);
  const bool a_kfast = (g.a_cs == 1);
  const bool b_nfast = (g.b_cs == 1);
  for (int64_t k0 = 0; k0 < g.k; k0 += BK) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int idx = tid + e * 256;
      int r, kk;
      if (a_kfast) { r = idx / BK; kk = idx % BK; } else { r = idx % BM; kk = idx / BM; }
      const int64_t gr = row0 + r, gk = k0 + kk;
      As[kk][r] = (gr < g.m && gk < g.k) ? A[gr * g.a_rs + gk * g.a_cs] : mk<T>(0, 0);
      int cc, kb;
      if (b_nfast) { cc = idx % BN; kb = idx / BN; } else { kb = idx % BK; cc = idx / BK; }
      const int64_t gc = col0 + cc, gkb = k0 + kb;
      Bs[kb][cc] = (gc < g.n && gkb < g.k) ? B[gkb * g.b_rs + gc * g.b_cs] : mk<T>(0, 0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      Z av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) cfma(acc[i][j], av[i], bv[j]);
    }
    __syncthreads();
  }
  const Z alpha = mk<T>(static_cast<T>(g.alpha.x), static_cast<T>(g.alpha.y));
  const Z beta = mk<T>(static_cast<T>(g.beta.x), static_cast<T>(g.beta.y));
  const bool use_beta = (g.beta.x != 0.0 || g.beta.y != 0.0);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gr = row0 + ty + 16 * i;
    if (gr >= g.m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gc = col0 + tx + 16 * j;
      if (gc >= g.n) continue;
      Z* dst = Cm + gr * g.c_rs + gc * g.c_cs;
      Z v = cmul(alpha, acc[i][j]);
      if (use_beta) v = cadd(v, cmul(beta, *dst));
      *dst = v;
    }
  }
}

template <typename T>
__global__ void transpose_kernel(const C<T>* __restrict__ in, C<T>* __restrict__ out, int rows, int cols) {
  using Z = C<T>;
  __shared__ Z tile[32][33];
  const int64_t b = blockIdx.z;
  const Z* src = in + b * rows * cols;
  Z* dst = out + b * rows * cols;
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = src[static_cast<int64_t>(r) * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[static_cast<int64_t>(c) * rows + r] = tile[threadIdx.x][i];
  }
}

__global__ void cast_kernel(const double2* __restrict__ in, float2* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = make_float2(static_cast<float>(in[i].x), static_cast<float>(in[i].y));
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <typename T, int WB, int UNR = (WB <= 2) ? 4 : 2>
int launch_cm(const void* DT, const void* U, void* V, int64_t K, int n0, int64_t w, const int* stop,
              cudaStream_t s) {
  constexpr int WARPS = 8;
  const int mtiles = (n0 + 31) / 32;
  const int64_t items = K * mtiles;
  const int64_t grid = items;
  binprod_cm_kernel<T, 1, WB, WARPS, UNR><<<static_cast<unsigned>(grid), WARPS * 32, 0, s>>>(
      static_cast<const C<T>*>(DT), static_cast<const C<T>*>(U), static_cast<C<T>*>(V), K, n0, w, mtiles, stop);
  TOEP_LAUNCHED();
  return TOEP_OK;
}

template <typename T, int MT, int STAGES = 6>
int launch_tma(const void* DT, const void* U, void* V, int64_t K, int n0, const int* stop, cudaStream_t s) {
  constexpr int RB = 32768 / (MT * sizeof(C<T>));  // 32 KB per stage
  using Cfg = TmaCfg<T, MT, RB, STAGES>;
  auto kern = binprod_tma_kernel<T, MT, RB, STAGES>;
  TOEP_CUDA(ensure_smem(kern, Cfg::kSmem));
  const int mtiles = n0 / MT;
  const int64_t items = K * mtiles;
  const int grid = static_cast<int>(std::min<int64_t>(items, sm_count()));
  return launch_k(kern, dim3(grid), dim3(kTmaThreads), Cfg::kSmem, s, static_cast<const C<T>*>(DT),
                  static_cast<const C<T>*>(U), static_cast<C<T>*>(V), n0, mtiles, items, stop);
}

template <typename T>
int launch_rm(const void* DT, const void* U, void* V, int64_t K, int n0, int64_t w, const int* stop,
              cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(K, 65535));
  if (w == 1)
    binprod_rm_kernel<T, 4, 1><<<grid, 256, 0, s>>>(static_cast<const C<T>*>(DT), static_cast<const C<T>*>(U),
                                                     static_cast<C<T>*>(V), K, n0, w, stop);
  else
    binprod_rm_kernel<T, 2, 4><<<grid, 256, 0, s>>>(static_cast<const C<T>*>(DT), static_cast<const C<T>*>(U),
                                                     static_cast<C<T>*>(V), K, n0, w, stop);
  TOEP_LAUNCHED();
  return TOEP_OK;
}

template <typename T>
int bin_product_t(const void* DT, const void* U, void* V, int64_t K, int n0, int64_t w, bool transpose,
                  const int* stop, cudaStream_t s) {
  if (transpose) return launch_rm<T>(DT, U, V, K, n0, w, stop, s);
  if (w >= 16) {
    // V_k (n0 x w) = D_k U_k with D_k[m][j] = DT[k][j][m]
    return gemm(sizeof(T) == 8 ? TOEP_C128 : TOEP_C64, n0, w, n0, make_double2(1, 0), DT, 1, n0,
                static_cast<int64_t>(n0) * n0, U, w, 1, static_cast<int64_t>(n0) * w, make_double2(0, 0), V, w, 1,
                static_cast<int64_t>(n0) * w, K, s, stop);
  }
  if (w == 1) {
    // whole-row bulk-copy stream (N_b = 128: one 32 KB DT row pair per stage), 64-column row
    // segments for the other multiples of 64, the SIMT column kernel otherwise
    if (n0 == 128) return launch_tma<T, 128>(DT, U, V, K, n0, stop, s);
    if (n0 % 64 == 0 && n0 <= 256) return launch_tma<T, 64>(DT, U, V, K, n0, stop, s);
    return launch_cm<T, 1>(DT, U, V, K, n0, w, stop, s);
  }
  if (w == 2) return launch_cm<T, 2>(DT, U, V, K, n0, w, stop, s);
  if (w <= 4) return launch_cm<T, 4>(DT, U, V, K, n0, w, stop, s);
  return launch_cm<T, 8>(DT, U, V, K, n0, w, stop, s);
}

}  // namespace

L2Prefetch binprod_prefetch_plan(int dtype, const void* DT, int64_t K, int n0, int side) {
  L2Prefetch pf;
  if (n0 != 128) return pf;  // only the whole-row TMA stream has this bin order
  // L2 prefetch of the head of every CTA's bin range, issued by the forward DFT (side 0) while it
  // computes: 48 MB measured best (+4 %); from the inverse DFT (side 1) or the GMRES
  // orthogonalisation (side 2) it measured no gain, so those budgets are 0
  constexpr int64_t budget[3] = {int64_t{48} << 20, 0, 0};
  const int64_t bin_bytes = static_cast<int64_t>(n0) * n0 * (dtype == TOEP_C64 ? 8 : 16);
  pf.ranges = static_cast<int>(std::min<int64_t>(K, sm_count()));
  const int64_t range_min = bin_bytes * (K / pf.ranges);
  auto share = [&](int64_t b) { return std::min<int64_t>(b / pf.ranges, range_min) / 32768 * 32768; };
  const int64_t fwd = share(budget[0]);
  int64_t head = 0;
  if (side == 0) {
    head = fwd;
  } else if (side == 1) {
    head = share(budget[1]);
  } else {
    pf.skip = fwd;
    head = std::min<int64_t>(share(budget[2]), range_min - fwd);
  }
  if (head <= 0) return L2Prefetch{};
  pf.base = DT;
  pf.bin_bytes = bin_bytes;
  pf.bytes = head;
  pf.K = K;
  return pf;
}

int bin_product(int dtype, const void* DT, const void* U, void* V, int64_t K, int n0, int64_t w, bool transpose,
                const int* stop, cudaStream_t s) {
  if (K == 0 || w == 0) return TOEP_OK;
  if (dtype == TOEP_C128) return bin_product_t<double>(DT, U, V, K, n0, w, transpose, stop, s);
  return bin_product_t<float>(DT, U, V, K, n0, w, transpose, stop, s);
}

// Skinny complex128 GEMM, all operands row-major, n <= NC columns: C = alpha A B + beta C.
// One CTA per RB rows of A (x batch); its 256 threads stride over K (coalesced 512-byte rows of
// A per warp, B rows from L2), then a fixed-order warp-shuffle + shared-memory reduction (no
// atomics: deterministic).  Used where the tile GEMM would launch only m/64 CTAs (n <= 8
// right-hand sides against a long K) and run at a fraction of HBM bandwidth.
template <int NC, int RB>
__global__ void __launch_bounds__(256) skinny_gemm_kernel(int64_t m, int n, int64_t k, double2 alpha,
                                                          const double2* __restrict__ A, int64_t lda, int64_t a_bs,
                                                          const double2* __restrict__ B, int64_t ldb, int64_t b_bs,
                                                          double2 beta, double2* C, int64_t ldc, int64_t c_bs) {
  __shared__ double2 red[8][RB][NC];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * RB;
  A += blockIdx.y * a_bs + r0 * lda;
  B += blockIdx.y * b_bs;
  C += blockIdx.y * c_bs;
  const int rows = static_cast<int>(std::min<int64_t>(RB, m - r0));
  double2 acc[RB][NC];
#pragma unroll
  for (int r = 0; r < RB; ++r)
#pragma unroll
    for (int j = 0; j < NC; ++j) acc[r][j] = make_double2(0, 0);
  for (int64_t kk = tid; kk < k; kk += 256) {
    double2 b[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) b[j] = j < n ? B[kk * ldb + j] : make_double2(0, 0);
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const double2 av = r < rows ? A[r * lda + kk] : make_double2(0, 0);
#pragma unroll
      for (int j = 0; j < NC; ++j) cfma(acc[r][j], av, b[j]);
    }
  }
#pragma unroll
  for (int r = 0; r < RB; ++r)
#pragma unroll
    for (int j = 0; j < NC; ++j) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        acc[r][j].x += __shfl_xor_sync(0xffffffffu, acc[r][j].x, off);
        acc[r][j].y += __shfl_xor_sync(0xffffffffu, acc[r][j].y, off);
      }
      if (lane == 0) red[warp][r][j] = acc[r][j];
    }
  __syncthreads();
  if (tid < RB * NC) {
    const int r = tid / NC, j = tid % NC;
    if (r < rows && j < n) {
      double2 sum = red[0][r][j];
      for (int w = 1; w < 8; ++w) sum = cadd(sum, red[w][r][j]);
      double2* cp = C + (r0 + r) * ldc + j;
      double2 out = cmul(alpha, sum);
      if (beta.x != 0.0 || beta.y != 0.0) cfma(out, beta, *cp);
      *cp = out;
    }
  }
}

template <int NC, int RB>
int skinny_launch(int64_t m, int64_t n, int64_t k, double2 alpha, const void* a, int64_t lda, int64_t a_bs,
                  const void* b, int64_t ldb, int64_t b_bs, double2 beta, void* c, int64_t ldc, int64_t c_bs,
                  int64_t batch, cudaStream_t s) {
  const dim3 grid(static_cast<unsigned>((m + RB - 1) / RB), static_cast<unsigned>(batch));
  skinny_gemm_kernel<NC, RB><<<grid, 256, 0, s>>>(m, static_cast<int>(n), k, alpha, static_cast<const double2*>(a), lda,
                                                  a_bs, static_cast<const double2*>(b), ldb, b_bs, beta,
                                                  static_cast<double2*>(c), ldc, c_bs);
  TOEP_LAUNCHED();
  return TOEP_OK;
}

int gemm(int dtype, int64_t m, int64_t n, int64_t k, double2 alpha, const void* a, int64_t a_rs, int64_t a_cs,
         int64_t a_bs, const void* b, int64_t b_rs, int64_t b_cs, int64_t b_bs, double2 beta, void* c, int64_t c_rs,
         int64_t c_cs, int64_t c_bs, int64_t batch, cudaStream_t s, const int* stop) {
  if (m == 0 || n == 0 || batch == 0) return TOEP_OK;
  if (dtype == TOEP_C128 && stop == nullptr && n <= 8 && k >= 256 && a_cs == 1 && b_cs == 1 &&
      c_cs == 1 && batch <= 65535 && (m + 3) / 4 <= 0x7fffffff) {
    if (n <= 4) return skinny_launch<4, 4>(m, n, k, alpha, a, a_rs, a_bs, b, b_rs, b_bs, beta, c, c_rs, c_bs, batch, s);
    return skinny_launch<8, 2>(m, n, k, alpha, a, a_rs, a_bs, b, b_rs, b_bs, beta, c, c_rs, c_bs, batch, s);
  }
  if (dtype == TOEP_C128 && m * n * k >= 32 * 32 * 32) {
    const int rc = zgemm_dmma(m, n, k, alpha, a, a_rs, a_cs, a_bs, b, b_rs, b_cs, b_bs, beta, c, c_rs, c_cs, c_bs,
                              batch, s, stop);
    if (rc >= 0) return rc;
  }
  GemmArgs g{m, n, k, alpha, beta, a, a_rs, a_cs, a_bs, b, b_rs, b_cs, b_bs, c, c_rs, c_cs, c_bs, stop};
  const int64_t gy = (m + BM - 1) / BM, gx = (n + BN - 1) / BN;
  TOEP_REQUIRE(gy <= 65535 && batch <= 65535 && gx <= 0x7fffffff, TOEP_ERR_ARG, "gemm grid too large");
  dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(gy), static_cast<unsigned>(batch));
  if (dtype == TOEP_C128) gemm_kernel<double><<<grid, 256, 0, s>>>(g);
  else gemm_kernel<float><<<grid, 256, 0, s>>>(g);
  TOEP_LAUNCHED();
  return TOEP_OK;
}

int transpose_batched(int dtype, const void* in, void* out, int64_t batch, int rows, int cols, cudaStream_t s) {
  if (batch == 0) return TOEP_OK;
  TOEP_REQUIRE(batch <= 65535, TOEP_ERR_ARG, "transpose batch too large");
  dim3 grid((cols + 31) / 32, (rows + 31) / 32, static_cast<unsigned>(batch));
  dim3 block(32, 8);
  if (dtype == TOEP_C128)
    transpose_kernel<double><<<grid, block, 0, s>>>(static_cast<const double2*>(in), static_cast<double2*>(out), rows, cols);
  else
    transpose_kernel<float><<<grid, block, 0, s>>>(static_cast<const float2*>(in), static_cast<float2*>(out), rows, cols);
  TOEP_LAUNCHED();
  return TOEP_OK;
}

int cast_c128_to_c64(const void* in, void* out, int64_t n, cudaStream_t s) {
  if (n == 0) return TOEP_OK;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
  cast_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(static_cast<const double2*>(in), static_cast<float2*>(out), n);
  TOEP_LAUNCHED();
  return TOEP_OK;
}

}  // namespace toep
