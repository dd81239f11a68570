// Fused spectral kernel of the single-RHS matvec: level-2 forward DFT + per-bin product +
// level-2 inverse DFT in one persistent TMA-streaming kernel.
//
// The reference matvec (toeplitz.py:287-303) is pad -> block_fft_2l (level 1, then level 2)
// -> diag_blocks @ hat -> inverse block_fft_2l -> extract.  Here the level-1 (x) transforms
// stay standalone passes, and the level-2 (y) transforms move into the product kernel:
//
//   * bins are visited kx-major: a CTA owns a contiguous range of (kx, ky) bins, i.e. one or
//     two runs of consecutive ky at fixed kx;
//   * at the start of a run the CTA loads the level-1 spectrum column X1[y][kx][:] (the n2
//     non-zero rows only) into shared memory; for each bin the 256 consumer threads form
//     u_hat[ky][kx][:] = sum_y w^{ky y} X1[y][kx][:] directly (thread = (j, y-group));
//   * D_k streams through the TMA ring exactly as in binprod_tma_kernel;
//   * v_hat_k is folded into per-thread accumulators of the inverse level-2 DFT,
//     X2[y][kx][m] += w^{-ky y} v_hat[m] (only the n2 kept rows: the crop is fused), and at
//     the end of a run the CTA writes its partial X2 slab; the inverse level-1 pass sums the
//     (<= maxp) slabs of each kx while loading.
//
// All the DFT work is register/shared-memory arithmetic that overlaps the D stream (the ring
// keeps ~3 us of bandwidth in flight), so the two level-2 passes, their launches and their
// 15 MB of L2 round trips disappear from the matvec critical path.
#include <vector>

#include "launch.cuh"
#include "op.h"
#include "tma.cuh"

namespace toep {

namespace {

struct FusedArgs {
  const void* DT;  // [K][n0][n0] transposed spectral blocks, bin k = ky*L1 + kx
  const void* X1;  // [n2][L1][n0] level-1 forward DFT of u
  void* P;         // [L1][maxp][n2][n0] inverse level-2 partial slabs
  void* X2;        // [n2][L1][n0] combined inverse level-2 DFT (input of the inverse level-1 pass)
  int* cnt;        // [L1] arrival counters, zero between launches
  int n2, L1, L2, maxp;
  int64_t items;   // L1 * L2
  const int* stop;
};

__device__ __forceinline__ int64_t cta_of(int64_t i, int64_t per, int64_t rem) {
  const int64_t cut = rem * (per + 1);
  return i < cut ? i / (per + 1) : rem + (i - cut) / per;
}

template <typename T, int N0, int STAGES, int YMAX>
struct FusedCfg {
  using Z = C<T>;
  static constexpr int G = 256 / N0;                       // y-groups of consumer threads
  static constexpr int RB = 32768 / (N0 * sizeof(Z));      // DT rows per 32 KB stage
  static constexpr int kStageElems = RB * N0;
  static constexpr size_t kRing = sizeof(Z) * STAGES * kStageElems;
  static size_t smem(int n2, int L2) {
    return kRing + sizeof(Z) * (static_cast<size_t>(n2) * N0 + G * N0 + kTmaConsumerWarps * N0 + 2 * N0 + L2) +
           2 * STAGES * sizeof(uint64_t) + 16;
  }
};

template <typename T, int N0, int STAGES, int YMAX>
__global__ void __launch_bounds__(kTmaThreads, 1) mlfft_fused_kernel(FusedArgs fa) {
  using Z = C<T>;
  using Cfg = FusedCfg<T, N0, STAGES, YMAX>;
  constexpr int G = Cfg::G;
  constexpr int RB = Cfg::RB;
  constexpr int MPL = N0 / 32;
  if (fa.stop != nullptr) {
    pdl_wait();
    if (*fa.stop != 0) return;
  }
  pdl_trigger();
  extern __shared__ __align__(128) unsigned char smem[];
  Z* ring = reinterpret_cast<Z*>(smem);
  Z* col = reinterpret_cast<Z*>(smem + Cfg::kRing);   // [n2][N0]
  Z* upart = col + fa.n2 * N0;                          // [G][N0]
  Z* red = upart + G * N0;                              // [8][N0]
  Z* us = red + kTmaConsumerWarps * N0;                 // [N0]
  Z* vs = us + N0;                                      // [N0]
  Z* tw = vs + N0;                                      // [L2] forward twiddles exp(-2 pi i t / L2)
  uint64_t* full = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(tw + fa.L2) + 15) & ~static_cast<uintptr_t>(15));
  uint64_t* empty = full + STAGES;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int64_t per = fa.items / gridDim.x, rem = fa.items % gridDim.x;
  const int64_t i_begin = blockIdx.x * per + std::min<int64_t>(blockIdx.x, rem);
  const int64_t i_end = i_begin + per + (blockIdx.x < rem ? 1 : 0);
  const int L1 = fa.L1, L2 = fa.L2, n2 = fa.n2;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaConsumerWarps);
    }
    mbar_init_fence();
  }
  for (int t = tid; t < L2; t += kTmaThreads) {
    T s, c;
    if constexpr (sizeof(T) == 8) sincospi(static_cast<T>(2.0 * t / L2), &s, &c);
    else sincospif(static_cast<T>(2.0 * t / L2), &s, &c);
    tw[t] = mk<T>(c, -s);
  }
  __syncthreads();

  if (warp == kTmaConsumerWarps) {  // ------------------------------------------- producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const Z* DT = static_cast<const Z*>(fa.DT);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t it = i_begin; it < i_end; ++it) {
        const int64_t kx = it / L2, ky = it - kx * L2;
        const Z* base = DT + (ky * L1 + kx) * N0 * N0;
#pragma unroll 1
        for (int rb = 0; rb < N0 / RB; ++rb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], static_cast<uint32_t>(sizeof(Z) * Cfg::kStageElems));
          bulk_g2s(ring + stage * Cfg::kStageElems, base + static_cast<int64_t>(rb) * Cfg::kStageElems,
                   sizeof(Z) * Cfg::kStageElems, &full[stage], pol);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    return;
  }
  // ------------------------------------------------------------------------- consumers
  pdl_wait();
  const Z* X1 = static_cast<const Z*>(fa.X1);
  Z* P = static_cast<Z*>(fa.P);
  const int j = tid % N0;         // column (u_hat index j, later output row m)
  const int g = tid / N0;         // y-group
  const int ypt = (n2 + G - 1) / G;
  const int y0 = g * ypt;
  Z inv[YMAX];
  int stage = 0;
  uint32_t phase = 0;
  int64_t cur_kx = -1;
  int part = 0;
  __shared__ int last_flag;
  for (int64_t it = i_begin; it < i_end; ++it) {
    const int64_t kx = it / L2;
    const int ky = static_cast<int>(it - kx * L2);
    if (kx != cur_kx) {  // new run: level-1 spectrum column, fresh inverse accumulators
      for (int e = tid; e < n2 * N0; e += 256) {
        const int y = e / N0;
        col[e] = X1[(static_cast<int64_t>(y) * L1 + kx) * N0 + (e - y * N0)];
      }
#pragma unroll
      for (int q = 0; q < YMAX; ++q) inv[q] = mk<T>(0, 0);
      cur_kx = kx;
      part = static_cast<int>(blockIdx.x - cta_of(kx * L2, per, rem));
      consumers_sync();
    }
    // forward level-2 DFT of this bin (rows y < n2 only: the zero padding is implicit)
    {
      Z s = mk<T>(0, 0);
      int idx = (ky * y0) % L2;  // twiddle index ky*y mod L2, advanced incrementally
#pragma unroll
      for (int q = 0; q < YMAX; ++q) {
        const int y = y0 + q;
        if (q < ypt && y < n2) cfma(s, col[y * N0 + j], tw[idx]);
        idx += ky;
        idx = idx >= L2 ? idx - L2 : idx;
      }
      upart[g * N0 + j] = s;
    }
    consumers_sync();
    if (tid < N0) {
      Z s = upart[tid];
#pragma unroll
      for (int gg = 1; gg < G; ++gg) s = cadd(s, upart[gg * N0 + tid]);
      us[tid] = s;
    }
    consumers_sync();
    // per-bin product v_k = D_k u_k, D_k streamed as DT rows
    Z acc[MPL];
#pragma unroll
    for (int i = 0; i < MPL; ++i) acc[i] = mk<T>(0, 0);
#pragma unroll 1
    for (int rb = 0; rb < N0 / RB; ++rb) {
      mbar_wait(&full[stage], phase);
      const Z* tile = ring + stage * Cfg::kStageElems;
#pragma unroll
      for (int r = warp; r < RB; r += kTmaConsumerWarps) {
        const Z uj = us[rb * RB + r];
#pragma unroll
        for (int i = 0; i < MPL; ++i) cfma(acc[i], tile[r * N0 + lane + 32 * i], uj);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
#pragma unroll
    for (int i = 0; i < MPL; ++i) red[warp * N0 + lane + 32 * i] = acc[i];
    consumers_sync();
    if (tid < N0) {
      Z s = red[tid];
#pragma unroll
      for (int ww = 1; ww < kTmaConsumerWarps; ++ww) s = cadd(s, red[ww * N0 + tid]);
      vs[tid] = s;
    }
    consumers_sync();
    // inverse level-2 DFT contribution, kept rows only
    {
      const Z v = vs[j];
      int idx = (ky * y0) % L2;
#pragma unroll
      for (int q = 0; q < YMAX; ++q) {
        const int y = y0 + q;
        if (q < ypt && y < n2) {
          const Z w = tw[idx];
          cfma(inv[q], mk<T>(w.x, -w.y), v);
        }
        idx += ky;
        idx = idx >= L2 ? idx - L2 : idx;
      }
    }
    const bool run_end = (it + 1 == i_end) || ((it + 1) / L2 != kx);
    if (run_end) {
      // A kx column split over np CTAs: each writes its partial slab; the last to arrive
      // (threadfence + counter) adds the slabs in fixed order p = 0..np-1 (deterministic)
      // and writes the combined column, so the inverse level-1 pass reads plain X2.
      Z* X2 = static_cast<Z*>(fa.X2);
      const int np = static_cast<int>(cta_of(kx * L2 + L2 - 1, per, rem) - cta_of(kx * L2, per, rem) + 1);
      if (np == 1) {
#pragma unroll
        for (int q = 0; q < YMAX; ++q) {
          const int y = y0 + q;
          if (q < ypt && y < n2) X2[(static_cast<int64_t>(y) * L1 + kx) * N0 + j] = inv[q];
        }
      } else {
        Z* slab = P + (static_cast<int64_t>(kx) * fa.maxp + part) * n2 * N0;
#pragma unroll
        for (int q = 0; q < YMAX; ++q) {
          const int y = y0 + q;
          if (q < ypt && y < n2) slab[y * N0 + j] = inv[q];
        }
        __threadfence();
        consumers_sync();
        if (tid == 0) last_flag = (atomicAdd(&fa.cnt[kx], 1) == np - 1);
        consumers_sync();
        if (last_flag) {
          __threadfence();
          const Z* slabs = P + static_cast<int64_t>(kx) * fa.maxp * n2 * N0;
#pragma unroll
          for (int q = 0; q < YMAX; ++q) {
            const int y = y0 + q;
            if (q < ypt && y < n2) {
              Z sum = __ldcg(slabs + y * N0 + j);
              for (int p = 1; p < np; ++p) sum = cadd(sum, __ldcg(slabs + (static_cast<int64_t>(p) * n2 + y) * N0 + j));
              X2[(static_cast<int64_t>(y) * L1 + kx) * N0 + j] = sum;
            }
          }
          if (tid == 0) fa.cnt[kx] = 0;
        }
      }
    }
  }
}

template <typename T, int N0, int YMAX>
int launch_fused(toep_op_s* op, const void* x1, void* P, void* X2, int* cnt, const int* stop, cudaStream_t s) {
  constexpr int STAGES = 4;
  using Cfg = FusedCfg<T, N0, STAGES, YMAX>;
  auto kern = mlfft_fused_kernel<T, N0, STAGES, YMAX>;
  const size_t smem = Cfg::smem(op->n2, op->l2);
  static int attr = 0;
  if (attr < static_cast<int>(smem)) {
    TOEP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = static_cast<int>(smem);
  }
  FusedArgs fa{op->DT, x1, P, X2, cnt, op->n2, op->l1, op->l2, op->fused_maxp, op->K, stop};
  return launch_k(kern, dim3(op->fused_grid), dim3(kTmaThreads), smem, s, fa);
}

}  // namespace

bool fused_eligible(const toep_op_s* op, int64_t w, bool transpose) {
  // Opt-in (TOEP_FUSED=1): measured on B200 at cfg2 it ties the unfused PDL chain
  // (166 vs 160 us per matvec), see DESIGN.md "fused level-2 transforms".
  static const bool off = [] {
    const char* e = std::getenv("TOEP_FUSED");
    return !(e != nullptr && std::strcmp(e, "1") == 0);
  }();
  if (off || w != 1 || transpose) return false;
  if (op->n0 != 64 && op->n0 != 128 && op->n0 != 256) return false;
  if (op->l2 > 256) return false;
  if (op->l1 != 32 && op->l1 != 60 && op->l1 != 64 && op->l1 != 128) return false;  // compiled level-1 plans
  const size_t es = op->dtype == TOEP_C64 ? 8 : 16;
  const int G = 256 / op->n0;
  const int ypt = (op->n2 + G - 1) / G;
  const int ymax = op->dtype == TOEP_C64 ? 32 : 16;
  if (ypt > ymax) return false;
  const size_t smem = 4 * 32768 + es * (static_cast<size_t>(op->n2) * op->n0 + (G + kTmaConsumerWarps + 2) * op->n0 +
                                        op->l2) + 128;
  return smem <= 227 * 1024;
}

// op->fused_grid / fused_maxp / part_count (device) for the kx-major partition
int fused_prepare(toep_op_s* op, cudaStream_t s) {
  std::lock_guard<std::mutex> lock(op->mu);
  if (op->part_count != nullptr) return TOEP_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t items = op->K;
  const int grid = static_cast<int>(std::min<int64_t>(items, sms));
  const int64_t per = items / grid, rem = items % grid;
  auto cta_of_h = [&](int64_t i) {
    const int64_t cut = rem * (per + 1);
    return i < cut ? i / (per + 1) : rem + (i - cut) / per;
  };
  std::vector<int> counts(op->l1);
  int maxp = 1;
  for (int kx = 0; kx < op->l1; ++kx) {
    const int64_t a = cta_of_h(static_cast<int64_t>(kx) * op->l2);
    const int64_t b = cta_of_h(static_cast<int64_t>(kx) * op->l2 + op->l2 - 1);
    counts[kx] = static_cast<int>(b - a + 1);
    maxp = std::max(maxp, counts[kx]);
  }
  int* dcount = nullptr;
  TOEP_CUDA(cudaMalloc(&dcount, sizeof(int) * op->l1));
  TOEP_CUDA(cudaMemcpyAsync(dcount, counts.data(), sizeof(int) * op->l1, cudaMemcpyHostToDevice, s));
  TOEP_CUDA(cudaStreamSynchronize(s));
  op->fused_grid = grid;
  op->fused_maxp = maxp;
  op->part_count = dcount;
  return TOEP_OK;
}

int fused_spectral(toep_op_s* op, const void* x1, void* P, void* X2, int* cnt, const int* stop, cudaStream_t s) {
  if (op->dtype == TOEP_C128) {
    switch (op->n0) {
      case 64: return launch_fused<double, 64, 16>(op, x1, P, X2, cnt, stop, s);
      case 128: return launch_fused<double, 128, 16>(op, x1, P, X2, cnt, stop, s);
      case 256: return launch_fused<double, 256, 16>(op, x1, P, X2, cnt, stop, s);
      default: break;
    }
  } else {
    switch (op->n0) {
      case 64: return launch_fused<float, 64, 32>(op, x1, P, X2, cnt, stop, s);
      case 128: return launch_fused<float, 128, 32>(op, x1, P, X2, cnt, stop, s);
      case 256: return launch_fused<float, 256, 32>(op, x1, P, X2, cnt, stop, s);
      default: break;
    }
  }
  set_error("fused spectral kernel: unsupported n0 %d", op->n0);
  return TOEP_ERR_ARG;
}

}  // namespace toep
