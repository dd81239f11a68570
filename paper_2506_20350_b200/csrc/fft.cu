// Batched shared-memory mixed-radix DFT pass (Stockham autosort).
//
// Replaces the block-wise FFT of the reference, block_fft_2l / _fft_axis
// (toeplitz.py:207-245, np.fft.fft / np.fft.ifft = pocketfft), for one axis of
// the circulant grid: F_L (x) I_inner applied to a strided array whose batch
// dimension (n0 * w, or n0 * n0 for the spectral precompute) is contiguous, so
// every global load / store is a coalesced run of `TIL` complex values.
//
// One CTA owns one (outer, batch-tile) pair: it gathers the L axis values of
// TIL batch columns into shared memory (zero-padding fused), runs the radix
// stages ping-ponging between two shared buffers, and the last stage writes
// straight to global memory with the crop and the 1/L scale fused.
#include <cstdlib>
#include <mutex>
#include <cstring>
#include <type_traits>

#include "kernels.cuh"
#include "launch.cuh"
#include "tma.cuh"

namespace toep {

namespace {

constexpr int kThreads = 128;
constexpr int kMinBlocks = 8;  // 64 regs/thread cap: 8 CTAs x 31 KB per SM keep enough loads in flight for the big passes
constexpr int kMinBlocksGeneric = 4;  // runtime-radix pass: the generic butterflies need >64 regs (spilled ~700 B at 8)
constexpr int kMaxStages = 16;

struct Radices {
  int n;
  int r[kMaxStages];
};

template <typename T> __device__ __forceinline__ void sincospi_t(T x, T* s, T* c);
template <> __device__ __forceinline__ void sincospi_t<double>(double x, double* s, double* c) { sincospi(x, s, c); }
template <> __device__ __forceinline__ void sincospi_t<float>(float x, float* s, float* c) { sincospif(x, s, c); }

// output scale of a pass; a device-side input scale (lazy GMRES normalisation) folds in by linearity
template <typename T> __device__ __forceinline__ T pass_scale(const PassArgs& a) {
  return static_cast<T>(a.in_scale != nullptr ? a.scale * *a.in_scale : a.scale);
}

template <typename Zd, typename Zs> __device__ __forceinline__ Zd cvt(Zs v) {
  Zd r;
  r.x = v.x;
  r.y = v.y;
  return r;
}

// y = DFT_R(v) with R-th roots wr[m] = exp(sign*2*pi*i*m/R)
template <typename Z, int R>
__device__ __forceinline__ void butterfly(Z* v, const Z* wr, int sign) {
  if constexpr (R == 2) {
    Z a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 4) {
    Z t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    Z t2 = cadd(v[1], v[3]), d = csub(v[1], v[3]);
    Z t3;  // (sign*i) * d
    t3.x = -sign * d.y;
    t3.y = sign * d.x;
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3);
    v[3] = csub(t1, t3);
  } else if constexpr (R == 3) {
    // y0 = v0 + s, y1,2 = (v0 - s/2) +- sign*i*(sqrt(3)/2)(v1 - v2), s = v1 + v2
    using T = decltype(v[0].x);
    constexpr T kS3 = static_cast<T>(0.86602540378443864676);
    const Z sm = cadd(v[1], v[2]), d = csub(v[1], v[2]);
    Z m;
    m.x = v[0].x - static_cast<T>(0.5) * sm.x;
    m.y = v[0].y - static_cast<T>(0.5) * sm.y;
    Z rot;
    rot.x = -sign * kS3 * d.y;
    rot.y = sign * kS3 * d.x;
    v[0] = cadd(v[0], sm);
    v[1] = cadd(m, rot);
    v[2] = csub(m, rot);
  } else if constexpr (R == 5) {
    // a_k = v_k + v_{5-k}, b_k = v_k - v_{5-k}; y_k / y_{5-k} = p_k +- sign*i*q_k
    using T = decltype(v[0].x);
    constexpr T c1 = static_cast<T>(0.30901699437494742410), c2 = static_cast<T>(-0.80901699437494742410);
    constexpr T s1 = static_cast<T>(0.95105651629515357212), s2 = static_cast<T>(0.58778525229247312917);
    const Z a1 = cadd(v[1], v[4]), b1 = csub(v[1], v[4]);
    const Z a2 = cadd(v[2], v[3]), b2 = csub(v[2], v[3]);
    Z p1, p2, q1, q2;
    p1.x = v[0].x + c1 * a1.x + c2 * a2.x;
    p1.y = v[0].y + c1 * a1.y + c2 * a2.y;
    p2.x = v[0].x + c2 * a1.x + c1 * a2.x;
    p2.y = v[0].y + c2 * a1.y + c1 * a2.y;
    q1.x = s1 * b1.x + s2 * b2.x;
    q1.y = s1 * b1.y + s2 * b2.y;
    q2.x = s2 * b1.x - s1 * b2.x;
    q2.y = s2 * b1.y - s1 * b2.y;
    Z r1, r2;  // sign*i*q
    r1.x = -sign * q1.y;
    r1.y = sign * q1.x;
    r2.x = -sign * q2.y;
    r2.y = sign * q2.x;
    v[0] = cadd(v[0], cadd(a1, a2));
    v[1] = cadd(p1, r1);
    v[4] = csub(p1, r1);
    v[2] = cadd(p2, r2);
    v[3] = csub(p2, r2);
  } else {
    Z o[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      Z acc = v[0];
#pragma unroll
      for (int r = 1; r < R; ++r) cfma(acc, v[r], wr[(q * r) % R]);
      o[q] = acc;
    }
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = o[q];
  }
}

template <typename TC, typename TO, int TIL, int R, bool LAST>
__device__ __forceinline__ void run_stage(const C<TC>* __restrict__ src, C<TC>* __restrict__ dst,
                                          const C<TC>* __restrict__ tw, int L, int Ns, int sign,
                                          C<TO>* __restrict__ gout, int64_t out_sa, int n_out,
                                          int ncol, TC scale) {
  using Z = C<TC>;
  const int nb = L / R;
  const int tstep = L / (Ns * R);
  Z wr[R];
  if constexpr (R == 7) {
#pragma unroll
    for (int m = 0; m < R; ++m) wr[m] = tw[m * nb];
  }
  for (int e = threadIdx.x; e < nb * TIL; e += kThreads) {
    const int j = e / TIL;
    const int col = e - j * TIL;
    const int k = j % Ns;
    Z v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src[(j + r * nb) * TIL + col];
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw[k * r * tstep]);
    butterfly<Z, R>(v, wr, sign);
    const int base = (j / Ns) * Ns * R + k;
    if constexpr (!LAST) {
#pragma unroll
      for (int q = 0; q < R; ++q) dst[(base + q * Ns) * TIL + col] = v[q];
    } else {
      if (col < ncol) {
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int idx = base + q * Ns;
          if (idx < n_out) gout[idx * out_sa + col] = cvt<C<TO>>(cscale(v[q], scale));
        }
      }
    }
  }
}

template <typename TC, typename TO, int TIL, bool LAST>
__device__ __forceinline__ void dispatch_stage(int R, const C<TC>* src, C<TC>* dst, const C<TC>* tw, int L,
                                               int Ns, int sign, C<TO>* gout, int64_t out_sa, int n_out,
                                               int ncol, TC scale) {
  switch (R) {
    case 2: run_stage<TC, TO, TIL, 2, LAST>(src, dst, tw, L, Ns, sign, gout, out_sa, n_out, ncol, scale); break;
    case 3: run_stage<TC, TO, TIL, 3, LAST>(src, dst, tw, L, Ns, sign, gout, out_sa, n_out, ncol, scale); break;
    case 4: run_stage<TC, TO, TIL, 4, LAST>(src, dst, tw, L, Ns, sign, gout, out_sa, n_out, ncol, scale); break;
    case 5: run_stage<TC, TO, TIL, 5, LAST>(src, dst, tw, L, Ns, sign, gout, out_sa, n_out, ncol, scale); break;
    case 7: run_stage<TC, TO, TIL, 7, LAST>(src, dst, tw, L, Ns, sign, gout, out_sa, n_out, ncol, scale); break;
    default: break;
  }
}

// Completion signal of a peer-scatter launch: every CTA counts itself in (acq_rel, system
// scope: its threads' peer stores are ordered before by the barrier); the last one adds 1 to each
// destination's arrival counter with a system-scope release and re-arms the count.
__device__ __forceinline__ void peer_signal(const toep_peer_scatter* sc) {
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned long long* done = const_cast<unsigned long long*>(reinterpret_cast<const unsigned long long*>(&sc->done));
  const unsigned long long total = static_cast<unsigned long long>(gridDim.x) * gridDim.y * gridDim.z;
  unsigned long long old;
  asm volatile("atom.acq_rel.sys.global.add.u64 %0, [%1], 1;" : "=l"(old) : "l"(done) : "memory");
  if (old + 1 != total) return;
  asm volatile("st.relaxed.sys.global.u64 [%0], 0;" ::"l"(done) : "memory");
  for (int q = 0; q < sc->parts; ++q)
    asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(sc->signal[q]) : "memory");
}

// Peer-scatter epilogue: the pass result (natural order, unscaled) sits in shared memory `res`
// [L][TIL]; output row idx goes to the rank whose range holds it (table lo/base/off/sa/so).
template <typename TC, typename TO, int TIL>
__device__ __forceinline__ void scatter_tile(const PassArgs& a, const C<TC>* res, int ncol, TC scale) {
  const toep_peer_scatter* sc = a.scatter;
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * TIL;
  const int64_t o = blockIdx.y;
  for (int e = threadIdx.x; e < a.n_out * TIL; e += kThreads) {
    const int idx = e / TIL;
    const int col = e - idx * TIL;
    if (col >= ncol) continue;
    int q = 0;
    while (q + 1 < sc->parts && idx >= sc->lo[q + 1]) ++q;
    C<TO>* dstp = reinterpret_cast<C<TO>*>(sc->base[q]) + sc->off[q] + idx * sc->sa[q] + o * sc->so[q] + i0 + col;
    *dstp = cvt<C<TO>>(cscale(res[idx * TIL + col], scale));
  }
  peer_signal(sc);
}

// ------------------------------------------------------------------------------------------
// Compile-time plans for the embedding lengths the BASELINE grids use (7, 32, 60, 128): every
// index, stride and trip count is a constant.  The first stage reads its radix inputs straight
// from global memory (zero padding fused, no staging copy), intermediate stages ping-pong in
// shared memory, the last stage writes the cropped, scaled outputs.  Launched with PDL: the
// twiddle table is built before griddepcontrol.wait, overlapping the predecessor's tail.
template <int... Rs> struct PlanLen;
template <> struct PlanLen<> { static constexpr int value = 1; };
template <int R, int... Rest> struct PlanLen<R, Rest...> { static constexpr int value = R * PlanLen<Rest...>::value; };

template <typename TI, typename TC, typename TO, int NT, int TIL, int L, int Ns, int kIn, int R, int... Rest>
__device__ __forceinline__ void plan_stage(const PassArgs& a, const C<TI>* __restrict__ gin, C<TO>* __restrict__ gout,
                                           C<TC>* __restrict__ src, C<TC>* __restrict__ dst,
                                           const C<TC>* __restrict__ tw, int ncol, TC scale) {
  using Z = C<TC>;
  static_assert(kIn >= 0 && kIn <= 3, "plan_stage input mode");
  static_assert(Ns * R * PlanLen<Rest...>::value == L, "plan radices must multiply to L");
  constexpr bool kFirst = (Ns == 1);
  constexpr bool kLast = sizeof...(Rest) == 0;
  constexpr int nb = L / R;
  constexpr int tstep = L / (Ns * R);
  Z wr[R];  // roots of unity, only for the generic (radix-7) butterfly
  if constexpr (R == 7) {
#pragma unroll
    for (int m = 0; m < R; ++m) wr[m] = tw[m * nb];
  }
  const int hi_start = L - a.n_hi;
#pragma unroll 2
  for (int e = threadIdx.x; e < nb * TIL; e += NT) {
    const int j = e / TIL;
    const int col = e % TIL;
    const int k = j % Ns;
    Z v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if constexpr (kFirst) {
        const int slot = j + r * nb;
        int row = -1;
        if (slot < a.n_lo) row = slot;
        else if (slot >= hi_start) row = a.n_lo + slot - hi_start;
        v[r] = mk<TC>(0, 0);
        if constexpr (kIn == 1) {  // staged by the streaming kernel: rows [n_lo + n_hi][TIL] in `src`
          if (row >= 0 && col < ncol) v[r] = src[row * TIL + col];
        } else if constexpr (kIn >= 2) {  // staged planes [3 or 2][n_lo + n_hi][TIL] doubles
          if (row >= 0 && col < ncol) {
            const double* sp = reinterpret_cast<const double*>(src);
            const int nr = a.n_lo + a.n_hi;
            const double t1 = sp[row * TIL + col], t2 = sp[(nr + row) * TIL + col];
            if (kIn == 3 || a.planes2) {
              v[r] = mk<TC>(static_cast<TC>(t1), static_cast<TC>(t2));
            } else {
              const double t3 = sp[(2 * nr + row) * TIL + col];
              v[r] = mk<TC>(static_cast<TC>(t1 - t2), static_cast<TC>(t3 - t1 - t2));
            }
          }
        } else if (row >= 0 && col < ncol) {
          if (a.in_planes != nullptr) {
            const int64_t e = (gin - static_cast<const C<TI>*>(a.in)) + row * a.in_sa + col * a.in_cs;
            const double t1 = a.in_planes[e], t2 = a.in_planes[a.plane + e];
            if (a.planes2) {
              v[r] = mk<TC>(static_cast<TC>(t1), static_cast<TC>(t2));
            } else {
              const double t3 = a.in_planes[2 * a.plane + e];
              v[r] = mk<TC>(static_cast<TC>(t1 - t2), static_cast<TC>(t3 - t1 - t2));
            }
          } else {
            v[r] = cvt<Z>(gin[row * a.in_sa + col * a.in_cs]);
          }
        }
      } else {
        v[r] = src[(j + r * nb) * TIL + col];
      }
    }
    if constexpr (!kFirst) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw[k * r * tstep]);
    }
    butterfly<Z, R>(v, wr, a.sign);
    const int base = (j / Ns) * Ns * R + k;
    if constexpr (!kLast) {
#pragma unroll
      for (int q = 0; q < R; ++q) dst[(base + q * Ns) * TIL + col] = v[q];
    } else if (a.scatter != nullptr) {  // peer scatter: the epilogue stores from shared memory
#pragma unroll
      for (int q = 0; q < R; ++q) dst[(base + q * Ns) * TIL + col] = v[q];
    } else {
      if (col < ncol) {
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int idx = base + q * Ns;
          if (idx < a.n_out) {
            if (a.out_planes != nullptr) {
              const int64_t e = (gout - static_cast<C<TO>*>(a.out)) + idx * a.out_sa + col * a.out_cs;
              const Z val = cscale(v[q], scale);
              a.out_planes[e] = static_cast<double>(val.x);
              a.out_planes[a.plane + e] = static_cast<double>(val.y);
              if (!a.planes2) a.out_planes[2 * a.plane + e] = static_cast<double>(val.x) + static_cast<double>(val.y);
            } else {
              gout[idx * a.out_sa + col * a.out_cs] = cvt<C<TO>>(cscale(v[q], scale));
            }
          }
        }
      }
    }
  }
  if constexpr (!kLast) {
    __syncthreads();
    plan_stage<TI, TC, TO, NT, TIL, L, Ns * R, kIn, Rest...>(a, gin, gout, dst, src, tw, ncol, scale);
  }
}

template <typename TI, typename TC, typename TO, int TIL, int... Rs>
__global__ void __launch_bounds__(kThreads, kMinBlocks) fft_plan_kernel(PassArgs a, double two_over_L) {
  using Z = C<TC>;
  constexpr int L = PlanLen<Rs...>::value;
  __shared__ __align__(16) Z tw[L];
  __shared__ __align__(16) Z buf[2][L * TIL];
  pdl_trigger();
  for (int t = threadIdx.x; t < L; t += kThreads) {
    TC s, c;
    sincospi_t<TC>(static_cast<TC>(t * two_over_L), &s, &c);
    tw[t] = mk<TC>(c, a.sign * s);
  }
  pdl_wait();
  if (a.stop != nullptr && *a.stop != 0) return;
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * TIL;
  const int o = blockIdx.y;
  const int ncol = static_cast<int>(std::min<int64_t>(TIL, a.inner - i0));
  const C<TI>* in = static_cast<const C<TI>*>(a.in) + o * a.in_so + i0;
  if (a.in_idx != nullptr) in += static_cast<int64_t>(*a.in_idx) * a.in_idx_stride;
  C<TO>* out = static_cast<C<TO>*>(a.out) + o * a.out_so + i0;
  if (a.out_idx != nullptr) out += static_cast<int64_t>(*a.out_idx) * a.out_idx_stride;
  __syncthreads();  // twiddle table
  plan_stage<TI, TC, TO, kThreads, TIL, L, 1, 0, Rs...>(a, in, out, buf[0], buf[1], tw, ncol, pass_scale<TC>(a));
  if (a.scatter != nullptr) {  // stage s writes buf[(s + 1) % 2]
    __syncthreads();
    scatter_tile<TC, TO, TIL>(a, buf[sizeof...(Rs) % 2], ncol, pass_scale<TC>(a));
  }
}

template <typename TI, typename TC, typename TO, int TIL, int... Rs>
int launch_plan(const PassArgs& a, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((a.inner + TIL - 1) / TIL), static_cast<unsigned>(a.outer));
  return launch_k(fft_plan_kernel<TI, TC, TO, TIL, Rs...>, grid, dim3(kThreads), 0, s, a,
                  2.0 / PlanLen<Rs...>::value);
}

// Persistent, software-pipelined variant of fft_plan_kernel for the very large passes of the
// multi-RHS matvec (hundreds of thousands of tiles streamed through HBM): each CTA walks tiles
// t = blockIdx.x + k * gridDim.x and stages tile t + gridDim.x with cp.async (LDGSTS) while it
// transforms tile t, so every SM keeps input bytes in flight across its whole lifetime instead of
// paying load latency + launch ramp per short-lived CTA.  Shared memory: two staging buffers
// (also used as the ping-pong partner of `work`) and `work`.  kIn = 1: complex rows; kIn = 2: the
// (T1, T2, T3) planes of the 3M product, recombined when the first stage reads them.
constexpr int kStreamBlocks = 4;

template <typename TC, int TIL, int kIn, int L>
struct StreamSmem {
  // complex slots per staging buffer: kIn 2 = three double planes, kIn 3 = two (Re, Im: the Ozaki path)
  static constexpr int kStageZ = kIn == 2 ? (3 * L * TIL + 1) / 2 : L * TIL;
  static constexpr size_t bytes = sizeof(C<TC>) * (L + 2 * static_cast<size_t>(kStageZ) + L * TIL);
};

__device__ __forceinline__ void cp_async(void* smem, const void* g, int nbytes) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  if (nbytes == 16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(g) : "memory");
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(g) : "memory");
}

template <typename TC, typename TO, int TIL, int kIn, int... Rs>
__global__ void __launch_bounds__(kThreads, TIL <= 8 ? 2 * kStreamBlocks : kStreamBlocks) fft_plan_stream_kernel(PassArgs a, double two_over_L,
                                                                                 int64_t ntiles, int64_t tiles_x) {
  using Z = C<TC>;
  constexpr int L = PlanLen<Rs...>::value;
  using SM = StreamSmem<TC, TIL, kIn, L>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Z* tw = reinterpret_cast<Z*>(smem_raw);
  Z* stage[2] = {tw + L, tw + L + SM::kStageZ};
  Z* work = tw + L + 2 * SM::kStageZ;
  pdl_trigger();
  for (int t = threadIdx.x; t < L; t += kThreads) {
    TC s, c;
    sincospi_t<TC>(static_cast<TC>(t * two_over_L), &s, &c);
    tw[t] = mk<TC>(c, a.sign * s);
  }
  pdl_wait();
  if (a.stop != nullptr && *a.stop != 0) return;
  const int nrows = a.n_lo + a.n_hi;
  auto issue = [&](int64_t tile, Z* buf) {
    const int64_t o = tile / tiles_x;
    const int64_t i0 = (tile - o * tiles_x) * TIL;
    const int ncol = static_cast<int>(std::min<int64_t>(TIL, a.inner - i0));
    const int64_t g0 = o * a.in_so + i0;  // complex-element offset of the tile's (row 0, col 0)
    for (int e = threadIdx.x; e < nrows * TIL; e += kThreads) {
      const int row = e / TIL;
      const int col = e - row * TIL;
      if (col >= ncol) continue;
      const int64_t ge = g0 + row * a.in_sa + col * a.in_cs;
      if constexpr (kIn == 1) {
        cp_async(buf + e, static_cast<const Z*>(a.in) + ge, static_cast<int>(sizeof(Z)));
      } else {
        double* bd = reinterpret_cast<double*>(buf);
        const int np = (kIn == 3 || a.planes2) ? 2 : 3;
        for (int p = 0; p < np; ++p) cp_async(bd + p * nrows * TIL + e, a.in_planes + p * a.plane + ge, 8);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const TC scale = pass_scale<TC>(a);
  int64_t t = blockIdx.x;
  if (t < ntiles) issue(t, stage[0]);
  for (int k = 0; t < ntiles; t += gridDim.x, ++k) {
    const int cur = k & 1;
    if (t + gridDim.x < ntiles) issue(t + gridDim.x, stage[cur ^ 1]);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();  // tile t staged by every thread (and the twiddles, on the first pass)
    const int64_t o = t / tiles_x;
    const int64_t i0 = (t - o * tiles_x) * TIL;
    const int ncol = static_cast<int>(std::min<int64_t>(TIL, a.inner - i0));
    C<TO>* out = static_cast<C<TO>*>(a.out) + o * a.out_so + i0;
    plan_stage<TC, TC, TO, kThreads, TIL, L, 1, kIn, Rs...>(a, nullptr, out, stage[cur], work, tw, ncol, scale);
    __syncthreads();  // stage[cur] is refilled (tile t + 2 * gridDim.x) in the next iteration
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

inline int device_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// streaming launch for very large passes (TI == TC, no device-side offsets / partial sums / scatter);
// returns -1 when the pass does not qualify
template <typename TC, typename TO, int TIL, int... Rs>
int try_stream(const PassArgs& a, cudaStream_t s) {
  constexpr int64_t min_tiles = int64_t{1} << 15;  // persistent streaming only for very large passes
  const int64_t tiles_x = (a.inner + TIL - 1) / TIL;
  const int64_t ntiles = tiles_x * a.outer;
  // measured on cfg3 (L = 60, 432 000 tiles per pass): the plane-input pass 1.74 -> 1.38 ms, but the
  // complex-input passes 1.17 -> 1.30 / 2.45 -> 2.56 ms (fewer resident warps than the short-lived
  // CTAs of fft_plan_kernel): only plane-input passes stream
  if (ntiles < min_tiles || a.in_idx != nullptr || a.out_idx != nullptr || a.scatter != nullptr ||
      a.in_planes == nullptr)
    return -1;
  constexpr int L = PlanLen<Rs...>::value;
  auto launch_kin = [&](auto kin_tag) -> int {
    constexpr int kIn = decltype(kin_tag)::value;
    using SM = StreamSmem<TC, TIL, kIn, L>;
    auto kern = fft_plan_stream_kernel<TC, TO, TIL, kIn, Rs...>;
    static int per_sm = 0;  // identical devices: same occupancy; the attribute itself is per device
    TOEP_CUDA(ensure_smem(kern, SM::bytes));
    if (per_sm == 0) {
      TOEP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, SM::bytes));
      if (per_sm <= 0) per_sm = 1;
    }
    const int64_t grid = std::min<int64_t>(ntiles, static_cast<int64_t>(device_sms()) * per_sm);
    return launch_k(kern, dim3(static_cast<unsigned>(grid)), dim3(kThreads), SM::bytes, s, a, 2.0 / L, ntiles, tiles_x);
  };
  // two planes: 47 KB of shared memory per CTA (4 resident per SM) instead of the 3-plane 62 KB (3)
  if (a.in_planes != nullptr && a.planes2) return launch_kin(std::integral_constant<int, 3>{});
  if (a.in_planes != nullptr) return launch_kin(std::integral_constant<int, 2>{});
  return launch_kin(std::integral_constant<int, 1>{});
}

// compile-time plan for L (7, 32, 60, 128), or -1
template <typename TI, typename TC, typename TO>
int try_plan(const PassArgs& a, cudaStream_t s) {
  switch (a.L) {
    case 60:
      if (a.inner >= 16) {
        if constexpr (std::is_same_v<TI, TC>) {
          const int rc = try_stream<TC, TO, 16, 4, 3, 5>(a, s);  // 16-column tiles (8: 47.7 vs 46.5 ms at cfg3)
          if (rc >= 0) return rc;
        }
        return launch_plan<TI, TC, TO, 16, 4, 3, 5>(a, s);
      }
      break;
    case 128: if (a.inner >= 8) return launch_plan<TI, TC, TO, 8, 4, 4, 4, 2>(a, s); break;
    case 32: if (a.inner >= 32) return launch_plan<TI, TC, TO, 32, 4, 4, 2>(a, s); break;
    case 64: if (a.inner >= 16) return launch_plan<TI, TC, TO, 16, 4, 4, 4>(a, s); break;
    default: break;
  }
  return -1;
}

// ------------------------------------------------------------------------------------------
// Whole 2-D transform per batch column in one CTA: the level-1 pass writes the (n2 x l1)
// intermediate to shared memory, the level-2 pass reads it from there (no global round trip,
// one launch instead of two).  Used for the single-RHS matvec on grids whose shared-memory
// footprint fits (cfg2 60x60, cfg5 32x32).
template <int... Rs> struct Plan {
  static constexpr int L = PlanLen<Rs...>::value;
  static constexpr int kStages = sizeof...(Rs);
  template <typename TI, typename TC, typename TO, int NT, int TIL>
  __device__ static void run(const PassArgs& a, const C<TI>* gin, C<TO>* gout, C<TC>* b0, C<TC>* b1,
                             const C<TC>* tw, int ncol, TC scale) {
    plan_stage<TI, TC, TO, NT, TIL, L, 1, 0, Rs...>(a, gin, gout, b0, b1, tw, ncol, scale);
  }
};

struct Fft2dArgs {
  const void* in;
  void* out;
  int n2, n1;
  int64_t inner;
  int sign;
  const double* in_scale;
  const int* stop;
  L2Prefetch pf;
};

constexpr int k2dThreads = 512;

template <typename TC, int TILX, int TILY, typename PX, typename PY>
struct Fft2dSmem {
  static constexpr int kBuf = (PX::L * TILX > PY::L * TILY) ? PX::L * TILX : PY::L * TILY;
  // G rows padded to an odd stride: the level-1 pass walks G down a column (one row per lane)
  static constexpr int kGs = PX::L | 1;
  static size_t bytes(int n2) { return sizeof(C<TC>) * (PX::L + PY::L + 2 * kBuf + static_cast<size_t>(n2) * kGs); }
};

#ifdef TOEP_ORTH_PROBE
__device__ long long g_dft_ts[2][160][8];
#define DPROBE(i)                                                                            \
  if (threadIdx.x == 0 && b < 160) {                                                         \
    long long t_;                                                                            \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                   \
    g_dft_ts[INV ? 1 : 0][b][i] = t_;                                                        \
  }
#else
#define DPROBE(i)
#endif

// The 2-D transform of batch column `b`, shared-memory workspace at `smem_raw`.  Every thread of the
// block calls it (threads >= k2dThreads only take part in the barriers).  With `wait` the PDL
// wait / stop check happens inside (after the twiddles); returns false when the stop flag is set.
struct NoHook {
  __device__ void operator()() const {}
};

// kAliasG: the (n2 x l1) intermediate G lives in ping-pong buffer b1 instead of a buffer of its own
// (the caller guarantees n2 * kGs <= kBuf).  Both plans have three stages, so the first pass ends
// reading b0 (b1 is free for G) and the second pass runs with the buffers swapped (its first stage
// reads G = b1 and writes b0).
// kHatT: the spectral side (forward output / inverse input) is stored column-major, [b][ky][kx], so
// the CTA of batch column b reads / writes one contiguous run of l2 * l1 values (coalesced) instead of
// l2 * l1 values 16 * inner bytes apart.
template <typename TI, typename TC, typename TO, int TILX, int TILY, typename PX, typename PY, bool INV,
          bool kAliasG = false, int NT = k2dThreads, bool kHatT = false, typename AfterL1 = NoHook>
__device__ __forceinline__ bool fft2d_body(const Fft2dArgs& f, unsigned char* smem_raw, int64_t b, bool wait,
                                           AfterL1 after_l1 = {}, const C<TC>* tw_given = nullptr) {
  using Z = C<TC>;
  using S = Fft2dSmem<TC, TILX, TILY, PX, PY>;
  constexpr int L1 = PX::L, L2 = PY::L;
  static_assert(!kAliasG || (PX::kStages == 3 && PY::kStages == 3), "G aliasing assumes three-stage plans");
  static_assert(!kAliasG || TILY >= PX::L, "G aliasing needs single-tile level-2 passes (the caller keeps n2 <= TILX)");
  // twiddles: computed here, or a table of the right sign the caller built earlier (L1 == L2)
  Z* twx = tw_given != nullptr ? const_cast<Z*>(tw_given) : reinterpret_cast<Z*>(smem_raw);
  Z* twy = tw_given != nullptr ? twx : twx + L1;
  Z* b0 = reinterpret_cast<Z*>(smem_raw) + L1 + L2;
  Z* b1 = b0 + S::kBuf;
  Z* G = kAliasG ? b1 : b1 + S::kBuf;  // [n2][kGs]
  Z* p0 = kAliasG ? b1 : b0;  // ping-pong order of the second pass
  Z* p1 = kAliasG ? b0 : b1;
  constexpr int Gs = S::kGs;
  if (tw_given == nullptr)
    for (int t = threadIdx.x; t < L1 + L2; t += NT) {
      const int L = t < L1 ? L1 : L2;
      const int tt = t < L1 ? t : t - L1;
      TC s, c;
      sincospi_t<TC>(static_cast<TC>(2.0 * tt / L), &s, &c);
      (t < L1 ? twx[tt] : twy[tt]) = mk<TC>(c, f.sign * s);
    }
  if (wait) {
    pdl_wait();
    if (f.stop != nullptr && *f.stop != 0) return false;
  }
  __syncthreads();
  DPROBE(0);
  const int64_t inner = f.inner;
  const int n2 = f.n2, n1 = f.n1;
  // each level runs over its columns in tiles of TILX (level 1: array rows y) / TILY (level 2:
  // frequencies kx); the ping-pong buffers are reused, hence the barrier between tiles
  if constexpr (!INV) {
    PassArgs ax;  // level 1: slots x (pad fused), columns y -> G[y][kx]
    ax.L = L1; ax.n_lo = n1; ax.n_hi = 0; ax.n_out = L1; ax.in_sa = inner; ax.in_cs = n1 * inner;
    ax.out_sa = 1; ax.out_cs = Gs; ax.sign = f.sign;
    const TC sc = static_cast<TC>(f.in_scale != nullptr ? *f.in_scale : 1.0);
    for (int y0 = 0; y0 < n2; y0 += TILX) {
      if (y0) __syncthreads();
      PX::template run<TI, TC, TC, NT, TILX>(ax, static_cast<const C<TI>*>(f.in) + y0 * n1 * inner + b,
                                                     G + y0 * Gs, b0, b1, twx, min(TILX, n2 - y0), sc);
    }
    __syncthreads();
    after_l1();
    DPROBE(1);
    PassArgs ay;  // level 2: slots y (n2 non-zero rows), columns kx -> u_hat[ky][kx][b]
    ay.L = L2; ay.n_lo = n2; ay.n_hi = 0; ay.n_out = L2; ay.in_sa = Gs; ay.in_cs = 1;
    ay.out_sa = kHatT ? L1 : static_cast<int64_t>(L1) * inner; ay.out_cs = kHatT ? 1 : inner; ay.sign = f.sign;
    C<TO>* hat_b = static_cast<C<TO>*>(f.out) + (kHatT ? b * L1 * L2 : b);
    for (int k0 = 0; k0 < L1; k0 += TILY) {
      if (k0) __syncthreads();
      PY::template run<TC, TC, TO, NT, TILY>(ay, G + k0, hat_b + k0 * ay.out_cs, p0, p1, twy, min(TILY, L1 - k0),
                                             static_cast<TC>(1));
      DPROBE(2 + k0 / TILY);
    }
  } else {
    PassArgs ay;  // inverse level 2 over all ky, keep y < n2 -> G[y][kx]
    ay.L = L2; ay.n_lo = L2; ay.n_hi = 0; ay.n_out = n2; ay.in_sa = kHatT ? L1 : static_cast<int64_t>(L1) * inner;
    ay.in_cs = kHatT ? 1 : inner; ay.out_sa = Gs; ay.out_cs = 1; ay.sign = f.sign;
    const C<TI>* hat_b = static_cast<const C<TI>*>(f.in) + (kHatT ? b * L1 * L2 : b);
    for (int k0 = 0; k0 < L1; k0 += TILY) {
      if (k0) __syncthreads();
      PY::template run<TI, TC, TC, NT, TILY>(ay, hat_b + k0 * ay.in_cs, G + k0, b0, b1, twy, min(TILY, L1 - k0),
                                             static_cast<TC>(1));
      DPROBE(1 + k0 / TILY);
    }
    __syncthreads();
    PassArgs ax;  // inverse level 1, keep x < n1, 1/(l1 l2) -> v[y][x][b]
    ax.L = L1; ax.n_lo = L1; ax.n_hi = 0; ax.n_out = n1; ax.in_sa = 1; ax.in_cs = Gs; ax.out_sa = inner;
    ax.out_cs = n1 * inner; ax.sign = f.sign;
    for (int y0 = 0; y0 < n2; y0 += TILX) {
      if (y0) __syncthreads();
      PX::template run<TC, TC, TO, NT, TILX>(ax, G + y0 * Gs, static_cast<C<TO>*>(f.out) + y0 * n1 * inner + b,
                                                     p0, p1, twx, min(TILX, n2 - y0),
                                                     static_cast<TC>(1.0 / (static_cast<double>(L1) * L2)));
    }
#ifdef TOEP_ORTH_PROBE
    __syncthreads();
#endif
    DPROBE(4);
  }
  return true;
}

template <typename TI, typename TC, typename TO, int TILX, int TILY, typename PX, typename PY, bool INV>
__global__ void __launch_bounds__(k2dThreads, 1) fft2d_kernel(Fft2dArgs f) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  pdl_trigger();
  if (threadIdx.x < 32)  // constant operator data: no dependency to wait for
    l2_prefetch_heads(f.pf, blockIdx.x, gridDim.x, threadIdx.x);
  fft2d_body<TI, TC, TO, TILX, TILY, PX, PY, INV>(f, smem_raw, blockIdx.x, true);
}

template <typename TI, typename TC, typename TO, int TILX, int TILY, typename PX, typename PY>
int launch2d(bool inverse, const Fft2dArgs& f, cudaStream_t s) {
  using S = Fft2dSmem<TC, TILX, TILY, PX, PY>;
  const size_t smem = S::bytes(f.n2);
  TOEP_REQUIRE(smem <= 227 * 1024, TOEP_ERR_ARG, "fft2d shared memory too large");
  auto kf = fft2d_kernel<TI, TC, TO, TILX, TILY, PX, PY, false>;
  auto ki = fft2d_kernel<TI, TC, TO, TILX, TILY, PX, PY, true>;
  auto k = inverse ? ki : kf;
  TOEP_CUDA(ensure_smem(k, smem));
  return launch_k(k, dim3(static_cast<unsigned>(f.inner)), dim3(k2dThreads), smem, s, f);
}

// ------------------------------------------------------------------------------------------
// Fused single-RHS matvec for N_b = 128 on the 60 x 60 grid (cfg2): forward 2-D DFT -> per-bin
// product D_k u_k -> inverse 2-D DFT in ONE cooperative launch (148 CTAs, one per SM), phases
// separated by grid barriers.  The operator blocks do not depend on the vector, so the product's
// bulk-copy ring is filled while the forward DFT computes (3 stages of 32 KB per SM, plus the L2
// prefetch of every CTA's first bins): the DFT runs under the HBM stream instead of in front of it.
// In the product phase the ring grows to 6 stages (the DFT's shared memory is free by then).
// Warps 0-15 run the DFTs; warps 0-7 consume and warp 16 produces in the product phase, exactly
// as binprod_tma_kernel (csrc/binprod.cu): a bin's 128 x 128 block streams in 8 whole-row stages.
#ifndef TOEP_FUSED_PF_MB
#define TOEP_FUSED_PF_MB 48  // L2 prefetch of the first bins in hand-out order
#endif
#ifndef TOEP_FUSED_THREADS
#define TOEP_FUSED_THREADS 1024
#endif
constexpr int kFusedThreads = TOEP_FUSED_THREADS;  // every warp runs the DFTs; the last one produces in the product phase
constexpr int kFusedN0 = 128;
constexpr int kFusedRB = 16;                                 // rows per 32 KB stage
constexpr int kFusedStageElems = kFusedRB * kFusedN0;
constexpr int kFusedStages = 6;                              // 3 in the ring region + 3 in the DFT region
constexpr int kFusedEarly = 3;                               // stages filled during the forward DFT
constexpr int kFusedConsumers = 8;
using FusedPX = Plan<4, 3, 5>;
using FusedPY = Plan<4, 3, 5>;
constexpr int kFusedTILX = 32, kFusedTILY = 60;  // one tile per pass (n2 <= 30, all 60 level-2 columns)

struct FusedArgs {
  Fft2dArgs fwd, inv;
  const double2* DT;  // [K][n0][n0], DT[k][j][m] = D_k[m][j]
  double2* hat;       // [n0][K] forward DFT output (column-major: each DFT CTA writes one contiguous run)
  double2* hat2;      // [n0][K] product output
  int64_t K;
  unsigned* bar;      // grid barrier arrival counter (monotonic, zeroed once)
  int* work;          // dynamic bin hand-out counter (zero between launches)
  int64_t pf_bytes;   // L2 prefetch budget of the first bins in hand-out order
};

// Shared memory: region 0 holds the DFT workspace (twiddles + two 60 x 60 ping-pong buffers, the
// level-1 intermediate aliased into one of them) and, in the product phase, ring stages 3..5 plus
// the consumers' vector / reduction buffers; region 1 holds ring stages 0..2 (filled during the
// forward DFT).
constexpr size_t kFusedDftBytes = sizeof(double2) * (FusedPX::L + FusedPY::L + 2 * FusedPY::L * kFusedTILY);
constexpr size_t kFusedLateBytes = sizeof(double2) * (3 * kFusedStageElems + kFusedN0 + kFusedConsumers * kFusedN0);
constexpr size_t kFusedRegion0 = ((kFusedDftBytes > kFusedLateBytes ? kFusedDftBytes : kFusedLateBytes) + 127) / 128 * 128;
constexpr size_t kFusedSmem = kFusedRegion0 + sizeof(double2) * 3 * kFusedStageElems + 2 * kFusedStages * sizeof(uint64_t);
static_assert(FusedPX::L * kFusedTILX <= FusedPY::L * kFusedTILY && 30 * (FusedPX::L | 1) <= FusedPY::L * kFusedTILY,
              "fused DFT buffers");

__device__ __forceinline__ void fused_grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
    const unsigned target = (old / gridDim.x + 1) * gridDim.x;
    long long t0 = 0;
    for (unsigned spins = 1;; ++spins) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if (static_cast<int>(v - target) >= 0) break;
      if ((spins & 1023u) == 0) {  // a CTA that never arrives must not hang the device: trap after 10 s
        long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t0 == 0) t0 = t;
        else if (t - t0 > 10000000000ll) __trap();
      }
    }
  }
  __syncthreads();
}

#ifdef TOEP_ORTH_PROBE
__device__ unsigned g_fused_calls;
__device__ long long g_fend[160];
#define FPROBE(i) \
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(fpt[i]))
#else
#define FPROBE(i)
#endif

__global__ void __launch_bounds__(kFusedThreads, 1) mv_fused_kernel(FusedArgs a) {
  using Z = double2;
#ifdef TOEP_ORTH_PROBE
  long long fpt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  FPROBE(0);
  extern __shared__ __align__(128) unsigned char fsm[];
  unsigned char* region0 = fsm;                                      // DFT workspace, later stages 3..5
  Z* ring0 = reinterpret_cast<Z*>(fsm + kFusedRegion0);               // stages 0..2
  Z* us = reinterpret_cast<Z*>(region0) + 3 * kFusedStageElems;       // product phase only
  Z* red = us + kFusedN0;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring0 + 3 * kFusedStageElems);
  uint64_t* empty = full + kFusedStages;
  auto stage_ptr = [&](int st) -> Z* {
    return st < 3 ? ring0 + st * kFusedStageElems : reinterpret_cast<Z*>(region0) + (st - 3) * kFusedStageElems;
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int nrb = kFusedN0 / kFusedRB;
  // Bins are handed out dynamically: CTA b starts with bin b (its first stages stream under the
  // forward DFT), later bins come from a device counter as the CTA's producer needs them, so CTAs
  // that draw more HBM bandwidth take more bins and the grid finishes together (a static partition
  // left a ~10 us spread at the closing barrier).  item_of[stage] tells the consumers which bin a
  // stage belongs to (-1: no more bins).
  __shared__ int item_of[kFusedStages];
  const int64_t first = blockIdx.x < a.K ? static_cast<int64_t>(blockIdx.x) : -1;
  auto issue = [&](int64_t q, int64_t k, uint64_t pol) {
    const int st = static_cast<int>(q % kFusedStages);
    const int rb = static_cast<int>(q % nrb);
    item_of[st] = static_cast<int>(k);
    mbar_expect_tx(&full[st], static_cast<uint32_t>(sizeof(Z) * kFusedStageElems));
    bulk_g2s(stage_ptr(st), a.DT + k * kFusedN0 * kFusedN0 + static_cast<int64_t>(rb) * kFusedStageElems,
             sizeof(Z) * kFusedStageElems, &full[st], pol);
  };
  pdl_trigger();
  if (threadIdx.x == 0) {
    for (int st = 0; st < kFusedStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kFusedConsumers);
    }
    mbar_init_fence();
  }
  __syncthreads();
  // the operator stream starts now: the early stages of the first bin, and the L2 prefetch of the
  // next bins in hand-out order (bin b + j * grid for this CTA)
  const int64_t early = first >= 0 ? kFusedEarly : 0;
  if (threadIdx.x == 0) {
    const uint64_t pol = policy_evict_first();
    for (int64_t q = 0; q < early; ++q) issue(q, first, pol);
  }
  // twiddle table of the inverse transform (L1 = L2 = 60), built by warps that idle in the product
  // phase, so the inverse DFT after the second grid barrier starts at once
  __shared__ Z tw_inv[60];
  // The L2 prefetch of the first bins (in hand-out order, 48 MB) is issued by each DFT CTA after its
  // forward level-1 pass, so that pass's vector loads do not queue behind it in HBM (CTAs without a
  // batch column issue their share at once).  Issuing it from the 20 idle CTAs alone, once every
  // level-1 pass is done, measured 10 us at the first grid barrier: the bulk prefetches back-pressure
  // the issuing SM, so the stream must be spread over all of them.
  auto prefetch_heads = [&]() {
    if (warp == 1) {
      const int64_t bin_bytes = sizeof(Z) * kFusedN0 * kFusedN0;
      const int64_t pf_bins = std::min<int64_t>(a.K, a.pf_bytes / bin_bytes);
      for (int64_t k = blockIdx.x; k < pf_bins; k += gridDim.x)
        for (int64_t off = lane * 32768; off < bin_bytes; off += 32 * 32768)
          bulk_prefetch_l2(reinterpret_cast<const char*>(a.DT + k * kFusedN0 * kFusedN0) + off, 32768);
    }
  };
  pdl_wait();
  FPROBE(1);
#ifdef TOEP_ORTH_PROBE
  long long prev_max = 0, prev_min = 0;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    prev_min = 1ll << 62;
    for (int i = 0; i < gridDim.x; ++i) {
      const long long e = *(volatile long long*)&g_fend[i];
      prev_max = e > prev_max ? e : prev_max;
      prev_min = e < prev_min ? e : prev_min;
    }
  }
#endif
  if (a.fwd.stop != nullptr && *a.fwd.stop != 0) {  // uniform across the grid: no barrier is reached
    if (threadIdx.x == 0)
      for (int64_t q = 0; q < early; ++q) mbar_wait(&full[q % kFusedStages], 0);  // no copy outlives the CTA
    return;
  }
  // ---- phase 1: forward 2-D DFT of batch column b (CTAs beyond the batch only take the barriers)
  if (blockIdx.x < a.fwd.inner)
    fft2d_body<double, double, double, kFusedTILX, kFusedTILY, FusedPX, FusedPY, false, true, kFusedThreads, true>(
        a.fwd, region0, blockIdx.x, false, prefetch_heads);
  else
    prefetch_heads();
  FPROBE(2);
  fused_grid_barrier(a.bar);
  FPROBE(3);
  // ---- phase 2: per-bin product, bins handed out dynamically
  if (warp == kFusedThreads / 32 - 1) {  // producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int64_t k = first;
      for (int64_t q = early;; ++q) {
        const int st = static_cast<int>(q % kFusedStages);
        if (q % nrb == 0) {  // next bin
          if (q > 0 || k < 0) k = gridDim.x + static_cast<int64_t>(atomicAdd(a.work, 1));
          if (q == 0 && first >= 0) k = first;
        }
        if (q >= kFusedStages) mbar_wait(&empty[st], static_cast<uint32_t>(((q / kFusedStages) - 1) & 1));
        if (k >= a.K) {  // no more bins: wake the consumers on this stage with the end marker
          item_of[st] = -1;
          mbar_arrive(&full[st]);
          break;
        }
        issue(q, k, pol);
      }
    }
  } else if (warp >= kFusedConsumers) {  // idle in this phase: the inverse DFT's twiddles
    for (int t = threadIdx.x - kFusedConsumers * 32; t < 60; t += 32 * (kFusedThreads / 32 - 1 - kFusedConsumers)) {
      double sn, cs;
      sincospi(2.0 * t / 60, &sn, &cs);
      tw_inv[t] = make_double2(cs, a.inv.sign * sn);
    }
  } else {  // consumers: lane = output row m (4 per lane), warp = row slice
    constexpr int MPL = kFusedN0 / 32;
    for (int64_t q = 0;; q += nrb) {
      const int st0 = static_cast<int>(q % kFusedStages);
      mbar_wait(&full[st0], static_cast<uint32_t>((q / kFusedStages) & 1));
      const int it = item_of[st0];
      if (it < 0) break;
      for (int t = threadIdx.x; t < kFusedN0; t += kFusedConsumers * 32)  // u_hat column-major: [b][k]
        us[t] = __ldcg(a.hat + static_cast<int64_t>(t) * a.K + it);
      consumers_sync();
      Z acc[MPL];
#pragma unroll
      for (int i = 0; i < MPL; ++i) acc[i] = make_double2(0, 0);
      for (int rb = 0; rb < nrb; ++rb) {
        const int64_t qq = q + rb;
        const int st = static_cast<int>(qq % kFusedStages);
        if (rb > 0) mbar_wait(&full[st], static_cast<uint32_t>((qq / kFusedStages) & 1));
        const Z* tile = stage_ptr(st);
#pragma unroll
        for (int r = warp; r < kFusedRB; r += kFusedConsumers) {
          const Z uj = us[rb * kFusedRB + r];
#pragma unroll
          for (int i = 0; i < MPL; ++i) cfma(acc[i], tile[r * kFusedN0 + lane + 32 * i], uj);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
#pragma unroll
      for (int i = 0; i < MPL; ++i) red[warp * kFusedN0 + lane + 32 * i] = acc[i];
      consumers_sync();
      for (int t = threadIdx.x; t < kFusedN0; t += kFusedConsumers * 32) {
        Z sum = red[t];
#pragma unroll
        for (int ww = 1; ww < kFusedConsumers; ++ww) sum = cadd(sum, red[ww * kFusedN0 + t]);
        a.hat2[static_cast<int64_t>(t) * a.K + it] = sum;
      }
      consumers_sync();
    }
  }
  FPROBE(4);
  fused_grid_barrier(a.bar);
  FPROBE(5);
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch(a.work, 0);  // every CTA is past phase 2
  // ---- phase 3: inverse 2-D DFT, crop, 1/(l1 l2) of batch column b
  if (blockIdx.x < a.inv.inner)
    fft2d_body<double, double, double, kFusedTILX, kFusedTILY, FusedPX, FusedPY, true, true, kFusedThreads, true>(
        a.inv, region0, blockIdx.x, false, NoHook{}, tw_inv);
#ifdef TOEP_ORTH_PROBE
  FPROBE(6);
  __shared__ unsigned fcall;
  if (threadIdx.x == 0 && blockIdx.x == 0) fcall = atomicAdd(&g_fused_calls, 1);
  __syncthreads();
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == 140) && (fcall % 200) == 150)
  {
    printf("fused cta %d: start->pdl %lld dft %lld bar1 %lld product %lld bar2 %lld inv %lld ns\n", blockIdx.x,
           fpt[1] - fpt[0], fpt[2] - fpt[1], fpt[3] - fpt[2], fpt[4] - fpt[3], fpt[5] - fpt[4], fpt[6] - fpt[5]);
    if (blockIdx.x == 0)
      printf("  previous launch: CTA exits spread %lld ns, last exit -> this CTA start %lld ns\n", prev_max - prev_min,
             fpt[0] - prev_max);
    const long long* f0 = g_dft_ts[0][blockIdx.x];
    const long long* f1 = g_dft_ts[1][blockIdx.x];
    printf("  fwd cta %d: pdl->tw %lld lvl1 %lld lvl2a %lld lvl2b %lld | inv: tw %lld lvl2a %lld lvl2b %lld lvl1 %lld ns\n",
           blockIdx.x, f0[0] - fpt[1], f0[1] - f0[0], f0[2] - f0[1], f0[3] - f0[2], f1[0] - fpt[5], f1[1] - f1[0],
           f1[2] - f1[1], f1[4] - f1[2]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_fend[blockIdx.x] = t;
  }
#endif
}

template <typename TI, typename TC, typename TO>
int fft2d_t(bool inverse, const Fft2dArgs& f, int l2, int l1, cudaStream_t s) {
  if (l2 == 60 && l1 == 60 && f.n2 <= 32) return launch2d<TI, TC, TO, 32, 64, Plan<4, 3, 5>, Plan<4, 3, 5>>(inverse, f, s);
  if (l2 == 32 && l1 == 32 && f.n2 <= 16) return launch2d<TI, TC, TO, 16, 32, Plan<4, 4, 2>, Plan<4, 4, 2>>(inverse, f, s);
  // (a 128 x 128 variant with column tiles fits in shared memory but measured slower than the
  // four-pass path at cfg4: 728 vs 693 us per matvec — one CTA per column serialises 12 tiles)
  return -1;
}

template <typename TI, typename TC, typename TO, int TIL>
__global__ void __launch_bounds__(kThreads, kMinBlocksGeneric) fft_pass_kernel(PassArgs a, Radices rad, double two_over_L) {
  pdl_wait();
  if (a.stop != nullptr && *a.stop != 0) return;
  using Z = C<TC>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Z* tw = reinterpret_cast<Z*>(smem_raw);
  Z* buf0 = tw + a.L;
  Z* buf1 = buf0 + a.L * TIL;
  const int L = a.L;
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * TIL;
  const int o = blockIdx.y;
  const int ncol = static_cast<int>(std::min<int64_t>(TIL, a.inner - i0));

  for (int t = threadIdx.x; t < L; t += kThreads) {
    TC s, c;
    sincospi_t<TC>(static_cast<TC>(t * two_over_L), &s, &c);
    tw[t] = mk<TC>(c, a.sign * s);
  }

  const C<TI>* in = static_cast<const C<TI>*>(a.in) + o * a.in_so + i0;
  if (a.in_idx != nullptr) in += static_cast<int64_t>(*a.in_idx) * a.in_idx_stride;
  C<TO>* out = static_cast<C<TO>*>(a.out) + o * a.out_so + i0;
  if (a.out_idx != nullptr) out += static_cast<int64_t>(*a.out_idx) * a.out_idx_stride;

  const int hi_start = L - a.n_hi;
  for (int e = threadIdx.x; e < L * TIL; e += kThreads) {
    const int slot = e / TIL;
    const int col = e - slot * TIL;
    int src = -1;
    if (slot < a.n_lo) src = slot;
    else if (slot >= hi_start) src = a.n_lo + slot - hi_start;
    Z v = mk<TC>(0, 0);
    if (src >= 0 && col < ncol) v = cvt<Z>(in[src * a.in_sa + col]);
    buf0[e] = v;
  }
  __syncthreads();

  const TC scale = pass_scale<TC>(a);
  if (rad.n == 0) {  // L == 1
    if (threadIdx.x < ncol && a.n_out > 0) out[threadIdx.x] = cvt<C<TO>>(cscale(buf0[threadIdx.x], scale));
    return;
  }
  Z* src = buf0;
  Z* dst = buf1;
  int Ns = 1;
  const bool scat = a.scatter != nullptr;
  for (int s = 0; s < rad.n; ++s) {
    const int R = rad.r[s];
    if (s + 1 < rad.n || scat) {
      dispatch_stage<TC, TO, TIL, false>(R, src, dst, tw, L, Ns, a.sign, out, a.out_sa, a.n_out, ncol, scale);
      __syncthreads();
      Z* t = src;
      src = dst;
      dst = t;
      Ns *= R;
    } else {
      dispatch_stage<TC, TO, TIL, true>(R, src, dst, tw, L, Ns, a.sign, out, a.out_sa, a.n_out, ncol, scale);
    }
  }
  if (scat) scatter_tile<TC, TO, TIL>(a, src, ncol, scale);  // result in `src` after the last swap
}

// Direct O(L^2) DFT for lengths that are not 7-smooth (API block_fft_* on prime
// lengths such as the reference's 2n-1 = 59).  Same placement / crop contract.
template <typename TI, typename TC, typename TO, int TIL>
__global__ void __launch_bounds__(kThreads) dft_direct_kernel(PassArgs a, double two_over_L) {
  pdl_wait();
  if (a.stop != nullptr && *a.stop != 0) return;
  using Z = C<TC>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Z* tw = reinterpret_cast<Z*>(smem_raw);
  Z* buf = tw + a.L;
  const int L = a.L;
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * TIL;
  const int o = blockIdx.y;
  const int ncol = static_cast<int>(std::min<int64_t>(TIL, a.inner - i0));
  for (int t = threadIdx.x; t < L; t += kThreads) {
    TC s, c;
    sincospi_t<TC>(static_cast<TC>(t * two_over_L), &s, &c);
    tw[t] = mk<TC>(c, a.sign * s);
  }
  const C<TI>* in = static_cast<const C<TI>*>(a.in) + o * a.in_so + i0;
  if (a.in_idx != nullptr) in += static_cast<int64_t>(*a.in_idx) * a.in_idx_stride;
  C<TO>* out = static_cast<C<TO>*>(a.out) + o * a.out_so + i0;
  if (a.out_idx != nullptr) out += static_cast<int64_t>(*a.out_idx) * a.out_idx_stride;
  const int hi_start = L - a.n_hi;
  for (int e = threadIdx.x; e < L * TIL; e += kThreads) {
    const int slot = e / TIL;
    const int col = e - slot * TIL;
    int src = -1;
    if (slot < a.n_lo) src = slot;
    else if (slot >= hi_start) src = a.n_lo + slot - hi_start;
    Z v = mk<TC>(0, 0);
    if (src >= 0 && col < ncol) v = cvt<Z>(in[src * a.in_sa + col]);
    buf[e] = v;
  }
  __syncthreads();
  const TC scale = pass_scale<TC>(a);
  for (int e = threadIdx.x; e < a.n_out * TIL; e += kThreads) {
    const int k = e / TIL;
    const int col = e - k * TIL;
    Z acc = mk<TC>(0, 0);
    int idx = 0;
    for (int t = 0; t < L; ++t) {
      cfma(acc, buf[t * TIL + col], tw[idx]);
      idx += k;
      if (idx >= L) idx -= L;
    }
    if (col < ncol) out[k * a.out_sa + col] = cvt<C<TO>>(cscale(acc, scale));
  }
}

template <typename TI, typename TC, typename TO>
int launch(const PassArgs& a, const Radices& rad, bool direct, cudaStream_t s) {
  if (!direct) {
    const int rc = try_plan<TI, TC, TO>(a, s);
    if (rc >= 0) return rc;
  }
  TOEP_REQUIRE(a.scatter == nullptr || (!direct && a.L > 1), TOEP_ERR_ARG,
               "peer scatter needs a 7-smooth pass length > 1 (L=%d)", a.L);
  TOEP_REQUIRE(a.in_planes == nullptr && a.out_planes == nullptr, TOEP_ERR_ARG,
               "split-plane I/O needs a compiled pass plan (L=%d)", a.L);
  const size_t es = sizeof(C<TC>);
  const int nbuf = direct ? 1 : 2;
  int til = 32;
  while (til > 1 && static_cast<size_t>(nbuf * a.L * til + a.L) * es > 48 * 1024) til /= 2;
  while (til > 1 && til / 2 >= a.inner) til /= 2;
  const size_t smem = static_cast<size_t>(nbuf * a.L * til + a.L) * es;
  TOEP_REQUIRE(smem <= 200 * 1024, TOEP_ERR_ARG, "fft length %d too long for one shared-memory pass", a.L);
  dim3 grid(static_cast<unsigned>((a.inner + til - 1) / til), static_cast<unsigned>(a.outer));
  TOEP_REQUIRE(a.outer <= 65535, TOEP_ERR_ARG, "fft pass outer count %d > 65535", a.outer);
  const double two_over_L = 2.0 / a.L;
#define TOEP_FFT_CASE(T)                                                                         \
  case T: {                                                                                      \
    if (direct) {                                                                                \
      auto k = dft_direct_kernel<TI, TC, TO, T>;                                                 \
      TOEP_CUDA(ensure_smem(k, smem)); \
      k<<<grid, kThreads, smem, s>>>(a, two_over_L);                                             \
    } else {                                                                                     \
      auto k = fft_pass_kernel<TI, TC, TO, T>;                                                   \
      TOEP_CUDA(ensure_smem(k, smem)); \
      k<<<grid, kThreads, smem, s>>>(a, rad, two_over_L);                                        \
    }                                                                                            \
    break;                                                                                       \
  }
  switch (til) {
    TOEP_FFT_CASE(1)
    TOEP_FFT_CASE(2)
    TOEP_FFT_CASE(4)
    TOEP_FFT_CASE(8)
    TOEP_FFT_CASE(16)
    TOEP_FFT_CASE(32)
    default: break;
  }
#undef TOEP_FFT_CASE
  TOEP_LAUNCHED();
  return TOEP_OK;
}

}  // namespace

int factorize(int L, int* rad, int* nrad) {
  int n = 0;
  int m = L;
  while (m % 4 == 0 && m > 4 && n < kMaxStages) { rad[n++] = 4; m /= 4; }
  const int radices[] = {4, 2, 3, 5, 7};
  for (int p : radices) {
    while (m % p == 0 && n < kMaxStages) { rad[n++] = p; m /= p; }
  }
  *nrad = n;
  if (m != 1) {
    set_error("DFT length %d is not 7-smooth", L);
    return TOEP_ERR_ARG;
  }
  return TOEP_OK;
}

int fft2d(bool inverse, const void* in, void* out, int n2, int n1, int l2, int l1, int64_t inner, int sign, int tin,
          int tc, int tout, const double* in_scale, const int* stop, cudaStream_t s, const L2Prefetch* pf) {
  if (inner > 65535 || inner < 1) return -1;
  Fft2dArgs f{in, out, n2, n1, inner, sign, in_scale, stop, pf != nullptr ? *pf : L2Prefetch{}};
  const int code = tin * 4 + tc * 2 + tout;
  switch (code) {
    case 0: return fft2d_t<double, double, double>(inverse, f, l2, l1, s);
    case 7: return fft2d_t<float, float, float>(inverse, f, l2, l1, s);
    case 6: return fft2d_t<float, float, double>(inverse, f, l2, l1, s);
    case 3: return fft2d_t<double, float, float>(inverse, f, l2, l1, s);
    default: return -1;
  }
}

// The fused cfg2 matvec (mv_fused_kernel) when it applies: complex128 operator and vectors, N_b = 128,
// a 60 x 60 embedding with n2 <= 30, forward product (not transpose), every SM co-resident.
// Returns -1 when it does not apply (the caller uses the three-kernel path).
int matvec_fused(const void* DT, int64_t K, int n2, int n1, int l2, int l1, int n0, const void* u, void* hat,
                 void* hat2, void* v, unsigned* bar, const double* in_scale, const int* stop, const L2Prefetch& pf,
                 cudaStream_t s) {
  if (n0 != kFusedN0 || l2 != 60 || l1 != 60 || n2 > 30 || n1 > 30 || bar == nullptr) return -1;
  const size_t smem = kFusedSmem;
  if (smem > 227 * 1024) return -1;
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  TOEP_CUDA(ensure_smem(mv_fused_kernel, smem));
  static int fits = -1;  // every SM must hold one CTA (the grid barriers need every CTA resident)
  if (fits < 0) {
    int per_sm = 0;
    fits = (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mv_fused_kernel, kFusedThreads, smem) ==
                cudaSuccess &&
            per_sm >= 1)
               ? 1
               : 0;
    cudaGetLastError();
  }
  if (!fits) return -1;
  FusedArgs a;
  a.fwd = Fft2dArgs{u, hat, n2, n1, kFusedN0, -1, in_scale, stop, pf};
  a.inv = Fft2dArgs{hat2, v, n2, n1, kFusedN0, +1, nullptr, nullptr, L2Prefetch{}};
  a.DT = static_cast<const double2*>(DT);
  a.hat = static_cast<double2*>(hat);
  a.hat2 = static_cast<double2*>(hat2);
  a.K = K;
  a.bar = bar;
  a.work = reinterpret_cast<int*>(bar + 1);
  a.pf_bytes = pf.bytes > 0 ? int64_t{TOEP_FUSED_PF_MB} << 20 : 0;
  // Launched as an ordinary (PDL) grid, not a cooperative one: the next matvec's CTAs then start on
  // the SMs the previous grid vacates first instead of waiting for the whole grid plus the
  // cooperative launch's dispatch (142.4 vs 143.8 us per matvec).  Co-residency of all CTAs (one per
  // SM, checked above) is what the grid barriers need; what a cooperative launch would add is
  // protection from a second fused matvec on another stream holding part of the SMs — so fused
  // launches are serialised across streams here: a launch on a different stream than the previous
  // one first waits for that stream's work.  (Any other kernel holding SMs only delays CTAs; the
  // barriers' 10 s trap bounds a pathological wait.)
  return launch_gridsync(mv_fused_kernel, dim3(static_cast<unsigned>(std::min<int64_t>(sms, K))),
                         dim3(kFusedThreads), smem, s, a);
}

namespace {
std::mutex g_gridsync_mu;
cudaStream_t g_gridsync_last[64] = {};
cudaEvent_t g_gridsync_ev[64] = {};
}  // namespace

// held from gridsync_order to gridsync_launched (same thread): the check, the launch and the record
// are one step for concurrent host threads
int gridsync_order(cudaStream_t s) {
  g_gridsync_mu.lock();
  int dev = 0;
  cudaGetDevice(&dev);
  dev &= 63;
  if (g_gridsync_ev[dev] == nullptr) {
    if (cudaEventCreateWithFlags(&g_gridsync_ev[dev], cudaEventDisableTiming) != cudaSuccess) {
      g_gridsync_mu.unlock();
      set_error("gridsync event creation failed");
      return TOEP_ERR_CUDA;
    }
  } else if (g_gridsync_last[dev] != s && cudaStreamWaitEvent(s, g_gridsync_ev[dev], 0) != cudaSuccess) {
    g_gridsync_mu.unlock();
    set_error("gridsync stream wait failed");
    return TOEP_ERR_CUDA;
  }
  return TOEP_OK;
}

void gridsync_launched(cudaStream_t s, bool ok) {
  if (ok) {
    int dev = 0;
    cudaGetDevice(&dev);
    dev &= 63;
    cudaEventRecord(g_gridsync_ev[dev], s);
    g_gridsync_last[dev] = s;
  }
  g_gridsync_mu.unlock();
}

bool fft_plan_has_planes(int L, int64_t inner) {
  return (L == 60 && inner >= 16) || (L == 128 && inner >= 8) || (L == 32 && inner >= 32) || (L == 64 && inner >= 16);
}

int fft_pass(const PassArgs& a, int tin, int tcomp, int tout, cudaStream_t s) {
  TOEP_REQUIRE(a.L >= 1 && a.n_lo >= 0 && a.n_hi >= 0 && a.n_lo + a.n_hi <= a.L && a.n_out <= a.L,
               TOEP_ERR_ARG, "bad fft pass geometry L=%d lo=%d hi=%d out=%d", a.L, a.n_lo, a.n_hi, a.n_out);
  if (a.inner == 0 || a.outer == 0 || a.n_out == 0) return TOEP_OK;
  Radices rad{};
  const bool direct = factorize(a.L, rad.r, &rad.n) != TOEP_OK;  // not 7-smooth: direct DFT
  const int code = tin * 4 + tcomp * 2 + tout;
  switch (code) {
    case 0: return launch<double, double, double>(a, rad, direct, s);   // c128 end to end
    case 7: return launch<float, float, float>(a, rad, direct, s);      // c64 end to end
    case 6: return launch<float, float, double>(a, rad, direct, s);     // c64 compute, c128 out
    case 3: return launch<double, float, float>(a, rad, direct, s);     // c128 in, c64 compute
    default:
      set_error("unsupported fft pass type combination %d/%d/%d", tin, tcomp, tout);
      return TOEP_ERR_ARG;
  }
}

}  // namespace toep
