// Hand-written FP64 tensor-core GEMMs for sm_100a (DMMA: mma.sync.aligned.m8n8k4.f64).
//
// sm_100a has no tcgen05 kind for f64 (ptxas rejects .kind::f64), so the FP64 tensor-core path on
// B200 is the warp-level DMMA instruction.  These kernels replace a library template for every
// FP64 product on the hot path:
//   * dgemm: real C = alpha A B + beta C — the three real products of the 3M (Gauss) complex block
//     products of the block-Rybicki recursion (rybicki.py:114-133) and of the multi-RHS per-bin
//     products on split planes (toeplitz.py:300 at W >= 16, when the int8 path is off);
//   * zgemm: complex C = alpha A B + beta C (four real DMMA per complex k-step) — the P_K fold into
//     the operator (precond.py:124-131), the LU trailing updates and triangular-solve updates of the
//     recursion's denominators, and the generic complex GEMM entry point.
//
// Tiling: a CTA owns a BM x BN output tile, 32 x 32 per warp (4 x 4 DMMA 8x8 accumulator tiles),
// and walks K in BK-deep stages through a STAGES-deep cp.async ring (zero-filled at the edges, so
// any m, n, k).  Operands keep their global orientation in shared memory (row-major A stays
// [m][k], column-major A is [k][m], likewise B) with row strides padded so that each DMMA
// fragment load (lane -> (row lane/4, k lane%4)) is bank-conflict free:
//   8-byte loads (16 lanes per phase): stride = 4 mod 16 doubles;
//   16-byte complex loads (8 lanes per phase): stride = 4 mod 8 ([x][k]) or 2 mod 8 ([k][x]).
// Any operand with one unit stride is covered; a column-major C is computed as C^T = B^T A^T.
#include "kernels.cuh"
#include "launch.cuh"

namespace toep {

void keep_pool();  // op.cu

namespace {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct GArgs {
  int64_t m, n, k;
  double2 alpha, beta;  // real kernel: .x only
  const void* a;
  int64_t lda, a_bs;
  const void* b;
  int64_t ldb, b_bs;
  void* c;
  int64_t ldc, c_bs;
  const int* stop;  // optional device flag: non-zero -> the launch is a no-op
  // real kernel: up to 3 independent operand triples ("planes", e.g. the re / im / re+im planes of
  // a 3M product) of identical shape and strides in ONE launch: blockIdx.z = batch * planes + plane
  int planes;
  const void* pa[3];
  const void* pb[3];
  void* pc[3];
  // real kernel split-K: blockIdx.z = (batch * planes + plane) * ksplit + split; with ksplit > 1
  // each split writes its raw partial tile to work[split][batch * planes + plane][m][n] and
  // dsplit_reduce forms C = alpha sum_s work[s] + beta C in a fixed order (deterministic)
  int ksplit;
  int ktiles_per_split;
  double* work;
};

// Copies of one operand tile per k-stage with the addressing fixed once per CTA: the non-k
// coordinate of each copy (and so its validity) never changes, only the k offset moves, and only
// the last k-tile needs a k bound check.  KC: k is the contiguous dimension of the tile's rows.
template <int E, int CH, int R, int CC, int S, int NT, bool KC>
struct TileLoader {
  static constexpr int EPC = CH / E, PER_ROW = CC / EPC, TOTAL = R * PER_ROW;
  static constexpr int N = (TOTAL + NT - 1) / NT;
  static_assert(CC % EPC == 0, "tile width");
  const char* src[N];  // address of the copy at k-tile 0
  int fixed[N];        // bytes the fixed coordinate allows (0: outside; -1: no copy)
  int64_t kstep;       // bytes per k-tile
  const char* any;     // a valid address for zero-filled copies

  __device__ __forceinline__ void init(const char* g, int64_t ld, int64_t x0, int64_t xmax, int bk) {
    any = g;
    kstep = KC ? static_cast<int64_t>(bk) * E : static_cast<int64_t>(bk) * ld * E;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const int i = j * NT + static_cast<int>(threadIdx.x);
      const int r = i / PER_ROW, c = (i - r * PER_ROW) * EPC;
      if (i >= TOTAL) { fixed[j] = -1; src[j] = g; continue; }
      if constexpr (KC) {  // rows: the non-k coordinate, columns: k
        const int64_t gx = x0 + r;
        fixed[j] = gx < xmax ? CH : 0;
        src[j] = g + (gx * ld + c) * E;
      } else {             // rows: k, columns: the non-k coordinate
        const int64_t gx = x0 + c;
        fixed[j] = gx < xmax ? static_cast<int>(std::min<int64_t>(EPC, xmax - gx)) * E : 0;
        src[j] = g + (static_cast<int64_t>(r) * ld + gx) * E;
      }
    }
  }
  // k-tile kt into the stage at `sm`; `full`: the whole tile lies below kmax
  __device__ __forceinline__ void load(char* sm, int kt, int bk, int64_t kmax, bool full) const {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if (TOTAL % NT != 0 && fixed[j] < 0) continue;
      const int i = j * NT + static_cast<int>(threadIdx.x);
      const int r = i / PER_ROW, c = (i - r * PER_ROW) * EPC;
      int valid = fixed[j];
      if (!full) {
        const int64_t kk = static_cast<int64_t>(kt) * bk + (KC ? c : r);
        if (kk >= kmax) valid = 0;
        else if (KC && valid) valid = static_cast<int>(std::min<int64_t>(EPC, kmax - kk)) * E;
      }
      const char* p = src[j] + kt * kstep;
      cp_async<CH>(sm + (r * S + c) * E, valid ? p : any, valid);
    }
  }
};

// ------------------------------------------------------------------------------------ real
// AK: A is row-major (k contiguous).  BKC: B is column-major (k contiguous).  VEC: 16-byte copies
// (every operand row start 16-byte aligned), else 8-byte copies.  Warp tile WM x WN (WM/8 x WN/8
// DMMA accumulator tiles per warp).
template <bool AK, bool BKC, int BM, int BN, int BK, int WM, int WN, int STAGES, bool VEC>
struct DCfg {
  static constexpr int kWarpsM = BM / WM, kWarpsN = BN / WN;
  static constexpr int kThreads = kWarpsM * kWarpsN * 32;
  static constexpr int MI = WM / 8, NJ = WN / 8;
  static constexpr int SA = AK ? BK + 4 : BM + 4;  // shared row stride (doubles)
  static constexpr int SB = BKC ? BK + 4 : BN + 4;
  static constexpr int kATile = (AK ? BM : BK) * SA;  // doubles per stage
  static constexpr int kBTile = (BKC ? BN : BK) * SB;
  static constexpr size_t kSmem = static_cast<size_t>(STAGES) * (kATile + kBTile) * sizeof(double);
  static_assert((SA % 16 == 4 || SA % 16 == 12) && (SB % 16 == 4 || SB % 16 == 12), "conflict-free fragment strides");
};

template <bool AK, bool BKC, int BM, int BN, int BK, int WM, int WN, int STAGES, bool VEC>
__global__ void __launch_bounds__(DCfg<AK, BKC, BM, BN, BK, WM, WN, STAGES, VEC>::kThreads)
    dgemm_kernel(GArgs g) {
  using Cfg = DCfg<AK, BKC, BM, BN, BK, WM, WN, STAGES, VEC>;
  constexpr int NT = Cfg::kThreads, SA = Cfg::SA, SB = Cfg::SB, MI = Cfg::MI, NJ = Cfg::NJ;
  constexpr int CH = VEC ? 16 : 8;
  if (g.stop != nullptr && *g.stop) return;
  extern __shared__ __align__(16) double dsm[];
  double* As = dsm;
  double* Bs = dsm + STAGES * Cfg::kATile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp % Cfg::kWarpsM, wn = warp / Cfg::kWarpsM;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM, n0 = static_cast<int64_t>(blockIdx.x) * BN;
  const int split = static_cast<int>(blockIdx.z % g.ksplit);
  const int64_t zz = blockIdx.z / g.ksplit;  // batch * planes + plane
  const int plane = static_cast<int>(zz % g.planes);
  const int64_t bz = zz / g.planes;
  const char* A = static_cast<const char*>(g.pa[plane]) + bz * g.a_bs * 8;
  const char* B = static_cast<const char*>(g.pb[plane]) + bz * g.b_bs * 8;
  double* C = static_cast<double*>(g.pc[plane]) + bz * g.c_bs;
  const int ktiles_all = static_cast<int>((g.k + BK - 1) / BK);
  const int kt0 = split * g.ktiles_per_split;
  const int kt1 = std::min(ktiles_all, kt0 + g.ktiles_per_split);
  const int ktiles = std::max(0, kt1 - kt0);

  TileLoader<8, CH, AK ? BM : BK, AK ? BK : BM, SA, NT, AK> la;
  TileLoader<8, CH, BKC ? BN : BK, BKC ? BK : BN, SB, NT, BKC> lb;
  la.init(A, g.lda, m0, g.m, BK);
  lb.init(B, g.ldb, n0, g.n, BK);
  auto load_stage = [&](int t, int slot) {  // t: k-tile index within this split
    const int kt = kt0 + t;
    const bool full = static_cast<int64_t>(kt + 1) * BK <= g.k;
    la.load(reinterpret_cast<char*>(As + slot * Cfg::kATile), kt, BK, g.k, full);
    lb.load(reinterpret_cast<char*>(Bs + slot * Cfg::kBTile), kt, BK, g.k, full);
  };

  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < ktiles) load_stage(st, st);
    cp_commit();
  }
  const int fr = lane >> 2, fk = lane & 3;
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    {  // refill the slot consumed STAGES-1 tiles ago (every warp is past it after the barrier)
      const int nk = kt + STAGES - 1;
      if (nk < ktiles) load_stage(nk, nk % STAGES);
      cp_commit();
    }
    const double* as = As + (kt % STAGES) * Cfg::kATile;
    const double* bs = Bs + (kt % STAGES) * Cfg::kBTile;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[MI], bf[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int r = wm * WM + i * 8 + fr;
        af[i] = AK ? as[r * SA + kk + fk] : as[(kk + fk) * SA + r];
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int c = wn * WN + j * 8 + fr;
        bf[j] = BKC ? bs[c * SB + kk + fk] : bs[(kk + fk) * SB + c];
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  if (g.ksplit > 1) {  // raw partial tile -> work[split][zz] (m x n, row-major)
    cp_wait<0>();
    const int64_t zcount = static_cast<int64_t>(gridDim.z) / g.ksplit;
    double* W = g.work + (static_cast<int64_t>(split) * zcount + zz) * g.m * g.n;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int64_t r = m0 + wm * WM + i * 8 + fr;
      if (r >= g.m) continue;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int64_t c = n0 + wn * WN + j * 8 + fk * 2;
        if (c + 1 < g.n && ((g.n & 1) == 0)) {
          *reinterpret_cast<double2*>(W + r * g.n + c) = make_double2(acc[i][j][0], acc[i][j][1]);
        } else {
          if (c < g.n) W[r * g.n + c] = acc[i][j][0];
          if (c + 1 < g.n) W[r * g.n + c + 1] = acc[i][j][1];
        }
      }
    }
    return;
  }
  cp_wait<0>();
  const double alpha = g.alpha.x, beta = g.beta.x;
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int64_t r = m0 + wm * WM + i * 8 + fr;
    if (r >= g.m) continue;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t c = n0 + wn * WN + j * 8 + fk * 2 + e;
        if (c < g.n) {
          double* cp = C + r * g.ldc + c;
          double v = alpha * acc[i][j][e];
          if (beta != 0.0) v = fma(beta, *cp, v);
          *cp = v;
        }
      }
    }
  }
}

// --------------------------------------------------------------------------------- complex
template <bool AK, bool BKC, int BM, int BN, int BK, int STAGES>
struct ZCfg {
  static constexpr int kWarpsM = BM / 32, kWarpsN = BN / 32;
  static constexpr int kThreads = kWarpsM * kWarpsN * 32;
  static constexpr int SA = AK ? BK + 4 : BM + 2;  // shared row stride (complex elements)
  static constexpr int SB = BKC ? BK + 4 : BN + 2;
  static constexpr int kATile = (AK ? BM : BK) * SA;
  static constexpr int kBTile = (BKC ? BN : BK) * SB;
  static constexpr size_t kSmem = static_cast<size_t>(STAGES) * (kATile + kBTile) * sizeof(double2);
  static_assert((AK ? SA % 8 == 4 : SA % 8 == 2) && (BKC ? SB % 8 == 4 : SB % 8 == 2), "conflict-free strides");
};

template <bool AK, bool BKC, int BM, int BN, int BK, int STAGES>
__global__ void __launch_bounds__(ZCfg<AK, BKC, BM, BN, BK, STAGES>::kThreads) zgemm_kernel(GArgs g) {
  using Cfg = ZCfg<AK, BKC, BM, BN, BK, STAGES>;
  constexpr int NT = Cfg::kThreads, SA = Cfg::SA, SB = Cfg::SB;
  if (g.stop != nullptr && *g.stop) return;
  extern __shared__ __align__(16) double2 zsm[];
  double2* As = zsm;
  double2* Bs = zsm + STAGES * Cfg::kATile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp % Cfg::kWarpsM, wn = warp / Cfg::kWarpsM;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM, n0 = static_cast<int64_t>(blockIdx.x) * BN;
  const char* A = static_cast<const char*>(g.a) + static_cast<int64_t>(blockIdx.z) * g.a_bs * 16;
  const char* B = static_cast<const char*>(g.b) + static_cast<int64_t>(blockIdx.z) * g.b_bs * 16;
  double2* C = static_cast<double2*>(g.c) + static_cast<int64_t>(blockIdx.z) * g.c_bs;
  const int ktiles = static_cast<int>((g.k + BK - 1) / BK);

  TileLoader<16, 16, AK ? BM : BK, AK ? BK : BM, SA, NT, AK> la;
  TileLoader<16, 16, BKC ? BN : BK, BKC ? BK : BN, SB, NT, BKC> lb;
  la.init(A, g.lda, m0, g.m, BK);
  lb.init(B, g.ldb, n0, g.n, BK);
  auto load_stage = [&](int kt, int slot) {
    const bool full = static_cast<int64_t>(kt + 1) * BK <= g.k;
    la.load(reinterpret_cast<char*>(As + slot * Cfg::kATile), kt, BK, g.k, full);
    lb.load(reinterpret_cast<char*>(Bs + slot * Cfg::kBTile), kt, BK, g.k, full);
  };

  double re[4][4][2], im[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) re[i][j][0] = re[i][j][1] = im[i][j][0] = im[i][j][1] = 0.0;

#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < ktiles) load_stage(st, st);
    cp_commit();
  }
  const int fr = lane >> 2, fk = lane & 3;
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < ktiles) load_stage(nk, nk % STAGES);
      cp_commit();
    }
    const double2* as = As + (kt % STAGES) * Cfg::kATile;
    const double2* bs = Bs + (kt % STAGES) * Cfg::kBTile;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double2 af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = wm * 32 + i * 8 + fr;
        af[i] = AK ? as[r * SA + kk + fk] : as[(kk + fk) * SA + r];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = wn * 32 + j * 8 + fr;
        bf[j] = BKC ? bs[c * SB + kk + fk] : bs[(kk + fk) * SB + c];
      }
      // (ar + i ai)(br + i bi): re += ar br - ai bi, im += ar bi + ai br
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double nai = -af[i].y;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dmma(re[i][j][0], re[i][j][1], af[i].x, bf[j].x);
          dmma(im[i][j][0], im[i][j][1], af[i].x, bf[j].y);
          dmma(re[i][j][0], re[i][j][1], nai, bf[j].y);
          dmma(im[i][j][0], im[i][j][1], af[i].y, bf[j].x);
        }
      }
    }
  }
  cp_wait<0>();
  const double2 alpha = g.alpha, beta = g.beta;
  const bool has_beta = beta.x != 0.0 || beta.y != 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = m0 + wm * 32 + i * 8 + fr;
    if (r >= g.m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t c = n0 + wn * 32 + j * 8 + fk * 2 + e;
        if (c < g.n) {
          double2* cp = C + r * g.ldc + c;
          double2 v = cmul(alpha, make_double2(re[i][j][e], im[i][j][e]));
          if (has_beta) cfma(v, beta, *cp);
          *cp = v;
        }
      }
    }
  }
}

// ------------------------------------------------------------------------------------ host
// Operand views in the kernels' terms: lda is the stride of the non-unit dimension.
struct Op {
  const void* p;
  int64_t ld, bs;
  bool kcontig;
};

// A (m x k, strides rs / cs) and B (k x n): unit stride required in one dimension each
bool view_a(const void* a, int64_t rs, int64_t cs, int64_t bs, Op* o) {
  if (cs == 1) { *o = {a, rs, bs, true}; return true; }
  if (rs == 1) { *o = {a, cs, bs, false}; return true; }
  return false;
}
bool view_b(const void* b, int64_t rs, int64_t cs, int64_t bs, Op* o) {
  if (rs == 1) { *o = {b, cs, bs, true}; return true; }
  if (cs == 1) { *o = {b, rs, bs, false}; return true; }
  return false;
}

template <typename K>
int launch_tile(K kern, size_t smem, int threads, int bm, int bn, const GArgs& g, int64_t batch, cudaStream_t s) {
  TOEP_CUDA(ensure_smem(kern, smem));
  const int64_t gy = (g.m + bm - 1) / bm, gx = (g.n + bn - 1) / bn;
  TOEP_REQUIRE(gy <= 65535 && batch <= 65535 && gx <= 0x7fffffff, TOEP_ERR_ARG, "dmma gemm grid too large");
  kern<<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy), static_cast<unsigned>(batch)), threads, smem, s>>>(g);
  TOEP_LAUNCHED();
  return TOEP_OK;
}

__global__ void dsplit_reduce(GArgs g, int64_t zcount) {
  const int64_t mn = g.m * g.n, total = zcount * mn;
  const double alpha = g.alpha.x, beta = g.beta.x;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t z = e / mn, rc = e - z * mn;
    double sum = 0.0;
    for (int sp = 0; sp < g.ksplit; ++sp) sum += __ldcs(g.work + (sp * zcount + z) * mn + rc);  // fixed order
    const int64_t r = rc / g.n, c = rc - r * g.n;
    const int plane = static_cast<int>(z % g.planes);
    double* cp = static_cast<double*>(g.pc[plane]) + (z / g.planes) * g.c_bs + r * g.ldc + c;
    double v = alpha * sum;
    if (beta != 0.0) v = fma(beta, *cp, v);
    *cp = v;
  }
}

int dev_sms() {
  static int n[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  dev &= 63;
  if (n[dev] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

// Split-K factor that evens out the per-SM load: `tiles` output tiles on `sms` SMs holding `slots`
// co-resident CTAs, `ktiles` k-tiles per tile.  CTAs are handed out as others finish, so an SM
// ends up with ceil(units / sms) units and the efficiency is units / (sms * ceil(units / sms)); a
// split must gain > 3 % over that (its partial tiles cost an extra write + reduction pass) and keep
// >= 32 k-tiles per split.  Grids of several full waves are never split.
int choose_ksplit(int64_t tiles, int64_t sms, int64_t slots, int ktiles) {
  if (tiles >= 3 * slots) return 1;
  auto eff = [&](int64_t units) {
    return static_cast<double>(units) / static_cast<double>(sms * ((units + sms - 1) / sms));
  };
  int best = 1;
  double best_eff = eff(tiles);
  for (int sp = 2; sp <= 8; ++sp) {
    if (ktiles / sp < 32) break;
    const double e = eff(tiles * sp) - 0.03;
    if (e > best_eff) {
      best_eff = e;
      best = sp;
    }
  }
  return best;
}

// real: CTA tile BM x BN x BK, warp tile WM x WN, STAGES-deep ring (tools/dmma_tune.cu sweep);
// split-K when the output tiles leave the last wave of co-resident CTAs mostly empty
template <bool AK, bool BKC, bool VEC, int BM = 64, int BN = 64, int BK = 16, int WM = 32, int WN = 32, int ST = 3>
int run_d(GArgs g, int64_t batch, cudaStream_t s, int force_split = 0) {
  using Cfg = DCfg<AK, BKC, BM, BN, BK, WM, WN, ST, VEC>;
  auto kern = dgemm_kernel<AK, BKC, BM, BN, BK, WM, WN, ST, VEC>;
  TOEP_CUDA(ensure_smem(kern, Cfg::kSmem));
  static int per_sm = 0;
  if (per_sm == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::kThreads, Cfg::kSmem) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    cudaGetLastError();
  }
  const int64_t gy = (g.m + BM - 1) / BM, gx = (g.n + BN - 1) / BN;
  const int64_t zcount = batch * g.planes;
  const int ktiles = static_cast<int>((g.k + BK - 1) / BK);
  // no split for stop-flag launches (GMRES speculative steps): the reduction would not see the flag
  int ks = g.stop != nullptr ? 1
           : force_split > 0 ? force_split
                             : choose_ksplit(gx * gy * zcount, dev_sms(), static_cast<int64_t>(per_sm) * dev_sms(),
                                             ktiles);
  ks = std::max(1, std::min(ks, std::max(ktiles, 1)));
  g.ktiles_per_split = (ktiles + ks - 1) / ks;
  g.ksplit = ks > 1 ? (ktiles + g.ktiles_per_split - 1) / g.ktiles_per_split : 1;
  if (g.ksplit <= 1) {
    g.ksplit = 1;
    g.ktiles_per_split = std::max(ktiles, 1);
    g.work = nullptr;
    return launch_tile(kern, Cfg::kSmem, Cfg::kThreads, BM, BN, g, zcount, s);
  }
  const size_t wbytes = static_cast<size_t>(g.ksplit) * zcount * g.m * g.n * sizeof(double);
  keep_pool();  // the workspace returns to the pool, not the driver, between calls
  if (cudaMallocAsync(reinterpret_cast<void**>(&g.work), wbytes, s) != cudaSuccess) {
    cudaGetLastError();
    set_error("out of device memory for the split-K workspace (%zu bytes)", wbytes);
    return TOEP_ERR_OOM;
  }
  int rc = launch_tile(kern, Cfg::kSmem, Cfg::kThreads, BM, BN, g, zcount * g.ksplit, s);
  if (rc == TOEP_OK) {
    const int64_t total = zcount * g.m * g.n;
    const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, static_cast<int64_t>(dev_sms()) * 8));
    dsplit_reduce<<<grid, 256, 0, s>>>(g, zcount);
    if (cudaGetLastError() != cudaSuccess) {
      set_error("split-K reduction launch failed");
      rc = TOEP_ERR_CUDA;
    }
  }
  cudaFreeAsync(g.work, s);
  return rc;
}

constexpr int kBM = 64, kBN = 64;

template <bool AK, bool BKC>
int run_z(const GArgs& g, int64_t batch, cudaStream_t s) {
  using Cfg = ZCfg<AK, BKC, kBM, kBN, 8, 3>;
  return launch_tile(zgemm_kernel<AK, BKC, kBM, kBN, 8, 3>, Cfg::kSmem, Cfg::kThreads, kBM, kBN, g, batch, s);
}

// Normalise to a row-major C: a column-major C is computed as C^T = B^T A^T.
bool normalise(int64_t& m, int64_t& n, const void*& a, int64_t& a_rs, int64_t& a_cs, int64_t& a_bs, const void*& b,
               int64_t& b_rs, int64_t& b_cs, int64_t& b_bs, int64_t& c_rs, int64_t& c_cs) {
  if (c_cs == 1 || n == 1) return true;
  if (c_rs != 1) return false;
  std::swap(m, n);
  std::swap(a, b);
  std::swap(a_bs, b_bs);
  const int64_t ars = a_rs, acs = a_cs;
  a_rs = b_cs; a_cs = b_rs;  // A' = B^T
  b_rs = acs; b_cs = ars;    // B' = A^T
  std::swap(c_rs, c_cs);
  return true;
}

}  // namespace

// Real C_p = alpha A_p B_p + beta C_p for `planes` (<= 3) operand triples of one shape in one
// launch, on the FP64 tensor cores; returns -1 if a stride pattern is not covered.
int dgemm_dmma_planes(int64_t m, int64_t n, int64_t k, double alpha, const double* const* a, int64_t a_rs,
                      int64_t a_cs, int64_t a_bs, const double* const* b, int64_t b_rs, int64_t b_cs, int64_t b_bs,
                      double beta, double* const* c, int64_t c_rs, int64_t c_cs, int64_t c_bs, int64_t batch,
                      int planes, cudaStream_t s, const int* stop) {
  if (m == 0 || n == 0 || batch == 0 || planes == 0) return TOEP_OK;
  if (planes < 1 || planes > 3) return -1;
  const void* av = a[0];
  const void* bv = b[0];
  const bool swapped = !(c_cs == 1 || n == 1);
  if (!normalise(m, n, av, a_rs, a_cs, a_bs, bv, b_rs, b_cs, b_bs, c_rs, c_cs)) return -1;
  Op A, B;
  if (!view_a(av, a_rs, a_cs, a_bs, &A) || !view_b(bv, b_rs, b_cs, b_bs, &B)) return -1;
  GArgs g{m, n, k, make_double2(alpha, 0), make_double2(beta, 0), A.p, A.ld, A.bs, B.p, B.ld, B.bs, c[0], c_rs, c_bs,
          stop, planes, {}, {}, {}};
  bool vec = true;
  auto al = [](const void* p, int64_t ld, int64_t bs) {
    return (reinterpret_cast<uintptr_t>(p) & 15) == 0 && (ld & 1) == 0 && (bs & 1) == 0;
  };
  for (int q = 0; q < planes; ++q) {
    g.pa[q] = swapped ? b[q] : a[q];
    g.pb[q] = swapped ? a[q] : b[q];
    g.pc[q] = c[q];
    // 16-byte copies when every copied row starts 16-byte aligned (odd extents end in a zero-filled half copy)
    vec = vec && al(g.pa[q], A.ld, A.bs) && al(g.pb[q], B.ld, B.bs);
  }
#define TOEP_DRUN(ak, bk)                                          \
  if (A.kcontig == ak && B.kcontig == bk)                          \
    return vec ? run_d<ak, bk, true>(g, batch, s) : run_d<ak, bk, false>(g, batch, s);
  TOEP_DRUN(true, false)
  TOEP_DRUN(false, false)
  TOEP_DRUN(true, true)
  TOEP_DRUN(false, true)
#undef TOEP_DRUN
  return -1;
}

int dgemm_dmma(int64_t m, int64_t n, int64_t k, double alpha, const double* a, int64_t a_rs, int64_t a_cs,
               int64_t a_bs, const double* b, int64_t b_rs, int64_t b_cs, int64_t b_bs, double beta, double* c,
               int64_t c_rs, int64_t c_cs, int64_t c_bs, int64_t batch, cudaStream_t s, const int* stop) {
  return dgemm_dmma_planes(m, n, k, alpha, &a, a_rs, a_cs, a_bs, &b, b_rs, b_cs, b_bs, beta, &c, c_rs, c_cs, c_bs,
                           batch, 1, s, stop);
}

// Complex C = alpha A B + beta C on the FP64 tensor cores; returns -1 if a stride pattern is not covered.
int zgemm_dmma(int64_t m, int64_t n, int64_t k, double2 alpha, const void* a, int64_t a_rs, int64_t a_cs, int64_t a_bs,
               const void* b, int64_t b_rs, int64_t b_cs, int64_t b_bs, double2 beta, void* c, int64_t c_rs,
               int64_t c_cs, int64_t c_bs, int64_t batch, cudaStream_t s, const int* stop) {
  if (m == 0 || n == 0 || batch == 0) return TOEP_OK;
  if (!normalise(m, n, a, a_rs, a_cs, a_bs, b, b_rs, b_cs, b_bs, c_rs, c_cs)) return -1;
  Op A, B;
  if (!view_a(a, a_rs, a_cs, a_bs, &A) || !view_b(b, b_rs, b_cs, b_bs, &B)) return -1;
  if ((reinterpret_cast<uintptr_t>(A.p) & 15) || (reinterpret_cast<uintptr_t>(B.p) & 15)) return -1;
  const int64_t ldc = c_rs;
  GArgs g{m, n, k, alpha, beta, A.p, A.ld, A.bs, B.p, B.ld, B.bs, c, ldc, c_bs, stop, 1, {}, {}, {}};
  if (A.kcontig && !B.kcontig) return run_z<true, false>(g, batch, s);
  if (!A.kcontig && !B.kcontig) return run_z<false, false>(g, batch, s);
  if (A.kcontig && B.kcontig) return run_z<true, true>(g, batch, s);
  return run_z<false, true>(g, batch, s);
}

}  // namespace toep

extern "C" int toep_dgemm(int64_t m, int64_t n, int64_t k, double alpha, const double* a, int64_t a_rs, int64_t a_cs,
                          int64_t a_bs, const double* b, int64_t b_rs, int64_t b_cs, int64_t b_bs, double beta,
                          double* c, int64_t c_rs, int64_t c_cs, int64_t c_bs, int64_t batch, void* stream) {
  TOEP_NVTX("toep_dgemm");
  TOEP_REQUIRE(m >= 0 && n >= 0 && k >= 0 && batch >= 0, TOEP_ERR_SHAPE, "negative gemm size");
  int64_t done = 0;
  while (done < batch) {
    const int64_t nb = std::min<int64_t>(batch - done, 65535);
    const int rc = toep::dgemm_dmma(m, n, k, alpha, a + done * a_bs, a_rs, a_cs, a_bs, b + done * b_bs, b_rs, b_cs,
                                    b_bs, beta, c + done * c_bs, c_rs, c_cs, c_bs, nb,
                                    static_cast<cudaStream_t>(stream), nullptr);
    if (rc < 0) {
      toep::set_error("toep_dgemm: each operand needs a unit stride in one dimension");
      return TOEP_ERR_ARG;
    }
    if (rc != TOEP_OK) return rc;
    done += nb;
  }
  return TOEP_OK;
}
