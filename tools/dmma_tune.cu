// Tile-shape sweep of the hand-written DMMA real GEMM (csrc/dmma.cu) on the solvers' shapes.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr \
//        -I paper_2506_20350_b200/csrc tools/dmma_tune.cu -o tools/dmma_tune && tools/dmma_tune
#include <cstdarg>
#include <cstdio>
#include <map>
#include <mutex>
#include <vector>

#include "../paper_2506_20350_b200/csrc/dmma.cu"

namespace toep {
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vfprintf(stderr, fmt, ap);
  va_end(ap);
  fprintf(stderr, "\n");
}
void keep_pool() {}
cudaError_t ensure_smem_attr(const void* func, size_t bytes) {
  return cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
}
}  // namespace toep

using namespace toep;

struct Shape {
  const char* name;
  int64_t m, n, k, batch;
  int planes;
  bool a_colmajor;
};

template <bool AK, int BM, int BN, int BK, int WM, int WN, int ST>
float time_cfg(const Shape& sh, double* A[3], double* B[3], double* Cc[3], int split = 0) {
  GArgs g{};
  g.m = sh.m; g.n = sh.n; g.k = sh.k;
  g.alpha = make_double2(1, 0); g.beta = make_double2(0, 0);
  g.lda = AK ? sh.k : sh.m;
  g.a_bs = sh.m * sh.k;
  g.ldb = sh.n; g.b_bs = sh.k * sh.n;
  g.ldc = sh.n; g.c_bs = sh.m * sh.n;
  g.planes = sh.planes;
  for (int q = 0; q < 3; ++q) { g.pa[q] = A[q]; g.pb[q] = B[q]; g.pc[q] = Cc[q]; }
  auto go = [&]() { return run_d<AK, false, true, BM, BN, BK, WM, WN, ST>(g, sh.batch, 0, split); };
  if (go() != TOEP_OK) return -1.f;
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 5;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) go();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  if (cudaGetLastError() != cudaSuccess) return -2.f;
  return ms / reps;
}

int main() {
  {  // as the library (op.cu keep_pool): freed stream-ordered memory stays in the pool
    cudaMemPool_t pool;
    cudaDeviceGetDefaultMemPool(&pool, 0);
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  std::vector<Shape> shapes = {
      {"blocksum_1024x1024x15360_p3", 1024, 1024, 15360, 1, 3, false},
      {"blocksum_1024x1024x4096_b2_p3", 1024, 1024, 4096, 2, 3, false},
      {"blocksum_1024x1024x1024_b2_p3", 1024, 1024, 1024, 2, 3, false},
      {"cross_1024x1024x1024_b15_p3", 1024, 1024, 1024, 15, 3, false},
      {"dgemm_4096_p1", 4096, 4096, 4096, 1, 1, false},
      {"perbin_256x900x256_b120_p3_acm", 256, 900, 256, 120, 3, true},
  };
  size_t maxe = 0;
  for (auto& s : shapes) maxe = std::max<size_t>(maxe, static_cast<size_t>(s.batch) * std::max({s.m * s.k, s.k * s.n, s.m * s.n}));
  double *A[3], *B[3], *C[3];
  for (int q = 0; q < 3; ++q) {
    cudaMalloc(&A[q], maxe * 8);
    cudaMalloc(&B[q], maxe * 8);
    cudaMalloc(&C[q], maxe * 8);
    cudaMemset(A[q], 0, maxe * 8);
    cudaMemset(B[q], 0, maxe * 8);
  }
  for (auto& sh : shapes) {
    const double fl = 2.0 * sh.m * sh.n * sh.k * sh.batch * sh.planes;
    printf("%s\n", sh.name);
#define CFG(BM, BN, BK, WM, WN, ST)                                                                     \
  {                                                                                                      \
    const float ms = sh.a_colmajor ? time_cfg<false, BM, BN, BK, WM, WN, ST>(sh, A, B, C)               \
                                   : time_cfg<true, BM, BN, BK, WM, WN, ST>(sh, A, B, C);               \
    printf("  %3d x %3d x %2d  warp %2d x %2d  st %d : %8.3f ms  %6.2f TFLOP/s\n", BM, BN, BK, WM, WN, ST, ms, \
           ms > 0 ? fl / (ms * 1e-3) / 1e12 : 0.0);                                                      \
    fflush(stdout);                                                                                      \
  }
    CFG(64, 64, 16, 32, 32, 3)
    CFG(64, 64, 16, 32, 32, 4)
    CFG(64, 64, 32, 32, 32, 3)
    CFG(128, 64, 16, 32, 32, 3)
    CFG(64, 128, 16, 32, 64, 3)
    CFG(64, 64, 8, 32, 32, 6)
    for (int sp = 1; sp <= 4; ++sp) {
      const float ms = sh.a_colmajor ? time_cfg<false, 64, 64, 16, 32, 32, 3>(sh, A, B, C, sp)
                                     : time_cfg<true, 64, 64, 16, 32, 32, 3>(sh, A, B, C, sp);
      printf("  64x64x16 st3 forced split %d : %8.3f ms  %6.2f TFLOP/s\n", sp, ms, fl / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
