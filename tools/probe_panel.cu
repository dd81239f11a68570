// Phase timing of the cluster LU panel (build: make -C tools probe; not part of the library).
#define TOEP_PANEL_PROBE 1
#include "../paper_2506_20350_b200/csrc/rybicki.cu"
#include <cstdio>
#include <random>
constexpr int kProbeRPT = (1024 / toep::kCL + toep::kRowsPass - 1) / toep::kRowsPass;
int main() {
  const int n = 1024;
  std::vector<double2> h(static_cast<size_t>(n) * n);
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  for (auto& v : h) v = make_double2(nd(rng), nd(rng));
  double2* A; int *ipiv, *info, *moves;
  cudaMalloc(&A, h.size() * 16); cudaMalloc(&ipiv, n * 4); cudaMalloc(&info, 4); cudaMalloc(&moves, 4 * 200);
  cudaMemset(info, 0, 4);
  cudaFuncSetAttribute(toep::lu_panel_cluster<kProbeRPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(A, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
    long long z[toep::kCL][8] = {};
    cudaMemcpyToSymbol(toep::g_probe, z, sizeof(z));
    cudaEventRecord(e0);
    toep::lu_panel_cluster<kProbeRPT><<<dim3(toep::kCL, 1), toep::kPanelThr2, toep::panel_smem(n, 0)>>>(A, 0, n, 0, ipiv, info, moves);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpyFromSymbol(z, toep::g_probe, sizeof(z));
    printf("rep %d: %.1f us  err=%s\n", rep, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
    for (int r = 0; r < 2; ++r) {
      printf("  rank %d cycles/phase:", r);
      for (int k = 0; k < 8; ++k) printf(" %lld", z[r][k] / 32);
      printf("\n");
    }
  }
}
