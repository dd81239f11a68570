// Timing of the fused 2-D transform kernels alone for several batch widths (not part of the library).
#include "../paper_2506_20350_b200/csrc/kernels.cuh"
#include <cstdio>
#include <vector>
int main() {
  const int n2 = 30, n1 = 30, l = 60;
  for (int inner : {16, 64, 128, 148, 256, 296}) {
    double2 *in, *out;
    cudaMalloc(&in, sizeof(double2) * (size_t)n2 * n1 * inner);
    cudaMalloc(&out, sizeof(double2) * (size_t)l * l * inner);
    cudaMemset(in, 0, sizeof(double2) * (size_t)n2 * n1 * inner);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int inv = 0; inv < 2; ++inv) {
      const void* src = inv ? (const void*)out : (const void*)in;
      void* dst = inv ? (void*)in : (void*)out;
      for (int w = 0; w < 5; ++w) toep::fft2d(inv, src, dst, n2, n1, l, l, inner, inv ? 1 : -1, 0, 0, 0, nullptr, nullptr, 0);
      cudaEventRecord(e0);
      const int reps = 200;
      for (int r = 0; r < reps; ++r) toep::fft2d(inv, src, dst, n2, n1, l, l, inner, inv ? 1 : -1, 0, 0, 0, nullptr, nullptr, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("inner %4d %s: %.2f us  (%s)\n", inner, inv ? "inv" : "fwd", ms * 1e3 / reps, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(in); cudaFree(out);
  }
}
