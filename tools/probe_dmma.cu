// DMMA shape probe: register-resident throughput of the f64 mma.sync shapes on sm_100a, and a
// numerical check of the m16n8k{4,8,16} fragment layouts against a host product.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/probe_dmma.cu -o tools/probe_dmma
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

__device__ __forceinline__ void mma884(double* c, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma1684(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
}
__device__ __forceinline__ void mma1688(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void mma16816(double* c, const double* a, const double* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
        "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int SHAPE>
__global__ void thr(double* out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) b[i] = 1e-3 * (threadIdx.x - i);
  double c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if constexpr (SHAPE == 0) mma884(c[t], a[t], b[t & 3]);
      if constexpr (SHAPE == 1) mma1684(c[t], a + (t & 3) * 2, b + (t & 3));
      if constexpr (SHAPE == 2) mma1688(c[t], a + (t & 1) * 4, b + (t & 1) * 2);
      if constexpr (SHAPE == 3) mma16816(c[t], a, b);
    }
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// layout check: one warp computes C(16x8) = A(16xK) B(Kx8) with the assumed fragment maps
template <int K>
__global__ void check(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double c[4] = {0, 0, 0, 0};
  double a[8], b[4];
  for (int q = 0; q < K / 4; ++q) {  // a[2q] = (g, t + 4q), a[2q+1] = (g + 8, t + 4q); b[q] = (t + 4q, g)
    a[2 * q] = A[g * K + t + 4 * q];
    a[2 * q + 1] = A[(g + 8) * K + t + 4 * q];
    b[q] = B[(t + 4 * q) * 8 + g];
  }
  if constexpr (K == 4) mma1684(c, a, b);
  if constexpr (K == 8) mma1688(c, a, b);
  if constexpr (K == 16) mma16816(c, a, b);
  // c0, c1 = (g, 2t + {0,1}); c2, c3 = (g + 8, 2t + {0,1})
  C[g * 8 + 2 * t] = c[0];
  C[g * 8 + 2 * t + 1] = c[1];
  C[(g + 8) * 8 + 2 * t] = c[2];
  C[(g + 8) * 8 + 2 * t + 1] = c[3];
}

template <int K>
void run_check() {
  std::vector<double> A(16 * K), B(K * 8), C(128), R(128, 0.0);
  for (auto& x : A) x = rand() / double(RAND_MAX) - 0.5;
  for (auto& x : B) x = rand() / double(RAND_MAX) - 0.5;
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 8; ++j)
      for (int k = 0; k < K; ++k) R[i * 8 + j] += A[i * K + k] * B[k * 8 + j];
  double *dA, *dB, *dC;
  cudaMalloc(&dA, A.size() * 8);
  cudaMalloc(&dB, B.size() * 8);
  cudaMalloc(&dC, 128 * 8);
  cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
  check<K><<<1, 32>>>(dA, dB, dC);
  cudaMemcpy(C.data(), dC, 128 * 8, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 128; ++i) err = fmax(err, fabs(C[i] - R[i]));
  printf("m16n8k%d layout check: max abs err %.3e (%s)\n", K, err, err < 1e-12 ? "OK" : "MISMATCH");
}

int main() {
  run_check<4>();
  run_check<8>();
  run_check<16>();
  double* out;
  cudaMalloc(&out, 148 * 8 * 256 * 8);
  const double macs_per_inst[4] = {8 * 8 * 4, 16 * 8 * 4, 16 * 8 * 8, 16 * 8 * 16};
  const char* names[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int sh = 0; sh < 4; ++sh) {
      const int iters = sh == 3 ? 512 : (sh == 2 ? 1024 : (sh == 1 ? 2048 : 4096));
      auto launch = [&]() {
        if (sh == 0) thr<0><<<148 * 2, warps * 32>>>(out, iters);
        if (sh == 1) thr<1><<<148 * 2, warps * 32>>>(out, iters);
        if (sh == 2) thr<2><<<148 * 2, warps * 32>>>(out, iters);
        if (sh == 3) thr<3><<<148 * 2, warps * 32>>>(out, iters);
      };
      launch();
      cudaDeviceSynchronize();
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flop = 2.0 * macs_per_inst[sh] * 8 * iters * (148.0 * 2 * warps);
      printf("%-9s %2d warps/CTA x 2 CTA/SM: %.3f ms  %.2f TFLOP/s\n", names[sh], warps, ms, flop / (ms * 1e-3) / 1e12);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
