// DFT pass configuration sweep for the cfg3 multi-RHS passes (L = 60, inner = n0 * W = 230 400):
// CTA width (threads) x batch-column tile x resident CTAs.  Not part of the library.
//   nvcc ... -I paper_2506_20350_b200/csrc tools/probe_pass.cu <library objects except fft.o>
#include "../paper_2506_20350_b200/csrc/fft.cu"
#include <cstdio>

namespace toep {
namespace {
template <typename TI, typename TC, typename TO, int NT, int MINB, int TIL, int... Rs>
__global__ void __launch_bounds__(NT, MINB) probe_plan_kernel(PassArgs a, double two_over_L) {
  using Z = C<TC>;
  constexpr int L = PlanLen<Rs...>::value;
  __shared__ __align__(16) Z tw[L];
  __shared__ __align__(16) Z buf[2][L * TIL];
  pdl_trigger();
  for (int t = threadIdx.x; t < L; t += NT) {
    TC s, c;
    sincospi_t<TC>(static_cast<TC>(t * two_over_L), &s, &c);
    tw[t] = mk<TC>(c, a.sign * s);
  }
  pdl_wait();
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * TIL;
  const int o = blockIdx.y;
  const int ncol = static_cast<int>(std::min<int64_t>(TIL, a.inner - i0));
  const C<TI>* in = static_cast<const C<TI>*>(a.in) + o * a.in_so + i0;
  C<TO>* out = static_cast<C<TO>*>(a.out) + o * a.out_so + i0;
  __syncthreads();
  plan_stage<TI, TC, TO, NT, TIL, L, 1, 0, Rs...>(a, in, out, buf[0], buf[1], tw, ncol, pass_scale<TC>(a));
}
}  // namespace
}  // namespace toep

using namespace toep;

template <int NT, int MINB, int TIL>
void run(const char* name, PassArgs a, double bytes) {
  auto k = probe_plan_kernel<double, double, double, NT, MINB, TIL, 4, 3, 5>;
  dim3 grid(static_cast<unsigned>((a.inner + TIL - 1) / TIL), static_cast<unsigned>(a.outer));
  for (int w = 0; w < 2; ++w) k<<<grid, NT>>>(a, 2.0 / 60);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<<<grid, NT>>>(a, 2.0 / 60);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 5;
  printf("%-10s NT %3d MINB %2d TIL %2d: %.3f ms  %.2f TB/s  %s\n", name, NT, MINB, TIL, ms, bytes / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int n2 = 30, n1 = 30, L = 60;
  const int64_t inner = 256LL * 900;
  double2 *u, *x1;
  cudaMalloc(&u, sizeof(double2) * n2 * n1 * inner);
  cudaMalloc(&x1, sizeof(double2) * n2 * L * inner);
  cudaMemset(u, 0, sizeof(double2) * n2 * n1 * inner);
  PassArgs a;  // the cfg3 level-1 forward pass: u [n2][n1][inner] -> x1 [n2][L][inner]
  a.in = u; a.out = x1; a.L = L; a.n_lo = n1; a.n_hi = 0; a.n_out = L; a.inner = inner; a.outer = n2;
  a.in_sa = inner; a.in_so = n1 * inner; a.out_sa = inner; a.out_so = L * inner; a.sign = -1; a.scale = 1.0;
  const double bytes = 16.0 * inner * n2 * (n1 + L);
  run<128, 8, 16>("level1", a, bytes);
  run<128, 8, 8>("level1", a, bytes);
  run<128, 4, 24>("level1", a, bytes);
  run<256, 4, 16>("level1", a, bytes);
  run<256, 4, 24>("level1", a, bytes);
  run<256, 2, 24>("level1", a, bytes);
  run<64, 16, 8>("level1", a, bytes);
  run<64, 16, 16>("level1", a, bytes);
  // inverse level 1: x1 [n2][L][inner] -> v [n2][n1][inner], crop
  PassArgs d;
  d.in = x1; d.out = u; d.L = L; d.n_lo = L; d.n_hi = 0; d.n_out = n1; d.inner = inner; d.outer = n2;
  d.in_sa = inner; d.in_so = L * inner; d.out_sa = inner; d.out_so = n1 * inner; d.sign = 1; d.scale = 1.0 / 3600;
  run<128, 8, 16>("inv-level1", d, bytes);
  run<128, 4, 24>("inv-level1", d, bytes);
  run<256, 4, 16>("inv-level1", d, bytes);
  run<256, 4, 24>("inv-level1", d, bytes);
  run<64, 16, 16>("inv-level1", d, bytes);
  return 0;
}
