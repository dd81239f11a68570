// Probe: can runtime-API kernels run on streams of green contexts (SM partitions), with memory from
// cudaMalloc?  Prints the SM ids each partition's kernel ran on.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <set>

__global__ void __cluster_dims__(8, 1, 1) cluster_k(int* out) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) out[blockIdx.x] = smid;
}

__global__ void which_sm(int* out, int n) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) out[blockIdx.x] = smid;
  long long t0 = clock64();
  while (clock64() - t0 < 2000000) {}
}

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); printf("%s -> %s\n", #x, s_); return 1; } } while (0)
#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("%s -> %s\n", #x, cudaGetErrorString(r_)); return 1; } } while (0)

int main() {
  RK(cudaSetDevice(0));
  RK(cudaFree(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUdevResource all;
  CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs %u\n", all.sm.smCount);
  unsigned n = 1;
  CUdevResource part[1], rest;
  CK(cuDevSmResourceSplitByCount(part, &n, &all, &rest, 0, 16));
  printf("groups %u: part %u SMs, rest %u SMs\n", n, part[0].sm.smCount, rest.sm.smCount);
  CUdevResourceDesc d1, d2;
  CK(cuDevResourceGenerateDesc(&d1, &part[0], 1));
  CK(cuDevResourceGenerateDesc(&d2, &rest, 1));
  CUgreenCtx g1, g2;
  CK(cuGreenCtxCreate(&g1, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CK(cuGreenCtxCreate(&g2, d2, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream s1, s2;
  CK(cuGreenCtxStreamCreate(&s1, g1, CU_STREAM_NON_BLOCKING, 0));
  CK(cuGreenCtxStreamCreate(&s2, g2, CU_STREAM_NON_BLOCKING, 0));
  int* buf;
  RK(cudaMalloc(&buf, 4096 * sizeof(int)));
  which_sm<<<296, 128, 0, (cudaStream_t)s1>>>(buf, 296);
  RK(cudaGetLastError());
  which_sm<<<296, 128, 0, (cudaStream_t)s2>>>(buf + 1024, 296);
  RK(cudaGetLastError());
  RK(cudaDeviceSynchronize());
  int h[2048];
  RK(cudaMemcpy(h, buf, sizeof(h), cudaMemcpyDeviceToHost));
  std::set<int> a(h, h + 296), b(h + 1024, h + 1024 + 296);
  printf("green 1 kernel ran on %zu distinct SMs, green 2 on %zu; overlap:", a.size(), b.size());
  int ov = 0;
  for (int x : a) ov += b.count(x);
  printf(" %d\n", ov);
  // clusters of 8 in the 16-SM partition, and an event recorded there waited on by the other
  cudaEvent_t ev;
  RK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  cluster_k<<<16, 128, 0, (cudaStream_t)s1>>>(buf + 3000);
  RK(cudaGetLastError());
  RK(cudaEventRecord(ev, (cudaStream_t)s1));
  RK(cudaStreamWaitEvent((cudaStream_t)s2, ev, 0));
  which_sm<<<8, 128, 0, (cudaStream_t)s2>>>(buf + 3500, 8);
  RK(cudaGetLastError());
  RK(cudaDeviceSynchronize());
  int hc[16];
  RK(cudaMemcpy(hc, buf + 3000, sizeof(hc), cudaMemcpyDeviceToHost));
  printf("cluster kernel SMs:");
  for (int i = 0; i < 16; ++i) printf(" %d", hc[i]);
  printf("\n");
  int maxc = 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16); cfg.blockDim = dim3(128); cfg.stream = (cudaStream_t)s1;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 8; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  printf("max active clusters in partition: %s\n", cudaOccupancyMaxActiveClusters(&maxc, (void*)cluster_k, &cfg) == cudaSuccess ? "ok" : "err");
  printf("  = %d\n", maxc);
  // default (primary-context) stream still sees everything
  which_sm<<<296, 128>>>(buf + 2048 - 1024, 296);
  RK(cudaDeviceSynchronize());
  printf("ok\n");
  return 0;
}
