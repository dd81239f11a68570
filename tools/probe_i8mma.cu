// Probe: one tcgen05.mma.kind::i8 tile (M=128, N=128, K=KT) from shared memory (no-swizzle
// K-major core-matrix layout), accumulator in TMEM, read back with tcgen05.ld.  Checks the
// descriptor encodings against a host reference, then times a many-CTA loop of MMAs.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I$CUTLASS tools/probe_i8mma.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cute/arch/mma_sm100_desc.hpp>

#ifndef NPROBE
#define NPROBE 128
#endif
constexpr int M = 128, N = NPROBE, KT = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// no-swizzle K-major operand: core matrices of 8 rows x 16 bytes; chunk c (16 K-bytes) of row group g
// at  g * sbo + c * lbo
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  cute::UMMA::SmemDescriptor d;
  d.desc_ = 0;
  d.start_address_ = static_cast<uint16_t>(saddr >> 4);
  d.leading_byte_offset_ = static_cast<uint16_t>(lbo >> 4);
  d.stride_byte_offset_ = static_cast<uint16_t>(sbo >> 4);
  d.version_ = 1;
  d.base_offset_ = 0;
  d.lbo_mode_ = 0;
  d.layout_type_ = 0;  // SWIZZLE_NONE
  return d.desc_;
}

__host__ __device__ constexpr uint32_t make_idesc() {
  // c_format S32 (2) bits 4-5, a/b signed (1) bits 7-9 / 10-12, K-major, n_dim = N>>3 bits 17-22,
  // m_dim = M>>4 bits 24-28
  return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) i8_tile(const int8_t* A, const int8_t* B, int32_t* C, int reps) {
  // smem: A [g=M/8][c=KT/16][8][16], B [g=N/8][c=KT/16][8][16]  (MODE 0: lbo = 128 (K), sbo = KT/16*128)
  //        MODE 1: [c][g][8][16] (lbo = M/8*128, sbo = 128)
  __shared__ __align__(1024) int8_t sa[M * KT];
  __shared__ __align__(1024) int8_t sb[N * KT];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int8_t* Ab = A + static_cast<size_t>(blockIdx.x % 4) * 0;  // same tile for every CTA
  for (int e = tid; e < M * KT / 16; e += 128) {  // 16-byte chunks
    const int row = e / (KT / 16), c = e % (KT / 16);
    const int g = row / 8, r = row % 8;
    const int off = MODE == 0 ? ((g * (KT / 16) + c) * 8 + r) * 16 : ((c * (M / 8) + g) * 8 + r) * 16;
    *reinterpret_cast<int4*>(sa + off) = *reinterpret_cast<const int4*>(Ab + row * KT + c * 16);
  }
  for (int e = tid; e < N * KT / 16; e += 128) {
    const int row = e / (KT / 16), c = e % (KT / 16);
    const int g = row / 8, r = row % 8;
    const int off = MODE == 0 ? ((g * (KT / 16) + c) * 8 + r) * 16 : ((c * (N / 8) + g) * 8 + r) * 16;
    *reinterpret_cast<int4*>(sb + off) = *reinterpret_cast<const int4*>(B + row * KT + c * 16);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t lboA = MODE == 0 ? 128 : (M / 8) * 128, sboA = MODE == 0 ? (KT / 16) * 128 : 128;
  const uint32_t lboB = MODE == 0 ? 128 : (N / 8) * 128, sboB = MODE == 0 ? (KT / 16) * 128 : 128;
  const uint32_t stepA = MODE == 0 ? 2 * 128 : 2 * lboA;  // start-address advance per K=32 MMA
  const uint32_t stepB = MODE == 0 ? 2 * 128 : 2 * lboB;
  constexpr uint32_t idesc = make_idesc();
  const uint64_t da0 = make_desc(smem_u32(sa), lboA, sboA);
  const uint64_t db0 = make_desc(smem_u32(sb), lboB, sboB);
  if (tid == 0) {
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
      for (int kk = 0; kk < KT / 32; ++kk) {
        const uint64_t da = da0 + ((kk * stepA) >> 4);
        const uint64_t db = db0 + ((kk * stepB) >> 4);
        const uint32_t acc = (rep > 0 || kk > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&mbar))
                 : "memory");
  }
  // wait for the MMAs (phase 0)
  asm volatile(
      "{\n\t.reg .pred done;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], 0;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(&mbar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + (tid & 31);
  for (int col = 0; col < N; col += 8) {
    uint32_t v[8];
    const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + col;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (blockIdx.x == 0)
      for (int j = 0; j < 8; ++j) C[row * N + col + j] = static_cast<int32_t>(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(N));
}

int main(int argc, char** argv) {
  std::vector<int8_t> a(M * KT), b(N * KT);
  srand(1);
  for (auto& x : a) x = static_cast<int8_t>(rand() % 255 - 127);
  for (auto& x : b) x = static_cast<int8_t>(rand() % 255 - 127);
  std::vector<int64_t> ref(M * N, 0);
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int64_t s = 0;
      for (int k = 0; k < KT; ++k) s += static_cast<int64_t>(a[i * KT + k]) * b[j * KT + k];
      ref[i * N + j] = s;
    }
  int8_t *da, *db;
  int32_t* dc;
  cudaMalloc(&da, a.size());
  cudaMalloc(&db, b.size());
  cudaMalloc(&dc, M * N * 4);
  cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dc, 0, M * N * 4);
    if (mode == 0) i8_tile<0><<<1, 128>>>(da, db, dc, 1);
    else i8_tile<1><<<1, 128>>>(da, db, dc, 1);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<int32_t> c(M * N);
    cudaMemcpy(c.data(), dc, M * N * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < M * N; ++i) bad += (c[i] != ref[i]);
    printf("mode %d: %s, mismatches %d / %d  (c[0]=%d ref %lld, c[1]=%d ref %lld, c[N]=%d ref %lld)\n", mode,
           cudaGetErrorString(e), bad, M * N, c[0], (long long)ref[0], c[1], (long long)ref[1], c[N],
           (long long)ref[N]);
    if (e != cudaSuccess) return 1;
  }
  // throughput: many CTAs, each looping MMAs on its resident tile
  const int reps = argc > 1 ? atoi(argv[1]) : 2000;
  for (int mode = 0; mode < 2; ++mode) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = 148;
    cudaEventRecord(e0);
    if (mode == 0) i8_tile<0><<<grid, 128>>>(da, db, dc, reps);
    else i8_tile<1><<<grid, 128>>>(da, db, dc, reps);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 2.0 * M * N * KT * reps * grid;
    printf("mode %d timing: %s  %.3f ms  %.1f TOPS\n", mode, cudaGetErrorString(e), ms, ops / (ms * 1e-3) / 1e12);
  }
  return 0;
}
