// Host-side helpers of the problem-file path (TBZ1, problems.py:219-322 of the reference).
#include <functional>

#include "common.cuh"
#include "op.h"

extern "C" int toep_fnv1a64(const void* data, uint64_t bytes, uint64_t* out) {
  TOEP_REQUIRE(out != nullptr && (data != nullptr || bytes == 0), TOEP_ERR_ARG, "bad fnv1a64 arguments");
  const unsigned char* p = static_cast<const unsigned char*>(data);
  uint64_t h = 0xCBF29CE484222325ull;  // offset basis
  for (uint64_t i = 0; i < bytes; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ull;  // FNV prime (wraps mod 2^64)
  }
  *out = h;
  return TOEP_OK;
}

// Page-locked host buffers for the host-in / host-out calls (toep_matvec_host).  cudaHostAlloc
// memory is read by the copy engines at the PCIe rate (1.84 MB H2D: 37 us = 50 GB/s on the B200
// boxes); torch's caching host allocator's blocks measured 17-19 GB/s in the same direction
// (tools/hostbuf_probe.py), so the Python layer stages host vectors in these.
extern "C" int toep_host_alloc(uint64_t bytes, void** out) {
  TOEP_REQUIRE(out != nullptr, TOEP_ERR_ARG, "null output pointer");
  *out = nullptr;
  if (bytes == 0) return TOEP_OK;
  const cudaError_t e = cudaHostAlloc(out, bytes, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *out = nullptr;
    toep::set_error("cudaHostAlloc of %llu bytes failed: %s", static_cast<unsigned long long>(bytes),
                    cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? TOEP_ERR_OOM : TOEP_ERR_CUDA;
  }
  return TOEP_OK;
}

extern "C" int toep_host_free(void* p) {
  if (p == nullptr) return TOEP_OK;
  TOEP_CUDA(cudaFreeHost(p));
  return TOEP_OK;
}

// ---- staged host -> device copies of pageable input (toep_matvec_host + TOEP_MV_STAGE_INPUT)
//
// A pageable buffer (a numpy array) cannot be read by the copy engines directly: the driver
// bounces it through its own pinned buffers (1.84 MB in 115-140 us on the B200 boxes against 45 us
// from page-locked memory, tools/hoststage_probe.cu).  Here the library's copy threads memcpy it
// into a page-locked staging buffer in parallel slices (5 threads: 1.84 MB in ~10 us, non-temporal
// stores), then one DMA.  The workers spin for up to 2 ms after a job (back-to-back calls find them
// awake; a condition-variable wake-up costs tens of microseconds), then sleep.
#include <immintrin.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace toep {
namespace {

class CopyPool {
 public:
  static constexpr int kWorkers = 4;
  // never destroyed: the workers live as long as the process (a destructor would have to join them
  // at exit, and a forked child holds thread handles that are not its own)
  static CopyPool& get() {
    static CopyPool* pool = new CopyPool();
    return *pool;
  }
  // chunk c of [0, n) is copied by participant c % (kWorkers + 1) (0 = the caller); on_ready(c) runs
  // on the caller, in chunk order, once chunks 0..c are staged.  Returns on_ready's first error.
  int run(int n, const std::function<void(int)>& job, const std::function<int(int)>& on_ready) {
    if (getpid() != pid_) {  // a forked child inherits no threads: copy on the caller alone
      int rc = TOEP_OK;
      for (int c = 0; c < n; ++c) {
        job(c);
        if (rc == TOEP_OK) rc = on_ready(c);
      }
      return rc;
    }
    std::lock_guard<std::mutex> run_lock(run_mu_);  // one staged copy at a time
    std::vector<std::atomic<int>> done(static_cast<size_t>(n));
    for (auto& d : done) d.store(0, std::memory_order_relaxed);
    job_ = &job;
    done_ = done.data();
    n_ = n;
    const uint64_t g = gen_.fetch_add(1, std::memory_order_acq_rel) + 1;
    {
      std::lock_guard<std::mutex> lk(mu_);  // pairs with the sleepers' predicate check
    }
    cv_.notify_all();
    int issued = 0, rc = TOEP_OK;
    auto issue_ready = [&]() {
      while (issued < n && done[issued].load(std::memory_order_acquire)) {
        if (rc == TOEP_OK) rc = on_ready(issued);
        ++issued;
      }
    };
    for (int c = 0; c < n; c += kWorkers + 1) {
      job(c);
      done[c].store(1, std::memory_order_release);
      issue_ready();
    }
    for (int w = 0; w < kWorkers; ++w)
      while (finished_[w].v.load(std::memory_order_acquire) != g) {
        issue_ready();
        _mm_pause();
      }
    issue_ready();
    return rc;
  }

 private:
  struct alignas(64) Slot {
    std::atomic<uint64_t> v{0};
  };
  CopyPool() : pid_(getpid()) {
    for (int i = 0; i < kWorkers; ++i) threads_.emplace_back([this, i] { loop(i); });
  }
  static int64_t now_ns() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
  }
  void loop(int w) {
    uint64_t seen = 0;
    for (;;) {
      int64_t t0 = now_ns();
      uint64_t g;
      for (unsigned spins = 0;; ++spins) {
        if (stop_.load(std::memory_order_acquire)) return;
        g = gen_.load(std::memory_order_acquire);
        if (g != seen) break;
        if ((spins & 1023u) == 0 && now_ns() - t0 > 2000000) {
          std::unique_lock<std::mutex> lk(mu_);
          cv_.wait(lk, [&] { return stop_.load() || gen_.load(std::memory_order_acquire) != seen; });
          t0 = now_ns();
          continue;
        }
        _mm_pause();
      }
      seen = g;
      const std::function<void(int)>& job = *job_;
      for (int c = w + 1; c < n_; c += kWorkers + 1) {
        job(c);
        done_[c].store(1, std::memory_order_release);
      }
      finished_[w].v.store(g, std::memory_order_release);
    }
  }
  std::vector<std::thread> threads_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_;
  const std::function<void(int)>* job_ = nullptr;
  std::atomic<int>* done_ = nullptr;
  int n_ = 0;
  std::atomic<uint64_t> gen_{0};
  std::atomic<bool> stop_{false};  // (never set: the pool lives for the whole process)
  pid_t pid_;
  Slot finished_[kWorkers];
};

}  // namespace

// memcpy with non-temporal stores: the staged bytes go to DRAM instead of sitting dirty in the CPU
// caches, where the DMA engine would have to snoop them out (a cached staging buffer transferred at
// 31 GB/s against 50 GB/s for a clean one)
void stream_copy(char* dst, const char* src, size_t n) {
  size_t i = 0;
  if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    for (; i + 64 <= n; i += 64) {
      const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
      const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
      const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
      const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
    }
    _mm_sfence();
  }
  if (i < n) std::memcpy(dst + i, src + i, n - i);
}

int staged_h2d(const void* src, void* dst_pinned, void* dev, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return TOEP_OK;
  // The copy threads stage one slice each in parallel; the DMA is ONE transfer issued when all are
  // staged: a transfer has ~9 us of fixed cost on these boxes (5 x 368 KB DMAs took 80 us against
  // 37 us for one 1.84 MB DMA, tools/e2e_timeline.py), more than pipelining slices saves.
  constexpr int kParts = CopyPool::kWorkers + 1;
  const size_t kChunk = std::max<size_t>(size_t{64} << 10, ((bytes + kParts - 1) / kParts + 4095) & ~size_t{4095});
  const int n = static_cast<int>((bytes + kChunk - 1) / kChunk);
  const char* sp = static_cast<const char*>(src);
  char* pp = static_cast<char*>(dst_pinned);
  auto len = [&](int c) { return std::min(kChunk, bytes - static_cast<size_t>(c) * kChunk); };
  const std::function<void(int)> job = [&](int c) {
    stream_copy(pp + static_cast<size_t>(c) * kChunk, sp + static_cast<size_t>(c) * kChunk, len(c));
  };
  const std::function<int(int)> ready = [&](int c) -> int {
    if (c + 1 < n) return TOEP_OK;  // all slices staged once the last one is (ready() runs in order)
    const cudaError_t e = cudaMemcpyAsync(dev, dst_pinned, bytes, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) {
      set_error("staged H2D copy failed: %s", cudaGetErrorString(e));
      return TOEP_ERR_CUDA;
    }
    return TOEP_OK;
  };
  return CopyPool::get().run(n, job, ready);
}

// Large pageable uploads (the generator blocks of toep_op_create, 0.9-4 GB at the BASELINE shapes):
// the driver's own pageable path moves them at 8-9 GB/s.  Here the library's copy threads stage
// 16 MB chunks into one of two page-locked buffers while the DMA of the previous chunk runs
// (double buffering, an event per buffer), so the upload runs near the DMA rate.  The staging
// buffers are process-lifetime and one upload runs at a time.
int pipelined_h2d(const void* src, void* dst, size_t bytes, cudaStream_t s) {
  constexpr size_t kChunk = size_t{16} << 20;
  if (bytes <= kChunk / 4) {  // small: the driver's path is fine
    TOEP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return TOEP_OK;
  }
  static std::mutex mu;
  static void* stage[2] = {nullptr, nullptr};
  static cudaEvent_t done[2] = {nullptr, nullptr};
  std::lock_guard<std::mutex> lock(mu);
  for (int h = 0; h < 2; ++h) {
    if (stage[h] == nullptr) {
      if (cudaHostAlloc(&stage[h], kChunk, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        stage[h] = nullptr;
        TOEP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));  // fall back to the driver's path
        return TOEP_OK;
      }
      TOEP_CUDA(cudaEventCreateWithFlags(&done[h], cudaEventDisableTiming));
      TOEP_CUDA(cudaEventRecord(done[h], s));
    }
  }
  const char* sp = static_cast<const char*>(src);
  char* dp = static_cast<char*>(dst);
  int h = 0;
  for (size_t off = 0; off < bytes; off += kChunk, h ^= 1) {
    const size_t len = std::min(kChunk, bytes - off);
    TOEP_CUDA(cudaEventSynchronize(done[h]));  // this buffer's previous DMA has read it
    TOEP_TRY(staged_h2d(sp + off, stage[h], dp + off, len, s));
    TOEP_CUDA(cudaEventRecord(done[h], s));
  }
  return TOEP_OK;
}

}  // namespace toep
