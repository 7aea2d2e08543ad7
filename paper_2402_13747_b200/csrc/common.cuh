// common.cuh — error mapping, stream-ordered device buffers and launch helpers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

namespace pcr {

// Errors surface through the C ABI as pcr_last_error(); messages reproduce the
// reference's std::runtime_error texts where one exists.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define PCR_CUDA(call)                                                                          \
  do {                                                                                          \
    cudaError_t pcr_e_ = (call);                                                                \
    if (pcr_e_ != cudaSuccess) {                                                                \
      throw ::pcr::Error(pcr_e_ == cudaErrorMemoryAllocation ? 3 : 2,                           \
                         std::string("cuda ") + #call + ": " + cudaGetErrorString(pcr_e_));    \
    }                                                                                           \
  } while (0)

// Wait for a stream by polling it: the host loops of the trace and refine stages read a
// few counters back per chunk, and a blocking / yielding wait can wake up milliseconds
// late on a busy host (measured: the same C2 trace stage 1.4-3.6 s across repetitions),
// so the library spins on cudaStreamQuery instead of sleeping in cudaStreamSynchronize.
inline void stream_wait(cudaStream_t s) {
  cudaError_t e;
  while ((e = cudaStreamQuery(s)) == cudaErrorNotReady) {
  }
  if (e != cudaSuccess)
    throw ::pcr::Error(e == cudaErrorMemoryAllocation ? 3 : 2, std::string("cuda stream wait: ") + cudaGetErrorString(e));
}

// Launch errors; with PCR_SYNC_LAUNCHES=1 in the environment every checked launch is
// also synchronised, so an asynchronous fault names the kernel's source line (debug aid).
bool sync_launches();
inline void launch_check(const char* file, int line) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && sync_launches()) e = cudaDeviceSynchronize();
  if (e != cudaSuccess)
    throw Error(e == cudaErrorMemoryAllocation ? 3 : 2,
                std::string("cuda launch at ") + file + ":" + std::to_string(line) + ": " + cudaGetErrorString(e));
}
#define PCR_LAUNCH_CHECK() ::pcr::launch_check(__FILE__, __LINE__)

// Stream-ordered device buffer (cudaMallocAsync pool); never copied, only moved.
template <typename T>
class DBuf {
 public:
  DBuf() = default;
  DBuf(size_t n, cudaStream_t s) { alloc(n, s); }
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept { swap(o); }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      swap(o);
    }
    return *this;
  }
  void alloc(size_t n, cudaStream_t s) {
    release();
    stream_ = s;
    n_ = n;
    if (n) PCR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), s));
  }
  // Grow to at least n elements, keeping the first `keep` elements.
  void reserve(size_t n, size_t keep, cudaStream_t s) {
    if (n <= n_) return;
    T* q = nullptr;
    PCR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&q), n * sizeof(T), s));
    if (keep && p_) PCR_CUDA(cudaMemcpyAsync(q, p_, keep * sizeof(T), cudaMemcpyDeviceToDevice, s));
    if (p_) cudaFreeAsync(p_, stream_);
    p_ = q;
    n_ = n;
    stream_ = s;
  }
  void release() {
    if (p_) cudaFreeAsync(p_, stream_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  void swap(DBuf& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    std::swap(stream_, o.stream_);
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
  cudaStream_t stream_ = nullptr;
};

inline unsigned blocks_for(uint64_t n, unsigned threads, unsigned cap = 148u * 64u) {
  uint64_t b = (n + threads - 1) / threads;
  if (b == 0) b = 1;
  return static_cast<unsigned>(b < cap ? b : cap);
}

// Launch and transfer accounting: every kernel launch and host<->device copy of the
// library goes through these counters so bench.py can report them per timed step.
extern uint64_t g_launch_count, g_h2d_bytes, g_d2h_bytes;
inline void count_launch() { ++g_launch_count; }

template <typename T>
void d2h(T* dst, const T* src, size_t n, cudaStream_t s) {
  if (n) {
    PCR_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    g_d2h_bytes += n * sizeof(T);
  }
}
template <typename T>
void h2d(T* dst, const T* src, size_t n, cudaStream_t s) {
  if (n) {
    PCR_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
    g_h2d_bytes += n * sizeof(T);
  }
}

}  // namespace pcr
