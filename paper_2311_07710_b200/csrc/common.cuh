// common.cuh — error handling, device buffers and arithmetic helpers shared by
// the rAPDHG B200 library. Everything here is fp64 and HBM-bound; no tensor
// cores are involved (nothing on this path is a dense contraction).
#pragma once

#include <type_traits>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <mutex>
#include <utility>
#include <vector>
#include <cstdlib>

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

#include "rapdhg_b200.h"

namespace rb {

// Exception carrying a C-ABI error code; the capi layer turns it into a return
// value + rapdhg_last_error() message, mirroring the reference's exception
// types (std::invalid_argument -> RAPDHG_E_INVALID_ARGUMENT, ...).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void invalid(const std::string& m) { throw Error(RAPDHG_E_INVALID_ARGUMENT, m); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw Error(RAPDHG_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                                   std::to_string(line) + ")");
}
#define RB_CUDA(x) ::rb::cuda_check((x), #x, __FILE__, __LINE__)
#define RB_LAUNCH_CHECK() ::rb::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// Owning device allocation (cudaMalloc'd, freed on destruction). Not copyable.
// Device memory comes from the device's default stream-ordered pool, which
// keeps freed memory (release threshold: unlimited), so repeated solves do not
// pay cudaMalloc/cudaFree (tens of ms each on large buffers). Allocation and
// free are ordered on the legacy default stream, which every solver stream
// (blocking streams) synchronises with. RAPDHG_POOL=0: plain cudaMalloc/Free.
inline bool pool_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("RAPDHG_POOL");
    return !(e && e[0] == '0');
  }();
  return on;
}
inline void pool_prepare() {
  static std::atomic<unsigned long long> done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return;
  const unsigned long long bit = 1ull << dev;
  if (done.load() & bit) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    unsigned long long keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    // RAPDHG_POOL_RESERVE_MB: map this much up front (growing the pool later
    // maps pages synchronously, which can stall a setup for 100+ ms)
    if (const char* r = std::getenv("RAPDHG_POOL_RESERVE_MB")) {
      const std::size_t bytes = static_cast<std::size_t>(std::atoll(r)) << 20;
      void* p = nullptr;
      if (bytes && cudaMallocAsync(&p, bytes, cudaStreamPerThread) == cudaSuccess) {
        cudaFreeAsync(p, cudaStreamPerThread);
        cudaStreamSynchronize(cudaStreamPerThread);
      }
    }
  }
  done.fetch_or(bit);
}
// Grow-only reservation of the current device's pool to at least `bytes`
// (one allocation + free of the difference): a solve's many large
// allocations are then carved from memory already mapped. Without it, repeated
// solves of one instance occasionally found no free block of the right size
// (the planner threads allocate concurrently, so the free-list layout varies)
// and grew the pool in the middle of the setup, stalling every stream of the
// device for 0.3-1.4 s (C4: setup 0.15 s typically, 0.8-1.5 s then).
inline void pool_reserve(std::size_t bytes) {
  if (!pool_enabled() || bytes == 0) return;
  static std::mutex mu;
  static std::size_t reserved[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return;
  std::lock_guard<std::mutex> g(mu);
  if (reserved[dev] >= bytes) return;
  pool_prepare();
  cudaStream_t s = nullptr;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return;
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes, s) == cudaSuccess) {
    cudaFreeAsync(p, s);
    reserved[dev] = bytes;
  } else {
    cudaGetLastError();  // not enough memory for the reservation: allocate as needed
  }
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
}

// The stream pool allocations and frees of this host thread are ordered on
// the stream of the work they serve: every solver object runs on its own
// NON-BLOCKING stream and enters an AllocStreamScope of it for each call, so
// a temporary freed at the end of a setup function is ordered after the
// kernels that read it. Outside any scope (objects destroyed after their
// stream was synchronised) the per-thread default stream is used. Nothing in
// the library touches the legacy stream: a legacy-stream operation would
// synchronise with (and invalidate the graph capture of) any blocking stream
// of the process, ours or the caller's.
inline cudaStream_t& alloc_stream() {
  thread_local cudaStream_t s = cudaStreamPerThread;
  return s;
}
struct AllocStreamScope {
  cudaStream_t prev;
  explicit AllocStreamScope(cudaStream_t s) : prev(alloc_stream()) { alloc_stream() = s; }
  ~AllocStreamScope() { alloc_stream() = prev; }
  AllocStreamScope(const AllocStreamScope&) = delete;
  AllocStreamScope& operator=(const AllocStreamScope&) = delete;
};
// A non-blocking stream owned by a solver object: declared before the
// object's device buffers, so it is destroyed after them (they are freed on
// the alloc stream once the owner has synchronised it).
class OwnedStream {
 public:
  OwnedStream() = default;
  ~OwnedStream() { reset(); }
  OwnedStream(const OwnedStream&) = delete;
  OwnedStream& operator=(const OwnedStream&) = delete;
  cudaStream_t create(int priority = 0) {
    reset();
    RB_CUDA(cudaStreamCreateWithPriority(&s_, cudaStreamNonBlocking, priority));
    return s_;
  }
  void reset() {
    if (s_) {
      cudaStreamSynchronize(s_);
      cudaStreamDestroy(s_);
      s_ = nullptr;
    }
  }
  cudaStream_t get() const { return s_; }

 private:
  cudaStream_t s_ = nullptr;
};
// Declared LAST in a solver object: synchronises its streams before any of
// the object's buffers are freed (also when its constructor throws).
struct SyncBeforeFree {
  const cudaStream_t* a;
  const cudaStream_t* b;
  ~SyncBeforeFree() {
    if (a && *a) cudaStreamSynchronize(*a);
    if (b && *b) cudaStreamSynchronize(*b);
  }
};

inline void* dev_alloc(std::size_t bytes) {
  void* p = nullptr;
  if (pool_enabled()) {
    pool_prepare();
    RB_CUDA(cudaMallocAsync(&p, bytes, alloc_stream()));
  } else {
    RB_CUDA(cudaMalloc(&p, bytes));
  }
  return p;
}
inline void dev_free(void* p) {
  if (!p) return;
  if (pool_enabled()) cudaFreeAsync(p, alloc_stream());
  else cudaFree(p);
}

template <typename T>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(std::size_t n) { alloc(n); }
  ~DevBuf() { reset(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr, o.n_ = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      reset();
      p_ = o.p_, n_ = o.n_;
      o.p_ = nullptr, o.n_ = 0;
    }
    return *this;
  }
  void alloc(std::size_t n) {
    reset();
    n_ = n;
    // always allocate at least one element so pointers are valid for empty sets
    p_ = static_cast<T*>(dev_alloc(sizeof(T) * (n ? n : 1)));
  }
  void reset() {
    dev_free(p_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  std::size_t size() const { return n_; }
  void upload(const T* h, std::size_t n, cudaStream_t s) {
    if (n) RB_CUDA(cudaMemcpyAsync(p_, h, sizeof(T) * n, cudaMemcpyHostToDevice, s));
  }
  void download(T* h, std::size_t n, cudaStream_t s) const {
    if (n) RB_CUDA(cudaMemcpyAsync(h, p_, sizeof(T) * n, cudaMemcpyDeviceToHost, s));
  }
  void zero(cudaStream_t s) { RB_CUDA(cudaMemsetAsync(p_, 0, sizeof(T) * (n_ ? n_ : 1), s)); }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
};

// Pinned host staging buffer.
// Page-locked host blocks are expensive to create (cudaMallocHost pins pages:
// milliseconds), so released blocks are cached for reuse (same size class:
// next power of two >= 4 KB).
struct PinnedCache {
  std::mutex mu;
  std::vector<std::pair<std::size_t, void*>> free;
  ~PinnedCache() = default;  // process exit releases the pages
};
inline PinnedCache& pinned_cache() {
  static PinnedCache* c = new PinnedCache();  // never destroyed (outlives static buffers)
  return *c;
}
inline std::size_t pinned_class(std::size_t bytes) {
  std::size_t c = 4096;
  while (c < bytes) c <<= 1;
  return c;
}
inline void* pinned_acquire(std::size_t bytes) {
  const std::size_t cls = pinned_class(bytes);
  PinnedCache& pc = pinned_cache();
  {
    std::lock_guard<std::mutex> g(pc.mu);
    for (std::size_t i = 0; i < pc.free.size(); ++i)
      if (pc.free[i].first == cls) {
        void* p = pc.free[i].second;
        pc.free[i] = pc.free.back();
        pc.free.pop_back();
        return p;
      }
  }
  void* p = nullptr;
  RB_CUDA(cudaMallocHost(&p, cls));
  return p;
}
inline void pinned_release(void* p, std::size_t bytes) {
  if (!p) return;
  PinnedCache& pc = pinned_cache();
  std::lock_guard<std::mutex> g(pc.mu);
  pc.free.emplace_back(pinned_class(bytes), p);
}

template <typename T>
class PinnedBuf {
 public:
  PinnedBuf() = default;
  ~PinnedBuf() { pinned_release(p_, bytes_); }
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  void alloc(std::size_t n) {
    pinned_release(p_, bytes_);
    bytes_ = sizeof(T) * (n ? n : 1);
    p_ = static_cast<T*>(pinned_acquire(bytes_));
    n_ = n;
  }
  T* get() const { return p_; }
  T& operator[](std::size_t i) { return p_[i]; }
  std::size_t size() const { return n_; }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0, bytes_ = 0;
};

// Phase timer printed to stderr when RAPDHG_TRACE is set (synchronises the
// stream at each mark, so only for diagnosis).
struct Tracer {
  bool on, sync;
  cudaStream_t st;
  std::chrono::steady_clock::time_point t;
  explicit Tracer(cudaStream_t s) : on(std::getenv("RAPDHG_TRACE") != nullptr), st(s), t(std::chrono::steady_clock::now()) {
    const char* e = std::getenv("RAPDHG_TRACE");
    sync = !(e && e[0] == 'h');  // RAPDHG_TRACE=host: host timestamps only, no stream syncs
  }
  void mark(const char* what) {
    if (!on) return;
    if (st && sync) cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[rapdhg] %-30s %9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// Captures body() on stream s (thread-local mode) into an executable graph.
// A failure inside ends and drops the capture, so the stream stays usable,
// then rethrows; the graph is destroyed once instantiated (or not).
template <class F>
cudaGraphExec_t capture_graph(cudaStream_t s, F&& body) {
  RB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  try {
    body();
  } catch (...) {
    cudaGraph_t broken = nullptr;
    cudaStreamEndCapture(s, &broken);
    if (broken) cudaGraphDestroy(broken);
    cudaGetLastError();
    throw;
  }
  cudaGraph_t g = nullptr;
  RB_CUDA(cudaStreamEndCapture(s, &g));
  cudaGraphExec_t exec = nullptr;
  const cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
  cudaGraphDestroy(g);
  RB_CUDA(e);
  return exec;
}

// Step gate (power iterations run in device batches, engine.cu): a launch
// tagged with step i does nothing once the device recorded a stop at a step
// before i (*stop < i). The stop is written by step j's own last kernel, so no
// kernel ever reads a gate its own blocks write.
struct StepGate {
  const int* stop = nullptr;
  int step = 0;
  __device__ __forceinline__ bool closed() const { return stop && *stop < step; }
};
template <class T, class = void>
struct HasGate {
  __device__ __forceinline__ static bool closed(const T&) { return false; }
};
template <class T>
struct HasGate<T, std::void_t<decltype(T::gate)>> {
  __device__ __forceinline__ static bool closed(const T& t) { return t.gate.closed(); }
};

constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace rb
