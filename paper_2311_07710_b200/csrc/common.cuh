// common.cuh — error handling, device buffers and arithmetic helpers shared by
// the rAPDHG B200 library. Everything here is fp64 and HBM-bound; no tensor
// cores are involved (nothing on this path is a dense contraction).
#pragma once

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
    RB_CUDA(cudaMalloc(&p_, sizeof(T) * (n ? n : 1)));
  }
  void reset() {
    if (p_) cudaFree(p_);
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
template <typename T>
class PinnedBuf {
 public:
  PinnedBuf() = default;
  ~PinnedBuf() {
    if (p_) cudaFreeHost(p_);
  }
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  void alloc(std::size_t n) {
    if (p_) cudaFreeHost(p_);
    RB_CUDA(cudaMallocHost(&p_, sizeof(T) * (n ? n : 1)));
    n_ = n;
  }
  T* get() const { return p_; }
  T& operator[](std::size_t i) { return p_[i]; }
  std::size_t size() const { return n_; }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
};

constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace rb
