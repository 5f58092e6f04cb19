// Shared runtime pieces of libxtsg: status/exception mapping, per-thread
// streams, host/device pointer staging, launch accounting.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/xtsg.h"

namespace xtsg {

// Internal exception carrying an ABI status code and payloads; converted at
// the C boundary by guard().
struct Status : std::runtime_error {
  int32_t code;
  int64_t p0, p1;
  Status(int32_t c, const std::string& m, int64_t a = 0, int64_t b = 0)
      : std::runtime_error(m), code(c), p0(a), p1(b) {}
};

[[noreturn]] inline void usage(const std::string& m) { throw Status(XTSG_E_USAGE, m); }
[[noreturn]] inline void data_error(const std::string& m) { throw Status(XTSG_E_DATA, m); }

struct ErrState {
  std::string msg;
  int64_t p0 = 0, p1 = 0;
};
ErrState& err_state();

template <class F>
int32_t guard(F&& f) {
  try {
    f();
    return XTSG_OK;
  } catch (const Status& s) {
    err_state() = {s.what(), s.p0, s.p1};
    return s.code;
  } catch (const std::exception& e) {
    err_state() = {e.what(), 0, 0};
    return XTSG_E_INTERNAL;
  } catch (...) {
    err_state() = {"unknown error", 0, 0};
    return XTSG_E_INTERNAL;
  }
}

#define XCUDA(call)                                                                    \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      throw ::xtsg::Status(XTSG_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Count of kernels launched through this library by the calling thread.
std::atomic<int64_t>& launch_counter();
inline void count_launch(int64_t n = 1) { launch_counter().fetch_add(n, std::memory_order_relaxed); }
#define XLAUNCH_CHECK()                                                                \
  do {                                                                                 \
    ::xtsg::count_launch();                                                            \
    XCUDA(cudaGetLastError());                                                         \
  } while (0)

// The calling thread's stream (created on first use, non-blocking).
cudaStream_t thread_stream();
// Throws XTSG_E_CUDA unless an sm_100 device is current.
void require_device();
int sm_count();

inline bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// RAII stream-ordered device buffer.
template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t n = 0;
  cudaStream_t st = nullptr;
  DevBuf() = default;
  DevBuf(size_t count, cudaStream_t s) : n(count), st(s) {
    if (n) XCUDA(cudaMallocAsync(reinterpret_cast<void**>(&ptr), n * sizeof(T), st));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), n(o.n), st(o.st) { o.ptr = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    ptr = o.ptr; n = o.n; st = o.st;
    o.ptr = nullptr; o.n = 0;
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (ptr) cudaFreeAsync(ptr, st);
    ptr = nullptr;
  }
  void zero() {
    if (n) XCUDA(cudaMemsetAsync(ptr, 0, n * sizeof(T), st));
  }
};

// Host -> device copy on stream s of a caller's host buffer. Pinned
// (page-locked / registered) memory goes straight to the copy engine;
// pageable memory of 8 MB and more is copied by the host worker threads into
// a pinned double buffer whose 64 MB chunks the copy engine moves while the
// next chunk is filled (a pageable cudaMemcpy runs at ~10 GB/s on one thread).
// Returns once the source may be reused (the last chunk has landed).
void h2d_copy(void* dst, const void* src, size_t bytes, cudaStream_t s);

// A caller-supplied buffer viewed on the device: device pointers are used in
// place, host pointers are staged through a temporary device copy.
template <class T>
struct InView {
  const T* dev = nullptr;
  DevBuf<T> tmp;
  InView(const T* p, size_t count, cudaStream_t s) {
    if (!p || count == 0) return;
    if (is_device_ptr(p)) {
      dev = p;
    } else {
      tmp = DevBuf<T>(count, s);
      h2d_copy(tmp.ptr, p, count * sizeof(T), s);
      dev = tmp.ptr;
    }
  }
};

template <class T>
struct OutView {
  T* dev = nullptr;
  T* host = nullptr;
  size_t n = 0;
  cudaStream_t st;
  DevBuf<T> tmp;
  OutView(T* p, size_t count, cudaStream_t s) : n(count), st(s) {
    if (!p || count == 0) return;
    if (is_device_ptr(p)) {
      dev = p;
    } else {
      host = p;
      tmp = DevBuf<T>(count, s);
      dev = tmp.ptr;
    }
  }
  // Copy back to host (if staged) and wait for the stream.
  void finish() {
    if (host) XCUDA(cudaMemcpyAsync(host, dev, n * sizeof(T), cudaMemcpyDeviceToHost, st));
    XCUDA(cudaStreamSynchronize(st));
  }
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Phase trace (XTSG_TRACE=1): device time between marks on one stream plus
// the host wall time, printed to stderr when the tracer goes out of scope.
// Diagnostics only; inactive (no events recorded) unless the variable is set.
struct PhaseTrace {
  const char* name;
  cudaStream_t st;
  bool on;
  std::vector<std::pair<const char*, cudaEvent_t>> ev;
  std::vector<double> host;
  PhaseTrace(const char* n, cudaStream_t s);
  void mark(const char* label);
  ~PhaseTrace();
};

}  // namespace xtsg
