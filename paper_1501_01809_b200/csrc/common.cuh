// common.cuh -- error convention, CUDA helpers and device buffers.
//
// Errors follow the reference: loam::Error(kind, message) (common.hpp:36-49)
// becomes an int code 1 + kind with a thread-local message.  Internally the
// engine throws loam_gpu::Error and the C ABI (capi.cu) converts.
#pragma once
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <exception>
#include <thread>
#include <utility>
#include <vector>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <stdexcept>
#include <string>

#include "loam_gpu.h"

namespace loam_gpu {

class Error : public std::runtime_error {
public:
  Error(int code, const std::string& what) : std::runtime_error(what), code_(code) {}
  int code() const { return code_; }

private:
  int code_;
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
inline void require(bool cond, int code, const std::string& msg) {
  if (!cond) fail(code, msg);
}

#define LG_CUDA(call)                                                                    \
  do {                                                                                   \
    cudaError_t err_ = (call);                                                           \
    if (err_ != cudaSuccess)                                                             \
      ::loam_gpu::fail(LOAM_GPU_ERR_CUDA, std::string(#call) + ": " +                    \
                                              cudaGetErrorString(err_) + " (" __FILE__ ":" + \
                                              std::to_string(__LINE__) + ")");           \
  } while (0)

// Number of kernels launched by this library (bench gpu_launches).
extern std::atomic<int64_t> g_launches;
inline void count_launch(int64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }
#define LG_LAUNCH_CHECK() LG_CUDA(cudaGetLastError())

// Owned device buffer (stream-ordered allocation from the default mempool).
template <class T>
class DevBuf {
public:
  DevBuf() = default;
  DevBuf(size_t n, cudaStream_t s) { alloc(n, s); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_), s_(o.s_) { o.p_ = nullptr; o.n_ = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_; n_ = o.n_; s_ = o.s_;
      o.p_ = nullptr; o.n_ = 0;
    }
    return *this;
  }
  void alloc(size_t n, cudaStream_t s) {
    release();
    s_ = s;
    n_ = n;
    if (n) LG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), s));
  }
  void release() {
    if (p_) cudaFreeAsync(p_, s_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  size_t bytes() const { return n_ * sizeof(T); }

private:
  T* p_ = nullptr;
  size_t n_ = 0;
  cudaStream_t s_ = nullptr;
};

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

// Raise a kernel's dynamic shared-memory limit to at least `smem`, once per
// kernel (keyed by the kernel's address: instantiations that share a function
// type must not share the cache).
inline void ensure_dynamic_smem(const void* kern, size_t smem) {
  static std::mutex m;
  static std::unordered_map<const void*, size_t> done;
  std::lock_guard<std::mutex> g(m);
  size_t& cur = done[kern];
  if (cur < smem) {
    LG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cur = smem;
  }
}

constexpr int kNumSMs = 148; // B200

// Developer phase timing of plan construction (LOAM_GPU_PLAN_TIMING=1):
// synchronises `s` and prints the host wall clock since the previous tick.
inline void plan_tick(const char* label, cudaStream_t s) {
  static const bool on = std::getenv("LOAM_GPU_PLAN_TIMING") != nullptr;
  if (!on) return;
  static auto last = std::chrono::steady_clock::now();
  cudaStreamSynchronize(s);
  const auto now = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[plan] %-28s %9.3f ms\n", label, std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

// Programmatic dependent launch (PDL): a kernel launched this way may start
// while the previous kernel in the stream drains; it must execute
// griddepcontrol.wait (async.cuh grid_dep_wait) before it reads anything a
// previous kernel may write or writes anything at all.  Only kernels written
// that way are launched through here.  LOAM_GPU_NO_PDL=1 disables it.
inline bool pdl_on() {
  static const bool on = std::getenv("LOAM_GPU_NO_PDL") == nullptr;
  return on;
}
template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_on() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (e != cudaSuccess) throw Error(LOAM_GPU_ERR_CUDA, std::string("cudaLaunchKernelEx: ") + cudaGetErrorString(e));
}

// Uploads the concatenation of host byte vectors (one per plan chunk) into one
// device buffer without building the concatenation on the host; returns the
// byte offset of every part.  The copies run from all host cores (the
// pageable-memory staging is CPU work).
template <class Parts>
std::vector<size_t> upload_parts(DevBuf<uint8_t>& dst, const Parts& parts, cudaStream_t s) {
  std::vector<size_t> off(parts.size() + 1, 0);
  for (size_t i = 0; i < parts.size(); ++i) off[i + 1] = off[i] + parts[i]->size();
  dst.alloc(off.back() + 16, s);
  LG_CUDA(cudaStreamSynchronize(s)); // the buffer exists before other threads copy into it
  uint8_t* base = dst.get();
  std::vector<std::thread> th;
  std::vector<cudaError_t> err(parts.size(), cudaSuccess);
  for (size_t i = 0; i < parts.size(); ++i)
    th.emplace_back([&, i] {
      if (!parts[i]->empty()) err[i] = cudaMemcpy(base + off[i], parts[i]->data(), parts[i]->size(), cudaMemcpyHostToDevice);
    });
  for (auto& x : th) x.join();
  for (auto e : err)
    if (e != cudaSuccess) throw Error(LOAM_GPU_ERR_CUDA, std::string("plan upload: ") + cudaGetErrorString(e));
  return off;
}

// Host arrays for plan builders: no value-initialisation (the copy that fills
// them is the first write), and their pages first-touched by all host cores
// -- single-threaded page faults were most of a 300 MB download's 140 ms.
template <class T>
struct NoInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = NoInitAlloc<U>;
  };
  NoInitAlloc() = default;
  template <class U>
  NoInitAlloc(const NoInitAlloc<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
};
template <class T>
using hvec = std::vector<T, NoInitAlloc<T>>;
inline void parallel_touch(void* p, size_t bytes) {
  const size_t chunk = (size_t)4 << 20;
  const size_t n = (bytes + chunk - 1) / chunk;
  if (n <= 1) {
    if (bytes) std::memset(p, 0, bytes);
    return;
  }
  const int T = std::max(1, std::min<int>((int)std::thread::hardware_concurrency(), (int)n));
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      for (size_t k = t; k < n; k += T) std::memset(static_cast<uint8_t*>(p) + k * chunk, 0, std::min(chunk, bytes - k * chunk));
    });
  for (auto& x : th) x.join();
}
template <class T>
hvec<T> host_array(size_t n) {
  hvec<T> v;
  v.resize(n);
  parallel_touch(v.data(), n * sizeof(T));
  return v;
}

// Device -> pageable host copies of a plan builder's inputs.
struct D2H {
  void* dst;
  const void* src;
  size_t bytes;
};
// (A pinned staging buffer measured slower here: cudaMallocHost of the ~300
// MB a P2 plan needs costs more than the pageable copies; threads per array
// did not overlap the pageable staging either.)
inline void parallel_d2h(const std::vector<D2H>& copies, cudaStream_t s) {
  for (const D2H& c : copies)
    if (c.bytes) LG_CUDA(cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
}

// Host-side plan construction runs on all host cores: parallel_chunks(n, f)
// splits [0, n) into contiguous chunks (at most one per thread, `align`-sized
// multiples) and calls f(chunk, begin, end) concurrently; the first exception
// is rethrown after every thread joined.  LOAM_GPU_PLAN_THREADS overrides the
// thread count (1 = serial).
inline int plan_threads() {
  static const int t = [] {
    const char* e = std::getenv("LOAM_GPU_PLAN_THREADS");
    int v = e ? std::atoi(e) : (int)std::thread::hardware_concurrency();
    return std::max(1, std::min(v, 64));
  }();
  return t;
}
template <class F>
int parallel_chunks(int64_t n, int64_t align, F&& f, int64_t min_chunk = 4096) {
  const int64_t units = (n + align - 1) / align;
  int T = (int)std::max<int64_t>(1, std::min<int64_t>(plan_threads(), (n + min_chunk - 1) / min_chunk));
  T = (int)std::max<int64_t>(1, std::min<int64_t>(T, units));
  std::vector<int64_t> cut(T + 1);
  for (int t = 0; t <= T; ++t) cut[t] = std::min<int64_t>(n, (units * t / T) * align);
  if (T == 1) {
    f(0, (int64_t)0, n);
    return 1;
  }
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> err(T);
  for (int t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      try {
        f(t, cut[t], cut[t + 1]);
      } catch (...) {
        err[t] = std::current_exception();
      }
    });
  for (auto& x : th) x.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
  return T;
}

} // namespace loam_gpu
