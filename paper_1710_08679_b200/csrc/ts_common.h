// ts_common.h — shared host/device plumbing for libtsgpu (error model, device
// buffers, launch helpers). Internal; the public boundary is include/tsgpu.h.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "../../include/tsgpu.h"

namespace tsg {

// Exception carrying a ts_status; translated to a return code at the C ABI.
// Mirrors the reference's exception hierarchy (errors.hpp:9-31).
struct Error : std::runtime_error {
  ts_status code;
  Error(ts_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(ts_status c, const std::string& m) { throw Error(c, m); }
[[noreturn]] inline void validation(const std::string& m) { throw Error(TS_ERR_VALIDATION, m); }

void set_last_error(const std::string& m);

#define TS_CUDA(x)                                                                      \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      ::tsg::fail(TS_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));        \
  } while (0)

#define TS_CUDA_LAUNCH() TS_CUDA(cudaGetLastError())

// Ensure a usable device exists; the product has no CPU fallback.
void require_device();

// Allocator whose value-initialising constructions default-initialise: a
// HostVec<T>(n) of scalars is NOT zero-filled, so big setup arrays are first
// touched (paged in) by the parallel loops that fill them, not by one thread.
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
  void construct(U* p) noexcept(std::is_nothrow_default_constructible<U>::value) {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
};
template <class T>
using HostVec = std::vector<T, NoInitAlloc<T>>;

// RAII device allocation.
template <typename T>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t n) { alloc(n); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_; n_ = o.n_;
      o.p_ = nullptr; o.n_ = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t n) {
    release();
    if (n) TS_CUDA(cudaMalloc(&p_, n * sizeof(T)));
    n_ = n;
  }
  // grow-only reallocation (contents not preserved)
  void ensure(size_t n) { if (n > n_) alloc(n); }
  void upload(const T* h, size_t n, cudaStream_t s = 0) {
    ensure(n);
    if (n) TS_CUDA(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  template <class A>
  void upload(const std::vector<T, A>& h, cudaStream_t s = 0) { upload(h.data(), h.size(), s); }
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

// NVTX range for the whole scope (solve, outer iterations, multigrid levels, EBE
// products, Green's batches): free without a profiler, named phases under nsys / ncu
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// setup phase timing to stderr when TSGPU_SETUP_PROFILE is set
void setup_mark(const char* what);

inline unsigned grid_for(int64_t n, int block) {
  const int64_t g = (n + block - 1) / block;
  return static_cast<unsigned>(g < 1 ? 1 : g);
}

// Host mesh (tetsolve::Mesh, mesh.hpp:26-42).
struct Mesh {
  std::vector<double> coords;       // [N][3]
  std::vector<int32_t> tets10;      // [E][10]
  std::vector<int32_t> material_id; // [E]
  int32_t vertex_count = 0;
  std::vector<int32_t> bc_node;
  std::vector<int8_t> bc_axis;
  int32_t n_nodes() const { return static_cast<int32_t>(coords.size() / 3); }
  int32_t n_elems() const { return static_cast<int32_t>(tets10.size() / 10); }
  std::vector<uint8_t> dirichlet_mask() const;
};

Mesh generate_box_mesh(const double ext[3], const int32_t div[3],
                       const std::vector<double>& interfaces, int fixed_boundary);

}  // namespace tsg

// opaque ABI handle
struct ts_mesh {
  tsg::Mesh m;
};
