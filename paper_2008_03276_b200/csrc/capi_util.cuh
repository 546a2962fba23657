// Error plumbing for the C ABI: no exceptions cross the boundary; the last
// error message is kept per thread and returned by paqif_last_error().
#pragma once
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
#include "../../include/paqif_b200.h"

namespace paqif {

inline char* last_error_buf() {
  static thread_local char buf[512] = "";
  return buf;
}

inline int set_arg_error(const char* what) {
  std::snprintf(last_error_buf(), 512, "argument error: %s", what);
  return PAQIF_E_ARG;
}

inline int set_cuda_error(const char* what, cudaError_t e) {
  std::snprintf(last_error_buf(), 512, "%s: %s", what, cudaGetErrorString(e));
  return PAQIF_E_CUDA;
}

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(what, e);
  return PAQIF_OK;
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(size_t count) {
    if (count && cudaMalloc(&p, count * sizeof(T)) != cudaSuccess) p = nullptr;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  bool ok() const { return p != nullptr; }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

}  // namespace paqif
