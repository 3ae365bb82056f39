// No C++ exception may cross the C ABI (include/rnnb.h): every entry point
// that allocates host memory runs its body through abi_guard, which maps
// std::bad_alloc / length_error to RNNB_ENOMEM and anything else to
// RNNB_EINVAL with the message kept for rnnb_last_error().
#pragma once
#include <new>
#include <stdexcept>
#include <string>

#include <cuda_runtime.h>

#include "../../include/rnnb.h"

namespace rnnb {
rnnb_status set_error(rnnb_status s, const std::string& msg);  // rnnb_api.cu

template <class F>
rnnb_status abi_guard(const char* where, F&& body) noexcept {
  try {
    return body();
  } catch (const std::bad_alloc&) {
    return set_error(RNNB_ENOMEM, std::string(where) + ": host allocation failed");
  } catch (const std::length_error&) {
    return set_error(RNNB_ENOMEM, std::string(where) + ": requested size too large");
  } catch (const std::exception& e) {
    return set_error(RNNB_EINVAL, std::string(where) + ": " + e.what());
  } catch (...) {
    return set_error(RNNB_EINVAL, std::string(where) + ": unknown C++ exception");
  }
}

// Makes `dev` current for the scope and restores the caller's device on
// every exit path (early error returns included).
struct DeviceGuard {
  int prev = 0;
  bool switched = false;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) {
      err = cudaSetDevice(dev);
      switched = err == cudaSuccess;
    }
  }
  ~DeviceGuard() {
    if (switched) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};
}  // namespace rnnb
