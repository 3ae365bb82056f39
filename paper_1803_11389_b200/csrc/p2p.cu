// Peer-memory plumbing for the multi-GPU partitions: device
// buffers exported to the other ranks' processes by CUDA IPC, peer access for
// ranks in one process, and stream-ordered flags.  The data itself moves by
// the layer kernels' own epilogue stores into mapped peer buffers
// (rnnb_forward_ex); a flag tells the consumer the rows are there.
//
// No kernel ever spins on a flag: a signal is a one-thread kernel that
// publishes with st.release.sys after everything earlier in its stream, and
// a wait is a stream wait-value operation (the stream does not start the
// next kernel until the flag reaches the value), so emulated ranks sharing
// one GPU cannot deadlock on residency.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "../../include/rnnb.h"

namespace rnnb {
rnnb_status set_error(rnnb_status s, const std::string& msg);  // rnnb_api.cu
}
using rnnb::set_error;

namespace {

#define P2P_TRY(expr)                                                                          \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e != cudaSuccess) return set_error(RNNB_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

__global__ void flag_signal_kernel(unsigned int* flag, unsigned int value) {
  // every earlier kernel of this stream has completed; make its stores (local
  // or to mapped peer memory) visible system-wide before the flag
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
}

typedef CUresult (*WaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*DevAttrFn)(int*, CUdevice_attribute, CUdevice);
typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);

AddrRangeFn addr_range_fn() {
  static AddrRangeFn fn = nullptr;
  static bool done = false;
  if (!done) {
    done = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<AddrRangeFn>(p);
  }
  return fn;
}

WaitValue32Fn wait_fn() {
  static WaitValue32Fn fn = nullptr;
  static bool done = false;
  if (!done) {
    done = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WaitValue32Fn>(p);
  }
  return fn;
}

// CU_STREAM_WAIT_VALUE_FLUSH where the device supports it: remote writes that
// reached the device before the wait was satisfied are visible downstream
bool can_flush(int device) {
  static int cache[64];
  static bool init[64];
  if (device < 0 || device >= 64) return false;
  if (!init[device]) {
    init[device] = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    int v = 0;
    if (cudaGetDriverEntryPoint("cuDeviceGetAttribute", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      reinterpret_cast<DevAttrFn>(p)(&v, CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES, (CUdevice)device);
    cache[device] = v;
  }
  return cache[device] != 0;
}

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DevGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

extern "C" {

rnnb_status rnnb_dev_alloc(int device, size_t bytes, void** ptr) {
  if (!ptr) return set_error(RNNB_EINVAL, "null ptr");
  *ptr = nullptr;
  if (bytes == 0) return set_error(RNNB_EINVAL, "zero-byte allocation");
  DevGuard g(device);
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaErrorMemoryAllocation) return set_error(RNNB_ENOMEM, "cudaMalloc: out of device memory");
  P2P_TRY(e);
  P2P_TRY(cudaMemset(p, 0, bytes));
  *ptr = p;
  return RNNB_OK;
}

rnnb_status rnnb_dev_free(int device, void* ptr) {
  if (!ptr) return RNNB_OK;
  DevGuard g(device);
  P2P_TRY(cudaFree(ptr));
  return RNNB_OK;
}

rnnb_status rnnb_ipc_handle(const void* ptr, void* handle, uint64_t* offset) {
  if (!ptr || !handle || !offset) return set_error(RNNB_EINVAL, "null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == RNNB_IPC_HANDLE_BYTES, "IPC handle size");
  // the handle names the whole cudaMalloc allocation (a caching allocator
  // may have sub-allocated ptr from it): report ptr's offset inside it
  AddrRangeFn range = addr_range_fn();
  if (!range) return set_error(RNNB_EUNSUPPORTED, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) return set_error(RNNB_EINVAL, "not a device allocation");
  cudaIpcMemHandle_t h;
  P2P_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  memcpy(handle, &h, sizeof(h));
  *offset = (uint64_t)((CUdeviceptr)ptr - base);
  return RNNB_OK;
}

rnnb_status rnnb_ipc_open(int device, const void* handle, void** ptr) {
  if (!handle || !ptr) return set_error(RNNB_EINVAL, "null argument");
  *ptr = nullptr;
  DevGuard g(device);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  P2P_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return RNNB_OK;
}

rnnb_status rnnb_ipc_close(int device, void* ptr) {
  if (!ptr) return RNNB_OK;
  DevGuard g(device);
  P2P_TRY(cudaIpcCloseMemHandle(ptr));
  return RNNB_OK;
}

rnnb_status rnnb_peer_access(int device, int peer) {
  if (device == peer) return RNNB_OK;
  int ok = 0;
  P2P_TRY(cudaDeviceCanAccessPeer(&ok, device, peer));
  if (!ok) return set_error(RNNB_EUNSUPPORTED, "no peer access between these devices");
  DevGuard g(device);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return RNNB_OK;
  }
  P2P_TRY(e);
  return RNNB_OK;
}

rnnb_status rnnb_flag_signal(int device, void* flag, uint32_t value, void* stream) {
  if (!flag) return set_error(RNNB_EINVAL, "null flag");
  DevGuard g(device);
  flag_signal_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<unsigned int*>(flag), value);
  P2P_TRY(cudaGetLastError());
  return RNNB_OK;
}

rnnb_status rnnb_flag_wait(int device, const void* flag, uint32_t value, void* stream) {
  if (!flag) return set_error(RNNB_EINVAL, "null flag");
  WaitValue32Fn fn = wait_fn();
  if (!fn) return set_error(RNNB_EUNSUPPORTED, "cuStreamWaitValue32 unavailable");
  DevGuard g(device);
  unsigned int fl = CU_STREAM_WAIT_VALUE_GEQ;
  if (can_flush(device)) fl |= CU_STREAM_WAIT_VALUE_FLUSH;
  CUresult r = fn(static_cast<CUstream>(stream), (CUdeviceptr)flag, value, fl);
  if (r != CUDA_SUCCESS) return set_error(RNNB_ECUDA, "cuStreamWaitValue32 failed");
  return RNNB_OK;
}

}  // extern "C"
