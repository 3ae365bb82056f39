// Shared device helpers for the blocked SRU/QRNN kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "paper_1803_11389_b200 kernels target sm_100a only"
#endif

namespace rnnb {

// LINEAR: a dense layer Y = X W^T (+ b) on the same kernels (no gates, no
// scan): the cfg3 acoustic model's input projection and logits
enum Cell : int { SRU = 1, QRNN = 2, LINEAR = 3 };
// Extra destinations of the last layer's h stores (peer GPUs' mapped buffers:
// the pipeline hand-off / all-gather rides on the epilogue's stores).
constexpr int kMaxPeers = 7;

// h store of a layer epilogue: the local output plus each peer destination
// (constant indices: no dynamic indexing into the kernel parameter block).
template <typename Args, typename T>
__device__ __forceinline__ void store_h(const Args& a, int64_t i, T h) {
  a.Hout[i] = h;
#pragma unroll
  for (int p = 0; p < kMaxPeers; ++p)
    if (p < a.npeer) a.Hpeer[p][i] = h;
}
// x-operand rounding applied inside the FFMA kernel so its numerics match the
// tensor-core modes (TF32: cvt.rna.tf32; BF16: round-to-nearest-even).
enum XRound : int { XR_NONE = 0, XR_BF16 = 1, XR_TF32 = 2 };

__device__ __forceinline__ float tanh_full(float x) { return tanhf(x); }
__device__ __forceinline__ double tanh_full(double x) { return tanh(x); }

// sigma(z) = 0.5 * (1 + tanh(0.5 z)), evaluated exactly in that order
// (rnnblock kernels.py:236-237): overflow-free and exactly symmetric.
template <typename T>
__device__ __forceinline__ T sigmoid_ref(T z) {
  return T(0.5) * (T(1) + tanh_full(T(0.5) * z));
}

__device__ __forceinline__ float round_x(float v, int xr) {
  if (xr == XR_BF16) return __bfloat162float(__float2bfloat16_rn(v));
  if (xr == XR_TF32) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
  }
  return v;
}
__device__ __forceinline__ double round_x(double v, int) { return v; }

// 16-byte async global->shared copy; src_bytes < 16 zero-fills the tail.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Vector of KV elements of T occupying 16 bytes (float: 4, double: 2).
template <typename T> struct Vec16;
template <> struct Vec16<float> { static constexpr int N = 4; float v[4]; };
template <> struct Vec16<double> { static constexpr int N = 2; double v[2]; };

template <typename T>
__device__ __forceinline__ Vec16<T> lds16(const T* p) {
  Vec16<T> r;
  *reinterpret_cast<float4*>(r.v) = *reinterpret_cast<const float4*>(p);
  return r;
}

// Weight fetch of KV elements converted to the accumulation type TA.
template <typename TA, typename TW> struct WLoad;
template <> struct WLoad<float, float> {
  static __device__ __forceinline__ void shared(const float* p, float (&w)[4]) {
    float4 v = *reinterpret_cast<const float4*>(p);
    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
  }
  static __device__ __forceinline__ void global(const float* p, float (&w)[4]) {
    float4 v = __ldg(reinterpret_cast<const float4*>(p));
    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
  }
};
template <> struct WLoad<float, __nv_bfloat16> {
  static __device__ __forceinline__ void cvt(uint2 u, float (&w)[4]) {
    w[0] = __uint_as_float(u.x << 16); w[1] = __uint_as_float(u.x & 0xffff0000u);
    w[2] = __uint_as_float(u.y << 16); w[3] = __uint_as_float(u.y & 0xffff0000u);
  }
  static __device__ __forceinline__ void shared(const __nv_bfloat16* p, float (&w)[4]) {
    cvt(*reinterpret_cast<const uint2*>(p), w);
  }
  static __device__ __forceinline__ void global(const __nv_bfloat16* p, float (&w)[4]) {
    cvt(__ldg(reinterpret_cast<const uint2*>(p)), w);
  }
};
template <> struct WLoad<double, double> {
  static __device__ __forceinline__ void shared(const double* p, double (&w)[2]) {
    double2 v = *reinterpret_cast<const double2*>(p);
    w[0] = v.x; w[1] = v.y;
  }
  static __device__ __forceinline__ void global(const double* p, double (&w)[2]) {
    double2 v = __ldg(reinterpret_cast<const double2*>(p));
    w[0] = v.x; w[1] = v.y;
  }
};

}  // namespace rnnb
