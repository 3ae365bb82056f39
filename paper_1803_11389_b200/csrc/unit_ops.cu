// Unit-level dense kernels and activations of the reference's kernels.py
// (rnnblock kernels.py:181-241) on the GPU, for callers that use them
// directly (the blocked path itself runs them fused inside the layer
// kernels).
//
//   strict (kernel "reference" / "tiled"): C[i,j] = sum_p A[i,p] B[p,j] summed
//     in ascending p with separately rounded multiply and add (__fmul_rn /
//     __fadd_rn: no FMA contraction) -- the reference kernel's exact chain
//     (kernels.py:55-75; "tiled" keeps the same chain, kernels.py:79-113),
//     so results are bitwise equal to it.
//   fast: the same ascending loop with fused multiply-add (the reference's
//     fast family may reassociate; it is tolerance-checked, kernels.py:116-178).
// One thread per output element, 32x32 SMEM tiles of A and B per K step.
#include <cuda_runtime.h>

#include <string>

#include "../../include/rnnb.h"
#include "common.cuh"

namespace rnnb {
rnnb_status set_error(rnnb_status s, const std::string& msg);  // rnnb_api.cu
}
using rnnb::set_error;

namespace {

constexpr int kT = 32;  // output tile side / K step

template <typename T> __device__ __forceinline__ T mul_rn(T a, T b);
template <> __device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
template <typename T> __device__ __forceinline__ T add_rn(T a, T b);
template <> __device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

template <typename T, bool STRICT>
__global__ void __launch_bounds__(kT * 8) gemm_kernel(const T* __restrict__ A, int64_t lda, const T* __restrict__ B,
                                                      int64_t ldb, T* __restrict__ C, int64_t ldc, int64_t m,
                                                      int64_t n, int64_t k) {
  // 32 x 8 threads, each 4 rows of the 32 x 32 output tile (rows ty, ty+8, ...)
  __shared__ T As[kT][kT + 1];
  __shared__ T Bs[kT][kT + 1];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t i0 = (int64_t)blockIdx.y * kT, j = (int64_t)blockIdx.x * kT + tx;
  T acc[4] = {T(0), T(0), T(0), T(0)};
  for (int64_t p0 = 0; p0 < k; p0 += kT) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int rr = ty + 8 * r;
      const int64_t ia = i0 + rr, pa = p0 + tx;
      As[rr][tx] = (ia < m && pa < k) ? A[ia * lda + pa] : T(0);
      const int64_t pb = p0 + rr;
      Bs[rr][tx] = (pb < k && j < n) ? B[pb * ldb + j] : T(0);
    }
    __syncthreads();
    const int pe = (k - p0) < kT ? (int)(k - p0) : kT;
    for (int p = 0; p < pe; ++p) {  // ascending p: the reference's chain
      const T b = Bs[p][tx];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const T a = As[ty + 8 * r][p];
        acc[r] = STRICT ? add_rn(acc[r], mul_rn(a, b)) : fma(a, b, acc[r]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t i = i0 + ty + 8 * r;
    if (i < m && j < n) C[i * ldc + j] = acc[r];
  }
}

// sigmoid(x) = 0.5 * (1 + tanh(0.5 x)) in exactly that order (kernels.py:236-237)
template <typename T>
__global__ void act_kernel(int which, const T* __restrict__ x, T* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = which == 0 ? rnnb::sigmoid_ref<T>(x[i]) : rnnb::tanh_full(x[i]);
}

template <typename T>
cudaError_t gemm_t(bool strict, const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                   int64_t m, int64_t n, int64_t k, cudaStream_t s) {
  const dim3 block(kT, 8), grid((unsigned)((n + kT - 1) / kT), (unsigned)((m + kT - 1) / kT));
  if (strict)
    gemm_kernel<T, true><<<grid, block, 0, s>>>(static_cast<const T*>(A), lda, static_cast<const T*>(B), ldb,
                                                 static_cast<T*>(C), ldc, m, n, k);
  else
    gemm_kernel<T, false><<<grid, block, 0, s>>>(static_cast<const T*>(A), lda, static_cast<const T*>(B), ldb,
                                                  static_cast<T*>(C), ldc, m, n, k);
  return cudaGetLastError();
}

// SplitMix64 (kernels.py:253-309): output j (0-based) of the stream seeded
// with `seed` is mix(seed + (j + 1) * gamma); the weight transform maps its
// top 24 bits u to (u / 2^24) * 0.2 - 0.1 in float64, then casts.  Every
// element is independent, so the stream is generated in parallel.
__device__ __forceinline__ uint64_t sm64_at(uint64_t seed, uint64_t j) {
  uint64_t z = seed + (j + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <typename T>
__global__ void splitmix_uniform_kernel(uint64_t seed, uint64_t offset, int64_t n, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t u = sm64_at(seed, offset + (uint64_t)i) >> 40;
    const double v = __dadd_rn(__dmul_rn(__ddiv_rn((double)u, 16777216.0), 0.2), -0.1);
    out[i] = (T)v;
  }
}

__global__ void splitmix_raw_kernel(uint64_t seed, uint64_t offset, int64_t n, uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = sm64_at(seed, offset + (uint64_t)i);
}

}  // namespace

extern "C" {

rnnb_status rnnb_splitmix_uniform(uint64_t seed, uint64_t offset, int64_t n, void* out, int dtype, void* stream) {
  if (n < 0) return set_error(RNNB_EINVAL, "negative length");
  if (n == 0) return RNNB_OK;
  if (!out) return set_error(RNNB_EINVAL, "null output");
  const int bs = 256;
  const int grid = (int)((n + bs - 1) / bs < 148 * 16 ? (n + bs - 1) / bs : 148 * 16);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == RNNB_DT_F32) splitmix_uniform_kernel<float><<<grid, bs, 0, s>>>(seed, offset, n, static_cast<float*>(out));
  else if (dtype == RNNB_DT_F64) splitmix_uniform_kernel<double><<<grid, bs, 0, s>>>(seed, offset, n, static_cast<double*>(out));
  else if (dtype == RNNB_DT_U64) splitmix_raw_kernel<<<grid, bs, 0, s>>>(seed, offset, n, static_cast<uint64_t*>(out));
  else return set_error(RNNB_EINVAL, "dtype must be f32, f64 or u64 (raw stream)");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(RNNB_ECUDA, std::string("splitmix launch: ") + cudaGetErrorString(e));
  return RNNB_OK;
}


rnnb_status rnnb_gemm(int strict, const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                      int64_t m, int64_t n, int64_t k, int dtype, void* stream) {
  if (!A || !B || !C) return set_error(RNNB_EINVAL, "null matrix");
  if (m < 1 || n < 1 || k < 1) return set_error(RNNB_EINVAL, "matrices must have at least one row and one column");
  if (lda < k || ldb < n || ldc < n) return set_error(RNNB_EINVAL, "leading dimension smaller than the row");
  if (m > (int64_t)65535 * kT) return set_error(RNNB_EUNSUPPORTED, "too many rows");
  cudaError_t e;
  if (dtype == RNNB_DT_F32) e = gemm_t<float>(strict != 0, A, lda, B, ldb, C, ldc, m, n, k, static_cast<cudaStream_t>(stream));
  else if (dtype == RNNB_DT_F64) e = gemm_t<double>(strict != 0, A, lda, B, ldb, C, ldc, m, n, k, static_cast<cudaStream_t>(stream));
  else return set_error(RNNB_EINVAL, "dtype must be f32 or f64");
  if (e != cudaSuccess) return set_error(RNNB_ECUDA, std::string("gemm launch: ") + cudaGetErrorString(e));
  return RNNB_OK;
}

rnnb_status rnnb_activation(int which, const void* x, void* y, int64_t n, int dtype, void* stream) {
  if (which != 0 && which != 1) return set_error(RNNB_EINVAL, "activation must be 0 (sigmoid) or 1 (tanh)");
  if (n < 0) return set_error(RNNB_EINVAL, "negative length");
  if (n == 0) return RNNB_OK;
  if (!x || !y) return set_error(RNNB_EINVAL, "null array");
  const int bs = 256;
  const int grid = (int)((n + bs - 1) / bs < 148 * 8 ? (n + bs - 1) / bs : 148 * 8);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == RNNB_DT_F32) act_kernel<float><<<grid, bs, 0, s>>>(which, static_cast<const float*>(x), static_cast<float*>(y), n);
  else if (dtype == RNNB_DT_F64) act_kernel<double><<<grid, bs, 0, s>>>(which, static_cast<const double*>(x), static_cast<double*>(y), n);
  else return set_error(RNNB_EINVAL, "dtype must be f32 or f64");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(RNNB_ECUDA, std::string("activation launch: ") + cudaGetErrorString(e));
  return RNNB_OK;
}

}  // extern "C"
