// Measures the FP32 FFMA throughput a B200 SM actually sustains, to use as
// the CUDA-core roofline denominator (MEASURED_PEAKS.json has no CUDA-core
// figure).  Variants:
//   reg3   : acc[i] = fma(a[i&7], b, acc[i])      3 distinct register sources
//   bcast  : acc[r][c] = fma(w[r], x[c], acc[r][c]) outer product (our kernel's shape)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma_peak ffma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
__global__ void __launch_bounds__(512) k_reg3(float* out, int iters, float s) {
  float acc[N];
  float a[8];
#pragma unroll
  for (int i = 0; i < N; ++i) acc[i] = threadIdx.x * 1e-7f + i;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = s * (i + 1);
  float b = s * 0.5f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = fmaf(a[i & 7], b, acc[i]);
    b = b * 0.999f;
  }
  float t = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) t += acc[i];
  if (t == 12345.f) out[threadIdx.x] = t;
}

// outer product R x C per k-step with w, x loaded from shared memory (broadcast w)
template <int R, int C>
__global__ void __launch_bounds__(512) k_outer(float* out, int iters) {
  __shared__ float4 ws[16 * R];
  __shared__ float4 xs[16 * 32];
  for (int i = threadIdx.x; i < 16 * R; i += blockDim.x) ws[i] = make_float4(1e-3f, 2e-3f, 3e-3f, 4e-3f);
  for (int i = threadIdx.x; i < 16 * 32; i += blockDim.x) xs[i] = make_float4(1.f, 0.5f, 0.25f, 0.125f);
  __syncthreads();
  float acc[R][C];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[r][c] = 0.f;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    const int k = (it & 15);
    float4 xv[C];
#pragma unroll
    for (int c = 0; c < C; ++c) xv[c] = xs[k * 32 + ((lane + c) & 31)];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float4 w = ws[k * R + r];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        acc[r][c] = fmaf(w.x, xv[c].x, acc[r][c]);
        acc[r][c] = fmaf(w.y, xv[c].y, acc[r][c]);
        acc[r][c] = fmaf(w.z, xv[c].z, acc[r][c]);
        acc[r][c] = fmaf(w.w, xv[c].w, acc[r][c]);
      }
    }
  }
  float t = 0;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) t += acc[r][c];
  if (t == 12345.f) out[threadIdx.x] = t;
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// packed FFMA2: acc pairs over (k even, k odd), operands straight from LDS.128
template <int R, int C>
__global__ void __launch_bounds__(512) k_outer2(float* out, int iters) {
  __shared__ float4 ws[16 * R];
  __shared__ float4 xs[16 * 32];
  for (int i = threadIdx.x; i < 16 * R; i += blockDim.x) ws[i] = make_float4(1e-3f, 2e-3f, 3e-3f, 4e-3f);
  for (int i = threadIdx.x; i < 16 * 32; i += blockDim.x) xs[i] = make_float4(1.f, 0.5f, 0.25f, 0.125f);
  __syncthreads();
  unsigned long long acc[R][C];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[r][c] = 0ull;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    const int k = (it & 15);
    ulonglong2 xv[C];
#pragma unroll
    for (int c = 0; c < C; ++c) xv[c] = reinterpret_cast<const ulonglong2*>(xs)[k * 32 + ((lane + c) & 31)];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      ulonglong2 w = reinterpret_cast<const ulonglong2*>(ws)[k * R + r];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        acc[r][c] = ffma2(w.x, xv[c].x, acc[r][c]);
        acc[r][c] = ffma2(w.y, xv[c].y, acc[r][c]);
      }
    }
  }
  float t = 0;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) t += __uint_as_float((unsigned)acc[r][c]) + __uint_as_float((unsigned)(acc[r][c] >> 32));
  if (t == 12345.f) out[threadIdx.x] = t;
}

template <int N>
__global__ void __launch_bounds__(512) k_reg2(float* out, int iters, float s) {
  unsigned long long acc[N], a[8];
#pragma unroll
  for (int i = 0; i < N; ++i) acc[i] = ((unsigned long long)__float_as_uint(threadIdx.x * 1e-7f + i) << 32) | __float_as_uint(1.f * i);
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = ((unsigned long long)__float_as_uint(s * (i + 1)) << 32) | __float_as_uint(s * (i + 2));
  unsigned long long b = ((unsigned long long)__float_as_uint(s * 0.5f) << 32) | __float_as_uint(s * 0.25f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = ffma2(a[i & 7], b, acc[i]);
    b ^= 1ull;
  }
  float t = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) t += __uint_as_float((unsigned)acc[i]) + __uint_as_float((unsigned)(acc[i] >> 32));
  if (t == 12345.f) out[threadIdx.x] = t;
}

template <typename F>
double time_it(F f, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  float* out;
  cudaMalloc(&out, 4096 * sizeof(float));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  for (int threads : {256, 512}) {
    double ms = time_it([&] { k_reg3<32><<<sms, threads>>>(out, iters, 1.0001f); });
    double fl = 2.0 * 32 * iters * threads * sms;
    printf("reg3  threads=%d: %.2f TFLOP/s (%.1f FMA/clk/SM @1965MHz)\n", threads, fl / ms / 1e9,
           fl / 2 / (ms * 1e-3) / sms / 1.965e9);
  }
  for (int threads : {256, 512}) {
    double ms = time_it([&] { k_outer<11, 2><<<sms, threads>>>(out, iters); });
    double fl = 2.0 * 11 * 2 * 4 * iters * threads * sms;
    printf("outer 11x2 threads=%d: %.2f TFLOP/s (%.1f FMA/clk/SM)\n", threads, fl / ms / 1e9,
           fl / 2 / (ms * 1e-3) / sms / 1.965e9);
    ms = time_it([&] { k_outer<21, 2><<<sms, threads>>>(out, iters); });
    fl = 2.0 * 21 * 2 * 4 * iters * threads * sms;
    printf("outer 21x2 threads=%d: %.2f TFLOP/s (%.1f FMA/clk/SM)\n", threads, fl / ms / 1e9,
           fl / 2 / (ms * 1e-3) / sms / 1.965e9);
    ms = time_it([&] { k_outer<8, 4><<<sms, threads>>>(out, iters); });
    fl = 2.0 * 8 * 4 * 4 * iters * threads * sms;
    printf("outer 8x4 threads=%d: %.2f TFLOP/s (%.1f FMA/clk/SM)\n", threads, fl / ms / 1e9,
           fl / 2 / (ms * 1e-3) / sms / 1.965e9);
  }
  for (int threads : {256, 512}) {
    double ms = time_it([&] { k_reg2<32><<<sms, threads>>>(out, iters, 1.0001f); });
    double fl = 2.0 * 2 * 32 * iters * threads * sms;
    printf("reg2 FFMA2 threads=%d: %.2f TFLOP/s (%.1f FMA/clk/SM)\n", threads, fl / ms / 1e9,
           fl / 2 / (ms * 1e-3) / sms / 1.965e9);
  }
  for (int threads : {256, 512}) {
    double ms = time_it([&] { k_outer2<11, 2><<<sms, threads>>>(out, iters); });
    double fl = 2.0 * 11 * 2 * 4 * iters * threads * sms;
    printf("outer2 FFMA2 11x2 threads=%d: %.2f TFLOP/s (%.1f FMA/clk/SM)\n", threads, fl / ms / 1e9,
           fl / 2 / (ms * 1e-3) / sms / 1.965e9);
    ms = time_it([&] { k_outer2<21, 2><<<sms, threads>>>(out, iters); });
    fl = 2.0 * 21 * 2 * 4 * iters * threads * sms;
    printf("outer2 FFMA2 21x2 threads=%d: %.2f TFLOP/s (%.1f FMA/clk/SM)\n", threads, fl / ms / 1e9,
           fl / 2 / (ms * 1e-3) / sms / 1.965e9);
  }
  return 0;
}
