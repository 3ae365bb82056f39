// Consumer inner-loop tiling study for the FFMA layer kernel (B200).
// Per k-vector (4 consecutive K columns) a lane loads R weight vectors
// (LDS.128, shared by the lanes of a k-group) and C x vectors (LDS.128,
// distinct per lane) and issues 2*R*C packed FFMA2 on (k even, k odd)
// accumulator pairs -- the shape of ffma_ws.cuh's consumer.  Reports the
// sustained FMA/clk/SM for several (R, C, warps/SM) points.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o outer_bench outer_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// KVS k-vectors staged; lanes: LT lanes over columns, 32/LT over k
template <int R, int C, int LT, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) k_tile(float* out, int iters) {
  constexpr int KVS = 64;
  constexpr int LK = 32 / LT;
  extern __shared__ __align__(16) float sm[];
  constexpr int RS = R | 1;                              // odd vector pitch: conflict-free over kq
  float4* ws = reinterpret_cast<float4*>(sm);            // [KVS][RS]
  float4* xs = ws + KVS * RS;                            // [C*LT rows][KVS + 1]
  for (int i = threadIdx.x; i < KVS * RS + C * LT * (KVS + 1); i += blockDim.x)
    ws[i] = make_float4(1e-3f * (i & 7), 2e-3f, 3e-3f, 4e-3f);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int tq = lane % LT, kq = lane / LT;
  unsigned long long acc[R][C];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[r][c] = 0ull;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 2
    for (int kb = 0; kb < KVS; kb += LK) {
      const int kv = kb + kq;
      ulonglong2 xv[C];
#pragma unroll
      for (int c = 0; c < C; ++c)
        xv[c] = reinterpret_cast<const ulonglong2*>(xs)[(tq + LT * c) * (KVS + 1) + kv];
      const ulonglong2* wp = reinterpret_cast<const ulonglong2*>(ws) + kv * RS;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const ulonglong2 w = wp[r];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          acc[r][c] = ffma2(w.x, xv[c].x, acc[r][c]);
          acc[r][c] = ffma2(w.y, xv[c].y, acc[r][c]);
        }
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

template <int R, int C, int LT, int THREADS>
void run(const char* name, int sms, float* out) {
  constexpr int KVS = 64;
  const size_t smem = (size_t)(KVS * (R | 1) + C * LT * (KVS + 1)) * 16;
  cudaFuncSetAttribute(k_tile<R, C, LT, THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int iters = 400;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_tile<R, C, LT, THREADS><<<sms, THREADS, smem>>>(out, iters);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) k_tile<R, C, LT, THREADS><<<sms, THREADS, smem>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  const double fma_sm = (double)iters * (KVS / (32 / LT)) * 32 * R * C * 4 * (THREADS / 32);
  printf("{\"tile\": \"%s\", \"R\": %d, \"C\": %d, \"LT\": %d, \"threads\": %d, \"ms\": %.4f, \"fma_per_clk_sm\": %.1f, "
         "\"tflops\": %.2f, \"err\": \"%s\"}\n",
         name, R, C, LT, THREADS, ms, fma_sm / (ms * 1e-3) / 1.965e9, 2 * fma_sm * sms / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
}


// scalar FFMA variant: acc[r][c] += w[r][e] * x[c][e] over the 4 k of a vector
template <int R, int C, int LT, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) k_tile_s(float* out, int iters) {
  constexpr int KVS = 64;
  constexpr int LK = 32 / LT;
  extern __shared__ __align__(16) float sm[];
  constexpr int RS = R | 1;
  float4* ws = reinterpret_cast<float4*>(sm);
  float4* xs = ws + KVS * RS;
  for (int i = threadIdx.x; i < KVS * RS + C * LT * (KVS + 1); i += blockDim.x)
    ws[i] = make_float4(1e-3f * (i & 7), 2e-3f, 3e-3f, 4e-3f);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int tq = lane % LT, kq = lane / LT;
  float acc[R][C];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[r][c] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 2
    for (int kb = 0; kb < KVS; kb += LK) {
      const int kv = kb + kq;
      float4 xv[C];
#pragma unroll
      for (int c = 0; c < C; ++c) xv[c] = xs[(tq + LT * c) * (KVS + 1) + kv];
      const float4* wp = ws + kv * RS;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float4 w = wp[r];
#pragma unroll
        for (int c = 0; c < C; ++c) acc[r][c] = fmaf(w.x, xv[c].x, acc[r][c]);
#pragma unroll
        for (int c = 0; c < C; ++c) acc[r][c] = fmaf(w.y, xv[c].y, acc[r][c]);
#pragma unroll
        for (int c = 0; c < C; ++c) acc[r][c] = fmaf(w.z, xv[c].z, acc[r][c]);
#pragma unroll
        for (int c = 0; c < C; ++c) acc[r][c] = fmaf(w.w, xv[c].w, acc[r][c]);
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

template <int R, int C, int LT, int THREADS>
void run_s(const char* name, int sms, float* out) {
  constexpr int KVS = 64;
  const size_t smem = (size_t)(KVS * (R | 1) + C * LT * (KVS + 1)) * 16;
  cudaFuncSetAttribute(k_tile_s<R, C, LT, THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int iters = 400;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_tile_s<R, C, LT, THREADS><<<sms, THREADS, smem>>>(out, iters);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) k_tile_s<R, C, LT, THREADS><<<sms, THREADS, smem>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  const double fma_sm = (double)iters * (KVS / (32 / LT)) * 32 * R * C * 4 * (THREADS / 32);
  printf("{\"tile\": \"scalar %s\", \"R\": %d, \"C\": %d, \"LT\": %d, \"threads\": %d, \"ms\": %.4f, \"fma_per_clk_sm\": %.1f, "
         "\"tflops\": %.2f, \"err\": \"%s\"}\n",
         name, R, C, LT, THREADS, ms, fma_sm / (ms * 1e-3) / 1.965e9, 2 * fma_sm * sms / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 4096 * sizeof(float));
  run_s<11, 4, 4, 256>("11x4", sms, out);
  run_s<11, 4, 4, 384>("11x4", sms, out);
  run_s<11, 4, 4, 512>("11x4", sms, out);
  run_s<11, 8, 4, 256>("11x8", sms, out);
  run_s<11, 8, 4, 384>("11x8", sms, out);
  run_s<8, 8, 4, 384>("8x8", sms, out);
  run_s<8, 8, 4, 512>("8x8", sms, out);
  run_s<7, 8, 4, 512>("7x8", sms, out);
  run_s<11, 2, 8, 512>("11x2", sms, out);
  run<11, 2, 8, 512>("11x2 (v2)", sms, out);
  run<11, 2, 8, 384>("11x2", sms, out);
  run<7, 4, 4, 384>("7x4", sms, out);
  run<7, 4, 4, 512>("7x4", sms, out);
  run<7, 4, 8, 384>("7x4 lt8", sms, out);
  run<8, 4, 4, 384>("8x4", sms, out);
  run<6, 4, 4, 512>("6x4", sms, out);
  run<11, 4, 4, 256>("11x4", sms, out);
  run<11, 4, 4, 384>("11x4", sms, out);
  run<7, 8, 4, 256>("7x8", sms, out);
  run<4, 8, 4, 384>("4x8", sms, out);
  run<7, 2, 8, 512>("7x2", sms, out);
  run<3, 8, 4, 512>("3x8", sms, out);
  return 0;
}
