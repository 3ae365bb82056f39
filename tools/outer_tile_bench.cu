// Consumer-tile ceiling of the FFMA kernel's shape: an R x C outer-product
// tile per lane on (k even, k odd) FFMA2 pairs, W broadcast from shared
// memory (4 distinct k-vectors per warp, as the kernel's 4 k-lanes), x from
// 32 distinct addresses, one CTA of T threads per SM.  Answers: how many
// consumer warps per SM, and which tile, the loop alone can use.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o outer_tile_bench outer_tile_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long f2(unsigned long long a, unsigned long long b, unsigned long long c) {
  const float2 r = __ffma2_rn(*reinterpret_cast<const float2*>(&a), *reinterpret_cast<const float2*>(&b),
                              *reinterpret_cast<const float2*>(&c));
  return *reinterpret_cast<const unsigned long long*>(&r);
}

template <int R, int C, int T>
__global__ void __launch_bounds__(T, 1) k_tile(float* out, int iters) {
  __shared__ float4 ws[16 * 4 * 24];
  __shared__ float4 xs[33 * 32];
  for (int i = threadIdx.x; i < 16 * 4 * 24; i += blockDim.x) ws[i] = make_float4(1e-3f, 2e-3f, 3e-3f, 4e-3f);
  for (int i = threadIdx.x; i < 33 * 32; i += blockDim.x) xs[i] = make_float4(1.f, 0.5f, 0.25f, 0.125f);
  __syncthreads();
  unsigned long long acc[R][C];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[r][c] = 0ull;
  const int lane = threadIdx.x & 31, kq = lane >> 3, tq = lane & 7;
  for (int it = 0; it < iters; ++it) {
    const int k = it & 15;
    ulonglong2 xv[C];
#pragma unroll
    for (int c = 0; c < C; ++c)
      xv[c] = reinterpret_cast<const ulonglong2*>(xs)[((k * 4 + kq) & 31) * 33 + tq + 8 * c];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const ulonglong2 w = reinterpret_cast<const ulonglong2*>(ws)[(k * 4 + kq) * 24 + r];
#pragma unroll
      for (int c = 0; c < C; ++c) acc[r][c] = f2(w.x, xv[c].x, acc[r][c]);
#pragma unroll
      for (int c = 0; c < C; ++c) acc[r][c] = f2(w.y, xv[c].y, acc[r][c]);
    }
  }
  float t = 0;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) t += __uint_as_float((unsigned)acc[r][c]) + __uint_as_float((unsigned)(acc[r][c] >> 32));
  if (t == 12345.f) out[threadIdx.x] = t;
}

template <int R, int C, int T>
static void run(float* out) {
  const int iters = 40000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_tile<R, C, T><<<148, T>>>(out, iters / 10);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int i = 0; i < 3; ++i) {
    cudaEventRecord(e0);
    k_tile<R, C, T><<<148, T>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double fl = 2.0 * R * C * 4 * (double)iters * T * 148;
  printf("tile %2dx%d  threads %3d (%2d warps): %.2f TFLOP/s\n", R, C, T, T / 32, fl / best / 1e9);
}

int main() {
  float* out;
  cudaMalloc(&out, 4096);
  run<11, 4, 256>(out);
  run<11, 4, 384>(out);
  run<11, 2, 256>(out);
  run<11, 2, 512>(out);
  run<7, 4, 384>(out);
  run<7, 4, 512>(out);
  run<8, 4, 384>(out);
  run<8, 4, 512>(out);
  run<14, 4, 256>(out);
  run<11, 3, 384>(out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
