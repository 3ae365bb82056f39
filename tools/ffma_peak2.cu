// FP32 FMA-pipe peak, second measurement: many independent accumulator
// chains per thread (no dependent instruction between an FMA and its next use
// for >= 16 issues), FFMA and packed FFMA2, 1-2 CTAs of 512 threads per SM,
// long enough (~1 s) for clocks to settle; run beside an nvidia-smi clock
// sampler (tools/ffma_peak2.sh).  Cross-checks tools/ffma_peak.cu's reg3
// figure, the CUDA-core roofline denominator.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma_peak2 ffma_peak2.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
__global__ void __launch_bounds__(512) k_ffma(float* out, int iters, float a, float b) {
  float acc[N];
#pragma unroll
  for (int i = 0; i < N; ++i) acc[i] = threadIdx.x * 1e-7f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = fmaf(acc[i], a, b);
  }
  float t = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) t += acc[i];
  if (t == 12345.f) out[threadIdx.x] = t;
}

template <int N>
__global__ void __launch_bounds__(512) k_ffma2(float* out, int iters, float a, float b) {
  float2 acc[N];
#pragma unroll
  for (int i = 0; i < N; ++i) acc[i] = make_float2(threadIdx.x * 1e-7f + i, i * 0.5f);
  const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = __ffma2_rn(acc[i], a2, b2);
  }
  float t = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) t += acc[i].x + acc[i].y;
  if (t == 12345.f) out[threadIdx.x] = t;
}

template <typename K>
static double run(K k, int ctas_per_sm, int iters, double fma_per_iter_thread) {
  float* out;
  cudaMalloc(&out, 4096);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = 148 * ctas_per_sm;
  k<<<grid, 512>>>(out, iters / 10, 0.999999f, 1e-7f);
  cudaDeviceSynchronize();
  double best = 0;
  for (int t = 0; t < 3; ++t) {
    cudaEventRecord(e0);
    k<<<grid, 512>>>(out, iters, 0.999999f, 1e-7f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tf = 2.0 * fma_per_iter_thread * iters * grid * 512 / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  cudaFree(out);
  return best;
}

int main() {
  const int iters = 200000;
  for (int c : {1, 2}) {
    printf("ffma  N=32 ctas/sm=%d: %.2f TFLOP/s\n", c, run(k_ffma<32>, c, iters, 32));
    printf("ffma2 N=16 ctas/sm=%d: %.2f TFLOP/s\n", c, run(k_ffma2<16>, c, iters, 32));
    printf("ffma2 N=32 ctas/sm=%d: %.2f TFLOP/s\n", c, run(k_ffma2<32>, c, iters / 2, 64));
  }
  return 0;
}
