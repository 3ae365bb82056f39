// Host <-> device transfer rates that bound rnnb_forward_host (the e2e
// number): copy-engine cudaMemcpyAsync vs kernels reading / writing PINNED
// host memory directly (zero-copy over PCIe), for the cfg2 sizes (8 MB each
// way).  Reads: a few CTAs (the SMs the streaming path leaves free) with
// several 16-byte loads in flight per thread; writes: every SM storing
// 512-byte row pieces, the tensor-core epilogue's pattern.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zc_probe zc_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_read(const float4* __restrict__ src, float4* __restrict__ dst, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    float4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride),
           d = __ldcs(src + i + 3 * stride);
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < n; i += stride) dst[i] = __ldcs(src + i);
}

// each CTA: 128 threads = 128 consecutive floats of a row; rows round-robin over CTAs
__global__ void k_write(float* __restrict__ dst, int rows, int width) {
  for (int r = blockIdx.x; r < rows * (width / 128); r += gridDim.x) {
    const int row = r / (width / 128), piece = r % (width / 128);
    dst[(size_t)row * width + piece * 128 + threadIdx.x] = (float)r;
  }
}

static float time_ms(cudaEvent_t e0, cudaEvent_t e1) {
  float ms;
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  const size_t bytes = 8u << 20;
  float *h_in, *h_out, *d_a, *d_b;
  cudaHostAlloc(&h_in, bytes, cudaHostAllocDefault);
  cudaHostAlloc(&h_out, bytes, cudaHostAllocDefault);
  cudaMalloc(&d_a, bytes);
  cudaMalloc(&d_b, bytes);
  for (size_t i = 0; i < bytes / 4; ++i) h_in[i] = (float)i;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  printf("{\n");
  auto best_of = [&](auto fn) {
    float best = 1e30f;
    for (int t = 0; t < 8; ++t) {
      cudaEventRecord(e0, s1);
      fn();
      cudaEventRecord(e1, s1);
      const float ms = time_ms(e0, e1);
      if (ms < best) best = ms;
    }
    return best;
  };
  float ms = best_of([&] { cudaMemcpyAsync(d_a, h_in, bytes, cudaMemcpyHostToDevice, s1); });
  printf("  \"memcpy_h2d_8MB\": {\"us\": %.1f, \"gbs\": %.1f},\n", ms * 1e3, bytes / ms / 1e6);
  ms = best_of([&] { cudaMemcpyAsync(h_out, d_a, bytes, cudaMemcpyDeviceToHost, s1); });
  printf("  \"memcpy_d2h_8MB\": {\"us\": %.1f, \"gbs\": %.1f},\n", ms * 1e3, bytes / ms / 1e6);
  ms = best_of([&] { cudaMemcpyAsync(d_a, h_in, 256 * 1024, cudaMemcpyHostToDevice, s1); });
  printf("  \"memcpy_h2d_256KB\": {\"us\": %.1f, \"gbs\": %.1f},\n", ms * 1e3, 256 * 1024 / ms / 1e6);
  // both directions at once (two streams), timed on the host
  {
    float best = 1e30f;
    for (int t = 0; t < 8; ++t) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, s1);
      cudaMemcpyAsync(d_a, h_in, bytes, cudaMemcpyHostToDevice, s1);
      cudaMemcpyAsync(h_out, d_b, bytes, cudaMemcpyDeviceToHost, s2);
      cudaEventRecord(e1, s1);
      cudaStreamSynchronize(s2);
      const float m = time_ms(e0, e1);
      if (m < best) best = m;
    }
    printf("  \"memcpy_h2d_with_d2h_concurrent_8MB\": {\"us\": %.1f},\n", best * 1e3);
  }
  for (int ctas : {1, 2, 4, 8, 16}) {
    for (int thr : {256, 1024}) {
      ms = best_of([&] { k_read<<<ctas, thr, 0, s1>>>((const float4*)h_in, (float4*)d_a, bytes / 16); });
      printf("  \"zc_read_%dcta_%dthr\": {\"us\": %.1f, \"gbs\": %.1f},\n", ctas, thr, ms * 1e3, bytes / ms / 1e6);
    }
  }
  for (int ctas : {16, 148, 592}) {
    ms = best_of([&] { k_write<<<ctas, 128, 0, s1>>>(h_out, 2048, 1024); });
    printf("  \"zc_write_%dcta\": {\"us\": %.1f, \"gbs\": %.1f},\n", ctas, ms * 1e3, bytes / ms / 1e6);
  }
  // read and write at once
  {
    float best = 1e30f;
    for (int t = 0; t < 8; ++t) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, s1);
      k_read<<<4, 1024, 0, s1>>>((const float4*)h_in, (float4*)d_a, bytes / 16);
      k_write<<<144, 128, 0, s2>>>(h_out, 2048, 1024);
      cudaEventRecord(e1, s1);
      cudaStreamSynchronize(s2);
      const float m = time_ms(e0, e1);
      if (m < best) best = m;
    }
    printf("  \"zc_read_4cta_with_write_concurrent\": {\"us\": %.1f},\n", best * 1e3);
  }
  // zero-copy read (SMs) with a copy-engine D2H at once, and copy-engine H2D with zero-copy writes
  {
    float best = 1e30f, best2 = 1e30f;
    for (int t = 0; t < 8; ++t) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, s1);
      k_read<<<2, 1024, 0, s1>>>((const float4*)h_in, (float4*)d_a, bytes / 16);
      cudaMemcpyAsync(h_out, d_b, bytes, cudaMemcpyDeviceToHost, s2);
      cudaEventRecord(e1, s1);
      cudaStreamSynchronize(s2);
      float m = time_ms(e0, e1);
      if (m < best) best = m;
      cudaDeviceSynchronize();
      cudaEventRecord(e0, s1);
      cudaMemcpyAsync(d_a, h_in, bytes, cudaMemcpyHostToDevice, s1);
      k_write<<<144, 128, 0, s2>>>(h_out, 2048, 1024);
      cudaEventRecord(e1, s1);
      cudaStreamSynchronize(s2);
      m = time_ms(e0, e1);
      if (m < best2) best2 = m;
    }
    printf("  \"zc_read_2cta_with_memcpy_d2h_concurrent\": {\"us\": %.1f},\n", best * 1e3);
    printf("  \"memcpy_h2d_with_zc_write_concurrent\": {\"us\": %.1f},\n", best2 * 1e3);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("  \"error\": \"%s\"\n}\n", cudaGetErrorString(e));
  return 0;
}
