// Measures the L2 -> SM read throughput a B200 sustains (all SMs reading an
// L2-resident buffer with 16-byte ld.global.cg, which bypasses L1), to use as
// the roofline denominator of the tensor-core modes, whose kernels stream
// every weight tile from L2 once per block (MEASURED_PEAKS.json has HBM and
// tensor peaks only).  A DRAM-sized buffer is read the same way as a check
// against MEASURED_PEAKS.json's copy bandwidth.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_peak l2_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) k_read(const uint4* __restrict__ buf, size_t n, int reps, uint4* out) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    // each rep starts at a rotated offset so consecutive reps do not reuse L1/L2 lines in the same order
    const size_t rot = (size_t)r * 4099 * 32 % n;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
      size_t j = i + rot;
      if (j >= n) j -= n;
      uint4 v;
      asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "l"(buf + j));
      acc.x ^= v.x;
      acc.y ^= v.y;
      acc.z ^= v.z;
      acc.w ^= v.w;
    }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x9e3779b9u) out[threadIdx.x] = acc;
}

static double run(size_t bytes, int reps, int ctas_per_sm) {
  uint4 *buf, *out;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&out, 512 * sizeof(uint4));
  cudaMemset(buf, 1, bytes);
  const size_t n = bytes / sizeof(uint4);
  const int grid = 148 * ctas_per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_read<<<grid, 512>>>(buf, n, 1, out);  // warm: brings the buffer into L2
  cudaDeviceSynchronize();
  double best = 0;
  for (int t = 0; t < 10; ++t) {
    cudaEventRecord(e0);
    k_read<<<grid, 512>>>(buf, n, reps, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gbs = (double)bytes * reps / (ms * 1e-3) / 1e9;
    if (gbs > best) best = gbs;
  }
  cudaFree(buf);
  cudaFree(out);
  return best;
}

int main() {
  const size_t mb = 1 << 20;
  printf("{\n");
  for (size_t sz : {16 * mb, 32 * mb, 48 * mb, 64 * mb})
    for (int c : {2, 4})
      printf("  \"l2_read_gbs_%zuMB_%dcta\": %.1f,\n", sz / mb, c, run(sz, 20, c));
  printf("  \"dram_read_gbs_2048MB\": %.1f\n", run(2048 * mb, 2, 4));
  printf("}\n");
  return 0;
}
