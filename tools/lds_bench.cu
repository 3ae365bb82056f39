// Shared-memory load throughput by lane -> address pattern (B200).
// Decides the consumer layout of the FFMA kernels: how many SMEM wavefronts
// an LDS.128 / LDS.64 / LDS.32 costs when lanes share addresses (broadcast)
// in various groupings.  Reports warp-level loads per clock per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_bench lds_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

// pattern -> 16-byte slot index for a lane
__device__ __forceinline__ int slot_of(int pat, int lane) {
  switch (pat) {
    case 0: return 0;                 // all lanes one address
    case 1: return lane >> 3;         // 4 distinct, one per quarter warp
    case 2: return lane & 3;          // 4 distinct, interleaved (every quarter has all 4)
    case 3: return lane >> 2;         // 8 distinct, 2 per quarter
    case 4: return lane & 7;          // 8 distinct, every quarter has all 8
    case 5: return lane;              // 32 distinct consecutive
    case 6: return lane >> 1;         // 16 distinct
    case 7: return (lane & 3) * 9;    // 4 distinct interleaved, strided (bank-spread)
    case 8: return (lane >> 3) * 9;   // 4 distinct per quarter, strided
    case 9: return (lane & 7) + 8 * 0; // same as 4 (control)
    case 10: return (lane >> 2) * 8 + 0; // 8 distinct, 128B apart -> bank conflicts
    default: return 0;
  }
}

template <int BYTES>
__global__ void __launch_bounds__(512) k_lds(unsigned* out, int iters, int pat) {
  __shared__ __align__(16) unsigned buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i * 2654435761u;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int s = slot_of(pat, lane);
  const unsigned base = (unsigned)__cvta_generic_to_shared(buf) + s * 16;
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const unsigned a = base + ((j * 1024) & 8191);
      if (BYTES == 16) {
        unsigned x, y, z, w;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a));
        acc ^= x ^ y ^ z ^ w;
      } else if (BYTES == 8) {
        unsigned x, y;
        asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(a));
        acc ^= x ^ y;
      } else {
        unsigned x;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(a));
        acc ^= x;
      }
    }
  }
  if (acc == 0x12345678u) out[threadIdx.x] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned* out;
  cudaMalloc(&out, 4096);
  const int iters = 20000, threads = 512;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("{\"sms\": %d, \"clock_khz\": %d, \"rows\": [\n", sms, clk);
  bool first = true;
  for (int bytes : {16, 8, 4}) {
    for (int pat = 0; pat <= 10; ++pat) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (bytes == 16) k_lds<16><<<sms, threads>>>(out, iters, pat);
        else if (bytes == 8) k_lds<8><<<sms, threads>>>(out, iters, pat);
        else k_lds<4><<<sms, threads>>>(out, iters, pat);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        if (rep == 0) continue;
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double warp_lds = (double)iters * 8 * (threads / 32);
        const double cycles = ms * 1e-3 * clk * 1e3;
        printf("%s{\"bytes\": %d, \"pattern\": %d, \"ms\": %.4f, \"clk_per_warp_lds\": %.3f}", first ? "" : ",\n",
               bytes, pat, ms, cycles / warp_lds);
        first = false;
      }
    }
  }
  printf("\n]}\n");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
