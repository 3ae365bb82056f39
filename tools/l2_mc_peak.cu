// L2 -> shared-memory throughput of the bulk-copy engine with CLUSTER
// MULTICAST: the C CTAs of a cluster each fetch 1/C of every 32 KB piece and
// multicast it into the same ring slot of all C CTAs (the weight-tile sharing
// a pair of CTAs working on the same unit tile would use).  Reported: bytes
// RECEIVED per second summed over SMs, for C = 1 (unicast, = l2_tma_peak.cu),
// 2 and 4, and for C = 1 on half the SMs (is the limit per SM or chip-wide?).
// Ring protocol as in the layer kernel: full[s] (tx bytes) / empty[s] (one
// arrival per CTA of the cluster, so a slot is refilled only when every CTA
// has consumed it).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_mc_peak l2_mc_peak.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kPiece = 32 * 1024;
constexpr int kStages = 6;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_par(uint64_t* bar, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}\n" ::"r"(su32(bar)),
      "r"(ph)
      : "memory");
}

template <int C>
__global__ void __launch_bounds__(64, 1) k_mc(const char* __restrict__ buf, size_t bytes, int reps, int* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kStages * kPiece);
  uint64_t* empty = full + kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t rank = 0;
  if (C > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(C));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (C > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  const size_t npieces = bytes / kPiece;
  const uint64_t total = (uint64_t)reps * npieces;
  const size_t cluster_id = blockIdx.x / C;
  if (warp == 0 && lane == 0) {
    // one thread plays both roles (as tools/l2_tma_peak.cu): before slot s is
    // refilled, the copy that filled it kStages iterations ago is waited for
    // ("consumed") and, with a cluster, every CTA is told so
    for (uint64_t it = 0; it < total + kStages; ++it) {
      const int s = (int)(it % kStages);
      if (it >= kStages) {
        wait_par(&full[s], (uint32_t)(((it / kStages) - 1) & 1));
        if (C > 1) {
          for (int c = 0; c < C; ++c) {
            uint32_t ra;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(su32(&empty[s])), "r"(c));
            asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
          }
        }
      }
      if (it >= total) continue;
      if (C > 1) wait_par(&empty[s], (uint32_t)(((it / kStages) & 1) ^ 1));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(kPiece)
                   : "memory");
      const size_t piece = (it + cluster_id * 7) % npieces;
      const char* src = buf + piece * kPiece + rank * (kPiece / C);
      const uint32_t dst = su32(sm + s * kPiece + rank * (kPiece / C));
      if (C == 1)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                     "l"(src), "r"(kPiece), "r"(su32(&full[s]))
                     : "memory");
      else
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
            "%4;" ::"r"(dst),
            "l"(src), "r"(kPiece / C), "r"(su32(&full[s])), "h"((uint16_t)((1u << C) - 1))
            : "memory");
    }
  }
  __syncthreads();
  if (C > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
}

template <int C>
static void run(const char* tag, int grid, char* buf, size_t bytes, int* out) {
  const size_t smem = kStages * kPiece + 256;
  cudaFuncSetAttribute(k_mc<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_mc<C>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(64);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int maxc = 0;
  cudaOccupancyMaxActiveClusters(&maxc, k_mc<C>, &cfg);
  if (maxc * C < grid) grid = maxc * C, cfg.gridDim = dim3(grid);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 8;
  cudaLaunchKernelEx(&cfg, k_mc<C>, (const char*)buf, bytes, 1, out);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int t = 0; t < 5; ++t) {
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k_mc<C>, (const char*)buf, bytes, reps, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double recv = (double)bytes * reps * grid / (best * 1e-3) / 1e9;
  printf("  \"%s\": {\"cluster\": %d, \"ctas\": %d, \"received_gbs\": %.1f, \"per_sm_gbs\": %.1f, \"l2_read_gbs\": %.1f},\n",
         tag, C, grid, recv, recv / grid, recv / C);
}

int main() {
  int* out;
  cudaMalloc(&out, 16);
  const size_t bytes = (size_t)48 << 20;
  char* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  printf("{\n");
  run<1>("unicast_148", 148, buf, bytes, out);
  run<1>("unicast_74", 74, buf, bytes, out);
  run<1>("unicast_37", 37, buf, bytes, out);
  run<2>("multicast2_148", 148, buf, bytes, out);
  run<4>("multicast4_148", 148, buf, bytes, out);
  run<2>("multicast2_74", 74, buf, bytes, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("  \"error\": \"%s\"\n}\n", cudaGetErrorString(e));
  return 0;
}
