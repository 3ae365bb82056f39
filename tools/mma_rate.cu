// tcgen05.mma issue-rate microbenchmark: cycles per kind::f16 (bf16) MMA of
// shape M x N x 16 with both operands in shared memory (SW128 K-major), for
// the shapes the blocked-layer kernel uses (M = 128, N = T_b in 16..64) and
// the alternatives it could use (N up to 256, M = 64, and the CTA pair
// M = 256 with cta_group::2).  One CTA (or CTA pair) per SM, one thread
// issues R MMAs back to back (4 K-steps inside one 64-wide k-tile, repeated),
// commits once, waits; the kernel time over R gives cycles per MMA per SM.
// Operand contents do not matter for timing (zeros).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_rate tools/mma_rate.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int CG, int MIMIC = 0>
__global__ void __launch_bounds__(128, 1) k_mma(int M, int N, int R, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  // A: 128 rows x 128 B (16 KB) (MIMIC: three such tiles), B: up to 256 rows x 128 B (32 KB)
  unsigned char* A = sm;
  unsigned char* B = sm + (MIMIC ? 3 * 16384 : 16384);
  __shared__ __align__(8) uint64_t bar, bar2;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < ((MIMIC ? 3 : 1) * 16384 + 32768) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  const uint32_t idesc = idesc_bf16(M, N);
  long long t0 = 0, t1 = 0;
  if ((MIMIC & 32) ? (warp == 0) : (threadIdx.x == 0 && rank == 0)) {
    const uint64_t ad = sw128_desc(su32(A)), bd = sw128_desc(su32(B));
    t0 = clock64();
    for (int r = 0; r < R; ++r) {
      const uint64_t koff = (uint64_t)((r & 3) * 2);  // 32 B = 16 bf16 along K, in 16-byte units
      if (MIMIC & 32) {  // one asm block per k-tile: 12 MMAs, descriptors advanced inside PTX
        if ((r % 12) == 0) {
          asm volatile(
              "{\n\t.reg .pred p, e;\n\t.reg .b64 a, b;\n\t.reg .b32 d;\n\t"
              "elect.sync _|e, 0xffffffff;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              // gate 0
              "mov.b64 a, %1;\n\tmov.b64 b, %2;\n\tmov.b32 d, %0;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [d], a, b, %3, p;\n\t"
              "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [d], a, b, %3, 1;\n\t"
              "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [d], a, b, %3, 1;\n\t"
              "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [d], a, b, %3, 1;\n\t"
              // gate 1
              "add.s64 a, %1, 1024;\n\tmov.b64 b, %2;\n\tadd.s32 d, %0, %5;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [d], a, b, %3, p;\n\t"
              "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [d], a, b, %3, 1;\n\t"
              "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [d], a, b, %3, 1;\n\t"
              "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [d], a, b, %3, 1;\n\t"
              // gate 2
              "add.s64 a, %1, 2048;\n\tmov.b64 b, %2;\n\tadd.s32 d, d, %5;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [d], a, b, %3, p;\n\t"
              "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [d], a, b, %3, 1;\n\t"
              "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [d], a, b, %3, 1;\n\t"
              "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [d], a, b, %3, 1;\n\t"
              "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%6];\n\t}\n" ::"r"(tmem),
              "l"(ad), "l"(bd), "r"(idesc), "r"(r), "r"(N), "r"(su32(&bar2))
              : "memory");
        }
      } else if (MIMIC) {  // the layer kernel's pattern: gate g = (r / 4) % 3 -> own A tile (bit 1),
                    // own accumulator (bit 2), commit every 12 MMAs (bit 4)
        const int g = (r >> 2) % 3;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + ((MIMIC & 2) ? g * N : 0)),
            "l"(ad + (uint64_t)(((MIMIC & 1) ? g : 0) * 16384 >> 4) + koff), "l"(bd + koff), "r"(idesc), "r"(r));
        const int every = (MIMIC & 8) ? 24 : (MIMIC & 16) ? 48 : 12;
        if ((MIMIC & 4) && r % every == every - 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           su32(&bar2))
                       : "memory");
      } else if (MIMIC & 128) {  // kind::tf32 (K = 8 per MMA: 128 rows x 32 B of A, same bytes as bf16)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(ad + koff), "l"(bd + koff), "r"((idesc & ~((7u << 7) | (7u << 10))) | (2u << 7) | (2u << 10)),
            "r"(r));
      } else if (CG == 1)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(ad + koff), "l"(bd + koff), "r"(idesc), "r"(r));
      else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(ad + koff), "l"(bd + koff), "r"(idesc), "r"(r));
    }
    if (CG == 1 && (MIMIC & 32))
      asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                   "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bar))
                   : "memory");
    else if (CG == 1)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                   : "memory");
    else
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              su32(&bar)),
          "h"((uint16_t)3)
          : "memory");
  }
  if (threadIdx.x == 0 && (CG == 2 || rank == 0)) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}\n" ::"r"(su32(&bar))
        : "memory");
    t1 = clock64();
    if (rank == 0) cyc[blockIdx.x / CG] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  if (warp == 0) {
    if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main(int argc, char** argv) {
  const int R = argc > 1 ? atoi(argv[1]) : 8192;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long* dcyc;
  cudaMalloc(&dcyc, nsm * sizeof(long long));
  const size_t smem = 3 * 16384 + 32768 + 1024;
  cudaFuncSetAttribute(k_mma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_mma<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_mma<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_mma<1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_mma<1, 7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_mma<1, 15>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_mma<1, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_mma<1, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_mma<1, 23>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_mma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  struct Shape { int cg, M, N; };
  // cg 3..6 = cta_group::1 in (parts of) the layer kernel's pattern: 3 = all
  // (3 gates: own A tile and accumulator each, commit every 12 MMAs), 4 = A
  // tile switch only, 5 = accumulator switch only, 6 = commits only
  // 7 / 8 = the full pattern with a commit every 24 / 48 MMAs
  // 9 = the full pattern issued as one asm block of 12 MMAs + commit per k-tile
  // 10 = kind::tf32 (flops counted at the bf16 K = 16 per MMA: halve for tf32)
  const Shape shapes[] = {{9, 128, 64}, {9, 128, 32}, {9, 128, 16}, {10, 128, 16}, {10, 128, 32}, {10, 128, 64},
                          {10, 128, 128}, {3, 128, 64}, {4, 128, 64}, {5, 128, 64}, {6, 128, 64}, {7, 128, 64}, {8, 128, 64},
                          {7, 128, 32}, {8, 128, 32}, {1, 128, 16}, {1, 128, 32}, {1, 128, 64}, {1, 128, 128}, {1, 128, 256}, {1, 64, 64},
                          {1, 64, 128}, {1, 64, 256}, {2, 256, 32}, {2, 256, 64}, {2, 256, 128}, {2, 256, 256}};
  printf("{\"R\": %d, \"sms\": %d, \"rows\": [\n", R, nsm);
  bool first = true;
  for (const Shape& s : shapes) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(nsm / 2 * 2);
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = s.cg == 2 ? 2 : 1;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaEventRecord(e0);
      cudaError_t e = s.cg == 1   ? cudaLaunchKernelEx(&cfg, k_mma<1>, s.M, s.N, R, dcyc)
                      : s.cg == 3 ? cudaLaunchKernelEx(&cfg, k_mma<1, 7>, s.M, s.N, R, dcyc)
                      : s.cg == 4 ? cudaLaunchKernelEx(&cfg, k_mma<1, 1>, s.M, s.N, R, dcyc)
                      : s.cg == 5 ? cudaLaunchKernelEx(&cfg, k_mma<1, 2>, s.M, s.N, R, dcyc)
                      : s.cg == 6 ? cudaLaunchKernelEx(&cfg, k_mma<1, 4>, s.M, s.N, R, dcyc)
                      : s.cg == 9 ? cudaLaunchKernelEx(&cfg, k_mma<1, 32>, s.M, s.N, R, dcyc)
                      : s.cg == 10 ? cudaLaunchKernelEx(&cfg, k_mma<1, 128>, s.M, s.N, R, dcyc)
                      : s.cg == 7 ? cudaLaunchKernelEx(&cfg, k_mma<1, 15>, s.M, s.N, R, dcyc)
                      : s.cg == 8 ? cudaLaunchKernelEx(&cfg, k_mma<1, 23>, s.M, s.N, R, dcyc)
                                  : cudaLaunchKernelEx(&cfg, k_mma<2>, s.M, s.N, R, dcyc);
      cudaEventRecord(e1);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        fprintf(stderr, "shape cg=%d M=%d N=%d: %s\n", s.cg, s.M, s.N, cudaGetErrorString(e));
        return 1;
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    long long cyc[256];
    const int per = s.cg == 2 ? 2 : 1;
    cudaMemcpy(cyc, dcyc, nsm / per * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < nsm / 2 * 2 / per; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
    const double flop = 2.0 * s.M * s.N * 16 * (double)R * (nsm / 2 * 2 / per);
    printf("%s{\"cta_group\": %d, \"M\": %d, \"N\": %d, \"cycles_per_mma\": %.1f, \"tflops\": %.1f, \"kernel_ms\": %.4f}",
           first ? "" : ",\n", s.cg, s.M, s.N, (double)mx / R, flop / (best * 1e-3) / 1e12, best);
    first = false;
  }
  printf("\n]}\n");
  return 0;
}
