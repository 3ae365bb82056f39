// L2 -> shared-memory throughput with the bulk-copy engine (cp.async.bulk,
// the path the tensor-core kernel streams weights on): every CTA (one per
// SM) copies 32 KB pieces of an L2-resident buffer into a 4-deep shared
// memory ring guarded by mbarriers, for many passes.  tools/l2_peak.cu
// measures the same with 16-byte ld.global.cg from registers, which ncu
// shows the TMA path exceeding (lts__t_bytes 15.6 TB/s in the bf16 T_b = 1
// kernel), so this is the roofline denominator for the weight stream.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_tma_peak l2_tma_peak.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kPiece = 32 * 1024;
constexpr int kStages = 6;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32, 1) k_tma(const char* __restrict__ buf, size_t bytes, int reps, int* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + kStages * kPiece);
  const int lane = threadIdx.x;
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const size_t npieces = bytes / kPiece;
  uint32_t acc = 0;
  if (lane == 0) {
    uint64_t it = 0;
    for (int r = 0; r < reps; ++r) {
      // each CTA walks the buffer from its own starting piece
      for (size_t k = 0; k < npieces; ++k, ++it) {
        const int s = (int)(it % kStages);
        if (it >= kStages) {  // wait for this stage's previous copy before reusing it
          const uint32_t ph = (uint32_t)(((it / kStages) - 1) & 1);
          asm volatile(
              "{\n\t.reg .pred p;\n"
              "W_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}\n" ::"r"(
                  su32(&bar[s])),
              "r"(ph)
              : "memory");
          acc += sm[s * kPiece];
        }
        const size_t piece = (k + blockIdx.x * 7) % npieces;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(kPiece)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(sm + s * kPiece)),
            "l"(buf + piece * kPiece), "r"(kPiece), "r"(su32(&bar[s]))
            : "memory");
      }
    }
    for (uint64_t j = (it >= kStages ? it - kStages : 0); j < it; ++j) {  // drain
      const int s = (int)(j % kStages);
      const uint32_t ph = (uint32_t)((j / kStages) & 1);
      asm volatile(
          "{\n\t.reg .pred p;\n"
          "D_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra D_%=;\n\t}\n" ::"r"(
              su32(&bar[s])),
          "r"(ph)
          : "memory");
    }
  }
  if (acc == 0xdeadbeef) out[0] = 1;
}

int main() {
  int* out;
  cudaMalloc(&out, 16);
  const size_t smem = kStages * kPiece + 64;
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  printf("{\n");
  for (size_t mb : {32, 48, 64}) {
    const size_t bytes = mb << 20;
    char* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 8;
    k_tma<<<148, 32, smem>>>(buf, bytes, 1, out);  // warm: bring the buffer into L2
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int t = 0; t < 5; ++t) {
      cudaEventRecord(e0);
      k_tma<<<148, 32, smem>>>(buf, bytes, reps, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    // every CTA copies the whole buffer reps times
    const double gbs = (double)bytes * reps * 148 / (best * 1e-3) / 1e9;
    printf("  \"l2_tma_gbs_%zuMB\": %.1f,\n", mb, gbs);
    cudaFree(buf);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("  \"error\": \"%s\"\n}\n", cudaGetErrorString(e));
  return 0;
}
