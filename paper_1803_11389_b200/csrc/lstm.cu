// LSTM partial precompute on B200: the reference's
// lstm_run_precomputed (rnnblock blocked.py:271-305), one layer.
//
//   pre_g[t] = (W_g x_t + b_g) + U_g h_{t-1}      g in {forget, input, output, cand}
//   f, i, o = sigma(pre), cand = tanh(pre);  c = f c + i cand;  h = o tanh(c)
//
// The reference batches the four W x products of a block into GEMMs and
// keeps the four U h products in the step loop ("nothing can move them
// out", blocked.py:274-279).  On the GPU:
//   * lstm_proj_kernel: the input-side products for the whole sequence in
//     one tiled FFMA GEMM (+ bias), Gx [L][4 Hp] with the four gate rows of a
//     unit adjacent (row 4u+g).  Block boundaries only decide where the
//     reference batches this product, never its value per element.
//   * lstm_rec_kernel: ONE persistent cooperative launch for the recurrence.
//     CTA j owns units [jU, jU+U): its 4U rows of U stay in shared memory for
//     the whole sequence (read from L2 when they do not fit), h_{t-1} is
//     gathered from a double-buffered global vector that every CTA publishes
//     its slice of, and per-CTA release flags (one line each, polled by one
//     warp per CTA) are the only grid-wide synchronisation per step.
// Deterministic: fixed summation orders, no atomics on data.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rnnb.h"
#include "abi_guard.h"
#include "common.cuh"

namespace rnnb {

rnnb_status set_error(rnnb_status s, const std::string& msg);  // rnnb_api.cu

constexpr int kProjBM = 64;   // time rows per CTA tile
constexpr int kProjBN = 128;  // gate rows per CTA tile
constexpr int kProjThreads = 256;

// Gx[t][n] = sum_k X[t][k] W[n][k] + b[n], ascending k (tiles of kProjBK).
// X [L][ldx] (K = D valid columns), W [N][Kp] (zero-padded to Kp), Gx [L][N].
template <typename T>
__global__ void __launch_bounds__(kProjThreads) lstm_proj_kernel(const T* __restrict__ X, int64_t ldx,
                                                                 const T* __restrict__ W, const T* __restrict__ b,
                                                                 T* __restrict__ Gx, int64_t L, int N, int D,
                                                                 int Kp) {
  constexpr int kProjBK = sizeof(T) == 8 ? 8 : 16;  // static smem stays under 48 KB for f64
  __shared__ T As[2][kProjBK][kProjBM + 4];
  __shared__ T Bs[2][kProjBK][kProjBN + 4];
  const int tid = threadIdx.x;
  const int ty = tid / 16, tx = tid % 16;  // thread tile: 4 time rows x 8 gate rows
  const int64_t m0 = (int64_t)blockIdx.y * kProjBM;
  const int n0 = blockIdx.x * kProjBN;
  T acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = T(0);
  // staging: A tile 64 x BK (BK/4 values per thread), B tile 128 x BK (BK/2 per thread)
  constexpr int AE = kProjBK / 4, BE = kProjBK / 2;
  const int ar = tid / 4, ak = (tid % 4) * AE;
  const int br = tid / 2, bk = (tid % 2) * BE;
  T ra[AE], rb[BE];
  auto load = [&](int k0) {
#pragma unroll
    for (int e = 0; e < AE; ++e) {
      const int64_t m = m0 + ar;
      const int k = k0 + ak + e;
      ra[e] = (m < L && k < D) ? X[m * ldx + k] : T(0);
    }
#pragma unroll
    for (int e = 0; e < BE; ++e) {
      const int n = n0 + br;
      const int k = k0 + bk + e;
      rb[e] = (n < N && k < Kp) ? W[(int64_t)n * Kp + k] : T(0);
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int e = 0; e < AE; ++e) As[buf][ak + e][ar] = ra[e];
#pragma unroll
    for (int e = 0; e < BE; ++e) Bs[buf][bk + e][br] = rb[e];
  };
  load(0);
  store(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < Kp; k0 += kProjBK) {
    const bool more = k0 + kProjBK < Kp;
    if (more) load(k0 + kProjBK);
#pragma unroll
    for (int kk = 0; kk < kProjBK; ++kk) {
      T a[4], w[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[buf][kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 8; ++j) w[j] = Bs[buf][kk][tx * 8 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], w[j], acc[i][j]);
    }
    if (more) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= L) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + tx * 8 + j;
      if (n < N) Gx[m * N + n] = acc[i][j] + b[n];  // (W x) + b, blocked.py:291-294
    }
  }
}

struct LstmRecArgs {
  const void* Gx;   // [L][4Hp]
  const void* Ur;   // [4Hp][Kh] recurrent rows 4u+g
  void* hval;       // [2][Kh] published h (double-buffered)
  int* flags;       // [grid][kFlagStride] per-CTA published step counts (zeroed before launch)
  void* Hout;       // [L][ldh]
  int64_t ldh;
  void* c_io;       // [H] in/out (nullptr: zero in, not written)
  void* h_io;       // [H] in/out
  int64_t L;
  int H, Hp, Kh, U;
  int resident;     // 1: the CTA's U rows live in shared memory
  int dbg;          // RNNB_DEBUG bit 5 (32): skip the grid wait (timing only; wrong results)
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr int kRecThreads = 512;  // 16 warps: <= 2 U rows per warp at U = 7

// Publication of h between CTAs: every CTA stores its slice of h_t into a
// double-buffered global vector, then one thread (after __syncthreads and
// __threadfence) release-stores the CTA's step count into its OWN flag, on
// its own 128-byte line.  A reader's warp 0 polls the G flags (lanes in
// parallel, back-off between rounds), then the CTA reads the vector from L2.
// Measured alternatives: one grid counter (G same-address atomics per step
// serialise in L2, ~3 us/step) and value+tag words polled by every thread
// (L2 hot-line contention, 3-7 us/step).  Double-buffered by step parity: a
// CTA can only publish h_t after it gathered h_{t-1}, i.e. after every CTA
// finished reading h_{t-2}.
constexpr int kFlagStride = 32;  // ints: one 128-byte line per CTA flag

template <typename T>
__device__ __forceinline__ T dot_row(const T* __restrict__ ur, const T* __restrict__ hs, int Kh, int lane) {
  if constexpr (sizeof(T) == 4) {
    // lane owns k = 4 lane + 128 j (float4); 4 rows of float4 loads in flight
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int k = 4 * lane;
    for (; k + 384 < Kh; k += 512) {
      float4 u[4], x[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        u[q] = *reinterpret_cast<const float4*>(ur + k + 128 * q);
        x[q] = *reinterpret_cast<const float4*>(hs + k + 128 * q);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc.x = fmaf(u[q].x, x[q].x, acc.x);
        acc.y = fmaf(u[q].y, x[q].y, acc.y);
        acc.z = fmaf(u[q].z, x[q].z, acc.z);
        acc.w = fmaf(u[q].w, x[q].w, acc.w);
      }
    }
    for (; k < Kh; k += 128) {
      const float4 u = *reinterpret_cast<const float4*>(ur + k);
      const float4 x = *reinterpret_cast<const float4*>(hs + k);
      acc.x = fmaf(u.x, x.x, acc.x);
      acc.y = fmaf(u.y, x.y, acc.y);
      acc.z = fmaf(u.z, x.z, acc.z);
      acc.w = fmaf(u.w, x.w, acc.w);
    }
    return (acc.x + acc.y) + (acc.z + acc.w);
  } else {
    T s4[4] = {T(0), T(0), T(0), T(0)};
    int k = lane;
    for (; k + 96 < Kh; k += 128) {
#pragma unroll
      for (int q = 0; q < 4; ++q) s4[q] = fma(ur[k + 32 * q], hs[k + 32 * q], s4[q]);
    }
    for (int q = 0; k < Kh; k += 32, ++q) s4[q] = fma(ur[k], hs[k], s4[q]);
    return (s4[0] + s4[1]) + (s4[2] + s4[3]);
  }
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// RES: the CTA's U rows are in shared memory (a compile-time fact, so the
// GEMV issues LDS rather than generic loads)
template <typename T, bool RES>
__global__ void __launch_bounds__(kRecThreads, 1) lstm_rec_kernel(LstmRecArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kRecThreads / 32;
  const int U = a.U, R = 4 * a.U, Kh = a.Kh;
  const int u0 = blockIdx.x * U;
  T* hs = reinterpret_cast<T*>(smem_raw);  // [Kh] h_{t-1}
  T* pre = hs + Kh;                        // [R] U h products of this step
  T* Us = pre + ((R + 3) / 4) * 4;         // [R][Kh] when resident
  const T* Ug = static_cast<const T*>(a.Ur) + (size_t)u0 * 4 * Kh;
  const T* Urow = RES ? Us : Ug;
  if (RES) {
    for (int i = tid; i < R * Kh; i += kRecThreads) Us[i] = Ug[i];
  }
  T* hv = static_cast<T*>(a.hval);
  const T* Gx = static_cast<const T*>(a.Gx);
  T* Hout = static_cast<T*>(a.Hout);
  const int G = gridDim.x;
  // CUTLASS-style generic barrier halves: bar.sync, then ONE thread's
  // gpu-scope release (cumulative over the CTA's writes ordered by the
  // barrier); readers: ld.acquire.gpu, then bar.sync.  No fence.sc
  // (__threadfence), which measured ~1-2 us per step on the critical path.
  auto signal = [&](int count) {
    __syncthreads();
    if (tid == 0) st_release(&a.flags[(size_t)blockIdx.x * kFlagStride], count);  // release = fence + store
  };
  // publish h_{-1} (this CTA's slice) into buffer 0
  T c = T(0), hcur = T(0);
  const bool own = tid < U && u0 + tid < a.H;
  if (own) {
    if (a.c_io) c = static_cast<const T*>(a.c_io)[u0 + tid];
    if (a.h_io) hcur = static_cast<const T*>(a.h_io)[u0 + tid];
    hv[u0 + tid] = hcur;
  }
  signal(1);
  // input-side pre-activations (independent of h), software-pipelined one
  // step ahead so their L2 latency never sits on the recurrence chain
  T gx[4] = {T(0), T(0), T(0), T(0)};
  T gn[4] = {T(0), T(0), T(0), T(0)};
  auto load_gx = [&](int64_t t, T (&dst)[4]) {
    if (own && t < a.L) {
      const T* gp = Gx + (size_t)t * 4 * a.Hp + (size_t)(u0 + tid) * 4;
#pragma unroll
      for (int g = 0; g < 4; ++g) dst[g] = gp[g];
    }
  };
  load_gx(0, gn);
  for (int64_t t = 0; t < a.L; ++t) {
#pragma unroll
    for (int g = 0; g < 4; ++g) gx[g] = gn[g];
    load_gx(t + 1, gn);
    // warp 0 waits for every CTA's h_{t-1} (relaxed polls, one acquire
    // fence after), then the CTA gathers it from L2
    if (warp == 0 && !(a.dbg & 32)) {
      const int want = (int)(t + 1);
      for (int j = lane; j < G; j += 32) {
        while (ld_relaxed(&a.flags[(size_t)j * kFlagStride]) < want) {
        }
      }
      __syncwarp();
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
    const T* hsrc = hv + (size_t)(t & 1) * Kh;
    for (int k = tid; k < Kh; k += kRecThreads) hs[k] = k < a.H ? __ldcg(hsrc + k) : T(0);
    __syncthreads();
    // U h for the CTA's 4U rows: warp per row (fixed per-lane order, then a
    // fixed butterfly across lanes)
    for (int r = warp; r < R; r += NW) {
      T s = dot_row<T>(Urow + (size_t)r * Kh, hs, Kh, lane);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) pre[r] = s;
    }
    __syncthreads();
    if (own) {
      const int r = tid * 4;
      const T f = sigmoid_ref<T>(gx[0] + pre[r + 0]);
      const T i = sigmoid_ref<T>(gx[1] + pre[r + 1]);
      const T o = sigmoid_ref<T>(gx[2] + pre[r + 2]);
      const T cand = tanh_full(gx[3] + pre[r + 3]);
      c = f * c + i * cand;
      hcur = o * tanh_full(c);
      hv[(size_t)((t + 1) & 1) * Kh + u0 + tid] = hcur;
      Hout[t * a.ldh + u0 + tid] = hcur;
    }
    signal((int)(t + 2));
  }
  if (own) {
    if (a.c_io) static_cast<T*>(a.c_io)[u0 + tid] = c;
    if (a.h_io) static_cast<T*>(a.h_io)[u0 + tid] = hcur;
  }
}

// Small layers (fp32, the whole of U fits in one 16-CTA cluster's shared
// memory -- d_h up to ~470): the recurrence runs inside ONE thread-block
// cluster.  Every CTA keeps h_{t-1} in a double-buffered shared vector that
// the owners of each unit write directly (st.async into every CTA of the
// cluster, completing bytes on that CTA's mbarrier for the buffer), so a
// CTA's wait on its own mbarrier replaces the global flags, the L2 gather
// and any fence: no global round trip and no memory barrier on the
// recurrence chain.  Unit ownership differs from the
// grid kernel (ceil(H/CS) units per CTA), the row layout of U and Gx does not.
constexpr int kClusterCTAs = 16;  // non-portable cluster size (B200 allows 16)
#ifndef RNNB_LSTM_RB
#define RNNB_LSTM_RB 6
#endif
constexpr int kRB = RNNB_LSTM_RB;  // rows per warp in flight in the cluster GEMV

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// h value into CTA `rank`'s vector, completing bytes on that CTA's mbarrier
// for the buffer (st.async: no fence, the receiver's mbarrier wait orders it)
__device__ __forceinline__ void st_async_f32(const float* local, const uint64_t* mbar, uint32_t rank, float v) {
  const uint32_t la = (uint32_t)__cvta_generic_to_shared(local), lb = (uint32_t)__cvta_generic_to_shared(mbar);
  uint32_t ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(la), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rb) : "r"(lb), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];\n" ::"r"(ra),
               "r"(__float_as_uint(v)), "r"(rb)
               : "memory");
}
__device__ __forceinline__ void cl_mbar_wait(const uint64_t* mbar, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "LW_%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra LW_%=;\n\t}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

__global__ void __launch_bounds__(kRecThreads, 1) lstm_cluster_kernel(LstmRecArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t hbar[2];  // one mbarrier per h buffer
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kRecThreads / 32;
  uint32_t rank, csize;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(csize));
  const int Uc = a.U, Kh = a.Kh;
  const int u0 = (int)rank * Uc;
  const int nu = a.H - u0 < Uc ? (a.H - u0 > 0 ? a.H - u0 : 0) : Uc;  // units this CTA owns
  const int R = 4 * nu;
  float* hs = reinterpret_cast<float*>(smem_raw);  // [2][Kh]: h_{t-1} by step parity
  float* pre = hs + 2 * Kh;                        // [4 Uc]
  float* Us = pre + ((4 * Uc + 3) / 4) * 4;        // [4 Uc][Kh]
  const float* Ug = static_cast<const float*>(a.Ur) + (size_t)u0 * 4 * Kh;
  for (int i = tid; i < R * Kh; i += kRecThreads) Us[i] = Ug[i];
  for (int i = tid; i < 2 * Kh; i += kRecThreads) hs[i] = 0.f;  // padding columns stay 0
  if (tid == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(&hbar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  const float* Gx = static_cast<const float*>(a.Gx);
  float* Hout = static_cast<float*>(a.Hout);
  const bool own = tid < nu;
  const uint32_t hbytes = 4u * (uint32_t)a.H;  // every unit's h once per buffer fill
  float c = 0.f, hcur = 0.f;
  if (own) {
    if (a.c_io) c = static_cast<const float*>(a.c_io)[u0 + tid];
    if (a.h_io) hcur = static_cast<const float*>(a.h_io)[u0 + tid];
  }
  cluster_sync_all();  // barriers initialised and vectors zeroed in every CTA
  if (own)
    for (uint32_t q = 0; q < csize; ++q) st_async_f32(&hs[u0 + tid], &hbar[0], q, hcur);
  float gx[4] = {0.f, 0.f, 0.f, 0.f}, gn[4] = {0.f, 0.f, 0.f, 0.f};
  auto load_gx = [&](int64_t t, float (&dst)[4]) {
    if (own && t < a.L) {
      const float* gp = Gx + (size_t)t * 4 * a.Hp + (size_t)(u0 + tid) * 4;
#pragma unroll
      for (int g = 0; g < 4; ++g) dst[g] = gp[g];
    }
  };
  load_gx(0, gn);
  // Buffer p = t & 1 holds h_{t-1}; its (t >> 1)-th fill.  A CTA sends h_t
  // into buffer (t+1) & 1 only after it received h_{t-1} from every CTA,
  // i.e. after every CTA finished reading h_{t-2} from that buffer: the data
  // flow alone orders the reuse, no cluster barrier per step.
  for (int64_t t = 0; t < a.L; ++t) {
    const int p = (int)(t & 1);
    if (tid == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&hbar[p])),
                   "r"(hbytes)
                   : "memory");
#pragma unroll
    for (int g = 0; g < 4; ++g) gx[g] = gn[g];
    load_gx(t + 1, gn);
    cl_mbar_wait(&hbar[p], (uint32_t)((t >> 1) & 1));
    const float* hsrc = hs + (size_t)p * Kh;
    // rows warp, warp + NW, ... kRB at a time (independent chains share
    // each h load); per row the same per-lane ascending-k float4 order and
    // butterfly as dot_row, so the products equal the grid kernel's bitwise
    for (int r0 = warp; r0 < R; r0 += kRB * NW) {
      float4 acc[kRB];
#pragma unroll
      for (int q = 0; q < kRB; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int k = 4 * lane; k < Kh; k += 128) {
        const float4 x = *reinterpret_cast<const float4*>(hsrc + k);
#pragma unroll
        for (int q = 0; q < kRB; ++q) {
          const int r = r0 + q * NW;
          if (r < R) {
            const float4 u = *reinterpret_cast<const float4*>(Us + (size_t)r * Kh + k);
            acc[q].x = fmaf(u.x, x.x, acc[q].x);
            acc[q].y = fmaf(u.y, x.y, acc[q].y);
            acc[q].z = fmaf(u.z, x.z, acc[q].z);
            acc[q].w = fmaf(u.w, x.w, acc[q].w);
          }
        }
      }
      float v[kRB];
#pragma unroll
      for (int q = 0; q < kRB; ++q) v[q] = (acc[q].x + acc[q].y) + (acc[q].z + acc[q].w);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < kRB; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
      if (lane == 0)
#pragma unroll
        for (int q = 0; q < kRB; ++q)
          if (r0 + q * NW < R) pre[r0 + q * NW] = v[q];
    }
    __syncthreads();
    if (own) {
      const int r = tid * 4;
      const float f = sigmoid_ref<float>(gx[0] + pre[r + 0]);
      const float i = sigmoid_ref<float>(gx[1] + pre[r + 1]);
      const float o = sigmoid_ref<float>(gx[2] + pre[r + 2]);
      const float cand = tanh_full(gx[3] + pre[r + 3]);
      c = f * c + i * cand;
      hcur = o * tanh_full(c);
      if (t + 1 < a.L) {  // the last h is nobody's input
        float* dst = hs + (size_t)(p ^ 1) * Kh + u0 + tid;
        for (uint32_t q = 0; q < csize; ++q) st_async_f32(dst, &hbar[p ^ 1], q, hcur);
      }
      Hout[t * a.ldh + u0 + tid] = hcur;
    }
    // no second barrier: pre[] is rewritten at step t+1 only after this
    // CTA's own h_t (sent above, after reading pre[]) has arrived
  }
  if (own) {
    if (a.c_io) static_cast<float*>(a.c_io)[u0 + tid] = c;
    if (a.h_io) static_cast<float*>(a.h_io)[u0 + tid] = hcur;
  }
  cluster_sync_all();  // no CTA leaves while a peer may still address its shared memory
}

}  // namespace rnnb

using namespace rnnb;

struct rnnb_lstm {
  int64_t din = 0, dh = 0;
  int mode = RNNB_F32, device = 0, num_sms = 148;
  int U = 1, grid = 1, Hp = 0, Kp = 0, Kh = 0;
  bool weights_set = false;
  void* W = nullptr;   // [4Hp][Kp]
  void* b = nullptr;   // [4Hp]
  void* Ur = nullptr;  // [4Hp][Kh]
  void* Gx = nullptr;
  size_t gx_bytes = 0;
  void* hval = nullptr;  // [2][Kh]
  int* flags = nullptr;  // [grid]
  void* hostX = nullptr;
  void* hostH = nullptr;
  size_t hx_bytes = 0, hh_bytes = 0;
  int64_t last_launches = 0;
  bool last_resident = false;
  int last_cluster = 0;  // CTAs of the cluster kernel in the last forward (0: grid kernel)
};

namespace {

size_t es_of(int mode) { return mode == RNNB_F64 ? 8 : 4; }

#define LSTM_CUDA_TRY(expr)                                                                   \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess) return set_error(RNNB_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

size_t rec_smem(const rnnb_lstm* h, bool resident) {
  const size_t es = es_of(h->mode);
  const int R = 4 * h->U;
  return es * ((size_t)h->Kh + (size_t)((R + 3) / 4) * 4 + (resident ? (size_t)R * h->Kh : 0));
}

template <typename T>
rnnb_status lstm_forward_t(rnnb_lstm* h, const T* X, int64_t ldx, int64_t L, T* H, int64_t ldh, T* c_io, T* h_io,
                           cudaStream_t s) {
  const int N = 4 * h->Hp;
  const size_t gxb = (size_t)L * N * sizeof(T);
  if (h->gx_bytes < gxb) {
    if (h->Gx) cudaFree(h->Gx);
    h->Gx = nullptr;
    h->gx_bytes = 0;
    LSTM_CUDA_TRY(cudaMalloc(&h->Gx, gxb));
    h->gx_bytes = gxb;
  }
  dim3 pg((N + kProjBN - 1) / kProjBN, (unsigned)((L + kProjBM - 1) / kProjBM));
  lstm_proj_kernel<T><<<pg, kProjThreads, 0, s>>>(X, ldx, static_cast<const T*>(h->W), static_cast<const T*>(h->b),
                                                  static_cast<T*>(h->Gx), L, N, (int)h->din, h->Kp);
  LSTM_CUDA_TRY(cudaGetLastError());
  LSTM_CUDA_TRY(cudaMemsetAsync(h->flags, 0, sizeof(int) * kFlagStride * h->grid, s));
  LstmRecArgs a{};
  a.Gx = h->Gx;
  a.Ur = h->Ur;
  a.hval = h->hval;
  a.flags = h->flags;
  a.Hout = H;
  a.ldh = ldh;
  a.c_io = c_io;
  a.h_io = h_io;
  a.L = L;
  a.H = (int)h->dh;
  a.Hp = h->Hp;
  a.Kh = h->Kh;
  a.U = h->U;
  a.dbg = getenv("RNNB_DEBUG") ? atoi(getenv("RNNB_DEBUG")) : 0;
  // one-cluster recurrence when the whole of U fits in the cluster (fp32)
  const char* env_cl = getenv("RNNB_LSTM_CLUSTER");
  if (sizeof(T) == 4 && !(env_cl && atoi(env_cl) == 0)) {
    const int CS = kClusterCTAs;
    const int Uc = (int)((h->dh + CS - 1) / CS);
    const size_t smem_cl = sizeof(float) * (2 * (size_t)h->Kh + (size_t)((4 * Uc + 3) / 4) * 4 + (size_t)4 * Uc * h->Kh);
    if (smem_cl <= 227 * 1024) {
      auto kc = lstm_cluster_kernel;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(CS);
      cfg.blockDim = dim3(kRecThreads);
      cfg.dynamicSmemBytes = smem_cl;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CS;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nclusters = 0;
      if (cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cl) == cudaSuccess &&
          cudaFuncSetAttribute(kc, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
          cudaOccupancyMaxActiveClusters(&nclusters, kc, &cfg) == cudaSuccess && nclusters >= 1) {
        a.U = Uc;
        a.resident = 1;
        LSTM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kc, a));
        h->last_launches = 2;
        h->last_resident = true;
        h->last_cluster = CS;
        return RNNB_OK;
      }
      cudaGetLastError();  // the attribute / occupancy probe failed: grid kernel below
    }
  }
  h->last_cluster = 0;
  const size_t smem_res = rec_smem(h, true);
  a.resident = smem_res <= 227 * 1024 ? 1 : 0;
  const size_t smem = rec_smem(h, a.resident);
  auto k = a.resident ? lstm_rec_kernel<T, true> : lstm_rec_kernel<T, false>;
  LSTM_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  void* params[] = {&a};
  LSTM_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k, dim3(h->grid), dim3(kRecThreads), params, smem, s));
  h->last_launches = 2;
  h->last_resident = a.resident != 0;
  return RNNB_OK;
}

}  // namespace

extern "C" {

rnnb_status rnnb_lstm_create(rnnb_lstm_t* out, int64_t d_in, int64_t d_h, int mode, int device) {
  if (!out) return set_error(RNNB_EINVAL, "null output handle");
  *out = nullptr;
  if (d_in < 1 || d_h < 1) return set_error(RNNB_EINVAL, "d_in and d_h must be >= 1");
  if (mode != RNNB_F32 && mode != RNNB_F64)
    return set_error(RNNB_EUNSUPPORTED, "LSTM supports the reference precisions f32 and f64");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return set_error(RNNB_ECUDA, "no CUDA device");
  if (device < 0 || device >= ndev) return set_error(RNNB_EINVAL, "device index out of range");
  DeviceGuard g(device);
  rnnb_lstm* h = new rnnb_lstm();
  h->din = d_in;
  h->dh = d_h;
  h->mode = mode;
  h->device = device;
  int coop = 0;
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
  if (!coop) {
    delete h;
    return set_error(RNNB_EUNSUPPORTED, "device does not support cooperative launch");
  }
  h->U = (int)((d_h + h->num_sms - 1) / h->num_sms);
  h->grid = (int)((d_h + h->U - 1) / h->U);
  h->Hp = h->grid * h->U;
  h->Kp = (int)((d_in + 3) / 4 * 4);
  h->Kh = (int)((d_h + 3) / 4 * 4);
  const size_t es = es_of(mode);
  cudaError_t e = cudaMalloc(&h->W, es * 4 * h->Hp * h->Kp);
  if (e == cudaSuccess) e = cudaMalloc(&h->b, es * 4 * h->Hp);
  if (e == cudaSuccess) e = cudaMalloc(&h->Ur, es * 4 * h->Hp * h->Kh);
  if (e == cudaSuccess) e = cudaMalloc(&h->hval, 8 * 2 * (size_t)h->Kh);
  if (e == cudaSuccess) e = cudaMalloc(&h->flags, sizeof(int) * kFlagStride * h->grid);
  if (e == cudaSuccess) e = cudaMemset(h->W, 0, es * 4 * h->Hp * h->Kp);
  if (e == cudaSuccess) e = cudaMemset(h->b, 0, es * 4 * h->Hp);
  if (e == cudaSuccess) e = cudaMemset(h->Ur, 0, es * 4 * h->Hp * h->Kh);
  if (e == cudaSuccess) e = cudaMemset(h->hval, 0, 8 * 2 * (size_t)h->Kh);
  if (e != cudaSuccess) {
    rnnb_lstm_destroy(h);
    return set_error(RNNB_ECUDA, std::string("LSTM allocation: ") + cudaGetErrorString(e));
  }
  *out = h;
  return RNNB_OK;
}

rnnb_status rnnb_lstm_destroy(rnnb_lstm_t h) {
  if (!h) return RNNB_OK;
  DeviceGuard g(h->device);
  for (void* p : {h->W, h->b, h->Ur, h->Gx, h->hval, static_cast<void*>(h->flags), h->hostX, h->hostH})
    if (p) cudaFree(p);
  delete h;
  return RNNB_OK;
}

rnnb_status rnnb_lstm_set_weights(rnnb_lstm_t h, const void* const* mats, int n_mats, int src_dtype) {
  if (!h) return set_error(RNNB_EINVAL, "null LSTM handle");
  if (n_mats != 12 || !mats) return set_error(RNNB_EINVAL, "LSTM needs 12 arrays (cells.py:46-58)");
  if (src_dtype != RNNB_DT_F32 && src_dtype != RNNB_DT_F64)
    return set_error(RNNB_EINVAL, "src dtype must be f32 or f64");
  for (int m = 0; m < 12; ++m)
    if (!mats[m]) return set_error(RNNB_EINVAL, "null weight array");
  const size_t es = es_of(h->mode);
  const int64_t din = h->din, dh = h->dh;
  auto get = [&](int m, int64_t idx) -> double {
    return src_dtype == RNNB_DT_F64 ? static_cast<const double*>(mats[m])[idx]
                                    : (double)static_cast<const float*>(mats[m])[idx];
  };
  std::vector<unsigned char> W((size_t)4 * h->Hp * h->Kp * es, 0), U((size_t)4 * h->Hp * h->Kh * es, 0),
      B((size_t)4 * h->Hp * es, 0);
  auto put = [&](std::vector<unsigned char>& v, size_t i, double x) {
    if (h->mode == RNNB_F64) std::memcpy(&v[i * 8], &x, 8);
    else {
      const float f = (float)x;
      std::memcpy(&v[i * 4], &f, 4);
    }
  };
  // gate slot g: 0 forget, 1 input, 2 output, 3 cand (mats 0-3 W, 4-7 U, 8-11 b)
  for (int64_t u = 0; u < dh; ++u)
    for (int g = 0; g < 4; ++g) {
      const size_t row = (size_t)u * 4 + g;
      for (int64_t k = 0; k < din; ++k) put(W, row * h->Kp + k, get(g, u * din + k));
      for (int64_t k = 0; k < dh; ++k) put(U, row * h->Kh + k, get(4 + g, u * dh + k));
      put(B, row, get(8 + g, u));
    }
  DeviceGuard gd(h->device);
  LSTM_CUDA_TRY(cudaMemcpy(h->W, W.data(), W.size(), cudaMemcpyHostToDevice));
  LSTM_CUDA_TRY(cudaMemcpy(h->Ur, U.data(), U.size(), cudaMemcpyHostToDevice));
  LSTM_CUDA_TRY(cudaMemcpy(h->b, B.data(), B.size(), cudaMemcpyHostToDevice));
  h->weights_set = true;
  return RNNB_OK;
}

rnnb_status rnnb_lstm_forward(rnnb_lstm_t h, const void* X, int64_t ldx, int64_t L, int64_t block_size, void* H,
                              int64_t ldh, void* c_state, void* h_state, void* stream) {
  if (!h) return set_error(RNNB_EINVAL, "null LSTM handle");
  if (!h->weights_set) return set_error(RNNB_EINVAL, "LSTM weights not set");
  if (L < 1) return set_error(RNNB_EINVAL, "seq_len must be >= 1");
  if (block_size < 1) return set_error(RNNB_EINVAL, "block_size must be >= 1");
  if (!X || !H) return set_error(RNNB_EINVAL, "null X or H");
  if (ldx < h->din) return set_error(RNNB_EINVAL, "ldx smaller than d_in");
  if (ldh < h->dh) return set_error(RNNB_EINVAL, "ldh smaller than d_h");
  DeviceGuard g(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (h->mode == RNNB_F64)
    return lstm_forward_t<double>(h, static_cast<const double*>(X), ldx, L, static_cast<double*>(H), ldh,
                                  static_cast<double*>(c_state), static_cast<double*>(h_state), s);
  return lstm_forward_t<float>(h, static_cast<const float*>(X), ldx, L, static_cast<float*>(H), ldh,
                               static_cast<float*>(c_state), static_cast<float*>(h_state), s);
}

rnnb_status rnnb_lstm_forward_host(rnnb_lstm_t h, const void* X, int64_t L, int64_t block_size, void* H,
                                   void* c_state, void* h_state, void* stream) {
  if (!h) return set_error(RNNB_EINVAL, "null LSTM handle");
  if (L < 1) return set_error(RNNB_EINVAL, "seq_len must be >= 1");
  if (!X || !H) return set_error(RNNB_EINVAL, "null X or H");
  DeviceGuard g(h->device);
  const size_t es = es_of(h->mode);
  const size_t xb = (size_t)L * h->din * es, hb = (size_t)L * h->dh * es, sb = (size_t)2 * h->dh * es;
  if (h->hx_bytes < xb + sb) {
    if (h->hostX) cudaFree(h->hostX);
    h->hostX = nullptr;
    h->hx_bytes = 0;
    LSTM_CUDA_TRY(cudaMalloc(&h->hostX, xb + sb));
    h->hx_bytes = xb + sb;
  }
  if (h->hh_bytes < hb) {
    if (h->hostH) cudaFree(h->hostH);
    h->hostH = nullptr;
    h->hh_bytes = 0;
    LSTM_CUDA_TRY(cudaMalloc(&h->hostH, hb));
    h->hh_bytes = hb;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* dX = static_cast<char*>(h->hostX);
  char* dC = dX + xb;
  char* dHs = dC + h->dh * es;
  LSTM_CUDA_TRY(cudaMemcpyAsync(dX, X, xb, cudaMemcpyHostToDevice, s));
  if (c_state) LSTM_CUDA_TRY(cudaMemcpyAsync(dC, c_state, h->dh * es, cudaMemcpyHostToDevice, s));
  if (h_state) LSTM_CUDA_TRY(cudaMemcpyAsync(dHs, h_state, h->dh * es, cudaMemcpyHostToDevice, s));
  rnnb_status st = rnnb_lstm_forward(h, dX, h->din, L, block_size, h->hostH, h->dh, c_state ? dC : nullptr,
                                     h_state ? dHs : nullptr, stream);
  if (st != RNNB_OK) return st;
  LSTM_CUDA_TRY(cudaMemcpyAsync(H, h->hostH, hb, cudaMemcpyDeviceToHost, s));
  if (c_state) LSTM_CUDA_TRY(cudaMemcpyAsync(c_state, dC, h->dh * es, cudaMemcpyDeviceToHost, s));
  if (h_state) LSTM_CUDA_TRY(cudaMemcpyAsync(h_state, dHs, h->dh * es, cudaMemcpyDeviceToHost, s));
  LSTM_CUDA_TRY(cudaStreamSynchronize(s));
  return RNNB_OK;
}

rnnb_status rnnb_lstm_query(rnnb_lstm_t h, int what, int64_t* value) {
  if (!h || !value) return set_error(RNNB_EINVAL, "null argument");
  const size_t es = es_of(h->mode);
  switch (what) {
    case 0: *value = (int64_t)(es * 4 * h->Hp * ((size_t)h->Kp + h->Kh + 1)); return RNNB_OK;
    case 1: *value = h->last_launches; return RNNB_OK;
    case 2: *value = h->U; return RNNB_OK;
    case 3: *value = h->last_resident ? 1 : 0; return RNNB_OK;
    case 4: *value = h->grid; return RNNB_OK;
    case 5: *value = h->last_cluster; return RNNB_OK;
    default: return set_error(RNNB_EINVAL, "unknown query");
  }
}

}  // extern "C"
