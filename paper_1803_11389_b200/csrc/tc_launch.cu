// Host launch of the tcgen05 layer kernel + the operand-conversion kernel.
#include <cstdlib>

#include "tc_dispatch.cuh"

namespace rnnb {

// X operand rows: row 0 = x_{-1} (carry or zeros), rows 1..L = x_t rounded to
// the MMA operand type (bf16 RNE, or tf32 RNA kept in fp32 containers).
template <int MODE>
__global__ void to_operand_kernel(const float* __restrict__ X, int64_t ldx, const float* __restrict__ xcarry,
                                  void* __restrict__ out, int64_t ldo, int64_t L, int D, int64_t prow,
                                  uint4* __restrict__ fill, size_t fill16) {
  // look-back state of the layer launch that follows: all-ones sentinel (tc_lookback)
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < fill16; i += (size_t)gridDim.x * blockDim.x)
    fill[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
  const int64_t n = (L + 1) * (int64_t)D;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / D;
    const int d = (int)(i - r * D);
    const float v = r == 0 ? (xcarry ? xcarry[d] : 0.f) : X[(r - 1) * ldx + d];
    if (MODE == TC_BF16) {
      reinterpret_cast<__nv_bfloat16*>(out)[r * ldo + d] = __float2bfloat16_rn(v);
    } else if (MODE == TC_TF32) {
      reinterpret_cast<float*>(out)[r * ldo + d] = round_x(v, XR_TF32);
    } else {  // 3xTF32: hi plane rows [0, L], lo plane rows [L+1, 2L+1]
      const float hi = round_x(v, XR_TF32);
      reinterpret_cast<float*>(out)[r * ldo + d] = hi;
      reinterpret_cast<float*>(out)[(r + prow) * ldo + d] = round_x(v - hi, XR_TF32);
    }
  }
}

// Same conversion, 4 columns per thread (16-byte loads, 8/16-byte stores),
// rows on grid.y: no per-element 64-bit division (the scalar kernel above
// ran at ~1.2 TB/s on cfg2).  Needs 16-byte aligned rows (host-checked).
template <int MODE>
__global__ void to_operand_v4_kernel(const float* __restrict__ X, int64_t ldx, const float* __restrict__ xcarry,
                                     void* __restrict__ out, int64_t ldo, int64_t L, int D, int64_t prow,
                                     uint4* __restrict__ fill, size_t fill16) {
  {  // look-back state of the layer launch that follows: all-ones sentinel (tc_lookback)
    const size_t nthr = (size_t)gridDim.x * gridDim.y * blockDim.x;
    for (size_t i = ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x; i < fill16; i += nthr)
      fill[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
  }
  const int nv = D >> 2;
  for (int64_t r = blockIdx.y; r <= L; r += gridDim.y) {
    const float* src = r == 0 ? xcarry : X + (r - 1) * ldx;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
      const int d = v << 2;
      const float4 x = src ? *reinterpret_cast<const float4*>(src + d) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (MODE == TC_BF16) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(x.x, x.y), hi = __floats2bfloat162_rn(x.z, x.w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&lo);
        pk.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out) + r * ldo + d) = pk;
      } else {
        const float4 h4 = make_float4(round_x(x.x, XR_TF32), round_x(x.y, XR_TF32), round_x(x.z, XR_TF32),
                                      round_x(x.w, XR_TF32));
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + r * ldo + d) = h4;
        if (MODE == TC_3XTF32) {
          const float4 l4 = make_float4(round_x(x.x - h4.x, XR_TF32), round_x(x.y - h4.y, XR_TF32),
                                        round_x(x.z - h4.z, XR_TF32), round_x(x.w - h4.w, XR_TF32));
          *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + (r + prow) * ldo + d) = l4;
        }
      }
    }
  }
}

// Operand rows 0..L of X (row r = x_{r-1}, row 0 = xcarry or zeros); the
// 3xTF32 lo plane starts prow rows after the hi plane (prow = L+1 for a whole
// sequence; a row range of a longer operand passes that operand's L+1).
cudaError_t tc_to_operand_rows(int mode, const float* X, int64_t ldx, const float* xcarry, void* out, int64_t ldo,
                               int64_t L, int D, int64_t prow, cudaStream_t s, void* fill, size_t fill_bytes) {
  uint4* f4 = static_cast<uint4*>(fill);
  const size_t f16 = fill ? fill_bytes / 16 : 0;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (D % 4 == 0 && ldx % 4 == 0 && ldo % 8 == 0 && al16(X) && (xcarry == nullptr || al16(xcarry)) && al16(out)) {
    const int nv = D / 4;
    const int bx = (nv + 255) / 256;
    const int64_t rows = L + 1;
    const int by = (int)(rows < 148 * 16 / bx ? rows : (148 * 16 / bx > 0 ? 148 * 16 / bx : 1));
    const dim3 grid(bx, by);
    if (mode == TC_BF16) to_operand_v4_kernel<TC_BF16><<<grid, 256, 0, s>>>(X, ldx, xcarry, out, ldo, L, D, prow, f4, f16);
    else if (mode == TC_TF32) to_operand_v4_kernel<TC_TF32><<<grid, 256, 0, s>>>(X, ldx, xcarry, out, ldo, L, D, prow, f4, f16);
    else to_operand_v4_kernel<TC_3XTF32><<<grid, 256, 0, s>>>(X, ldx, xcarry, out, ldo, L, D, prow, f4, f16);
    return cudaGetLastError();
  }
  const int64_t n = (L + 1) * (int64_t)D;
  const int bs = 256;
  const int grid = (int)((n + bs - 1) / bs < 148 * 16 ? (n + bs - 1) / bs : 148 * 16);
  if (mode == TC_BF16) to_operand_kernel<TC_BF16><<<grid, bs, 0, s>>>(X, ldx, xcarry, out, ldo, L, D, prow, f4, f16);
  else if (mode == TC_TF32) to_operand_kernel<TC_TF32><<<grid, bs, 0, s>>>(X, ldx, xcarry, out, ldo, L, D, prow, f4, f16);
  else to_operand_kernel<TC_3XTF32><<<grid, bs, 0, s>>>(X, ldx, xcarry, out, ldo, L, D, prow, f4, f16);
  return cudaGetLastError();
}

cudaError_t tc_to_operand(int mode, const float* X, int64_t ldx, const float* xcarry, void* out, int64_t ldo,
                          int64_t L, int D, cudaStream_t s, void* fill, size_t fill_bytes) {
  return tc_to_operand_rows(mode, X, ldx, xcarry, out, ldo, L, D, L + 1, s, fill, fill_bytes);
}

// Streaming conversion (rnnb_forward_host): ONE persistent launch converts
// the whole sequence while the copy engine is still landing it.  X rows
// arrive in copy segments (TcSegTab) on two alternating copy streams; a
// stream write-value after each segment's copy tags seg_flag[j] with the
// call's epoch.  Groups of `group` rows go round-robin over the worker
// CTAs (blockIdx >= 1): a worker converts its group as soon as the rows are
// there (16-byte loads, 8 in flight per thread) and release-stores the call's
// epoch into flags[g].  CTA 0 is the PUBLISHER: one warp polls 32 group flags
// at a time and advances *ready = rows converted, the in-order counter the
// layer kernel's TMA producer waits on.  Workers never wait on each other,
// so they need not be co-resident (they fill the SMs the layer launch leaves
// free and whatever register space is left beside its CTAs).
// History: per-segment conversion launches were latency-bound on the two free
// SMs (60-90 us per 512-row segment against a 40 us copy); workers
// publishing the counter themselves in order made every group wait an L2
// round trip on its predecessor (a 128-hop serial chain).
// Rows that do not arrive within kStreamTimeoutNs (a profiler serialising
// the streams) set *fail, release the consumer and end the kernel.
template <int MODE>
__global__ void __launch_bounds__(256, 4)
    to_operand_stream_kernel(const float* __restrict__ X, int64_t ldx, const float* __restrict__ xcarry,
                             void* __restrict__ out, int64_t ldo, int64_t L, int D, int64_t prow,
                             const TcSegTab segs, const int* seg_flag, int* ready, int* fail, int* flags,
                             int* next_group, int epoch, int group) {
  const int nv = D >> 2;
  const int ngroups = (int)((L + group - 1) / group);
  uint64_t t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  auto timed_out = [&]() {
    uint64_t now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    return now - t_start > kStreamTimeoutNs;
  };
  if (blockIdx.x == 0) {
    // ---- publisher ----
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    int base = 0;
    while (base < ngroups) {
      int v = 0;
      if (base + lane < ngroups)
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flags + base + lane) : "memory");
      const unsigned m = __ballot_sync(0xffffffffu, v == epoch);
      const int n = __ffs(~m) - 1;  // leading groups done (m == all ones: __ffs(0) - 1 = -1 -> 32)
      const int adv = n < 0 ? 32 : n;
      if (adv > 0) {
        base += adv;
        if (base > ngroups) base = ngroups;
        const int64_t rows = (int64_t)base * group < L ? (int64_t)base * group : L;
        if (lane == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(ready), "r"((int)rows) : "memory");
      } else {
        int f = 0;
        if (lane == 0) {
          asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(fail) : "memory");
          if (!f && timed_out()) {
            atomicExch(fail, 1);
            f = 1;
          }
        }
        f = __shfl_sync(0xffffffffu, f, 0);
        if (f) {  // a worker or this warp gave up: let the consumer run on (the host redoes the call)
          if (lane == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(ready), "r"(0x7fffffff) : "memory");
          return;
        }
        __nanosleep(100);
      }
    }
    return;
  }
  // ---- workers ----
  __shared__ int s_fail, s_g;
  if (threadIdx.x == 0) s_fail = 0;
  __syncthreads();
  auto convert = [&](int64_t r, int v, const float4 x) {  // operand row r, 4 columns from 4v
    const int d = v << 2;
    if (MODE == TC_BF16) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(x.x, x.y), hi = __floats2bfloat162_rn(x.z, x.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out) + r * ldo + d) = pk;
    } else {
      const float4 h4 = make_float4(round_x(x.x, XR_TF32), round_x(x.y, XR_TF32), round_x(x.z, XR_TF32),
                                    round_x(x.w, XR_TF32));
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + r * ldo + d) = h4;
      if (MODE == TC_3XTF32) {
        const float4 l4 = make_float4(round_x(x.x - h4.x, XR_TF32), round_x(x.y - h4.y, XR_TF32),
                                      round_x(x.z - h4.z, XR_TF32), round_x(x.w - h4.w, XR_TF32));
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + (r + prow) * ldo + d) = l4;
      }
    }
  };
  // groups are claimed from a queue, in order: the workers that are resident
  // convert the next rows to land (a static round-robin would leave holes at
  // the groups of workers still waiting for an SM, and the in-order counter
  // would stall on them)
  while (true) {
    if (threadIdx.x == 0) s_g = atomicAdd(next_group, 1);
    __syncthreads();
    const int g = s_g;
    if (g >= ngroups) return;
    const int64_t r0 = (int64_t)g * group, r1 = (r0 + group) < L ? (r0 + group) : L;  // X rows [r0, r1)
    if (threadIdx.x == 0) {
      // the copy segment holding the group's last row (the segments land in
      // order on two alternating copy streams; a segment's write-value tags
      // its flag with the call's epoch once all of it is in device memory).
      // A group inside one segment needs only that flag; one that spans two
      // needs both.
      int j1 = 0;
      while (j1 < segs.n - 1 && segs.end[j1] < (int)r1) ++j1;
      int j0 = j1;
      while (j0 > 0 && segs.end[j0 - 1] > (int)r0) --j0;
      for (int j = j0; j <= j1 && !s_fail; ++j) while (true) {
        int have = 0;
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(have) : "l"(seg_flag + j) : "memory");
        if (have == epoch) break;
        if (timed_out()) {
          atomicExch(fail, 1);
          s_fail = 1;
          break;
        }
        __nanosleep(200);
      }
    }
    __syncthreads();
    if (s_fail) return;
    if (g == 0)  // operand row 0 = x_{-1}: the carry or zeros
      for (int v = threadIdx.x; v < nv; v += blockDim.x)
        convert(0, v, xcarry ? *reinterpret_cast<const float4*>(xcarry + (v << 2)) : make_float4(0.f, 0.f, 0.f, 0.f));
    const int n = (int)(r1 - r0) * nv;
    const int stride = blockDim.x;
    int i = threadIdx.x;
    for (; i + 7 * stride < n; i += 8 * stride) {  // 8 independent 16-byte loads in flight per thread
      float4 x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = i + k * stride, rr = j / nv, v = j - rr * nv;
        x[k] = __ldcs(reinterpret_cast<const float4*>(X + (r0 + rr) * ldx) + v);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = i + k * stride, rr = j / nv, v = j - rr * nv;
        convert(r0 + rr + 1, v, x[k]);
      }
    }
    for (; i < n; i += stride) {
      const int rr = i / nv, v = i - rr * nv;
      convert(r0 + rr + 1, v, __ldcs(reinterpret_cast<const float4*>(X + (r0 + rr) * ldx) + v));
    }
    __syncthreads();  // the CTA's stores happen-before thread 0's release below
    if (threadIdx.x == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flags + g), "r"(epoch) : "memory");
  }
}

bool tc_to_operand_stream_ok(const float* X, int64_t ldx, const float* xcarry, const void* out, int64_t ldo, int D) {
  // Load the kernels NOW (CUDA loads a kernel's code lazily at its first
  // launch, and that load waits for the device): the conversion is launched
  // while the layer kernel is already spinning on its row counter, so a first
  // launch there stalled until the layer kernel's 2 s time-out.
  static bool loaded = false;
  if (!loaded) {
    cudaFuncAttributes fa;
    (void)cudaFuncGetAttributes(&fa, to_operand_stream_kernel<TC_BF16>);
    (void)cudaFuncGetAttributes(&fa, to_operand_stream_kernel<TC_TF32>);
    (void)cudaFuncGetAttributes(&fa, to_operand_stream_kernel<TC_3XTF32>);
    loaded = true;
  }
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return D % 4 == 0 && ldx % 4 == 0 && ldo % 8 == 0 && al16(X) && (xcarry == nullptr || al16(xcarry)) && al16(out);
}

cudaError_t tc_to_operand_stream(int mode, const float* X, int64_t ldx, const float* xcarry, void* out, int64_t ldo,
                                 int64_t L, int D, const TcSegTab& segs, const int* seg_flag, int* ready, int* fail,
                                 int* flags, int* next_group, int epoch, int group, int workers, cudaStream_t s) {
  const int grid = workers + 1;  // + the publisher (CTA 0)
  if (mode == TC_BF16)
    to_operand_stream_kernel<TC_BF16><<<grid, 256, 0, s>>>(X, ldx, xcarry, out, ldo, L, D, L + 1, segs, seg_flag, ready, fail,
                                                           flags, next_group, epoch, group);
  else if (mode == TC_TF32)
    to_operand_stream_kernel<TC_TF32><<<grid, 256, 0, s>>>(X, ldx, xcarry, out, ldo, L, D, L + 1, segs, seg_flag, ready, fail,
                                                           flags, next_group, epoch, group);
  else
    to_operand_stream_kernel<TC_3XTF32><<<grid, 256, 0, s>>>(X, ldx, xcarry, out, ldo, L, D, L + 1, segs, seg_flag, ready,
                                                             fail, flags, next_group, epoch, group);
  return cudaGetLastError();
}

static bool make_map(CUtensorMap* tm, CUtensorMapDataType dt, int es, const void* base, uint64_t inner,
                     uint64_t outer, uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return false;
  cuuint64_t gdim[2] = {inner, outer};
  cuuint64_t gstride[1] = {ld_elems * (uint64_t)es};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return enc(tm, dt, 2, const_cast<void*>(base), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// grid == 0: only load the kernel and set its attribute (CUDA loads kernel code
// lazily at the first launch, and that load waits for the device -- fatal for
// a first launch made while another kernel spins on this one's progress)
template <int CELL, int MODE, int N, int EG = 1>
static cudaError_t launch_tc(const TcArgs& a, const CUtensorMap& tw, const CUtensorMap& tx, int grid,
                             cudaStream_t s) {
  if constexpr (EG == 1 && MODE != TC_3XTF32) {
    // bf16 / tf32: the two-epilogue-group variant when the host asks for it
    // (grid == 0, the preload, loads both)
    if (grid == 0) {
      cudaError_t e = launch_tc<CELL, MODE, N, 2>(a, tw, tx, 0, s);
      if (e != cudaSuccess) return e;
    } else if (a.egroups == 2) {
      return launch_tc<CELL, MODE, N, 2>(a, tw, tx, grid, s);
    }
  }
  using C = TcCfg<MODE, N, EG>;
  auto k = tc_layer_kernel<CELL, MODE, N, EG>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (grid == 0) return cudaSuccess;
  // programmatic dependent launch: the CTAs set up (barriers, TMEM, tensor-map
  // prefetch) while the preceding kernel -- usually the operand conversion --
  // drains, then wait on griddepcontrol before touching global memory
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, a, tw, tx);
}

cudaError_t tc_layer_preload(int cell, int mode, int T_b);

int tc_max_n(int mode) { return mode == TC_3XTF32 ? 32 : 128; }

int tc_pick_n(int T_b) {
  if (T_b <= 16) return 16;
  if (T_b <= 32) return 32;
  if (T_b <= 64) return 64;
  return 128;
}

template <int CELL, int MODE>
static cudaError_t run_n(int N, const TcArgs& a, const CUtensorMap& tw, const CUtensorMap& tx, int grid,
                         cudaStream_t s) {
  switch (N) {
    case 16: return launch_tc<CELL, MODE, 16>(a, tw, tx, grid, s);
    case 32: return launch_tc<CELL, MODE, 32>(a, tw, tx, grid, s);
    default:
      // 3xTF32 keeps the 3N chunk partials in registers: N <= 32
      if constexpr (MODE == TC_3XTF32) return cudaErrorInvalidValue;
      else if (N == 64) return launch_tc<CELL, MODE, 64>(a, tw, tx, grid, s);
      else return launch_tc<CELL, MODE, 128>(a, tw, tx, grid, s);
  }
}

cudaError_t tc_layer_run(int cell, int mode, TcArgs a, const void* Wtc, int Kp, const void* Xop, int64_t ldop_in,
                         int num_sms, cudaStream_t s, int* grid_out) {
  const int N = tc_pick_n(a.T_b);
  const int es = mode == TC_BF16 ? 2 : 4;
  const int KT = mode == TC_BF16 ? 64 : 32;
  const int planes = mode == TC_3XTF32 ? 2 : 1;
  const CUtensorMapDataType dt = mode == TC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUtensorMap tw, tx;
  if (!make_map(&tw, dt, es, Wtc, (uint64_t)Kp, (uint64_t)3 * planes * a.Hpad, (uint64_t)Kp, KT, 128))
    return cudaErrorInvalidValue;
  // operand X has L+1 rows per plane (row 0 = x_{-1}); the kernel addresses row t+1
  if (!make_map(&tx, dt, es, Xop, (uint64_t)a.D, (uint64_t)planes * (a.L + 1), (uint64_t)ldop_in, KT, N))
    return cudaErrorInvalidValue;
  const int nitems = a.nU * a.nB;
  const int grid = nitems < num_sms ? nitems : num_sms;  // (num_sms: the caller may reserve SMs)
  // no split last wave unless the caller set one up (zero-initialised args)
  if (a.split_start <= 0 || a.split_start > nitems || mode != TC_3XTF32) a.split_start = nitems;
  if (grid_out) *grid_out = grid;
  if (cell == LINEAR) {
    // dense layers: bf16 / tf32 products, or 3xTF32 for fp32 layers large enough to fill the GPU
    if (mode == TC_BF16) return run_n<LINEAR, TC_BF16>(N, a, tw, tx, grid, s);
    if (mode == TC_TF32) return run_n<LINEAR, TC_TF32>(N, a, tw, tx, grid, s);
    return run_n<LINEAR, TC_3XTF32>(N, a, tw, tx, grid, s);  // fp32 dense layers: fp32-accurate split products
  }
  if (cell == SRU) {
    if (mode == TC_BF16) return run_n<SRU, TC_BF16>(N, a, tw, tx, grid, s);
    if (mode == TC_TF32) return run_n<SRU, TC_TF32>(N, a, tw, tx, grid, s);
    return run_n<SRU, TC_3XTF32>(N, a, tw, tx, grid, s);
  }
  if (mode == TC_BF16) return run_n<QRNN, TC_BF16>(N, a, tw, tx, grid, s);
  if (mode == TC_TF32) return run_n<QRNN, TC_TF32>(N, a, tw, tx, grid, s);
  return run_n<QRNN, TC_3XTF32>(N, a, tw, tx, grid, s);
}

cudaError_t tc_layer_preload(int cell, int mode, int T_b) {
  const int N = tc_pick_n(T_b);
  const TcArgs a{};
  const CUtensorMap tm{};
  if (cell == LINEAR) {
    if (mode == TC_BF16) return run_n<LINEAR, TC_BF16>(N, a, tm, tm, 0, nullptr);
    if (mode == TC_TF32) return run_n<LINEAR, TC_TF32>(N, a, tm, tm, 0, nullptr);
    return run_n<LINEAR, TC_3XTF32>(N, a, tm, tm, 0, nullptr);
  }
  if (cell == SRU) {
    if (mode == TC_BF16) return run_n<SRU, TC_BF16>(N, a, tm, tm, 0, nullptr);
    if (mode == TC_TF32) return run_n<SRU, TC_TF32>(N, a, tm, tm, 0, nullptr);
    return run_n<SRU, TC_3XTF32>(N, a, tm, tm, 0, nullptr);
  }
  if (mode == TC_BF16) return run_n<QRNN, TC_BF16>(N, a, tm, tm, 0, nullptr);
  if (mode == TC_TF32) return run_n<QRNN, TC_TF32>(N, a, tm, tm, 0, nullptr);
  return run_n<QRNN, TC_3XTF32>(N, a, tm, tm, 0, nullptr);
}

}  // namespace rnnb
