// Register-resident fused blocked SRU/QRNN layer kernel (fp32, FFMA2), v3.
//
// Same math and reference mapping as ffma_layer.cuh (rnnblock blocked.py:
// 123-193, 221-268).  For small T_b the shared-memory kernel (ffma_ws.cuh)
// is bound by shared-memory bandwidth: every weight is re-read from SMEM
// for only T_b FMAs.  Here the CTA's weight slice (U units = 3U gate rows,
// K = taps*D <= 1024) lives in REGISTERS for the whole sequence: thread t
// owns k-vector t (4 consecutive K columns) of all 21 rows, packed as 11
// row pairs for fma.rn.f32x2 (row 21 is a zero pad).  Per time step:
//   FMA warps: one 16-byte x load (x_t for the current tap, x_{t-1} for the
//     previous one, prefetched a step ahead), 44 FFMA2, a warp
//     reduce-scatter that leaves row j's warp partial in lane j, one STS;
//   epilogue warp: sums the warp partials in fixed order, bias +
//     activations (lane = gate row), gathers the 3 gates of a unit with
//     shuffles, c = f c + (1-f) z, h = o tanh(c) [+ (1-o) x], stores h.
// Partials are double-buffered; FMA warps and the epilogue warp hand off
// through named barriers (bar.arrive / bar.sync), so step t's epilogue
// overlaps step t+1's products.  Every time step is computed the same way
// whatever T_b is (weights are fetched once per launch for every T_b).
#pragma once
#include "ffma_ws.cuh"

namespace rnnb {


__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void unpack2(unsigned long long v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

// v[0..31] (rows >= 22 are zero) summed over the warp; afterwards lane l
// holds row l's sum in v[0].  Recursive halving: at offset o a lane keeps
// the half of its live slots selected by (lane & o).
template <int NS>
__device__ __forceinline__ void reduce_scatter_step(float (&v)[32], int lane, int live, int o) {
  const bool upper = (lane & o) != 0;
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    const float send = upper ? v[i] : v[i + NS];
    const float keep = upper ? v[i + NS] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
  }
}

template <int CELL, int U>
__global__ void __maxnreg__(U == 7 ? 160 : 96) ffma_reg_kernel(LayerArgs<float, float> a) {
  constexpr int kRegRows = 3 * U;               // gate rows of the CTA's U units
  constexpr int kRegPairs = (kRegRows + 1) / 2;  // row pairs for fma.rn.f32x2
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int nfma = blockDim.x - 32;  // FMA threads; the last warp is the epilogue
  const int nfw = nfma >> 5;
  const int nthr = blockDim.x;
  const int TAPS = CELL == QRNN ? 2 : 1;
  const int Kp = TAPS * a.Dp;
  const int NKV = Kp / 4;
  const int u0 = blockIdx.x * U;
  __shared__ float red[2][16][24];

  if (warp < nfw) {
    // ---------------- FMA warps ----------------
    const bool active = tid < NKV;
    const int kv = active ? tid : 0;
    const int tap = (TAPS == 2 && kv * 4 >= a.Dp) ? 1 : 0;
    const int d = kv * 4 - tap * a.Dp;
    const float* Wg = a.W + (size_t)u0 * 3 * Kp + (size_t)kv * 4;
    unsigned long long w2[kRegPairs][4];
#pragma unroll
    for (int p = 0; p < kRegPairs; ++p) {
      float4 lo = active ? __ldg(reinterpret_cast<const float4*>(Wg + (size_t)(2 * p) * Kp))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 hi = (active && 2 * p + 1 < kRegRows)
                      ? __ldg(reinterpret_cast<const float4*>(Wg + (size_t)(2 * p + 1) * Kp))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
      w2[p][0] = pack2(lo.x, hi.x);
      w2[p][1] = pack2(lo.y, hi.y);
      w2[p][2] = pack2(lo.z, hi.z);
      w2[p][3] = pack2(lo.w, hi.w);
    }
    // x for step t: row t - tap (row -1 = x_carry or zeros); padded columns are 0
    auto load_x = [&](int64_t t) -> float4 {
      const int64_t r = t - tap;
      if (!active || d >= a.D) return make_float4(0.f, 0.f, 0.f, 0.f);
      const float* src = r >= 0 ? a.X + r * a.ldx + d : (a.xcarry ? a.xcarry + d : nullptr);
      if (!src) return make_float4(0.f, 0.f, 0.f, 0.f);
      return __ldg(reinterpret_cast<const float4*>(src));
    };
    float4 xn = load_x(0);
    for (int64_t t = 0; t < a.L; ++t) {
      const float4 x = xn;
      if (t + 1 < a.L) xn = load_x(t + 1);
      const unsigned long long xx0 = pack2(x.x, x.x), xx1 = pack2(x.y, x.y);
      const unsigned long long xx2 = pack2(x.z, x.z), xx3 = pack2(x.w, x.w);
      float v[32];
#pragma unroll
      for (int p = 0; p < kRegPairs; ++p) {
        unsigned long long acc = ffma2(w2[p][0], xx0, 0ull);
        acc = ffma2(w2[p][1], xx1, acc);
        acc = ffma2(w2[p][2], xx2, acc);
        acc = ffma2(w2[p][3], xx3, acc);
        unpack2(acc, v[2 * p], v[2 * p + 1]);
      }
#pragma unroll
      for (int i = 2 * kRegPairs; i < 32; ++i) v[i] = 0.f;
      reduce_scatter_step<16>(v, lane, 32, 16);
      reduce_scatter_step<8>(v, lane, 16, 8);
      reduce_scatter_step<4>(v, lane, 8, 4);
      reduce_scatter_step<2>(v, lane, 4, 2);
      reduce_scatter_step<1>(v, lane, 2, 1);
      // lane l now holds the warp partial of slot l (bit order matches: the
      // upper half was kept when the lane bit is set)
      const int buf = (int)(t & 1);
      if (t >= 2) bar_sync(3 + buf, nthr);  // epilogue released this buffer
      if (lane < 2 * kRegPairs) red[buf][warp][lane] = v[0];
      bar_arrive(1 + buf, nthr);
    }
  } else {
    // ---------------- epilogue warp ----------------
    float c = 0.f;
    const int g = lane % 3, ul = lane / 3;  // gate row lane -> (unit, gate)
    if (lane < U && a.c_in != nullptr && u0 + lane < a.H) c = a.c_in[u0 + lane];
    float bias = 0.f;
    if (CELL == SRU && lane < kRegRows && g > 0 && a.bias) bias = a.bias[(size_t)(u0 + ul) * 2 + g - 1];
    for (int64_t t = 0; t < a.L; ++t) {
      const int buf = (int)(t & 1);
      bar_sync(1 + buf, nthr);
      float s = 0.f;
      if (lane < kRegRows)
        for (int w = 0; w < nfw; ++w) s += red[buf][w][lane];
      bar_arrive(3 + buf, nthr);
      float act;
      if (CELL == SRU) act = g == 0 ? s : sigmoid_ref<float>(s + bias);
      else act = g == 0 ? tanh_full(s) : sigmoid_ref<float>(s);
      const float z = __shfl_sync(0xffffffffu, act, (3 * lane) & 31);
      const float f = __shfl_sync(0xffffffffu, act, (3 * lane + 1) & 31);
      const float o = __shfl_sync(0xffffffffu, act, (3 * lane + 2) & 31);
      if (lane < U && u0 + lane < a.H) {
        c = f * c + (1.f - f) * z;
        float h = o * tanh_full(c);
        if (CELL == SRU) h = h + (1.f - o) * a.Xhw[t * a.ldhw + u0 + lane];
        store_h(a, t * a.ldh + u0 + lane, h);
      }
    }
    if (lane < U && a.c_out != nullptr && u0 + lane < a.H) a.c_out[u0 + lane] = c;
  }
}

}  // namespace rnnb
