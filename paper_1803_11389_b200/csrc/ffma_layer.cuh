// Fused blocked SRU/QRNN layer kernel on the FFMA (CUDA-core) pipe.
//
// Reference path (rnnblock, /root/reference/pkg/src/rnnblock):
//   run_blocked            blocked.py:221-268  (per layer, per block)
//   precompute_gates_*     blocked.py:123-150  (block projection + bias + act)
//   recurrence_sweep       blocked.py:153-176  (c_t = f c_{t-1} + (1-f) x-hat)
//   finalize_outputs       blocked.py:179-193  (h = o tanh c [+ (1-r) x])
// One launch runs one layer over the whole sequence.  Each CTA owns U hidden
// units (their 3 gate rows, gate-interleaved, K = taps*D columns) and that
// slice's c state for the whole sequence, so there is no cross-CTA
// dependency at all.  Per block of T_b steps the CTA
//   1. streams the input frames x[t0-1 .. t0+l) through shared memory in
//      K-chunks (cp.async double buffer) -- the QRNN x_{t-1} tap is the same
//      slab shifted one row, row -1 being the carried x (blocked.py:143,262);
//   2. multiplies them with its weight rows: weights live in shared memory
//      for the whole sequence when they fit (fetched from HBM once per
//      launch), otherwise they are re-read from L2 once per pass;
//   3. reduces across lanes/warps, applies bias + activations, runs the
//      sequential c-scan for the block in shared memory, and writes h.
// Gate pre-activations never leave the SM.
//
// Work mapping per pass of NT columns: 8 warps split K; inside a warp
// LANES_T lanes split the columns and LANES_K = 32/LANES_T lanes split K
// (lane = tq + LANES_T*kq).  Weight vectors are broadcast across the
// LANES_T lanes of one kq; x vectors come from a padded shared slab whose
// row stride makes each 8-lane phase hit 8 distinct 16-byte bank groups.
#pragma once
#include "common.cuh"

namespace rnnb {

template <typename TA, typename TW>
struct LayerArgs {
  const TW* W;         // [Upad*3][Kp] rows 3u+g (g: 0 cand, 1 forget, 2 out/highway); Kp = taps*Dp
  const TA* bias;      // SRU: [Upad][2] (b_forget, b_highway); QRNN: nullptr
  const TA* X;         // [L][ldx] layer input, rows are time steps
  int64_t ldx;
  const TA* xcarry;    // [D] x_{-1} for QRNN (nullptr: zeros)
  const TA* Xhw;       // SRU highway source, normally == X
  int64_t ldhw;
  TA* Hout;            // [L][ldh]
  int64_t ldh;         // may be negative (rows stored in reverse time order)
  TA* Hpeer[kMaxPeers];  // same layout as Hout on peer GPUs (mapped), npeer used
  int npeer;
  const TA* c_in;      // [H] initial c (nullptr: zeros)
  TA* c_out;           // [H] final c (nullptr: not written)
  TA* G;               // gates-out mode: [3][H][ldg] activated gates, no scan
  int64_t ldg;
  int64_t L;
  int T_b;
  int D, Dp, H;
  int KC;              // K-chunk (elements per tap) staged per pipeline step
  int KCB;             // TMA box width inside a chunk (ws kernel)
  int xround;          // XRound
  int dbg;             // debug switches (RNNB_DEBUG): bit0 consumers skip the x-ready wait
  // streaming (ws kernel only; rnnb_forward_host): rows of X present in
  // device memory so far (written by the copy stream), and per-chunk counts
  // of CTAs whose h rows of that chunk are stored (read by the copy-out stream)
  const int* x_ready;
  int* h_done;
  int h_chunk;
  int* stream_fail;    // set by the kernel if streamed rows did not arrive in time
  // weight-streaming ws kernel (layers whose weights do not fit in shared
  // memory): per-(CTA, chunk) weight images, see ws_stream_pack
  const TW* Wst;
};

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

template <typename TA, typename TW, int CELL, int NT, int U>
struct FfmaCfg {
  static constexpr int KV = 16 / (int)sizeof(TA);
  static constexpr int TAPS = CELL == QRNN ? 2 : 1;
  static constexpr int R = 3 * U;
  static constexpr int LANES_T = NT < 8 ? NT : 8;
  static constexpr int CT = NT / LANES_T;
  static constexpr int LANES_K = 32 / LANES_T;
  static constexpr int KL = kWarps * LANES_K;
  static constexpr int PADV = KV * (8 / LANES_T);  // row padding (elements)
};

__host__ __device__ inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

template <typename TA, typename TW, int CELL, int NT, int U>
__host__ __device__ inline size_t ffma_smem_bytes(int Dp, int KC, bool wsmem) {
  using C = FfmaCfg<TA, TW, CELL, NT, U>;
  size_t off = 0;
  if (wsmem) off = align_up((size_t)C::R * C::TAPS * Dp * sizeof(TW), 16);
  off += 2 * (size_t)(NT + 1) * (KC + C::PADV) * sizeof(TA);
  off += (size_t)kWarps * C::R * NT * sizeof(TA);
  off += (size_t)3 * U * NT * sizeof(TA);
  off += align_up((size_t)U * sizeof(TA), 16);
  return off;
}

template <typename TA, typename TW, int CELL, int NT, int U, bool WSMEM>
__global__ void __launch_bounds__(kThreads, 1) ffma_layer_kernel(LayerArgs<TA, TW> a) {
  using C = FfmaCfg<TA, TW, CELL, NT, U>;
  constexpr int KV = C::KV, TAPS = C::TAPS, R = C::R;
  constexpr int LANES_T = C::LANES_T, CT = C::CT, LANES_K = C::LANES_K, KL = C::KL;
  const int KC = a.KC;
  const int XS = KC + C::PADV;
  const int Dp = a.Dp;
  const int Kp = TAPS * Dp;

  extern __shared__ __align__(16) unsigned char smem[];
  size_t off = 0;
  TW* Ws = reinterpret_cast<TW*>(smem);
  if (WSMEM) off = align_up((size_t)R * Kp * sizeof(TW), 16);
  TA* Xs = reinterpret_cast<TA*>(smem + off);
  off += 2 * (size_t)(NT + 1) * XS * sizeof(TA);
  TA* red = reinterpret_cast<TA*>(smem + off);
  off += (size_t)kWarps * R * NT * sizeof(TA);
  TA* gate = reinterpret_cast<TA*>(smem + off);
  off += (size_t)3 * U * NT * sizeof(TA);
  TA* cst = reinterpret_cast<TA*>(smem + off);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int tq = lane % LANES_T, kq = lane / LANES_T;
  const int kl = warp * LANES_K + kq;
  const int u0 = blockIdx.x * U;
  const TW* Wg = a.W + (size_t)u0 * 3 * Kp;

  // vector staging needs 16-byte aligned rows; otherwise element-wise
  const bool xvec = ((a.ldx % KV) == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0) &&
                    (a.xcarry == nullptr || (reinterpret_cast<uintptr_t>(a.xcarry) & 15) == 0);

  if (WSMEM) {
    const int nvec = R * Kp * (int)sizeof(TW) / 16;
    for (int i = tid; i < nvec; i += kThreads)
      cp_async16(reinterpret_cast<char*>(Ws) + 16 * (size_t)i,
                 reinterpret_cast<const char*>(Wg) + 16 * (size_t)i, 16);
    cp_async_commit();
  }
  if (tid < U) {
    const int unit = u0 + tid;
    cst[tid] = (a.c_in != nullptr && unit < a.H) ? a.c_in[unit] : TA(0);
  }

  // stage x rows [tp-1, tp+nt) x [d0, d0+kcs) into buffer `buf`
  auto stage = [&](int buf, int64_t tp, int nt, int d0, int kcs) {
    TA* xb = Xs + (size_t)buf * (NT + 1) * XS;
    const int r0 = TAPS == 2 ? 0 : 1;
    const int nrow = nt + 1 - r0;
    if (xvec) {
      const int nv = kcs / KV;
      for (int i = tid; i < nrow * nv; i += kThreads) {
        const int r = r0 + i / nv, v = i % nv;
        const int d = d0 + v * KV;
        const int64_t gr = tp - 1 + r;
        const TA* src = a.X;
        int bytes = 0;
        if (gr >= 0) {
          src = a.X + gr * a.ldx + d;
          bytes = (a.D - d) * (int)sizeof(TA);
        } else if (a.xcarry != nullptr) {
          src = a.xcarry + d;
          bytes = (a.D - d) * (int)sizeof(TA);
        }
        bytes = bytes < 0 ? 0 : (bytes > 16 ? 16 : bytes);
        if (bytes == 0) src = a.X;
        cp_async16(xb + (size_t)r * XS + v * KV, src, bytes);
      }
    } else {
      for (int i = tid; i < nrow * kcs; i += kThreads) {
        const int r = r0 + i / kcs, e = i % kcs;
        const int d = d0 + e;
        const int64_t gr = tp - 1 + r;
        const TA* src = a.X;
        int bytes = 0;
        if (d < a.D) {
          if (gr >= 0) { src = a.X + gr * a.ldx + d; bytes = sizeof(TA); }
          else if (a.xcarry != nullptr) { src = a.xcarry + d; bytes = sizeof(TA); }
        }
        if (sizeof(TA) == 4) cp_async4(xb + (size_t)r * XS + e, src, bytes);
        else cp_async8(xb + (size_t)r * XS + e, src, bytes);
      }
    }
  };

  const int nchunk = (Dp + KC - 1) / KC;
  for (int64_t t0 = 0; t0 < a.L; t0 += a.T_b) {
    const int l = (int)((a.L - t0) < a.T_b ? (a.L - t0) : a.T_b);
    for (int p0 = 0; p0 < l; p0 += NT) {
      const int nt = (l - p0) < NT ? (l - p0) : NT;
      const int64_t tp = t0 + p0;

      TA acc[R][CT];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int ct = 0; ct < CT; ++ct) acc[r][ct] = TA(0);

      stage(0, tp, nt, 0, KC < Dp ? KC : Dp);
      cp_async_commit();
      for (int ch = 0; ch < nchunk; ++ch) {
        cp_async_wait<0>();
        __syncthreads();
        const int d0 = ch * KC;
        const int kcs = (Dp - d0) < KC ? (Dp - d0) : KC;
        if (ch + 1 < nchunk) {
          const int d1 = d0 + KC;
          stage((ch + 1) & 1, tp, nt, d1, (Dp - d1) < KC ? (Dp - d1) : KC);
          cp_async_commit();
        }
        const TA* xb = Xs + (size_t)(ch & 1) * (NT + 1) * XS;
        const int nv = kcs / KV;
        const int items = TAPS * nv;
        for (int it = kl; it < items; it += KL) {
          const int tap = (TAPS == 2 && it >= nv) ? 1 : 0;
          const int dv = it - tap * nv;
          TA xv[CT][KV];
#pragma unroll
          for (int ct = 0; ct < CT; ++ct) {
            const int row = tq + LANES_T * ct + 1 - tap;
            Vec16<TA> v = lds16<TA>(xb + (size_t)row * XS + dv * KV);
#pragma unroll
            for (int e = 0; e < KV; ++e) xv[ct][e] = round_x(v.v[e], a.xround);
          }
          const int kg = tap * Dp + d0 + dv * KV;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            TA w[KV];
            if (WSMEM) WLoad<TA, TW>::shared(Ws + (size_t)r * Kp + kg, w);
            else WLoad<TA, TW>::global(Wg + (size_t)r * Kp + kg, w);
#pragma unroll
            for (int ct = 0; ct < CT; ++ct)
#pragma unroll
              for (int e = 0; e < KV; ++e) acc[r][ct] = fma(w[e], xv[ct][e], acc[r][ct]);
          }
        }
      }

      // lanes sharing tq hold partial sums over disjoint K: butterfly over kq
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int ct = 0; ct < CT; ++ct) {
          TA v = acc[r][ct];
#pragma unroll
          for (int o = LANES_T; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          acc[r][ct] = v;
        }
      if (kq == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int ct = 0; ct < CT; ++ct)
            red[((size_t)warp * R + r) * NT + tq + LANES_T * ct] = acc[r][ct];
      }
      __syncthreads();

      // cross-warp sum in fixed order, bias, activations (blocked.py:128-130,144-149)
      for (int i = tid; i < R * nt; i += kThreads) {
        const int r = i / nt, col = i - (i / nt) * nt;
        TA s = TA(0);
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s += red[((size_t)w * R + r) * NT + col];
        const int u = r / 3, g = r - 3 * (r / 3);
        TA v;
        if (CELL == SRU) {
          v = g == 0 ? s : sigmoid_ref<TA>(s + a.bias[(size_t)(u0 + u) * 2 + g - 1]);
        } else {
          v = g == 0 ? tanh_full(s) : sigmoid_ref<TA>(s);
        }
        gate[((size_t)g * U + u) * NT + col] = v;
      }
      __syncthreads();

      if (a.G != nullptr) {  // unit-level precompute_gates_*: activated gates out
        for (int i = tid; i < 3 * U * nt; i += kThreads) {
          const int col = i % nt, gu = i / nt, g = gu / U, u = gu % U;
          if (u0 + u < a.H)
            a.G[((size_t)g * a.H + u0 + u) * a.ldg + tp + col] = gate[((size_t)g * U + u) * NT + col];
        }
        __syncthreads();
        continue;
      }

      // sequential c-scan across the pass (blocked.py:153-162); c carried in smem
      if (tid < U) {
        TA c = cst[tid];
        TA* cand = gate + (size_t)tid * NT;
        const TA* fg = gate + (size_t)(U + tid) * NT;
        for (int col = 0; col < nt; ++col) {
          const TA f = fg[col];
          c = f * c + (TA(1) - f) * cand[col];
          cand[col] = c;
        }
        cst[tid] = c;
      }
      __syncthreads();

      // output mix (blocked.py:179-193)
      for (int i = tid; i < U * nt; i += kThreads) {
        const int u = i % U, col = i / U;
        const int unit = u0 + u;
        if (unit < a.H) {
          const TA c = gate[(size_t)u * NT + col];
          const TA o = gate[((size_t)2 * U + u) * NT + col];
          TA h = o * tanh_full(c);
          if (CELL == SRU) h = h + (TA(1) - o) * a.Xhw[(tp + col) * a.ldhw + unit];
          store_h(a, (tp + col) * a.ldh + unit, h);
        }
      }
    }
  }
  if (WSMEM) { cp_async_wait<0>(); }
  __syncthreads();
  if (tid < U && a.c_out != nullptr && u0 + tid < a.H) a.c_out[u0 + tid] = cst[tid];
}

}  // namespace rnnb
