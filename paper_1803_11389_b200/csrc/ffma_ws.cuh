// Warp-specialised fused blocked SRU/QRNN layer kernel (FFMA pipe), v2.
//
// Same math and reference mapping as ffma_layer.cuh (rnnblock blocked.py:
// 123-193, 221-268), re-organised for B200:
//   * weights for the CTA's U units live in shared memory for the whole
//     sequence in a k-vector-major layout Ws[kv][Rs][KV], so the 3U rows of
//     one k-vector sit at compile-time offsets (one address per item);
//   * warp 8 is a TMA producer: cp.async.bulk copies of x-row chunks into a
//     STAGES-deep ring guarded by full/empty mbarriers (no __syncthreads in
//     the main loop);
//   * warps 0-7 are FFMA consumers (K split across warps and lanes);
//   * warp 9 is the epilogue: cross-warp sums, bias + activations, the
//     sequential c-scan, the output mix and the h stores of pass p run
//     while the consumers already multiply pass p+1.
// Requirements (checked on the host): D % 8 == 0, 16-byte aligned X /
// x_carry rows, ldx % 4 == 0 and the weight slice fits in shared memory.
#pragma once
#include <cuda.h>  // CUtensorMap (type only; encoded via the runtime's driver entry point)

#include <type_traits>

#include "ffma_layer.cuh"

namespace rnnb {

#ifndef RNNB_PROD_SLEEP_NS
#define RNNB_PROD_SLEEP_NS 1024  // producer back-off cap while waiting for a free ring slot
#endif
#ifndef RNNB_WIDE_MIN_NT
#define RNNB_WIDE_MIN_NT 1
#endif
#ifndef RNNB_NT32_NRED
#define RNNB_NT32_NRED 1  // 32-column passes: double-buffered cross-warp partials (1) or single (0)
#endif
#ifndef RNNB_NT32_STAGES
#define RNNB_NT32_STAGES 3
#endif
// Epilogue warps: 3 beside the 8 consumer warps of the wide fp32 tile (the
// epilogue competes with the consumers for issue slots and falls behind with
// 2: 3 measured +1.4 % at T_b=32, +2.5 % at T_b=8; 1 -> -3 %; 4 lowers the
// register cap to 152 -> spills); 2 beside 16 consumer warps (96-register cap).
#ifndef RNNB_EPI_WARPS
#define RNNB_EPI_WARPS 3
#endif

// named barrier 1 over the epilogue warpgroup only
template <int NTHR>
__device__ __forceinline__ void epi_bar_sync() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(NTHR) : "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t tx) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(
                   smem_u32(bar)),
               "r"(tx)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t tx) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// off-critical-path wait (producer / epilogue): back off with nanosleep so the
// spinning warp does not steal issue slots from the FFMA consumers
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t max_ns = 1024) {
  uint32_t ns = 32;
  while (true) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    __nanosleep(ns);
    ns = ns < max_ns ? ns * 2 : max_ns;
  }
}
// 2-D TMA tile load (tensor map in param space), completion on `bar`
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// packed fp32x2 FMA (sm_100): d = a * b + c on (lo, hi) float pairs
// Two spellings, same instruction: the compiler builtin lets ptxas coalesce
// accumulators in place (no register-rotation moves) but costs registers;
// the inline-asm form is kept for kernels that run at the 96-register cap.
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  const float2 r = __ffma2_rn(*reinterpret_cast<const float2*>(&a), *reinterpret_cast<const float2*>(&b),
                              *reinterpret_cast<const float2*>(&c));
  return *reinterpret_cast<const unsigned long long*>(&r);
}
__device__ __forceinline__ unsigned long long ffma2_asm(unsigned long long a, unsigned long long b,
                                                        unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
template <bool kBuiltin>
__device__ __forceinline__ unsigned long long ffma2_sel(unsigned long long a, unsigned long long b,
                                                        unsigned long long c) {
  if constexpr (kBuiltin) return ffma2(a, b, c);
  else return ffma2_asm(a, b, c);
}
// streaming input: spin (with back-off) until `need` rows of X are in device
// memory, then order the following TMA (async-proxy) reads after that.  If
// the rows do not arrive within kStreamTimeoutNs of kernel start (e.g. a
// profiler serialises the copy stream behind this kernel) the kernel stops
// waiting, flags *fail and runs to completion on whatever is there -- the
// host sees the flag and recomputes without streaming.  Returns false on
// time-out.
constexpr uint64_t kStreamTimeoutNs = 2000000000ull;
__device__ __forceinline__ int wait_rows(const int* ready, int need, uint64_t t_start, int* fail) {
  // returns the row count observed (>= need), or -1 after the time-out
  int have = 0;
  if ((threadIdx.x & 31) == 0) {
    uint32_t ns = 32;
    while (true) {
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(have) : "l"(ready) : "memory");
      if (have >= need) break;
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t_start > kStreamTimeoutNs) {
        atomicExch(fail, 1);
        have = -1;
        break;
      }
      __nanosleep(ns);
      ns = ns < 256 ? ns * 2 : 256;
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  return __shfl_sync(0xffffffffu, have, 0);
}
// 1-D TMA bulk copy global -> shared, completion counted on `bar` in bytes
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Consumer mapping: CW = KG k-groups x RG row-groups of consumer warps.  A
// warp owns RH = ceil(R/RG) rows over its k-group's share of K; inside the
// warp LANES_T lanes split the NT columns (CT columns each) and LANES_K lanes
// split K.  A weight LDS feeds CT*KV FMAs and an x LDS RH*KV, so the wide
// tile (CT = 4, fp32, NT >= 16) halves the LDS per FMA of the narrow one;
// it needs ~2x the accumulator registers, so it runs 8 consumer warps
// (KG = 4) with up to 168 registers each instead of 16 with 96.
template <typename TA, typename TW, int CELL, int NT, int U, bool WSTR = false>
struct WsCfg {
  static constexpr int KV = 16 / (int)sizeof(TA);
  static constexpr int TAPS = CELL == QRNN ? 2 : 1;
  static constexpr int R = 3 * U;
  static constexpr int CTW = (sizeof(TA) == 4 && NT >= RNNB_WIDE_MIN_NT) ? 4 : 2;
  // more rows per CTA (U = 14, weight-streaming layers) -> more row groups,
  // same per-warp tile and warp count
  static constexpr int RG = R > 24 ? 4 : 2;
  static constexpr int KG = (CTW == 4 ? 8 : 16) / RG;
  static constexpr int CW = KG * RG;                       // consumer warps
  static constexpr int EPIW = CW == 8 ? RNNB_EPI_WARPS : 2;  // epilogue warps
  static constexpr int EPIT = EPIW * 32;
  static constexpr int THREADS = (CW + 1 + EPIW) * 32;  // + producer + epilogue group
  static constexpr int RH = (R + RG - 1) / RG;
  static constexpr int Rpad = RH * RG;
  // smem row count per k-vector: odd so consecutive kv (lanes kq) hit distinct
  // 16-byte bank groups; rows [R, Rpad) read garbage that is never used
  static constexpr int Rs = (R % 2) ? R : R + 1;
  static constexpr int LANES_T = NT >= CTW ? NT / CTW : 1;
  static constexpr int CT = NT / LANES_T;
  static constexpr int LANES_K = 32 / LANES_T;
  static constexpr int KL = KG * LANES_K;
  // padded x row pitch: each 8-lane phase (LANES_T rows x 8/LANES_T k-vectors)
  // must hit 8 distinct 16-byte bank groups; one row needs no padding
  static constexpr int PADV = LANES_T == 1 ? 0 : KV * (LANES_T >= 8 ? 1 : 8 / LANES_T);
  // the 32-column pass (fp32, T_b >= 32) double-buffers the cross-warp partials
  // so consumers reduce pass p+1 while the epilogue still reads pass p; it
  // pays for the second buffer with one x stage
  // (also the short fp32 passes, NT <= 8, where a pass lasts ~1 us and the
  // buffers cost < 3 KB)
  static constexpr int NRED = (NT == 32 ? RNNB_NT32_NRED : (sizeof(TA) == 4 && NT <= 8)) ? 2 : 1;
  // WSTR: weights are not resident, so the ring can be deeper; each stage
  // also carries the chunk's weight image
  static constexpr int STAGES = WSTR ? 6 : (NT == 32 ? RNNB_NT32_STAGES : 4);
};

// Reduce-scatter of NR partials over the lanes whose bits are O, 2O, .., 16:
// at each level a lane keeps the half of its live partials selected by its
// lane bit and adds the partner's copy of that half, so partial j ends in one
// lane; odd counts are padded by one zero (not the old padding of NR up to a
// multiple of the lane count: at NT = 1, 11 partials over 32 lanes cost 13
// shuffles instead of 31).  Once one partial is left, the remaining levels
// are a butterfly: both partners hold the sum and the upper one is marked
// `dup`.  Afterwards a lane holds partials jb .. jb + ws_rs_final - 1, of
// which the first `nreal` are real (the rest are padding: with odd counts
// a padded slot's index can coincide with a real partial of another lane).
template <int CUR, int O>
__host__ __device__ constexpr int ws_rs_final() {
  if constexpr (O >= 32) return CUR;
  else return ws_rs_final<(CUR > 1 ? (CUR + 1) / 2 : 1), O * 2>();
}
template <typename TA, int CUR, int O, int N>
__device__ __forceinline__ void ws_reduce_scatter(TA (&v)[N], int lane, int& jb, bool& dup, int& nreal) {
  if constexpr (O < 32) {
    const bool upper = (lane & O) != 0;
    if constexpr (CUR > 1) {
      constexpr int HALF = (CUR + 1) / 2;
#pragma unroll
      for (int i = 0; i < HALF; ++i) {
        const TA hi = (i + HALF < CUR) ? v[i + HALF] : TA(0);
        const TA send = upper ? v[i] : hi;
        const TA keep = upper ? hi : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, O);
      }
      if (upper) {
        jb += HALF;
        nreal = nreal > HALF ? nreal - HALF : 0;
      } else {
        nreal = nreal < HALF ? nreal : HALF;
      }
      ws_reduce_scatter<TA, HALF, O * 2>(v, lane, jb, dup, nreal);
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], O);
      if (upper) dup = true;
      ws_reduce_scatter<TA, 1, O * 2>(v, lane, jb, dup, nreal);
    }
  }
}

// x chunk of KC columns = KC/BW TMA boxes of [NT+1 rows x (BW + PADV) cols],
// each box at a 128-byte aligned stride inside the stage buffer
template <typename TA, typename TW, int CELL, int NT, int U, bool WSTR = false>
__host__ __device__ inline size_t ws_box_elems(int BW) {
  using C = WsCfg<TA, TW, CELL, NT, U, WSTR>;
  return align_up((size_t)(NT + 1) * (BW + C::PADV), 128 / sizeof(TA));
}

// WSTR: one chunk's weight image in global memory and in a stage, elements:
// [tap][kv of the chunk][Rs][KV] (the resident layout restricted to a chunk)
template <typename TA, typename TW, int CELL, int NT, int U, bool WSTR = false>
__host__ __device__ inline size_t ws_wimg_elems(int KC) {
  using C = WsCfg<TA, TW, CELL, NT, U, WSTR>;
  return (size_t)C::TAPS * (KC / C::KV) * C::Rs * C::KV;
}

template <typename TA, typename TW, int CELL, int NT, int U, bool WSTR = false>
__host__ __device__ inline size_t ws_smem_bytes(int Dp, int KC, int BW) {
  using C = WsCfg<TA, TW, CELL, NT, U, WSTR>;
  size_t off = WSTR ? 0 : align_up((size_t)C::TAPS * Dp / C::KV * C::Rs * C::KV * sizeof(TW) + 16 * C::RG, 128);
  off += (size_t)C::STAGES * align_up(((KC + BW - 1) / BW) * ws_box_elems<TA, TW, CELL, NT, U, WSTR>(BW) * sizeof(TA) +
                                          (WSTR ? ws_wimg_elems<TA, TW, CELL, NT, U, WSTR>(KC) * sizeof(TW) : 0),
                                      128);
  off += (size_t)C::NRED * C::KG * C::Rpad * NT * sizeof(TA);
  off += (size_t)3 * U * NT * sizeof(TA);
  off = align_up(off, 8);
  off += (2 * C::STAGES + 2 * C::NRED) * sizeof(uint64_t);
  return off;
}

// STREAM: X arrives while the kernel runs (rnnb_forward_host streaming); a
// separate instantiation so the plain kernel's code is untouched.
// WSTR: the layer's weights do not fit in shared memory (BASELINE cfg4 fp32):
// each stage of the ring also carries the chunk's weight image, bulk-copied
// from a pre-tiled copy (a.Wst: [CTA][chunk][tap][kv][Rs][KV]), so every
// weight is fetched once per pass of NT columns.
template <typename TA, typename TW, int CELL, int NT, int U, int XR, bool STREAM = false, bool WSTR = false>
__global__ void __launch_bounds__(WsCfg<TA, TW, CELL, NT, U, WSTR>::THREADS, 1)
    ffma_ws_kernel(LayerArgs<TA, TW> a, const __grid_constant__ CUtensorMap tmx) {
  using C = WsCfg<TA, TW, CELL, NT, U, WSTR>;
  constexpr int KV = C::KV, TAPS = C::TAPS, R = C::R, Rs = C::Rs, KG = C::KG, RH = C::RH, Rpad = C::Rpad;
  constexpr int LANES_T = C::LANES_T, CT = C::CT, LANES_K = C::LANES_K, KL = C::KL;
  constexpr int STAGES = C::STAGES;
  constexpr int CW = C::CW, NTHR = C::THREADS;
  const int KC = a.KC;
  const int BW = a.KCB;                  // TMA box width (columns)
  const int BXS = BW + C::PADV;          // padded row pitch inside a box
  const int LVPB = __ffs(BW / KV) - 1;   // log2(k-vectors per box); BW is a power of 2
  const int MVPB = BW / KV - 1;
  const int BOXS = (int)ws_box_elems<TA, TW, CELL, NT, U, WSTR>(BW);
  const int Dp = a.Dp;
  const int Kv = TAPS * Dp / KV;  // k-vectors per row

  extern __shared__ __align__(128) unsigned char smem[];
  size_t off = 0;
  TW* Ws = reinterpret_cast<TW*>(smem);
  if constexpr (!WSTR) off = align_up((size_t)Kv * Rs * KV * sizeof(TW) + 16 * C::RG, 128);  // TMA dst: 128-B aligned
  TA* Xr = reinterpret_cast<TA*>(smem + off);
  const size_t xstage_bytes = (size_t)((KC + BW - 1) / BW) * BOXS * sizeof(TA);
  const size_t wimg_elems = WSTR ? ws_wimg_elems<TA, TW, CELL, NT, U, WSTR>(KC) : 0;
  // stage = x boxes [+ weight image]; the weight image follows the boxes
  const size_t stage_bytes = align_up(xstage_bytes + wimg_elems * sizeof(TW), 128);
  off += (size_t)STAGES * stage_bytes;
  constexpr int NRED = C::NRED;
  constexpr size_t red_elems = (size_t)KG * Rpad * NT;
  TA* red = reinterpret_cast<TA*>(smem + off);
  off += (size_t)NRED * red_elems * sizeof(TA);
  TA* gate = reinterpret_cast<TA*>(smem + off);
  off += (size_t)3 * U * NT * sizeof(TA);
  off = align_up(off, 8);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + off);
  uint64_t* empty = full + STAGES;
  uint64_t* redfull = empty + STAGES;    // [NRED]
  uint64_t* redempty = redfull + NRED;   // [NRED]

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int u0 = blockIdx.x * U;
  const TW* Wg = a.W + (size_t)u0 * 3 * TAPS * Dp;

  // weights -> Ws[kv][r][:], once per launch (rows of Wg are [R][Kp])
  if constexpr (!WSTR) {
    constexpr int VB = KV * (int)sizeof(TW);  // bytes per (kv, r) vector
    const int nvec = R * Kv;
    for (int i = tid; i < nvec; i += NTHR) {
      const int r = i / Kv, kv = i - (i / Kv) * Kv;
      char* dst = reinterpret_cast<char*>(Ws) + ((size_t)kv * Rs + r) * VB;
      const char* src = reinterpret_cast<const char*>(Wg) + ((size_t)r * Kv + kv) * VB;
      if (VB == 16) cp_async16(dst, src, 16);
      else cp_async8(dst, src, 8);
    }
    cp_async_commit();
  }
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    for (int b = 0; b < NRED; ++b) {
      mbar_init(&redfull[b], CW);
      mbar_init(&redempty[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  cp_async_wait<0>();
  __syncthreads();

  const int nchunk = (Dp + KC - 1) / KC;
  const int rot = (int)(blockIdx.x % (unsigned)nchunk);
  const int r0 = TAPS == 2 ? 0 : 1;  // SRU never reads row 0 (x_{t-1})

  if (warp == CW) {
    // ---------------- producer: TMA bulk copies of x-row chunks ----------------
    uint32_t seq = 0;
    bool timed_out = false;
    uint64_t t_start = 0;
    int rows_seen = 0;  // STREAM: rows of X known to be resident
    if constexpr (STREAM) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    for (int64_t t0 = 0; t0 < a.L; t0 += a.T_b) {
      const int l = (int)((a.L - t0) < a.T_b ? (a.L - t0) : a.T_b);
      for (int p0 = 0; p0 < l; p0 += NT) {
        const int nt = (l - p0) < NT ? (l - p0) : NT;
        const int64_t tp = t0 + p0;
        for (int ch = 0; ch < nchunk; ++ch, ++seq) {
          const int s = seq % STAGES;
          const uint32_t ph = (seq / STAGES) & 1;
          if (a.dbg & 1) continue;
          mbar_wait_sleep(&empty[s], ph ^ 1, RNNB_PROD_SLEEP_NS);
          if constexpr (STREAM) {
            // rows already seen resident need no new acquire round trip
            const int need = (int)((tp + NT) < a.L ? (tp + NT) : a.L);
            if (ch == 0 && !timed_out && need > rows_seen) {
              const int got = wait_rows(a.x_ready, need, t_start, a.stream_fail);
              if (got < 0) timed_out = true;
              else rows_seen = got;
            }
          }
          const int d0 = ((ch + rot) % nchunk) * KC;  // per-CTA chunk rotation spreads L2 hot lines
          const int kcs = (Dp - d0) < KC ? (Dp - d0) : KC;
          TA* xb = reinterpret_cast<TA*>(reinterpret_cast<char*>(Xr) + (size_t)s * stage_bytes);
          const bool carry_row = (r0 == 0 && tp == 0 && a.xcarry != nullptr);
          if constexpr (WSTR) {
            // this chunk's weight image: one bulk copy, counted on the same barrier
            if (lane == 0) {
              const uint32_t wb = (uint32_t)(wimg_elems * sizeof(TW));
              mbar_expect_tx(&full[s], wb);  // no arrival: the x copies below arrive once
              const TW* src = a.Wst + ((size_t)blockIdx.x * nchunk + (size_t)(d0 / KC)) * wimg_elems;
              bulk_g2s(reinterpret_cast<char*>(xb) + xstage_bytes, src, wb, &full[s]);
            }
          }
          if (!carry_row) {
            // one 2-D TMA box [NT+1-r0 rows x XS cols] per chunk: box rows land at
            // pitch XS (the padding columns are real neighbours, never read), rows
            // before 0 or past L and columns past D are zero-filled by the TMA unit
            if (lane == 0) {
              const int nb = (kcs + BW - 1) / BW;
              mbar_arrive_expect_tx(&full[s], (uint32_t)(nb * (NT + 1) * BXS * sizeof(TA)));
              for (int b = 0; b < nb; ++b) tma_load_2d(xb + (size_t)b * BOXS, &tmx, d0 + b * BW, (int)(tp - 1), &full[s]);
            }
            continue;
          }
          // first pass with a carried x_{-1}: row 0 from x_carry, rows 1.. per row
          const int nb = (kcs + BW - 1) / BW;
          __syncwarp();
          if (lane == 0) mbar_arrive_expect_tx(&full[s], (uint32_t)((nt + 1) * kcs * sizeof(TA)));
          __syncwarp();
          for (int i = lane; i < (nt + 1) * nb; i += 32) {
            const int r = i / nb, b = i - (i / nb) * nb;
            const int64_t gr = tp - 1 + r;
            const int w = (kcs - b * BW) < BW ? (kcs - b * BW) : BW;
            const TA* src = gr >= 0 ? a.X + gr * a.ldx + d0 + b * BW : a.xcarry + d0 + b * BW;
            bulk_g2s(xb + (size_t)b * BOXS + (size_t)r * BXS, src, (uint32_t)(w * sizeof(TA)), &full[s]);
          }
        }
      }
    }
  } else if (warp > CW) {
    // ------------- epilogue warpgroup: sums, activations, scan, output -------------
    const int et = tid - (CW + 1) * 32;  // 0 .. EPIT-1
    TA c = TA(0);
    if (et < U && a.c_in != nullptr && u0 + et < a.H) c = a.c_in[u0 + et];
    uint32_t pass = 0;
    for (int64_t t0 = 0; t0 < a.L; t0 += a.T_b) {
      const int l = (int)((a.L - t0) < a.T_b ? (a.L - t0) : a.T_b);
      for (int p0 = 0; p0 < l; p0 += NT, ++pass) {
        const int nt = (l - p0) < NT ? (l - p0) : NT;
        const int64_t tp = t0 + p0;
        const int rb = NRED == 2 ? (int)(pass & 1) : 0;
        const uint32_t rph = (NRED == 2 ? pass >> 1 : pass) & 1;
        const TA* redb = red + rb * red_elems;
        mbar_wait_sleep(&redfull[rb], rph, NT <= 8 ? 128u : 1024u);  // short passes: wake promptly
        for (int i = et; i < ((a.dbg & 4) ? 0 : R * nt); i += C::EPIT) {
          const int r = i / nt, col = i - (i / nt) * nt;
          TA s = TA(0);
#pragma unroll
          for (int w = 0; w < KG; ++w) s += redb[((size_t)w * Rpad + r) * NT + col];
          const int u = r / 3, g = r - 3 * (r / 3);
          TA v;
          if (CELL == SRU)
            v = g == 0 ? s : sigmoid_ref<TA>(s + (u0 + u < a.H ? a.bias[(size_t)(u0 + u) * 2 + g - 1] : TA(0)));
          else v = g == 0 ? tanh_full(s) : sigmoid_ref<TA>(s);
          gate[((size_t)g * U + u) * NT + col] = v;
        }
        epi_bar_sync<C::EPIT>();
        if (et == 0) mbar_arrive(&redempty[rb]);
        if (et < U && !(a.dbg & 4)) {
          TA* cand = gate + (size_t)et * NT;
          const TA* fg = gate + (size_t)(U + et) * NT;
          for (int col = 0; col < nt; ++col) {
            const TA f = fg[col];
            c = f * c + (TA(1) - f) * cand[col];
            cand[col] = c;
          }
        }
        epi_bar_sync<C::EPIT>();
        for (int i = et; i < ((a.dbg & 4) ? 0 : U * nt); i += C::EPIT) {
          const int u = i % U, col = i / U;
          const int unit = u0 + u;
          if (unit < a.H) {
            const TA cc = gate[(size_t)u * NT + col];
            const TA o = gate[((size_t)2 * U + u) * NT + col];
            TA h = o * tanh_full(cc);
            if (CELL == SRU) h = h + (TA(1) - o) * a.Xhw[(tp + col) * a.ldhw + unit];
            store_h(a, (tp + col) * a.ldh + unit, h);
          }
        }
        epi_bar_sync<C::EPIT>();
        if constexpr (STREAM) {
          if (et == 0 && ((tp + nt) % a.h_chunk == 0 || tp + nt == a.L)) {
            __threadfence();  // this CTA's h rows of the chunk (ordered by the barrier) before the count
            atomicAdd(&a.h_done[(tp + nt - 1) / a.h_chunk], 1);
          }
        }
      }
    }
    if (et < U && a.c_out != nullptr && u0 + et < a.H) a.c_out[u0 + et] = c;
  } else {
    // ---------------- consumers: FFMA over the staged chunks ----------------
    const int tq = lane % LANES_T, kq = lane / LANES_T;
    const int rg = warp / KG, kg = warp - (warp / KG) * KG;
    const int kl = kg * LANES_K + kq;
    const int rbase = rg * RH;
    // lane-constant x offset: box of k-vector kl, row tq+1 (tap 0, column tq)
    const int xlane = (kl >> LVPB) * BOXS + (tq + 1) * BXS + (kl & MVPB) * KV;
    const TA* xlane_base = Xr + xlane;
    const size_t stage_elems = stage_bytes / sizeof(TA);
    const TW* wlane_base = WSTR ? reinterpret_cast<const TW*>(reinterpret_cast<const char*>(Xr) + xstage_bytes) +
                                      ((size_t)kl * Rs + rbase) * KV
                                : Ws + ((size_t)kl * Rs + rbase) * KV;
    const size_t w_chunk = (size_t)(KC / KV) * Rs * KV;  // weights of one chunk (all rows)
    // tap stride inside the weights a lane reads: the resident array holds all
    // of K per tap, a streamed chunk image one chunk per tap
    const size_t w_tap = WSTR ? w_chunk : (size_t)(Dp / KV) * Rs * KV;
    const size_t stage_tw = stage_bytes / sizeof(TW);
    const int kv_last = (Dp - (nchunk - 1) * KC) / KV;    // k-vectors in the last chunk
    // One-column fp32 passes (T_b = 1) are bound by shared-memory bandwidth:
    // every weight is re-read for one FMA.  Each lane keeps its weights of
    // chunk 0 (TAPS x RH vectors = 88 registers at U = 7) in registers for the
    // whole sequence and reads only the other chunks from shared memory
    // (cfg2 T_b = 1: 0.87 -> 0.93 M steps/s; at NT = 2 the extra registers
    // cost more than they save: 1.52 -> 1.33, so NT = 1 only).
    constexpr bool kRegW = sizeof(TA) == 4 && sizeof(TW) == 4 && XR == XR_NONE && !WSTR && NT == 1;
    ulonglong2 wreg[kRegW ? TAPS : 1][kRegW ? RH : 1];
    if constexpr (kRegW) {
      const bool has0 = nchunk > 1 || kl < kv_last;  // chunk 0 is partial only when it is the only chunk
#pragma unroll
      for (int tap = 0; tap < TAPS; ++tap)
#pragma unroll
        for (int r = 0; r < RH; ++r)
          wreg[tap][r] = has0 ? *reinterpret_cast<const ulonglong2*>(wlane_base + (size_t)tap * w_tap + r * KV)
                              : make_ulonglong2(0ull, 0ull);
    }
    uint32_t seq = 0, pass = 0;
    for (int64_t t0 = 0; t0 < a.L; t0 += a.T_b) {
      const int l = (int)((a.L - t0) < a.T_b ? (a.L - t0) : a.T_b);
      for (int p0 = 0; p0 < l; p0 += NT, ++pass) {
        // fp32 with fp32 weights: packed FFMA2 (Blackwell fma.rn.f32x2) on
        // (k even, k odd) accumulator pairs -- half the FMA issue slots; the
        // pair halves are summed after the K loop
        constexpr bool kPacked = sizeof(TA) == 4 && sizeof(TW) == 4 && XR == XR_NONE;
        TA acc[RH][CT];
        unsigned long long acc2[kPacked ? RH : 1][kPacked ? CT : 1];
#pragma unroll
        for (int r = 0; r < RH; ++r)
#pragma unroll
          for (int ct = 0; ct < CT; ++ct) acc[r][ct] = TA(0);
        if (kPacked) {
#pragma unroll
          for (int r = 0; r < (kPacked ? RH : 1); ++r)
#pragma unroll
            for (int ct = 0; ct < (kPacked ? CT : 1); ++ct) acc2[r][ct] = 0ull;
        }
        constexpr int kUnrollCh = 1;
        // chunk index cc runs rot, rot+1, .. (mod nchunk) -- the producer's order;
        // kept incrementally (no per-chunk division)
        int cc = rot;
#pragma unroll kUnrollCh
        for (int ch = 0; ch < nchunk; ++ch, ++seq) {
          const int s = seq % STAGES;
          if (!(a.dbg & 1)) mbar_wait(&full[s], (seq / STAGES) & 1);
          const int ccur = cc;
          cc = cc + 1 == nchunk ? 0 : cc + 1;
          // KC == KL*KV (host): every lane owns exactly one k-vector per tap per
          // chunk, at a lane-constant offset inside the staged box; only the
          // last chunk of a row can be partial
          if (ccur != nchunk - 1 || kl < kv_last) {
            const TA* xl = xlane_base + (size_t)s * stage_elems;
            const TW* wl = WSTR ? wlane_base + (size_t)s * stage_tw : wlane_base + (size_t)ccur * w_chunk;
#pragma unroll
            for (int tap = 0; tap < TAPS; ++tap) {
              const TW* wp = wl + (size_t)tap * w_tap;
              if constexpr (kPacked) {
                ulonglong2 xp[CT];
#pragma unroll
                for (int ct = 0; ct < CT; ++ct)
                  xp[ct] = *reinterpret_cast<const ulonglong2*>(xl + (size_t)(LANES_T * ct - tap) * BXS);
                auto rows = [&](auto from_regs) {
#pragma unroll
                  for (int r = 0; r < RH; ++r) {
                    ulonglong2 w;
                    if constexpr (decltype(from_regs)::value) w = wreg[kRegW ? tap : 0][kRegW ? r : 0];
                    else w = *reinterpret_cast<const ulonglong2*>(wp + r * KV);
                    // both k-pair halves of a row: CT independent FFMA2 between
                    // the two updates of one accumulator
#pragma unroll
                    for (int ct = 0; ct < CT; ++ct) acc2[r][ct] = ffma2_sel<C::CTW == 4>(w.x, xp[ct].x, acc2[r][ct]);
#pragma unroll
                    for (int ct = 0; ct < CT; ++ct) acc2[r][ct] = ffma2_sel<C::CTW == 4>(w.y, xp[ct].y, acc2[r][ct]);
                  }
                };
                if (kRegW && ccur == 0) rows(std::integral_constant<bool, kRegW>{});
                else rows(std::false_type{});
              } else {
                TA xv[CT][KV];
#pragma unroll
                for (int ct = 0; ct < CT; ++ct) {
                  Vec16<TA> v = lds16<TA>(xl + (size_t)(LANES_T * ct - tap) * BXS);
#pragma unroll
                  for (int e = 0; e < KV; ++e) xv[ct][e] = round_x(v.v[e], XR);
                }
#pragma unroll
                for (int r = 0; r < RH; ++r) {
                  TA w[KV];
                  WLoad<TA, TW>::shared(wp + r * KV, w);
#pragma unroll
                  for (int ct = 0; ct < CT; ++ct)
#pragma unroll
                    for (int e = 0; e < KV; ++e) acc[r][ct] = fma(w[e], xv[ct][e], acc[r][ct]);
                }
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
        }
        if constexpr (kPacked) {
#pragma unroll
          for (int r = 0; r < RH; ++r)
#pragma unroll
            for (int ct = 0; ct < CT; ++ct)
              acc[r][ct] = __uint_as_float((unsigned)acc2[r][ct]) + __uint_as_float((unsigned)(acc2[r][ct] >> 32));
        }
        // reduce-scatter over the LANES_K lanes of the k-group.  Short passes
        // (NT <= 4: 32 lanes split K, few partials) use the minimal-padding
        // ws_reduce_scatter; wider passes pad the partials to a multiple of
        // LANES_K (little padding there, and it fits the 168-register budget)
        constexpr int NR = RH * CT;
        constexpr bool kMinPad = NT <= 4;
        constexpr int NV = kMinPad ? NR : (NR + LANES_K - 1) / LANES_K * LANES_K;
        TA v[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) v[j] = j < NR ? acc[j / CT][j % CT] : TA(0);
        int jb = 0, nreal = NV;
        bool dup = false;
        if constexpr (kMinPad) {
          ws_reduce_scatter<TA, NR, LANES_T>(v, lane, jb, dup, nreal);
        } else {
#pragma unroll
          for (int o = LANES_T, ns = NV / 2; o < 32; o <<= 1, ns >>= 1) {
            const bool upper = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < ns; ++i) {
              const TA send = upper ? v[i] : v[i + ns];
              const TA keep = upper ? v[i + ns] : v[i];
              v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
          }
          // lane bits (LANES_T, 2 LANES_T, ...) chose offsets (NV/2, NV/4, ...)
#pragma unroll
          for (int o = LANES_T, ns = NV / 2; o < 32; o <<= 1, ns >>= 1) jb += (lane & o) ? ns : 0;
        }
        constexpr int NF = kMinPad ? ws_rs_final<NR, LANES_T>() : NV / LANES_K;
        const int rb = NRED == 2 ? (int)(pass & 1) : 0;
        const uint32_t rph = (NRED == 2 ? pass >> 1 : pass) & 1;
        TA* redb = red + rb * red_elems;
        mbar_wait(&redempty[rb], rph ^ 1);
#pragma unroll
        for (int i = 0; i < NF; ++i) {
          const int j = jb + i;
          if (!dup && i < nreal && j < NR) {
            const int r = j / CT, ct = j - (j / CT) * CT;
            redb[((size_t)kg * Rpad + rbase + r) * NT + tq + LANES_T * ct] = v[i];
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&redfull[rb]);
      }
    }
  }
}

}  // namespace rnnb
