// Tensor-core (tcgen05 + TMEM + TMA) blocked SRU/QRNN layer kernel, sm_100a.
//
// Reference path: rnnblock run_blocked (blocked.py:221-268) with the block
// projection precompute_gates_* (blocked.py:123-150), the c-sweep
// (blocked.py:153-176) and finalize_outputs (blocked.py:179-193) fused.
//
// Work item = (unit tile u of 128 hidden units, time block b of T_b steps).
// For one item the CTA computes, per gate g in {cand, forget, out/highway},
//     P_g[128 x N] = W_g[u-tile, :] . X_block^T          (N = T_b padded to 16)
// with K = taps*D: the QRNN x_{t-1} tap multiplies the SAME x tile fetched one
// row earlier (row -1 is zero-filled by TMA), exactly Xprev of blocked.py:143.
// The three accumulators live in TMEM (3*N columns, double-buffered when
// they fit) and never touch HBM; the epilogue warps read them with
// tcgen05.ld (thread = TMEM lane = hidden unit), apply bias/activations, run
// the sequential c-scan over the block and write h.
//
// Items are processed time-block-major by a persistent grid, so different
// time blocks' projections run concurrently on different SMs (the weights of
// a layer stay L2-resident and are re-read once per block, the reference's
// "one weight fetch per block" model); only the cheap scan is chained: the
// epilogue of (u, b) composes the carry maps earlier blocks of the same unit
// published (decoupled look-back, tc_lookback: the value is the flag).  Items
// are claimed in increasing order and every dependency points to a smaller
// item, so with all CTAs co-resident the chain cannot deadlock.
//
// Roles: warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer (the
// converged warp; elect.sync picks the issuing lane), then epilogue groups of
// four warps (TMEM lane quadrant w%4): one group (192 threads) for 3xTF32, two
// groups taking alternate items (320 threads) for bf16 / tf32.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "ffma_ws.cuh"  // mbarrier / TMA helpers

namespace rnnb {

// TC_3XTF32: fp32-accurate split products on the tf32 pipe,
//   a.b ~= a_hi.b_hi + a_hi.b_lo + a_lo.b_hi  (hi = tf32(x), lo = tf32(x - hi))
enum TcMode : int { TC_BF16 = 0, TC_TF32 = 1, TC_3XTF32 = 2 };

struct TcArgs {
  const float* Xhw;   // SRU highway source x (fp32, raw), row stride ldhw
  int64_t ldhw;
  float* Hout;        // fp32 h [L][ldh]
  int64_t ldh;        // may be negative (rows stored in reverse time order)
  float* Hpeer[kMaxPeers];  // same layout as Hout on peer GPUs (mapped), npeer used
  int npeer;
  void* Hop;          // optional MMA-operand copy of h for the next layer (bf16 or tf32-rounded f32), [L][ldop]
  int64_t ldop;
  const float* bias;  // SRU [Hpad][2] (b_forget, b_highway) or nullptr
  const float* c_in;  // [H] c_0 (nullptr: zeros); never written by the launch
  float* c_out;       // [H] c_T (nullptr: not written); must not alias c_in
  int epoch;          // this launch's tag of the split-last-wave flags (fixflag holds 4*epoch + 3):
                      // values of earlier launches read as "none"
  // look-back state, "the value is the flag": the launch's predecessor (the
  // operand conversion, or a memset) fills both arrays with kLbSentinel bits
  // (a NaN pattern the publishers never store), a published value is whatever
  // differs from it
  unsigned long long* agg;  // [nB][Hpad] block carry map c_out = A c_in + B as the pair (A, B)
  unsigned int* incl;       // [nB][Hpad] c after the block (inclusive prefix), fp32 bits
  int64_t L;
  int T_b;
  int H, Hpad, D;
  int nK;             // k-tiles per row (taps * Dp / KT)
  int nKtap;          // k-tiles per tap
  int nU, nB;
  // streaming (rnnb_forward_host, single-layer stacks): the MMA operand rows
  // are converted while the kernel runs; *x_ready = operand rows resident
  // (sequence rows [0, *x_ready)), and each item, after its h rows are
  // stored, adds 1 to h_done[t0 / h_gran] (nullptr: not streaming)
  const int* x_ready;
  int* h_done;
  int h_gran;
  int* stream_fail;   // set when the input did not arrive in time (see wait_rows)
  // RNNB_STREAM_TRACE (tuning only): globaltimer stamps, [0] kernel start,
  // [1 + b] block b's rows seen resident (unit tile 0), [1 + nB + b] block b's
  // last unit tile stored
  unsigned long long* trace;
  // 3xTF32 only: items from split_start on (the last, partial wave) are
  // split in two halves on two CTAs (see tc_work); fix holds the first
  // halves' K-chunk sums [slot][3N][128], fixflag their release tags
  int split_start;
  float* fix;
  int* fixflag;
  int ck0;            // 3xTF32: k-tiles in each of an item's first two K chunks (x3_chunk_start)
  int egroups;        // epilogue warp groups in use (1 or 2; <= the kernel's EGROUPS; 0 = all)
  int dbg;            // RNNB_DEBUG bits, timing experiments only (results wrong): 16 no look-back,
                      // 32 no epilogue, 64 no MMAs, 128 no loads, 512 no scan/stores, 1024 no activations
};

template <int MODE> struct TcT;
template <> struct TcT<TC_BF16> {
  static constexpr int ES = 2;   // operand element bytes
  static constexpr int KT = 64;  // k-tile: 128 bytes = one SW128 row
  static constexpr int UK = 16;  // K per tcgen05.mma (kind::f16)
  static constexpr uint32_t FMT = 1;  // BF16
};
template <> struct TcT<TC_TF32> {
  static constexpr int ES = 4;
  static constexpr int KT = 32;
  static constexpr int UK = 8;   // K per tcgen05.mma (kind::tf32)
  static constexpr uint32_t FMT = 2;  // TF32
};
template <> struct TcT<TC_3XTF32> : TcT<TC_TF32> {};

constexpr int kTcThreads = 192;
constexpr int kLB = 32;  // look-back depth (aggregates composed per block)

// ---- tcgen05 wrappers (PTX ISA 8.7, sm_100a) ----
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst_smem)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// D[tmem] (+)= A[smem desc] . B[smem desc]^T, kind selected by MODE
template <int MODE>
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  if (MODE == TC_BF16)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
// arrive on an mbarrier once all previously issued tcgen05.mma have completed
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
// ---- one k-tile of MMAs as ONE asm block, executed by the whole (converged)
// MMA warp with elect.sync inside: the descriptors are warp-uniform, so ptxas
// issues the UTCHMMAs back to back from uniform registers.  Issued from a
// lane-0-only branch, each MMA sat in an ELECT/BRA.U.ANY loop with dependent
// uniform-register moves: 82 cycles per 128xNx16 MMA vs 56 this way
// (tools/mma_rate.cu, profiles/mma_rate_r2.json; the hardware floor is ~51
// cycles for any N <= 64).  Gate g: A tile a0 + g*16 KB, accumulator d0 + g*N;
// K-step kk: start address + 32 B.  acc == 0 starts the accumulation.
#define RNNB_MMA(KIND, ACCP) "@e tcgen05.mma.cta_group::1.kind::" KIND " [d], a, b, %3, " ACCP ";\n\t"
#define RNNB_KSTEP(KIND) "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t" RNNB_MMA(KIND, "1")
#define RNNB_GATE(KIND, G)                                                                        \
  "add.s64 a, %1, " #G "*1024;\n\tmov.b64 b, %2;\n\tmad.lo.s32 d, %5, " #G ", %0;\n\t" RNNB_MMA(KIND, "p") \
      RNNB_KSTEP(KIND) RNNB_KSTEP(KIND) RNNB_KSTEP(KIND)
#define RNNB_KTILE(KIND)                                                                            \
  "{\n\t.reg .pred p, e;\n\t.reg .b64 a, b;\n\t.reg .b32 d;\n\telect.sync _|e, 0xffffffff;\n\t" \
  "setp.ne.b32 p, %4, 0;\n\t" RNNB_GATE(KIND, 0) RNNB_GATE(KIND, 1) RNNB_GATE(KIND, 2) "}\n"
// 3xTF32 in TWO MMAs per gate and K-step instead of three: the x tile holds
// [x_hi ; x_lo] as 2N rows, so W_hi . [x_hi | x_lo] is ONE N' = 2N MMA (idesc
// %3) writing hi.hi to accumulator columns [0, N) and hi.lo to [N, 2N); then
// W_lo . x_hi (N columns, idesc %6) accumulates into [N, 2N).  The issue floor
// is ~51 cycles per MMA for any N <= 64, so this is 1.5x fewer issue slots;
// the epilogue adds the two column halves.  W_lo = W_hi + 3 tiles (%5 =
// 3*16 KB in 16-byte units); gate g: accumulator d0 + 2N*g (%7 = 2N).
#define RNNB_X3STEP(ACCP)                                                          \
  "@e tcgen05.mma.cta_group::1.kind::tf32 [d], a, b, %3, " ACCP ";\n\t"           \
  "add.s64 al, a, %5;\n\t@e tcgen05.mma.cta_group::1.kind::tf32 [dc], al, b, %6, 1;\n\t"
#define RNNB_X3NEXT "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t" RNNB_X3STEP("1")
#define RNNB_X3GATE(G)                                                                            \
  "add.s64 a, %1, " #G "*1024;\n\tmov.b64 b, %2;\n\tmad.lo.s32 d, %7, " #G ", %0;\n\t"         \
  "shr.u32 dc, %7, 1;\n\tadd.s32 dc, d, dc;\n\t" RNNB_X3STEP("p") RNNB_X3NEXT RNNB_X3NEXT RNNB_X3NEXT
template <int MODE>
__device__ __forceinline__ void tc_issue_ktile(uint32_t d0, uint64_t a0, uint64_t b0, uint32_t idesc, uint32_t acc,
                                               uint32_t n, uint32_t idesc_n, uint64_t lo16) {
  if constexpr (MODE == TC_BF16)
    asm volatile(RNNB_KTILE("f16") ::"r"(d0), "l"(a0), "l"(b0), "r"(idesc), "r"(acc), "r"(n));
  else if constexpr (MODE == TC_TF32)
    asm volatile(RNNB_KTILE("tf32") ::"r"(d0), "l"(a0), "l"(b0), "r"(idesc), "r"(acc), "r"(n));
  else  // idesc: N' = 2n (W_hi . [x_hi | x_lo]); idesc_n: N = n (W_lo . x_hi)
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 a, b, al;\n\t.reg .b32 d, dc;\n\telect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t" RNNB_X3GATE(0) RNNB_X3GATE(1) RNNB_X3GATE(2) "}\n" ::"r"(d0),
        "l"(a0), "l"(b0), "r"(idesc), "r"(acc), "l"(lo16), "r"(idesc_n), "r"(2 * n));
}
// One 3xTF32 k-tile on the fine-grained ring as ONE asm block: the three
// gates' W slots are consecutive (32 KB = 2048 sixteen-byte units apart, W_lo
// 16 KB after W_hi), and each gate's slot is RELEASED by its own commit right
// after its 8 MMAs (empty barriers 8 B apart), the x slot after the last
// gate.  Per gate: 4 K-steps x (W_hi . [x_hi | x_lo] into [d, d+2N), then
// W_lo . x_hi into [d+N, d+2N)).  One block per k-tile, not per gate: every
// asm block costs ptxas ~60 uniform-datapath instructions of operand set-up
// that the tensor pipe's short queue does not hide (per-gate blocks: MMA-only
// time 151 -> 189 us on cfg2).  Releasing in two halves of three tiles (one
// mid-stream commit instead of three) was measured too: 201 vs 198 us -- the
// finer release is worth more than the commits cost.
#define RNNB_G3STEP(ACCP)                                                   \
  "@e tcgen05.mma.cta_group::1.kind::tf32 [d], a, b, %3, " ACCP ";\n\t"     \
  "add.s64 al, a, 1024;\n\t@e tcgen05.mma.cta_group::1.kind::tf32 [dc], al, b, %6, 1;\n\t"
#define RNNB_G3NEXT "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t" RNNB_G3STEP("1")
#define RNNB_G3GATE(G)                                                                               \
  "add.s64 a, %1, " #G "*2048;\n\tmov.b64 b, %2;\n\tmad.lo.s32 d, %8, " #G ", %0;\n\tadd.s32 dc, d, %5;\n\t" \
  RNNB_G3STEP("p") RNNB_G3NEXT RNNB_G3NEXT RNNB_G3NEXT                                               \
  "add.s32 eb, %7, " #G "*8;\n\t"                                                                    \
  "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [eb];\n\t"
__device__ __forceinline__ void tc_issue_ktile_x3_fine(uint32_t d0, uint64_t a0, uint64_t b0, uint32_t idesc_2n,
                                                       uint32_t acc, uint32_t n, uint32_t idesc_n, uint32_t emptyw0,
                                                       uint32_t gcols, uint32_t emptyx) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 a, b, al;\n\t.reg .b32 d, dc, eb;\n\telect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t" RNNB_G3GATE(0) RNNB_G3GATE(1) RNNB_G3GATE(2)
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%9];\n\t}\n" ::"r"(d0),
      "l"(a0), "l"(b0), "r"(idesc_2n), "r"(acc), "r"(n), "r"(idesc_n), "r"(emptyw0), "r"(gcols), "r"(emptyx)
      : "memory");
}
#undef RNNB_G3STEP
#undef RNNB_G3NEXT
#undef RNNB_G3GATE
#undef RNNB_MMA
#undef RNNB_KSTEP
#undef RNNB_GATE
#undef RNNB_KTILE
#undef RNNB_X3STEP
#undef RNNB_X3NEXT
#undef RNNB_X3GATE
// tcgen05.commit from the converged MMA warp, one elected lane
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
// 32 lanes x 32 bit, 16 consecutive columns -> 16 registers per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// tcgen05.ld without the wait: issue several, then one tmem_wait_ld() and a
// reg_fence per destination array (the empty volatile asm "redefines" the
// registers after the wait, so no use can be scheduled before it)
__device__ __forceinline__ void tmem_ld16_raw(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void reg_fence(uint32_t (&r)[16]) {
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]));
}
// the three gate accumulators of 16 columns, one wait
__device__ __forceinline__ void tmem_ld_gates16(uint32_t tz, uint32_t tf, uint32_t to, float (&z)[16], float (&f)[16],
                                                float (&o)[16]) {
  uint32_t rz[16], rf[16], ro[16];
  tmem_ld16_raw(tz, rz);
  tmem_ld16_raw(tf, rf);
  tmem_ld16_raw(to, ro);
  tmem_wait_ld();
  reg_fence(rz);
  reg_fence(rf);
  reg_fence(ro);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    z[i] = __uint_as_float(rz[i]);
    f[i] = __uint_as_float(rf[i]);
    o[i] = __uint_as_float(ro[i]);
  }
}

// K-major, 128-byte-swizzled operand tile (rows of 128 B, 8-row atoms 1 KB apart)
__device__ __forceinline__ uint64_t sw128_desc(const void* smem_tile) {
  const uint64_t addr = smem_u32(smem_tile);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;        // start address
  d |= (uint64_t)1 << 16;              // leading byte offset (ignored for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;    // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1 << 46;              // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;              // layout: SWIZZLE_128B
  return d;
}

template <int MODE>
__host__ __device__ constexpr uint32_t tc_idesc(int M, int N) {
  return (1u << 4)                      // D format F32
         | (TcT<MODE>::FMT << 7)        // A format
         | (TcT<MODE>::FMT << 10)       // B format
         | ((uint32_t)(N >> 3) << 17)   // N / 8
         | ((uint32_t)(M >> 4) << 24);  // M / 16
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ float ld_cg(const float* p) {
  float v;
  asm volatile("ld.global.cg.f32 %0, [%1];\n" : "=f"(v) : "l"(p) : "memory");
  return v;
}
// Branch-free tanh for the epilogue.  |x| >= 0.4: 1 - 2 / (e^{2|x|} + 1) on
// MUFU ex2 / rcp (|x| clamped at 15, where tanh rounds to 1 in fp32), relative
// error <= ~4e-7.  |x| < 0.4: the odd Taylor polynomial to x^13 (truncation
// 4e-9 relative; 6e-8 measured in fp32), because the exp form's ~2e-7
// ABSOLUTE error is a large RELATIVE error for small |x|, and deep stacks
// drive the gate pre-activations and c toward 0 (cfg4: the output scale
// shrinks ~3x per layer, so layer 8 saw 1.7e-3 normwise error vs the
// rounded-operand oracle before this select; the FFMA path's tanhf saw
// none).  Both halves are computed and selected: the library tanhf branches
// on |x| and, with one epilogue warp per scheduler, its dependent MUFU chain
// made the epilogue latency-bound.
__device__ __forceinline__ float tc_tanh(float x) {
  const float ax = fabsf(x);
  const float e = __expf(2.f * fminf(ax, 15.f));
  const float big = 1.f - __fdividef(2.f, e + 1.f);
  const float x2 = x * x;
  float p = 21844.f / 6081075.f;
  p = fmaf(p, x2, -1382.f / 155925.f);
  p = fmaf(p, x2, 62.f / 2835.f);
  p = fmaf(p, x2, -17.f / 315.f);
  p = fmaf(p, x2, 2.f / 15.f);
  p = fmaf(p, x2, -1.f / 3.f);
  const float small = fmaf(p * x2, ax, ax);
  return copysignf(ax < 0.4f ? small : big, x);
}
// 1 / (1 + e^{-z}): relative error a few ulp for every z (no cancellation;
// e^{-z} overflowing to inf gives 0, underflowing gives 1)
__device__ __forceinline__ float tc_sigmoid(float z) { return __fdividef(1.f, 1.f + __expf(-z)); }

// named barrier 2 over the four epilogue warps
__device__ __forceinline__ void tc_epi_sync(int eg = 0) { asm volatile("bar.sync %0, 128;\n" ::"r"(2 + eg) : "memory"); }

// Streaming output: once the 128 epilogue threads stored this item's h rows
// (ordered by the barrier), one gpu-scope fence and one count per item on
// the item's output granule; the host's copy-out stream waits until a
// granule holds nU x (its blocks) counts.
__device__ __forceinline__ void tc_count_done(const TcArgs& a, int64_t t0, int et, int eg = 0) {
  if (a.trace && et == 0) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    atomicMax(&a.trace[1 + a.nB + (int)(t0 / a.T_b)], now);
  }
  if (a.h_done == nullptr) return;
  tc_epi_sync(eg);
  if (et == 0) {
    __threadfence();
    atomicAdd(&a.h_done[t0 / a.h_gran], 1);
  }
}

// Decoupled look-back, "the value is the flag".  Publish block b's AGGREGATE
// carry map (A, B) as ONE 8-byte store, fetch the aggregates of blocks b-1 ..
// b-kLB of the same unit (and the INCLUSIVE carry of block b-kLB-1, or c_0) --
// each a single-copy-atomic load that is re-issued while it still returns the
// sentinel the arrays were filled with before the launch -- compose them in
// FIXED order (timing never changes the arithmetic: results are run-to-run
// and chunking / GPU-count invariant), publish block b's inclusive carry and
// return c_in.  Every thread works on its own unit: no barrier, no fence, no
// status word; a ready predecessor costs one L2 round trip.  (The first
// version published per-tile status words: store, barrier, release, 32 lanes
// polling with acquires, barrier, loads -- three L2 round trips and two
// barriers on every item's critical path: 14-26 % of a cfg2 bf16 launch at
// T_b = 64-16.)  Real NaNs are re-coded so they can never equal the sentinel.
constexpr unsigned int kLbSentinel = 0xFFFFFFFFu;
__device__ __forceinline__ unsigned int lb_bits(float v) {
  const unsigned int u = __float_as_uint(v);
  return u == kLbSentinel ? 0x7FC00000u : u;
}
__device__ __forceinline__ unsigned long long lb_load64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned int lb_load32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float tc_lookback(const TcArgs& a, int b, int u, int unit, int et, float Ablk,
                                             float Bblk) {
  (void)u;
  (void)et;
  const size_t sidx = (size_t)b * a.Hpad + unit;
  const unsigned long long mine = (unsigned long long)lb_bits(Ablk) | ((unsigned long long)lb_bits(Bblk) << 32);
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;\n" ::"l"(a.agg + sidx), "l"(mine) : "memory");
  const int jlo = b - kLB > 0 ? b - kLB : 0;  // oldest aggregate used
  // all kLB loads (and the anchor) in flight at once, constant register
  // indices; identity maps (A = 1, B = 0) past jlo leave the composed map
  // bitwise unchanged (x*1 and fma(x, 0, y) are exact)
  constexpr unsigned long long kPair = ((unsigned long long)kLbSentinel << 32) | kLbSentinel;
  unsigned long long pj[kLB];
#pragma unroll
  for (int k = 0; k < kLB; ++k) {
    const int j = b - 1 - k;
    pj[k] = j >= jlo ? lb_load64(a.agg + (size_t)j * a.Hpad + unit) : 0ull;
  }
  unsigned int anc = 0;
  if (jlo > 0) anc = lb_load32(a.incl + (size_t)(jlo - 1) * a.Hpad + unit);
#pragma unroll
  for (int k = 0; k < kLB; ++k) {
    const int j = b - 1 - k;
    if (j >= jlo)
      while (pj[k] == kPair) pj[k] = lb_load64(a.agg + (size_t)j * a.Hpad + unit);
  }
  if (jlo > 0)
    while (anc == kLbSentinel) anc = lb_load32(a.incl + (size_t)(jlo - 1) * a.Hpad + unit);
  const float anchor = jlo > 0 ? __uint_as_float(anc) : (a.c_in != nullptr && unit < a.H ? a.c_in[unit] : 0.f);
  float Aacc = 1.f, Bacc = 0.f;  // map from c after block jlo-1 to c after block b-1
#pragma unroll
  for (int k = 0; k < kLB; ++k) {
    const bool v = b - 1 - k >= jlo;
    const float Aj = v ? __uint_as_float((unsigned int)pj[k]) : 1.f;
    const float Bj = v ? __uint_as_float((unsigned int)(pj[k] >> 32)) : 0.f;
    Bacc = Aacc * Bj + Bacc;
    Aacc = Aacc * Aj;
  }
  const float cin = Aacc * anchor + Bacc;
  // the INCLUSIVE carry is only ever read as the anchor of block b+kLB+1
  if (b + kLB + 1 < a.nB)
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;\n" ::"l"(a.incl + sidx), "r"(lb_bits(Ablk * cin + Bblk))
                 : "memory");
  return cin;
}

#ifndef RNNB_X3_CK
#define RNNB_X3_CK 8  // 3xTF32 K chunk in k-tiles (8 x 32 = 256-deep; 128-deep: 8 % slower, half the error)
#endif
// 3xTF32 chunk plan of an item's nK k-tiles: two chunks of ck0 k-tiles, then
// chunks of CK (ck0 = TcArgs::ck0, chosen by the host).  While the epilogue
// warps finish an item (activations, look-back, scan, stores) the MMA warp
// can run only two chunks of the next item ahead (two TMEM buffers; TMEM is
// full), and every chunk costs the epilogue a TMEM read + add pass.
//  * Short reductions (nK <= 32, i.e. K <= 1024: cfg3): ck0 = 16 -- an item is
//    two 512-deep chunks instead of four 256-deep ones: cfg3 f32 T_b = 32
//    1.81 -> 1.30 ms, T_b = 8 4.44 -> 3.97 ms; the total depth is small, so
//    the accumulation error stays low (cfg3 logits within the fp32 bound).
//  * Long reductions (cfg2, cfg4): ck0 = CK = 8.  Longer first chunks there
//    were measured: 12: 1.6 % faster, 25 % more error; 16: slower (207 vs
//    198 us) and cfg4's 8-layer error 4.2e-6 -> 5.4e-6 -- not adopted.
__host__ __device__ __forceinline__ int x3_chunk_start(int c, int ck0) {
  return c <= 2 ? c * ck0 : 2 * ck0 + (c - 2) * RNNB_X3_CK;
}
__host__ __device__ __forceinline__ int x3_chunk_of(int kt, int ck0) {
  return kt < 2 * ck0 ? kt / ck0 : 2 + (kt - 2 * ck0) / RNNB_X3_CK;
}
__host__ __device__ __forceinline__ int x3_nchunks(int nK, int ck0) { return x3_chunk_of(nK - 1, ck0) + 1; }
__host__ __device__ __forceinline__ int x3_pick_ck0(int nK) { return nK <= 32 ? 16 : RNNB_X3_CK; }

template <int MODE, int N, int EG = 1>
struct TcCfg {
  static constexpr int ES = TcT<MODE>::ES, KT = TcT<MODE>::KT, UK = TcT<MODE>::UK;
  static constexpr int A_BYTES = 128 * 128;  // one gate tile: 128 rows x 128 B
  static constexpr int B_BYTES = N * 128;
  static constexpr int SPLIT = MODE == TC_3XTF32 ? 2 : 1;  // hi (+ lo) planes per operand
  // stage layout: A tiles [plane][gate] (plane 0 = hi), then the x tile of
  // every plane stacked as ONE B tile of SPLIT*N rows ([x_hi ; x_lo]: the
  // 3xTF32 MMA W_hi . [x_hi | x_lo] reads both planes as N' = 2N columns)
  static constexpr int B_OFF = SPLIT * 3 * A_BYTES;
  static constexpr int STAGE_BYTES = SPLIT * (3 * A_BYTES + B_BYTES);
  static constexpr int STAGES = (4 * STAGE_BYTES + 2048 <= 227 * 1024)   ? 4
                                : (3 * STAGE_BYTES + 2048 <= 227 * 1024) ? 3
                                                                          : 2;
  // accumulator columns per gate: N, or for 3xTF32 2N ([hi.hi | hi.lo + lo.hi])
  static constexpr int GCOLS = (MODE == TC_3XTF32 ? 2 : 1) * N;
  static constexpr int ACC_COLS = 3 * GCOLS;
  // accumulator buffers in TMEM: up to 4 for the non-chunked modes (N <= 32:
  // the MMA warp runs up to three items ahead of an epilogue held up in the
  // look-back), 2 for 3xTF32 (alternating K chunks) and N = 64
  static constexpr int NACC = MODE == TC_3XTF32 ? 2 : (4 * ACC_COLS <= 512) ? 4 : (2 * ACC_COLS <= 512) ? 2 : 1;
  // 3xTF32: the tensor cores' fp32 accumulation error grows linearly with the
  // reduction length (measured), so K is accumulated in CK-k-tile chunks
  // (K = 128) in alternating TMEM buffers and the chunk partials are summed
  // in fp32 registers by the epilogue (keeps 3xTF32 inside the fp32 bound)
  static constexpr bool CHUNKED = MODE == TC_3XTF32;
  static constexpr int CK = RNNB_X3_CK;
  static_assert(!CHUNKED || (N <= 32 && NACC == 2), "chunked accumulation keeps 3N partials in registers");
  // 3xTF32: 3N more columns stash the first half's chunk sum (see the epilogue)
  static constexpr int USED_COLS = NACC * ACC_COLS + (CHUNKED ? 3 * N : 0);
  static constexpr int TMEM_COLS = (USED_COLS <= 32) ? 32 : (USED_COLS <= 64) ? 64
                                   : (USED_COLS <= 128) ? 128 : (USED_COLS <= 256) ? 256 : 512;
  static_assert(USED_COLS <= 512, "TMEM holds 512 columns");
  // 3xTF32: FINE-grained ring.  A 104 KB stage (both planes of a k-tile) left
  // room for two stages only, and a stage is refilled only after ALL its 24
  // MMAs: half the buffer was idle while the other half was read, and the
  // L2 feed (which, like the MMA issue, needs ~0.65 us per k-tile) could not
  // overlap it (loads + MMAs 199 us vs 152 us for either alone on cfg2).  Now
  // a W slot holds one gate's hi + lo tiles (32 KB, freed after that gate's 8
  // MMAs) and the x tiles ([x_hi ; x_lo], shared by the three gates) have
  // their own small ring.
  // Epilogue warp groups.  The non-chunked modes run TWO groups of four warps
  // that take alternate items (each on its own TMEM buffers): with short
  // reductions (cfg3's K = 1024: 5 us of MMAs per item) one group's ~5 us per
  // item was the bottleneck (cfg3 bf16 T_b = 8 1.41 -> 1.02 ms, tf32 T_b = 32
  // 0.79 -> 0.57 ms); possible since the look-back needs no barrier across a
  // group's items any more.  Where the MMA stream bounds an item (cfg2's K =
  // 2048) the second group gains nothing or costs a few % (tf32 T_b = 64), so
  // the host picks the one- or the two-group kernel per launch
  // (TcArgs::egroups; a 320-thread kernel with the second group idle still
  // cost cfg2 bf16 3 % at T_b = 8-16).  3xTF32 keeps one group (its 254
  // registers per thread do not fit 320 threads).
  static constexpr int EGROUPS = CHUNKED ? 1 : EG;  // (EG: template parameter, two kernel variants)
  static constexpr int THREADS = 64 + 128 * EGROUPS;
  static constexpr bool FINE = CHUNKED;
  static constexpr int W_SLOT = 2 * A_BYTES;
  static constexpr int X_SLOT = SPLIT * B_BYTES;
  static constexpr int NW = 6;
  static constexpr int NX = (227 * 1024 - 2048 - NW * W_SLOT) / X_SLOT < 4 ? (227 * 1024 - 2048 - NW * W_SLOT) / X_SLOT : 4;
  static_assert(!FINE || NX >= 2, "x ring too small");
  static constexpr int RING_BYTES = FINE ? NW * W_SLOT + NX * X_SLOT : STAGES * STAGE_BYTES;
  static constexpr int NFULL = FINE ? NW + NX : STAGES;  // full barriers (then as many empty ones)
  static constexpr size_t SMEM = (size_t)RING_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static_assert(2 * NFULL * 8 + 64 + 8 <= 256, "barrier area");
};

// This CTA's k-th unit of work.  Whole items blockIdx.x + k*grid below
// a.split_start (round-robin, time-block-major, as before); then, when the
// last wave is split (3xTF32 only; the host guarantees 2R <= grid for its R
// items), one half of a last-wave item: part 0 = K chunks [0, nch/2) whose
// sum goes to the fixup buffer, part 1 = chunks [nch/2, nch), which finishes
// the item.  Every item -- split or not -- sums its chunks as
// S = (chunks [0, nch/2)) + (chunks [nch/2, nch)), so the split never
// changes a bit of the result and any grid gives the same numbers.
struct TcWork {
  int item, kt0, kt1, part;  // part: -1 whole item, 0 / 1 halves
};
template <int CK>
__device__ __forceinline__ bool tc_work(const TcArgs& a, int nitems, int k, TcWork& w) {
  const int bx = blockIdx.x, G = gridDim.x;
  const int nwhole = a.split_start > bx ? (a.split_start - bx + G - 1) / G : 0;
  if (k < nwhole) {
    w = TcWork{bx + k * G, 0, a.nK, -1};
    return true;
  }
  if (k == nwhole && a.split_start < nitems && bx < 2 * (nitems - a.split_start)) {
    const int kmid = x3_chunk_start(x3_nchunks(a.nK, a.ck0) / 2, a.ck0);
    const int part = bx & 1;
    w = TcWork{a.split_start + bx / 2, part ? kmid : 0, part ? a.nK : kmid, part};
    return true;
  }
  return false;
}

template <int CELL, int MODE, int N, int EG = 1>
__global__ void __launch_bounds__((TcCfg<MODE, N, EG>::THREADS), 1)
    tc_layer_kernel(TcArgs a, const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX) {
  using C = TcCfg<MODE, N, EG>;
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  unsigned char* tsm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  // FINE: full = [W slots | x slots], empty likewise
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm + (size_t)C::RING_BYTES);
  uint64_t* empty = full + C::NFULL;
  uint64_t* acc_full = empty + C::NFULL;
  uint64_t* acc_empty = acc_full + 4;
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(acc_empty + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nitems = a.nU * a.nB;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NFULL; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < C::NACC; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) tmem_alloc(tmem_base_smem, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_base_smem;
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
  }
  // launched with programmatic stream serialization: everything above ran
  // while the previous kernel in the stream finished; its writes (the x
  // operand, the look-back state, the previous layer's h) are visible after this
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      uint32_t it = 0;
      uint64_t t_start = 0;
      int rows_seen = 0;
      bool timed_out = false;
      if (a.x_ready) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
      TcWork w;
      for (int k = 0; tc_work<C::CK>(a, nitems, k, w); ++k) {
        const int item = w.item;
        const int b = item / a.nU, u = item - (item / a.nU) * a.nU;
        const int t0 = b * a.T_b;
        if (a.x_ready && !timed_out) {
          // streaming input: this block's operand rows must be resident
          // before the first x tile of the item is fetched (rows already
          // seen need no new acquire round trip)
          const int need = (int)((t0 + N) < a.L ? (t0 + N) : a.L);
          while (rows_seen < need) {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(rows_seen) : "l"(a.x_ready) : "memory");
            if (rows_seen >= need) break;
            uint64_t now;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            if (now - t_start > kStreamTimeoutNs) {  // profiler serialising the streams: give up (host redoes)
              atomicExch(a.stream_fail, 1);
              timed_out = true;
              break;
            }
            __nanosleep(64);
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");  // TMA reads after the acquire
          if (a.trace && u == 0 && w.part != 1) {
            unsigned long long now;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            a.trace[1 + b] = now;
            if (item == 0) a.trace[0] = t_start;
          }
        }
        if constexpr (C::FINE) {
          // ONE full barrier per k-tile (ring of two: k-tile parity) counts the
          // bytes of its x slot and its three W slots -- the MMA warp waits
          // once per k-tile (four waits per k-tile left the tensor pipe's
          // short queue dry: MMA-only time 151 -> 182 us); the slots are
          // still loaded one by one, as soon as each is released
          for (int kt = w.kt0; kt < w.kt1; ++kt, ++it) {
            const int tap = kt >= a.nKtap ? 1 : 0;
            const int kx = (kt - tap * a.nKtap) * C::KT;
            const int xs = it % C::NX;
            uint64_t* fk = &full[it & 1];
            mbar_wait(&empty[C::NW + xs], ((it / C::NX) & 1) ^ 1);
            // the k-tile's first W slot is free only after the MMA warp has
            // passed this barrier's previous phase (k-tile it-2): arm it after
            // that wait, never twice in one phase
            mbar_wait(&empty[(it & 1) * 3], ((it >> 1) & 1) ^ 1);
            unsigned char* xt = tsm + C::NW * C::W_SLOT + (size_t)xs * C::X_SLOT;
            if (!(a.dbg & 128)) {
              mbar_arrive_expect_tx(fk, C::X_SLOT + 3 * C::W_SLOT);
#pragma unroll
              for (int p = 0; p < C::SPLIT; ++p)
                tma_load_2d(xt + p * C::B_BYTES, &tmX, kx, (int)(p * (a.L + 1)) + t0 + 1 - tap, fk);
            }
            for (int g = 0; g < 3; ++g) {
              const int ws = (it & 1) * 3 + g;
              if (g > 0) mbar_wait(&empty[ws], ((it >> 1) & 1) ^ 1);
              unsigned char* wt = tsm + (size_t)ws * C::W_SLOT;
              if (a.dbg & 128) continue;
#pragma unroll
              for (int p = 0; p < C::SPLIT; ++p)
                tma_load_2d(wt + p * C::A_BYTES, &tmW, kt * C::KT, (p * 3 + g) * a.Hpad + u * 128, fk);
            }
            if (a.dbg & 128) mbar_arrive(fk);  // timing experiment: no loads
          }
          continue;
        }
        for (int kt = w.kt0; kt < w.kt1; ++kt, ++it) {
          const int s = it % C::STAGES;
          // plain try_wait (the instruction suspends in hardware): a
          // nanosleep back-off here overshot the stage release by up to ~1 us
          // with each stage's MMAs taking ~0.3 us, starving the ring
          mbar_wait(&empty[s], ((it / C::STAGES) & 1) ^ 1);
          unsigned char* st = tsm + (size_t)s * C::STAGE_BYTES;
          if (a.dbg & 128) {  // timing experiment: no loads (MMAs read stale tiles)
            mbar_arrive(&full[s]);
            continue;
          }
          mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
          const int tap = kt >= a.nKtap ? 1 : 0;
          const int kx = (kt - tap * a.nKtap) * C::KT;
#pragma unroll
          for (int p = 0; p < C::SPLIT; ++p) {  // hi plane, then lo plane (3xTF32)
            for (int g = 0; g < 3; ++g)
              tma_load_2d(st + (p * 3 + g) * C::A_BYTES, &tmW, kt * C::KT, (p * 3 + g) * a.Hpad + u * 128,
                          &full[s]);
            // operand row r holds x_{r-1}: block rows t0.. for tap 0, t0-1.. for tap 1
            tma_load_2d(st + C::B_OFF + p * C::B_BYTES, &tmX, kx, (int)(p * (a.L + 1)) + t0 + 1 - tap, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: the whole warp, one elected lane issues ----------------
    {
      constexpr uint32_t idesc = tc_idesc<MODE>(128, N);
      static_assert(C::A_BYTES == 16384 && C::KT / C::UK == 4 && (C::UK * C::ES) == 32,
                    "tc_issue_ktile hard-codes 16 KB gate tiles and 4 K-steps of 32 B");
      constexpr uint32_t idesc_n = tc_idesc<MODE>(128, N);
      constexpr uint32_t idesc_2n = tc_idesc<MODE>(128, C::SPLIT * N);  // 3xTF32: [x_hi | x_lo]
      uint32_t it = 0, acc_it = 0;
      TcWork w;
      for (int k = 0; tc_work<C::CK>(a, nitems, k, w); ++k) {
        int ab = acc_it % C::NACC;
        uint32_t dbase = tmem + ab * C::ACC_COLS;
        if (!C::CHUNKED) {
          mbar_wait(&acc_empty[ab], ((acc_it / C::NACC) & 1) ^ 1);
          tc_fence_after();
        }
        for (int kt = w.kt0; kt < w.kt1; ++kt, ++it) {
          const int kch = C::CHUNKED ? x3_chunk_of(kt, a.ck0) : 0;
          const int kc = C::CHUNKED ? kt - x3_chunk_start(kch, a.ck0) : kt;  // k-tile index inside the accumulation
          const bool kc_last = C::CHUNKED && (kt + 1 == x3_chunk_start(kch + 1, a.ck0) || kt == w.kt1 - 1);
          if (C::CHUNKED && kc == 0) {  // a new K-chunk accumulates into a fresh buffer
            ab = acc_it % C::NACC;
            dbase = tmem + ab * C::ACC_COLS;
            mbar_wait(&acc_empty[ab], ((acc_it / C::NACC) & 1) ^ 1);
            tc_fence_after();
          }
          if constexpr (C::FINE) {
            static_assert(C::NW == 6, "a k-tile's three W slots are consecutive: slots {0,1,2} / {3,4,5}");
            const int xs = it % C::NX;
            const int wb = (it & 1) * 3;  // first W slot of this k-tile
            const uint32_t wph = (it >> 1) & 1;
            mbar_wait(&full[it & 1], wph);
            tc_fence_after();
            if (a.dbg & 2048) {  // timing experiment: the old coarse issue block + software arrives (no per-gate commits)
              tc_issue_ktile<MODE>(dbase, sw128_desc(tsm + (size_t)wb * C::W_SLOT),
                                   sw128_desc(tsm + C::NW * C::W_SLOT + (size_t)xs * C::X_SLOT), idesc_2n, kc != 0, N,
                                   idesc_n, (uint64_t)(C::A_BYTES >> 4));
              if (lane == 0) {
                mbar_arrive(&empty[wb]);
                mbar_arrive(&empty[wb + 1]);
                mbar_arrive(&empty[wb + 2]);
              }
              __syncwarp();
              tc_commit_elect(&empty[C::NW + xs]);
            } else if (!(a.dbg & 64)) {
              tc_issue_ktile_x3_fine(dbase, sw128_desc(tsm + (size_t)wb * C::W_SLOT),
                                     sw128_desc(tsm + C::NW * C::W_SLOT + (size_t)xs * C::X_SLOT), idesc_2n, kc != 0, N,
                                     idesc_n, smem_u32(&empty[wb]), C::GCOLS, smem_u32(&empty[C::NW + xs]));
            } else {
              tc_commit_elect(&empty[wb]);
              tc_commit_elect(&empty[wb + 1]);
              tc_commit_elect(&empty[wb + 2]);
              tc_commit_elect(&empty[C::NW + xs]);
            }
            if (kc_last) {
              tc_commit_elect(&acc_full[ab]);  // this K-chunk's partial products complete
              ++acc_it;
            }
            continue;
          }
          const int s = it % C::STAGES;
          mbar_wait(&full[s], (it / C::STAGES) & 1);
          tc_fence_after();
          unsigned char* st = tsm + (size_t)s * C::STAGE_BYTES;
          if (!(a.dbg & 64))  // dbg 64 (timing): no MMAs
            tc_issue_ktile<MODE>(dbase, sw128_desc(st), sw128_desc(st + C::B_OFF),
                                 C::CHUNKED ? idesc_2n : idesc, kc != 0, N, idesc_n,
                                 (uint64_t)((3 * C::A_BYTES) >> 4));
          tc_commit_elect(&empty[s]);  // frees the smem stage once these MMAs have read it
          if (kc_last) {
            tc_commit_elect(&acc_full[ab]);  // this K-chunk's partial products complete
            ++acc_it;
          }
        }
        if (!C::CHUNKED) {
          tc_commit_elect(&acc_full[ab]);  // accumulators of this item complete
          ++acc_it;
        }
      }
    }
  } else {
    // ---------------- epilogue: 4 warps, thread = TMEM lane = unit ----------------
    // Per item: (A) activations for every step of the block, written back over
    // the accumulators with tcgen05.st, and the block's affine carry map
    // c_out = Ablk * c_in + Bblk (independent of earlier blocks) published as
    // an AGGREGATE; (B) decoupled look-back over earlier blocks' aggregates /
    // INCLUSIVE carries of the same unit tile to get c_in, then publish this
    // block's INCLUSIVE carry; (C) the sequential c-recurrence of the block from
    // c_in (blocked.py:153-162) and the output mix, h stores.
    const int q = warp & 3;                 // TMEM lane quadrant this warp may access
    const int row = q * 32 + lane;          // unit within the tile
    const int eg = (warp - 2) >> 2;         // epilogue group (takes items k = eg mod EGROUPS)
    const int et = threadIdx.x - 64 - eg * 128;  // 0..127 within the group
    // groups in use: the second one only pays where the epilogue, not the MMA
    // stream, bounds an item (short reductions, tiny blocks); the host decides
    const int neg = (a.egroups >= 1 && a.egroups < C::EGROUPS) ? a.egroups : C::EGROUPS;
    uint32_t acc_it = 0;
    TcWork w;
    for (int k = 0; eg < neg && tc_work<C::CK>(a, nitems, k, w); ++k) {
      if (C::EGROUPS > 1 && (k % neg) != eg) {  // the other group's item (one accumulator buffer each)
        ++acc_it;
        continue;
      }
      const int item = w.item;
      const int b = item / a.nU, u = item - (item / a.nU) * a.nU;
      const int64_t t0 = (int64_t)b * a.T_b;
      const int l = (int)((a.L - t0) < a.T_b ? (a.L - t0) : a.T_b);
      const int unit = u * 128 + row;
      if (a.dbg & 32) {  // timing experiment: epilogue only hands the accumulators back
        const int nacc = C::CHUNKED ? x3_chunk_of(w.kt1 - 1, a.ck0) - x3_chunk_of(w.kt0, a.ck0) + 1 : 1;
        for (int ch = 0; ch < nacc; ++ch, ++acc_it) {
          const int ab = acc_it % C::NACC;
          mbar_wait(&acc_full[ab], (acc_it / C::NACC) & 1);
          tc_fence_after();
          tc_fence_before();
          mbar_arrive(&acc_empty[ab]);
        }
        continue;
      }
      if constexpr (CELL == LINEAR && !C::CHUNKED) {
        // dense layer: gate plane g holds output columns [g*Hpad, (g+1)*Hpad);
        // accumulators + bias straight to Y (a warp stores 128 contiguous bytes per row)
        const int ab = acc_it % C::NACC;
        mbar_wait(&acc_full[ab], (acc_it / C::NACC) & 1);
        tc_fence_after();
        const uint32_t tb = tmem + ab * C::ACC_COLS + ((uint32_t)(q * 32) << 16);
#pragma unroll
        for (int g = 0; g < 3; ++g) {
          const int col = g * a.Hpad + unit;
          const bool live = col < a.H;
          const float bias = (live && a.bias) ? a.bias[col] : 0.f;
          float* yp = a.Hout + t0 * a.ldh + col;
          for (int c0 = 0; c0 < N && c0 < l; c0 += 16) {
            float v[16];
            tmem_ld16(tb + g * N + c0, v);
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (live && c0 + j < l) yp[(int64_t)(c0 + j) * a.ldh] = v[j] + bias;
          }
        }
        tc_fence_before();
        mbar_arrive(&acc_empty[ab]);
        ++acc_it;
        continue;
      }
      float bf = 0.f, br = 0.f;
      if (CELL == SRU && a.bias) {
        bf = a.bias[(size_t)unit * 2];
        br = a.bias[(size_t)unit * 2 + 1];
      }
      float Ablk = 1.f, Bblk = 0.f;
      if constexpr (C::CHUNKED) {
        // sum the K-chunk partials in fp32 registers, then all phases from registers
        float rz[N], rf[N], ro[N];
#pragma unroll
        for (int j = 0; j < N; ++j) rz[j] = rf[j] = ro[j] = 0.f;
        const int nch = x3_nchunks(a.nK, a.ck0);
        const int hch = nch / 2;  // first chunk of the second half (see tc_work)
        const int c_lo = w.part == 1 ? hch : 0, c_hi = w.part == 0 ? hch : nch;
        // the first half's sum waits in TMEM columns past the accumulators
        const uint32_t stash = tmem + C::NACC * C::ACC_COLS + ((uint32_t)(q * 32) << 16);
        for (int ch = c_lo; ch < c_hi; ++ch, ++acc_it) {
          if (w.part < 0 && ch == hch && hch > 0) {  // whole item: set the first half aside
#pragma unroll
            for (int c0 = 0; c0 < N; c0 += 16) {
              tmem_st16(stash + 0 * N + c0, *reinterpret_cast<float(*)[16]>(rz + c0));
              tmem_st16(stash + 1 * N + c0, *reinterpret_cast<float(*)[16]>(rf + c0));
              tmem_st16(stash + 2 * N + c0, *reinterpret_cast<float(*)[16]>(ro + c0));
            }
            tmem_st_wait();
#pragma unroll
            for (int j = 0; j < N; ++j) rz[j] = rf[j] = ro[j] = 0.f;
          }
          const int ab = acc_it % C::NACC;
          mbar_wait(&acc_full[ab], (acc_it / C::NACC) & 1);
          tc_fence_after();
          const uint32_t tb = tmem + ab * C::ACC_COLS + ((uint32_t)(q * 32) << 16);
#pragma unroll
          for (int c0 = 0; c0 < N; c0 += 16) {
            // per gate: columns [0, N) hi.hi, [N, 2N) hi.lo + lo.hi
            float pz[16], pf[16], po[16], cz[16], cf[16], co[16];
            tmem_ld_gates16(tb + 0 * C::GCOLS + c0, tb + 1 * C::GCOLS + c0, tb + 2 * C::GCOLS + c0, pz, pf, po);
            tmem_ld_gates16(tb + 0 * C::GCOLS + N + c0, tb + 1 * C::GCOLS + N + c0, tb + 2 * C::GCOLS + N + c0, cz,
                            cf, co);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              rz[c0 + j] += pz[j] + cz[j];
              rf[c0 + j] += pf[j] + cf[j];
              ro[c0 + j] += po[j] + co[j];
            }
          }
          tc_fence_before();
          mbar_arrive(&acc_empty[ab]);
        }
        const int slot = item - a.split_start;
        if (w.part == 0) {  // first half of a split item: hand the sum on, nothing else
          float* fx = a.fix + (size_t)slot * 3 * N * 128 + row;
#pragma unroll
          for (int j = 0; j < N; ++j) {
            fx[(size_t)(0 * N + j) * 128] = rz[j];
            fx[(size_t)(1 * N + j) * 128] = rf[j];
            fx[(size_t)(2 * N + j) * 128] = ro[j];
          }
          tc_epi_sync();
          if (et == 0) st_release(&a.fixflag[slot], 4 * a.epoch + 3);
          continue;
        }
        if (w.part == 1) {  // second half: S = (first half, from the other CTA) + this half
          if (et == 0) while (ld_acquire(&a.fixflag[slot]) < 4 * a.epoch + 3) __nanosleep(64);
          tc_epi_sync();
          const float* fx = a.fix + (size_t)slot * 3 * N * 128 + row;
#pragma unroll
          for (int j = 0; j < N; ++j) {
            rz[j] = __ldcg(fx + (size_t)(0 * N + j) * 128) + rz[j];
            rf[j] = __ldcg(fx + (size_t)(1 * N + j) * 128) + rf[j];
            ro[j] = __ldcg(fx + (size_t)(2 * N + j) * 128) + ro[j];
          }
        } else if (hch > 0) {  // whole item: S = (stashed first half) + second half
#pragma unroll
          for (int c0 = 0; c0 < N; c0 += 16) {
            float sz[16], sf[16], so[16];
            tmem_ld_gates16(stash + 0 * N + c0, stash + 1 * N + c0, stash + 2 * N + c0, sz, sf, so);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              rz[c0 + j] = sz[j] + rz[c0 + j];
              rf[c0 + j] = sf[j] + rf[c0 + j];
              ro[c0 + j] = so[j] + ro[c0 + j];
            }
          }
        }
        if constexpr (CELL == LINEAR) {
          // dense layer on the fp32-accurate path: plane g holds output columns
          // [g*Hpad, (g+1)*Hpad); chunk sums + bias straight to Y
          float* const rg[3] = {rz, rf, ro};
#pragma unroll
          for (int g = 0; g < 3; ++g) {
            const int col = g * a.Hpad + unit;
            const bool lv = col < a.H;
            const float bias = (lv && a.bias) ? a.bias[col] : 0.f;
            float* yp = a.Hout + t0 * a.ldh + col;
#pragma unroll
            for (int j = 0; j < N; ++j)
              if (lv && j < l) yp[(int64_t)j * a.ldh] = rg[g][j] + bias;
          }
          continue;
        }
#pragma unroll
        for (int j = 0; j < N; ++j) {
          if (a.dbg & 1024) {  // timing experiment: no activation math
          } else if (CELL == SRU) {
            rf[j] = tc_sigmoid(rf[j] + bf);
            ro[j] = tc_sigmoid(ro[j] + br);
          } else {
            rz[j] = tc_tanh(rz[j]);
            rf[j] = tc_sigmoid(rf[j]);
            ro[j] = tc_sigmoid(ro[j]);
          }
          // steps past the block end are identity steps (f = 1, z = 0): branch-free
          if (j >= l) rf[j] = 1.f, rz[j] = 0.f;
        }
#pragma unroll
        for (int j = 0; j < N; ++j) {
          Bblk = rf[j] * Bblk + (1.f - rf[j]) * rz[j];
          Ablk = rf[j] * Ablk;
        }
        const float cin = (a.dbg & 16) ? 0.f : tc_lookback(a, b, u, unit, et, Ablk, Bblk);  // 16: no look-back (timing)
        float c = cin;
        const bool live = unit < a.H && !(a.dbg & 512);  // 512: no stores (timing)
#pragma unroll
        for (int j = 0; j < N; ++j) {  // the c chain alone (one FMA per step) ...
          c = rf[j] * c + (1.f - rf[j]) * rz[j];
          rz[j] = c;
        }
#pragma unroll
        for (int j = 0; j < N; ++j) {  // ... then the independent outputs
          float h = ro[j] * tc_tanh(rz[j]);
          if (j < l && live) {
            if (CELL == SRU) h = h + (1.f - ro[j]) * a.Xhw[(t0 + j) * a.ldhw + unit];
            store_h(a, (t0 + j) * a.ldh + unit, h);
          }
        }
        if (b == a.nB - 1 && a.c_out != nullptr && live) a.c_out[unit] = c;  // c_T of the sequence
        tc_count_done(a, t0, et);
        continue;
      }
      const int ab = acc_it % C::NACC;
      mbar_wait(&acc_full[ab], (acc_it / C::NACC) & 1);
      tc_fence_after();
      const uint32_t tb = tmem + ab * C::ACC_COLS + ((uint32_t)(q * 32) << 16);
      // (A) activations + block aggregate
      // Branch-free per 16 columns: the three loads share one wait, the 48
      // activations are independent (ILP for the one epilogue warp per
      // scheduler), steps past the block end become identity steps (f = 1,
      // z = 0: the aggregate and, in phase C, c are left exactly unchanged).
      for (int c0 = 0; c0 < N && c0 < l; c0 += 16) {
        float pz[16], pf[16], po[16];
        tmem_ld_gates16(tb + 0 * N + c0, tb + 1 * N + c0, tb + 2 * N + c0, pz, pf, po);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (a.dbg & 1024) {  // timing experiment: no activation math
          } else if (CELL == SRU) {
            pf[j] = tc_sigmoid(pf[j] + bf);
            po[j] = tc_sigmoid(po[j] + br);
          } else {
            pz[j] = tc_tanh(pz[j]);
            pf[j] = tc_sigmoid(pf[j]);
            po[j] = tc_sigmoid(po[j]);
          }
          if (c0 + j >= l) pf[j] = 1.f, pz[j] = 0.f;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          Bblk = pf[j] * Bblk + (1.f - pf[j]) * pz[j];
          Ablk = pf[j] * Ablk;
        }
        tmem_st16(tb + 0 * N + c0, pz);
        tmem_st16(tb + 1 * N + c0, pf);
        tmem_st16(tb + 2 * N + c0, po);
      }
      tmem_st_wait();
      const float cin = (a.dbg & 16) ? 0.f : tc_lookback(a, b, u, unit, et, Ablk, Bblk);  // 16: no look-back (timing)
      // (C) sequential recurrence from c_in and the output mix
      // row pointers advanced by a stride per step (no 64-bit index
      // arithmetic per store); the uniform peer / operand-copy tests hoisted
      float c = cin;
      const bool live = unit < a.H;
      const int64_t ldh = a.ldh, ldhw = a.ldhw, ldop = a.ldop;
      const int npeer = a.npeer;
      float* hp = a.Hout + t0 * ldh + unit;
      const float* xp = CELL == SRU ? a.Xhw + t0 * ldhw + unit : nullptr;
      unsigned char* op = a.Hop ? static_cast<unsigned char*>(a.Hop) +
                                      (t0 * ldop + unit) * (MODE == TC_BF16 ? 2 : 4)
                                : nullptr;
      for (int c0 = 0; c0 < N && c0 < l && !(a.dbg & 512); c0 += 16) {  // 512: no scan / stores (timing)
        float z[16], f[16], o[16], xh[16];
        if (CELL == SRU) {  // highway inputs first: their latency overlaps the TMEM loads and the chain
#pragma unroll
          for (int j = 0; j < 16; ++j) xh[j] = (c0 + j < l && live) ? xp[(int64_t)(c0 + j) * ldhw] : 0.f;
        }
        tmem_ld_gates16(tb + 0 * N + c0, tb + 1 * N + c0, tb + 2 * N + c0, z, f, o);
        // the c chain alone (one FMA per step; f = 1, z = 0 past the block end) ...
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          c = f[j] * c + (1.f - f[j]) * z[j];
          z[j] = c;
        }
        // ... then 16 independent outputs
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float h = o[j] * tc_tanh(z[j]);
          if (CELL == SRU) h = h + (1.f - o[j]) * xh[j];
          f[j] = h;
        }
        if (npeer == 0 && op == nullptr) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c0 + j < l && live) hp[(int64_t)(c0 + j) * ldh] = f[j];
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int col = c0 + j;
            if (col < l && live) {
              const float h = f[j];
              hp[(int64_t)col * ldh] = h;
              const int64_t i = (t0 + col) * ldh + unit;
#pragma unroll
              for (int p = 0; p < kMaxPeers; ++p)
                if (p < npeer) a.Hpeer[p][i] = h;
              if (op != nullptr) {
                if (MODE == TC_BF16)
                  reinterpret_cast<__nv_bfloat16*>(op)[(int64_t)col * ldop] = __float2bfloat16_rn(h);
                else
                  reinterpret_cast<float*>(op)[(int64_t)col * ldop] = round_x(h, XR_TF32);
              }
            }
          }
        }
      }
      // TMEM buffer can be refilled
      tc_fence_before();
      mbar_arrive(&acc_empty[ab]);
      ++acc_it;
      if (b == a.nB - 1 && a.c_out != nullptr && unit < a.H) a.c_out[unit] = c;  // c_T of the sequence
      tc_count_done(a, t0, et, eg);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
}

}  // namespace rnnb
