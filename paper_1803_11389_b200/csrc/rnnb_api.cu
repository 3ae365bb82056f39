// C ABI of the blocked SRU/QRNN path (see include/rnnb.h).
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rnnb.h"
#include "abi_guard.h"
#include "ffma_dispatch.cuh"
#include "tc_dispatch.cuh"

using namespace rnnb;

namespace {

thread_local std::string g_err;

rnnb_status fail(rnnb_status s, const std::string& msg) {
  g_err = msg;
  return s;
}
rnnb_status cuda_fail(cudaError_t e, const char* where) {
  return fail(RNNB_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
}  // namespace

namespace rnnb {
// shared with lstm.cu: one thread-local last-error string per process
rnnb_status set_error(rnnb_status s, const std::string& msg) { return fail(s, msg); }
}  // namespace rnnb

namespace {

#define CUDA_TRY(expr)                                  \
  do {                                                  \
    cudaError_t _e = (expr);                            \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
  } while (0)

#define CU_TRY(expr)                                                                      \
  do {                                                                                    \
    CUresult _r = (expr);                                                                 \
    if (_r != CUDA_SUCCESS) return fail(RNNB_ECUDA, "stream memory operation failed: " #expr); \
  } while (0)

struct Layer {
  int64_t din = 0, dh = 0;
  int Dp = 0;        // d_in padded to a multiple of 8
  int U = 7;         // units per CTA
  int Upad = 0;      // d_h padded to a multiple of U
  void* W = nullptr; // [Upad*3][taps*Dp] gate-interleaved
  void* bias = nullptr;
  size_t wbytes = 0;
  bool loaded = false;
  FfmaPlan last;
  int grid = 0;
  // tensor-core path (BF16/TF32 stacks): gate-major operand weights
  void* Wtc = nullptr;  // [3*Hpad128][tcKp] bf16 or tf32-rounded f32
  int tcKp = 0;         // taps * Dtc, Dtc = d_in padded to the k-tile
  int Hpad128 = 0;
  bool last_tc = false;
  float* bias_tc = nullptr;  // [Hpad128][2]
  int64_t hw_off = 0;        // SRU highway reads x[:, hw_off + unit] (wide / sharded SRU)
  // fp32 layers too large for shared memory: per-(CTA, chunk) weight images
  // for the weight-streaming ws kernel, built on first use (ws_stream_pack)
  void* Wst = nullptr;
};

}  // namespace

struct rnnb_stack {
  int kind = 0, n_layers = 0, mode = 0, device = 0, num_sms = 148;
  std::vector<Layer> layers;
  void* ws[2] = {nullptr, nullptr};
  size_t ws_bytes = 0;
  int64_t last_launches = 0;
  void* rev = nullptr;    // time-reversed copy of the input for the FFMA paths (ldx < 0), [L][d_in]
  size_t rev_bytes = 0;
  void* op = nullptr;     // tensor-core operand copy of a layer input, [L+1][maxD]
  size_t op_bytes = 0;
  float* cbuf = nullptr;  // tensor-core c_T scratch + look-back state (carry maps, inclusive carries)
  int tc_epoch = 0;       // launch tag of the split-last-wave flags
  int* tc_status = nullptr;  // [kFixSlots] split-last-wave flags, cleared only on (re)allocation
  size_t tc_status_n = 0;
  float* fix = nullptr;      // 3xTF32 split last wave: first halves' chunk sums
  size_t fix_bytes = 0;
  int* flags = nullptr;
  size_t cf_bytes = 0;
  void* hostX = nullptr;  // e2e device staging
  void* hostH = nullptr;
  size_t hx_bytes = 0, hh_bytes = 0;
  // rnnb_forward_host pipeline: copy-in / copy-out streams and per-chunk events
  cudaStream_t s_in = nullptr, s_in2 = nullptr, s_out = nullptr;
  cudaEvent_t ev[2 * 8 + 2] = {};
  // tcgen05 streaming: the operand-conversion stream and one event per copy-in segment
  cudaStream_t s_cv = nullptr;
  std::vector<cudaEvent_t> sev;
  // streaming forward_host (single-layer fp32 stacks): counters the copy
  // streams and the layer kernel hand rows through
  int* stream_ctr = nullptr;  // [0] rows of X resident, [1] kernel time-out flag, [2..] per-chunk CTA counts
  int* stream_flag_host = nullptr;  // pinned copy of the time-out flag
  const int* stream_ready = nullptr;
  int* stream_done = nullptr;
  int stream_chunk = 0;
  unsigned long long* stream_trace = nullptr;  // RNNB_STREAM_TRACE: in-kernel time stamps (tuning)
  int* stream_flags = nullptr;  // tcgen05 streaming conversion: per-group flags (epoch-tagged)
  size_t stream_flags_n = 0;
  int stream_epoch = 0;
  int stream_free_sms = 2;  // SMs the streaming layer launch leaves to the operand conversion
  bool stream_refused = false;
  // set after a streaming time-out (a serialising profiler, a stalled copy
  // engine): later rnnb_forward_host calls on this handle use the chunked
  // pipeline.  A handle is not meant for concurrent calls (the peer and
  // streaming fields below are per call); the flag is atomic so a racing
  // reader sees either value, never a torn one.
  std::atomic<bool> stream_disabled{false};
  // rnnb_forward_ex: extra h destinations of the LAST layer (peer GPUs'
  // mapped buffers); cur_peers is non-zero only while that layer launches
  int n_peers = 0, cur_peers = 0;
  void* peer_H[kMaxPeers] = {};
};

namespace {

constexpr int64_t kMaxStreamChunks = 64;

// Stream memory operations (driver API, fetched through the runtime so the
// library does not link libcuda): write a 32-bit value / wait for one.
typedef CUresult (*StreamWriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*StreamWaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct StreamOps {
  StreamWriteValue32Fn write = nullptr;
  StreamWaitValue32Fn wait = nullptr;
};
StreamOps stream_ops() {
  static StreamOps ops;
  static bool done = false;
  if (!done) {
    done = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      ops.write = reinterpret_cast<StreamWriteValue32Fn>(p);
    p = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      ops.wait = reinterpret_cast<StreamWaitValue32Fn>(p);
  }
  return ops;
}

size_t elem_size(int mode) { return mode == RNNB_F64 ? 8 : 4; }
size_t wsize(int mode) { return mode == RNNB_F64 ? 8 : (mode == RNNB_BF16 ? 2 : 4); }
int taps(int kind) { return kind == RNNB_QRNN ? 2 : 1; }

int choose_units(int64_t dh, int num_sms) {
  // enough CTAs to cover the SMs, U from the instantiated set {2, 4, 7}
  if (dh >= 7LL * num_sms * 0.85) return 7;
  if (dh >= 4LL * num_sms * 0.85) return 4;
  if (dh > 2LL * num_sms) return 4;
  return 2;
}

// Weight repack on the GPU: the caller's gate matrices are staged in device
// memory as they are and ONE kernel writes both device layouts (gate-
// interleaved FFMA rows, gate-major tensor-core planes) with the mode's
// rounding -- the host used to do this element by element (40-50 ms for cfg2,
// which made the reference-signature run_blocked, one upload per call, slower
// than the CPU reference).
struct PackArgs {
  const void* m[6];   // SRU: W, W_f, W_r, b_f, b_r ; QRNN: (cand, forget, out) x (tap 0, tap 1)
  int kind, mode, T;
  int64_t dh, din, Dp, Kp;        // FFMA layout W[3*Upad][Kp], row 3u+g, columns [tap][Dp]
  void* W;
  void* Wtc;                      // tensor-core layout [planes][3*Hpad][tcKp], row g*Hpad+u, columns [tap][Dtc]
  int64_t Hpad, tcKp, Dtc, lo_off;  // lo_off: elements from the hi to the lo plane (3xTF32), 0: one plane
  void* bias;                     // SRU [Upad][2] in the stack's element type
  float* bias_tc;                 // SRU [Hpad][2]
};
template <typename S>
__global__ void pack_layer_kernel(const PackArgs a) {
  const int64_t n = a.dh * 3 * a.T * a.din;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i % a.din;
    int64_t r = i / a.din;
    const int tap = (int)(r % a.T);
    r /= a.T;
    const int g = (int)(r % 3);
    const int64_t u = r / 3;
    const int slot = a.kind == RNNB_SRU ? g : 2 * g + tap;
    const double v = (double)static_cast<const S*>(a.m[slot])[u * a.din + k];
    const float vf = (float)v;
    const int64_t dst = (3 * u + g) * a.Kp + (int64_t)tap * a.Dp + k;
    switch (a.mode) {
      case RNNB_F64: static_cast<double*>(a.W)[dst] = v; break;
      case RNNB_BF16: static_cast<__nv_bfloat16*>(a.W)[dst] = __float2bfloat16_rn(vf); break;
      case RNNB_TF32: static_cast<float*>(a.W)[dst] = rnnb::round_x(vf, rnnb::XR_TF32); break;
      default: static_cast<float*>(a.W)[dst] = vf; break;
    }
    if (a.Wtc) {
      const int64_t d2 = ((int64_t)g * a.Hpad + u) * a.tcKp + (int64_t)tap * a.Dtc + k;
      if (a.mode == RNNB_BF16) {
        static_cast<__nv_bfloat16*>(a.Wtc)[d2] = __float2bfloat16_rn(vf);
      } else {
        const float hi = rnnb::round_x(vf, rnnb::XR_TF32);
        static_cast<float*>(a.Wtc)[d2] = hi;
        if (a.lo_off) static_cast<float*>(a.Wtc)[d2 + a.lo_off] = rnnb::round_x(vf - hi, rnnb::XR_TF32);
      }
    }
  }
  if (a.kind == RNNB_SRU)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.dh * 2; i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t u = i >> 1;
      const int j = (int)(i & 1);
      const double v = (double)static_cast<const S*>(a.m[3 + j])[u];
      if (a.mode == RNNB_F64) static_cast<double*>(a.bias)[i] = v;
      else static_cast<float*>(a.bias)[i] = (float)v;
      if (a.bias_tc) a.bias_tc[i] = (float)v;
    }
}

rnnb_status ensure_ws(rnnb_stack* h, size_t bytes) {
  if (h->ws_bytes >= bytes) return RNNB_OK;
  for (auto& p : h->ws)
    if (p) cudaFree(p), p = nullptr;
  h->ws_bytes = 0;
  CUDA_TRY(cudaMalloc(&h->ws[0], bytes));
  CUDA_TRY(cudaMalloc(&h->ws[1], bytes));
  h->ws_bytes = bytes;
  return RNNB_OK;
}

template <typename TA, typename TW>
LayerArgs<TA, TW> make_args(const rnnb_stack* h, const Layer& ly) {
  LayerArgs<TA, TW> a{};
  a.W = static_cast<const TW*>(ly.W);
  a.bias = static_cast<const TA*>(ly.bias);
  a.D = (int)ly.din;
  a.Dp = ly.Dp;
  a.H = (int)ly.dh;
  a.dbg = getenv("RNNB_DEBUG") ? atoi(getenv("RNNB_DEBUG")) : 0;
  a.xround = h->mode == RNNB_BF16 ? XR_BF16 : (h->mode == RNNB_TF32 ? XR_TF32 : XR_NONE);
  a.x_ready = h->stream_ready;
  a.h_done = h->stream_done;
  a.stream_fail = h->stream_ready ? h->stream_ctr + 1 : nullptr;
  a.h_chunk = h->stream_chunk;
  a.npeer = h->cur_peers;
  for (int p = 0; p < h->cur_peers; ++p) a.Hpeer[p] = static_cast<TA*>(h->peer_H[p]);
  return a;
}

// Tensor-core path selection.  bf16/tf32: small T_b too (N = 16 with masked
// columns below 16 -- one weight stream per block still beats the FFMA
// kernel); f32x3: 16..32 (below 16 the exact FFMA kernel is faster).
bool use_tc(const rnnb_stack* h, int64_t Tb) {
  if (getenv("RNNB_NO_TC") != nullptr) return false;
  const char* mn = getenv("RNNB_TC_MIN");
  // measured on cfg2: bf16 TC beats the FFMA kernel from T_b = 1 (1.26 vs 0.86 M
  // steps/s), tf32 from T_b = 2 (1.29 vs 0.95)
  const int lo = mn ? atoi(mn) : (h->mode == RNNB_BF16 ? 1 : 2);
  if (h->mode == RNNB_BF16 || h->mode == RNNB_TF32) return Tb >= lo && Tb <= 128;
  // f32x3: T_b >= 16 (below, the exact FFMA kernel is faster); blocks longer
  // than 32 steps run as 32-step tensor-core blocks (the 3N chunk partials
  // live in registers: N <= 32), i.e. each weight is read into the tensor
  // pipe once per 32 steps -- the same cap as the FFMA kernel's 32-column
  // passes (cfg2 T_b=64: 2.9 M steps/s on the FFMA fallback before)
  if (h->mode == RNNB_F32X3) return Tb >= 8;
  // fp32 (the reference precision): the same fp32-accurate 3xTF32 tcgen05
  // path from T_b = 8 on (N = 16 accumulator columns, half of them masked:
  // cfg2 3.04 vs 2.65 M steps/s on the FFMA kernel, cfg3 0.97 vs 0.65 M; at
  // T_b = 4 the FFMA kernel wins 2.18 vs 1.54 M; RNNB_F32_TC_MIN) (normwise error 1e-6 .. 6e-6 against the oracle on
  // the BASELINE shapes, inside the 1e-5 bound: tests/test_gpu_full_shapes.py;
  // 2.5x the FFMA kernel at cfg2 T_b = 32).  RNNB_F32_TC=0 keeps every T_b
  // on the FFMA kernels (bitwise invariant to how calls chunk the sequence).
  if (h->mode == RNNB_F32) {
    const char* e = getenv("RNNB_F32_TC");
    const char* m = getenv("RNNB_F32_TC_MIN");
    return !(e && e[0] == '0') && Tb >= (m ? atoi(m) : 8);
  }
  return false;
}

// fp32 mode: the tcgen05 path only when its items fill the GPU (a short
// sequence of a narrow layer -- cfg1: 4 unit tiles x 16 blocks = 64 items --
// runs faster on the FFMA kernel's 128+ CTAs)
bool use_tc_layer(const rnnb_stack* h, const Layer& ly, int64_t L, int64_t Tb) {
  if (!use_tc(h, Tb)) return false;
  if (h->mode != RNNB_F32) return true;
  const int64_t Tbe = Tb > 32 ? 32 : Tb;
  const int64_t items = (ly.dh + 127) / 128 * ((L + Tbe - 1) / Tbe);
  return items >= h->num_sms;
}

int tc_mode_of(int mode) {
  return mode == RNNB_BF16 ? TC_BF16 : (mode == RNNB_TF32 ? TC_TF32 : TC_3XTF32);  // f32, f32x3: 3xTF32
}

// one layer on the tcgen05 path (tc_layer.cuh)
// time steps per tensor-core block (3xTF32 caps blocks at 32 steps, see use_tc)
int64_t tc_block(const rnnb_stack* h, int64_t Tb_req) {
  return (tc_mode_of(h->mode) == TC_3XTF32 && Tb_req > 32) ? 32 : Tb_req;
}

// the MMA-operand copy of a layer input: [planes][L+1][ldop] (row 0 = x_{-1})
rnnb_status ensure_tc_op(rnnb_stack* h, int li, int64_t L, int64_t* ldop_out) {
  const int mode = tc_mode_of(h->mode);
  const int es = mode == TC_BF16 ? 2 : 4;
  const int64_t ldop = (h->layers[li].din + 7) / 8 * 8;
  const size_t opb = (size_t)(mode == TC_3XTF32 ? 2 : 1) * (L + 1) * ldop * es;
  if (h->op_bytes < opb) {
    if (h->op) cudaFree(h->op);
    h->op = nullptr;
    h->op_bytes = 0;
    CUDA_TRY(cudaMalloc(&h->op, opb));
    h->op_bytes = opb;
  }
  *ldop_out = ldop;
  return RNNB_OK;
}

// flags of the split last wave (one per split item)
constexpr size_t kFixSlots = 128;

// Scratch of one tensor-core layer launch, (re)allocated when too small.
// cudaMalloc / cudaFree wait for the device, so the streaming host path calls
// this BEFORE it launches anything that spins on rows still to be enqueued.
rnnb_status tc_layer_scratch(rnnb_stack* h, Layer& ly, int64_t nB, int nU, int N, bool x3, cudaStream_t s) {
  // cbuf [Hpad] (c_T scratch) | aggA, aggB, incl [nB][Hpad]: written before read
  const size_t plane = (size_t)nB * ly.Hpad128;
  const size_t cfb = ((size_t)ly.Hpad128 + 3 * plane) * sizeof(float);
  if (h->cf_bytes < cfb) {
    if (h->cbuf) cudaFree(h->cbuf);
    h->cbuf = nullptr;
    h->cf_bytes = 0;
    CUDA_TRY(cudaMalloc(&h->cbuf, cfb));
    h->cf_bytes = cfb;
  }
  // the split last wave's kFixSlots flags, tagged 4*epoch + 3 by each launch
  // (cleared only when allocated or when the epoch wraps); the look-back
  // itself needs no status words any more (tc_lookback)
  (void)nU;
  if (h->tc_status_n < kFixSlots || h->tc_epoch >= (1 << 28)) {
    if (h->tc_status_n < kFixSlots) {
      if (h->tc_status) cudaFree(h->tc_status);
      h->tc_status = nullptr;
      h->tc_status_n = 0;
      CUDA_TRY(cudaMalloc(&h->tc_status, kFixSlots * sizeof(int)));
      h->tc_status_n = kFixSlots;
    }
    CUDA_TRY(cudaMemsetAsync(h->tc_status, 0, h->tc_status_n * sizeof(int), s));
    h->tc_epoch = 0;
  }
  if (x3) {
    const size_t fb = kFixSlots * 3 * (size_t)N * 128 * sizeof(float);
    if (h->fix_bytes < fb) {
      if (h->fix) cudaFree(h->fix);
      h->fix = nullptr;
      h->fix_bytes = 0;
      CUDA_TRY(cudaMalloc(&h->fix, fb));
      h->fix_bytes = fb;
    }
  }
  return RNNB_OK;
}

rnnb_status tc_layer_launch(rnnb_stack* h, int li, const float* X, int64_t ldx, int64_t L, int64_t Tb_req,
                            float* Hout, int64_t ldh, float* c_io, float* xc_io, cudaStream_t s) {
  Layer& ly = h->layers[li];
  const int mode = tc_mode_of(h->mode);
  const int64_t Tb = tc_block(h, Tb_req);
  int64_t ldop = 0;
  rnnb_status ost = ensure_tc_op(h, li, L, &ldop);
  if (ost != RNNB_OK) return ost;
  // streaming (rnnb_forward_host): the operand rows are converted by the
  // copy-in stream while this launch runs; two SMs stay free for them
  const bool streaming = h->stream_ready != nullptr;
  const int nU = ly.Hpad128 / 128;
  const int64_t nB = (L + Tb - 1) / Tb;
  rnnb_status sst = tc_layer_scratch(h, ly, nB, nU, tc_pick_n((int)Tb), mode == TC_3XTF32, s);
  if (sst != RNNB_OK) return sst;
  const size_t plane = (size_t)nB * ly.Hpad128;
  float* aggA = h->cbuf + ly.Hpad128;
  ++h->tc_epoch;
  // the look-back arrays start as all-ones sentinels: filled by the operand
  // conversion kernel (no extra launch), or by a memset when the conversion
  // streams beside the layer kernel
  const size_t lb_bytes = 3 * plane * sizeof(float);
  if (!streaming)
    CUDA_TRY(tc_to_operand(mode, X, ldx, h->kind == RNNB_QRNN ? xc_io : nullptr, h->op, ldop, L, (int)ly.din, s,
                           aggA, lb_bytes));
  else
    CUDA_TRY(cudaMemsetAsync(aggA, 0xFF, lb_bytes, s));
  TcArgs a{};
  a.Xhw = X + ly.hw_off;
  a.ldhw = ldx;
  a.Hout = Hout;
  a.ldh = ldh;
  a.Hop = nullptr;
  a.npeer = h->cur_peers;
  for (int p = 0; p < h->cur_peers; ++p) a.Hpeer[p] = static_cast<float*>(h->peer_H[p]);
  a.bias = ly.bias_tc;
  a.c_in = c_io;                          // read only (anchor of the look-back)
  a.c_out = c_io ? h->cbuf : nullptr;     // c_T to scratch, copied to c_io after the launch
  a.epoch = h->tc_epoch;
  a.agg = reinterpret_cast<unsigned long long*>(aggA);
  a.incl = reinterpret_cast<unsigned int*>(aggA + 2 * plane);
  a.L = L;
  a.T_b = (int)Tb;
  a.H = (int)ly.dh;
  a.Hpad = ly.Hpad128;
  a.D = (int)ly.din;
  const int KT = mode == TC_BF16 ? 64 : 32;
  a.nKtap = (int)((ly.din + KT - 1) / KT);
  a.nK = ly.tcKp / KT;
  a.nU = nU;
  a.nB = (int)nB;
  a.dbg = getenv("RNNB_DEBUG") ? atoi(getenv("RNNB_DEBUG")) : 0;
  {
    // second epilogue warp group (bf16 / tf32): when an item's MMA stream is
    // shorter than ~8 us (51.3 cycles per MMA, 12 per k-tile) or the blocks are
    // tiny, the epilogue bounds the item (measured: cfg3 K = 1024 +15..56 %,
    // cfg2 K = 2048 -6..+3 % except T_b <= 4)
    const double mma_us = (double)a.nK * 12 * 51.3 / 1965.0;
    const char* eg = getenv("RNNB_TC_EGROUPS");
    // (SRU's epilogue also gathers the highway x: cfg3 tf32, 10 us of MMAs per item, still gains 37 %)
    a.egroups = eg ? atoi(eg) : ((mma_us < 8.0 || Tb <= 4 || (h->kind == RNNB_SRU && mma_us < 14.0)) ? 2 : 1);
  }
  // 3xTF32: split the last, partial wave's items in two K halves on two CTAs
  // (tc_work in tc_layer.cuh; the arithmetic is the same split or not)
  const int nitems = nU * (int)nB;
  const int G = nitems < h->num_sms - (streaming ? h->stream_free_sms : 0) ? nitems : h->num_sms - (streaming ? h->stream_free_sms : 0);
  a.split_start = nitems;
  {  // 3xTF32 K-chunk plan (x3_chunk_start): deeper first chunks for short reductions
    const char* env_ck = getenv("RNNB_X3_CK0");
    a.ck0 = env_ck ? atoi(env_ck) : x3_pick_ck0(a.nK);
    if (a.ck0 < 1) a.ck0 = RNNB_X3_CK;
  }
  const char* env_sp = getenv("RNNB_TC_SPLIT");
  if (mode == TC_3XTF32 && !(env_sp && env_sp[0] == '0')) {
    int W = nitems / G, R = nitems - W * G;
    const int nch = x3_nchunks(a.nK, a.ck0);
    if (streaming && nitems > G) {
      // input-bound launch (rows arrive slower than the kernel consumes them):
      // what counts is how soon the LAST blocks finish after their rows land,
      // so the last G/2 items are split whatever the wave structure
      R = G / 2 < (int)kFixSlots ? G / 2 : (int)kFixSlots;
      W = 1;
    }
    if (W >= 1 && R > 0 && 2 * R <= G && R <= (int)kFixSlots && nch >= 2) {
      a.split_start = nitems - R;
      a.fix = h->fix;
      a.fixflag = h->tc_status;
    }
  }
  int grid = 0;
  if (streaming) {
    a.x_ready = h->stream_ready;
    a.h_done = h->stream_done;
    a.h_gran = h->stream_chunk;
    a.trace = h->stream_trace;
    a.stream_fail = h->stream_ctr + 1;
  }
  cudaError_t e = tc_layer_run(h->kind, mode, a, ly.Wtc, ly.tcKp, h->op, ldop, h->num_sms - (streaming ? h->stream_free_sms : 0), s,
                               &grid);
  if (e != cudaSuccess) return cuda_fail(e, "tc_layer launch");
  if (c_io) CUDA_TRY(cudaMemcpyAsync(c_io, h->cbuf, ly.dh * sizeof(float), cudaMemcpyDeviceToDevice, s));
  ly.last_tc = true;
  ly.grid = grid;
  ly.last = FfmaPlan{};
  ly.last.nt = tc_pick_n((int)Tb);
  h->last_launches += 2;  // operand conversion + layer kernel
  return RNNB_OK;
}

// one layer over [L x din] -> [L x dh]
template <typename TA, typename TW>
rnnb_status layer_launch(rnnb_stack* h, int li, const TA* X, int64_t ldx, int64_t L, int64_t Tb,
                         TA* Hout, int64_t ldh, TA* c_io, TA* xc_io, TA* G, int64_t ldg,
                         cudaStream_t s) {
  if constexpr (sizeof(TA) == 4) {
    if (G == nullptr && use_tc_layer(h, h->layers[li], L, Tb))
      return tc_layer_launch(h, li, reinterpret_cast<const float*>(X), ldx, L, Tb, reinterpret_cast<float*>(Hout),
                             ldh, reinterpret_cast<float*>(c_io), reinterpret_cast<float*>(xc_io), s);
  }
  Layer& ly = h->layers[li];
  ly.last_tc = false;
  LayerArgs<TA, TW> a = make_args<TA, TW>(h, ly);
  if constexpr (sizeof(TA) == 4 && sizeof(TW) == 4) {
    // weights beyond what a CTA can keep in shared memory: stream per-chunk
    // weight images through the ws kernel's ring (T_b >= 32 passes)
    const size_t res_bytes = (size_t)3 * ly.U * taps(h->kind) * ly.Dp * sizeof(float);
    const char* env = getenv("RNNB_WSTREAM");
    if (G == nullptr && Tb >= 32 && a.xround == XR_NONE && h->stream_ready == nullptr &&
        res_bytes + 44 * 1024 > kMaxSmem && !(env && env[0] == '0') && ly.din % 8 == 0) {
      // (the resident plans need ~44 KB of ring + partials beside the weights)
      if (!ly.Wst) {
        const size_t n = ws_stream_elems(h->kind, ly.Dp, (int)ly.dh);
        CUDA_TRY(cudaMalloc(&ly.Wst, n * sizeof(float)));
        CUDA_TRY(ws_stream_pack(h->kind, static_cast<const float*>(ly.W), 3 * ly.Upad, ly.Dp, (int)ly.dh,
                                static_cast<float*>(ly.Wst), s));
      }
      a.Wst = static_cast<const TW*>(ly.Wst);
    }
  }
  a.X = X;
  a.ldx = ldx;
  a.xcarry = h->kind == RNNB_QRNN ? xc_io : nullptr;
  a.Xhw = X + ly.hw_off;
  a.ldhw = ldx;
  a.Hout = Hout;
  a.ldh = ldh;
  a.c_in = c_io;
  a.c_out = c_io;
  a.G = G;
  a.ldg = ldg;
  a.L = L;
  a.T_b = (int)(Tb > (int64_t)1 << 30 ? (int64_t)1 << 30 : Tb);
  FfmaPlan plan;
  cudaError_t e = ffma_layer_run<TA, TW>(h->kind, ly.U, a, true, s, &plan);
  if (e == cudaErrorNotSupported && a.x_ready != nullptr) {
    h->stream_refused = true;  // streaming needs the ws kernel; nothing was launched
    return fail(RNNB_EINVAL, "streaming input not supported for this layer");
  }
  if (e != cudaSuccess) return cuda_fail(e, "ffma_layer launch");
  ly.last = plan;
  ly.grid = plan.grid ? plan.grid : (int)((ly.dh + ly.U - 1) / ly.U);
  h->last_launches += 1;
  return RNNB_OK;
}

// Rows of a time-reversed input view (row t at X + t*ldx, ldx < 0) into a
// dense [L][D] buffer, 16-byte vectors when aligned.
template <typename T>
__global__ void reverse_rows_kernel(const T* __restrict__ X, int64_t ldx, T* __restrict__ out, int64_t L, int D) {
  for (int64_t r = blockIdx.y; r < L; r += gridDim.y) {
    const T* src = X + r * ldx;
    T* dst = out + r * D;
    for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < D; d += gridDim.x * blockDim.x) dst[d] = src[d];
  }
}

template <typename TA, typename TW>
rnnb_status forward_t(rnnb_stack* h, const TA* X, int64_t ldx, int64_t L, int64_t Tb, TA* H,
                      int64_t ldh, TA* c_state, TA* x_carry, cudaStream_t s) {
  if (ldx < 0 && !(sizeof(TA) == 4 && use_tc_layer(h, h->layers[0], L, Tb))) {
    // Time-reversed input (the backward direction of a bidirectional stack).
    // The tcgen05 path reads it directly: its operand conversion walks the
    // rows with the negative stride.  The FFMA kernels fetch x with TMA
    // boxes, whose strides are unsigned, so they get a dense reversed copy.
    const int64_t din = h->layers[0].din;
    const size_t rb = (size_t)L * din * sizeof(TA);
    if (h->rev_bytes < rb) {
      if (h->rev) cudaFree(h->rev);
      h->rev = nullptr;
      h->rev_bytes = 0;
      CUDA_TRY(cudaMalloc(&h->rev, rb));
      h->rev_bytes = rb;
    }
    const int bx = (int)((din + 255) / 256);
    const int by = (int)(L < 4096 ? L : 4096);
    reverse_rows_kernel<TA><<<dim3(bx, by), 256, 0, s>>>(X, ldx, static_cast<TA*>(h->rev), L, (int)din);
    CUDA_TRY(cudaGetLastError());
    rnnb_status st = forward_t<TA, TW>(h, static_cast<const TA*>(h->rev), din, L, Tb, H, ldh, c_state, x_carry, s);
    h->last_launches += 1;
    return st;
  }
  int64_t maxw = 0;
  for (auto& ly : h->layers) maxw = ly.dh > maxw ? ly.dh : maxw;
  if (h->n_layers > 1) {
    rnnb_status st = ensure_ws(h, (size_t)L * maxw * sizeof(TA));
    if (st != RNNB_OK) return st;
  }
  h->last_launches = 0;
  const TA* in = X;
  int64_t ldin = ldx;
  int64_t coff = 0, xoff = 0;
  for (int li = 0; li < h->n_layers; ++li) {
    Layer& ly = h->layers[li];
    const bool last = li == h->n_layers - 1;
    TA* out = last ? H : static_cast<TA*>(h->ws[li & 1]);
    const int64_t ldo = last ? ldh : ly.dh;
    TA* c_io = c_state ? c_state + coff : nullptr;
    TA* xc_io = x_carry ? x_carry + xoff : nullptr;
    h->cur_peers = last ? h->n_peers : 0;
    rnnb_status st = layer_launch<TA, TW>(h, li, in, ldin, L, Tb, out, ldo, c_io, xc_io, nullptr, 0, s);
    h->cur_peers = 0;
    if (st != RNNB_OK) return st;
    if (xc_io && h->kind == RNNB_QRNN) {
      // carried x for the next call = last input row of this layer (blocked.py:262)
      CUDA_TRY(cudaMemcpyAsync(xc_io, in + (L - 1) * ldin, ly.din * sizeof(TA), cudaMemcpyDeviceToDevice, s));
      h->last_launches += 1;
    }
    coff += ly.dh;
    xoff += ly.din;
    in = out;
    ldin = ldo;
  }
  return RNNB_OK;
}

rnnb_status check_stack(rnnb_stack* h) {
  if (!h) return fail(RNNB_EINVAL, "null stack handle");
  for (int i = 0; i < h->n_layers; ++i)
    if (!h->layers[i].loaded) return fail(RNNB_EINVAL, "layer " + std::to_string(i) + " has no weights");
  return RNNB_OK;
}

template <typename T>
__global__ void sweep_kernel(const T* __restrict__ F, const T* __restrict__ Xh, const T* __restrict__ c0,
                             T* __restrict__ C, int64_t d, int64_t T_) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= d) return;
  T c = c0[i];
  for (int64_t t = 0; t < T_; ++t) {
    T f = F[i * T_ + t];
    c = f * c + (T(1) - f) * Xh[i * T_ + t];
    C[i * T_ + t] = c;
  }
}

template <typename T>
__global__ void finalize_kernel(int kind, const T* __restrict__ O, const T* __restrict__ C,
                                const T* __restrict__ Xb, T* __restrict__ H, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  T o = O[i];
  T h = o * tanh_full(C[i]);
  if (kind == RNNB_SRU) h = h + (T(1) - o) * Xb[i];
  H[i] = h;
}

}  // namespace

extern "C" {

const char* rnnb_last_error(void) { return g_err.c_str(); }
const char* rnnb_version(void) { return "rnnb-b200 0.1.0 (sm_100a)"; }

rnnb_status rnnb_plan_blocks(int64_t seq_len, int64_t block_size, int64_t* n_blocks, int64_t* last_len) {
  if (seq_len < 1) return fail(RNNB_EINVAL, "seq_len must be >= 1");
  if (block_size < 1) return fail(RNNB_EINVAL, "block_size must be >= 1");
  int64_t nb = (seq_len + block_size - 1) / block_size;
  if (n_blocks) *n_blocks = nb;
  if (last_len) *last_len = seq_len - (nb - 1) * block_size;
  return RNNB_OK;
}

rnnb_status rnnb_stack_create(rnnb_stack_t* out, int kind, int n_layers, const int64_t* d_in,
                              const int64_t* d_h, int mode, int device) {
  return rnnb_stack_create_ex(out, kind, n_layers, d_in, d_h, mode, device, 0);
}

static rnnb_status rnnb_stack_create_ex_impl(rnnb_stack_t* out, int kind, int n_layers, const int64_t* d_in,
                                 const int64_t* d_h, int mode, int device, int flags) {
  const bool wide = (flags & RNNB_FLAG_WIDE_SRU) != 0;
  if (!out) return fail(RNNB_EINVAL, "out is null");
  *out = nullptr;
  if (kind != RNNB_SRU && kind != RNNB_QRNN)
    return fail(RNNB_EINVAL, "blocked execution covers SRU and QRNN; use lstm_run_precomputed for LSTM");
  if (n_layers < 1) return fail(RNNB_EINVAL, "n_layers must be >= 1");
  if (mode < RNNB_F32 || mode > RNNB_F32X3) return fail(RNNB_EINVAL, "unknown compute mode");
  if (!d_in || !d_h) return fail(RNNB_EINVAL, "null dimension arrays");
  for (int l = 0; l < n_layers; ++l) {
    if (d_in[l] < 1 || d_h[l] < 1) return fail(RNNB_EINVAL, "d_in and d_h must be >= 1");
    if (kind == RNNB_SRU && !wide && d_in[l] != d_h[l]) return fail(RNNB_EINVAL, "SRU requires d_in == d_h");
    if (kind == RNNB_SRU && wide && d_in[l] < d_h[l]) return fail(RNNB_EINVAL, "wide SRU needs d_in >= d_h");
    if (l > 0 && !wide && d_in[l] != d_h[l - 1])
      return fail(RNNB_EINVAL, "layer " + std::to_string(l) + " input width does not match previous layer width");
    if (d_in[l] > (1 << 24) || d_h[l] > (1 << 24)) return fail(RNNB_EUNSUPPORTED, "dimension too large");
  }
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(RNNB_EINVAL, "bad device ordinal");
  auto* h = new rnnb_stack();
  h->kind = kind;
  h->n_layers = n_layers;
  h->mode = mode;
  h->device = device;
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
  h->layers.resize(n_layers);
  for (int l = 0; l < n_layers; ++l) {
    Layer& ly = h->layers[l];
    ly.din = d_in[l];
    ly.dh = d_h[l];
    ly.Dp = (int)((d_in[l] + 7) / 8 * 8);
    ly.U = choose_units(d_h[l], h->num_sms);
    ly.Upad = (int)((d_h[l] + ly.U - 1) / ly.U * ly.U);
  }
  *out = h;
  return RNNB_OK;
}

rnnb_status rnnb_stack_create_ex(rnnb_stack_t* out, int kind, int n_layers, const int64_t* d_in,
                                 const int64_t* d_h, int mode, int device, int flags) {
  return abi_guard("rnnb_stack_create_ex", [&]() { return rnnb_stack_create_ex_impl(out, kind, n_layers, d_in, d_h, mode, device, flags); });
}

rnnb_status rnnb_stack_destroy(rnnb_stack_t h) {
  if (!h) return RNNB_OK;
  DeviceGuard dg(h->device);
  for (auto& ly : h->layers) {
    if (ly.W) cudaFree(ly.W);
    if (ly.Wst) cudaFree(ly.Wst);
    if (ly.bias) cudaFree(ly.bias);
    if (ly.Wtc) cudaFree(ly.Wtc);
    if (ly.bias_tc) cudaFree(ly.bias_tc);
  }
  if (h->op) cudaFree(h->op);
  if (h->rev) cudaFree(h->rev);
  if (h->cbuf) cudaFree(h->cbuf);
  if (h->tc_status) cudaFree(h->tc_status);
  if (h->fix) cudaFree(h->fix);
  for (auto& p : h->ws)
    if (p) cudaFree(p);
  if (h->hostX) cudaFree(h->hostX);
  if (h->hostH) cudaFree(h->hostH);
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  if (h->stream_ctr) cudaFree(h->stream_ctr);
  if (h->stream_flags) cudaFree(h->stream_flags);
  if (h->stream_flag_host) cudaFreeHost(h->stream_flag_host);
  if (h->s_in) cudaStreamDestroy(h->s_in);
  if (h->s_in2) cudaStreamDestroy(h->s_in2);
  if (h->s_cv) cudaStreamDestroy(h->s_cv);
  for (auto& e : h->sev) cudaEventDestroy(e);
  if (h->s_out) cudaStreamDestroy(h->s_out);
  delete h;
  return RNNB_OK;
}

static rnnb_status rnnb_stack_set_layer_impl(rnnb_stack_t h, int layer, const void* const* mats, int n_mats, int src_dtype) {
  if (!h) return fail(RNNB_EINVAL, "null stack handle");
  if (layer < 0 || layer >= h->n_layers) return fail(RNNB_EINVAL, "layer index out of range");
  const int need = h->kind == RNNB_SRU ? 5 : 6;
  if (!mats || n_mats != need) return fail(RNNB_EINVAL, "expected " + std::to_string(need) + " weight arrays");
  if (src_dtype != RNNB_DT_F32 && src_dtype != RNNB_DT_F64) return fail(RNNB_EINVAL, "src dtype must be f32 or f64");
  for (int i = 0; i < n_mats; ++i)
    if (!mats[i]) return fail(RNNB_EINVAL, "null weight array");
  Layer& ly = h->layers[layer];
  const int T = taps(h->kind);
  const int64_t Kp = (int64_t)T * ly.Dp;
  const int64_t rows = (int64_t)ly.Upad * 3;
  const size_t ws = wsize(h->mode);
  const size_t ses = src_dtype == RNNB_DT_F64 ? 8 : 4;
  DeviceGuard dg(h->device);
  CUDA_TRY(dg.err);
  for (void** p : {(void**)&ly.W, (void**)&ly.Wst, (void**)&ly.bias, (void**)&ly.Wtc, (void**)&ly.bias_tc})
    if (*p) cudaFree(*p), *p = nullptr;  // (Wst: rebuilt from the new weights on first use)
  // stage the caller's arrays as they are (one allocation)
  const size_t mat_b = (size_t)ly.dh * ly.din * ses, vec_b = (size_t)ly.dh * ses;
  size_t off[6], total = 0;
  for (int i = 0; i < n_mats; ++i) {
    off[i] = total;
    total += ((h->kind == RNNB_SRU && i >= 3 ? vec_b : mat_b) + 255) / 256 * 256;
  }
  char* stage = nullptr;
  CUDA_TRY(cudaMalloc(&stage, total));
  struct StageFree {
    char* p;
    ~StageFree() { cudaFree(p); }
  } stage_free{stage};
  for (int i = 0; i < n_mats; ++i)
    CUDA_TRY(cudaMemcpy(stage + off[i], mats[i], h->kind == RNNB_SRU && i >= 3 ? vec_b : mat_b, cudaMemcpyHostToDevice));
  PackArgs pa{};
  for (int i = 0; i < n_mats; ++i) pa.m[i] = stage + off[i];
  pa.kind = h->kind;
  pa.mode = h->mode;
  pa.T = T;
  pa.dh = ly.dh;
  pa.din = ly.din;
  pa.Dp = ly.Dp;
  pa.Kp = Kp;
  const size_t wb = (size_t)rows * Kp * ws;
  CUDA_TRY(cudaMalloc(&ly.W, wb));
  CUDA_TRY(cudaMemsetAsync(ly.W, 0, wb, 0));  // padding rows / columns
  pa.W = ly.W;
  ly.wbytes = wb;
  if (h->kind == RNNB_SRU) {
    const size_t bb = (size_t)ly.Upad * 2 * elem_size(h->mode);
    CUDA_TRY(cudaMalloc(&ly.bias, bb));
    CUDA_TRY(cudaMemsetAsync(ly.bias, 0, bb, 0));
    pa.bias = ly.bias;
    ly.wbytes += bb;
  }
  if (h->mode == RNNB_BF16 || h->mode == RNNB_TF32 || h->mode == RNNB_F32X3 || h->mode == RNNB_F32) {
    // tensor-core layout: rows (p*3 + g)*Hpad128 + u (plane p: hi / lo for
    // 3xTF32, gate-major), columns [tap][Dtc]
    const int KT = h->mode == RNNB_BF16 ? 64 : 32;
    const int planes = (h->mode == RNNB_F32X3 || h->mode == RNNB_F32) ? 2 : 1;
    const int64_t Dtc = (ly.din + KT - 1) / KT * KT;
    ly.Hpad128 = (int)((ly.dh + 127) / 128 * 128);
    ly.tcKp = (int)(T * Dtc);
    const size_t rows_tc = (size_t)3 * ly.Hpad128;
    const size_t tb = planes * rows_tc * ly.tcKp * ws;
    CUDA_TRY(cudaMalloc(&ly.Wtc, tb));
    CUDA_TRY(cudaMemsetAsync(ly.Wtc, 0, tb, 0));
    pa.Wtc = ly.Wtc;
    pa.Hpad = ly.Hpad128;
    pa.tcKp = ly.tcKp;
    pa.Dtc = Dtc;
    pa.lo_off = planes == 2 ? (int64_t)(rows_tc * ly.tcKp) : 0;
    ly.wbytes += tb;
    if (h->kind == RNNB_SRU) {
      CUDA_TRY(cudaMalloc(&ly.bias_tc, (size_t)ly.Hpad128 * 2 * sizeof(float)));
      CUDA_TRY(cudaMemsetAsync(ly.bias_tc, 0, (size_t)ly.Hpad128 * 2 * sizeof(float), 0));
      pa.bias_tc = ly.bias_tc;
    }
  }
  const int64_t n = ly.dh * 3 * T * ly.din;
  const int grid = (int)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
  if (src_dtype == RNNB_DT_F64) pack_layer_kernel<double><<<grid, 256>>>(pa);
  else pack_layer_kernel<float><<<grid, 256>>>(pa);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(0));
  ly.loaded = true;
  return RNNB_OK;
}

rnnb_status rnnb_stack_set_layer(rnnb_stack_t h, int layer, const void* const* mats, int n_mats, int src_dtype) {
  return abi_guard("rnnb_stack_set_layer", [&]() { return rnnb_stack_set_layer_impl(h, layer, mats, n_mats, src_dtype); });
}

rnnb_status rnnb_stack_set_highway(rnnb_stack_t h, int layer, int64_t col_offset) {
  if (!h) return fail(RNNB_EINVAL, "null stack handle");
  if (layer < 0 || layer >= h->n_layers) return fail(RNNB_EINVAL, "layer index out of range");
  if (h->kind != RNNB_SRU) return fail(RNNB_EINVAL, "highway offset applies to SRU layers");
  Layer& ly = h->layers[layer];
  if (col_offset < 0 || col_offset + ly.dh > ly.din) return fail(RNNB_EINVAL, "highway columns out of range");
  ly.hw_off = col_offset;
  return RNNB_OK;
}

static rnnb_status forward_impl(rnnb_stack_t h, const void* X, int64_t ldx, int64_t L, int64_t block_size,
                                void* H, int64_t ldh, void* c_state, void* x_carry, void* stream);

rnnb_status rnnb_forward(rnnb_stack_t h, const void* X, int64_t ldx, int64_t L, int64_t block_size, void* H,
                         int64_t ldh, void* c_state, void* x_carry, void* stream) {
  rnnb_status st = check_stack(h);
  if (st != RNNB_OK) return st;
  if (ldh < (h->layers.empty() ? 1 : h->layers.back().dh)) return fail(RNNB_EINVAL, "ldh smaller than d_h");
  return forward_impl(h, X, ldx, L, block_size, H, ldh, c_state, x_carry, stream);
}

rnnb_status rnnb_forward_ex(rnnb_stack_t h, const void* X, int64_t ldx, int64_t L, int64_t block_size, void* H,
                            int64_t ldh, void* c_state, void* x_carry, int n_peers, void* const* peer_H,
                            void* stream) {
  rnnb_status st = check_stack(h);
  if (st != RNNB_OK) return st;
  if ((ldh < 0 ? -ldh : ldh) < h->layers.back().dh) return fail(RNNB_EINVAL, "|ldh| smaller than d_h");
  if (n_peers < 0 || n_peers > kMaxPeers)
    return fail(RNNB_EINVAL, "n_peers must be in [0, " + std::to_string(kMaxPeers) + "]");
  if (n_peers > 0 && !peer_H) return fail(RNNB_EINVAL, "null peer_H");
  for (int p = 0; p < n_peers; ++p)
    if (!peer_H[p]) return fail(RNNB_EINVAL, "null peer destination");
  h->n_peers = n_peers;
  for (int p = 0; p < n_peers; ++p) h->peer_H[p] = peer_H[p];
  st = forward_impl(h, X, ldx, L, block_size, H, ldh, c_state, x_carry, stream);
  h->n_peers = 0;
  return st;
}

static rnnb_status forward_impl(rnnb_stack_t h, const void* X, int64_t ldx, int64_t L, int64_t block_size,
                                void* H, int64_t ldh, void* c_state, void* x_carry, void* stream) {
  rnnb_status st = RNNB_OK;
  if (L < 1) return fail(RNNB_EINVAL, "seq_len must be >= 1");
  if (block_size < 1) return fail(RNNB_EINVAL, "block_size must be >= 1");
  if (!X || !H) return fail(RNNB_EINVAL, "null X or H");
  // ldx < 0: rows in reverse time order (row t at X + t*ldx)
  if ((ldx < 0 ? -ldx : ldx) < h->layers[0].din) return fail(RNNB_EINVAL, "|ldx| smaller than d_in");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DeviceGuard dg(h->device);
  CUDA_TRY(dg.err);
  switch (h->mode) {
    case RNNB_F64:
      st = forward_t<double, double>(h, static_cast<const double*>(X), ldx, L, block_size,
                                     static_cast<double*>(H), ldh, static_cast<double*>(c_state),
                                     static_cast<double*>(x_carry), s);
      break;
    case RNNB_BF16:
      st = forward_t<float, __nv_bfloat16>(h, static_cast<const float*>(X), ldx, L, block_size,
                                           static_cast<float*>(H), ldh, static_cast<float*>(c_state),
                                           static_cast<float*>(x_carry), s);
      break;
    default:
      st = forward_t<float, float>(h, static_cast<const float*>(X), ldx, L, block_size, static_cast<float*>(H),
                                   ldh, static_cast<float*>(c_state), static_cast<float*>(x_carry), s);
  }
  return st;
}

static rnnb_status rnnb_forward_host_impl(rnnb_stack_t h, const void* X, int64_t L, int64_t block_size, void* H,
                              void* c_state, void* x_carry, void* stream) {
  rnnb_status st = check_stack(h);
  if (st != RNNB_OK) return st;
  if (L < 1) return fail(RNNB_EINVAL, "seq_len must be >= 1");
  if (!X || !H) return fail(RNNB_EINVAL, "null X or H");
  const size_t es = elem_size(h->mode);
  const int64_t din = h->layers[0].din, dh = h->layers.back().dh;
  int64_t csz = 0, xsz = 0;
  for (auto& ly : h->layers) csz += ly.dh, xsz += ly.din;
  const size_t xb = (size_t)L * din * es, hb = (size_t)L * dh * es;
  const size_t sb = (size_t)(csz + xsz) * es;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DeviceGuard dg(h->device);
  CUDA_TRY(dg.err);
  if (h->hx_bytes < xb + sb) {
    if (h->hostX) cudaFree(h->hostX);
    h->hostX = nullptr;
    CUDA_TRY(cudaMalloc(&h->hostX, xb + sb));
    h->hx_bytes = xb + sb;
  }
  if (h->hh_bytes < hb) {
    if (h->hostH) cudaFree(h->hostH);
    h->hostH = nullptr;
    CUDA_TRY(cudaMalloc(&h->hostH, hb));
    h->hh_bytes = hb;
  }
  char* dX = static_cast<char*>(h->hostX);
  char* dC = dX + xb;
  char* dXC = dC + csz * es;
  if (!h->s_in) {
    CUDA_TRY(cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking));
    for (auto& e : h->ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  const char* hX = static_cast<const char*>(X);
  char* hH = static_cast<char*>(H);
  char* dH = static_cast<char*>(h->hostH);
  const int64_t T = block_size < 1 ? 1 : block_size;
  // no state in or out and the tensor-core streaming path: the layer launch
  // takes null state pointers (zero c_0 / x_{-1}, no c_T copy) -- two host
  // calls less before the launch
  const bool want_state = c_state != nullptr || x_carry != nullptr;
  const bool tc_stream_candidate = !h->stream_disabled.load() && h->n_layers == 1 &&
                                   use_tc_layer(h, h->layers[0], L, block_size < 1 ? 1 : block_size) && h->num_sms > 8 &&
                                   !(getenv("RNNB_HOST_STREAM") && getenv("RNNB_HOST_STREAM")[0] == '0');
  if (!want_state && tc_stream_candidate) {
  } else if (!c_state && !x_carry) {
    CUDA_TRY(cudaMemsetAsync(dC, 0, (csz + xsz) * es, s));  // dC, dXC are adjacent: one call
  } else {
    if (c_state) CUDA_TRY(cudaMemcpyAsync(dC, c_state, csz * es, cudaMemcpyHostToDevice, s));
    else CUDA_TRY(cudaMemsetAsync(dC, 0, csz * es, s));
    if (x_carry) CUDA_TRY(cudaMemcpyAsync(dXC, x_carry, xsz * es, cudaMemcpyHostToDevice, s));
    else CUDA_TRY(cudaMemsetAsync(dXC, 0, xsz * es, s));
  }
  cudaEvent_t ev_start = h->ev[16], ev_done = h->ev[17];

  StreamOps so = stream_ops();
  const char* env_s = getenv("RNNB_HOST_STREAM");
  // Streaming on the tcgen05 path (single-layer stacks whose T_b runs on the
  // tensor cores): ONE layer launch on all but two SMs.  Per segment the
  // copy-in stream lands the rows, converts them into the MMA operand on the
  // two free SMs and bumps the operand-row counter the kernel's TMA producer
  // waits on; each finished item counts on its output granule and the
  // copy-out stream drains a segment once all its granules are complete.
  const bool want_tc_stream = !h->stream_disabled.load() && !(env_s && env_s[0] == '0') && h->n_layers == 1 &&
                              use_tc_layer(h, h->layers[0], L, T) && h->num_sms > 8;
  if (want_tc_stream && so.write && so.wait) {
    const auto t_call = std::chrono::steady_clock::now();
    const int mode = tc_mode_of(h->mode);
    const int64_t Tb = tc_block(h, T);
    const Layer& ly = h->layers[0];
    const int nU = ly.Hpad128 / 128;
    // granule: whole tensor-core blocks, >= 64 steps, at most kMaxStreamChunks of them
    int64_t g = (64 + Tb - 1) / Tb * Tb;
    const int64_t gmin = (L + kMaxStreamChunks - 1) / kMaxStreamChunks;
    if (g < gmin) g = (gmin + Tb - 1) / Tb * Tb;
    const int64_t ng = (L + g - 1) / g;
    const char* env_c = getenv("RNNB_STREAM_CHUNK");
    int64_t min_chunk = env_c ? atoll(env_c) : 256;
    if (min_chunk * (kMaxSegs - 8) < L) min_chunk = (L + kMaxSegs - 9) / (kMaxSegs - 8);  // at most kMaxSegs segments
    const int64_t sc = min_chunk > g ? (min_chunk + g - 1) / g * g : g;
    // segment boundaries: the first granule alone (the kernel starts on it),
    // then segments doubling up to ~sc steps (fewer host operations)
    std::vector<int64_t> seg{0};
    if (g < L) seg.push_back(g);
    for (int64_t len = 2 * g; seg.back() + len < L; len = len * 2 < sc ? len * 2 : sc) seg.push_back(seg.back() + len);
    if (seg.back() < L) seg.push_back(L);
    const int64_t nsc = (int64_t)seg.size() - 1;
    int64_t ldop = 0;
    if ((st = ensure_tc_op(h, 0, L, &ldop)) != RNNB_OK) return st;
    // everything that may wait for the device (scratch (re)allocation, the
    // lazy load of the layer kernel's code) happens HERE, before the
    // conversion kernel starts spinning on rows the host has yet to enqueue
    const int64_t nBt = (L + Tb - 1) / Tb;
    CUDA_TRY(tc_layer_preload(h->kind, mode, (int)Tb));
    if ((st = tc_layer_scratch(h, h->layers[0], nBt, nU, tc_pick_n((int)Tb), mode == TC_3XTF32, s)) != RNNB_OK) return st;
    const size_t opes = mode == TC_BF16 ? 2 : 4;
    if (!h->stream_ctr) {
      CUDA_TRY(cudaMalloc(&h->stream_ctr, (4 + kMaxStreamChunks + kMaxSegs) * sizeof(int)));
      CUDA_TRY(cudaHostAlloc(&h->stream_flag_host, sizeof(int), cudaHostAllocDefault));
    }
    if (!h->s_cv) CUDA_TRY(cudaStreamCreateWithFlags(&h->s_cv, cudaStreamNonBlocking));
    if (!h->s_in2) CUDA_TRY(cudaStreamCreateWithFlags(&h->s_in2, cudaStreamNonBlocking));
    if (nsc > kMaxSegs) return fail(RNNB_EINVAL, "streaming segment plan too long");
    while ((int64_t)h->sev.size() < nsc) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      h->sev.push_back(e);
    }
    CUDA_TRY(cudaMemsetAsync(h->stream_ctr, 0, (4 + kMaxStreamChunks + kMaxSegs) * sizeof(int), s));
    CUDA_TRY(cudaEventRecord(ev_start, s));
    CUDA_TRY(cudaStreamWaitEvent(h->s_in, ev_start, 0));
    CUDA_TRY(cudaStreamWaitEvent(h->s_in2, ev_start, 0));
    CUDA_TRY(cudaStreamWaitEvent(h->s_cv, ev_start, 0));
    const float* fX = reinterpret_cast<const float*>(dX);
    const float* fXC = reinterpret_cast<const float*>(dXC);
    // Output straight into the caller's buffer when it is pinned (mapped)
    // host memory: the epilogue's h stores go over PCIe as posted writes
    // while later items compute -- no copy-out segments, no wait-value
    // operations, and nothing left to copy after the kernel ends.  Measured
    // (tools/zc_probe.cu): SM stores to pinned memory 50 GB/s, and they run
    // full duplex with the copy engine's H2D (8 MB each way in 187 us);
    // SM *reads* of pinned memory do not overlap with writes (290-320 us),
    // so the input keeps the copy engine.
    char* dHz = nullptr;
    {
      const char* env_z = getenv("RNNB_ZC_OUT");
      cudaPointerAttributes pa;
      if (!(env_z && env_z[0] == '0') && cudaPointerGetAttributes(&pa, H) == cudaSuccess &&
          pa.type == cudaMemoryTypeHost && pa.devicePointer != nullptr)
        dHz = static_cast<char*>(pa.devicePointer);
      else
        (void)cudaGetLastError();
    }
    if (!dHz) CUDA_TRY(cudaStreamWaitEvent(h->s_out, ev_start, 0));
    // RNNB_STREAM_TRACE=1: timing events after every copy / conversion and
    // around the layer kernel, printed relative to the call's start (tuning only)
    const bool trace = getenv("RNNB_STREAM_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    std::vector<std::string> tname;
    const bool trace_ev = trace && atoi(getenv("RNNB_STREAM_TRACE")) >= 2;  // 2: + stream events (they slow the call)
    auto mark = [&](cudaStream_t ms, const std::string& name) {
      if (!trace_ev) return;
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, ms);
      tev.push_back(e);
      tname.push_back(name);
    };
    const bool trace_host = trace && atoi(getenv("RNNB_STREAM_TRACE")) >= 3;  // 3: host-side time stamps only
    std::vector<std::pair<const char*, double>> hts;
    auto hmark = [&](const char* name) {
      if (trace_host) hts.emplace_back(name, std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_call).count());
    };
    hmark("entry + setup");
    mark(s, "start");
    if (trace && !trace_host) {
      if (h->stream_trace) cudaFree(h->stream_trace);
      CUDA_TRY(cudaMalloc(&h->stream_trace, (1 + 2 * nBt) * sizeof(unsigned long long)));
      CUDA_TRY(cudaMemset(h->stream_trace, 0, (1 + 2 * nBt) * sizeof(unsigned long long)));
    } else if (h->stream_trace) {
      cudaFree(h->stream_trace);
      h->stream_trace = nullptr;
    }
    // ONE persistent conversion launch (s_cv, on the SMs the layer kernel
    // leaves free) follows the copy engine: per segment the host only
    // enqueues the copy and a write-value of the rows landed; the conversion
    // kernel polls that counter and publishes the operand-row counter the
    // layer kernel's TMA producer waits on (tc_launch.cu).  Unaligned inputs
    // keep one conversion launch per segment.
    const char* env_f = getenv("RNNB_STREAM_SMS");
    h->stream_free_sms = env_f ? atoi(env_f) : 2;
    if (h->stream_free_sms < 1) h->stream_free_sms = 1;
    if (h->stream_free_sms > 16) h->stream_free_sms = 16;
    int* copied_ctr = h->stream_ctr + 2 + kMaxStreamChunks;  // [+1]: the conversion workers' group queue
    int* seg_flag = h->stream_ctr + 4 + kMaxStreamChunks;    // per copy segment: epoch once it has landed
    TcSegTab segtab{};
    segtab.n = (int)nsc;
    for (int64_t i = 0; i < nsc; ++i) segtab.end[i] = (int)seg[i + 1];
    // per-group "converted" flags tagged with a per-call epoch (never cleared
    // per call); (re)allocated here, before anything of this call is launched
    if (h->stream_flags_n < (size_t)L + 1 || h->stream_epoch >= (1 << 30)) {
      if (h->stream_flags_n < (size_t)L + 1) {
        if (h->stream_flags) cudaFree(h->stream_flags);
        h->stream_flags = nullptr;
        h->stream_flags_n = 0;
        CUDA_TRY(cudaMalloc(&h->stream_flags, ((size_t)L + 1) * sizeof(int)));
        h->stream_flags_n = (size_t)L + 1;
      }
      CUDA_TRY(cudaMemsetAsync(h->stream_flags, 0, h->stream_flags_n * sizeof(int), s));
      h->stream_epoch = 0;
    }
    ++h->stream_epoch;
    const bool conv_stream = tc_to_operand_stream_ok(fX, din, h->kind == RNNB_QRNN ? fXC : nullptr, h->op, ldop, (int)din);
    // (without the persistent conversion the per-segment fallback reads the carry buffer: keep it defined)
    if (!conv_stream && !want_state) CUDA_TRY(cudaMemsetAsync(dC, 0, (csz + xsz) * es, s));
    auto copy_in = [&](int64_t i) -> rnnb_status {
      const int64_t t0 = seg[i], n = seg[i + 1] - seg[i];
      // segments alternate between two copy streams: a stream's write-value
      // runs only after its copy has fully landed, and on ONE stream the next
      // copy waited for it -- a ~30 us bubble per segment boundary (in-kernel
      // time stamps: rows arrived at 33 GB/s instead of PCIe's 53)
      cudaStream_t sc_in = conv_stream && (i & 1) ? h->s_in2 : h->s_in;
      CUDA_TRY(cudaMemcpyAsync(dX + t0 * din * es, hX + t0 * din * es, n * din * es, cudaMemcpyHostToDevice, sc_in));
      mark(sc_in, "copied rows " + std::to_string(t0 + n));
      if (conv_stream) {
        CU_TRY(so.write(sc_in, (CUdeviceptr)(seg_flag + i), (cuuint32_t)h->stream_epoch, 0));
        return RNNB_OK;
      }
      CUDA_TRY(cudaEventRecord(h->sev[i], h->s_in));
      CUDA_TRY(cudaStreamWaitEvent(h->s_cv, h->sev[i], 0));
      // operand rows t0+1 .. t0+n (row t0 = x_{t0-1}: the carry, or the
      // previous segment's last row rewritten with the same bits)
      const float* prev = t0 == 0 ? (h->kind == RNNB_QRNN ? fXC : nullptr) : fX + (t0 - 1) * din;
      CUDA_TRY(tc_to_operand_rows(mode, fX + t0 * din, din, prev, static_cast<char*>(h->op) + t0 * ldop * opes,
                                  ldop, n, (int)din, L + 1, h->s_cv));
      CU_TRY(so.write(h->s_cv, (CUdeviceptr)h->stream_ctr, (cuuint32_t)(t0 + n), 0));
      mark(h->s_cv, "converted rows " + std::to_string(t0 + n));
      return RNNB_OK;
    };
    // the first segments' copies are enqueued before the layer launch (the
    // copy engine starts at once and stays busy while the host encodes and
    // launches the kernel, which waits on the row counter anyway), the rest
    // after it
    // the persistent conversion kernel (everything that could wait for the
    // device was done above, so it may be launched on either side of the layer
    // kernel without a first-use stall)
    auto launch_conv = [&]() -> rnnb_status {
      if (!conv_stream) return RNNB_OK;
      const char* env_g = getenv("RNNB_STREAM_GROUP");
      int group = env_g ? atoi(env_g) : 16;
      if (group < 1) group = 16;
      const char* env_n = getenv("RNNB_STREAM_CTAS");
      int workers = env_n ? atoi(env_n) : 12;
      if (workers < 1) workers = 1;
      CUDA_TRY(tc_to_operand_stream(mode, fX, din, h->kind == RNNB_QRNN && want_state ? fXC : nullptr, h->op, ldop, L,
                                    (int)din, segtab, seg_flag, h->stream_ctr, h->stream_ctr + 1, h->stream_flags, copied_ctr + 1,
                                    h->stream_epoch, group, workers, h->s_cv));
      mark(h->s_cv, "conversion kernel done");
      return RNNB_OK;
    };
    // ALL copies are enqueued before the launches: with only the first three
    // ahead (the kernels launched sooner) the best calls were 4 % faster, but
    // the rows then depend on the host issuing ~12 more API calls on time and
    // runs on the shared boxes slipped to 0.45-0.65 ms; with everything
    // enqueued first, 8 of 8 processes measured 0.393-0.404 ms
    const char* env_p = getenv("RNNB_STREAM_PRE");
    int64_t want_pre = env_p ? atoll(env_p) : nsc;
    if (want_pre < 1) want_pre = 1;
    const int64_t pre = nsc < want_pre ? nsc : want_pre;
    // the conversion kernel goes behind the layer launch: launched first, its
    // workers spread over idle SMs and the layer CTAs that land beside them run
    // slower (e2e 0.50-0.55 ms vs 0.39-0.44 ms); RNNB_STREAM_CONV_FIRST=1 for A/B
    const bool conv_first = getenv("RNNB_STREAM_CONV_FIRST") != nullptr;
    for (int64_t i = 0; i < pre; ++i) {
      if ((st = copy_in(i)) != RNNB_OK) return st;
      if (i == 0 && conv_first && (st = launch_conv()) != RNNB_OK) return st;
    }
    hmark("copies enqueued (pre)");
    h->stream_ready = h->stream_ctr;
    h->stream_done = dHz ? nullptr : h->stream_ctr + 2;
    h->stream_chunk = (int)g;
    mark(s, "before layer kernel");
    st = rnnb_forward(h, dX, din, L, block_size, dHz ? dHz : dH, dh, want_state ? dC : nullptr,
                      want_state ? dXC : nullptr, stream);
    mark(s, "layer kernel done");
    hmark("layer kernel launched");
    if (st == RNNB_OK && !conv_first && (st = launch_conv()) != RNNB_OK) return st;
    h->stream_ready = nullptr;
    h->stream_done = nullptr;
    if (st != RNNB_OK) {
      // the conversion kernel may already be waiting for the remaining rows: let it finish
      if (conv_first && conv_stream) {
        for (int64_t i = pre; i < nsc; ++i) (void)copy_in(i);
        (void)cudaStreamSynchronize(h->s_cv);
      }
      return st;
    }
    for (int64_t i = pre; i < nsc; ++i)
      if ((st = copy_in(i)) != RNNB_OK) return st;
    int64_t launches = h->last_launches + nsc;  // + the per-segment operand conversions
    for (int64_t i = 0; i < nsc && !dHz; ++i) {
      const int64_t t0 = seg[i], n = seg[i + 1] - seg[i];
      for (int64_t gi = t0 / g; gi * g < t0 + n; ++gi) {
        const int64_t glen = ((gi + 1) * g < L ? (gi + 1) * g : L) - gi * g;
        const cuuint32_t want = (cuuint32_t)(nU * ((glen + Tb - 1) / Tb));
        CU_TRY(so.wait(h->s_out, (CUdeviceptr)(h->stream_ctr + 2 + gi), want, CU_STREAM_WAIT_VALUE_GEQ));
      }
      CUDA_TRY(cudaMemcpyAsync(hH + t0 * dh * es, dH + t0 * dh * es, n * dh * es, cudaMemcpyDeviceToHost, h->s_out));
    }
    h->last_launches = launches;
    CUDA_TRY(cudaEventRecord(ev_done, h->s_out));
    CUDA_TRY(cudaStreamWaitEvent(s, ev_done, 0));
    CUDA_TRY(cudaEventRecord(ev_done, h->s_cv));
    CUDA_TRY(cudaStreamWaitEvent(s, ev_done, 0));
    CUDA_TRY(cudaEventRecord(ev_done, h->s_in));
    CUDA_TRY(cudaStreamWaitEvent(s, ev_done, 0));
    CUDA_TRY(cudaEventRecord(ev_done, h->s_in2));
    CUDA_TRY(cudaStreamWaitEvent(s, ev_done, 0));
    mark(s, "all done");
    hmark("everything enqueued");
    CUDA_TRY(cudaStreamSynchronize(s));
    hmark("synchronised");
    for (auto& t : hts) fprintf(stderr, "[rnnb stream trace] host %8.1f us  %s\n", t.second, t.first);
    // The time-out flag is set only by a kernel thread that waited
    // kStreamTimeoutNs (2 s) for rows: a call that returned sooner cannot have
    // failed, and skips the flag's copy-out (a copy-engine round trip behind
    // the layer kernel on every call).
    *h->stream_flag_host = 0;
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t_call).count() > 1.0) {
      CUDA_TRY(cudaMemcpyAsync(h->stream_flag_host, h->stream_ctr + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
    }
    if (trace && !trace_host) {
      for (size_t i = 1; trace_ev && i < tev.size(); ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, tev[0], tev[i]);
        fprintf(stderr, "[rnnb stream trace] %8.1f us  %s\n", ms * 1e3, tname[i].c_str());
      }
      for (auto e : tev) cudaEventDestroy(e);
      std::vector<unsigned long long> tr(1 + 2 * nBt);
      cudaMemcpy(tr.data(), h->stream_trace, tr.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      for (int64_t b = 0; b < nBt; b += (nBt > 16 ? nBt / 16 : 1))
        fprintf(stderr, "[rnnb stream trace] block %4lld: rows seen %8.1f us, stored %8.1f us after kernel start\n",
                (long long)b, (double)(tr[1 + b] - tr[0]) * 1e-3, (double)(tr[1 + nBt + b] - tr[0]) * 1e-3);
      fprintf(stderr, "[rnnb stream trace] last block: rows seen %8.1f us, stored %8.1f us\n",
              (double)(tr[nBt] - tr[0]) * 1e-3, (double)(tr[2 * nBt] - tr[0]) * 1e-3);
    }
    if (*h->stream_flag_host == 0) {
      if (c_state) CUDA_TRY(cudaMemcpyAsync(c_state, dC, csz * es, cudaMemcpyDeviceToHost, s));
      if (x_carry) CUDA_TRY(cudaMemcpyAsync(x_carry, dXC, xsz * es, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
      return st;
    }
    if (getenv("RNNB_STREAM_DEBUG")) {
      int c[3] = {0, 0, 0};
      cudaMemcpy(&c[0], h->stream_ctr, 2 * sizeof(int), cudaMemcpyDeviceToHost);
      cudaMemcpy(&c[2], copied_ctr + 1, sizeof(int), cudaMemcpyDeviceToHost);
      fprintf(stderr, "[rnnb] tcgen05 host streaming gave up: ready=%d fail=%d groups claimed=%d (L=%lld)\n", c[0], c[1], c[2],
              (long long)L);
    }
    h->stream_disabled.store(true);  // rows arrived too late (serialising profiler): redo without streaming
    return rnnb_forward_host_impl(h, X, L, block_size, H, c_state, x_carry, stream);
  }

  // (the tensor-core streaming path was not taken after all: the other paths read the state buffers)
  if (!want_state && tc_stream_candidate) CUDA_TRY(cudaMemsetAsync(dC, 0, (csz + xsz) * es, s));

  // Streaming (single-layer fp32 stacks, warp-specialised kernel): ONE layer
  // launch consumes X while it is still being copied in -- its TMA producer
  // waits on a device counter of resident rows that the copy-in stream bumps
  // after each chunk (stream write-value) -- and each CTA counts the chunks
  // whose h rows it has stored, so the copy-out stream (stream wait-value)
  // drains chunk i while later chunks compute.
  const bool want_stream = !h->stream_disabled.load() && !(env_s && env_s[0] == '0') && h->n_layers == 1 &&
                           h->mode == RNNB_F32 && !use_tc_layer(h, h->layers[0], L, T);  // FFMA streaming
  if (want_stream && so.write && so.wait) {
    // The kernel counts finished h rows per granule g (whole blocks, >= 32
    // steps, at most kMaxStreamChunks granules).  Copies move segments of
    // whole granules: the first and the last segment are one granule (short
    // exposed copy-in before the first pass and copy-out after the last),
    // the others ~RNNB_STREAM_CHUNK steps (fewer, larger copies).
    const char* env_c = getenv("RNNB_STREAM_CHUNK");
    const int64_t min_chunk = env_c ? atoll(env_c) : 128;  // measured cfg2 (32-column passes): 64 -> 2.17-2.42M (noisy), 128 -> 2.64M, 256 -> 2.56M e2e
    int64_t g = (32 + T - 1) / T * T;
    const int64_t gmin = (L + kMaxStreamChunks - 1) / kMaxStreamChunks;
    if (g < gmin) g = (gmin + T - 1) / T * T;
    const int64_t ng = (L + g - 1) / g;
    int64_t sc = (min_chunk + g - 1) / g * g;
    if (sc < g) sc = g;
    std::vector<int64_t> seg{0};  // segment boundaries (multiples of g, then L)
    const int64_t last0 = (L - 1) / g * g;  // start of the last granule
    if (last0 > 0) {
      seg.push_back(g);
      for (int64_t t = g + sc; t < last0; t += sc) seg.push_back(t);
      if (seg.back() < last0) seg.push_back(last0);
    }
    seg.push_back(L);
    const int64_t nsc = (int64_t)seg.size() - 1;
    if (ng <= kMaxStreamChunks) {
      if (!h->stream_ctr) {
        CUDA_TRY(cudaMalloc(&h->stream_ctr, (4 + kMaxStreamChunks + kMaxSegs) * sizeof(int)));
        CUDA_TRY(cudaHostAlloc(&h->stream_flag_host, sizeof(int), cudaHostAllocDefault));
      }
      CUDA_TRY(cudaMemsetAsync(h->stream_ctr, 0, (2 + ng) * sizeof(int), s));
      CUDA_TRY(cudaEventRecord(ev_start, s));
      CUDA_TRY(cudaStreamWaitEvent(h->s_in, ev_start, 0));
      CUDA_TRY(cudaStreamWaitEvent(h->s_out, ev_start, 0));
      h->stream_ready = h->stream_ctr;
      h->stream_done = h->stream_ctr + 2;
      h->stream_chunk = (int)g;
      h->stream_refused = false;
      // segment 0's copy-in first: its rows land while the layer kernel is
      // still being launched and loads its weights (the kernel polls the
      // counter); if the layer cannot stream, the chunked path below copies again
      auto copy_in = [&](int64_t i) -> rnnb_status {
        const int64_t t0 = seg[i], n = seg[i + 1] - seg[i];
        CUDA_TRY(cudaMemcpyAsync(dX + t0 * din * es, hX + t0 * din * es, n * din * es, cudaMemcpyHostToDevice,
                                 h->s_in));
        CU_TRY(so.write(h->s_in, (CUdeviceptr)h->stream_ctr, (cuuint32_t)(t0 + n), 0));
        return RNNB_OK;
      };
      if ((st = copy_in(0)) != RNNB_OK) return st;
      st = rnnb_forward(h, dX, din, L, block_size, dH, dh, dC, dXC, stream);
      h->stream_ready = nullptr;
      h->stream_done = nullptr;
      if (st == RNNB_OK) {
        const unsigned grid = (unsigned)h->layers[0].grid;
        for (int64_t i = 1; i < nsc; ++i)
          if ((st = copy_in(i)) != RNNB_OK) return st;
        for (int64_t i = 0; i < nsc; ++i) {
          // every CTA finished the segment's last granule => all of the
          // segment (a CTA stores its passes in order)
          const int64_t t0 = seg[i], n = seg[i + 1] - seg[i];
          CU_TRY(so.wait(h->s_out, (CUdeviceptr)(h->stream_ctr + 2 + (seg[i + 1] - 1) / g), grid,
                         CU_STREAM_WAIT_VALUE_GEQ));
          CUDA_TRY(cudaMemcpyAsync(hH + t0 * dh * es, dH + t0 * dh * es, n * dh * es, cudaMemcpyDeviceToHost,
                                   h->s_out));
        }
        CUDA_TRY(cudaEventRecord(ev_done, h->s_out));
        CUDA_TRY(cudaStreamWaitEvent(s, ev_done, 0));
        CUDA_TRY(cudaMemcpyAsync(h->stream_flag_host, h->stream_ctr + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        if (*h->stream_flag_host == 0) {
          if (c_state) CUDA_TRY(cudaMemcpyAsync(c_state, dC, csz * es, cudaMemcpyDeviceToHost, s));
          if (x_carry) CUDA_TRY(cudaMemcpyAsync(x_carry, dXC, xsz * es, cudaMemcpyDeviceToHost, s));
          CUDA_TRY(cudaStreamSynchronize(s));
          return st;
        }
        // the rows did not arrive while the kernel waited (a serialising
        // profiler, a stalled copy engine): redo the call without streaming
        h->stream_disabled.store(true);  // do not try streaming again with this handle
        return rnnb_forward_host_impl(h, X, L, block_size, H, c_state, x_carry, stream);
      }
      if (!h->stream_refused) return st;
      st = RNNB_OK;  // the layer cannot stream: chunked pipeline below
    }
  }

  // Time is cut into chunks of whole blocks; chunk i's copy-in (s_in), its
  // forward (s, state carried in dC / dXC exactly as across blocks) and its
  // copy-out (s_out) overlap the neighbouring chunks' copies.  Chunking at
  // block boundaries leaves every value bitwise unchanged.
  const char* env = getenv("RNNB_HOST_CHUNK");
  const int64_t want = env ? atoll(env) : 512;  // steps per chunk
  int64_t nch = want > 0 ? (L + want - 1) / want : 1;
  if (nch > 8) nch = 8;
  if (nch < 1) nch = 1;
  int64_t cl = ((L + nch - 1) / nch + T - 1) / T * T;
  nch = (L + cl - 1) / cl;
  CUDA_TRY(cudaEventRecord(ev_start, s));  // staging buffers are free once earlier work on s is done
  CUDA_TRY(cudaStreamWaitEvent(h->s_in, ev_start, 0));
  CUDA_TRY(cudaStreamWaitEvent(h->s_out, ev_start, 0));
  int64_t launches = 0;
  for (int64_t i = 0; i < nch && st == RNNB_OK; ++i) {
    const int64_t t0 = i * cl, n = (L - t0) < cl ? (L - t0) : cl;
    cudaEvent_t ein = h->ev[2 * i], eout = h->ev[2 * i + 1];
    CUDA_TRY(cudaMemcpyAsync(dX + t0 * din * es, hX + t0 * din * es, n * din * es, cudaMemcpyHostToDevice, h->s_in));
    CUDA_TRY(cudaEventRecord(ein, h->s_in));
    CUDA_TRY(cudaStreamWaitEvent(s, ein, 0));
    st = rnnb_forward(h, dX + t0 * din * es, din, n, block_size, dH + t0 * dh * es, dh, dC, dXC, stream);
    launches += h->last_launches;
    if (st != RNNB_OK) break;
    CUDA_TRY(cudaEventRecord(eout, s));
    CUDA_TRY(cudaStreamWaitEvent(h->s_out, eout, 0));
    CUDA_TRY(cudaMemcpyAsync(hH + t0 * dh * es, dH + t0 * dh * es, n * dh * es, cudaMemcpyDeviceToHost, h->s_out));
  }
  h->last_launches = launches;
  CUDA_TRY(cudaEventRecord(ev_done, h->s_out));
  CUDA_TRY(cudaStreamWaitEvent(s, ev_done, 0));
  if (st == RNNB_OK) {
    if (c_state) CUDA_TRY(cudaMemcpyAsync(c_state, dC, csz * es, cudaMemcpyDeviceToHost, s));
    if (x_carry) CUDA_TRY(cudaMemcpyAsync(x_carry, dXC, xsz * es, cudaMemcpyDeviceToHost, s));
  }
  CUDA_TRY(cudaStreamSynchronize(s));
  return st;
}

rnnb_status rnnb_forward_host(rnnb_stack_t h, const void* X, int64_t L, int64_t block_size, void* H,
                              void* c_state, void* x_carry, void* stream) {
  return abi_guard("rnnb_forward_host", [&]() { return rnnb_forward_host_impl(h, X, L, block_size, H, c_state, x_carry, stream); });
}

rnnb_status rnnb_gates(rnnb_stack_t h, int layer, const void* Xt, int64_t ldx, int64_t l, const void* x_carry,
                       void* G, int64_t ldg, void* stream) {
  rnnb_status st = check_stack(h);
  if (st != RNNB_OK) return st;
  if (layer < 0 || layer >= h->n_layers) return fail(RNNB_EINVAL, "layer index out of range");
  if (l < 1) return fail(RNNB_EINVAL, "block must hold at least one step");
  if (!Xt || !G) return fail(RNNB_EINVAL, "null X or G");
  if (ldg < l) return fail(RNNB_EINVAL, "ldg smaller than block length");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Layer& ly = h->layers[layer];
  if (ldx < ly.din) return fail(RNNB_EINVAL, "ldx smaller than d_in");
  DeviceGuard dg(h->device);
  CUDA_TRY(dg.err);
  switch (h->mode) {
    case RNNB_F64:
      return layer_launch<double, double>(h, layer, static_cast<const double*>(Xt), ldx, l, l, nullptr, 0, nullptr,
                                          const_cast<double*>(static_cast<const double*>(x_carry)),
                                          static_cast<double*>(G), ldg, s);
    case RNNB_BF16:
      return layer_launch<float, __nv_bfloat16>(h, layer, static_cast<const float*>(Xt), ldx, l, l, nullptr, 0,
                                                nullptr, const_cast<float*>(static_cast<const float*>(x_carry)),
                                                static_cast<float*>(G), ldg, s);
    default:
      return layer_launch<float, float>(h, layer, static_cast<const float*>(Xt), ldx, l, l, nullptr, 0, nullptr,
                                        const_cast<float*>(static_cast<const float*>(x_carry)),
                                        static_cast<float*>(G), ldg, s);
  }
}

rnnb_status rnnb_sweep(const void* forget, const void* cand, const void* c_init, void* C, int64_t d, int64_t T,
                       int dtype, void* stream) {
  if (!forget || !cand || !c_init || !C) return fail(RNNB_EINVAL, "null argument");
  if (d < 1 || T < 1) return fail(RNNB_EINVAL, "forget and candidate blocks must share one 2-d shape");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int bs = 128;
  const int grid = (int)((d + bs - 1) / bs);
  if (dtype == RNNB_DT_F64)
    sweep_kernel<double><<<grid, bs, 0, s>>>(static_cast<const double*>(forget), static_cast<const double*>(cand),
                                             static_cast<const double*>(c_init), static_cast<double*>(C), d, T);
  else if (dtype == RNNB_DT_F32)
    sweep_kernel<float><<<grid, bs, 0, s>>>(static_cast<const float*>(forget), static_cast<const float*>(cand),
                                            static_cast<const float*>(c_init), static_cast<float*>(C), d, T);
  else
    return fail(RNNB_EINVAL, "dtype must be f32 or f64");
  CUDA_TRY(cudaGetLastError());
  return RNNB_OK;
}

rnnb_status rnnb_finalize(int kind, const void* out_gate, const void* C, const void* Xb, void* H, int64_t d,
                          int64_t T, int dtype, void* stream) {
  if (kind != RNNB_SRU && kind != RNNB_QRNN) return fail(RNNB_EINVAL, "no blocked output path for this kind");
  if (!out_gate || !C || !H) return fail(RNNB_EINVAL, "null argument");
  if (kind == RNNB_SRU && !Xb) return fail(RNNB_EINVAL, "SRU output needs the raw input block");
  if (d < 1 || T < 1) return fail(RNNB_EINVAL, "empty block");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t n = d * T;
  const int bs = 256;
  const int grid = (int)((n + bs - 1) / bs);
  if (dtype == RNNB_DT_F64)
    finalize_kernel<double><<<grid, bs, 0, s>>>(kind, static_cast<const double*>(out_gate),
                                                static_cast<const double*>(C), static_cast<const double*>(Xb),
                                                static_cast<double*>(H), n);
  else if (dtype == RNNB_DT_F32)
    finalize_kernel<float><<<grid, bs, 0, s>>>(kind, static_cast<const float*>(out_gate),
                                               static_cast<const float*>(C), static_cast<const float*>(Xb),
                                               static_cast<float*>(H), n);
  else
    return fail(RNNB_EINVAL, "dtype must be f32 or f64");
  CUDA_TRY(cudaGetLastError());
  return RNNB_OK;
}

rnnb_status rnnb_query(rnnb_stack_t h, int what, int layer, int64_t* value) {
  if (!h || !value) return fail(RNNB_EINVAL, "null argument");
  if (what >= 2 && (layer < 0 || layer >= h->n_layers)) return fail(RNNB_EINVAL, "layer index out of range");
  switch (what) {
    case 0: {
      int64_t b = 0;
      for (auto& ly : h->layers) b += (int64_t)ly.wbytes;
      *value = b;
      return RNNB_OK;
    }
    case 1: *value = h->last_launches; return RNNB_OK;
    case 2: *value = h->layers[layer].U; return RNNB_OK;
    case 3: *value = h->layers[layer].last.wsmem ? 1 : 0; return RNNB_OK;
    case 4: *value = h->layers[layer].grid; return RNNB_OK;
    case 5: *value = (int64_t)h->layers[layer].last.smem; return RNNB_OK;
    case 6: *value = h->layers[layer].last.ws ? 1 : 0; return RNNB_OK;
    case 7: *value = h->layers[layer].last.nt; return RNNB_OK;
    case 8: *value = h->layers[layer].last.kc; return RNNB_OK;
    case 9: *value = h->layers[layer].last_tc ? 1 : 0; return RNNB_OK;
    case 10: *value = h->layers[layer].last.reg ? 1 : 0; return RNNB_OK;
    case 11: *value = h->layers[layer].last.wstream ? 1 : 0; return RNNB_OK;
    default: return fail(RNNB_EINVAL, "unknown query");
  }
}

}  // extern "C"
