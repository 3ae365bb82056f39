// Host-side launch of the FFMA layer kernel: picks the pass width NT from
// T_b, the shared-memory plan (weights resident or streamed from L2) and
// instantiates the kernel for one (accumulate, weight) type pair.
#pragma once
#include <cstdlib>
#include "ffma_reg.cuh"

namespace rnnb {

constexpr size_t kMaxSmem = 227 * 1024;

inline int pick_nt(int T_b) {
  if (T_b >= 16) return 16;
  int n = 1;
  while (n < T_b) n <<= 1;
  return n;
}

template <typename TA, typename TW, int CELL, int NT, int U, bool WSMEM>
static cudaError_t launch_one(const LayerArgs<TA, TW>& a, int grid, size_t smem, cudaStream_t s) {
  auto k = ffma_layer_kernel<TA, TW, CELL, NT, U, WSMEM>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  k<<<grid, kThreads, smem, s>>>(a);
  return cudaGetLastError();
}

struct FfmaPlan {
  int nt = 1;
  bool wsmem = false;
  bool ws = false;  // warp-specialised TMA/mbarrier kernel (ffma_ws.cuh)
  bool reg = false; // register-resident weights kernel (ffma_reg.cuh)
  bool wstream = false;  // ws kernel with per-chunk weight images streamed through the ring
  int grid = 0;          // CTAs launched when it differs from ceil(H / U)
  int kc = 0;
  size_t smem = 0;
};

template <typename TA, typename TW, int CELL, int NT, int U, int XR>
static cudaError_t launch_ws_xr(const LayerArgs<TA, TW>& a, const CUtensorMap& tm, int grid, size_t smem,
                                cudaStream_t s) {
  auto k = ffma_ws_kernel<TA, TW, CELL, NT, U, XR>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  if constexpr (XR == XR_NONE && sizeof(TA) == 4 && sizeof(TW) == 4) {
    if (a.x_ready != nullptr) {
      auto ks = ffma_ws_kernel<TA, TW, CELL, NT, U, XR, true>;
      static bool attr_s = false;
      if (!attr_s) {
        cudaError_t e = cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem);
        if (e != cudaSuccess) return e;
        attr_s = true;
      }
      ks<<<grid, WsCfg<TA, TW, CELL, NT, U>::THREADS, smem, s>>>(a, tm);
      return cudaGetLastError();
    }
  } else {
    if (a.x_ready != nullptr) return cudaErrorNotSupported;
  }
  k<<<grid, WsCfg<TA, TW, CELL, NT, U>::THREADS, smem, s>>>(a, tm);
  return cudaGetLastError();
}

// x rounding is a template parameter of the warp-specialised kernel
template <typename TA, typename TW, int CELL, int NT, int U>
static cudaError_t launch_ws(const LayerArgs<TA, TW>& a, const CUtensorMap& tm, int grid, size_t smem,
                             cudaStream_t s) {
  if (sizeof(TW) == 2) return launch_ws_xr<TA, TW, CELL, NT, U, XR_BF16>(a, tm, grid, smem, s);
  if (sizeof(TA) == 4 && a.xround == XR_TF32) return launch_ws_xr<TA, TW, CELL, NT, U, XR_TF32>(a, tm, grid, smem, s);
  return launch_ws_xr<TA, TW, CELL, NT, U, XR_NONE>(a, tm, grid, smem, s);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D map over the layer input X [L x D] (row stride ldx); box = NT+1 rows x
// (KC + PADV) columns so TMA writes rows at the padded smem pitch.
template <typename TA>
static bool make_x_map(CUtensorMap* tm, const TA* X, int64_t D, int64_t L, int64_t ldx, int box_cols, int box_rows) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return false;
  cuuint64_t gdim[2] = {(cuuint64_t)D, (cuuint64_t)L};
  cuuint64_t gstride[1] = {(cuuint64_t)(ldx * (int64_t)sizeof(TA))};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(tm, sizeof(TA) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                   const_cast<TA*>(X), gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// The warp-specialised kernel needs 16-byte rows it can bulk-copy.
template <typename TA, typename TW>
static bool ws_eligible(const LayerArgs<TA, TW>& a) {
  const int KV = 16 / (int)sizeof(TA);
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return a.G == nullptr && a.D == a.Dp && (a.ldx % KV) == 0 && al(a.X) &&
         (a.xcarry == nullptr || al(a.xcarry)) && getenv("RNNB_NO_WS") == nullptr;
}

template <typename TA, typename TW, int CELL, int NT, int U>
static FfmaPlan plan_nt(int Dp, bool allow_wsmem) {
  FfmaPlan p;
  p.nt = NT;
  constexpr int KV = 16 / (int)sizeof(TA);
  if (allow_wsmem) {
    for (int kc : {256, 128, 64, 32, 16, 8}) {
      int k = kc < Dp ? kc : Dp;
      if (k % KV) continue;
      size_t s = ffma_smem_bytes<TA, TW, CELL, NT, U>(Dp, k, true);
      if (s <= kMaxSmem) { p.wsmem = true; p.kc = k; p.smem = s; return p; }
    }
  }
  p.wsmem = false;
  p.kc = 256 < Dp ? 256 : Dp;
  p.smem = ffma_smem_bytes<TA, TW, CELL, NT, U>(Dp, p.kc, false);
  return p;
}

// Register-resident fp32 kernel (ffma_reg.cuh): U in {4, 7}, aligned 16-byte
// x rows, K = taps*D small enough that the FMA warps + epilogue warp fit the
// register file (U=7: 84 weight registers, <= 8 FMA warps -> K <= 1024; U=4:
// 48 weight registers, <= 16 FMA warps -> K <= 2048).  Chosen for small T_b,
// where the shared-memory kernel re-reads every weight from SMEM for only
// T_b FMAs (RNNB_REG=0/1 overrides).
template <typename TA, typename TW, int CELL, int U>
static bool reg_eligible(const LayerArgs<TA, TW>& a) {
  if constexpr (!(sizeof(TA) == 4 && sizeof(TW) == 4 && (U == 7 || U == 4))) {
    return false;
  } else {
    const int taps = CELL == QRNN ? 2 : 1;
    auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    const int kmax = U == 7 ? 1024 : 2048;
    if (a.G != nullptr || a.xround != XR_NONE || (a.D % 4) != 0 || taps * a.Dp > kmax) return false;
    if ((a.ldx % 4) != 0 || !al(a.X) || (a.xcarry != nullptr && !al(a.xcarry))) return false;
    const char* env = getenv("RNNB_REG");
    if (env) return env[0] == '1';
    // measured crossover: T_b = 1 only since the shared-memory kernel's short
    // passes got cheaper (cfg1 T_b=2: 2.13 reg vs 2.26 M steps/s ws; cfg3:
    // 0.302 vs 0.326 M; at T_b=1 reg still wins: cfg1 2.13 vs 1.53, cfg3 0.302 vs 0.180)
    return a.T_b <= 1;
  }
}

template <int CELL, int U>
static cudaError_t launch_reg(const LayerArgs<float, float>& a, int grid, cudaStream_t s) {
  const int taps = CELL == QRNN ? 2 : 1;
  const int nkv = taps * a.Dp / 4;
  const int threads = (nkv + 31) / 32 * 32 + 32;
  ffma_reg_kernel<CELL, U><<<grid, threads, 0, s>>>(a);
  return cudaGetLastError();
}

// Warp-specialised kernel (ffma_ws.cuh) when its shared-memory plan fits.
// Returns false (nothing launched) when the kernel cannot take this layer.
template <typename TA, typename TW, int CELL, int NT, int U>
static bool try_ws(LayerArgs<TA, TW> a, int grid, cudaStream_t s, FfmaPlan* out, cudaError_t* err) {
  if (!ws_eligible(a)) return false;
  using WC = WsCfg<TA, TW, CELL, NT, U>;
  constexpr int BWMAX = 512 / (int)sizeof(TA);  // 512-byte TMA boxes
  // one k-vector per consumer lane per tap per chunk (see ffma_ws.cuh)
  int kc = WC::KL * WC::KV;
  if (kc > a.Dp) kc = a.Dp;
  int bw = WC::KV;  // power-of-two box width >= the chunk, capped at 512 bytes
  while (bw < kc && bw < BWMAX) bw <<= 1;
  const int nbox = (kc + bw - 1) / bw;
  const size_t sm = ws_smem_bytes<TA, TW, CELL, NT, U>(a.Dp, nbox * bw, bw);
  if (sm > kMaxSmem) return false;
  CUtensorMap tm;
  if (!make_x_map<TA>(&tm, a.X, a.D, a.L, a.ldx, bw + WC::PADV, NT + 1)) return false;
  FfmaPlan p;
  p.nt = NT; p.wsmem = true; p.ws = true; p.kc = kc; p.smem = sm;
  a.KC = kc;
  a.KCB = bw;
  if (out) *out = p;
  if constexpr (NT == 32) *err = launch_ws_xr<TA, TW, CELL, NT, U, XR_NONE>(a, tm, grid, sm, s);  // fp32 only
  else *err = launch_ws<TA, TW, CELL, NT, U>(a, tm, grid, sm, s);
  return true;
}

// ---- weight-streaming ws kernel (weights larger than shared memory) ----
// 32-column passes, kStreamU units per CTA (ceil(2048 / 14) = 147 CTAs for
// BASELINE cfg4's H = 2048: one CTA per SM), K in chunks of KL*KV columns.
constexpr int kStreamU = 14;

template <int CELL>
using WsStreamCfg = WsCfg<float, float, CELL, 32, kStreamU, true>;

template <int CELL>
inline int ws_stream_kc(int Dp) {
  const int kc = WsStreamCfg<CELL>::KL * WsStreamCfg<CELL>::KV;
  return kc < Dp ? kc : Dp;
}

// [CTA][chunk][tap][kv][Rs][KV] images from the gate-interleaved W [rows][TAPS*Dp]
template <int CELL>
__global__ void ws_stream_pack_kernel(const float* __restrict__ W, int rows_src, int Dp, int kc, int nchunk,
                                      int64_t total, float* __restrict__ out) {
  using C = WsStreamCfg<CELL>;
  constexpr int KV = C::KV, Rs = C::Rs, R = C::R, TAPS = C::TAPS;
  const int nkv = kc / KV;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t q = i;
    const int e = (int)(q % KV); q /= KV;
    const int r = (int)(q % Rs); q /= Rs;
    const int kv = (int)(q % nkv); q /= nkv;
    const int tap = (int)(q % TAPS); q /= TAPS;
    const int ch = (int)(q % nchunk); q /= nchunk;
    const int64_t cta = q;
    const int64_t row = cta * R + r;
    const int col = ch * kc + kv * KV + e;
    out[i] = (r < R && row < rows_src && col < Dp) ? W[row * (int64_t)(TAPS * Dp) + tap * Dp + col] : 0.f;
  }
}

template <int CELL>
size_t ws_stream_elems_t(int Dp, int H) {
  const int kc = ws_stream_kc<CELL>(Dp);
  const int nchunk = (Dp + kc - 1) / kc;
  const int grid = (H + kStreamU - 1) / kStreamU;
  return (size_t)grid * nchunk * ws_wimg_elems<float, float, CELL, 32, kStreamU, true>(kc);
}

inline size_t ws_stream_elems(int cell, int Dp, int H) {
  return cell == SRU ? ws_stream_elems_t<SRU>(Dp, H) : ws_stream_elems_t<QRNN>(Dp, H);
}

inline cudaError_t ws_stream_pack(int cell, const float* W, int rows_src, int Dp, int H, float* out, cudaStream_t s) {
  const int64_t total = (int64_t)ws_stream_elems(cell, Dp, H);
  const int bs = 256;
  const int grid = (int)((total + bs - 1) / bs < 148 * 32 ? (total + bs - 1) / bs : 148 * 32);
  if (cell == SRU) {
    const int kc = ws_stream_kc<SRU>(Dp);
    ws_stream_pack_kernel<SRU><<<grid, bs, 0, s>>>(W, rows_src, Dp, kc, (Dp + kc - 1) / kc, total, out);
  } else {
    const int kc = ws_stream_kc<QRNN>(Dp);
    ws_stream_pack_kernel<QRNN><<<grid, bs, 0, s>>>(W, rows_src, Dp, kc, (Dp + kc - 1) / kc, total, out);
  }
  return cudaGetLastError();
}

template <typename TA, typename TW, int CELL>
static bool try_ws_stream(LayerArgs<TA, TW> a, cudaStream_t s, FfmaPlan* out, cudaError_t* err) {
  if constexpr (!(sizeof(TA) == 4 && sizeof(TW) == 4)) {
    return false;
  } else {
    if (!ws_eligible(a) || a.Wst == nullptr) return false;
    constexpr int NT = 32, U = kStreamU;
    using WC = WsStreamCfg<CELL>;
    constexpr int BWMAX = 512 / (int)sizeof(TA);
    const int kc = ws_stream_kc<CELL>(a.Dp);
    int bw = WC::KV;
    while (bw < kc && bw < BWMAX) bw <<= 1;
    const int nbox = (kc + bw - 1) / bw;
    const size_t sm = ws_smem_bytes<TA, TW, CELL, NT, U, true>(a.Dp, nbox * bw, bw);
    if (sm > kMaxSmem) return false;
    CUtensorMap tm;
    if (!make_x_map<TA>(&tm, a.X, a.D, a.L, a.ldx, bw + WC::PADV, NT + 1)) return false;
    a.KC = kc;
    a.KCB = bw;
    auto k = ffma_ws_kernel<TA, TW, CELL, NT, U, XR_NONE, false, true>;
    static bool attr_done = false;
    if (!attr_done) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem);
      if (e != cudaSuccess) {
        *err = e;
        return true;
      }
      attr_done = true;
    }
    const int grid = (a.H + U - 1) / U;
    k<<<grid, WC::THREADS, sm, s>>>(a, tm);
    *err = cudaGetLastError();
    if (out) {
      FfmaPlan p;
      p.nt = NT; p.wsmem = false; p.ws = true; p.wstream = true; p.kc = kc; p.smem = sm; p.grid = grid;
      *out = p;
    }
    return true;
  }
}

template <typename TA, typename TW, int CELL, int NT, int U>
static cudaError_t run_nt(LayerArgs<TA, TW> a, int grid, bool allow_wsmem, cudaStream_t s, FfmaPlan* out) {
  if constexpr (sizeof(TA) == 4 && sizeof(TW) == 4 && (U == 7 || U == 4)) {
    if (reg_eligible<TA, TW, CELL, U>(a)) {
      // streaming input needs the ws kernel; refuse rather than change kernels
      // (the caller falls back, so results stay identical to rnnb_forward)
      if (a.x_ready != nullptr) return cudaErrorNotSupported;
      FfmaPlan p;
      p.nt = 1; p.wsmem = false; p.ws = false; p.reg = true; p.kc = 0; p.smem = 0;
      if (out) *out = p;
      return launch_reg<CELL, U>(a, grid, s);
    }
  }
  if (allow_wsmem) {
    cudaError_t e;
    if (try_ws<TA, TW, CELL, NT, U>(a, grid, s, out, &e)) return e;
  }
  if (a.x_ready != nullptr) return cudaErrorNotSupported;  // streaming needs the ws kernel; nothing launched
  FfmaPlan p = plan_nt<TA, TW, CELL, NT, U>(a.Dp, allow_wsmem);
  a.KC = p.kc;
  if (out) *out = p;
  if (p.wsmem) return launch_one<TA, TW, CELL, NT, U, true>(a, grid, p.smem, s);
  return launch_one<TA, TW, CELL, NT, U, false>(a, grid, p.smem, s);
}

template <typename TA, typename TW, int CELL, int U>
static cudaError_t run_u(const LayerArgs<TA, TW>& a, int grid, bool allow_wsmem, cudaStream_t s, FfmaPlan* out) {
  switch (pick_nt(a.T_b)) {
    case 1: return run_nt<TA, TW, CELL, 1, U>(a, grid, allow_wsmem, s, out);
    case 2: return run_nt<TA, TW, CELL, 2, U>(a, grid, allow_wsmem, s, out);
    case 4: return run_nt<TA, TW, CELL, 4, U>(a, grid, allow_wsmem, s, out);
    case 8: return run_nt<TA, TW, CELL, 8, U>(a, grid, allow_wsmem, s, out);
    default:
      // fp32: a 32-column pass (double-buffered partials, 3 x stages) halves
      // the per-pass reduction / hand-off cost: cfg2 2.89 -> 3.01 M steps/s.
      // Falls back to NT = 16 when its shared-memory plan does not fit
      // (RNNB_NT32=0 forces NT = 16).
      if constexpr (sizeof(TA) == 4 && sizeof(TW) == 4) {
        if (a.Wst != nullptr && a.T_b >= 32 && a.xround == XR_NONE && a.x_ready == nullptr) {
          cudaError_t e;
          if (try_ws_stream<TA, TW, CELL>(a, s, out, &e)) return e;
        }
        const char* env = getenv("RNNB_NT32");
        if (allow_wsmem && a.T_b >= 32 && a.xround == XR_NONE && !(env && env[0] == '0')) {
          cudaError_t e;
          if (try_ws<TA, TW, CELL, 32, U>(a, grid, s, out, &e)) return e;
        }
      }
      return run_nt<TA, TW, CELL, 16, U>(a, grid, allow_wsmem, s, out);
  }
}

// Units per CTA: the supported set; the weight layout is padded to a
// multiple of U units with zero rows.
inline bool valid_units(int U) { return U == 2 || U == 4 || U == 7; }

template <typename TA, typename TW>
cudaError_t ffma_layer_run(int cell, int U, const LayerArgs<TA, TW>& a, bool allow_wsmem,
                           cudaStream_t s, FfmaPlan* out) {
  const int grid = (a.H + U - 1) / U;
  if (cell == SRU) {
    if (U == 2) return run_u<TA, TW, SRU, 2>(a, grid, allow_wsmem, s, out);
    if (U == 4) return run_u<TA, TW, SRU, 4>(a, grid, allow_wsmem, s, out);
    return run_u<TA, TW, SRU, 7>(a, grid, allow_wsmem, s, out);
  }
  if (U == 2) return run_u<TA, TW, QRNN, 2>(a, grid, allow_wsmem, s, out);
  if (U == 4) return run_u<TA, TW, QRNN, 4>(a, grid, allow_wsmem, s, out);
  return run_u<TA, TW, QRNN, 7>(a, grid, allow_wsmem, s, out);
}

// explicit instantiations live in ffma_<mode>.cu
extern template cudaError_t ffma_layer_run<float, float>(int, int, const LayerArgs<float, float>&, bool, cudaStream_t, FfmaPlan*);
extern template cudaError_t ffma_layer_run<float, __nv_bfloat16>(int, int, const LayerArgs<float, __nv_bfloat16>&, bool, cudaStream_t, FfmaPlan*);
extern template cudaError_t ffma_layer_run<double, double>(int, int, const LayerArgs<double, double>&, bool, cudaStream_t, FfmaPlan*);

}  // namespace rnnb
