// Dense layers Y[L x d_out] = X[L x d_in] W^T (+ b) for the BASELINE cfg3
// acoustic model: the 120 -> 1024 input projection and the 1024 -> 2000
// logits.  The reference has no such layer type; the
// product it restates is kernels.gemm(W, X^T) (rnnblock kernels.py:203-225).
//
//   f32 / f64 (and f32x3): a register-blocked FFMA GEMM, 128 x 128 output
//     tile per CTA, 8 x 8 per thread, K staged through shared memory in
//     16-deep slices with the next slice's loads in flight; every output is
//     one ascending-k fp32 (fp64) chain, so results are deterministic.
//   bf16 / tf32: the tcgen05 layer kernel with the LINEAR cell (TMA weight
//     and x tiles, TMEM accumulators, epilogue = bias + store), the same MMA
//     operand rounding as the recurrent layers.
#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <vector>

#include "../../include/rnnb.h"
#include "abi_guard.h"
#include "tc_dispatch.cuh"

using namespace rnnb;

struct rnnb_linear {
  int64_t din = 0, dout = 0;
  int mode = RNNB_F32, device = 0, num_sms = 148;
  void* W = nullptr;      // FFMA path: [dout][din] (f32 or f64)
  void* bias = nullptr;   // [dout] of the element type (nullptr: no bias)
  void* Wtc = nullptr;    // tensor-core path: [3*Hpad][tcKp] bf16 / tf32-rounded f32
  float* bias_f = nullptr;
  int Hpad = 0, tcKp = 0;
  void* op = nullptr;     // MMA-operand copy of X, [L+1][ldop]
  size_t op_bytes = 0;
  bool loaded = false, last_tc = false;
  int64_t launches = 0;
};

namespace {

constexpr int kBK = 16, kThreads = 256;

// Y[m][n] = sum_k X[m][k] W[n][k] + b[n].  CTA: 16*TM rows (time steps) x
// 16*TM outputs; thread (tx, ty) in 16 x 16 owns rows ty*TM.. and outputs
// tx*TM.. (TM = 8 for fp32: a 128 x 128 tile; 4 for fp64, whose doubled
// staging would not fit the 48 KB of static shared memory otherwise)
template <typename T, int TM>
__global__ void __launch_bounds__(kThreads) linear_ffma_kernel(const T* __restrict__ X, int64_t ldx,
                                                               const T* __restrict__ W, const T* __restrict__ b,
                                                               T* __restrict__ Y, int64_t ldy, int64_t M, int N,
                                                               int K) {
  constexpr int BM = 16 * TM, TPR = 16 / TM;  // tile side, loader threads per row
  __shared__ __align__(16) T Xs[2][kBK][BM + 4];
  __shared__ __align__(16) T Ws[2][kBK][BM + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int n0 = blockIdx.x * BM;
  // loader mapping: each thread brings TM consecutive k of one row of X and
  // of W per 16-deep slice
  const int lr = tid / TPR, lk = (tid % TPR) * TM;
  T xr[TM], wr[TM];
  auto load = [&](int k0) {
    const int64_t m = m0 + lr;
    const int n = n0 + lr;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int k = k0 + lk + i;
      xr[i] = (m < M && k < K) ? X[m * ldx + k] : T(0);
      wr[i] = (n < N && k < K) ? W[(int64_t)n * K + k] : T(0);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      Xs[buf][lk + i][lr] = xr[i];
      Ws[buf][lk + i][lr] = wr[i];
    }
  };
  T acc[TM][TM];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TM; ++j) acc[i][j] = T(0);
  const int nk = (K + kBK - 1) / kBK;
  load(0);
  stash(0);
  __syncthreads();
  for (int s = 0; s < nk; ++s) {
    const int buf = s & 1;
    if (s + 1 < nk) load((s + 1) * kBK);  // next slice's global loads in flight during the FMAs
#pragma unroll
    for (int k = 0; k < kBK; ++k) {
      T a[TM], w[TM];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = Xs[buf][k][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TM; ++j) w[j] = Ws[buf][k][tx * TM + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TM; ++j) acc[i][j] = fma(a[i], w[j], acc[i][j]);
    }
    if (s + 1 < nk) stash(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t m = m0 + ty * TM + i;
    if (m >= M) break;
#pragma unroll
    for (int j = 0; j < TM; ++j) {
      const int n = n0 + tx * TM + j;
      if (n < N) Y[m * ldy + n] = acc[i][j] + (b ? b[n] : T(0));
    }
  }
}

rnnb_status fail(rnnb_status s, const std::string& m) { return set_error(s, m); }

#define LCUDA_TRY(expr)                                                                        \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e != cudaSuccess) return fail(RNNB_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

bool tensor_mode(int mode) { return mode == RNNB_BF16 || mode == RNNB_TF32; }

float tf32_rna(float v) {
  uint32_t u;
  std::memcpy(&u, &v, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
  std::memcpy(&v, &u, 4);
  return v;
}
uint16_t bf16_rne(float v) {
  uint32_t u;
  std::memcpy(&u, &v, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return (uint16_t)((u >> 16) | ((u & 0xffff) ? 0x40 : 0));
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

void free_all(rnnb_linear* h) {
  for (void* p : {h->W, h->bias, h->Wtc, (void*)h->bias_f, h->op})
    if (p) cudaFree(p);
  h->W = h->bias = h->Wtc = h->op = nullptr;
  h->bias_f = nullptr;
  h->op_bytes = 0;
}

rnnb_status linear_set(rnnb_linear* h, const void* W, const void* bias, int src_dtype) {
  if (!h) return fail(RNNB_EINVAL, "null linear handle");
  if (!W) return fail(RNNB_EINVAL, "null weight matrix");
  if (src_dtype != RNNB_DT_F32 && src_dtype != RNNB_DT_F64) return fail(RNNB_EINVAL, "src dtype must be f32 or f64");
  DeviceGuard dg(h->device);
  LCUDA_TRY(dg.err);
  auto get = [&](const void* p, int64_t i) -> double {
    return src_dtype == RNNB_DT_F64 ? static_cast<const double*>(p)[i] : (double)static_cast<const float*>(p)[i];
  };
  const int64_t n = h->din * h->dout;
  free_all(h);
  if (tensor_mode(h->mode)) {
    const int KT = h->mode == RNNB_BF16 ? 64 : 32;
    const int64_t Dtc = (h->din + KT - 1) / KT * KT;
    h->Hpad = (int)(((h->dout + 2) / 3 + 127) / 128 * 128);
    h->tcKp = (int)Dtc;
    const size_t rows = (size_t)3 * h->Hpad, es = h->mode == RNNB_BF16 ? 2 : 4;
    std::vector<unsigned char> tc(rows * Dtc * es, 0);
    for (int64_t r = 0; r < h->dout; ++r)
      for (int64_t k = 0; k < h->din; ++k) {
        const float v = (float)get(W, r * h->din + k);
        const size_t dst = (size_t)r * Dtc + k;
        if (h->mode == RNNB_BF16) reinterpret_cast<uint16_t*>(tc.data())[dst] = bf16_rne(v);
        else reinterpret_cast<float*>(tc.data())[dst] = tf32_rna(v);
      }
    LCUDA_TRY(cudaMalloc(&h->Wtc, tc.size()));
    LCUDA_TRY(cudaMemcpy(h->Wtc, tc.data(), tc.size(), cudaMemcpyHostToDevice));
    if (bias) {
      std::vector<float> bf((size_t)h->dout);
      for (int64_t r = 0; r < h->dout; ++r) bf[(size_t)r] = (float)get(bias, r);
      LCUDA_TRY(cudaMalloc(&h->bias_f, bf.size() * 4));
      LCUDA_TRY(cudaMemcpy(h->bias_f, bf.data(), bf.size() * 4, cudaMemcpyHostToDevice));
    }
  } else {
    if (h->mode == RNNB_F32) {
      // + tf32 hi / lo planes for the fp32-accurate 3xTF32 tensor-core path
      // (layers whose items fill the GPU; linear_forward)
      const int KT = 32;
      const int64_t Dtc = (h->din + KT - 1) / KT * KT;
      h->Hpad = (int)(((h->dout + 2) / 3 + 127) / 128 * 128);
      h->tcKp = (int)Dtc;
      const size_t rows = (size_t)3 * h->Hpad;
      std::vector<float> tc(2 * rows * Dtc, 0.f);
      for (int64_t r = 0; r < h->dout; ++r)
        for (int64_t k = 0; k < h->din; ++k) {
          const float v = (float)get(W, r * h->din + k);
          const float hi = tf32_rna(v);
          tc[(size_t)r * Dtc + k] = hi;
          tc[(rows + (size_t)r) * Dtc + k] = tf32_rna(v - hi);
        }
      LCUDA_TRY(cudaMalloc(&h->Wtc, tc.size() * 4));
      LCUDA_TRY(cudaMemcpy(h->Wtc, tc.data(), tc.size() * 4, cudaMemcpyHostToDevice));
      if (bias) {
        std::vector<float> bf((size_t)h->dout);
        for (int64_t r = 0; r < h->dout; ++r) bf[(size_t)r] = (float)get(bias, r);
        LCUDA_TRY(cudaMalloc(&h->bias_f, bf.size() * 4));
        LCUDA_TRY(cudaMemcpy(h->bias_f, bf.data(), bf.size() * 4, cudaMemcpyHostToDevice));
      }
    }
    const size_t es = h->mode == RNNB_F64 ? 8 : 4;
    std::vector<unsigned char> w((size_t)n * es);
    for (int64_t i = 0; i < n; ++i) {
      if (es == 8) reinterpret_cast<double*>(w.data())[i] = get(W, i);
      else reinterpret_cast<float*>(w.data())[i] = (float)get(W, i);
    }
    LCUDA_TRY(cudaMalloc(&h->W, w.size()));
    LCUDA_TRY(cudaMemcpy(h->W, w.data(), w.size(), cudaMemcpyHostToDevice));
    if (bias) {
      std::vector<unsigned char> bb((size_t)h->dout * es);
      for (int64_t r = 0; r < h->dout; ++r) {
        if (es == 8) reinterpret_cast<double*>(bb.data())[r] = get(bias, r);
        else reinterpret_cast<float*>(bb.data())[r] = (float)get(bias, r);
      }
      LCUDA_TRY(cudaMalloc(&h->bias, bb.size()));
      LCUDA_TRY(cudaMemcpy(h->bias, bb.data(), bb.size(), cudaMemcpyHostToDevice));
    }
  }
  h->loaded = true;
  return RNNB_OK;
}

rnnb_status linear_forward(rnnb_linear* h, const void* X, int64_t ldx, int64_t L, void* Y, int64_t ldy,
                           void* stream) {
  if (!h) return fail(RNNB_EINVAL, "null linear handle");
  if (!h->loaded) return fail(RNNB_EINVAL, "linear layer has no weights");
  if (!X || !Y) return fail(RNNB_EINVAL, "null X or Y");
  if (L < 1) return fail(RNNB_EINVAL, "seq_len must be >= 1");
  if (ldx < h->din) return fail(RNNB_EINVAL, "ldx smaller than d_in");
  if (ldy < h->dout) return fail(RNNB_EINVAL, "ldy smaller than d_out");
  DeviceGuard dg(h->device);
  LCUDA_TRY(dg.err);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  h->launches = 0;
  // fp32: the 3xTF32 tcgen05 path when its (128-column plane triple, 32-row
  // block) items fill the GPU (cfg3's projection and logits), else the FFMA GEMM
  bool x3 = false;
  if (h->mode == RNNB_F32 && h->Wtc != nullptr) {
    const char* e = getenv("RNNB_F32_TC");
    const int64_t items = (int64_t)(h->Hpad / 128) * ((L + 31) / 32);
    x3 = !(e && e[0] == '0') && getenv("RNNB_NO_TC") == nullptr && items >= h->num_sms;
  }
  if (tensor_mode(h->mode) || x3) {
    const int mode = x3 ? TC_3XTF32 : h->mode == RNNB_BF16 ? TC_BF16 : TC_TF32;
    const int es = mode == TC_BF16 ? 2 : 4;
    const int64_t ldop = (h->din + 7) / 8 * 8;
    const size_t opb = (size_t)(x3 ? 2 : 1) * (L + 1) * ldop * es;
    if (h->op_bytes < opb) {
      if (h->op) cudaFree(h->op);
      h->op = nullptr;
      h->op_bytes = 0;
      LCUDA_TRY(cudaMalloc(&h->op, opb));
      h->op_bytes = opb;
    }
    LCUDA_TRY(tc_to_operand(mode, static_cast<const float*>(X), ldx, nullptr, h->op, ldop, L, (int)h->din, s));
    TcArgs a{};
    a.Hout = static_cast<float*>(Y);
    a.ldh = ldy;
    a.bias = h->bias_f;
    a.L = L;
    a.T_b = x3 ? 32 : 64;  // N = 64: double-buffered TMEM accumulators, epilogue overlaps the next item's MMAs
                           // (3xTF32 keeps its chunk partials in registers: N = 32)
    a.H = (int)h->dout;
    a.Hpad = h->Hpad;
    a.D = (int)h->din;
    const int KT = mode == TC_BF16 ? 64 : 32;
    a.nKtap = (int)((h->din + KT - 1) / KT);
    a.nK = h->tcKp / KT;
    a.nU = h->Hpad / 128;
    a.nB = (int)((L + a.T_b - 1) / a.T_b);
    a.egroups = 2;  // dense layers: short K, the store epilogue bounds an item
    a.ck0 = x3_pick_ck0(a.nK);
    int grid = 0;
    cudaError_t e = tc_layer_run(LINEAR, mode, a, h->Wtc, h->tcKp, h->op, ldop, h->num_sms, s, &grid);
    if (e != cudaSuccess) return fail(RNNB_ECUDA, std::string("tc linear launch: ") + cudaGetErrorString(e));
    h->last_tc = true;
    h->launches = 2;
    return RNNB_OK;
  }
  if (h->mode == RNNB_F64) {
    const dim3 grid((unsigned)((h->dout + 63) / 64), (unsigned)((L + 63) / 64));
    linear_ffma_kernel<double, 4><<<grid, kThreads, 0, s>>>(static_cast<const double*>(X), ldx,
                                                            static_cast<const double*>(h->W),
                                                            static_cast<const double*>(h->bias),
                                                            static_cast<double*>(Y), ldy, L, (int)h->dout,
                                                            (int)h->din);
  } else {
    const dim3 grid((unsigned)((h->dout + 127) / 128), (unsigned)((L + 127) / 128));
    linear_ffma_kernel<float, 8><<<grid, kThreads, 0, s>>>(static_cast<const float*>(X), ldx,
                                                           static_cast<const float*>(h->W),
                                                           static_cast<const float*>(h->bias), static_cast<float*>(Y),
                                                           ldy, L, (int)h->dout, (int)h->din);
  }
  LCUDA_TRY(cudaGetLastError());
  h->last_tc = false;
  h->launches = 1;
  return RNNB_OK;
}

}  // namespace

extern "C" {

rnnb_status rnnb_linear_create(rnnb_linear_t* out, int64_t d_in, int64_t d_out, int mode, int device) {
  return abi_guard("rnnb_linear_create", [&]() -> rnnb_status {
    if (!out) return fail(RNNB_EINVAL, "out is null");
    *out = nullptr;
    if (d_in < 1 || d_out < 1) return fail(RNNB_EINVAL, "d_in and d_out must be >= 1");
    if (d_in > (1 << 24) || d_out > (1 << 24)) return fail(RNNB_EUNSUPPORTED, "dimension too large");
    if (mode < RNNB_F32 || mode > RNNB_F32X3) return fail(RNNB_EINVAL, "unknown compute mode");
    int ndev = 0;
    LCUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(RNNB_EINVAL, "bad device ordinal");
    auto* h = new rnnb_linear();
    h->din = d_in;
    h->dout = d_out;
    // f32x3 dense layers run the exact FFMA kernel (fp32 products)
    h->mode = mode == RNNB_F32X3 ? RNNB_F32 : mode;
    h->device = device;
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
    *out = h;
    return RNNB_OK;
  });
}

rnnb_status rnnb_linear_destroy(rnnb_linear_t h) {
  if (!h) return RNNB_OK;
  DeviceGuard dg(h->device);
  free_all(h);
  delete h;
  return RNNB_OK;
}

rnnb_status rnnb_linear_set_weights(rnnb_linear_t h, const void* W, const void* bias, int src_dtype) {
  return abi_guard("rnnb_linear_set_weights", [&]() { return linear_set(h, W, bias, src_dtype); });
}

rnnb_status rnnb_linear_forward(rnnb_linear_t h, const void* X, int64_t ldx, int64_t L, void* Y, int64_t ldy,
                                void* stream) {
  return abi_guard("rnnb_linear_forward", [&]() { return linear_forward(h, X, ldx, L, Y, ldy, stream); });
}

rnnb_status rnnb_linear_query(rnnb_linear_t h, int what, int64_t* value) {
  if (!h || !value) return fail(RNNB_EINVAL, "null argument");
  switch (what) {
    case 0: *value = h->last_tc ? 1 : 0; return RNNB_OK;
    case 1: *value = h->launches; return RNNB_OK;
    default: return fail(RNNB_EINVAL, "unknown query");
  }
}

}  // extern "C"
