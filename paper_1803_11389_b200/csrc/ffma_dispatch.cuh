// Host-side launch of the FFMA layer kernel: picks the pass width NT from
// T_b, the shared-memory plan (weights resident or streamed from L2) and
// instantiates the kernel for one (accumulate, weight) type pair.
#pragma once
#include "ffma_layer.cuh"

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
  int kc = 0;
  size_t smem = 0;
};

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

template <typename TA, typename TW, int CELL, int NT, int U>
static cudaError_t run_nt(LayerArgs<TA, TW> a, int grid, bool allow_wsmem, cudaStream_t s, FfmaPlan* out) {
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
    default: return run_nt<TA, TW, CELL, 16, U>(a, grid, allow_wsmem, s, out);
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
