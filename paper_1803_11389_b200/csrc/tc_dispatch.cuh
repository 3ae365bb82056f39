// Host interface of the tcgen05 layer path (tc_launch.cu).
#pragma once
#include "ffma_dispatch.cuh"  // encode_tiled()
#include "tc_layer.cuh"

namespace rnnb {

// MMA-operand copy of a layer input with a leading x_{-1} row.
// `fill` (16-byte multiple): the following layer launch's look-back state, set
// to the all-ones sentinel by the same kernel (no extra launch)
cudaError_t tc_to_operand(int mode, const float* X, int64_t ldx, const float* xcarry, void* out, int64_t ldo,
                          int64_t L, int D, cudaStream_t s, void* fill = nullptr, size_t fill_bytes = 0);
// rows of a longer operand (3xTF32 lo plane prow rows after the hi plane)
cudaError_t tc_to_operand_rows(int mode, const float* X, int64_t ldx, const float* xcarry, void* out, int64_t ldo,
                               int64_t L, int D, int64_t prow, cudaStream_t s, void* fill = nullptr,
                               size_t fill_bytes = 0);

// copy segments of a streamed input: segment j = X rows [end[j-1], end[j])
constexpr int kMaxSegs = 48;
struct TcSegTab {
  int n;
  int end[kMaxSegs];
};
// streaming conversion: one persistent launch (`workers` CTAs + a publisher)
// following the copy engine (seg_flag[j] == epoch: segment j landed), per-group flags tagged
// with the call's epoch, *ready = rows converted in order
bool tc_to_operand_stream_ok(const float* X, int64_t ldx, const float* xcarry, const void* out, int64_t ldo, int D);
cudaError_t tc_to_operand_stream(int mode, const float* X, int64_t ldx, const float* xcarry, void* out, int64_t ldo,
                                 int64_t L, int D, const TcSegTab& segs, const int* seg_flag, int* ready, int* fail,
                                 int* flags, int* next_group, int epoch, int group, int workers, cudaStream_t s);

// One layer on the tensor-core path.  Wtc: [3*Hpad][Kp] gate-major operand
// weights; Xop: [L+1][ldop_in] operand input (row 0 = x_{-1}).
cudaError_t tc_layer_run(int cell, int mode, TcArgs a, const void* Wtc, int Kp, const void* Xop, int64_t ldop_in,
                         int num_sms, cudaStream_t s, int* grid_out);

// load one layer-kernel variant without launching it (see launch_tc)
cudaError_t tc_layer_preload(int cell, int mode, int T_b);

int tc_pick_n(int T_b);
int tc_max_n(int mode);

}  // namespace rnnb
