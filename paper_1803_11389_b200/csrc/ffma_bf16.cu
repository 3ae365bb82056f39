// Explicit instantiation of the FFMA layer kernels for (float accumulate, __nv_bfloat16 weights).
#include "ffma_dispatch.cuh"
namespace rnnb {
template cudaError_t ffma_layer_run<float, __nv_bfloat16>(int, int, const LayerArgs<float, __nv_bfloat16>&, bool, cudaStream_t, FfmaPlan*);
}
