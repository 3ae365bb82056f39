// Explicit instantiation of the FFMA layer kernels for (float accumulate, float weights).
#include "ffma_dispatch.cuh"
namespace rnnb {
template cudaError_t ffma_layer_run<float, float>(int, int, const LayerArgs<float, float>&, bool, cudaStream_t, FfmaPlan*);
}
