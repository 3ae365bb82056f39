// Explicit instantiation of the FFMA layer kernels for (double accumulate, double weights).
#include "ffma_dispatch.cuh"
namespace rnnb {
template cudaError_t ffma_layer_run<double, double>(int, int, const LayerArgs<double, double>&, bool, cudaStream_t, FfmaPlan*);
}
