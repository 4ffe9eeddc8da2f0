// One instantiation set of the step kernel, compiled six times by the
// Makefile (precision mode x scene features) so the translation units build
// in parallel:
//   RSB_MODE_NS  mirror | f32 | f64fast  (+ _feat), namespace of the launchers
//   RSB_MODE_ID  0 (mirror: --fmad=false, IEEE div/sqrt: bitwise with the
//                reference) or 1 (fast: contraction allowed)
//   RSB_REAL     double | float
//   RSB_FEAT     0 plain step, 1 with the mesh-contact and self-collision phases
// MODE is part of the kernel's template arguments: identical arguments in
// two TUs built with different flags would otherwise be one symbol and the
// CUDA runtime would launch whichever module registered it.
#include "rod_launch.cuh"

namespace rsb {
namespace RSB_MODE_NS {
template cudaError_t launch_step<RSB_REAL>(int, int, int, const StepArgs<RSB_REAL>&, int, int, size_t, int,
                                           cudaStream_t);
template cudaError_t occupancy<RSB_REAL>(int, int, int, int, size_t, int, int*);
#if !RSB_FEAT
template cudaError_t batch_step<RSB_REAL>(int, int, const StepArgs<RSB_REAL>*, int, cudaStream_t, int*);
template cudaError_t warp_step<RSB_REAL>(int, int, const StepArgs<RSB_REAL>*, int, cudaStream_t);
template cudaError_t halo_step<RSB_REAL>(int, int, int, int, int, int, const StepArgs<RSB_REAL>*, int, int,
                                         cudaStream_t, int*);
#endif
}  // namespace RSB_MODE_NS
}  // namespace rsb
