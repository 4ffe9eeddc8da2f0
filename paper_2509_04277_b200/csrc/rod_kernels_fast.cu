// "fast" mode: FMA contraction allowed.  fp32 (tolerance-checked against the
// oracle) and a fast fp64 variant.
#define RSB_MODE_NS fast
#define RSB_MODE_ID 1
#include "rod_launch.cuh"

namespace rsb {
namespace fast {
template cudaError_t launch_step<float>(int, int, bool, const StepArgs<float>&, int, int, size_t, int, cudaStream_t);
template cudaError_t launch_step<double>(int, int, bool, const StepArgs<double>&, int, int, size_t, int, cudaStream_t);
template cudaError_t occupancy<float>(int, int, bool, int, size_t, int, int*);
template cudaError_t occupancy<double>(int, int, bool, int, size_t, int, int*);
}  // namespace fast
}  // namespace rsb
