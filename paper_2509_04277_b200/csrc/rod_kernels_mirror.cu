// fp64 "mirror" mode: compiled with --fmad=false and IEEE div/sqrt so every
// operation rounds exactly as the reference's compiled core (no FMA, same
// expression trees) -- the bitwise parity mode.
#define RSB_MODE_NS mirror
#define RSB_MODE_ID 0
#include "rod_launch.cuh"

namespace rsb {
namespace mirror {
template cudaError_t launch_step<double>(int, int, int, const StepArgs<double>&, int, int, size_t, int, cudaStream_t);
template cudaError_t occupancy<double>(int, int, int, int, size_t, int, int*);
}  // namespace mirror
}  // namespace rsb

// Self-test hook: IEEE a/b against the reciprocal-based div_rn used by the
// step kernel, compiled under the same flags (tests/test_gpu_selftest.py).
namespace rsb {
namespace mirror {
__global__ void div_selftest_kernel(const double* a, const double* b, int64_t n, double* q_ieee,
                                    double* q_fast) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const double rb = 1.0 / b[i];
        q_ieee[i] = a[i] / b[i];
        q_fast[i] = div_rn(a[i], b[i], rb);
    }
}
cudaError_t div_selftest(const double* a, const double* b, int64_t n, double* q_ieee, double* q_fast) {
    div_selftest_kernel<<<592, 256>>>(a, b, n, q_ieee, q_fast);
    return cudaDeviceSynchronize();
}
}  // namespace mirror
}  // namespace rsb
