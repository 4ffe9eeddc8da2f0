// "fast" mode: FMA contraction allowed.  fp32 (tolerance-checked against the
// oracle) and a fast fp64 variant.
#define RSB_MODE_NS fast
#define RSB_MODE_ID 1
#include "rod_launch.cuh"

namespace rsb {
namespace fast {
template cudaError_t launch_step<float>(int, int, int, const StepArgs<float>&, int, int, size_t, int, cudaStream_t);
template cudaError_t launch_step<double>(int, int, int, const StepArgs<double>&, int, int, size_t, int, cudaStream_t);
template cudaError_t occupancy<float>(int, int, int, int, size_t, int, int*);
template cudaError_t occupancy<double>(int, int, int, int, size_t, int, int*);

// Issue-rate microbenchmark for the compute cross-check of the roofline:
// `kind` 0 = DFMA, 1 = DADD, 2 = DMUL, 3 = FFMA; 8 independent chains per
// thread so the pipe, not latency, binds.  Returns operations executed.
template <typename T, int KIND>
__global__ void pipe_peak_kernel(T* out, int iters, T a, T b) {
    T x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = T(threadIdx.x + c) * T(1e-3);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if constexpr (KIND == 0 || KIND == 3) x[c] = fma(x[c], a, b);
            else if constexpr (KIND == 1) x[c] = x[c] + b;
            else x[c] = x[c] * a;
        }
    }
    T s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c];
    if (s == T(12345.678)) out[0] = s;
}

cudaError_t pipe_peak(int kind, int blocks, int threads, int iters, float* ms, double* ops) {
    void* buf = nullptr;
    cudaError_t e = cudaMalloc(&buf, 64);
    if (e != cudaSuccess) return e;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&]() {
        switch (kind) {
            case 0: pipe_peak_kernel<double, 0><<<blocks, threads>>>((double*)buf, iters, 0.999999, 1e-9); break;
            case 1: pipe_peak_kernel<double, 1><<<blocks, threads>>>((double*)buf, iters, 0.999999, 1e-9); break;
            case 2: pipe_peak_kernel<double, 2><<<blocks, threads>>>((double*)buf, iters, 0.999999, 1e-9); break;
            default: pipe_peak_kernel<float, 3><<<blocks, threads>>>((float*)buf, iters, 0.999999f, 1e-9f); break;
        }
    };
    run();
    cudaEventRecord(e0);
    run();
    cudaEventRecord(e1);
    e = cudaEventSynchronize(e1);
    cudaEventElapsedTime(ms, e0, e1);
    *ops = double(blocks) * threads * iters * 8.0;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    if (e == cudaSuccess) e = cudaGetLastError();
    return e;
}
}  // namespace fast
}  // namespace rsb
