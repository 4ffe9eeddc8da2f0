// rod_micro.cu -- latency microbenchmarks behind the single-rod latency
// roofline t_floor = n_sync * (t_sync + t_chain) + t_launch / K:
// dependent fp64 chains (the per-phase critical path is built from these),
// shared-memory load latency, and the three barrier scopes the step kernel
// uses (bar.sync in a CTA, barrier.cluster across a cluster, DSMEM reads).
// Compiled with the mirror flags (--fmad=false, IEEE div/sqrt) so the chains
// are the instruction sequences the fp64 mirror kernel issues.
#include <cuda_runtime.h>
#include <stdint.h>

#include "rod_math.cuh"

namespace rsb {
namespace micro {

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// out[0] = cycles per op, out[1] = ns per op (thread 0, dependent chain)
template <int KIND>
__global__ void chain_kernel(double* out, int iters, double a, double b) {
    if (threadIdx.x != 0) return;
    double x = a, rb = 1.0 / b;
    const long long c0 = clock64();
    const uint64_t t0 = gtimer();
    for (int i = 0; i < iters; ++i) {
        if constexpr (KIND == 0) x = x + b;
        else if constexpr (KIND == 1) x = x * b;
        else if constexpr (KIND == 2) x = fma(x, b, a);
        else if constexpr (KIND == 3) x = x / b;
        else if constexpr (KIND == 4) x = sqrt(x) + a;
        else if constexpr (KIND == 5) x = div_rn(x, b, rb);
        else if constexpr (KIND == 6) x = 1.0 / x;
    }
    const long long c1 = clock64();
    const uint64_t t1 = gtimer();
    out[0] = double(c1 - c0) / iters;
    out[1] = double(t1 - t0) / iters;
    if (x == 12345.678) out[2] = x;
}

// shared-memory pointer chase: cycles per dependent LDS
__global__ void lds_kernel(double* out, int iters) {
    __shared__ int nxt[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) nxt[i] = (i + 97) & 1023;
    __syncthreads();
    if (threadIdx.x != 0) return;
    int p = 0;
    const long long c0 = clock64();
    for (int i = 0; i < iters; ++i) p = nxt[p];
    const long long c1 = clock64();
    out[0] = double(c1 - c0) / iters;
    out[1] = 0;
    if (p == -1) out[2] = p;
}

// CTA barrier: ns per bar.sync with blockDim threads, each with a little
// shared-memory traffic per phase like the step kernel's
__global__ void bar_kernel(double* out, int iters) {
    __shared__ double buf[1024];
    const int t = threadIdx.x;
    buf[t] = t;
    __syncthreads();
    const uint64_t t0 = gtimer();
    const long long c0 = clock64();
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        acc += buf[(t + i) & (blockDim.x - 1)];
        __syncthreads();
        buf[t] = acc;
        __syncthreads();
    }
    const long long c1 = clock64();
    const uint64_t t1 = gtimer();
    if (t == 0) {
        out[0] = double(c1 - c0) / (2.0 * iters);
        out[1] = double(t1 - t0) / (2.0 * iters);
    }
    if (acc == -1.0) out[2] = acc;
}

// cluster barrier (arrive.release + wait.acquire) with one DSMEM read of the
// neighbour's slot per phase: ns per phase
__global__ void cluster_bar_kernel(double* out, int iters) {
    __shared__ double buf[32];
    unsigned rank, nrank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(nrank));
    if (threadIdx.x < 32) buf[threadIdx.x] = rank;
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(buf)), remote;
    const unsigned nb = (rank + 1) % nrank;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(nb));
    double acc = 0;
    const uint64_t t0 = gtimer();
    const long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        double v;
        asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote) : "memory");
        acc += v;
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    const long long c1 = clock64();
    const uint64_t t1 = gtimer();
    if (rank == 0 && threadIdx.x == 0) {
        out[0] = double(c1 - c0) / iters;
        out[1] = double(t1 - t0) / iters;
    }
    if (acc == -1.0) out[2] = acc;
}

// Neighbour-only synchronisation across a cluster (a chain of CTAs, like a
// rod split over the cluster): per phase bar.sync, thread 0 arrives on the
// left and right neighbours' mbarriers (remote, release.cluster) and waits on
// its own two (acquire.cluster), bar.sync -- with one DSMEM read of the
// neighbour's slot per phase, as in the cluster barrier benchmark.
__global__ void nb_sync_kernel(double* out, int iters) {
    __shared__ __align__(8) uint64_t nbar[2][2];   // [from left / from right][parity]
    __shared__ double buf[32];
    unsigned rank, nrank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(nrank));
    const bool has_l = rank > 0, has_r = rank + 1 < nrank;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                             static_cast<uint32_t>(__cvta_generic_to_shared(&nbar[i / 2][i % 2]))) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) buf[threadIdx.x] = rank;
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    const uint32_t local_buf = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
    uint32_t nb_buf;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(nb_buf) : "r"(local_buf), "r"(has_r ? rank + 1 : rank));
    auto remote_bar = [&](int side, int b, unsigned to) {
        uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(&nbar[side][b])), r;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(to));
        return r;
    };
    double acc = 0;
    const uint64_t t0 = gtimer();
    const long long c0 = clock64();
    for (int ph = 0; ph < iters; ++ph) {
        double v;
        asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(nb_buf) : "memory");
        acc += v;
        __syncthreads();
        if (threadIdx.x == 0) {
            const int b = ph & 1;
            const uint32_t par = (ph >> 1) & 1;
            if (has_l) asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar(1, b, rank - 1)) : "memory");
            if (has_r) asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar(0, b, rank + 1)) : "memory");
            for (int side = 0; side < 2; ++side) {
                if (side == 0 ? !has_l : !has_r) continue;
                const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(&nbar[side][b]));
                asm volatile(
                    "{\n\t.reg .pred p;\n"
                    "NBW_%=:\n\t"
                    "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
                    "@!p bra NBW_%=;\n}" ::"r"(a), "r"(par) : "memory");
            }
        }
        __syncthreads();
    }
    const long long c1 = clock64();
    const uint64_t t1 = gtimer();
    if (rank == 0 && threadIdx.x == 0) {
        out[0] = double(c1 - c0) / iters;
        out[1] = double(t1 - t0) / iters;
    }
    if (acc == -1.0) out[2] = acc;
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Neighbour-only exchange across a co-resident grid (the wide-halo kernel's
// grid exchange, rod_halo.cuh): per round every CTA writes a halo word,
// bar.sync, thread 0 fences, publishes its flag (release.gpu) and acquires
// both neighbours', bar.sync, then reads the neighbour's word through L2.
// mode 0: __threadfence + st.release + ld.acquire polls (the kernel's);
//      1: st.release + ld.acquire, no fence (release cumulativity over the
//         CTA barrier); 2: no fence, relaxed polls + one fence.acq_rel after
__global__ void grid_flag_kernel(double* out, int* flags, double* halo, int iters, int mode) {
    const int rank = blockIdx.x, n = gridDim.x;
    const bool has_l = rank > 0, has_r = rank + 1 < n;
    double acc = 0;
    __syncthreads();
    const uint64_t t0 = gtimer();
    const long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (threadIdx.x == 0) halo[2 * rank + (it & 1) * 2 * n] = double(it);
        __syncthreads();
        if (threadIdx.x == 0) {
            if (mode == 0) __threadfence();
            asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(flags + rank), "r"(it + 1) : "memory");
            int v;
            if (mode < 2) {
                if (has_l)
                    do asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(flags + rank - 1) : "memory");
                    while (v < it + 1);
                if (has_r)
                    do asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(flags + rank + 1) : "memory");
                    while (v < it + 1);
            } else {
                int vl = it + 1, vr = it + 1;
                do {
                    if (has_l) asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(vl) : "l"(flags + rank - 1) : "memory");
                    if (has_r) asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(vr) : "l"(flags + rank + 1) : "memory");
                } while (vl < it + 1 || vr < it + 1);
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && has_r) acc += __ldcg(halo + 2 * (rank + 1) + (it & 1) * 2 * n);
    }
    const long long c1 = clock64();
    const uint64_t t1 = gtimer();
    if (rank == 0 && threadIdx.x == 0) {
        out[0] = double(c1 - c0) / iters;
        out[1] = double(t1 - t0) / iters;
    }
    if (acc == -1.0) out[2] = acc;
}

// DSMEM dependent remote load latency (thread 0 of rank 0 chases through
// rank 1's shared memory)
__global__ void dsmem_kernel(double* out, int iters) {
    __shared__ int nxt[256];
    unsigned rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    for (int i = threadIdx.x; i < 256; i += blockDim.x) nxt[i] = (i + 31) & 255;
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (rank == 0 && threadIdx.x == 0) {
        uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(nxt)), rbase;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbase) : "r"(base), "r"(1));
        int p = 0;
        const long long c0 = clock64();
        for (int i = 0; i < iters; ++i) {
            int v;
            asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(rbase + 4u * p) : "memory");
            p = v;
        }
        const long long c1 = clock64();
        out[0] = double(c1 - c0) / iters;
        out[1] = 0;
        if (p == -1) out[2] = p;
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// kind: 0 DADD, 1 DMUL, 2 DFMA, 3 IEEE div, 4 sqrt(+add), 5 div_rn, 6 1/x
//       (chains; param unused), 7 LDS chase, 8 bar.sync (param = threads),
//       9 cluster barrier (param = CTAs), 10 DSMEM chase (2-CTA cluster),
//       11 neighbour mbarrier sync (param = CTAs), 12 grid neighbour flag
//       exchange (param = CTAs)
cudaError_t run(int kind, int param, double* res) {
    double* buf = nullptr;
    cudaError_t e = cudaMalloc(&buf, 4 * sizeof(double));
    if (e != cudaSuccess) return e;
    const int iters = 4096;
    auto launch = [&]() -> cudaError_t {
        switch (kind) {
            case 0: chain_kernel<0><<<1, 32>>>(buf, iters, 1.0, 1e-9); break;
            case 1: chain_kernel<1><<<1, 32>>>(buf, iters, 1.0, 1.0000001); break;
            case 2: chain_kernel<2><<<1, 32>>>(buf, iters, 1e-9, 0.999); break;
            case 3: chain_kernel<3><<<1, 32>>>(buf, iters, 1.0, 1.0000001); break;
            case 4: chain_kernel<4><<<1, 32>>>(buf, iters, 0.5, 1.0); break;
            case 5: chain_kernel<5><<<1, 32>>>(buf, iters, 1.0, 1.0000001); break;
            case 6: chain_kernel<6><<<1, 32>>>(buf, iters, 1.5, 1.0); break;
            case 7: lds_kernel<<<1, 32>>>(buf, iters); break;
            case 8: bar_kernel<<<1, param>>>(buf, iters); break;
            case 9:
            case 10:
            case 11: {
                cudaLaunchConfig_t cfg = {};
                const int c = kind == 10 ? 2 : param;
                cfg.gridDim = dim3(c);
                cfg.blockDim = dim3(kind == 10 ? 32 : 128);
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = c;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                if (kind == 11) {
                    if (c > 8) cudaFuncSetAttribute(nb_sync_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                    return cudaLaunchKernelEx(&cfg, nb_sync_kernel, buf, iters);
                }
                if (kind == 9) {
                    if (c > 8) cudaFuncSetAttribute(cluster_bar_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                    return cudaLaunchKernelEx(&cfg, cluster_bar_kernel, buf, iters);
                }
                return cudaLaunchKernelEx(&cfg, dsmem_kernel, buf, iters);
            }
            case 12: {   // grid neighbour exchange, param CTAs (co-resident)
                int* flags = nullptr;
                double* halo = nullptr;
                const int np_ = param & 0xffff;
                cudaError_t e2 = cudaMalloc(&flags, sizeof(int) * np_);
                if (e2 == cudaSuccess) e2 = cudaMalloc(&halo, sizeof(double) * 4 * np_);
                if (e2 == cudaSuccess) e2 = cudaMemset(flags, 0, sizeof(int) * np_);
                if (e2 == cudaSuccess) {
                    int it = iters, mode = param >> 16, n = param & 0xffff;
                    void* args[] = {&buf, &flags, &halo, &it, &mode};
                    e2 = cudaLaunchCooperativeKernel((const void*)grid_flag_kernel, dim3(n), dim3(128), args, 0, nullptr);
                }
                if (e2 == cudaSuccess) e2 = cudaDeviceSynchronize();
                cudaFree(flags);
                cudaFree(halo);
                return e2;
            }
            default: return cudaErrorInvalidValue;
        }
        return cudaGetLastError();
    };
    e = launch();   // warm-up
    if (e == cudaSuccess) e = launch();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(res, buf, 2 * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(buf);
    return e;
}

// Issue-rate microbenchmark for the compute cross-check of the roofline:
// `kind` 0 = DFMA, 1 = DADD, 2 = DMUL, 3 = FFMA; 8 independent chains per
// thread so the pipe, not latency, binds (explicit fma / + / *, so the TU's
// contraction flag does not change what is measured).
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

// Self-test hook: IEEE a/b against the reciprocal-based div_rn of the step
// kernel, compiled with the same mirror flags (tests/test_gpu_selftest.py).
__global__ void div_selftest_kernel(const double* a, const double* b, int64_t n, double* q_ieee,
                                    double* q_fast) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const double rb = 1.0 / b[i];
        q_ieee[i] = a[i] / b[i];
        q_fast[i] = div_rn(a[i], b[i], rb);
    }
}
// kind 0: 1/a, kind 1: sqrt(a) -- the compiler's IEEE result and the
// branch-free fast-path restatement (rcp_rn / sqrt_rn) the batched kernel uses
__global__ void fn_selftest_kernel(int kind, const double* a, int64_t n, double* r_ieee, double* r_fast) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const double x = a[i];
        r_ieee[i] = kind == 0 ? 1.0 / x : sqrt(x);
        r_fast[i] = kind == 0 ? rcp_rn(x) : sqrt_rn(x);
    }
}
cudaError_t fn_selftest(int kind, const double* a, int64_t n, double* r_ieee, double* r_fast) {
    fn_selftest_kernel<<<1184, 256>>>(kind, a, n, r_ieee, r_fast);
    return cudaDeviceSynchronize();
}
cudaError_t div_selftest(const double* a, const double* b, int64_t n, double* q_ieee, double* q_fast) {
    div_selftest_kernel<<<592, 256>>>(a, b, n, q_ieee, q_fast);
    return cudaDeviceSynchronize();
}

}  // namespace micro
}  // namespace rsb

extern "C" int rs_micro(int kind, int param, double* cycles_ns) {
    return rsb::micro::run(kind, param, cycles_ns) == cudaSuccess ? 0 : -2;
}
