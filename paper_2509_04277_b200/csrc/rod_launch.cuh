// rod_launch.cuh -- instantiation table and launchers for rod_step_kernel.
// Included by one translation unit per arithmetic mode; RSB_MODE_NS names
// the mode (mirror: --fmad=false fp64, bit-identical to the reference;
// fast: contraction allowed, fp32 and fp64).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>

#include "rod_step.cuh"
#if !RSB_FEAT
#include "rod_batch.cuh"
#include "rod_halo.cuh"
#include "rod_warp.cuh"
#endif

#if !defined(RSB_MODE_NS) || !defined(RSB_MODE_ID) || !defined(RSB_FEAT)
#error "define RSB_MODE_NS, RSB_MODE_ID and RSB_FEAT before including rod_launch.cuh"
#endif

namespace rsb {
namespace RSB_MODE_NS {

// (slots per thread S, slot capacity per CTA CAP): up to max_threads(S, CAP)
// threads cover S slots each (S odd: strided, S even: paired), CAP leaves
// room for the tail slot.
//   V0 (1,132)  V1 (1,258)  V2 (1,514)  V3 (2,770)  V4 (4,1154)
//   V5 (1,130) and V6 (2,130): batches of 129-point rods, 5 CTAs per SM
//   V7 (2,136): the same without the TMA staging buffer, 8 CTAs per SM
// Cluster tier: V0, V1, V2, V4; grid tier: V2, V4.  Each precision mode is
// compiled twice (RSB_FEAT 0 / 1): without and with the contact and
// self-collision phases; the feature TUs carry the CTA V0-V2, V4, cluster and
// grid variants only (the planner keeps such scenes on those).

// The kernel's function attributes, once per kernel and device (two driver
// calls per launch otherwise -- a haptic frame is one launch): the dynamic
// shared-memory limit at the opt-in maximum (the limit only gates launches;
// occupancy follows the size a launch or query passes) and all of the
// unified L1/shared array as shared memory -- several CTAs (rods) per SM
// are what hides latency in the batched case.
constexpr int kMaxDynSmem = 232448;   // 227 KB opt-in per CTA on sm_100
template <typename Fn>
static cudaError_t configure_once(Fn fn, std::atomic<bool>* done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64 && done[dev].load(std::memory_order_acquire)) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                             int(cudaSharedmemCarveoutMaxShared));
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) done[dev].store(true, std::memory_order_release);
    return cudaSuccess;
}

// clusters of more than 8 CTAs (non-portable sizes): the function attribute
// is set once per device like the ones above, not before every launch (a
// driver call that cost K = 1 launches of 16-CTA clusters host time)
template <typename Fn>
static cudaError_t allow_wide_clusters(Fn fn, std::atomic<bool>* done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64 && done[dev].load(std::memory_order_acquire)) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) done[dev].store(true, std::memory_order_release);
    return cudaSuccess;
}

template <typename Real, int S, int CAP, int TIER, int UNI>
static std::atomic<bool>* configured_flags() {
    static std::atomic<bool> done[64];
    return done;
}

template <typename Real, int S, int CAP, int TIER, int UNI>
static cudaError_t launch_one(const StepArgs<Real>& a, int ncta, int threads,
                              size_t smem, int cluster, cudaStream_t st) {
    auto fn = rod_step_kernel<Real, S, CAP, TIER, UNI, RSB_MODE_ID>;
    cudaError_t e = configure_once(fn, configured_flags<Real, S, CAP, TIER, UNI>());
    if (e != cudaSuccess) return e;
    if constexpr (TIER == TIER_CLUSTER) {
        if (cluster > 8) {
            static std::atomic<bool> wide[64];
            e = allow_wide_clusters(fn, wide);
            if (e != cudaSuccess) return e;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ncta);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cluster;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        // programmatic dependent launch (the kernel waits on the previous
        // grid before touching memory): hides the launch gap of K = 1 epochs
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 2;
        return cudaLaunchKernelEx(&cfg, fn, a);
    } else if constexpr (TIER == TIER_GRID) {
        void* args[] = {const_cast<StepArgs<Real>*>(&a)};
        return cudaLaunchCooperativeKernel((const void*)fn, dim3(ncta), dim3(threads), args, smem, st);
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ncta);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, fn, a);
    }
}

template <typename Real, int S, int CAP, int TIER, int UNI>
static cudaError_t occupancy_one(int threads, size_t smem, int cluster, int* out) {
    auto fn = rod_step_kernel<Real, S, CAP, TIER, UNI, RSB_MODE_ID>;
    cudaError_t e = configure_once(fn, configured_flags<Real, S, CAP, TIER, UNI>());
    if (e != cudaSuccess) return e;
    if constexpr (TIER == TIER_CLUSTER) {
        if (cluster > 8) {
            static std::atomic<bool> wide[64];
            e = allow_wide_clusters(fn, wide);
            if (e != cudaSuccess) return e;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cluster);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cluster;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaOccupancyMaxActiveClusters(out, (void*)fn, &cfg);
    } else {
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, fn, threads, smem);
    }
}

// what: 0 = launch, 1 = occupancy query
// cfg = uni + 3 feat.  uni: material constants 0 per slot, 1 CTA-uniform
// (registers), 2 launch-uniform (kernel parameters); feat: the scene has
// mesh contacts or self-collision (those phases are compiled only into the
// feat kernels -- they cost the plain step registers).  The stream tier has
// no feat kernels (the planner keeps such scenes off it).
template <typename Real, int S, int CAP, int TIER>
static cudaError_t dispatch_uni(int what, int cfg, const StepArgs<Real>* a, int ncta, int threads,
                                size_t smem, int cluster, cudaStream_t st, int* out) {
    // this translation unit holds cfg 3 RSB_FEAT .. 3 RSB_FEAT + 2
    constexpr int C0 = 3 * RSB_FEAT;
#define RSB_U(C)                                                                                          \
    case C:                                                                                               \
        return what == 0 ? launch_one<Real, S, CAP, TIER, C0 + C>(*a, ncta, threads, smem, cluster, st) \
                         : occupancy_one<Real, S, CAP, TIER, C0 + C>(threads, smem, cluster, out);
    switch (cfg - C0) {
        RSB_U(0)
        RSB_U(1)
        RSB_U(2)
    }
#undef RSB_U
    return cudaErrorInvalidValue;
}

// cfg 6..8: the speculative batched kernel (stream tier, variant 7 only)
template <typename Real, int S, int CAP, int TIER>
static cudaError_t dispatch_spec(int what, int cfg, const StepArgs<Real>* a, int ncta, int threads,
                                 size_t smem, int cluster, cudaStream_t st, int* out) {
#define RSB_U(C)                                                                                          \
    case C:                                                                                               \
        return what == 0 ? launch_one<Real, S, CAP, TIER, 6 + C>(*a, ncta, threads, smem, cluster, st) \
                         : occupancy_one<Real, S, CAP, TIER, 6 + C>(threads, smem, cluster, out);
    switch (cfg - 6) {
        RSB_U(0)
        RSB_U(1)
        RSB_U(2)
    }
#undef RSB_U
    return cudaErrorInvalidValue;
}

template <typename Real>
static cudaError_t dispatch(int what, int variant, int tier, int uni, const StepArgs<Real>* a,
                            int ncta, int threads, size_t smem, int cluster, cudaStream_t st,
                            int* out) {
#define RSB_D(S, CAP, TIER) dispatch_uni<Real, S, CAP, TIER>(what, uni, a, ncta, threads, smem, cluster, st, out)
#if RSB_FEAT
    // scenes with contacts / self-collision: plain CTA, cluster, grid only
    if (tier == TIER_CTA) {
        switch (variant) {
            case 0: return RSB_D(1, 132, TIER_CTA);
            case 1: return RSB_D(1, 258, TIER_CTA);
            case 2: return RSB_D(1, 514, TIER_CTA);
            case 4: return RSB_D(4, 1154, TIER_CTA);
        }
    }
#else
    if (tier == TIER_CTA) {
        if (uni >= 6) {   // speculative single-rod kernels
            if (variant == 0)
                return dispatch_spec<Real, 1, 132, TIER_CTA>(what, uni, a, ncta, threads, smem, cluster, st, out);
            return cudaErrorInvalidValue;
        }
        switch (variant) {
            case 0: return RSB_D(1, 132, TIER_CTA);
            case 1: return RSB_D(1, 258, TIER_CTA);
            case 2: return RSB_D(1, 514, TIER_CTA);
            case 3: return RSB_D(2, 770, TIER_CTA);
            case 4: return RSB_D(4, 1154, TIER_CTA);
            case 5: return RSB_D(1, 130, TIER_CTA);
            case 6: return RSB_D(2, 130, TIER_CTA);
            case 7: return RSB_D(2, 136, TIER_CTA);
        }
    } else if (tier == TIER_STREAM) {
        if (uni >= 6 && variant == 7)
            return dispatch_spec<Real, 2, 136, TIER_STREAM>(what, uni, a, ncta, threads, smem, cluster, st, out);
        switch (variant) {
            case 5: return RSB_D(1, 130, TIER_STREAM);
            case 6: return RSB_D(2, 130, TIER_STREAM);
            case 7: return RSB_D(2, 136, TIER_STREAM);
        }
    }
#endif
    if (tier == TIER_CLUSTER) {
        switch (variant) {
            case 0: return RSB_D(1, 132, TIER_CLUSTER);
            case 1: return RSB_D(1, 258, TIER_CLUSTER);
            case 2: return RSB_D(1, 514, TIER_CLUSTER);
            case 4: return RSB_D(4, 1154, TIER_CLUSTER);
        }
    } else if (tier == TIER_GRID) {
        switch (variant) {
            case 2: return RSB_D(1, 514, TIER_GRID);
            case 4: return RSB_D(4, 1154, TIER_GRID);
        }
    }
#undef RSB_D
    return cudaErrorInvalidValue;
}

template <typename Real>
cudaError_t launch_step(int variant, int tier, int uni, const StepArgs<Real>& a, int ncta,
                        int threads, size_t smem, int cluster, cudaStream_t st) {
    return dispatch<Real>(0, variant, tier, uni, &a, ncta, threads, smem, cluster, st, nullptr);
}

template <typename Real>
cudaError_t occupancy(int variant, int tier, int uni, int threads, size_t smem, int cluster, int* out) {
    return dispatch<Real>(1, variant, tier, uni, nullptr, 0, threads, smem, cluster, nullptr, out);
}


#if !RSB_FEAT
// The warp-per-rod batched kernel (rod_batch.cuh): launch shape `shape`
// (kBwShapes), `grid` persistent CTAs.
template <typename Real, int SH, bool GEN>
static cudaError_t batch_one(int what, const StepArgs<Real>* a, int grid, cudaStream_t st, int* out) {
    constexpr BwShape sh = kBwShapes[SH];
    auto fn = rod_batch_kernel<Real, RSB_MODE_ID, sh.wpc, sh.minb, GEN, sh.shst>;
    static std::atomic<bool> done[64];
    cudaError_t e = configure_once(fn, done);
    if (e != cudaSuccess) return e;
    // RSB_BW_PAD (bytes, tuning experiments): extra shared memory per CTA,
    // i.e. fewer resident CTAs per SM
    static const size_t pad = [] {
        const char* e = getenv("RSB_BW_PAD");
        return e ? size_t(atol(e)) : size_t(0);
    }();
    const size_t smem = bw_smem_bytes<Real>(sh.wpc, sh.shst) + pad;
    if (what == 1) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, fn, 32 * sh.wpc, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(32 * sh.wpc);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fn, *a);
}

// The one-warp single-rod kernel (rod_warp.cuh): one warp per task.
template <typename Real, bool GEN, int FORM>
static cudaError_t warp_one(const StepArgs<Real>* a, int grid, cudaStream_t st) {
    auto fn = FORM == 1 ? rod_warp1_kernel<Real, RSB_MODE_ID, GEN> : rod_warp_kernel<Real, RSB_MODE_ID, GEN>;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fn, *a);
}
// form 1: one point per lane (rods <= 31 elements); 2: two per lane (32..63)
template <typename Real>
cudaError_t warp_step(int gen, int form, const StepArgs<Real>* a, int grid, cudaStream_t st) {
    switch (form) {
        case 1: return gen ? warp_one<Real, true, 1>(a, grid, st) : warp_one<Real, false, 1>(a, grid, st);
        case 2: return gen ? warp_one<Real, true, 2>(a, grid, st) : warp_one<Real, false, 2>(a, grid, st);
    }
    return cudaErrorInvalidValue;
}

// The wide-halo cluster kernel (rod_halo.cuh): one cluster of ncta CTAs.
template <typename Real, bool GEN, bool BIND, int TB, bool GX, bool XF>
static cudaError_t halo_one(int what, const StepArgs<Real>* a, int ncta, int threads, cudaStream_t st, int* out) {
    auto fn = rod_halo_kernel<Real, RSB_MODE_ID, GEN, BIND, TB, GX, XF>;
    static std::atomic<bool> done[64];
    cudaError_t e = configure_once(fn, done);
    if (e != cudaSuccess) return e;
    if constexpr (GX) {   // co-resident grid (cooperative launch)
        const size_t smem = halo_smem_bytes(threads, sizeof(Real));
        if (what == 1) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, fn, threads, smem);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ncta);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, fn, *a);
    }
    if (ncta > 8) {
        static std::atomic<bool> wide[64];
        e = allow_wide_clusters(fn, wide);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ncta);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = halo_smem_bytes(threads, sizeof(Real));
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ncta;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    if (what == 1) {
        cfg.numAttrs = 1;
        return cudaOccupancyMaxActiveClusters(out, (void*)fn, &cfg);
    }
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, fn, *a);
}
// what: 0 launch, 1 occupancy query (cluster: active clusters, grid: CTAs
// per SM); tb: 256 or 512; gx: grid exchange instead of one cluster; xf:
// grabs / live launches / barrier accounting compiled in
template <typename Real, bool XF>
static cudaError_t halo_sel(int what, int sel, const StepArgs<Real>* a, int ncta, int threads, cudaStream_t st,
                            int* out) {
    switch (sel) {
#define RSB_H(S, G, B, T, X) \
    case S: return halo_one<Real, G, B, T, X, XF>(what, a, ncta, threads, st, out);
        RSB_H(0, false, false, 256, false)
        RSB_H(1, true, false, 256, false)
        RSB_H(2, false, true, 256, false)
        RSB_H(3, true, true, 256, false)
        RSB_H(4, false, false, 512, false)
        RSB_H(5, true, false, 512, false)
        RSB_H(6, false, true, 512, false)
        RSB_H(7, true, true, 512, false)
        RSB_H(8, false, false, 256, true)
        RSB_H(9, true, false, 256, true)
        RSB_H(10, false, true, 256, true)
        RSB_H(11, true, true, 256, true)
        RSB_H(12, false, false, 512, true)
        RSB_H(13, true, false, 512, true)
        RSB_H(14, false, true, 512, true)
        RSB_H(15, true, true, 512, true)
#undef RSB_H
    }
    return cudaErrorInvalidValue;
}
template <typename Real>
cudaError_t halo_step(int what, int gen, int bind, int tb, int gx, int xf, const StepArgs<Real>* a, int ncta,
                      int threads, cudaStream_t st, int* out) {
    const int sel = (gen ? 1 : 0) | (bind ? 2 : 0) | (tb > 256 ? 4 : 0) | (gx ? 8 : 0);
    return xf ? halo_sel<Real, true>(what, sel, a, ncta, threads, st, out)
              : halo_sel<Real, false>(what, sel, a, ncta, threads, st, out);
}

// shape in [0, kBwNumShapes) with gen = false, or kBwNumShapes + shape for
// the GEN kernel (extensible elements / external forces: kBwGenShape only)
template <typename Real>
cudaError_t batch_step(int what, int sel, const StepArgs<Real>* a, int grid, cudaStream_t st, int* out) {
    switch (sel) {
        case 0: return batch_one<Real, 0, false>(what, a, grid, st, out);
        case 1: return batch_one<Real, 1, false>(what, a, grid, st, out);
        case 2: return batch_one<Real, 2, false>(what, a, grid, st, out);
        case 3: return batch_one<Real, 3, false>(what, a, grid, st, out);
        case kBwNumShapes + kBwGenShape: return batch_one<Real, kBwGenShape, true>(what, a, grid, st, out);
    }
    return cudaErrorInvalidValue;
}
#endif

}  // namespace RSB_MODE_NS
}  // namespace rsb
