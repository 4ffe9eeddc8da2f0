// rodsim_capi.cu -- host side of the C ABI (include/rodsim_b200.h):
// device mirrors of the World arrays, the launch planner (CTA / cluster /
// grid tiers), epoch execution, command ring and snapshot.
//
// The planner's job is to map the reference's "block" decomposition
// (partition.py, _core.pyx:360-377) onto the B200: whole rods are packed into
// CTAs; a rod (or a set of rods coupled by bindings) too large for one CTA is
// split across the CTAs of a thread-block cluster; a rod too large for a
// 16-CTA cluster runs on a cooperative grid.  The oracle is bitwise invariant
// to the partition, so the mapping is free.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/rodsim_b200.h"
#include "rod_common.h"
#include "rod_batch.cuh"
#include "rod_halo.cuh"
#include "rod_warp.cuh"
#include "rod_step.cuh"

// launchers of the six kernel translation units (csrc/rod_kernels.cu)
#define RSB_DECLARE_MODE(NS)                                                                       \
    namespace rsb {                                                                                \
    namespace NS {                                                                                 \
    template <typename Real>                                                                       \
    cudaError_t launch_step(int, int, int, const StepArgs<Real>&, int, int, size_t, int, cudaStream_t); \
    template <typename Real>                                                                       \
    cudaError_t occupancy(int, int, int, int, size_t, int, int*);                                 \
    template <typename Real>                                                                       \
    cudaError_t batch_step(int, int, const StepArgs<Real>*, int, cudaStream_t, int*);             \
    template <typename Real>                                                                       \
    cudaError_t warp_step(int, int, const StepArgs<Real>*, int, cudaStream_t);                    \
    template <typename Real>                                                                       \
    cudaError_t halo_step(int, int, int, int, int, int, const StepArgs<Real>*, int, int, cudaStream_t, int*); \
    }                                                                                              \
    }
RSB_DECLARE_MODE(mirror)
RSB_DECLARE_MODE(mirror_feat)
RSB_DECLARE_MODE(f32)
RSB_DECLARE_MODE(f32_feat)
RSB_DECLARE_MODE(f64fast)
RSB_DECLARE_MODE(f64fast_feat)
#undef RSB_DECLARE_MODE

using namespace rsb;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e_ = (x);                                                       \
        if (e_ != cudaSuccess)                                                      \
            return fail(RS_E_CUDA, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                        \
    } while (0)

struct Variant {
    int S, CAP;
    // slots the threads cover; one more (the element-less tail) fits in CAP
    constexpr int cover() const { return S * max_threads(S, CAP); }
};
// capacity-ordered variants 0..4, then the batched variants 5 (strided, 128
// threads) and 6 (paired, 64 threads) for 129-point rods
constexpr Variant kVariants[] = {{1, 132}, {1, 258}, {1, 514}, {2, 770}, {4, 1154}, {1, 130}, {2, 130}, {2, 136}};
constexpr int kNumVariants = 8;
constexpr int kNumCapVariants = 5;
constexpr int kBatchVariant = 7;   // batches of short rods; 5 and 6 on request
// Cluster CTAs, smallest first: a rod (or bound set) above kCtaMaxPoints is
// spread over as many CTAs (<= 16) of the smallest of these as it needs.
// Measured (profiles/, cfg4 N = 1024): one 256-thread CTA 24.7 us/step, a
// 9-CTA cluster of 128-point CTAs 13.8 us/step -- below ~512 points the
// cluster barrier (~300 ns) costs more than the single CTA's extra work.
constexpr int kClusterVariants[] = {0, 1, 2, 4};
constexpr int kCtaMaxPoints = 513;   // variant 2 covers 512 slots + the tail
// A rod without distance-projected elements steps in 3 phases (no colour
// sweeps), so its one CTA is bound by that SM's fp64 issue rather than by
// barriers, and a cluster pays from ~320 points on (extensible rods, K = 10:
// 384 points 4.88 -> 4.52 us/step, 512: 5.69 -> 4.70; 256: 3.77 vs 4.11,
// tools/ext_sweep.py).  Applied to worlds of a few rods only -- a batch
// keeps one rod per CTA.
constexpr int kCtaMaxPointsNoDist = 320;
constexpr int kFewSegments = 8;
constexpr int kMaxCluster = 16;
constexpr int kMaxStepsPerLaunch = 1 << 16;
constexpr size_t kMaxSmem = 232448;   // 227 KB opt-in per CTA on sm_100

struct Segment {     // consecutive rods that must share a CTA / cluster / grid
    int r0, r1;      // rods [r0, r1]
    int64_t p0, p1;  // points [p0, p1)
};

struct Group {       // one kernel launch
    int tier = TIER_CTA;
    int variant = 0;
    int uni = 0;                    // constants: 0 per slot, 1 per CTA, 2 per launch
    bool any_dist = true;           // some element of the launch is distance-projected
    int32_t e_launch = 0;           // element standing for the launch (uni == 2)
    int task_begin = 0, ncta = 0;   // tasks (one CTA each, except stream)
    int grid = 0;                   // CTAs launched (stream: persistent)
    int threads = 0;
    int cluster = 1;
    int bind_cap = 0, drv_cap = 0;
    size_t smem = 0;
    int32_t* d_flags = nullptr;   // grid tier
    void* d_halo = nullptr;
    // stream groups of 129-point World rods: the speculative launch runs the
    // warp-per-rod kernel (rod_batch.cuh) in launch shape bw_shape on
    // bw_grid persistent CTAs (-1: not eligible); bw_gen: extensible
    // elements (the general variant of the kernel, shape kBwGenShape on
    // bw_grid_gen CTAs -- also taken when external forces appear)
    int bw_shape = -1;
    bool bw_gen = false;
    int bw_grid_gen = 0;
    // CTA-tier groups of single rods of <= 64 elements: the speculative
    // launch runs the one-warp register-resident kernel (rod_warp.cuh)
    bool rw = false;
    bool rw_gen = false;            // ... with extensible elements (GEN kernel)
    int rw_form = 0;                // 1: every rod <= 31 elements (one point per lane),
                                    // 2: 32..63 (two per lane)
    int bw_grid = 0;
    // cluster groups of one rod or two rods bound point to point at the same
    // local index: the wide-halo kernel (rod_halo.cuh) takes the speculative
    // launch -- one cluster barrier per step instead of one per phase
    bool halo = false;
    bool h_gen = false, h_bind = false;
    int h_cta = 0, h_threads = 0, h_tb = 256, h_w = 0, h_g = 0, h_nr = 0, h_np = 0, h_iters = 0;
    int h_s = 1;                    // steps per ghost exchange (ghost width h_s (2I+1))
    int32_t h_poff[2] = {0, 0}, h_eoff[2] = {0, 0};
    bool h_gx = false;              // grid exchange (co-resident grid) instead of one cluster
    bool h_short = false;           // only for epochs shorter than kSpecMinSteps
    bool halo_only = false;         // no general kernel can step the group (coupled, past a cluster)
    std::vector<HaloTask> h_tasks;
    HaloTask* d_htask = nullptr;
    int32_t* d_hflags = nullptr;    // grid exchange: per-CTA flags, arrival count, vote OR
    int64_t* d_hfail = nullptr;     // lazy redo word (StepArgs::hfail)
    mutable int lazy_skip = 0;      // lazy one-warp launches paused after a replay
    void* d_hhalo = nullptr;        // grid exchange: (2, C, 2, NR, G, 13) halo records
};

// groups with speculative kernels: the batched stream variant and the
// smallest single-rod CTA variant (plain scenes -- the scene-feature kernels
// keep their fallbacks).  Larger one-CTA rods stay exact: a planar rod's
// torques carry rounding noise (~1e-300) below the fast path's window, and
// a 256-element sweep rod redid every launch (6.4 -> 9.9 us/step).
constexpr int kSpecMinSteps = 32;
constexpr int kHaloCtaMinPoints = 100;
constexpr int kHaloCtaShortPoints = 2;   // every one-CTA rod (tools/short_probe.py)
constexpr int kHaloGridSteps = 3;
constexpr int kSpecBackoff = 64;
bool spec_group(const Group& g) {
    return (g.tier == TIER_STREAM && g.variant == 7) || (g.tier == TIER_CTA && g.variant == 0);
}


struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

}  // namespace

struct rs_handle_s {
    rs_world_desc d{};
    int prec = RS_F64_MIRROR;
    size_t rsz = 8;                 // sizeof(Real) on the device
    cudaStream_t st = nullptr;
    cudaStream_t st_in = nullptr, st_out = nullptr;   // pipelined host epochs: H2D, D2H
    std::vector<cudaEvent_t> ev_in, ev_k;             // per-chunk copy / kernel events
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;   // per-epoch kernel timing
    cudaEvent_t tm0 = nullptr, tm1 = nullptr;   // caller-bracketed spans
    bool timing = false;
    bool timed = false;
    double last_ms = 0.0;
    int64_t launches = 0;
    int64_t launches_pipelined = 0;   // epochs run by run_epoch_pipelined
    int num_sms = 0;
    int debug = 0;                  // RSB_DEBUG env: bit 0 poisons smem
    bool spec = true;               // speculative batched launches (RSB_SPEC=0: off)
    bool bw_on = true;              // warp-per-rod batched kernel (RSB_BW=0: off)
    bool rw_on = true;              // one-warp single-rod kernel (RSB_RW=0: off)
    bool rw1_on = true;             // its one-point-per-lane form (RSB_RW1=0: off)
    bool halo_on = true;            // wide-halo cluster kernel (RSB_HALO=0: off)
    int halo_ctas = 0;              // its CTA count (RSB_HALO_CTAS; 0: the planner's)
    int halo_grid = -1;             // RSB_HALO_GRID: 1 grid exchange, 0 cluster only, -1 the planner's
    int halo_width = 128;           // RSB_HALO_W: target threads per CTA of the grid exchange
    int halo_steps = 0;             // RSB_HALO_STEPS: steps per exchange (0: the planner's)
    int max_k = kMaxStepsPerLaunch; // RSB_MAX_K: steps per launch cap (launch-cost probes)
    int halo_short = kHaloCtaShortPoints;   // RSB_HALO_SHORT: smallest one-CTA rod on the halo kernel
    bool rw_lazy = true;            // RSB_RW_LAZY=0: one-warp rods only with a consume launch, K >= 32
    int pipe_chunks = 16;           // RSB_PIPE_CHUNKS: chunks of a pipelined host epoch
    bool halo_pending = false;      // wide-halo launches not yet checked for a failed vote
    bool halo_check_enqueued = false;   // their redo words are on the way to h_hfail
    int64_t* h_hfail = nullptr;     // pinned, one per group
    size_t h_hfail_n = 0;
    bool last_halo = false;         // the last launch was a wide-halo launch
    int64_t halo_redone = 0;        // groups replayed exactly at the last check
    int halo_cta = -1;              // RSB_HALO_CTA: one-CTA segments (-1: from kHaloCtaMinPoints)
    int bw_shape = -1;              // its launch shape (RSB_BW_SHAPE, kBwShapes; -1: the planner's)
    DevBuf redo_list, redo_count;   // rods the speculative launch left to the exact one
    bool last_spec = false;         // the last launch speculated (rs_last_redo_count)
    // speculation back-off of one-CTA / one-warp rod groups: a rod whose
    // dividends keep leaving the fast path's window (rounding noise below
    // 2^-400) would pay the exact redo launch every epoch.  The redo count
    // of each speculative launch is copied back asynchronously; three
    // launches in a row that needed the redo turn speculation off for the
    // group's next kSpecBackoff launches.
    std::vector<int> spec_streak, spec_skip;
    std::vector<cudaEvent_t> redo_ev;
    std::vector<char> redo_ev_live;
    int32_t* h_redo = nullptr;      // pinned, one slot per group
    bool dry = false;               // planning only (rs_plan_dry): no CUDA calls

    // device mirrors
    DevBuf pos, vel, q, w;
    DevBuf rest, ustar, inert, ks, kp, gt, gr, kb, mass, invm, fext, drv_v, drv_rot;
    DevBuf pflags, pt_elem, tasks, binds, drvs, grabs;
    DevBuf hdrv, hbind;             // wide-halo kernel: per-point driver rods, binding codes
    std::vector<int32_t> h_hdrv, h_hbind;
    // mesh contacts: tree + mesh (static), contact slots (state)
    DevBuf nmin, nmax, verts, nstart, ncount, torder, tris, cradii, cmask;
    DevBuf cact, cnorm, cdepth, cacc_n, cacc_t;
    // self-collision: group table (static), pair list (state), count (device)
    DevBuf grp_rod, grp_gi, grp_s, grp_e, grp_c, gp_count, pair_a, pair_b, pair_md, pair_acc;
    int32_t* d_pairs = nullptr;             // CNT_PAIRS, persistent like the ctx counter
    int contacts_on = 0;                    // any contact machinery needed
    unsigned long long* d_contacts = nullptr;
    unsigned long long* h_contacts = nullptr;   // pinned
    unsigned long long* d_err = nullptr;
    unsigned long long* h_err = nullptr;   // pinned
    unsigned long long* d_prof = nullptr;  // RSB_DEBUG bit 1: per-phase cycles (CTA 0)
    bool bar_timing = false;               // rs_barrier_timing: barrier wait cycles
    unsigned long long* d_bar = nullptr;
    unsigned long long* h_bar = nullptr;   // pinned
    int clock_khz = 0;                     // SM clock for cycles -> ns
    int64_t prof_steps = 0;
    int has_fext = 0;

    // plan
    std::vector<CtaTask> h_tasks;
    std::vector<BindEntry> h_binds;
    std::vector<DrvEntry> h_drvs;
    std::vector<GrabEntry> h_grabs;
    std::vector<Group> groups;
    std::vector<int64_t> task_p0_sorted;   // (p0, task) lookup for grabs
    std::vector<int> task_by_p0;
    std::vector<int> task_group;
    bool planned = false;

    // counters, ring, snapshot
    int64_t step = 0;
    int64_t err_step = -1;
    bool err_pending = false;       // d_err changed since the last read-back
    std::mutex ring_mu;
    LiveRing* ring = nullptr;       // page-locked, device-mapped (rod_common.h)
    LiveRing* ring_dev = nullptr;   // its device address
    bool live = false;              // the plan is one CTA / one cluster: the
                                    // kernel drains the ring at every step
    DevBuf g_act_d, g_pt_d, g_tgt_d;   // world grab slots on the device (live)
    LiveSnap* snap = nullptr;          // live per-step snapshot, mapped host memory
    LiveSnap* snap_dev = nullptr;
    double *snap_pos = nullptr, *snap_q = nullptr;         // (2,P,3), (2,E,4) mapped
    double *snap_pos_dev = nullptr, *snap_q_dev = nullptr;
    int64_t snap_version = 0;          // published snapshot version (host view)
    bool snap_on = false;              // per-step snapshots requested (rs_live_snapshots)
    bool control_dirty = false;
    std::vector<char> static_snap;  // static arrays at the last RS_STATIC upload
    // last uploaded controls (upload_control skips unchanged ones)
    bool ctl_valid = false;
    std::vector<double> ctl_drv_v, ctl_drv_rot, ctl_g_tgt;
    std::vector<uint8_t> ctl_g_act;
    std::vector<int64_t> ctl_g_pt;
    int64_t snap_seq = 0, snap_step = 0;

    // host staging (pinned) for precision conversion
    void* stage = nullptr;
    size_t stage_bytes = 0;
    std::vector<void*> registered;
    double* map_state[4] = {nullptr, nullptr, nullptr, nullptr};   // device aliases of pos, vel, q, w
    bool xfer_on = true;            // RSB_XFER=0: small worlds' host epochs through copy commands
};

namespace {

int dev_alloc(DevBuf& b, size_t bytes) {
    if (b.bytes >= bytes && b.p) return RS_OK;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    if (bytes == 0) return RS_OK;
    // +64 B: the stream tier's 16-byte-aligned bulk copies may read up to
    // 15 bytes past the last rod's block
    CK(cudaMalloc(&b.p, bytes + 64));
    b.bytes = bytes;
    return RS_OK;
}

int ensure_stage(rs_handle h, size_t bytes) {
    if (h->stage_bytes >= bytes) return RS_OK;
    if (h->stage) {
        cudaStreamSynchronize(h->st);
        cudaFreeHost(h->stage);
    }
    h->stage = nullptr;
    h->stage_bytes = 0;
    CK(cudaMallocHost(&h->stage, bytes));
    h->stage_bytes = bytes;
    return RS_OK;
}

// host double array -> device Real array
// Several copies between the World's host arrays and the device, collected
// and issued back to back on one stream (one cudaMemcpyAsync per array).
struct CopyBatch {
    void* dst[8];
    void* src[8];
    size_t size[8];
    size_t n = 0;
    void add(void* d, const void* s, size_t bytes) {
        if (bytes == 0) return;
        dst[n] = d;
        src[n] = const_cast<void*>(s);
        size[n] = bytes;
        ++n;
    }
};

int flush_batch(rs_handle h, CopyBatch& b, cudaStream_t st = nullptr) {
    if (!st) st = h->st;
    for (size_t i = 0; i < b.n; ++i)
        CK(cudaMemcpyAsync(b.dst[i], b.src[i], b.size[i], cudaMemcpyDefault, st));
    b.n = 0;
    return RS_OK;
}

int put_real(rs_handle h, DevBuf& b, const double* src, size_t count) {
    int rc = dev_alloc(b, std::max<size_t>(count, 1) * h->rsz);
    if (rc) return rc;
    if (count == 0 || !src) return RS_OK;
    if (h->rsz == sizeof(double)) {
        CK(cudaMemcpyAsync(b.p, src, count * sizeof(double), cudaMemcpyHostToDevice, h->st));
    } else {
        rc = ensure_stage(h, count * sizeof(float));
        if (rc) return rc;
        CK(cudaStreamSynchronize(h->st));   // staging buffer reuse
        float* s = static_cast<float*>(h->stage);
        for (size_t i = 0; i < count; ++i) s[i] = float(src[i]);
        CK(cudaMemcpyAsync(b.p, s, count * sizeof(float), cudaMemcpyHostToDevice, h->st));
        CK(cudaStreamSynchronize(h->st));
    }
    return RS_OK;
}

// device Real array -> host double array (synchronous for fp32)
int get_real(rs_handle h, const DevBuf& b, double* dst, size_t count) {
    if (count == 0 || !dst) return RS_OK;
    if (h->rsz == sizeof(double)) {
        CK(cudaMemcpyAsync(dst, b.p, count * sizeof(double), cudaMemcpyDeviceToHost, h->st));
    } else {
        int rc = ensure_stage(h, count * sizeof(float));
        if (rc) return rc;
        CK(cudaMemcpyAsync(h->stage, b.p, count * sizeof(float), cudaMemcpyDeviceToHost, h->st));
        CK(cudaStreamSynchronize(h->st));
        const float* s = static_cast<const float*>(h->stage);
        for (size_t i = 0; i < count; ++i) dst[i] = double(s[i]);
    }
    return RS_OK;
}

// host int64 array -> device int32 (mesh indices; validated < 2^31)
int put_i32(rs_handle h, DevBuf& b, const int64_t* src, size_t count) {
    std::vector<int32_t> v(count);
    for (size_t i = 0; i < count; ++i) {
        if (src[i] < INT32_MIN || src[i] > INT32_MAX) return fail(RS_E_INVALID, "mesh index out of int32 range");
        v[i] = int32_t(src[i]);
    }
    int rc = dev_alloc(b, std::max<size_t>(count, 1) * sizeof(int32_t));
    if (rc) return rc;
    if (count) CK(cudaMemcpyAsync(b.p, v.data(), count * sizeof(int32_t), cudaMemcpyHostToDevice, h->st));
    CK(cudaStreamSynchronize(h->st));
    return RS_OK;
}

int put_u8(rs_handle h, DevBuf& b, const uint8_t* src, size_t count) {
    int rc = dev_alloc(b, std::max<size_t>(count, 1));
    if (rc) return rc;
    if (count) CK(cudaMemcpyAsync(b.p, src, count, cudaMemcpyHostToDevice, h->st));
    return RS_OK;
}

template <typename T>
int put_vec(rs_handle h, DevBuf& b, const std::vector<T>& v) {
    int rc = dev_alloc(b, std::max<size_t>(v.size(), 1) * sizeof(T));
    if (rc) return rc;
    if (!v.empty()) CK(cudaMemcpyAsync(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, h->st));
    // the vectors may be rebuilt before the copy runs
    CK(cudaStreamSynchronize(h->st));
    return RS_OK;
}

int64_t rod_of(const rs_world_desc& d, int64_t p) {
    const int64_t* o = d.rod_offsets;
    return int64_t(std::upper_bound(o, o + d.R + 1, p) - o) - 1;
}

// ---- launch planning --------------------------------------------------------

// kernel configuration: material-constant storage + scene features
// (barrier timing: the feature kernels, where the group's variant has one)
bool has_feat_kernel(const Group& g) {
    return g.tier == TIER_CLUSTER || g.tier == TIER_GRID ||
           (g.tier == TIER_CTA && g.variant <= 4 && g.variant != 3);
}

int launch_cfg(rs_handle h, const Group& g) {
    const bool feat = ((h->contacts_on || h->d.has_self || h->live) && g.tier != TIER_STREAM) ||
                      (h->bar_timing && has_feat_kernel(g));
    return g.uni + (feat ? 3 : 0);
}

int occupancy_query(rs_handle h, int variant, int tier, int uni, int threads, size_t smem,
                    int cluster, int* out) {
    cudaError_t e;
    if (h->prec == RS_F64_MIRROR)
        e = uni >= 3 ? mirror_feat::occupancy<double>(variant, tier, uni, threads, smem, cluster, out)
                     : mirror::occupancy<double>(variant, tier, uni, threads, smem, cluster, out);
    else if (h->prec == RS_F32)
        e = uni >= 3 ? f32_feat::occupancy<float>(variant, tier, uni, threads, smem, cluster, out)
                     : f32::occupancy<float>(variant, tier, uni, threads, smem, cluster, out);
    else
        e = uni >= 3 ? f64fast_feat::occupancy<double>(variant, tier, uni, threads, smem, cluster, out)
                     : f64fast::occupancy<double>(variant, tier, uni, threads, smem, cluster, out);
    if (e != cudaSuccess)
        return fail(RS_E_CUDA, "occupancy query failed: %s", cudaGetErrorString(e));
    return RS_OK;
}

int batch_occupancy(rs_handle h, int shape, int* out) {
    cudaError_t e;
    if (h->prec == RS_F64_MIRROR) e = mirror::batch_step<double>(1, shape, nullptr, 0, nullptr, out);
    else if (h->prec == RS_F32) e = f32::batch_step<float>(1, shape, nullptr, 0, nullptr, out);
    else e = f64fast::batch_step<double>(1, shape, nullptr, 0, nullptr, out);
    if (e != cudaSuccess) return fail(RS_E_CUDA, "batch kernel occupancy query failed: %s", cudaGetErrorString(e));
    return RS_OK;
}

bool elem_consts_equal(const rs_world_desc& d, int64_t a, int64_t b) {
    auto eq = [](double x, double y) { return std::memcmp(&x, &y, sizeof x) == 0; };
    if (!eq(d.rest[a], d.rest[b]) || !eq(d.ks[a], d.ks[b]) || !eq(d.kp[a], d.kp[b]) ||
        !eq(d.gt[a], d.gt[b]) || !eq(d.gr[a], d.gr[b]))
        return false;
    for (int k = 0; k < 3; ++k)
        if (!eq(d.kb[3 * a + k], d.kb[3 * b + k]) || !eq(d.ustar[3 * a + k], d.ustar[3 * b + k]) ||
            !eq(d.inert[3 * a + k], d.inert[3 * b + k]))
            return false;
    return true;
}

int halo_query(rs_handle h, const Group& g, int* out);

// Wide-halo kernel (rod_halo.cuh) for cluster groups: one rod, or two rods of
// equal length bound point to point at the same local index (a matching), with
// the structural flags of World rods (junctions inside a rod, colours by local
// index), launch-uniform material constants and no scene features.  Each CTA
// owns ~np / C consecutive local indices plus G = 2I + 1 ghost points per
// side; the planner takes the largest cluster (<= 16) whose CTAs own at least
// G points each.
int plan_halo_groups(rs_handle h, const std::vector<uint32_t>& pflags, const std::vector<int32_t>& pt_elem);
int plan_halo(rs_handle h, const std::vector<uint32_t>& pflags, const std::vector<int32_t>& pt_elem) {
    int rc = plan_halo_groups(h, pflags, pt_elem);
    if (rc) return rc;
    for (const Group& g : h->groups)
        if (g.halo_only && !g.halo)
            return fail(RS_E_UNSUPPORTED, "coupled rods larger than a %d-CTA cluster need the wide-halo kernel "
                        "(two equal rods bound at the same local index, launch-uniform material)", kMaxCluster);
    return RS_OK;
}
int plan_halo_groups(rs_handle h, const std::vector<uint32_t>& pflags, const std::vector<int32_t>& pt_elem) {
    const rs_world_desc& d = h->d;
    const int64_t P = d.P;
    h->h_hdrv.assign(size_t(2 * P), -1);
    h->h_hbind.assign(size_t(P), -1);
    for (int64_t r = 0; r < d.R; ++r) {   // rod order: the last rod driving a point wins
        if (d.drv_pt[r] >= 0 && d.drv_pt[r] < P) h->h_hdrv[size_t(2 * d.drv_pt[r])] = int32_t(r);
        if (d.drv_fr[r] >= 0 && d.drv_fr[r] < d.E) h->h_hdrv[size_t(2 * d.elem_point[d.drv_fr[r]] + 1)] = int32_t(r);
    }
    for (Group& g : h->groups) {
        g.halo = false;
        // one-CTA segments (a single task) of >= kHaloCtaMinPoints points:
        // spread over a cluster as well (cfg4, K = 100: 128 elements 4.31 ->
        // 3.93 us/step, 256: 6.23 -> 3.97, 512: 9.59 -> 4.06; the 64-element
        // cantilever stays on its CTA, 3.80 vs 3.91).  RSB_HALO_CTA: 0 never,
        // 1 at any size
        // (two tasks: two equal rods, one per CTA -- the same column layout
        // as a bound pair, without the bindings)
        // Smaller one-CTA rods (kHaloCtaShortPoints .. kHaloCtaMinPoints)
        // take it as ONE CTA, no ghosts (cfg4, K = 100: 96 points 4.04 ->
        // 3.83 us per step, 64 elements 3.81 -> 3.75; K = 10: 4.23 -> 4.10,
        // 4.19 -> 3.99; 2-38 elements, K = 1 / 10: 6.9-7.4 -> 5.8-5.9 /
        // 4.0-4.2 -> 3.8-3.9); rods the one-warp kernels take (<= 63
        // elements) only for epochs shorter than kSpecMinSteps, where those
        // do not run
        const int cta_np = h->h_tasks[g.task_begin].np;
        const bool cta_ok = g.tier == TIER_CTA && g.ncta <= 2 && h->halo_cta != 0 &&
                            (h->halo_cta == 1 || cta_np >= h->halo_short);
        const bool one_cta = g.tier == TIER_CTA && h->halo_cta != 1 && cta_np < kHaloCtaMinPoints;
        g.h_short = one_cta && g.rw;
        if ((g.tier != TIER_CLUSTER && g.tier != TIER_GRID && !cta_ok) || g.uni != 2 || !h->halo_on ||
            d.has_self || d.force_ctas > 0 || d.force_variant >= 0)
            continue;
        const CtaTask& tf = h->h_tasks[g.task_begin];
        const CtaTask& tl = h->h_tasks[g.task_begin + g.ncta - 1];
        const int64_t p0 = tf.p0, p1 = int64_t(tl.p0) + tl.np;
        const int64_t r0 = rod_of(d, p0), r1 = rod_of(d, p1 - 1);
        const int nr = int(r1 - r0 + 1);
        if (nr > 2 || d.rod_offsets[r0] != p0 || d.rod_offsets[r1 + 1] != p1) continue;
        const int64_t np = d.rod_offsets[r0 + 1] - d.rod_offsets[r0];
        if (nr == 2 && d.rod_offsets[r1 + 1] - d.rod_offsets[r1] != np) continue;
        bool ok = true, gen = false;
        for (int64_t r = r0; r <= r1 && ok; ++r) {
            const int64_t o = d.rod_offsets[r];
            const int64_t ne = np - 1;
            for (int64_t j = 0; j < np && ok; ++j) {
                const uint32_t f = pflags[size_t(o + j)];
                const uint32_t want = (j < ne ? uint32_t(SF_HAS_ELEM) : 0u) | (j > 0 ? uint32_t(SF_HAS_PREV) : 0u) |
                                      (j < ne - 1 ? uint32_t(SF_JVALID) : 0u) |
                                      (j > 0 && j < ne ? uint32_t(SF_JPREV) : 0u) |
                                      (j < ne && (j & 1) ? uint32_t(SF_PARITY) : 0u);
                const uint32_t mask = SF_HAS_ELEM | SF_HAS_PREV | SF_JVALID | SF_JPREV | SF_PARITY;
                ok = (f & mask) == want && pt_elem[size_t(o + j)] == (j < ne ? int32_t(o + j - r) : -1);
                gen |= (f & SF_EXT) != 0;
            }
        }
        // bindings of the segment: across the two rods, same local index, a matching
        bool bind = false;
        std::vector<uint8_t> used;
        for (int64_t k = 0; k < d.nbind && ok; ++k) {
            const int64_t a = d.bind_a[k], b = d.bind_b[k];
            const bool ina = a >= p0 && a < p1, inb = b >= p0 && b < p1;
            if (!ina && !inb) continue;
            const int64_t ra = rod_of(d, a), rb = rod_of(d, b);
            if (nr != 2 || ra == rb || a - d.rod_offsets[ra] != b - d.rod_offsets[rb]) {
                ok = false;
                break;
            }
            if (used.empty()) used.assign(size_t(p1 - p0), 0);
            if (used[size_t(a - p0)] || used[size_t(b - p0)]) {
                ok = false;
                break;
            }
            used[size_t(a - p0)] = used[size_t(b - p0)] = 1;
            bind = true;
        }
        if (!ok) continue;
        // ghost width: the step's dependency radius (scatter 1, gather 1,
        // one per colour phase; without distance-projected elements or
        // bindings there are no sweeps)
        const int R1 = (g.any_dist || bind) ? int(2 * d.iters + 1) : 1;
        // Layout candidates, first feasible wins: one cluster of up to 16
        // CTAs while they stay within 256 threads (no spills); else a
        // co-resident grid of CTAs of ~halo_width threads (more, thinner
        // CTAs: a phase's issue per SM is what bounds its latency); else a
        // cluster of up to 512-thread CTAs.  Steps per exchange S: the grid's
        // exchange (an L2 round trip, 1-4 us) is amortised over up to
        // kHaloGridSteps steps while the ghosts stay within ~96 points
        // (cfg4 N = 16384, S = 1 / 2 / 3: 11.1 / 8.5 / 7.3 us per step; N = 8192:
        // 9.8 / 7.5 / 7.1); a cluster barrier is worth wider ghosts only when
        // they are one point per step (no colour sweeps: cfg2 3.80 -> 3.67 us
        // at S = 2).  Live launches: one cluster, an exchange every step.
        auto layout = [&](int c, int G, std::vector<HaloTask>& ts, int& wmax) {
            ts.clear();
            wmax = 0;
            const int64_t base = np / c, rem = np % c;
            int64_t o = 0;
            for (int k = 0; k < c; ++k) {
                const int64_t sz = base + (k < rem ? 1 : 0);
                HaloTask t{};
                t.o0 = int32_t(o);
                t.o1 = int32_t(o + sz);
                t.x0 = int32_t(std::max<int64_t>(0, o - G));
                t.x1 = int32_t(std::min<int64_t>(np, o + sz + G));
                wmax = std::max(wmax, int(t.x1 - t.x0));
                ts.push_back(t);
                o += sz;
            }
        };
        struct Cand {
            bool gx;
            int S, G, C, threads, wmax;
            std::vector<HaloTask> ts;
        };
        auto make_cand = [&](bool cgx, int s_cap) -> Cand {
            Cand c{};
            c.gx = cgx;
            c.S = h->live ? 1 : h->halo_steps > 0 ? h->halo_steps
                              : cgx ? std::max(1, std::min({kHaloGridSteps, 96 / R1, s_cap})) : (R1 == 1 ? 2 : 1);
            c.G = c.S * R1;
            int C;
            if (!cgx) {
                C = h->halo_ctas > 0 ? h->halo_ctas : (one_cta ? 1 : kMaxCluster);
                C = std::min(C, kMaxCluster);
            } else {
                // (wider CTAs once the grid passes ~96 CTAs: cfg4 N = 16384 at
                // 128 / 192 / 256 threads: 10.7 / 9.7 / 9.5 us per step)
                int width = h->halo_width;
                auto ctas_for = [&](int wdt) {
                    const int m_t = std::max(c.G, wdt / nr - 2 * c.G);
                    return int((np + m_t - 1) / m_t);
                };
                while (h->halo_ctas <= 0 && ctas_for(width) > 96 && width < 256) width += 32;
                C = h->halo_ctas > 0 ? h->halo_ctas : ctas_for(width);
                C = std::min(C, h->num_sms > 0 ? h->num_sms : 148);
            }
            // (one CTA holds the whole rod: no ghosts, any length)
            c.C = one_cta && !cgx ? 1 : int(std::min<int64_t>(C, np / c.G));
            if (c.C < 1) {
                c.threads = 1 << 30;
                return c;
            }
            layout(c.C, c.G, c.ts, c.wmax);
            c.threads = (nr * c.wmax + 31) / 32 * 32;
            return c;
        };
        // the grid candidate: the longest exchange period whose CTAs fit 512 threads
        auto grid_cand = [&]() -> Cand {
            Cand gr = make_cand(true, kHaloGridSteps);
            for (int sc = gr.S - 1; sc >= 1 && gr.threads > 512; --sc) gr = make_cand(true, sc);
            return gr;
        };
        std::vector<Cand> cands;
        if (h->halo_grid == 1 && !h->live) {
            cands.push_back(grid_cand());
        } else if (h->halo_grid == 0 || h->live) {
            cands.push_back(make_cand(false, 1));
        } else {
            Cand cl = make_cand(false, 1);
            if (cl.threads <= 256) {
                cands.push_back(cl);
            } else {
                Cand gr = grid_cand();
                if (gr.threads < cl.threads) cands.push_back(gr);   // (thinner CTAs than the cluster's)
                cands.push_back(cl);
                cands.push_back(gr);
            }
        }
        const Cand* pick = nullptr;
        for (const Cand& c : cands)
            if (c.threads <= 512 && (c.gx ? c.C >= 2 : c.C <= kMaxCluster)) {
                pick = &c;
                break;
            }
        if (!pick) continue;
        const bool gx = pick->gx;
        const int S = pick->S, G = pick->G, C = pick->C, threads = pick->threads, wmax = pick->wmax;
        const std::vector<HaloTask>& ts = pick->ts;
        g.h_tasks = ts;
        g.h_gx = gx;
        g.h_cta = C;
        g.h_w = wmax;
        g.h_threads = threads;
        g.h_tb = threads > 256 ? 512 : 256;
        g.h_g = G;
        g.h_s = S;
        g.h_iters = int(d.iters);
        g.h_nr = nr;
        g.h_np = int(np);
        g.h_gen = gen;
        g.h_bind = bind;
        for (int r = 0; r < 2; ++r) {
            const int64_t rr = std::min<int64_t>(r0 + r, r1);
            g.h_poff[r] = int32_t(d.rod_offsets[rr]);
            g.h_eoff[r] = int32_t(d.rod_offsets[rr] - rr);
        }
        if (bind)
            for (int64_t k = 0; k < d.nbind; ++k) {
                const int64_t a = d.bind_a[k], b = d.bind_b[k];
                if (a < p0 || a >= p1) continue;
                const int32_t mode = d.bind_mode[k] != 0 ? 2 : 0;
                h->h_hbind[size_t(a)] = 1 | mode;
                h->h_hbind[size_t(b)] = mode;
            }
        if (h->dry) {
            g.halo = true;
            continue;
        }
        int occ = 0;
        int rc = halo_query(h, g, &occ);
        if (rc) return rc;
        if (occ < 1 || (gx && int64_t(occ) * h->num_sms < C)) continue;
        CK(cudaMalloc(&g.d_hfail, sizeof(int64_t)));
        CK(cudaMemset(g.d_hfail, 0, sizeof(int64_t)));
        if (gx) {
            CK(cudaMalloc(&g.d_hflags, sizeof(int32_t) * size_t(C + 2)));
            const size_t words = size_t(2) * C * 2 * nr * G * HL_NSTATE;
            CK(cudaMalloc(&g.d_hhalo, h->rsz * words));
        }
        CK(cudaMalloc(&g.d_htask, sizeof(HaloTask) * ts.size()));
        CK(cudaMemcpy(g.d_htask, ts.data(), sizeof(HaloTask) * ts.size(), cudaMemcpyHostToDevice));
        g.halo = true;
    }
    return RS_OK;
}

int plan(rs_handle h, std::vector<uint32_t>& pflags, std::vector<int32_t>& pt_elem) {
    const rs_world_desc& d = h->d;
    const int64_t P = d.P, R = d.R;
    if (P >= (int64_t(1) << 31)) return fail(RS_E_INVALID, "too many points for int32 indexing");

    // -- per-point flags and element map (validates the flat layout) ------
    pflags.assign(P, 0u);
    pt_elem.assign(P, -1);
    for (int64_t r = 0; r < R; ++r) {
        const int64_t o = d.rod_offsets[r], np = d.rod_offsets[r + 1] - o;
        if (np < 2) return fail(RS_E_INVALID, "rod %lld has fewer than two points", (long long)r);
        for (int64_t i = 0; i < np; ++i) {
            const int64_t p = o + i;
            uint32_t f = 0;
            if (d.plock[p]) f |= SF_PLOCK;
            if (i > 0) f |= SF_HAS_PREV;
            if (i < np - 1) {
                const int64_t e = p - r;
                f |= SF_HAS_ELEM;
                pt_elem[p] = int32_t(e);
                if (d.elem_point[e] != p)
                    return fail(RS_E_INVALID, "elem_point[%lld] != %lld: non-standard layout",
                                (long long)e, (long long)p);
                if (d.jvalid[e]) {
                    if (i >= np - 2)
                        return fail(RS_E_INVALID, "junction_valid[%lld] set at a rod end", (long long)e);
                    f |= SF_JVALID;
                }
                if (e > 0 && d.jvalid[e - 1]) {
                    if (i == 0)
                        return fail(RS_E_INVALID, "junction_valid[%lld] crosses rods", (long long)(e - 1));
                    f |= SF_JPREV;
                }
                if (d.flock[e]) f |= SF_FLOCK;
                if (d.ext[e] != 0.0) f |= SF_EXT;
                else f |= SF_DIST;
                const int64_t par = d.elem_parity[e];
                if (par != 0 && par != 1)
                    return fail(RS_E_INVALID, "elem_parity[%lld] must be 0 or 1", (long long)e);
                if (par) f |= SF_PARITY;
            }
            pflags[p] = f;
        }
    }

    // -- segments: rods coupled by bindings must share a CTA / cluster ------
    std::vector<int> lo(R), hi(R);
    std::iota(lo.begin(), lo.end(), 0);
    std::iota(hi.begin(), hi.end(), 0);
    std::vector<int64_t> rodA(d.nbind), rodB(d.nbind);
    for (int64_t k = 0; k < d.nbind; ++k) {
        const int64_t a = d.bind_a[k], b = d.bind_b[k];
        if (a < 0 || a >= P || b < 0 || b >= P)
            return fail(RS_E_INVALID, "binding %lld endpoint out of range", (long long)k);
        rodA[k] = rod_of(d, a);
        rodB[k] = rod_of(d, b);
    }
    // reach[r] = furthest rod that must share a segment with r
    std::vector<int> reach(R);
    std::iota(reach.begin(), reach.end(), 0);
    if (d.has_self) reach[0] = int(R - 1);   // pairs may couple any two points
    for (int64_t k = 0; k < d.nbind; ++k) {
        const int a = int(std::min(rodA[k], rodB[k])), b = int(std::max(rodA[k], rodB[k]));
        reach[a] = std::max(reach[a], b);
    }
    std::vector<Segment> segs;
    for (int r = 0; r < R;) {
        int end = reach[r];
        for (int x = r; x <= end; ++x) end = std::max(end, reach[x]);
        segs.push_back({r, end, d.rod_offsets[r], d.rod_offsets[end + 1]});
        r = end + 1;
    }

    // the paired stream variants take colour p from slot parity p: every
    // rod's element colours must alternate from its first element
    bool colours_aligned = true;
    for (int64_t r = 0; r < R && colours_aligned; ++r)
        for (int64_t p = d.rod_offsets[r]; p < d.rod_offsets[r + 1] - 1; ++p)
            if (((pflags[p] & SF_PARITY) != 0) != (((p - d.rod_offsets[r]) & 1) != 0)) {
                colours_aligned = false;
                break;
            }

    // -- choose tiers --------------------------------------------------------
    // (self-colliding scenes: any one CTA -- the pair list couples arbitrary
    // points -- up to the largest variant)
    const int cta_cap = (d.force_tier == TIER_CTA || d.has_self) ? kVariants[kNumCapVariants - 1].cover() + 1
                                                                 : kCtaMaxPoints;
    const int clu_cap = kVariants[kNumCapVariants - 1].cover();
    std::vector<int> seg_tier(segs.size());
    std::vector<char> seg_halo_only(segs.size(), 0);
    int64_t max_cta_seg = 0;
    for (size_t i = 0; i < segs.size(); ++i) {
        const int64_t np = segs[i].p1 - segs[i].p0;
        int cap_i = cta_cap;
        if (d.force_tier < 0 && !d.has_self && !d.has_mesh && segs.size() <= size_t(kFewSegments) &&
            segs[i].r0 == segs[i].r1) {
            bool dist = false;
            for (int64_t p = segs[i].p0; p < segs[i].p1 && !dist; ++p) dist = (pflags[p] & SF_DIST) != 0;
            if (!dist) cap_i = kCtaMaxPointsNoDist;
        }
        int tier = np <= cap_i ? TIER_CTA : (np <= int64_t(kMaxCluster) * clu_cap ? TIER_CLUSTER : TIER_GRID);
        if (d.force_tier >= 0) tier = d.force_tier;
        if (d.has_self && tier != TIER_CTA)
            return fail(RS_E_UNSUPPORTED, "self-collision scenes must fit one CTA (%d points, have %lld)", cta_cap,
                        (long long)np);
        if (tier == TIER_CTA && np > cta_cap)
            return fail(RS_E_INVALID, "segment of %lld points does not fit one CTA", (long long)np);
        // coupled rods past one cluster: the wide-halo kernel's grid exchange
        // only (the general grid tier cannot bind across CTAs)
        if (tier == TIER_GRID && segs[i].r0 != segs[i].r1) {
            if (!h->halo_on || d.force_tier >= 0)
                return fail(RS_E_UNSUPPORTED, "coupled rods larger than a %d-CTA cluster", kMaxCluster);
            seg_halo_only[i] = 1;
        }
        seg_tier[i] = tier;
        if (tier == TIER_CTA) max_cta_seg = std::max(max_cta_seg, np);
    }

    for (Group& g : h->groups) {
        if (g.d_flags) cudaFree(g.d_flags);
        if (g.d_halo) cudaFree(g.d_halo);
        if (g.d_htask) cudaFree(g.d_htask);
        if (g.d_hflags) cudaFree(g.d_hflags);
        if (g.d_hhalo) cudaFree(g.d_hhalo);
        if (g.d_hfail) cudaFree(g.d_hfail);
    }
    h->h_tasks.clear();
    h->h_binds.clear();
    h->h_drvs.clear();
    h->groups.clear();

    // point -> (task, slot) for bindings and drivers
    std::vector<int32_t> task_of(P, -1);

    auto new_task = [&](int64_t p0, int64_t np) {
        CtaTask t{};
        t.p0 = int32_t(p0);
        t.np = int32_t(np);
        t.e_uni = -1;
        t.e0 = pt_elem[p0];
        int nrods = 0;   // rods lying entirely inside the range
        for (int64_t p = p0; p < p0 + np; ++p) {
            task_of[p] = int32_t(h->h_tasks.size());
            if (!(pflags[p] & SF_HAS_PREV) && p + 1 < p0 + np) {
                const int64_t r = rod_of(d, p);
                if (d.rod_offsets[r + 1] <= p0 + np) ++nrods;
            }
        }
        t.nrods = nrods;
        h->h_tasks.push_back(t);
    };

    // CTA tier: pack consecutive CTA-tier segments into CTAs
    if (max_cta_seg > 0) {
        int v = 0;
        while (kVariants[v].cover() + 1 < max_cta_seg) ++v;
        // the scene-feature kernels (contacts, self-collision, live) carry
        // the CTA variants 0-2 and 4
        if (v == 3 && (h->contacts_on || d.has_self || d.live)) v = 4;
        // batches of short rods: one rod per 64-thread CTA, 5 CTAs per SM
        int64_t cta_points = 0;
        for (size_t i = 0; i < segs.size(); ++i)
            if (seg_tier[i] == TIER_CTA) cta_points += segs[i].p1 - segs[i].p0;
        if (max_cta_seg <= kVariants[kBatchVariant].cover() + 1 &&
            cta_points >= int64_t(2) * kVariants[kBatchVariant].CAP * h->num_sms)
            v = colours_aligned ? kBatchVariant : 5;
        if (d.force_variant >= 0) {
            if (d.force_variant >= kNumVariants || kVariants[d.force_variant].cover() + 1 < max_cta_seg)
                return fail(RS_E_INVALID, "force_variant %d cannot hold %lld points", d.force_variant,
                            (long long)max_cta_seg);
            v = d.force_variant;
        }
        Group g;
        g.tier = TIER_CTA;
        g.variant = v;
        g.task_begin = int(h->h_tasks.size());
        // packed tasks end at a rod end, so the tail slot is usable
        const int cap = std::min(kVariants[v].CAP, kVariants[v].cover() + 1);
        int64_t cur0 = -1, cur1 = -1;
        for (size_t i = 0; i < segs.size(); ++i) {
            if (seg_tier[i] != TIER_CTA) {
                if (cur0 >= 0) new_task(cur0, cur1 - cur0);
                cur0 = -1;
                continue;
            }
            const int64_t np = segs[i].p1 - segs[i].p0;
            if (cur0 >= 0 && (cur1 - cur0) + np <= cap) {
                cur1 = segs[i].p1;
            } else {
                if (cur0 >= 0) new_task(cur0, cur1 - cur0);
                cur0 = segs[i].p0;
                cur1 = segs[i].p1;
            }
        }
        if (cur0 >= 0) new_task(cur0, cur1 - cur0);
        g.ncta = int(h->h_tasks.size()) - g.task_begin;
        h->groups.push_back(g);
    }
    // cluster / grid tiers: one launch per segment
    for (size_t i = 0; i < segs.size(); ++i) {
        if (seg_tier[i] == TIER_CTA) continue;
        const int64_t np = segs[i].p1 - segs[i].p0;
        Group g;
        g.tier = seg_tier[i];
        g.variant = 4;
        if (g.tier == TIER_CLUSTER)
            for (int v : kClusterVariants)
                if ((np + kVariants[v].cover() - 1) / kVariants[v].cover() <= kMaxCluster) {
                    g.variant = v;
                    break;
                }
        if (d.force_variant >= 0 && d.force_variant <= 4 && d.force_variant != 3 &&
            (g.tier == TIER_CLUSTER || d.force_variant == 2 || d.force_variant == 4))
            g.variant = d.force_variant;
        const int cap = kVariants[g.variant].cover();
        int c = int((np + cap - 1) / cap);
        if (d.force_ctas > 0) c = std::max(c, int(d.force_ctas));
        c = int(std::min<int64_t>(c, np));
        if (g.tier == TIER_CLUSTER && c > kMaxCluster)
            return fail(RS_E_UNSUPPORTED, "rod needs %d CTAs, more than a %d-CTA cluster", c, kMaxCluster);
        if (c < 1) c = 1;
        g.task_begin = int(h->h_tasks.size());
        // balanced split, sizes differ by at most one (partition.py:39-51)
        const int64_t base = np / c, rem = np % c;
        int64_t p = segs[i].p0;
        for (int k = 0; k < c; ++k) {
            const int64_t sz = base + (k < rem ? 1 : 0);
            new_task(p, sz);
            p += sz;
        }
        g.ncta = c;
        g.cluster = g.tier == TIER_CLUSTER ? c : 1;
        g.halo_only = seg_halo_only[i] != 0;
        h->groups.push_back(g);
    }

    // -- bindings ------------------------------------------------------------
    // group the binding list by segment, keeping the reference order
    std::vector<int> seg_of_rod(R);
    for (size_t i = 0; i < segs.size(); ++i)
        for (int r = segs[i].r0; r <= segs[i].r1; ++r) seg_of_rod[r] = int(i);
    std::vector<std::vector<int64_t>> seg_binds(segs.size());
    for (int64_t k = 0; k < d.nbind; ++k) seg_binds[seg_of_rod[rodA[k]]].push_back(k);
    std::vector<std::vector<BindEntry>> per_task(h->h_tasks.size());
    std::vector<int> task_seq(h->h_tasks.size(), 0);
    std::vector<uint8_t> used(P, 0);
    for (size_t i = 0; i < segs.size(); ++i) {
        if (seg_binds[i].empty()) continue;
        bool matching = true;
        for (int64_t k : seg_binds[i]) {
            const int64_t a = d.bind_a[k], b = d.bind_b[k];
            if (used[a] || used[b] || a == b) matching = false;
            used[a] = used[b] = 1;
        }
        for (int64_t k : seg_binds[i]) used[d.bind_a[k]] = used[d.bind_b[k]] = 0;
        const int ta = task_of[segs[i].p0];
        const Group* gp = nullptr;
        for (const Group& g : h->groups)
            if (ta >= g.task_begin && ta < g.task_begin + g.ncta) gp = &g;
        for (int64_t k : seg_binds[i]) {
            const int64_t a = d.bind_a[k], b = d.bind_b[k];
            const int tka = task_of[a], tkb = task_of[b];
            BindEntry be{};
            be.a_rank = gp->tier == TIER_CLUSTER ? tka - gp->task_begin : 0;
            be.b_rank = gp->tier == TIER_CLUSTER ? tkb - gp->task_begin : 0;
            be.a_slot = int32_t(a - h->h_tasks[tka].p0);
            be.b_slot = int32_t(b - h->h_tasks[tkb].p0);
            be.mode = int32_t(d.bind_mode[k]);
            if (gp->tier == TIER_CTA && tka != tkb)
                return fail(RS_E_INVALID, "internal: binding split across CTAs");
            // parallel: the CTA owning `a` applies it; sequential: rank 0
            const int owner = matching ? tka : (gp->tier == TIER_CLUSTER ? gp->task_begin : tka);
            per_task[owner].push_back(be);
            if (!matching) task_seq[owner] = 1;
        }
    }
    for (size_t t = 0; t < h->h_tasks.size(); ++t) {
        h->h_tasks[t].bind_begin = int32_t(h->h_binds.size());
        h->h_tasks[t].bind_count = int32_t(per_task[t].size());
        h->h_tasks[t].bind_seq = task_seq[t];
        h->h_binds.insert(h->h_binds.end(), per_task[t].begin(), per_task[t].end());
    }

    // -- drivers (rod order; the last rod driving a point wins) -------------
    std::vector<std::vector<DrvEntry>> per_drv(h->h_tasks.size());
    auto add_drv = [&](int64_t p, int kind, int64_t r) -> int {
        if (p < 0) return RS_OK;
        if (p >= P) return fail(RS_E_INVALID, "driver index out of range");
        int64_t slot_p = p;
        if (kind == 1) {   // frame e lives in the slot of its lower point
            if (p >= d.E) return fail(RS_E_INVALID, "driven frame out of range");
            slot_p = d.elem_point[p];
        }
        const int t = task_of[slot_p];
        const int slot = int(slot_p - h->h_tasks[t].p0);
        auto& v = per_drv[t];
        const uint32_t bit = kind == 0 ? SF_DRV_PT : SF_DRV_FR;
        const int shift = kind == 0 ? SF_DRV_PT_SHIFT : SF_DRV_FR_SHIFT;
        if (pflags[slot_p] & bit) {   // already driven: later rod overrides
            const int idx = int((pflags[slot_p] >> shift) & 0xffu);
            v[idx].rod = int32_t(r);
            return RS_OK;
        }
        if (int(v.size()) >= MAX_DRV_PER_CTA) return fail(RS_E_UNSUPPORTED, "too many drivers in one CTA");
        DrvEntry e{};
        e.slot = slot;
        e.kind = kind;
        e.rod = int32_t(r);
        pflags[slot_p] |= bit | (uint32_t(v.size()) << shift);
        v.push_back(e);
        return RS_OK;
    };
    for (int64_t r = 0; r < R; ++r) {
        int rc = add_drv(d.drv_pt[r], 0, r);
        if (rc) return rc;
        rc = add_drv(d.drv_fr[r], 1, r);
        if (rc) return rc;
    }
    for (size_t t = 0; t < h->h_tasks.size(); ++t) {
        h->h_tasks[t].drv_begin = int32_t(h->h_drvs.size());
        h->h_tasks[t].drv_count = int32_t(per_drv[t].size());
        h->h_drvs.insert(h->h_drvs.end(), per_drv[t].begin(), per_drv[t].end());
    }

    // -- per-launch uniformity, sizes and occupancy checks -------------------
    for (Group& g : h->groups) {
        const Variant var = kVariants[g.variant];
        bool uni = true, launch_uni = true;   // per CTA / across the whole launch
        int64_t g_e0 = -1;
        int max_np = 0, bcap = 0, dcap = 0;
        for (int t = g.task_begin; t < g.task_begin + g.ncta; ++t) {
            CtaTask& tk = h->h_tasks[t];
            max_np = std::max(max_np, tk.np);
            bcap = std::max(bcap, tk.bind_seq ? 0 : tk.bind_count);
            dcap = std::max(dcap, tk.drv_count);
            int64_t e0 = -1;
            for (int64_t p = tk.p0; p < tk.p0 + tk.np; ++p) {
                if (pt_elem[p] < 0) continue;
                if (e0 < 0) {
                    e0 = pt_elem[p];
                } else if (uni && !elem_consts_equal(d, e0, pt_elem[p])) {
                    uni = false;
                }
            }
            tk.e_uni = int32_t(std::max<int64_t>(e0, 0));
            if (e0 >= 0) {
                if (g_e0 < 0) g_e0 = e0;
                else if (launch_uni && !elem_consts_equal(d, g_e0, e0)) launch_uni = false;
            }
        }
        g.uni = uni ? (launch_uni && g_e0 >= 0 ? 2 : 1) : 0;
        g.any_dist = false;
        for (int t = g.task_begin; t < g.task_begin + g.ncta && !g.any_dist; ++t)
            for (int64_t p = h->h_tasks[t].p0; p < h->h_tasks[t].p0 + h->h_tasks[t].np; ++p)
                if (pflags[p] & SF_DIST) {
                    g.any_dist = true;
                    break;
                }
        g.e_launch = int32_t(std::max<int64_t>(g_e0, 0));
        g.bind_cap = bcap;
        g.drv_cap = std::max(dcap, 1);
        // slots the threads must cover: a task whose last slot is a rod end
        // (no element) leaves it to thread 0 as the tail slot
        int need = 0;
        for (int t = g.task_begin; t < g.task_begin + g.ncta; ++t) {
            const CtaTask& tk = h->h_tasks[t];
            const bool tail_ok = !(pflags[tk.p0 + tk.np - 1] & SF_HAS_ELEM);
            need = std::max(need, tk.np - (tail_ok ? 1 : 0));
        }
        const int maxT = max_threads(var.S, var.CAP);
        g.threads = std::max(32, ((need + var.S - 1) / var.S + 31) / 32 * 32);
        if (g.threads > maxT || max_np > var.CAP || max_np > var.S * g.threads + 1)
            return fail(RS_E_INVALID, "variant %d (S=%d, CAP=%d) cannot hold a %d-point task", g.variant, var.S,
                        var.CAP, max_np);
        // batches of whole single rods with no bindings: persistent stream
        // tier (TMA prefetch of the next rod while the current one steps)
        if (g.tier == TIER_CTA && g.variant >= 5 && d.force_tier < 0 && !h->contacts_on &&
            (colours_aligned || !paired(var.S))) {
            bool single = true;
            for (int t = g.task_begin; t < g.task_begin + g.ncta && single; ++t)
                single = h->h_tasks[t].nrods == 1 && h->h_tasks[t].bind_count == 0;
            if (single) g.tier = TIER_STREAM;
        }
        // warp-per-rod batched kernel: every task one 129-point rod whose
        // flags are the structural ones of a World rod (elements, junctions
        // and colours by local index; no drivers), launch-uniform constants
        if (g.tier == TIER_STREAM && g.variant == kBatchVariant && g.uni == 2 && h->bw_on) {
            bool ok = true;
            for (int t = g.task_begin; t < g.task_begin + g.ncta && ok; ++t) {
                const CtaTask& tk = h->h_tasks[t];
                ok = tk.np == BW_NP && tk.nrods == 1 && tk.drv_count == 0 && tk.bind_count == 0;
                for (int j = 0; j < BW_NP && ok; ++j) {
                    const uint32_t f = pflags[tk.p0 + j];
                    const uint32_t want = (j < BW_NE ? uint32_t(SF_HAS_ELEM) : 0u) | (j > 0 ? uint32_t(SF_HAS_PREV) : 0u) |
                                          (j < BW_NE - 1 ? uint32_t(SF_JVALID) : 0u) |
                                          (j > 0 && j < BW_NE ? uint32_t(SF_JPREV) : 0u) |
                                          (j < BW_NE && (j & 1) ? uint32_t(SF_PARITY) : 0u);
                    const uint32_t mask = SF_HAS_ELEM | SF_HAS_PREV | SF_JVALID | SF_JPREV | SF_PARITY | SF_DRV_PT | SF_DRV_FR;
                    ok = (f & mask) == want && pt_elem[tk.p0 + j] == (j < BW_NE ? tk.e0 + j : -1);
                }
            }
            bool gen = false;   // (external forces are checked at launch: h->has_fext)
            for (int t = g.task_begin; t < g.task_begin + g.ncta && ok && !gen; ++t)
                for (int j = 0; j < BW_NE && !gen; ++j) gen = (pflags[h->h_tasks[t].p0 + j] & SF_EXT) != 0;
            g.bw_gen = gen;
            // rods sharing their mass and inverse-mass arrays bit for bit:
            // the statics live once per CTA (more warps per SM)
            bool shared = ok;
            const int64_t q0 = h->h_tasks[g.task_begin].p0;
            for (int t = g.task_begin + 1; t < g.task_begin + g.ncta && shared; ++t) {
                const int64_t p = h->h_tasks[t].p0;
                shared = std::memcmp(d.mass + p, d.mass + q0, sizeof(double) * BW_NP) == 0 &&
                         std::memcmp(d.invm + p, d.invm + q0, sizeof(double) * BW_NP) == 0;
            }
            int shape = h->bw_shape >= 0 ? h->bw_shape : (shared ? 3 : 1);
            if (kBwShapes[shape].shst && !shared) shape = 1;
            g.bw_shape = ok ? shape : -1;
        }
        // one-warp kernel: every task one rod of <= 64 elements with the
        // structural flags of a World rod, launch-uniform constants
        g.rw = false;
        if (g.tier == TIER_CTA && g.variant == 0 && g.uni == 2 && h->rw_on && !h->contacts_on && !d.has_self &&
            !d.live) {
            bool ok = true;
            for (int t = g.task_begin; t < g.task_begin + g.ncta && ok; ++t) {
                const CtaTask& tk = h->h_tasks[t];
                const int ne = tk.np - 1;
                ok = tk.nrods == 1 && ne >= 1 && ne <= RW_MAX_EL && tk.drv_count == 0 && tk.bind_count == 0;
                for (int j = 0; j <= ne && ok; ++j) {
                    const uint32_t f = pflags[tk.p0 + j];
                    const uint32_t want = (j < ne ? uint32_t(SF_HAS_ELEM) : 0u) | (j > 0 ? uint32_t(SF_HAS_PREV) : 0u) |
                                          (j < ne - 1 ? uint32_t(SF_JVALID) : 0u) |
                                          (j > 0 && j < ne ? uint32_t(SF_JPREV) : 0u) |
                                          (j < ne && (j & 1) ? uint32_t(SF_PARITY) : 0u);
                    const uint32_t mask = SF_HAS_ELEM | SF_HAS_PREV | SF_JVALID | SF_JPREV | SF_PARITY | SF_DRV_PT | SF_DRV_FR;
                    ok = (f & mask) == want && pt_elem[tk.p0 + j] == (j < ne ? tk.e0 + j : -1);
                }
            }
            int ne_min = 1 << 30, ne_max = 0;
            for (int t = g.task_begin; t < g.task_begin + g.ncta; ++t) {
                ne_min = std::min(ne_min, h->h_tasks[t].np - 1);
                ne_max = std::max(ne_max, h->h_tasks[t].np - 1);
            }
            g.rw_form = (ne_max <= RW1_MAX_EL && h->rw1_on) ? 1 : (ne_max <= RW_MAX_EL ? 2 : 0);
            (void)ne_min;
            g.rw = ok && g.rw_form > 0;
            g.rw_gen = false;
            for (int t = g.task_begin; t < g.task_begin + g.ncta && ok && !g.rw_gen; ++t)
                for (int j = 0; j < h->h_tasks[t].np - 1 && !g.rw_gen; ++j)
                    g.rw_gen = (pflags[h->h_tasks[t].p0 + j] & SF_EXT) != 0;
        }
        const bool stream = g.tier == TIER_STREAM && stream_staged(var.S, var.CAP);
        size_t smem = h->prec == RS_F32 ? SmemLayout<float>(var.CAP, g.bind_cap, g.drv_cap, stream).total
                                        : SmemLayout<double>(var.CAP, g.bind_cap, g.drv_cap, stream).total;
        const int stage_cap = BIND_FIELDS * var.CAP / BIND_REALS;
        if ((smem > kMaxSmem || g.bind_cap > stage_cap) && g.bind_cap > 0) {
            // no room to stage binding constants: apply bindings in order
            for (int t = g.task_begin; t < g.task_begin + g.ncta; ++t) {
                CtaTask& tk = h->h_tasks[t];
                if (tk.bind_count == 0) continue;
                if (g.tier == TIER_CLUSTER && t != g.task_begin)
                    return fail(RS_E_UNSUPPORTED, "bindings too many for shared memory in cluster");
                tk.bind_seq = 1;
            }
            g.bind_cap = 0;
            smem = h->prec == RS_F32 ? SmemLayout<float>(var.CAP, 0, g.drv_cap).total
                                     : SmemLayout<double>(var.CAP, 0, g.drv_cap).total;
        }
        if (smem > kMaxSmem) return fail(RS_E_UNSUPPORTED, "shared memory plan %zu B too large", smem);
        g.smem = smem;
        g.grid = g.tier == TIER_STREAM ? std::min(g.ncta, min_blocks(var.S, var.CAP) * h->num_sms) : g.ncta;
        if (h->dry) continue;
        int occ = 0;
        int rc = occupancy_query(h, g.variant, g.tier, launch_cfg(h, g), g.threads, g.smem, g.cluster, &occ);
        if (rc) return rc;
        if (g.tier == TIER_CLUSTER && occ < 1)
            return fail(RS_E_UNSUPPORTED, "a %d-CTA cluster of %zu B smem cannot be resident", g.cluster, g.smem);
        if (g.tier == TIER_GRID && !g.halo_only && int64_t(occ) * h->num_sms < g.ncta)
            return fail(RS_E_UNSUPPORTED, "grid tier needs %d co-resident CTAs, device holds %d", g.ncta,
                        occ * h->num_sms);
        if ((g.tier == TIER_CTA || g.tier == TIER_STREAM) && occ < 1)
            return fail(RS_E_UNSUPPORTED, "CTA plan cannot be resident (%zu B smem, %d threads)", g.smem,
                        g.threads);
        if (g.tier == TIER_STREAM) {
            // persistent CTAs per SM: the occupancy limit, or fewer on request
            // (RSB_STREAM_CTAS, tuning experiments)
            int per_sm = occ;
            if (const char* e = getenv("RSB_STREAM_CTAS")) per_sm = std::max(1, std::min(occ, atoi(e)));
            g.grid = std::min(g.ncta, per_sm * h->num_sms);
        }
        if (g.bw_shape >= 0) {
            int bocc = 0, bocc_gen = 0;   // both kernels: external forces may appear later
            int rcb = batch_occupancy(h, g.bw_shape, &bocc);
            if (!rcb) rcb = batch_occupancy(h, kBwNumShapes + kBwGenShape, &bocc_gen);
            if (rcb) return rcb;
            if (bocc < 1 || bocc_gen < 1) {
                g.bw_shape = -1;
            } else {
                const int wpc = kBwShapes[g.bw_shape].wpc, wpg = kBwShapes[kBwGenShape].wpc;
                g.bw_grid = std::min((g.ncta + wpc - 1) / wpc, bocc * h->num_sms);
                g.bw_grid_gen = std::min((g.ncta + wpg - 1) / wpg, bocc_gen * h->num_sms);
            }
        }
        if (spec_group(g) && !h->dry) {   // the speculative launch's redo list
            int rc2 = dev_alloc(h->redo_list, sizeof(int32_t) * size_t(g.ncta));
            if (!rc2) rc2 = dev_alloc(h->redo_count, sizeof(int32_t));
            if (rc2) return rc2;
        }
        if (g.tier == TIER_GRID) {
            CK(cudaMalloc(&g.d_flags, sizeof(int32_t) * g.ncta));
            CK(cudaMalloc(&g.d_halo, h->rsz * 2 * HALO_WORDS * size_t(g.ncta)));
            CK(cudaMemset(g.d_halo, 0, h->rsz * 2 * HALO_WORDS * size_t(g.ncta)));
        }
    }

    // sorted p0 index for grab placement
    h->task_by_p0.resize(h->h_tasks.size());
    std::iota(h->task_by_p0.begin(), h->task_by_p0.end(), 0);
    std::sort(h->task_by_p0.begin(), h->task_by_p0.end(),
              [&](int a, int b) { return h->h_tasks[a].p0 < h->h_tasks[b].p0; });
    h->task_p0_sorted.resize(h->h_tasks.size());
    for (size_t i = 0; i < h->task_by_p0.size(); ++i) h->task_p0_sorted[i] = h->h_tasks[h->task_by_p0[i]].p0;
    h->task_group.assign(h->h_tasks.size(), 0);
    for (size_t gi = 0; gi < h->groups.size(); ++gi)
        for (int t = h->groups[gi].task_begin; t < h->groups[gi].task_begin + h->groups[gi].ncta; ++t)
            h->task_group[t] = int(gi);
    // one CTA or one cluster: the kernel itself drains staged commands at
    // every step boundary (commands posted while an epoch runs apply at the
    // next step, like the reference's parallel backend)
    h->live = d.live != 0 && h->groups.size() == 1 &&
              ((h->groups[0].tier == TIER_CTA && h->groups[0].ncta == 1 && h->groups[0].variant <= 4 &&
                h->groups[0].variant != 3) ||
               h->groups[0].tier == TIER_CLUSTER);
    int rc_h = plan_halo(h, pflags, pt_elem);
    if (rc_h) return rc_h;
    h->planned = true;
    return RS_OK;
}

int find_task(rs_handle h, int64_t p) {
    auto it = std::upper_bound(h->task_p0_sorted.begin(), h->task_p0_sorted.end(), p);
    const int i = int(it - h->task_p0_sorted.begin()) - 1;
    if (i < 0) return -1;
    const int t = h->task_by_p0[i];
    const CtaTask& tk = h->h_tasks[t];
    return (p >= tk.p0 && p < tk.p0 + tk.np) ? t : -1;
}

// Rebuild the per-CTA grab tables from the World's grab slots.
int build_grabs(rs_handle h) {
    const rs_world_desc& d = h->d;
    std::vector<std::vector<GrabEntry>> per(h->h_tasks.size());
    for (int64_t k = 0; k < d.ngrab; ++k) {
        if (!d.g_act[k]) continue;
        const int64_t p = d.g_pt[k];
        if (p < 0 || p >= d.P) return fail(RS_E_INVALID, "active grab %lld has no point", (long long)k);
        const int t = find_task(h, p);
        if (t < 0) return fail(RS_E_INVALID, "internal: grab point unplaced");
        GrabEntry g{};
        g.slot = int32_t(p - h->h_tasks[t].p0);
        g.world_slot = int32_t(k);
        for (int c = 0; c < 3; ++c) g.tgt[c] = d.g_tgt[3 * k + c];
        if (per[t].size() >= size_t(GRAB_SM)) return fail(RS_E_UNSUPPORTED, "too many grabs in one CTA");
        per[t].push_back(g);
    }
    h->h_grabs.clear();
    for (size_t t = 0; t < h->h_tasks.size(); ++t) {
        h->h_tasks[t].grab_begin = int32_t(h->h_grabs.size());
        h->h_tasks[t].grab_count = int32_t(per[t].size());
        h->h_grabs.insert(h->h_grabs.end(), per[t].begin(), per[t].end());
    }
    int rc = put_vec(h, h->grabs, h->h_grabs);
    if (rc) return rc;
    return put_vec(h, h->tasks, h->h_tasks);
}

// Contact slots: only a mesh, or slots set by hand, make the contact
// machinery do anything (every step resets the accumulators and, on
// detection steps, the slots, _core.pyx:730-741).  Hand-set slots in a world
// without a mesh are seen at bind time / the next RS_STATIC upload.
bool contacts_needed(const rs_world_desc& d) {
    bool on = d.has_mesh != 0;
    for (int64_t i = 0; i < d.P && !on; ++i)
        on = d.cact[i] != 0 || d.cacc_n[i] != 0.0 || d.cacc_t[i] != 0.0 || std::signbit(d.cacc_n[i]) ||
             std::signbit(d.cacc_t[i]);
    return on;
}

// The static arrays' bytes, in a fixed order: what RS_STATIC_IF_CHANGED
// compares against the last static upload (the reference reads these arrays
// live every step, so an in-place edit must take effect at the next epoch).
std::vector<std::pair<const void*, size_t>> static_spans(const rs_world_desc& d) {
    const size_t P = size_t(d.P), E = size_t(d.E), R = size_t(d.R), f = sizeof(double), i = sizeof(int64_t);
    return {{d.rest, E * f},        {d.ustar, 3 * E * f},    {d.mass, P * f},       {d.invm, P * f},
            {d.inert, 3 * E * f},   {d.fext, 3 * P * f},     {d.ks, E * f},         {d.kp, E * f},
            {d.gt, E * f},          {d.gr, E * f},           {d.ext, E * f},        {d.kb, 3 * E * f},
            {d.plock, P},           {d.flock, E},            {d.jvalid, E},         {d.elem_point, E * i},
            {d.elem_parity, E * i}, {d.drv_pt, R * i},       {d.drv_fr, R * i},     {d.bind_a, size_t(d.nbind) * i},
            {d.bind_b, size_t(d.nbind) * i}, {d.bind_mode, size_t(d.nbind) * i}, {d.cradii, P * f},
            {d.cmask, P}};
}

void snapshot_static(rs_handle h) {
    h->static_snap.clear();
    for (auto& sp : static_spans(h->d)) {
        const char* p = static_cast<const char*>(sp.first);
        if (p) h->static_snap.insert(h->static_snap.end(), p, p + sp.second);
    }
}

bool static_changed(rs_handle h) {
    size_t off = 0;
    for (auto& sp : static_spans(h->d)) {
        if (!sp.first) continue;
        if (off + sp.second > h->static_snap.size() ||
            std::memcmp(h->static_snap.data() + off, sp.first, sp.second) != 0)
            return true;
        off += sp.second;
    }
    return off != h->static_snap.size();
}

int upload_static(rs_handle h) {
    const rs_world_desc& d = h->d;
    std::vector<uint32_t> pflags;
    std::vector<int32_t> pt_elem;
    h->contacts_on = contacts_needed(d);
    snapshot_static(h);
    int rc = plan(h, pflags, pt_elem);
    if (rc) return rc;
    const size_t P = size_t(d.P), E = size_t(d.E), R = size_t(d.R);
    if ((rc = put_real(h, h->rest, d.rest, E))) return rc;
    if ((rc = put_real(h, h->ustar, d.ustar, 3 * E))) return rc;
    if ((rc = put_real(h, h->inert, d.inert, 3 * E))) return rc;
    if ((rc = put_real(h, h->ks, d.ks, E))) return rc;
    if ((rc = put_real(h, h->kp, d.kp, E))) return rc;
    if ((rc = put_real(h, h->gt, d.gt, E))) return rc;
    if ((rc = put_real(h, h->gr, d.gr, E))) return rc;
    if ((rc = put_real(h, h->kb, d.kb, 3 * E))) return rc;
    if ((rc = put_real(h, h->mass, d.mass, P))) return rc;
    if ((rc = put_real(h, h->invm, d.invm, P))) return rc;
    h->has_fext = 0;
    for (size_t i = 0; i < 3 * P; ++i)
        if (d.fext[i] != 0.0 || std::signbit(d.fext[i])) {
            h->has_fext = 1;
            break;
        }
    if (h->has_fext) {
        if ((rc = put_real(h, h->fext, d.fext, 3 * P))) return rc;
    } else if ((rc = dev_alloc(h->fext, h->rsz))) {
        return rc;
    }
    (void)R;
    if ((rc = put_vec(h, h->pflags, pflags))) return rc;
    if ((rc = put_vec(h, h->pt_elem, pt_elem))) return rc;
    if (d.has_mesh) {   // make_context's tree binding (_core.pyx:301-315)
        if (d.mesh_depth + 1 > CONTACT_STACK)
            return fail(RS_E_RUNTIME, "tree deeper than the traversal stack capacity");
        if (d.n_nodes < 1 || d.n_tris < 1 || d.n_verts < 1) return fail(RS_E_INVALID, "empty mesh");
        for (int64_t i = 0; i < 3 * d.n_tris; ++i)
            if (d.tris[i] < 0 || d.tris[i] >= d.n_verts) return fail(RS_E_INVALID, "triangle vertex out of range");
        for (int64_t i = 0; i < d.n_nodes; ++i)
            if (d.ncount[i] > 0 && (d.nstart[i] < 0 || d.nstart[i] + d.ncount[i] > d.n_tris))
                return fail(RS_E_INVALID, "tree leaf range out of bounds");
        for (int64_t i = 0; i < d.n_tris; ++i)
            if (d.torder[i] < 0 || d.torder[i] >= d.n_tris) return fail(RS_E_INVALID, "tree order out of range");
        if ((rc = put_real(h, h->nmin, d.nmin, 3 * size_t(d.n_nodes)))) return rc;
        if ((rc = put_real(h, h->nmax, d.nmax, 3 * size_t(d.n_nodes)))) return rc;
        if ((rc = put_real(h, h->verts, d.verts, 3 * size_t(d.n_verts)))) return rc;
        if ((rc = put_i32(h, h->nstart, d.nstart, size_t(d.n_nodes)))) return rc;
        if ((rc = put_i32(h, h->ncount, d.ncount, size_t(d.n_nodes)))) return rc;
        if ((rc = put_i32(h, h->torder, d.torder, size_t(d.n_tris)))) return rc;
        if ((rc = put_i32(h, h->tris, d.tris, 3 * size_t(d.n_tris)))) return rc;
    }
    if (d.coll_interval < 1) return fail(RS_E_INVALID, "collision_interval must be >= 1");
    if (d.has_self) {
        if (d.n_groups < 1 || d.pair_cap < 1) return fail(RS_E_INVALID, "self-collision needs groups and pair buffers");
        for (int64_t g = 0; g < d.n_groups; ++g)
            if (d.grp_s[g] < 0 || d.grp_e[g] > d.P || d.grp_s[g] >= d.grp_e[g])
                return fail(RS_E_INVALID, "self-collision group %lld out of range", (long long)g);
        if ((rc = put_i32(h, h->grp_rod, d.grp_rod, size_t(d.n_groups)))) return rc;
        if ((rc = put_i32(h, h->grp_gi, d.grp_gi, size_t(d.n_groups)))) return rc;
        if ((rc = put_i32(h, h->grp_s, d.grp_s, size_t(d.n_groups)))) return rc;
        if ((rc = put_i32(h, h->grp_e, d.grp_e, size_t(d.n_groups)))) return rc;
        if ((rc = dev_alloc(h->grp_c, h->rsz * 3 * size_t(d.n_groups)))) return rc;
        const size_t ngp = size_t(d.n_groups) * size_t(d.n_groups - 1) / 2;
        // (per-thread pair counts of the broad phase's scan: one CTA)
        if ((rc = dev_alloc(h->gp_count, sizeof(int32_t) * std::max<size_t>(ngp, 1024)))) return rc;
    }

    if ((rc = put_real(h, h->cradii, d.cradii, P))) return rc;
    if ((rc = put_u8(h, h->cmask, d.cmask, P))) return rc;
    if ((rc = put_vec(h, h->binds, h->h_binds))) return rc;
    if ((rc = put_vec(h, h->drvs, h->h_drvs))) return rc;
    if ((rc = put_vec(h, h->hdrv, h->h_hdrv))) return rc;
    if ((rc = put_vec(h, h->hbind, h->h_hbind))) return rc;
    return build_grabs(h);
}

// Driver velocities/rotations and grab slots, re-sent only when they differ
// from the last upload (they are read every epoch, like the reference's live
// reads of the World arrays, but rarely change between epochs).
int upload_control(rs_handle h) {
    const rs_world_desc& d = h->d;
    const size_t R = size_t(d.R), G = size_t(d.ngrab);
    auto same = [](const auto& v, const auto* p, size_t n) {
        return v.size() == n && (n == 0 || std::memcmp(v.data(), p, n * sizeof(*p)) == 0);
    };
    // drivers and grabs separately: a haptic frame changes a driver velocity
    // (two asynchronous copies); the grab slots and tables (copies through
    // temporaries, with synchronisations) only when a grab changed
    const bool valid = h->ctl_valid && h->planned;
    const bool drv_same = valid && same(h->ctl_drv_v, d.drv_v, 3 * R) && same(h->ctl_drv_rot, d.drv_rot, R);
    const bool grab_same = valid && same(h->ctl_g_act, d.g_act, G) && same(h->ctl_g_pt, d.g_pt, G) &&
                           same(h->ctl_g_tgt, d.g_tgt, 3 * G);
    if (drv_same && grab_same) return RS_OK;
    int rc = RS_OK;
    if (!drv_same) {
        h->ctl_drv_v.assign(d.drv_v, d.drv_v + 3 * R);
        h->ctl_drv_rot.assign(d.drv_rot, d.drv_rot + R);
        if ((rc = put_real(h, h->drv_v, d.drv_v, 3 * size_t(d.R)))) return rc;
        if ((rc = put_real(h, h->drv_rot, d.drv_rot, size_t(d.R)))) return rc;
    }
    h->ctl_valid = h->planned;
    if (grab_same) return RS_OK;
    h->ctl_g_act.assign(d.g_act, d.g_act + G);
    h->ctl_g_pt.assign(d.g_pt, d.g_pt + G);
    h->ctl_g_tgt.assign(d.g_tgt, d.g_tgt + 3 * G);
    {   // the world's grab slots, as the live kernel drains commands into them
        std::vector<int64_t> act(G);
        for (size_t g = 0; g < G; ++g) act[g] = d.g_act[g];
        if ((rc = put_i32(h, h->g_act_d, act.data(), G))) return rc;
        if ((rc = put_i32(h, h->g_pt_d, d.g_pt, G))) return rc;
        if ((rc = put_real(h, h->g_tgt_d, d.g_tgt, 3 * G))) return rc;
    }
    if (!h->planned) return RS_OK;
    return build_grabs(h);
}

int upload_state(rs_handle h) {
    const rs_world_desc& d = h->d;
    const size_t P = size_t(d.P), E = size_t(d.E);
    int rc = RS_OK;
    if (h->rsz == sizeof(double) && d.pos && d.vel && d.q && d.w) {
        if ((rc = dev_alloc(h->pos, 8 * 3 * std::max<size_t>(P, 1))) || (rc = dev_alloc(h->vel, 8 * 3 * std::max<size_t>(P, 1))) ||
            (rc = dev_alloc(h->q, 8 * 4 * std::max<size_t>(E, 1))) || (rc = dev_alloc(h->w, 8 * 3 * std::max<size_t>(E, 1))))
            return rc;
        CopyBatch b;
        b.add(h->pos.p, d.pos, 8 * 3 * P);
        b.add(h->vel.p, d.vel, 8 * 3 * P);
        b.add(h->q.p, d.q, 8 * 4 * E);
        b.add(h->w.p, d.w, 8 * 3 * E);
        if ((rc = flush_batch(h, b))) return rc;
    } else {
        if ((rc = put_real(h, h->pos, d.pos, 3 * P))) return rc;
        if ((rc = put_real(h, h->vel, d.vel, 3 * P))) return rc;
        if ((rc = put_real(h, h->q, d.q, 4 * E))) return rc;
        if ((rc = put_real(h, h->w, d.w, 3 * E))) return rc;
    }
    if (d.has_self) {
        if ((rc = put_i32(h, h->pair_a, d.pair_a, size_t(d.pair_cap)))) return rc;
        if ((rc = put_i32(h, h->pair_b, d.pair_b, size_t(d.pair_cap)))) return rc;
        if ((rc = put_real(h, h->pair_md, d.pair_md, size_t(d.pair_cap)))) return rc;
        if ((rc = put_real(h, h->pair_acc, d.pair_acc, size_t(d.pair_cap)))) return rc;
    }
    if (!h->contacts_on) return RS_OK;
    if ((rc = put_u8(h, h->cact, d.cact, P))) return rc;
    if ((rc = put_real(h, h->cnorm, d.cnorm, 3 * P))) return rc;
    if ((rc = put_real(h, h->cdepth, d.cdepth, P))) return rc;
    if ((rc = put_real(h, h->cacc_n, d.cacc_n, P))) return rc;
    return put_real(h, h->cacc_t, d.cacc_t, P);
}

// Apply staged commands at the step boundary (ph_boundary, _core.pyx:477-506)
// -- the host's drain, for launches that are not live.
void drain_ring(rs_handle h) {
    std::lock_guard<std::mutex> lk(h->ring_mu);
    rs_world_desc& d = h->d;
    volatile LiveRing* R = h->ring;
    while (R->head < R->tail) {
        const int slot = int(R->head % RING_CAP);
        double r[6];
        for (int k = 0; k < 6; ++k) r[k] = R->rows[slot][k];
        const int op = int(r[0]);
        const int64_t i0 = int64_t(r[1]), i1 = int64_t(r[2]);
        if (op == 0 && i0 >= 0 && i0 < d.R) {
            for (int k = 0; k < 3; ++k) d.drv_v[3 * i0 + k] = r[3 + k];
        } else if (op == 1 && i0 >= 0 && i0 < d.R) {
            d.drv_rot[i0] = r[3];
        } else if (op == 2 && i0 >= 0 && i0 < d.ngrab) {
            d.g_pt[i0] = i1;
            for (int k = 0; k < 3; ++k) d.g_tgt[3 * i0 + k] = r[3 + k];
            d.g_act[i0] = 1;
        } else if (op == 3 && i0 >= 0 && i0 < d.ngrab) {
            d.g_act[i0] = 0;
            d.g_pt[i0] = -1;
        }
        R->apply[slot] = h->step;
        R->head = R->head + 1;
        h->control_dirty = true;
    }
}

template <typename Real>
StepArgs<Real> make_args(rs_handle h, const Group& g, int64_t step0, int steps) {
    StepArgs<Real> a{};
    a.pos = static_cast<Real*>(h->pos.p);
    a.vel = static_cast<Real*>(h->vel.p);
    a.q = static_cast<Real*>(h->q.p);
    a.w = static_cast<Real*>(h->w.p);
    a.rest = static_cast<const Real*>(h->rest.p);
    a.ustar = static_cast<const Real*>(h->ustar.p);
    a.inert = static_cast<const Real*>(h->inert.p);
    a.ks = static_cast<const Real*>(h->ks.p);
    a.kp = static_cast<const Real*>(h->kp.p);
    a.gt = static_cast<const Real*>(h->gt.p);
    a.gr = static_cast<const Real*>(h->gr.p);
    a.kb = static_cast<const Real*>(h->kb.p);
    a.mass = static_cast<const Real*>(h->mass.p);
    a.invm = static_cast<const Real*>(h->invm.p);
    a.fext = static_cast<const Real*>(h->fext.p);
    a.drv_v = static_cast<const Real*>(h->drv_v.p);
    a.drv_rot = static_cast<const Real*>(h->drv_rot.p);
    a.pflags = static_cast<const uint32_t*>(h->pflags.p);
    a.pt_elem = static_cast<const int32_t*>(h->pt_elem.p);
    a.tasks = static_cast<const CtaTask*>(h->tasks.p) + g.task_begin;
    a.binds = static_cast<const BindEntry*>(h->binds.p);
    a.grabs = static_cast<const GrabEntry*>(h->grabs.p);
    a.drvs = static_cast<const DrvEntry*>(h->drvs.p);
    a.flags = g.d_flags;
    a.halo = static_cast<Real*>(g.d_halo);
    a.err_step = h->d_err;
    a.step0 = step0;
    a.steps = steps;
    a.iters = int32_t(h->d.iters);
    a.bind_cap = g.bind_cap;
    a.drv_cap = g.drv_cap;
    a.has_fext = h->has_fext;
    a.ncta = g.ncta;
    a.ntasks = g.ncta;
    a.debug = h->debug;
    a.prof = h->d_prof;
    for (int t = g.task_begin; t < g.task_begin + g.ncta; ++t) {
        a.any_binds |= h->h_tasks[t].bind_count > 0;
        a.any_grabs |= h->h_tasks[t].grab_count > 0;
    }
    a.any_dist = g.any_dist;
    if (g.uni == 2) {   // the same arithmetic the kernel's load_elem_consts does
        const int64_t e = g.e_launch;
        const rs_world_desc& d = h->d;
        a.u.l = Real(d.rest[e]);
        a.u.il = Real(1.0) / a.u.l;
        a.u.kpl = Real(d.kp[e]) * a.u.l;
        a.u.ks = Real(d.ks[e]);
        a.u.gt = Real(d.gt[e]);
        a.u.gr = Real(d.gr[e]);
        for (int k = 0; k < 3; ++k) {
            a.u.kb[k] = Real(d.kb[3 * e + k]);
            a.u.us[k] = Real(d.ustar[3 * e + k]);
            a.u.I[k] = Real(d.inert[3 * e + k]);
            a.u.rI[k] = Real(1.0) / a.u.I[k];
        }
    }
    a.contacts_on = h->contacts_on;
    a.has_mesh = int32_t(h->d.has_mesh != 0);
    a.n_nodes = int32_t(h->d.n_nodes);
    a.coll_interval = int32_t(h->d.coll_interval);
    a.nmin = static_cast<const Real*>(h->nmin.p);
    a.nmax = static_cast<const Real*>(h->nmax.p);
    a.verts = static_cast<const Real*>(h->verts.p);
    a.nstart = static_cast<const int32_t*>(h->nstart.p);
    a.ncount = static_cast<const int32_t*>(h->ncount.p);
    a.torder = static_cast<const int32_t*>(h->torder.p);
    a.tris = static_cast<const int32_t*>(h->tris.p);
    a.cradii = static_cast<const Real*>(h->cradii.p);
    a.cmask = static_cast<const uint8_t*>(h->cmask.p);
    a.cact = static_cast<uint8_t*>(h->cact.p);
    a.cnorm = static_cast<Real*>(h->cnorm.p);
    a.cdepth = static_cast<Real*>(h->cdepth.p);
    a.cacc_n = static_cast<Real*>(h->cacc_n.p);
    a.cacc_t = static_cast<Real*>(h->cacc_t.p);
    a.contacts = h->d_contacts;
    a.has_self = int32_t(h->d.has_self != 0);
    a.n_groups = int32_t(h->d.n_groups);
    a.excl = int32_t(h->d.excl);
    a.pair_cap = int32_t(std::min<int64_t>(h->d.pair_cap, INT32_MAX));
    a.grp_rod = static_cast<const int32_t*>(h->grp_rod.p);
    a.grp_gi = static_cast<const int32_t*>(h->grp_gi.p);
    a.grp_s = static_cast<const int32_t*>(h->grp_s.p);
    a.grp_e = static_cast<const int32_t*>(h->grp_e.p);
    a.grp_c = static_cast<Real*>(h->grp_c.p);
    a.gp_count = static_cast<int32_t*>(h->gp_count.p);
    a.pair_a = static_cast<int32_t*>(h->pair_a.p);
    a.pair_b = static_cast<int32_t*>(h->pair_b.p);
    a.pair_md = static_cast<Real*>(h->pair_md.p);
    a.pair_acc = static_cast<Real*>(h->pair_acc.p);
    a.pair_count = h->d_pairs;
    a.live = h->live ? h->ring_dev : nullptr;
    a.snap = (h->live && h->snap_on) ? h->snap_dev : nullptr;
    a.snap_pos = h->snap_pos_dev;
    a.snap_q = h->snap_q_dev;
    a.snap_base = h->snap_version;
    a.snap_P = h->d.P;
    a.snap_E = h->d.E;
    a.drv_v_live = static_cast<Real*>(h->drv_v.p);
    a.drv_rot_live = static_cast<Real*>(h->drv_rot.p);
    a.g_act = static_cast<int32_t*>(h->g_act_d.p);
    a.g_pt = static_cast<int32_t*>(h->g_pt_d.p);
    a.g_tgt = static_cast<Real*>(h->g_tgt_d.p);
    a.ngrab = int32_t(h->d.ngrab);
    a.nrods = int32_t(h->d.R);
    a.touch = Real(h->d.touch);
    a.broad = Real(h->d.broad);
    a.coll_margin = Real(h->d.coll_margin);
    a.restitution = Real(h->d.restitution);
    a.mu = Real(h->d.mu);
    a.dt = Real(h->d.dt);
    a.beta = Real(h->d.beta);
    a.gx = Real(h->d.gx);
    a.gy = Real(h->d.gy);
    a.gz = Real(h->d.gz);
    a.bar_cycles = h->bar_timing ? h->d_bar : nullptr;
    a.htask = g.d_htask;
    a.hdrv = static_cast<const int32_t*>(h->hdrv.p);
    a.hbind = static_cast<const int32_t*>(h->hbind.p);
    a.h_nr = g.h_nr;
    a.h_np = g.h_np;
    a.h_w = g.h_w;
    a.h_g = g.h_g;
    a.h_s = g.h_s;
    a.hfail = g.d_hfail;
    for (int r = 0; r < 2; ++r) {
        a.h_poff[r] = g.h_poff[r];
        a.h_eoff[r] = g.h_eoff[r];
    }
    return a;
}

int halo_query(rs_handle h, const Group& g, int* out) {
    cudaError_t e;
    const int gen = g.h_gen ? 1 : 0, bind = g.h_bind ? 1 : 0;
    if (h->prec == RS_F64_MIRROR)
        e = mirror::halo_step<double>(1, gen, bind, g.h_tb, g.h_gx, 1, nullptr, g.h_cta, g.h_threads, nullptr, out);
    else if (h->prec == RS_F32)
        e = f32::halo_step<float>(1, gen, bind, g.h_tb, g.h_gx, 1, nullptr, g.h_cta, g.h_threads, nullptr, out);
    else
        e = f64fast::halo_step<double>(1, gen, bind, g.h_tb, g.h_gx, 1, nullptr, g.h_cta, g.h_threads, nullptr, out);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *out = 0;   // not launchable here: the group keeps the general kernel
    }
    return RS_OK;
}

// Launch one group, or (t_cnt >= 0, CTA/stream tiers only) the task
// sub-range [t_off, t_off + t_cnt) of it: tasks of those tiers are
// independent, so a sub-range is a complete launch of its own.
int launch_group(rs_handle h, const Group& g, int64_t step0, int steps, int t_off = 0, int t_cnt = -1,
                 bool exact = false) {
    if (g.tier == TIER_GRID) CK(cudaMemsetAsync(g.d_flags, 0, sizeof(int32_t) * g.ncta, h->st));
    const int nt = t_cnt < 0 ? g.ncta : t_cnt;
    const int grid_full = t_cnt < 0 ? g.grid : (g.tier == TIER_STREAM ? std::min(g.grid, nt) : nt);
    const int cfg0 = launch_cfg(h, g);
    // batched rods (stream tier, variant 7): a speculative launch whose
    // quotients never take the IEEE fallback, then the exact kernel over the
    // rods it listed (almost always none: the exact launch finds an empty
    // list and returns)
    // (one-CTA rods only for long epochs: the exact launch over the redo
    // list costs a few microseconds, a whole K = 1 step on a short rod)
    // (a single one-warp rod: lazy launches, below)
    bool lazy_rw = !exact && h->rw_lazy && h->spec && g.rw && g.d_hfail && g.tier == TIER_CTA && g.ncta == 1 &&
                   t_cnt < 0 && cfg0 < 3 && h->h_grabs.empty() && !h->live;
    if (lazy_rw && g.lazy_skip > 0) {
        --g.lazy_skip;
        lazy_rw = false;
    }
    bool spec = !exact && !lazy_rw && h->spec && spec_group(g) && cfg0 < 3 && h->redo_count.p &&
                (g.tier != TIER_CTA || steps >= kSpecMinSteps);
    const int gi = int(&g - h->groups.data());
    const bool backoff = g.tier == TIER_CTA && gi >= 0 && gi < int(h->groups.size());
    if (spec && backoff) {
        const size_t ng = h->groups.size();
        if (h->spec_streak.size() != ng) {
            h->spec_streak.assign(ng, 0);
            h->spec_skip.assign(ng, 0);
            for (cudaEvent_t e : h->redo_ev)
                if (e) cudaEventDestroy(e);
            h->redo_ev.assign(ng, nullptr);
            h->redo_ev_live.assign(ng, 0);
            if (h->h_redo) cudaFreeHost(h->h_redo);
            h->h_redo = nullptr;
            CK(cudaMallocHost(&h->h_redo, sizeof(int32_t) * ng));
        }
        // the previous speculative launch's redo count, if it has arrived
        if (h->redo_ev_live[gi] && cudaEventQuery(h->redo_ev[gi]) == cudaSuccess) {
            h->redo_ev_live[gi] = 0;
            h->spec_streak[gi] = h->h_redo[gi] > 0 ? h->spec_streak[gi] + 1 : 0;
            if (h->spec_streak[gi] >= 3) {
                h->spec_streak[gi] = 0;
                h->spec_skip[gi] = kSpecBackoff;
            }
        }
        if (h->spec_skip[gi] > 0) {
            --h->spec_skip[gi];
            spec = false;
        }
    }
    h->last_spec = spec;
    if (spec) CK(cudaMemsetAsync(h->redo_count.p, 0, sizeof(int32_t), h->st));
    auto one = [&](int cfg, int redo_mode) -> cudaError_t {
        // the stream tier's consume launch walks the redo list (almost
        // always empty) with one CTA per SM, not the full persistent grid
        const int grid = (redo_mode == 1 && g.tier == TIER_STREAM) ? std::min(grid_full, std::max(h->num_sms, 1))
                                                                    : grid_full;
        auto finish = [&](auto& a) {
            a.tasks += t_off;
            a.ntasks = nt;
            if (spec) {
                a.redo_list = static_cast<int32_t*>(h->redo_list.p);
                a.redo_count = static_cast<int32_t*>(h->redo_count.p);
                a.redo_mode = redo_mode;
            }
        };
        const bool feat = cfg >= 3 && cfg < 6;
        if (h->prec == RS_F64_MIRROR) {
            auto a = make_args<double>(h, g, step0, steps);
            finish(a);
            return feat ? mirror_feat::launch_step<double>(g.variant, g.tier, cfg, a, grid, g.threads, g.smem, g.cluster, h->st)
                        : mirror::launch_step<double>(g.variant, g.tier, cfg, a, grid, g.threads, g.smem, g.cluster, h->st);
        } else if (h->prec == RS_F32) {
            auto a = make_args<float>(h, g, step0, steps);
            finish(a);
            return feat ? f32_feat::launch_step<float>(g.variant, g.tier, cfg, a, grid, g.threads, g.smem, g.cluster, h->st)
                        : f32::launch_step<float>(g.variant, g.tier, cfg, a, grid, g.threads, g.smem, g.cluster, h->st);
        }
        auto a = make_args<double>(h, g, step0, steps);
        finish(a);
        return feat ? f64fast_feat::launch_step<double>(g.variant, g.tier, cfg, a, grid, g.threads, g.smem, g.cluster, h->st)
                    : f64fast::launch_step<double>(g.variant, g.tier, cfg, a, grid, g.threads, g.smem, g.cluster, h->st);
    };
    // the warp-per-rod kernel takes the speculative launch of an eligible
    // group when no grab is active (grab anchors run on the general kernel)
    const bool bw = spec && g.bw_shape >= 0 && h->h_grabs.empty();
    auto one_bw = [&]() -> cudaError_t {
        const bool gen = g.bw_gen || h->has_fext;
        const int bsel = gen ? kBwNumShapes + kBwGenShape : g.bw_shape;
        const int wpc = kBwShapes[gen ? kBwGenShape : g.bw_shape].wpc;
        const int full = gen ? g.bw_grid_gen : g.bw_grid;
        const int bgrid = t_cnt < 0 ? full : std::min(full, (nt + wpc - 1) / wpc);
        auto go = [&](auto a) {
            a.tasks += t_off;
            a.ntasks = nt;
            a.redo_list = static_cast<int32_t*>(h->redo_list.p);
            a.redo_count = static_cast<int32_t*>(h->redo_count.p);
            a.redo_mode = 0;
            return a;
        };
        if (h->prec == RS_F64_MIRROR) {
            auto a = go(make_args<double>(h, g, step0, steps));
            return mirror::batch_step<double>(0, bsel, &a, bgrid, h->st, nullptr);
        } else if (h->prec == RS_F32) {
            auto a = go(make_args<float>(h, g, step0, steps));
            return f32::batch_step<float>(0, bsel, &a, bgrid, h->st, nullptr);
        }
        auto a = go(make_args<double>(h, g, step0, steps));
        return f64fast::batch_step<double>(0, bsel, &a, bgrid, h->st, nullptr);
    };
    const bool rw = spec && g.rw && h->h_grabs.empty() && !h->live;
    auto one_rw = [&]() -> cudaError_t {
        const int gen = (h->has_fext || g.rw_gen) ? 1 : 0;
        auto go = [&](auto a) {
            a.tasks += t_off;
            a.ntasks = nt;
            a.redo_list = static_cast<int32_t*>(h->redo_list.p);
            a.redo_count = static_cast<int32_t*>(h->redo_count.p);
            a.redo_mode = 0;
            return a;
        };
        if (h->prec == RS_F64_MIRROR) {
            auto a = go(make_args<double>(h, g, step0, steps));
            return mirror::warp_step<double>(gen, g.rw_form, &a, nt, h->st);
        } else if (h->prec == RS_F32) {
            auto a = go(make_args<float>(h, g, step0, steps));
            return f32::warp_step<float>(gen, g.rw_form, &a, nt, h->st);
        }
        auto a = go(make_args<double>(h, g, step0, steps));
        return f64fast::warp_step<double>(gen, g.rw_form, &a, nt, h->st);
    };
    // A single rod on a one-warp kernel (<= 63 elements) at any epoch length:
    // launched lazily like the wide-halo kernel -- a failed vote writes
    // nothing back and leaves the launch's first step in the group's redo
    // word, later launches return at once, and the host replays the exact
    // kernel at its next synchronisation -- so no consume launch follows it
    // (which had kept these kernels off epochs shorter than kSpecMinSteps).
    // A group that needed a replay runs without speculation for a while.
    if (lazy_rw) {
        const int gen = (h->has_fext || g.rw_gen) ? 1 : 0;
        auto go = [&](auto a) {
            a.ntasks = 1;
            a.redo_mode = 2;
            return a;
        };
        cudaError_t el;
        if (h->prec == RS_F64_MIRROR) {
            auto a = go(make_args<double>(h, g, step0, steps));
            el = mirror::warp_step<double>(gen, g.rw_form, &a, 1, h->st);
        } else if (h->prec == RS_F32) {
            auto a = go(make_args<float>(h, g, step0, steps));
            el = f32::warp_step<float>(gen, g.rw_form, &a, 1, h->st);
        } else {
            auto a = go(make_args<double>(h, g, step0, steps));
            el = f64fast::warp_step<double>(gen, g.rw_form, &a, 1, h->st);
        }
        if (el != cudaSuccess)
            return fail(RS_E_CUDA, "one-warp launch failed: %s", cudaGetErrorString(el));
        h->halo_pending = true;
        h->last_halo = true;
        h->last_spec = false;
        h->launches += 1;
        return RS_OK;
    }
    // the wide-halo kernel takes the launch of an eligible group (no grabs,
    // not live, ghost width still covering the iterations); a failed vote is
    // replayed exactly by resolve_halo at the next synchronisation
    const bool halo = !exact && g.halo && h->halo_on && (!g.h_short || steps < kSpecMinSteps) &&
                      (g.h_g == g.h_s || g.h_s * (2 * h->d.iters + 1) <= g.h_g) && t_cnt < 0;
    if (halo) {
        if (g.h_gx) CK(cudaMemsetAsync(g.d_hflags, 0, sizeof(int32_t) * size_t(g.h_cta + 2), h->st));
        const int gen = (g.h_gen || h->has_fext) ? 1 : 0, bind = g.h_bind ? 1 : 0;
        // grabs, live launches, barrier accounting: the XF kernels
        const int xf = (!h->h_grabs.empty() || h->live || h->bar_timing || h->contacts_on) ? 1 : 0;
        // the halo launch's own exchange buffers
        auto hx = [&](auto a) {
            a.flags = g.d_hflags;
            a.halo = static_cast<decltype(a.halo)>(g.d_hhalo);
            return a;
        };
        cudaError_t eh;
        if (h->prec == RS_F64_MIRROR) {
            auto a = hx(make_args<double>(h, g, step0, steps));
            eh = mirror::halo_step<double>(0, gen, bind, g.h_tb, g.h_gx, xf, &a, g.h_cta, g.h_threads, h->st, nullptr);
        } else if (h->prec == RS_F32) {
            auto a = hx(make_args<float>(h, g, step0, steps));
            eh = f32::halo_step<float>(0, gen, bind, g.h_tb, g.h_gx, xf, &a, g.h_cta, g.h_threads, h->st, nullptr);
        } else {
            auto a = hx(make_args<double>(h, g, step0, steps));
            eh = f64fast::halo_step<double>(0, gen, bind, g.h_tb, g.h_gx, xf, &a, g.h_cta, g.h_threads, h->st, nullptr);
        }
        if (eh != cudaSuccess)
            return fail(RS_E_CUDA, "wide-halo launch (%d CTAs x %d threads) failed: %s", g.h_cta, g.h_threads,
                        cudaGetErrorString(eh));
        h->halo_pending = true;
        h->last_halo = true;
        h->last_spec = false;
        h->launches += 1;
        return RS_OK;
    }
    h->last_halo = false;
    if (g.halo_only)
        return fail(RS_E_UNSUPPORTED, exact ? "wide-halo launch failed (degenerate geometry or non-finite forces) on "
                                              "coupled rods past one cluster: no exact fallback"
                                            : "coupled rods past one cluster need the wide-halo kernel (RSB_HALO, "
                                              "iterations beyond the planned ghost width)");
    cudaError_t e = bw ? one_bw() : rw ? one_rw() : (spec ? one(cfg0 + 6, 0) : one(cfg0, 0));
    if (e == cudaSuccess && spec) e = one(cfg0, 1);
    if (e == cudaSuccess && spec && backoff && !h->redo_ev_live[gi]) {
        if (!h->redo_ev[gi]) CK(cudaEventCreateWithFlags(&h->redo_ev[gi], cudaEventDisableTiming));
        CK(cudaMemcpyAsync(h->h_redo + gi, h->redo_count.p, sizeof(int32_t), cudaMemcpyDeviceToHost, h->st));
        CK(cudaEventRecord(h->redo_ev[gi], h->st));
        h->redo_ev_live[gi] = 1;
    }
    if (e != cudaSuccess)
        return fail(RS_E_CUDA, "kernel launch (tier %d variant %d, %d CTAs x %d threads, %zu B smem) failed: %s",
                    g.tier, g.variant, g.ncta, g.threads, g.smem, cudaGetErrorString(e));
    h->launches += spec ? 2 : 1;
    return RS_OK;
}

// Wide-halo launches whose cluster vote failed wrote nothing back and left
// their first step in the group's redo word (later launches of the group
// returned at once): replay the exact general kernel from that step to the
// current one.  Called before anything reads or replaces the device state
// or changes what a replay would compute (synchronisation, download, upload,
// staged commands, parameters).
// The groups' redo words come back to pinned host memory with one
// asynchronous copy each (enqueue_halo_check), read after a synchronisation
// the caller does anyway (finish_halo_check): a download costs no extra
// round trip in the common case.
int enqueue_halo_check(rs_handle h) {
    if (!h->halo_pending || h->halo_check_enqueued) return RS_OK;
    const size_t ng = h->groups.size();
    if (h->h_hfail_n < ng) {
        if (h->h_hfail) cudaFreeHost(h->h_hfail);
        h->h_hfail = nullptr;
        CK(cudaMallocHost(&h->h_hfail, sizeof(int64_t) * ng));
        h->h_hfail_n = ng;
    }
    for (size_t gi = 0; gi < ng; ++gi) {
        h->h_hfail[gi] = 0;
        if (h->groups[gi].d_hfail)
            CK(cudaMemcpyAsync(h->h_hfail + gi, h->groups[gi].d_hfail, sizeof(int64_t), cudaMemcpyDeviceToHost,
                               h->st));
    }
    h->halo_check_enqueued = true;
    return RS_OK;
}
// after a synchronisation of h->st: replay failed groups; *replayed: any
int finish_halo_check(rs_handle h, bool* replayed) {
    if (replayed) *replayed = false;
    if (!h->halo_check_enqueued) return RS_OK;
    h->halo_check_enqueued = false;
    h->halo_pending = false;
    int64_t redone = 0;
    for (size_t gi = 0; gi < h->groups.size(); ++gi) {
        const Group& g = h->groups[gi];
        const int64_t v = h->h_hfail[gi];
        if (!g.d_hfail || !v) continue;
        CK(cudaMemsetAsync(g.d_hfail, 0, sizeof(int64_t), h->st));
        if (g.rw) g.lazy_skip = kSpecBackoff;   // (a rod that fails keeps failing: planar noise)
        const bool lh = h->last_halo;
        for (int64_t s0 = v - 1; s0 < h->step;) {
            const int k = int(std::min<int64_t>(h->step - s0, kMaxStepsPerLaunch));
            int rc = launch_group(h, g, s0, k, 0, -1, true);
            if (rc) return rc;
            s0 += k;
        }
        h->last_halo = lh;
        ++redone;
    }
    h->halo_redone = redone;
    if (replayed) *replayed = redone > 0;
    return RS_OK;
}
int resolve_halo(rs_handle h) {
    if (!h->halo_pending) return RS_OK;
    int rc = enqueue_halo_check(h);
    if (rc) return rc;
    CK(cudaStreamSynchronize(h->st));
    return finish_halo_check(h, nullptr);
}

// page-locked (async copies, no staging) and mapped: the device alias lets
// one kernel move a small world's state (xfer_kernel) instead of a copy
// command per array
double* register_host(rs_handle h, void* p, size_t bytes) {
    if (!p || bytes == 0) return nullptr;
    if (cudaHostRegister(p, bytes, cudaHostRegisterMapped) != cudaSuccess) {
        cudaGetLastError();   // (page-locked without the mapping: copy commands only)
        if (cudaHostRegister(p, bytes, cudaHostRegisterDefault) == cudaSuccess)
            h->registered.push_back(p);
        else
            cudaGetLastError();
        return nullptr;
    }
    h->registered.push_back(p);
    void* dp = nullptr;
    if (cudaHostGetDevicePointer(&dp, p, 0) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return static_cast<double*>(dp);
}

// A small world's state between the World's mapped host arrays and the
// device mirrors in one launch (and, device -> host, the error stamp and the
// groups' redo words into pinned memory, so the host epoch needs a single
// synchronisation).
struct XferArgs {
    const double* src[4];
    double* dst[4];
    int64_t n[4];
    const unsigned long long* wsrc[5];
    unsigned long long* wdst[5];
    int nw;
};
__global__ void xfer_kernel(const XferArgs x) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    const int64_t t0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
#pragma unroll
    for (int a = 0; a < 4; ++a)
        for (int64_t i = t0; i < x.n[a]; i += stride) x.dst[a][i] = x.src[a][i];
    if (t0 < x.nw) *x.wdst[t0] = *x.wsrc[t0];
}

// whether a host epoch of this world can move its state with xfer_kernel
bool xfer_ok(rs_handle h) {
    if (!h->xfer_on || h->rsz != sizeof(double) || h->d.has_self || h->contacts_on || h->live) return false;
    for (double* m : h->map_state)
        if (!m) return false;
    const size_t bytes = 8 * (6 * size_t(h->d.P) + 7 * size_t(h->d.E));
    return bytes <= (size_t(8) << 20) && h->groups.size() <= 4;
}

int launch_xfer(rs_handle h, bool up) {
    const rs_world_desc& d = h->d;
    XferArgs x{};
    double* dev[4] = {static_cast<double*>(h->pos.p), static_cast<double*>(h->vel.p), static_cast<double*>(h->q.p),
                      static_cast<double*>(h->w.p)};
    const int64_t n[4] = {3 * d.P, 3 * d.P, 4 * d.E, 3 * d.E};
    int64_t tot = 0;
    for (int a = 0; a < 4; ++a) {
        x.src[a] = up ? h->map_state[a] : dev[a];
        x.dst[a] = up ? dev[a] : h->map_state[a];
        x.n[a] = n[a];
        tot += n[a];
    }
    if (!up) {   // the error stamp and the groups' redo words ride along
        void* he = nullptr;
        CK(cudaHostGetDevicePointer(&he, h->h_err, 0));
        x.wsrc[x.nw] = h->d_err;
        x.wdst[x.nw++] = static_cast<unsigned long long*>(he);
        if (h->halo_pending) {
            const size_t ng = h->groups.size();
            if (h->h_hfail_n < ng) {
                if (h->h_hfail) cudaFreeHost(h->h_hfail);
                h->h_hfail = nullptr;
                CK(cudaMallocHost(&h->h_hfail, sizeof(int64_t) * ng));
                h->h_hfail_n = ng;
            }
            void* hf = nullptr;
            CK(cudaHostGetDevicePointer(&hf, h->h_hfail, 0));
            for (size_t gi = 0; gi < ng; ++gi) {
                h->h_hfail[gi] = 0;
                if (!h->groups[gi].d_hfail) continue;
                x.wsrc[x.nw] = reinterpret_cast<const unsigned long long*>(h->groups[gi].d_hfail);
                x.wdst[x.nw++] = reinterpret_cast<unsigned long long*>(static_cast<int64_t*>(hf) + gi);
            }
            h->halo_check_enqueued = true;
        }
    }
    const int threads = 256;
    const int grid = int(std::min<int64_t>(std::max<int64_t>((tot + threads * 4 - 1) / (threads * 4), 1),
                                           std::max(h->num_sms, 1)));
    xfer_kernel<<<grid, threads, 0, h->st>>>(x);
    CK(cudaGetLastError());
    return RS_OK;
}

}  // namespace

// ph_boundary at the epoch's first step: staged commands, dirty controls
int epoch_prelude(rs_handle h) {
    // (staged commands or new controls would reach a replay of earlier steps)
    if (h->halo_pending && (h->control_dirty || (h->ring && h->ring->tail != h->ring->head))) {
        int rc = resolve_halo(h);
        if (rc) return rc;
    }
    if (!h->live) drain_ring(h);   // live launches drain in the kernel
    if (h->control_dirty) {
        int rc = upload_control(h);
        if (rc) return rc;
        h->control_dirty = false;
    }
    return RS_OK;
}

// after the epoch's launches (on h->st): error stamp read-back, counters
int epoch_epilogue(rs_handle h, int64_t steps, int64_t* contacts, int64_t* barrier_ns) {
    if (h->timing) CK(cudaEventRecord(h->ev1, h->st));
    h->timed = h->timing;
    // the error stamp (a running maximum on the device) is read back when
    // someone synchronises, not after every launch
    h->err_pending = true;
    h->step += steps;
    h->snap_seq += 2 * steps;
    h->snap_step = h->step;
    if (contacts) {
        *contacts = 0;
        if (h->contacts_on || h->d.has_self) {   // epoch_results: contacts + pairs after the last step
            CK(cudaMemcpyAsync(h->h_contacts, h->d_contacts, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                               h->st));
            CK(cudaStreamSynchronize(h->st));
            *contacts = int64_t(*h->h_contacts);
        }
    }
    if (barrier_ns) {
        *barrier_ns = 0;
        if (h->bar_timing) {   // epoch_results' barrier sum: cycles at the SM clock
            CK(cudaMemcpyAsync(h->h_bar, h->d_bar, sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->st));
            CK(cudaStreamSynchronize(h->st));
            *barrier_ns = int64_t(double(*h->h_bar) * 1e6 / double(std::max(h->clock_khz, 1)));
        }
    }
    return RS_OK;
}


// One epoch with the state coming from and going back to the host arrays,
// the copies of chunk c+1 (H2D) and c-1 (D2H) overlapping the launch on
// chunk c.  Chunks are contiguous task ranges of a single CTA/stream-tier
// group (whole rods, no cross-task coupling), so each chunk's launch is a
// complete step of its rods and the result is identical to the unchunked
// epoch.
int run_epoch_pipelined(rs_handle h, int64_t steps, int64_t* contacts, int64_t* barrier_ns) {
    const Group& g = h->groups[0];
    const rs_world_desc& d = h->d;
    // chunk boundaries: equal chunks in the middle, the first and last ones
    // ramped down (1/8, 1/4, 1/2 of a chunk), so the pipeline's fill (H2D of
    // the first chunk alone) and drain (D2H of the last alone) are short
    std::vector<double> w;
    for (double f : {0.125, 0.25, 0.5}) w.push_back(f);
    for (int i = 0; i < h->pipe_chunks - 6; ++i) w.push_back(1.0);
    for (double f : {0.5, 0.25, 0.125}) w.push_back(f);
    double wsum = 0;
    for (double x : w) wsum += x;
    std::vector<int> cut{0};
    double acc = 0;
    for (double x : w) {
        acc += x;
        const int t = int(std::llround(double(g.ncta) * acc / wsum));
        if (t > cut.back()) cut.push_back(std::min(t, g.ncta));
    }
    if (cut.back() != g.ncta) cut.push_back(g.ncta);
    const int C = int(cut.size()) - 1;
    if (!h->st_in) {
        CK(cudaStreamCreateWithFlags(&h->st_in, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&h->st_out, cudaStreamNonBlocking));
    }
    while (int(h->ev_in.size()) < C + 1) {
        cudaEvent_t a, b;
        CK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
        h->ev_in.push_back(a);
        h->ev_k.push_back(b);
    }
    // everything already queued on the compute stream (control uploads,
    // earlier epochs) precedes this epoch's copies
    CK(cudaEventRecord(h->ev_k[C], h->st));
    CK(cudaStreamWaitEvent(h->st_in, h->ev_k[C], 0));
    if (h->timing) CK(cudaEventRecord(h->ev0, h->st));
    if (h->bar_timing) CK(cudaMemsetAsync(h->d_bar, 0, sizeof(unsigned long long), h->st));
    double* const hp[4] = {d.pos, d.vel, d.q, d.w};
    DevBuf* const dp[4] = {&h->pos, &h->vel, &h->q, &h->w};
    const int width[4] = {3, 3, 4, 3};
    for (int c = 0; c < C; ++c) {
        const int t0 = cut[c], t1 = cut[c + 1];
        const CtaTask& a = h->h_tasks[g.task_begin + t0];
        const CtaTask& b = h->h_tasks[g.task_begin + t1 - 1];
        const int64_t P0 = a.p0, P1 = int64_t(b.p0) + b.np;
        const int64_t E0 = P0 - rod_of(d, P0), E1 = P1 - (rod_of(d, P1 - 1) + 1);
        CopyBatch up;   // the chunk's four state slices, one driver call
        for (int f = 0; f < 4; ++f) {
            const int64_t r0 = f < 2 ? P0 : E0, r1 = f < 2 ? P1 : E1;
            const size_t off = size_t(r0) * width[f], cnt = size_t(r1 - r0) * width[f];
            up.add(static_cast<double*>(dp[f]->p) + off, hp[f] + off, cnt * sizeof(double));
        }
        if (int rc0 = flush_batch(h, up, h->st_in)) return rc0;
        CK(cudaEventRecord(h->ev_in[c], h->st_in));
        CK(cudaStreamWaitEvent(h->st, h->ev_in[c], 0));
        int rc = launch_group(h, g, h->step, int(steps), t0, t1 - t0);
        if (rc) return rc;
        CK(cudaEventRecord(h->ev_k[c], h->st));
        CK(cudaStreamWaitEvent(h->st_out, h->ev_k[c], 0));
        CopyBatch down;
        for (int f = 0; f < 4; ++f) {
            const int64_t r0 = f < 2 ? P0 : E0, r1 = f < 2 ? P1 : E1;
            const size_t off = size_t(r0) * width[f], cnt = size_t(r1 - r0) * width[f];
            down.add(hp[f] + off, static_cast<const double*>(dp[f]->p) + off, cnt * sizeof(double));
        }
        if (int rc1 = flush_batch(h, down, h->st_out)) return rc1;
    }
    int rc = epoch_epilogue(h, steps, contacts, barrier_ns);
    if (rc) return rc;
    CK(cudaStreamSynchronize(h->st_out));
    return rs_synchronize(h);
}

// ---- C ABI --------------------------------------------------------------------

extern "C" {

const char* rs_last_error(void) { return g_err.c_str(); }

int rs_create(const rs_world_desc* desc, rs_handle* out) {
    if (!desc || !out) return fail(RS_E_INVALID, "null argument");
    *out = nullptr;
    if (desc->abi_version != RS_ABI_VERSION) return fail(RS_E_INVALID, "ABI version mismatch");
    if (desc->P < 2 || desc->R < 1 || desc->E != desc->P - desc->R)
        return fail(RS_E_INVALID, "inconsistent world sizes");
    if (desc->dt <= 0.0 || desc->iters < 1) return fail(RS_E_INVALID, "dt must be positive and iters >= 1");
    if (desc->precision < 0 || desc->precision > 2) return fail(RS_E_INVALID, "unknown precision");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (desc->device < 0 || desc->device >= ndev) return fail(RS_E_INVALID, "no CUDA device %d", desc->device);
    CK(cudaSetDevice(desc->device));
    auto h = new rs_handle_s();
    h->d = *desc;
    h->prec = desc->precision;
    h->rsz = h->prec == RS_F32 ? sizeof(float) : sizeof(double);
    h->step = desc->step_index;
    if (const char* dbg = getenv("RSB_DEBUG")) h->debug = atoi(dbg);
    if (const char* sp = getenv("RSB_SPEC")) h->spec = atoi(sp) != 0;
    if (const char* e = getenv("RSB_HALO")) h->halo_on = atoi(e) != 0;
    if (const char* e = getenv("RSB_HALO_CTAS")) h->halo_ctas = atoi(e);
    if (const char* e = getenv("RSB_HALO_GRID")) h->halo_grid = atoi(e);
    if (const char* e = getenv("RSB_HALO_W")) h->halo_width = std::max(64, atoi(e));
    if (const char* e = getenv("RSB_HALO_STEPS")) h->halo_steps = std::max(0, atoi(e));
    if (const char* e = getenv("RSB_XFER")) h->xfer_on = atoi(e) != 0;
    if (const char* e = getenv("RSB_PIPE_CHUNKS")) h->pipe_chunks = std::max(7, std::min(256, atoi(e)));
    if (const char* e = getenv("RSB_RW_LAZY")) h->rw_lazy = atoi(e) != 0;
    if (const char* e = getenv("RSB_HALO_SHORT")) h->halo_short = std::max(2, atoi(e));
    if (const char* e = getenv("RSB_MAX_K")) h->max_k = std::max(1, std::min(kMaxStepsPerLaunch, atoi(e)));
    if (const char* e = getenv("RSB_HALO_CTA")) h->halo_cta = atoi(e);
    if (const char* sp = getenv("RSB_BW")) h->bw_on = atoi(sp) != 0;
    if (const char* sp = getenv("RSB_RW")) h->rw_on = atoi(sp) != 0;
    if (const char* sp = getenv("RSB_RW1")) h->rw1_on = atoi(sp) != 0;
    if (const char* sp = getenv("RSB_BW_SHAPE")) h->bw_shape = std::max(0, std::min(kBwNumShapes - 1, atoi(sp)));
    if (cudaHostAlloc(reinterpret_cast<void**>(&h->ring), sizeof(LiveRing), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->ring_dev), h->ring, 0) != cudaSuccess) {
        cudaGetLastError();
        h->ring = nullptr;
        delete h;
        return fail(RS_E_CUDA, "mapped command ring allocation failed");
    }
    std::memset(h->ring, 0, sizeof(LiveRing));
    for (int i = 0; i < RING_CAP; ++i) h->ring->apply[i] = -1;
    if (desc->live) {   // per-step snapshot buffers of live launches
        const size_t P = size_t(desc->P), E = size_t(desc->E);
        auto mapped = [&](void** hp, void** dp, size_t bytes) {
            return cudaHostAlloc(hp, bytes, cudaHostAllocMapped) == cudaSuccess &&
                   cudaHostGetDevicePointer(dp, *hp, 0) == cudaSuccess;
        };
        if (!mapped(reinterpret_cast<void**>(&h->snap), reinterpret_cast<void**>(&h->snap_dev), sizeof(LiveSnap)) ||
            !mapped(reinterpret_cast<void**>(&h->snap_pos), reinterpret_cast<void**>(&h->snap_pos_dev),
                    2 * 3 * P * sizeof(double)) ||
            !mapped(reinterpret_cast<void**>(&h->snap_q), reinterpret_cast<void**>(&h->snap_q_dev),
                    2 * 4 * E * sizeof(double))) {
            cudaGetLastError();
            rs_destroy(h);
            return fail(RS_E_CUDA, "mapped snapshot allocation failed");
        }
        std::memcpy(h->snap_pos, desc->pos, 3 * P * sizeof(double));   // version 0: the bound state
        std::memcpy(h->snap_q, desc->q, 4 * E * sizeof(double));
        h->snap->pub = 0;
        h->snap->step[0] = h->snap->step[1] = desc->step_index;
    }
    int rc = RS_OK;
    auto bail = [&](int code) {
        rs_destroy(h);
        return code;
    };
    if (cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, desc->device) != cudaSuccess)
        return bail(fail(RS_E_CUDA, "device query failed"));
    if (cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&h->ev0) != cudaSuccess || cudaEventCreate(&h->ev1) != cudaSuccess ||
        cudaEventCreate(&h->tm0) != cudaSuccess || cudaEventCreate(&h->tm1) != cudaSuccess ||
        cudaMalloc(&h->d_err, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMallocHost(&h->h_err, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&h->d_contacts, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&h->d_pairs, sizeof(int32_t)) != cudaSuccess || cudaMemset(h->d_pairs, 0, sizeof(int32_t)) != cudaSuccess ||
        cudaMallocHost(&h->h_contacts, sizeof(unsigned long long)) != cudaSuccess)
        return bail(fail(RS_E_CUDA, "CUDA resource creation failed"));
    *h->h_err = 0;
    if (cudaMemset(h->d_err, 0, sizeof(unsigned long long)) != cudaSuccess)
        return bail(fail(RS_E_CUDA, "memset failed"));
    if ((h->debug & 6) && (cudaMalloc(&h->d_prof, PROF_SLOTS * sizeof(unsigned long long)) != cudaSuccess ||
                           cudaMemset(h->d_prof, 0, PROF_SLOTS * sizeof(unsigned long long)) != cudaSuccess))
        return bail(fail(RS_E_CUDA, "profile buffer allocation failed"));
    if (h->rsz == sizeof(double)) {
        h->map_state[0] = register_host(h, h->d.pos, 3 * sizeof(double) * size_t(h->d.P));
        h->map_state[1] = register_host(h, h->d.vel, 3 * sizeof(double) * size_t(h->d.P));
        h->map_state[2] = register_host(h, h->d.q, 4 * sizeof(double) * size_t(h->d.E));
        h->map_state[3] = register_host(h, h->d.w, 3 * sizeof(double) * size_t(h->d.E));
    }
    if ((rc = upload_control(h))) return bail(rc);
    if ((rc = upload_static(h))) return bail(rc);
    if ((rc = upload_state(h))) return bail(rc);
    if (cudaStreamSynchronize(h->st) != cudaSuccess) return bail(fail(RS_E_CUDA, "sync failed"));
    h->snap_seq = 2;
    h->snap_step = h->step;
    *out = h;
    return RS_OK;
}

// the handle's device current on this thread (cudaSetDevice only when it
// is not: every entry point calls this, one-step launches included)
static cudaError_t use_device(int dev) {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur == dev) return cudaSuccess;
    return cudaSetDevice(dev);
}

int rs_upload(rs_handle h, uint32_t mask) {
    if (!h) return fail(RS_E_INVALID, "null handle");
    CK(use_device(h->d.device));
    if (int rc = resolve_halo(h)) return rc;
    int rc = RS_OK;
    if (mask & RS_CONTROL) {
        if ((rc = upload_control(h))) return rc;
        h->control_dirty = false;
    }
    if ((mask & RS_STATIC) || ((mask & RS_STATIC_IF_CHANGED) && static_changed(h))) {
        CK(cudaStreamSynchronize(h->st));
        if ((rc = upload_static(h))) return rc;
    }
    if (mask & RS_STATE)
        if ((rc = upload_state(h))) return rc;
    return RS_OK;
}

int rs_run_epoch(rs_handle h, int64_t steps, int64_t* contacts, int64_t* barrier_ns) {
    if (!h) return fail(RS_E_INVALID, "null handle");
    if (steps < 1) return fail(RS_E_INVALID, "steps must be >= 1");
    CK(use_device(h->d.device));
    int rc = epoch_prelude(h);
    if (rc) return rc;
    if (h->timing) CK(cudaEventRecord(h->ev0, h->st));
    if (h->bar_timing) CK(cudaMemsetAsync(h->d_bar, 0, sizeof(unsigned long long), h->st));
    int64_t done = 0;
    while (done < steps) {
        const int k = int(std::min<int64_t>(steps - done, h->max_k));
        if (h->contacts_on || h->d.has_self)
            CK(cudaMemsetAsync(h->d_contacts, 0, sizeof(unsigned long long), h->st));
        for (const Group& g : h->groups) {
            int rc = launch_group(h, g, h->step + done, k);
            if (rc) return rc;
        }
        if (h->live && h->snap && h->snap_on) h->snap_version += k;   // one snapshot per step
        done += k;
    }
    h->prof_steps += steps;
    return epoch_epilogue(h, steps, contacts, barrier_ns);
}

int rs_synchronize(rs_handle h) {
    if (!h) return fail(RS_E_INVALID, "null handle");
    CK(use_device(h->d.device));
    if (int rc = resolve_halo(h)) return rc;
    if (h->err_pending) {
        CK(cudaMemcpyAsync(h->h_err, h->d_err, sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->st));
        h->err_pending = false;
    }
    CK(cudaStreamSynchronize(h->st));
    if (*h->h_err) h->err_step = std::max<int64_t>(h->err_step, int64_t(*h->h_err) - 1);
    if (h->timed) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
        h->last_ms = ms;
        h->timed = false;
    }
    return RS_OK;
}

// After a live epoch the device holds the authoritative driver and grab
// slots (commands were applied to them mid-launch): copy them back into the
// World's arrays, which the reference mutates in place.
int download_control(rs_handle h) {
    const rs_world_desc& d = h->d;
    const size_t R = size_t(d.R), G = size_t(d.ngrab);
    int rc = get_real(h, h->drv_v, d.drv_v, 3 * R);
    if (rc) return rc;
    if ((rc = get_real(h, h->drv_rot, d.drv_rot, R))) return rc;
    if ((rc = get_real(h, h->g_tgt_d, d.g_tgt, 3 * G))) return rc;
    std::vector<int32_t> act(G), pt(G);
    if (G) {
        CK(cudaMemcpyAsync(act.data(), h->g_act_d.p, G * sizeof(int32_t), cudaMemcpyDeviceToHost, h->st));
        CK(cudaMemcpyAsync(pt.data(), h->g_pt_d.p, G * sizeof(int32_t), cudaMemcpyDeviceToHost, h->st));
    }
    CK(cudaStreamSynchronize(h->st));
    for (size_t g = 0; g < G; ++g) {
        d.g_act[g] = uint8_t(act[g] != 0);
        d.g_pt[g] = pt[g];
    }
    h->ctl_valid = false;   // re-sync the upload cache with what is now on the host
    return RS_OK;
}

int rs_download(rs_handle h, uint32_t mask) {
    if (!h) return fail(RS_E_INVALID, "null handle");
    CK(use_device(h->d.device));
    // the redo words travel with the state; a replay (rare) downloads again
    if (int rc = enqueue_halo_check(h)) return rc;
    const rs_world_desc& d = h->d;
    int rc = RS_OK;
    if ((mask & (RS_STATE | RS_CONTROL)) && h->live && h->planned)
        if ((rc = download_control(h))) return rc;
    if (mask & RS_STATE) {
        if (h->rsz == sizeof(double)) {
            CopyBatch b;
            if (d.pos) b.add(d.pos, h->pos.p, 8 * 3 * size_t(d.P));
            if (d.vel) b.add(d.vel, h->vel.p, 8 * 3 * size_t(d.P));
            if (d.q) b.add(d.q, h->q.p, 8 * 4 * size_t(d.E));
            if (d.w) b.add(d.w, h->w.p, 8 * 3 * size_t(d.E));
            if ((rc = flush_batch(h, b))) return rc;
        } else {
            if ((rc = get_real(h, h->pos, d.pos, 3 * size_t(d.P)))) return rc;
            if ((rc = get_real(h, h->vel, d.vel, 3 * size_t(d.P)))) return rc;
            if ((rc = get_real(h, h->q, d.q, 4 * size_t(d.E)))) return rc;
            if ((rc = get_real(h, h->w, d.w, 3 * size_t(d.E)))) return rc;
        }
        if (d.has_self) {
            const size_t n = size_t(d.pair_cap);
            std::vector<int32_t> ia(n), ib(n);
            CK(cudaMemcpyAsync(ia.data(), h->pair_a.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, h->st));
            CK(cudaMemcpyAsync(ib.data(), h->pair_b.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, h->st));
            if ((rc = get_real(h, h->pair_md, d.pair_md, n))) return rc;
            if ((rc = get_real(h, h->pair_acc, d.pair_acc, n))) return rc;
            CK(cudaStreamSynchronize(h->st));
            for (size_t i = 0; i < n; ++i) {
                d.pair_a[i] = ia[i];
                d.pair_b[i] = ib[i];
            }
        }
        if (h->contacts_on) {
            const size_t P = size_t(d.P);
            CK(cudaMemcpyAsync(d.cact, h->cact.p, P, cudaMemcpyDeviceToHost, h->st));
            if ((rc = get_real(h, h->cnorm, d.cnorm, 3 * P))) return rc;
            if ((rc = get_real(h, h->cdepth, d.cdepth, P))) return rc;
            if ((rc = get_real(h, h->cacc_n, d.cacc_n, P))) return rc;
            if ((rc = get_real(h, h->cacc_t, d.cacc_t, P))) return rc;
        }
    }
    if (h->halo_check_enqueued) {
        CK(cudaStreamSynchronize(h->st));
        bool replayed = false;
        if ((rc = finish_halo_check(h, &replayed))) return rc;
        if (replayed) return rs_download(h, mask);
    }
    return rs_synchronize(h);
}

int rs_run_epoch_host(rs_handle h, int64_t steps, int64_t* contacts, int64_t* barrier_ns) {
    if (!h) return fail(RS_E_INVALID, "null handle");
    if (steps < 1) return fail(RS_E_INVALID, "steps must be >= 1");
    CK(use_device(h->d.device));
    if (int rc = resolve_halo(h)) return rc;
    const bool pipelined = h->rsz == sizeof(double) && h->groups.size() == 1 && !h->contacts_on &&
                           !h->d.has_mesh && !h->d.has_self &&
                           (h->groups[0].tier == TIER_CTA || h->groups[0].tier == TIER_STREAM) &&
                           h->groups[0].ncta >= 2 && steps <= kMaxStepsPerLaunch &&
                           !(h->groups[0].halo && h->halo_on);   // (a wide-halo launch covers the group)
    if (!pipelined && xfer_ok(h)) {
        // small worlds: state in and out by one kernel each, one synchronisation
        int rc = launch_xfer(h, true);
        if (rc) return rc;
        if ((rc = rs_run_epoch(h, steps, contacts, barrier_ns))) return rc;
        if ((rc = launch_xfer(h, false))) return rc;
        h->err_pending = false;   // (the stamp came back with the state)
        CK(cudaStreamSynchronize(h->st));
        bool replayed = false;
        if ((rc = finish_halo_check(h, &replayed))) return rc;
        if (replayed) {   // exact replay: its error stamp and the state again
            h->err_pending = true;
            return rs_download(h, RS_STATE);
        }
        if (*h->h_err) h->err_step = std::max<int64_t>(h->err_step, int64_t(*h->h_err) - 1);
        if (h->timed) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
            h->last_ms = ms;
            h->timed = false;
        }
        return RS_OK;
    }
    if (!pipelined) {
        int rc = upload_state(h);
        if (rc) return rc;
        if ((rc = rs_run_epoch(h, steps, contacts, barrier_ns))) return rc;
        return rs_download(h, RS_STATE);
    }
    int rc = epoch_prelude(h);
    if (rc) return rc;
    h->launches_pipelined += 1;
    return run_epoch_pipelined(h, steps, contacts, barrier_ns);
}

int64_t rs_error_step(rs_handle h) {
    if (!h) return -1;
    rs_synchronize(h);
    return h->err_step;
}

int64_t rs_step_counter(rs_handle h) { return h ? h->step : -1; }

int rs_update_params(rs_handle h, double dt, int64_t iters) {
    if (!h) return fail(RS_E_INVALID, "null handle");
    if (h->halo_pending) {   // a replay runs with the parameters of its steps
        CK(use_device(h->d.device));
        if (int rc = resolve_halo(h)) return rc;
    }
    if (dt <= 0.0 || iters < 1) return fail(RS_E_INVALID, "dt must be positive and iters >= 1");
    h->d.dt = dt;
    const bool more = iters > h->d.iters;
    h->d.iters = iters;
    // more iterations than a wide-halo group's ghosts cover: plan again (the
    // ghost width is 2I + 1 points per exchanged step)
    bool replan = false;
    if (more && h->planned)
        for (const Group& g : h->groups)
            replan = replan || (g.halo && g.h_g != g.h_s && g.h_s * (2 * iters + 1) > g.h_g);
    if (replan) {
        CK(use_device(h->d.device));
        CK(cudaStreamSynchronize(h->st));
        if (int rc = upload_static(h)) return rc;
    }
    return RS_OK;
}

int rs_barrier_timing(rs_handle h, int on) {
    if (!h) return fail(RS_E_INVALID, "null handle");
    CK(use_device(h->d.device));
    if (on && !h->d_bar) {
        CK(cudaMalloc(&h->d_bar, sizeof(unsigned long long)));
        CK(cudaMallocHost(&h->h_bar, sizeof(unsigned long long)));
        CK(cudaDeviceGetAttribute(&h->clock_khz, cudaDevAttrClockRate, h->d.device));
    }
    h->bar_timing = on != 0;
    return RS_OK;
}

int rs_stage_commands(rs_handle h, const double* ops, int64_t n, int64_t* slots) {
    if (!h || (n > 0 && !ops)) return fail(RS_E_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(h->ring_mu);
    volatile LiveRing* R = h->ring;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t tail = R->tail;
        if (tail - R->head >= RING_CAP) return fail(RS_E_RING_FULL, "command ring full and not draining");
        const int slot = int(tail % RING_CAP);
        R->apply[slot] = -1;
        for (int k = 0; k < 6; ++k) R->rows[slot][k] = ops[6 * i + k];
        if (slots) slots[i] = tail;
        // rows before tail (x86 stores are ordered; the fence keeps the
        // compiler from reordering them)
        std::atomic_thread_fence(std::memory_order_release);
        R->tail = tail + 1;
    }
    return RS_OK;
}

int64_t rs_applied_step_for(rs_handle h, int64_t global_slot) {
    if (!h) return -1;
    volatile LiveRing* R = h->ring;
    if (global_slot < 0 || global_slot >= R->tail || global_slot < R->tail - RING_CAP) return -1;
    return R->apply[global_slot % RING_CAP];
}

int rs_live_snapshots(rs_handle h, int on) {
    if (!h) return fail(RS_E_INVALID, "null handle");
    if (on && !h->snap) return fail(RS_E_INVALID, "per-step snapshots need a live handle (desc.live = 1)");
    if (on && !h->snap_on) {   // the last published buffer must hold the current state
        CK(cudaStreamSynchronize(h->st));
        const int b = int(h->snap_version & 1);
        std::memcpy(h->snap_pos + size_t(b) * 3 * size_t(h->d.P), h->d.pos, sizeof(double) * 3 * size_t(h->d.P));
        std::memcpy(h->snap_q + size_t(b) * 4 * size_t(h->d.E), h->d.q, sizeof(double) * 4 * size_t(h->d.E));
        h->snap->step[b] = h->step;
        h->snap->pub = h->snap_version;
    }
    h->snap_on = on != 0;
    return RS_OK;
}

int rs_read_snapshot(rs_handle h, double* pos, double* q, int64_t* seq, int64_t* step) {
    if (!h) return fail(RS_E_INVALID, "null handle");
    if (h->live && h->snap && h->snap_on) {   // the kernel publishes one per step (ph_publish)
        volatile LiveSnap* S = h->snap;
        for (int tries = 0; tries < (1 << 20); ++tries) {
            const int64_t v1 = S->pub;
            std::atomic_thread_fence(std::memory_order_acquire);
            const int b = int(v1 & 1);
            if (pos) std::memcpy(pos, h->snap_pos + size_t(b) * 3 * size_t(h->d.P), sizeof(double) * 3 * size_t(h->d.P));
            if (q) std::memcpy(q, h->snap_q + size_t(b) * 4 * size_t(h->d.E), sizeof(double) * 4 * size_t(h->d.E));
            const int64_t st = S->step[b];
            std::atomic_thread_fence(std::memory_order_acquire);
            if (S->pub == v1) {
                if (seq) *seq = 2 * v1;
                if (step) *step = st;
                return RS_OK;
            }
        }
        return fail(RS_E_RUNTIME, "snapshot read kept tearing");
    }
    // the host arrays hold the state of the last completed download
    if (pos) std::memcpy(pos, h->d.pos, sizeof(double) * 3 * size_t(h->d.P));
    if (q) std::memcpy(q, h->d.q, sizeof(double) * 4 * size_t(h->d.E));
    if (seq) *seq = h->snap_seq;
    if (step) *step = h->snap_step;
    return RS_OK;
}

void rs_destroy(rs_handle h) {
    if (!h) return;
    use_device(h->d.device);
    if (h->st) cudaStreamSynchronize(h->st);
    for (DevBuf* b : {&h->pos, &h->vel, &h->q, &h->w, &h->rest, &h->ustar, &h->inert, &h->ks, &h->kp, &h->gt,
                      &h->gr, &h->kb, &h->mass, &h->invm, &h->fext, &h->drv_v, &h->drv_rot, &h->pflags,
                      &h->pt_elem, &h->tasks, &h->binds, &h->drvs, &h->grabs, &h->nmin, &h->nmax, &h->verts,
                      &h->nstart, &h->ncount, &h->torder, &h->tris, &h->cradii, &h->cmask, &h->cact, &h->cnorm,
                      &h->cdepth, &h->cacc_n, &h->cacc_t, &h->grp_rod, &h->grp_gi, &h->grp_s, &h->grp_e,
                      &h->grp_c, &h->gp_count, &h->pair_a, &h->pair_b, &h->pair_md, &h->pair_acc, &h->g_act_d, &h->g_pt_d,
                      &h->g_tgt_d, &h->redo_list, &h->redo_count, &h->hdrv, &h->hbind})
        if (b->p) cudaFree(b->p);
    for (Group& g : h->groups) {
        if (g.d_flags) cudaFree(g.d_flags);
        if (g.d_halo) cudaFree(g.d_halo);
        if (g.d_htask) cudaFree(g.d_htask);
        if (g.d_hflags) cudaFree(g.d_hflags);
        if (g.d_hhalo) cudaFree(g.d_hhalo);
        if (g.d_hfail) cudaFree(g.d_hfail);
    }
    for (void* p : h->registered) cudaHostUnregister(p);
    for (cudaEvent_t e : h->redo_ev)
        if (e) cudaEventDestroy(e);
    if (h->h_redo) cudaFreeHost(h->h_redo);
    if (h->h_hfail) cudaFreeHost(h->h_hfail);
    if (h->d_prof && (h->debug & 4)) {   // wide-halo failed checks (RSB_DEBUG bit 2)
        unsigned long long v = 0;
        if (cudaMemcpy(&v, h->d_prof + PROF_SLOTS - 1, sizeof v, cudaMemcpyDeviceToHost) == cudaSuccess)
            fprintf(stderr, "rsb-halo-fail-mask 0x%llx\n", v);
    }
    if (h->d_prof) {   // per-phase profile (RSB_DEBUG=2): cycles per step, CTA 0
        unsigned long long v[PROF_SLOTS];
        if (cudaMemcpy(v, h->d_prof, sizeof v, cudaMemcpyDeviceToHost) == cudaSuccess && h->prof_steps > 0) {
            fprintf(stderr, "rsb-prof steps=%lld cycles/step per phase:", (long long)h->prof_steps);
            double tot = 0;
            for (int i = 0; i < PROF_SLOTS && v[i]; ++i) {
                fprintf(stderr, " %.0f", double(v[i]) / double(h->prof_steps));
                tot += double(v[i]) / double(h->prof_steps);
            }
            fprintf(stderr, " | total %.0f\n", tot);
        }
        cudaFree(h->d_prof);
    }
    if (h->d_err) cudaFree(h->d_err);
    if (h->h_err) cudaFreeHost(h->h_err);
    if (h->d_contacts) cudaFree(h->d_contacts);
    if (h->d_pairs) cudaFree(h->d_pairs);
    if (h->h_contacts) cudaFreeHost(h->h_contacts);
    if (h->d_bar) cudaFree(h->d_bar);
    if (h->h_bar) cudaFreeHost(h->h_bar);
    if (h->stage) cudaFreeHost(h->stage);
    if (h->ring) cudaFreeHost(h->ring);
    if (h->snap) cudaFreeHost(h->snap);
    if (h->snap_pos) cudaFreeHost(h->snap_pos);
    if (h->snap_q) cudaFreeHost(h->snap_q);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    if (h->tm0) cudaEventDestroy(h->tm0);
    if (h->tm1) cudaEventDestroy(h->tm1);
    for (cudaEvent_t e : h->ev_in) cudaEventDestroy(e);
    for (cudaEvent_t e : h->ev_k) cudaEventDestroy(e);
    if (h->st_in) cudaStreamDestroy(h->st_in);
    if (h->st_out) cudaStreamDestroy(h->st_out);
    if (h->st) cudaStreamDestroy(h->st);
    delete h;
}

int rs_enable_timing(rs_handle h, int on) {
    if (!h) return fail(RS_E_INVALID, "null handle");
    h->timing = on != 0;
    return RS_OK;
}

double rs_last_kernel_ms(rs_handle h) {
    if (!h) return -1.0;
    rs_synchronize(h);
    return h->last_ms;
}

int64_t rs_launch_count(rs_handle h) { return h ? h->launches : -1; }

int64_t rs_last_redo_count(rs_handle h) {
    if (!h) return -1;
    if (h->last_halo) {   // wide-halo groups replayed exactly at the last check
        if (use_device(h->d.device) != cudaSuccess || resolve_halo(h) != RS_OK) return -1;
        return h->halo_redone;
    }
    if (!h->redo_count.p || !h->last_spec) return 0;   // the last launch did not speculate
    if (use_device(h->d.device) != cudaSuccess) return -1;
    int32_t n = 0;
    if (cudaMemcpyAsync(&n, h->redo_count.p, sizeof(n), cudaMemcpyDeviceToHost, h->st) != cudaSuccess ||
        cudaStreamSynchronize(h->st) != cudaSuccess)
        return -1;
    return n;
}

int rs_timer_start(rs_handle h) {
    if (!h) return fail(RS_E_INVALID, "null handle");
    CK(cudaEventRecord(h->tm0, h->st));
    return RS_OK;
}

int rs_timer_stop(rs_handle h) {
    if (!h) return fail(RS_E_INVALID, "null handle");
    CK(cudaEventRecord(h->tm1, h->st));
    return RS_OK;
}

double rs_timer_ms(rs_handle h) {
    if (!h) return -1.0;
    if (cudaEventSynchronize(h->tm1) != cudaSuccess) return -1.0;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, h->tm0, h->tm1) != cudaSuccess) return -1.0;
    return ms;
}

int rs_plan_json(rs_handle h, char* buf, int64_t len) {
    if (!h || !buf || len <= 0) return fail(RS_E_INVALID, "bad argument");
    std::string s = "{\"precision\": " + std::to_string(h->prec) + ", \"groups\": [";
    for (size_t i = 0; i < h->groups.size(); ++i) {
        const Group& g = h->groups[i];
        const Variant v = kVariants[g.variant];
        int64_t pts = 0;
        for (int t = g.task_begin; t < g.task_begin + g.ncta; ++t) pts += h->h_tasks[t].np;
        static const char* names[] = {"cta", "cluster", "grid", "stream"};
        // barriers per step, as the kernel issues them (rod_step.cuh): scatter,
        // gather, integrate + per iteration the two colour phases (when any
        // element is distance-projected or bindings are staged) and one each
        // for contacts, self-collision pairs, bindings, grabs
        bool binds = false, grabs = false;
        for (int t = g.task_begin; t < g.task_begin + g.ncta; ++t) {
            binds |= h->h_tasks[t].bind_count > 0;
            grabs |= h->h_tasks[t].grab_count > 0;
        }
        const bool feat_k = g.tier != TIER_STREAM;
        const int per_it = ((g.any_dist || binds) ? 2 : 0) + ((h->contacts_on && feat_k) ? 1 : 0) +
                           ((h->d.has_self && feat_k) ? 1 : 0) + (binds ? 1 : 0) + (grabs ? 1 : 0);
        const int64_t n_sync = 3 + h->d.iters * per_it;
        // the warp-per-rod kernel (rod_batch.cuh) that takes the group's
        // speculative launches: shape (warps per CTA), persistent CTAs
        char bwj[160] = "null";
        if (g.bw_shape >= 0)
            snprintf(bwj, sizeof bwj, "{\"shape\": %d, \"warps_per_cta\": %d, \"grid\": %d, \"shared_statics\": %s, \"general\": %s}",
                     g.bw_shape, kBwShapes[g.bw_shape].wpc, g.bw_grid, kBwShapes[g.bw_shape].shst ? "true" : "false",
                     g.bw_gen ? "true" : "false");
        // the wide-halo cluster kernel (rod_halo.cuh) that takes the
        // group's launches: CTAs, threads, ghost width; one cluster barrier
        // per step, the phases' barriers CTA-local
        char hj[200] = "null";
        if (g.halo)
            snprintf(hj, sizeof hj, "{\"ctas\": %d, \"threads\": %d, \"ghost\": %d, \"rods\": %d, \"bindings\": %s, "
                     "\"exchange\": \"%s\", \"steps_per_exchange\": %d, \"short_epochs_only\": %s}",
                     g.h_cta, g.h_threads, g.h_g, g.h_nr, g.h_bind ? "true" : "false", g.h_gx ? "grid" : "cluster", g.h_s,
                     g.h_short ? "true" : "false");
        char tmp[1200];
        snprintf(tmp, sizeof tmp,
                 "%s{\"tier\": \"%s\", \"variant\": %d, \"slots_per_thread\": %d, \"cap\": %d, "
                 "\"uniform\": %s, \"ctas\": %d, \"grid\": %d, \"threads\": %d, \"cluster\": %d, "
                 "\"smem\": %zu, \"points\": %lld, \"bind_cap\": %d, \"any_dist\": %s, "
                 "\"bindings\": %s, \"grabs\": %s, \"contacts\": %s, \"self_collision\": %s, "
                 "\"sync_per_iteration\": %d, \"sync_per_step\": %lld, \"warp_per_rod\": %s, \"one_warp_rod\": %s, "
                 "\"halo\": %s}",
                 i ? ", " : "", names[g.tier], g.variant, v.S, v.CAP, g.uni == 2 ? "\"launch\"" : (g.uni ? "true" : "false"), g.ncta,
                 g.grid, g.threads, g.cluster, g.smem, (long long)pts, g.bind_cap, g.any_dist ? "true" : "false",
                 binds ? "true" : "false", grabs ? "true" : "false", h->contacts_on ? "true" : "false",
                 h->d.has_self ? "true" : "false", per_it, (long long)n_sync, bwj, g.rw ? (g.rw_form == 1 ? "\"point_per_lane\"" : "\"two_per_lane\"") : "false",
                 (g.halo && h->halo_on) ? hj : "null");
        s += tmp;
    }
    s += std::string("], \"live\": ") + (h->live ? "true" : "false") + "}";
    if (int64_t(s.size()) + 1 > len) return fail(RS_E_INVALID, "buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return RS_OK;
}

int rs_plan_dry(const rs_world_desc* desc, int32_t num_sms, char* buf, int64_t len) {
    if (!desc) return fail(RS_E_INVALID, "null argument");
    if (desc->P < 2 || desc->R < 1 || desc->E != desc->P - desc->R)
        return fail(RS_E_INVALID, "inconsistent world sizes");
    rs_handle_s h;
    h.d = *desc;
    h.prec = desc->precision;
    h.rsz = h.prec == RS_F32 ? sizeof(float) : sizeof(double);
    h.num_sms = num_sms;
    h.dry = true;
    h.contacts_on = contacts_needed(*desc);
    std::vector<uint32_t> pflags;
    std::vector<int32_t> pt_elem;
    int rc = plan(&h, pflags, pt_elem);
    if (rc) return rc;
    return rs_plan_json(&h, buf, len);
}

int rs_device_ptr(rs_handle h, int32_t which, void** out) {
    if (!h || !out) return fail(RS_E_INVALID, "null argument");
    if (h->halo_pending) {   // the buffers must hold every launched step
        CK(use_device(h->d.device));
        if (int rc = resolve_halo(h)) return rc;
    }
    const DevBuf* b[] = {&h->pos, &h->vel, &h->q, &h->w};
    if (which < 0 || which > 3) return fail(RS_E_INVALID, "unknown array");
    *out = b[which]->p;
    return RS_OK;
}

}  // extern "C"

namespace rsb {
namespace micro {   // csrc/rod_micro.cu
cudaError_t div_selftest(const double*, const double*, int64_t, double*, double*);
cudaError_t fn_selftest(int, const double*, int64_t, double*, double*);
cudaError_t pipe_peak(int kind, int blocks, int threads, int iters, float* ms, double* ops);
}  // namespace micro
}  // namespace rsb

extern "C" int rs_pipe_peak(int kind, double* ops_per_s) {
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    float ms = 0.f;
    double ops = 0.0;
    CK(rsb::micro::pipe_peak(kind, sms * 8, 256, 4096, &ms, &ops));
    *ops_per_s = ops / (double(ms) * 1e-3);
    return RS_OK;
}

extern "C" int rs_selftest_fn(int32_t kind, const double* a, int64_t n, double* r_ieee, double* r_fast) {
    if (kind < 0 || kind > 1 || n < 0) return fail(RS_E_INVALID, "bad argument");
    double *da = nullptr, *dr = nullptr, *df = nullptr;
    const size_t bytes = sizeof(double) * size_t(std::max<int64_t>(n, 1));
    CK(cudaMalloc(&da, bytes));
    CK(cudaMalloc(&dr, bytes));
    CK(cudaMalloc(&df, bytes));
    CK(cudaMemcpy(da, a, sizeof(double) * size_t(n), cudaMemcpyHostToDevice));
    CK(rsb::micro::fn_selftest(kind, da, n, dr, df));
    CK(cudaMemcpy(r_ieee, dr, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(r_fast, df, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost));
    cudaFree(da);
    cudaFree(dr);
    cudaFree(df);
    return RS_OK;
}

extern "C" int rs_selftest_div(const double* a, const double* b, int64_t n, double* q_ieee,
                               double* q_fast) {
    double *da = nullptr, *db = nullptr, *dq = nullptr, *df = nullptr;
    const size_t bytes = sizeof(double) * size_t(n);
    CK(cudaMalloc(&da, bytes));
    CK(cudaMalloc(&db, bytes));
    CK(cudaMalloc(&dq, bytes));
    CK(cudaMalloc(&df, bytes));
    CK(cudaMemcpy(da, a, bytes, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, b, bytes, cudaMemcpyHostToDevice));
    CK(rsb::micro::div_selftest(da, db, n, dq, df));
    CK(cudaMemcpy(q_ieee, dq, bytes, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(q_fast, df, bytes, cudaMemcpyDeviceToHost));
    cudaFree(da);
    cudaFree(db);
    cudaFree(dq);
    cudaFree(df);
    return RS_OK;
}
