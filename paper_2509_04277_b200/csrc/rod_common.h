// rod_common.h -- structures shared by the host planner (rodsim_capi.cu) and
// the sm_100a step kernels (rod_step.cuh).
//
// Vocabulary: a rod has P_r mass points and E_r = P_r - 1
// elements; element j spans points j, j+1 and carries frame j.  On the device
// a *slot* is one point of a CTA's contiguous point range together with the
// element whose lower point it is (absent for the last point of a rod).
#pragma once
#include <stdint.h>

namespace rsb {

// per-point flags (uint32), built on the host from the World arrays
enum SlotFlag : uint32_t {
    SF_HAS_ELEM = 1u << 0,   // point is not the last of its rod: element e exists
    SF_HAS_PREV = 1u << 1,   // point is not the first of its rod (pt_ehi >= 0)
    SF_JVALID   = 1u << 2,   // junction e|e+1 valid (world.junction_valid[e])
    SF_JPREV    = 1u << 3,   // junction e-1|e valid
    SF_PLOCK    = 1u << 4,   // world.point_locked[p]
    SF_FLOCK    = 1u << 5,   // world.frame_locked[e]
    SF_EXT      = 1u << 6,   // world.extensible[e] != 0
    SF_PARITY   = 1u << 7,   // world.elem_parity[e] & 1
    SF_DRV_PT   = 1u << 8,   // point velocity overwritten by a driver
    SF_DRV_FR   = 1u << 9,   // frame angular velocity overwritten by a driver
    SF_DIST     = 1u << 10,  // element takes part in the distance projection
    // bits 16..23 / 24..31: index into the CTA's driver table for the point
    // (DRV_PT) and the frame (DRV_FR) driver of this slot
};
constexpr int SF_DRV_PT_SHIFT = 16;
constexpr int SF_DRV_FR_SHIFT = 24;
constexpr int MAX_DRV_PER_CTA = 255;

// One CTA's share of the world: a contiguous point range [p0, p0+np).
struct CtaTask {
    int32_t p0;          // first global point
    int32_t np;          // number of points (slots) owned
    int32_t bind_begin;  // range in the binding table
    int32_t bind_count;
    int32_t grab_begin;  // range in the per-epoch grab table
    int32_t grab_count;
    int32_t drv_begin;   // range in the driver table
    int32_t drv_count;
    int32_t bind_seq;    // 1: bindings overlap (not a matching) -> ordered
    int32_t e_uni;       // element whose constants stand for the whole CTA
                         // when the launch uses CTA-uniform constants
    int32_t e0;          // element of the first slot (single-rod tasks)
    int32_t nrods;       // whole rods in the range (0: part of one rod)
};

// Wide-halo cluster kernel (rod_halo.cuh): one CTA's local point-index
// ranges along the rod(s) of the launch -- owned [o0, o1), held [x0, x1)
// (owned plus up to G ghost points per side)
struct HaloTask {
    int32_t o0, o1, x0, x1;
};

// A binding endpoint pair resolved to (cta rank within the cluster, slot).
struct BindEntry {
    int32_t a_rank, a_slot;
    int32_t b_rank, b_slot;
    int32_t mode;        // 0 one-way (a dominates), 1 bidirectional
    int32_t pad;
};

struct GrabEntry {
    int32_t slot;        // local slot of the grabbed point
    int32_t world_slot;  // grab slot index in the World (ordering key)
    double tgt[3];
};

struct DrvEntry {
    int32_t slot;        // local slot
    int32_t kind;        // 0 point velocity, 1 frame rotation
    int32_t rod;         // row of world.driver_velocity / driver_rotation
    int32_t pad;
};

// TIER_STREAM: persistent CTAs, each stepping a sequence of single-rod tasks
// and prefetching the next rod's state with TMA bulk copies (batches).
enum Tier : int { TIER_CTA = 0, TIER_CLUSTER = 1, TIER_GRID = 2, TIER_STREAM = 3 };

// Element material constants of a launch whose elements all share them
// (batches of identical rods): passed by value in the kernel parameters, so
// the step reads them as constant-bank operands instead of registers.
template <typename Real>
struct UniConsts {
    Real l, il, kpl, ks, gt, gr;   // rest length, 1/l, K_p l, K_s, gamma_t, gamma_r
    Real kb[3], us[3], I[3], rI[3];  // bend/twist stiffness, u*, inertia, 1/inertia
};

// The staged-command ring (_core.pyx:1151-1184, ph_boundary 477-506) in
// page-locked, device-mapped host memory: the host appends rows and
// publishes `tail`; the drainer -- the host at an epoch boundary, or, in a
// live launch, the step kernel at every step boundary -- applies rows in
// order, stamps each row's apply step and publishes `head`.
constexpr int RING_CAP = 64;
struct LiveRing {
    int64_t tail;                   // rows published by the host
    int64_t head;                   // rows applied
    int64_t apply[RING_CAP];        // core step each row was applied at (-1: not yet)
    double rows[RING_CAP][6];       // [op, i0, i1, f0, f1, f2]
};

// Per-step snapshot of a live launch (ph_publish, _core.pyx:1045-1052), in
// mapped host memory: two position/frame buffers; the step after which each
// was written; `pub` = version, the readable buffer being version & 1.  The
// kernel writes the other buffer during step s and flips `pub` (release,
// system scope) after the barrier that ends it; a reader copies the buffer
// and retries if `pub` moved meanwhile.
struct LiveSnap {
    int64_t pub;
    int64_t step[2];
};

// Kernel arguments; device pointers, AoS layouts identical to world.py.
template <typename Real>
struct StepArgs {
    Real *pos, *vel, *q, *w;                       // (P,3) (P,3) (E,4) (E,3)
    const Real *rest, *ustar, *inert, *ks, *kp, *gt, *gr, *kb;  // per element
    const Real *mass, *invm, *fext;                // per point
    const Real *drv_v, *drv_rot;                   // (R,3), (R)
    const uint32_t *pflags;                        // (P)
    const int32_t *pt_elem;                        // (P) element or -1
    const CtaTask *tasks;
    const BindEntry *binds;
    const GrabEntry *grabs;
    const DrvEntry *drvs;
    // grid tier: neighbour flags and double-buffered boundary halos
    int32_t *flags;                                // (ncta)
    Real *halo;                                    // (2, ncta, HALO_WORDS)
    unsigned long long *err_step;                  // max erroring step + 1 (0 = none)
    int64_t step0;                                 // core step counter at launch
    int32_t steps;                                 // K steps per launch
    int32_t iters;
    int32_t bind_cap;                              // smem binding slots per CTA
    int32_t drv_cap;                               // smem driver slots per CTA
    int32_t has_fext;
    int32_t ncta;
    int32_t debug;                                 // bit 0: poison smem (NaN) first,
                                                   // bit 1: per-phase cycles -> prof
    unsigned long long *prof;                      // (PROF_SLOTS) phase cycle sums
    // speculative batched launches: rods whose quotients left the fast
    // path's window are listed here (not written back) and stepped again by
    // the exact kernel, which then reads its tasks from the list
    int32_t *redo_list, *redo_count;
    int redo_mode;                                 // 1: tasks = redo_list[0 .. *redo_count)
    int32_t any_binds;                             // launch has bindings (cluster/grid:
    int32_t any_grabs;                             //   barrier count must be uniform)
    int32_t any_dist;                              // launch has distance-projected elements
    int32_t ntasks;                                // stream tier: tasks for gridDim CTAs
    Real dt, beta, gx, gy, gz;
    UniConsts<Real> u;                             // UNI == 2 launches
    // mesh contacts (_core.pyx:509-662, 730-741, 906-947); contacts_on == 0:
    // no contact slot is ever set, the machinery (and its barrier) is off
    int32_t contacts_on, has_mesh, n_nodes, coll_interval;
    const Real *nmin, *nmax, *verts;               // tree boxes (nodes,3), vertices (V,3)
    const int32_t *nstart, *ncount, *torder, *tris;
    const Real *cradii;                            // (P) contact radius
    const uint8_t *cmask;                          // (P) collides with the mesh
    uint8_t *cact;                                 // (P) contact slots (state)
    Real *cnorm, *cdepth, *cacc_n, *cacc_t;        // (P,3) (P) (P) (P)
    unsigned long long *contacts;                  // active contacts after the last step
    Real coll_margin, restitution, mu;
    // self-collision (_core.pyx:665-708, 956-980): CTA tier; broad phase by
    // the whole CTA (list order kept by a prefix sum), pair impulses thread 0
    int32_t has_self, n_groups, excl, pair_cap;
    const int32_t *grp_rod, *grp_gi, *grp_s, *grp_e;
    Real* grp_c;                                   // (G,3) scratch
    int32_t* gp_count;                             // (G(G-1)/2) scratch: pairs per group pair
    int32_t *pair_a, *pair_b, *pair_count;         // pair list, CNT_PAIRS (persistent)
    Real *pair_md, *pair_acc;
    Real touch, broad;
    // live launch (single CTA / single cluster): commands drained at every
    // step boundary from the mapped ring into the device control arrays
    LiveRing* live;                                // null: not live
    Real *drv_v_live, *drv_rot_live;               // = drv_v / drv_rot, writable
    int32_t *g_act, *g_pt;                         // (ngrab) world grab slots
    Real* g_tgt;                                   // (ngrab,3)
    int32_t ngrab, nrods;
    LiveSnap* snap;                                // live per-step snapshot (or null)
    double *snap_pos, *snap_q;                     // (2, P, 3), (2, E, 4)
    int64_t snap_base, snap_P, snap_E;             // version at launch start, sizes
    // barrier wait accounting (the reference's per-block barrier_wait_ns,
    // _core.pyx:453-471): scene-feature kernels only; thread 0 of every CTA
    // adds the SM cycles it spent inside barriers (null: off)
    unsigned long long* bar_cycles;
    // wide-halo cluster kernel: per-CTA ranges, per-point driver rods
    // (2 per point: point driver, frame driver; -1 none), per-point binding
    // code (-1 none; bit 0: endpoint a, bit 1: bidirectional), the launch's
    // rods (NR <= 2, np points each, first point / element), thread stride
    // per rod W and ghost width G
    const HaloTask* htask;
    const int32_t *hdrv, *hbind;
    int32_t h_nr, h_np, h_w, h_g, h_s;   // (h_s: steps per ghost exchange)
    int32_t h_poff[2], h_eoff[2];
    // the group's lazy-redo word: 0, or 1 + the first step of a launch
    // whose vote failed (later launches of the group then skip; the host
    // replays the exact kernel from that step at its next synchronisation)
    int64_t* hfail;
};

constexpr int PROF_SLOTS = 64;

// grid-tier halo record per CTA and buffer (Real words)
constexpr int HALO_WORDS = 32;
// layout inside a halo record
enum HaloOff : int {
    H_FIRST_POS = 0, H_FIRST_VEL = 3, H_FIRST_Q = 6, H_FIRST_W = 10,   // slot 0
    H_LAST_POS = 13, H_LAST_VEL = 16,                                    // last slot
    H_LAST_EF = 19, H_LAST_FN = 22, H_LAST_JT = 26,                      // last slot
};

}  // namespace rsb
