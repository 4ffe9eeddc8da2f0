/*
 * rodsim_b200.h -- C ABI of the B200-native CoRdE rod step.
 *
 * Drop-in boundary for the reference's compiled core (rodsim._core,
 * pkg/src/rodsim/_core.pyx).  The reference binds the World's numpy arrays
 * by raw pointer (make_context, _core.pyx:219-403) and steps them in place;
 * this library does the same from the host's point of view -- the World
 * arrays are described by plain pointers and sizes, stay authoritative
 * between epochs, and are mirrored in HBM while a kernel runs.  No torch or
 * CUDA types appear in the signatures.
 *
 * Entry point                      replaces (reference file:line)
 * -------------------------------  ------------------------------------------
 * rs_create                        _core.make_context          _core.pyx:219
 * rs_upload / rs_download          zero-copy pointer binding   _core.pyx:192-216
 * rs_run_epoch                     step_serial x K / begin_epoch +
 *                                  run_epoch_worker + epoch_results
 *                                                              _core.pyx:1058-1139
 * rs_error_step                    _core.error_step            _core.pyx:1142
 * rs_step_counter                  _core.step_counter          _core.pyx:1147
 * rs_update_params                 _core.update_params         _core.pyx:1083
 * rs_barrier_timing                barrier wait accounting     _core.pyx:453-471
 * rs_stage_commands                _core.stage_commands        _core.pyx:1151
 * rs_applied_step_for              _core.applied_step_for      _core.pyx:1181
 * rs_read_snapshot                 SnapshotBuffer.read         engine.py:113
 * rs_destroy                       (context GC)
 * rs_last_error                    exception text of the above
 *
 * Error convention: functions return RS_OK (0) or a negative RS_E* code and
 * leave a message for rs_last_error().  Like the reference, the kernel never
 * aborts on non-finite forces or zero-length segments: it records the step
 * (rs_error_step) and the caller raises FloatingPointError (engine.py:328).
 */
#ifndef RODSIM_B200_H
#define RODSIM_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_ABI_VERSION 2

enum rs_status {
    RS_OK = 0,
    RS_E_INVALID = -1,      /* bad argument (ValueError) */
    RS_E_CUDA = -2,         /* CUDA runtime failure (RuntimeError) */
    RS_E_UNSUPPORTED = -3,  /* scene feature outside this build's scope */
    RS_E_RING_FULL = -4,    /* command ring full (RuntimeError) */
    RS_E_RUNTIME = -5       /* scene rejected at bind time (RuntimeError) */
};

enum rs_precision {
    RS_F64_MIRROR = 0,      /* fp64, no FMA, reference rounding: bitwise parity */
    RS_F32 = 1,             /* fp32 with FMA: tolerance parity */
    RS_F64_FAST = 2         /* fp64 with FMA: 1e-9 parity on well-conditioned scenes */
};

/* upload / download masks */
#define RS_STATE   0x1u     /* positions, velocities, frames, angular velocities */
#define RS_STATIC  0x2u     /* material arrays, masses, locks, bindings, maps */
#define RS_CONTROL 0x4u     /* drivers and grab anchors */
#define RS_STATIC_IF_CHANGED 0x8u  /* RS_STATIC only if a static array differs
                                      from the last static upload (memcmp) */

/* Host view of a World (world.py:77-182).  All arrays are C-contiguous,
 * float64 / int64 / uint8 exactly as the reference World holds them, and
 * must outlive the handle (the reference keeps them alive via ctx.refs). */
typedef struct rs_world_desc {
    int32_t abi_version;    /* RS_ABI_VERSION */
    int32_t precision;      /* enum rs_precision */
    int32_t device;         /* CUDA device ordinal */
    int32_t force_tier;     /* -1 auto; 0 CTA, 1 cluster, 2 grid (testing) */
    int32_t force_ctas;     /* 0 auto; >0 CTAs per rod for cluster/grid tiers */
    int32_t force_variant;  /* -1 auto; else CTA-tier variant index (testing) */
    int64_t P, E, R;        /* points, elements, rods */
    int64_t iters;          /* solver.iterations */
    int64_t step_index;     /* world.step_index: initial core step counter */
    double dt, beta, gx, gy, gz;
    const int64_t *rod_offsets;       /* (R+1) first point of each rod, P */
    /* dynamic state (rs_upload RS_STATE / rs_download RS_STATE) */
    double *pos, *vel, *q, *w;        /* (P,3) (P,3) (E,4) (E,3) */
    /* constants (RS_STATIC) */
    const double *rest, *ustar, *mass, *invm, *inert, *fext;
    const double *ks, *kp, *gt, *gr, *ext, *kb;
    const uint8_t *plock, *flock, *jvalid;
    const int64_t *elem_point, *elem_parity;
    const int64_t *drv_pt, *drv_fr;   /* (R) driven point / frame or -1 */
    int64_t nbind;
    const int64_t *bind_a, *bind_b, *bind_mode;
    /* control (RS_CONTROL); also mutated by staged commands */
    double *drv_v, *drv_rot;          /* (R,3) (R) */
    int64_t ngrab;
    uint8_t *g_act;
    int64_t *g_pt;
    double *g_tgt;                    /* (ngrab,3) */
    /* mesh contacts (ABI 2).  The tree is the reference's TriMeshBvh
     * (bvh.py:22-44): implicit-heap AABB nodes, <= 2 triangles per leaf;
     * has_mesh 0 leaves the tree pointers unused.  The contact slots
     * (world.py:157-161) are state: uploaded / downloaded with RS_STATE. */
    int64_t has_mesh, n_nodes, mesh_depth, n_tris, n_verts;
    const double *nmin, *nmax;        /* (n_nodes,3) node boxes */
    const int64_t *nstart, *ncount;   /* (n_nodes) leaf range / count (-1 unused) */
    const int64_t *torder, *tris;     /* (n_tris) leaf order, (n_tris,3) */
    const double *verts;              /* (n_verts,3) */
    const double *cradii;             /* (P) world.contact_radii */
    const uint8_t *cmask;             /* (P) world.collide_mesh_mask */
    uint8_t *cact;                    /* (P) contact_active */
    double *cnorm, *cdepth;           /* (P,3) (P) contact_normal / depth */
    double *cacc_n, *cacc_t;          /* (P) contact_acc_n / acc_t */
    int64_t coll_interval;            /* world.collision_interval */
    double coll_margin;               /* world.collision_margin */
    double restitution, mu;           /* solver.restitution, solver.mu */
    /* self-collision (ABI 2; has_self 0: none): the point-group table as
     * make_context builds it (_core.pyx:316-345) and the world's pair
     * buffers (world.py:164-168, state).  All rods must fit one CTA-tier
     * segment (<= 513 points): the pairs couple arbitrary points and are
     * applied in list order. */
    int64_t has_self, n_groups, excl, pair_cap;
    const int64_t *grp_rod, *grp_gi, *grp_s, *grp_e;   /* (n_groups) */
    double touch, broad;              /* 2 point_radius, 2 sphere_radius */
    int64_t *pair_a, *pair_b;         /* (pair_cap) */
    double *pair_md, *pair_acc;       /* (pair_cap) */
    /* 1: live launches -- for a plan of one CTA or one cluster the kernel
     * drains staged commands at every step boundary, so commands staged while
     * an epoch runs apply at the next step (the reference's parallel backend,
     * engine.py:177-198); 0: they apply at the next epoch.  Live launches use
     * the heavier scene-feature kernels. */
    int64_t live;
} rs_world_desc;

typedef struct rs_handle_s *rs_handle;

int rs_create(const rs_world_desc *desc, rs_handle *out);
int rs_upload(rs_handle h, uint32_t mask);
/* Advance `steps` time steps on the device state (K steps per launch).
 * Applies commands staged with rs_stage_commands at the first step boundary.
 * contacts: active mesh contacts + self-collision pairs after the last
 * step (epoch_results, _core.pyx:1133; waits for the epoch when the scene
 * has contacts); barrier_ns: with rs_barrier_timing on, the summed time the
 * CTAs (thread 0 of each) spent waiting in the step's barriers, the
 * counterpart of the reference's per-block spin-barrier wait
 * (_core.pyx:453-471, epoch_results 1133-1139; waits for the epoch); else 0.
 * Either pointer may be NULL. */
int rs_run_epoch(rs_handle h, int64_t steps, int64_t *contacts, int64_t *barrier_ns);
int rs_download(rs_handle h, uint32_t mask);
/* rs_upload(RS_STATE) + rs_run_epoch + rs_download(RS_STATE) as one call
 * (the host arrays are authoritative before and after, like the reference's
 * in-place step_serial x K, _core.pyx:1058-1080).  For a plan of
 * independent rods (one CTA/stream-tier launch, fp64) the epoch runs in
 * chunks of rods on three streams so the H2D copy of chunk c+1 and the D2H
 * copy of chunk c-1 overlap the launch on chunk c; results are identical
 * to the sequential sequence.  Synchronous. */
int rs_run_epoch_host(rs_handle h, int64_t steps, int64_t *contacts, int64_t *barrier_ns);
int rs_synchronize(rs_handle h);
int64_t rs_error_step(rs_handle h);
int64_t rs_step_counter(rs_handle h);
int rs_update_params(rs_handle h, double dt, int64_t iters);
/* 1: account barrier waits (rs_run_epoch's barrier_ns) -- launches use the
 * scene-feature kernels, whose barriers read the SM clock around the wait;
 * batched stream-tier launches (independent rods, one CTA each) report 0.
 * 0 (default): no accounting, the plain kernels. */
int rs_barrier_timing(rs_handle h, int on);
/* ops: (n,6) rows [op, i0, i1, f0, f1, f2], ops 0..3 = driver velocity,
 * driver rotation, grab, release (engine.py:30-34). slots: (n) out. */
int rs_stage_commands(rs_handle h, const double *ops, int64_t n, int64_t *slots);
int64_t rs_applied_step_for(rs_handle h, int64_t global_slot);
/* Snapshot of the last completed epoch: pos (P,3), q (E,4). */
int rs_read_snapshot(rs_handle h, double *pos, double *q, int64_t *seq, int64_t *step);
/* Live handles: 1 = the kernel publishes a snapshot after every step
 * (ph_publish, _core.pyx:1045-1052; double-buffered in mapped host memory,
 * read by rs_read_snapshot while a launch runs); 0 = snapshots at epoch
 * boundaries only (the default: per-step publishing costs PCIe writes). */
int rs_live_snapshots(rs_handle h, int on);
void rs_destroy(rs_handle h);
const char *rs_last_error(void);

/* Measurement helpers (bench / tests). */
/* Time the kernels of the last rs_run_epoch with CUDA events on the
 * launching stream; returns milliseconds of the last epoch's launches. */
int rs_enable_timing(rs_handle h, int on);
double rs_last_kernel_ms(rs_handle h);
/* CUDA events on the launching stream around any span of epochs:
 * rs_timer_start, rs_run_epoch..., rs_timer_stop, rs_timer_ms (syncs). */
int rs_timer_start(rs_handle h);
int rs_timer_stop(rs_handle h);
double rs_timer_ms(rs_handle h);
/* Number of kernel launches issued so far (a speculative batched step is
 * two: the speculative kernel and the exact one over its redo list). */
int64_t rs_launch_count(rs_handle h);
/* Rods the last speculative batched launch handed to the exact kernel
 * (quotients outside the fast path's window); 0 when none or when the
 * handle has no speculative launches.  Synchronises the stream. */
int64_t rs_last_redo_count(rs_handle h);
/* JSON description of the launch plan (tiers, CTAs, threads, variants). */
int rs_plan_json(rs_handle h, char *buf, int64_t len);
/* The same plan computed without a device (no CUDA calls, no occupancy
 * checks) for a device with `num_sms` SMs: host-logic tests on CPU. */
int rs_plan_dry(const rs_world_desc *desc, int32_t num_sms, char *buf, int64_t len);
/* Raw device pointer of a state array: 0 pos, 1 vel, 2 q, 3 w (element
 * type double for RS_F64_*, float for RS_F32). */
int rs_device_ptr(rs_handle h, int32_t which, void **out);
/* Self-test: IEEE a/b and the kernel's reciprocal-based quotient for n
 * pairs, computed on the device with the fp64 mirror build flags. */
int rs_selftest_div(const double *a, const double *b, int64_t n, double *q_ieee,
                    double *q_fast);
/* Self-test: kind 0 1/a, kind 1 sqrt(a): the compiler's IEEE result and the
 * branch-free fast-path restatement the batched kernel uses (rod_math.cuh
 * rcp_rn / sqrt_rn), for n inputs on the device. */
int rs_selftest_fn(int32_t kind, const double *a, int64_t n, double *r_ieee, double *r_fast);
/* Measured issue rate of one pipe on the current device (operations/s):
 * kind 0 DFMA, 1 DADD, 2 DMUL, 3 FFMA.  Compute cross-check for the bench. */
int rs_pipe_peak(int kind, double *ops_per_s);
/* Latency microbenchmark for the single-rod latency roofline: kind 0 DADD,
 * 1 DMUL, 2 DFMA, 3 IEEE div, 4 sqrt+add, 5 reciprocal-based div, 6 1/x
 * (dependent chains), 7 shared-memory load chase, 8 bar.sync with `param`
 * threads, 9 barrier.cluster across `param` CTAs (+ one DSMEM read per
 * phase), 10 DSMEM load chase, 11 neighbour-only mbarrier sync along a
 * chain of `param` cluster CTAs (+ one DSMEM read per phase).  out[0] = cycles, out[1] = ns (0 if not
 * measured) per operation / barrier. */
int rs_micro(int kind, int param, double *out);

#ifdef __cplusplus
}
#endif
#endif
