// rod_halo.cuh -- wide-halo cluster kernel: a rod (or a pair of rods bound
// point to point) spread over the CTAs of a thread-block cluster with ONE
// cluster barrier per time step.
//
// The general cluster tier (rod_step.cuh) issues a cluster barrier after each
// of the 2I+3 (3I+3 with bindings) phases of a step, ~300 ns each: 33 x 300 ns
// is ~10 us of the cfg3 pair's 22 us step.  Here every CTA owns a contiguous
// range [o0, o1) of local point indices and also keeps G = 2I+1 ghost points
// on either side, whose state it receives from its neighbours once per step.
// A step's dependency radius along a rod is scatter 1 (element i reads point
// i+1) + gather 1 (point i reads element i-1) + one per colour phase (2I);
// bindings couple the same local index of the two rods (radius 0, both rods'
// columns live in the same CTA).  Computing the whole step redundantly on
// [o0-G, o1+G) therefore leaves the owned range exact, and the only
// inter-CTA exchange is the owned boundary state (pos, vel, q, w of G points
// per side) pushed into the neighbours' ghost slots through distributed
// shared memory before the step's one cluster barrier.  Every other phase
// boundary is a CTA barrier (bar.sync, 15-50 ns).
//
// Layout: thread t = r W + j holds point i = x0 + j of rod r (r < NR <= 2;
// W = the widest extended range of the launch) and the element i -- one point
// per thread, its state in registers, neighbours through shared memory.  The
// colour phases use the one-warp kernel's formulation (rod_warp1.cuh): both
// endpoints of an element compute its impulse from the same inputs with the
// same operations (the upper end holding the tangent negated), so each
// thread moves only its own point and a phase is one shared-memory round trip
// through a ping-pong velocity buffer.  Bindings are done the same way by
// the two threads of a bound column.
//
// Exchange periods: with S steps per exchange the ghost width is S (2I+1)
// (the grid exchange, an L2 round trip of 1-4 us, is amortised over S
// steps; the ghosts step along redundantly in between).
//
// Shared memory: the per-thread state fields are double-buffered by
// exchange-period parity -- the owned boundary points at the end of period p
// are pushed into the neighbours' buffer (p+1)&1 while a slower neighbour may
// still read buffer p&1 (the cluster barrier ending period p orders the
// reuse).
//
// Quotients outside the fast path's window take the IEEE division inline
// (one warp-uniform test per group of quotients); dividends below 2^-400 --
// the rounding noise a planar rod carries in its out-of-plane components --
// are first scaled by 2^700 for the correctly rounded reciprocal-based
// quotient and scaled back (exact while the quotient is a normal number), so
// only quotients that come out subnormal take that branch.  What remains
// speculative -- degenerate segments, non-finite forces (both stamp the
// reference's error step), colour-phase and binding dividends outside the
// window -- is ANDed into a per-thread flag, for the results the owned range
// depends on (a ghost's result of a phase matters while its distance outside
// the owned range is within the radius still to come; the outer ghost shell
// computes garbage from missing neighbours).  At the end of the launch the
// cluster votes; if anything failed, nothing is written back and the launch's
// first step goes into the group's redo word: later launches of the group
// return at once, and the host, at its next synchronisation, replays the
// exact general kernel from that step (results do not depend on how steps
// are split into launches) -- no second launch per epoch in the common case.
//
// Arithmetic: the reference's expression order (oracle/rod_oracle.c cites
// _core.pyx), identical to rod_warp1.cuh / rod_step.cuh.
#pragma once

#include "rod_warp1.cuh"

namespace rsb {

// the state fields (double-buffered) and the per-step fields, T Reals each
enum HaloField : int {
    HL_P = 0, HL_V = 3, HL_Q = 6, HL_W = 10,                    // x 2 (parity)
    HL_CA = 13, HL_CN = 14, HL_CD = 17,                          // contact slot (mesh scenes)
    HL_NSTATE = 18,
    HL_EF = 36, HL_FN = 39, HL_JT = 43, HL_NN = 46, HL_B = 49,  // scatter outputs
    HL_VA = 50, HL_VB = 53,                                      // colour ping-pong
    HL_NF = 56,
};
__host__ __device__ constexpr size_t halo_smem_bytes(int threads, size_t rsz) {
    return align16(size_t(HL_NF) * size_t(threads) * rsz) + 16;
}

// a / b for a dividend of any magnitude whose quotient is a normal number
// (fp64 mirror mode): dividends below the window are scaled by 2^600 (exact),
// divided with the correctly rounded reciprocal-based quotient, and scaled
// back (exact for a normal quotient, so the bits are IEEE a / b's).  The
// scaling factors are 1 for every other dividend, so the instruction stream
// is the same for all.  The operand checks are ANDed into ok.
template <typename R>
__device__ __forceinline__ R hl_quot(R a, R b, R rb, bool& ok) {
#if defined(RSB_MODE_ID) && RSB_MODE_ID == 0
    if constexpr (sizeof(R) == 8) {
        const unsigned ha = unsigned(__double2hiint(a)) & 0x7fffffffu;
        const bool tiny = ha < ((1023u - 400u) << 20);   // [0, 2^-400): x 2^700 -> [0, 2^300)
        const R s = tiny ? R(0x1p700) : R(1.0);
        const R si = tiny ? R(0x1p-700) : R(1.0);
        const R as = a * s;
        const R q = bw_quot(as, b, rb) * si;
        const unsigned eq = unsigned(__double2hiint(q)) & 0x7ff00000u;
        ok = ok & dividend_ok(as) & (!tiny | is_zero(a) | (eq != 0u));
        return q;
    }
#endif
    ok = ok & dividend_ok(a);
    return bw_quot(a, b, rb);
}
// N quotients by one divisor (window b_ok checked by the caller), exact: a
// lane whose operands leave the fast path's range and whose result matters
// (need) takes the IEEE division, behind one warp-uniform test -- dividends
// whose quotient is subnormal (decaying out-of-plane noise) reach it.
template <int N, typename R>
__device__ __forceinline__ void hl_div(const R (&a)[N], R b, R rb, bool b_ok, bool need, R (&q)[N]) {
    bool qok = b_ok;
#pragma unroll
    for (int k = 0; k < N; ++k) q[k] = hl_quot(a[k], b, rb, qok);
    const bool slow = need & !qok;
    if (__any_sync(0xffffffffu, slow)) {
        if (slow)
#pragma unroll
            for (int k = 0; k < N; ++k) q[k] = div_ieee(a[k], b);
    }
}

// TB: the launch's thread bound (registers: 256 -> up to 255, 512 -> 128).
// GX: a co-resident grid instead of one cluster (rods longer than 16 CTAs
// hold, or spread thinner): the owned boundary state goes through a
// double-buffered global halo record per CTA and side, published with a
// release flag per CTA that the two neighbours acquire -- still one exchange
// per step.
// XF: grab anchors, live launches (kernel-side ring drain, snapshots) and
// barrier-wait accounting compiled in -- a plain launch carries none of it
// (with the code present but idle, cfg4 N = 256 ran 4.2 -> 4.7 us per step).
template <typename Real, int MODE, bool GEN, bool BIND, int TB, bool GX, bool XF>
__global__ void __launch_bounds__(TB, 1) rod_halo_kernel(const StepArgs<Real> A) {
    // Programmatic dependent launch: the next launch of the stream may be
    // scheduled at once; this one waits for the previous grid (and its
    // writes) only after the loads of data no kernel writes -- the plan's
    // task and offset tables, point flags, masses -- so their round trips
    // overlap the previous launch's tail (griddepcontrol.wait below).
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    namespace cg = cooperative_groups;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Real* sm = reinterpret_cast<Real*>(smem_raw);
    const int T = blockDim.x, t = threadIdx.x;
    const unsigned rank = GX ? blockIdx.x : cluster_rank();
    const unsigned ncl = gridDim.x;   // one cluster (or one co-resident grid) per launch
    const HaloTask tk = A.htask[rank];
    const int NR = A.h_nr, W = A.h_w, np = A.h_np, ne = np - 1;
    // bound rods interleaved: thread t = 2 j + r holds point j of rod r, so a
    // bound column's two points sit on adjacent lanes of one warp and the
    // binding takes its partner by shuffle; otherwise rod r's points are the
    // threads r W .. r W + W - 1.  ST: the thread distance of neighbouring
    // points of a rod (a compile-time constant on every neighbour access).
    constexpr int ST = BIND ? 2 : 1;
    const int r = BIND ? (t & 1) : t / W, j = BIND ? (t >> 1) : t - (t / W) * W;
    const int i = tk.x0 + j;                        // local index along the rod
    const bool pv = r < NR && i < tk.x1;            // thread holds a point
    const bool ev = pv && i < ne;                   // ... and its element
    const bool own = pv && i >= tk.o0 && i < tk.o1;
    const int rr = pv ? r : 0;
    const int pt = A.h_poff[rr] + (pv ? i : 0);
    const int el = A.h_eoff[rr] + (ev ? i : 0);
#define HS(f, x) sm[(f) * T + (x)]
    const Real dt = A.dt, beta = A.beta;
    const Real rdt = Real(1.0) / dt;
    const bool dt_ok = in_window(dt);
    const Real grav[3] = {A.gx, A.gy, A.gz};
    const bool l_ok = in_window(A.u.l);
    const bool I_ok = in_window(A.u.I[0]) & in_window(A.u.I[1]) & in_window(A.u.I[2]);
    bool ok = true;
    unsigned why = 0;   // RSB_DEBUG bit 2: which checks failed (rs_destroy prints the mask)
#define OKC(bit, cond)                      \
    do {                                    \
        const bool c_ = (cond);             \
        ok = ok & c_;                       \
        if (A.debug & 4) why |= c_ ? 0u : unsigned(bit); \
    } while (0)
    // Which results the owned range depends on: a thread's result of a
    // phase matters while its distance outside [o0, o1) is within the
    // dependency radius still to come (the outer ghost shell computes garbage
    // from missing neighbours and must neither fail the vote nor take the
    // IEEE fallback).  The ghosts are exchanged every S = A.h_s steps; a
    // step's radius is R1 = 2I + 1 with colour sweeps (scatter 1, gather 1,
    // one per colour phase), 1 without; B: the radius still to come in the
    // exchange period at the start of a step.
    const int d_l = tk.o0 - i, d_r = i - (tk.o1 - 1);
    const int dout = max(max(d_l, d_r), 0);
    const int S = A.h_s;
    const bool sweeps = BIND || A.any_dist;
    const int R1 = sweeps ? 2 * A.iters + 1 : 1;
    const bool m_ga0 = pv && dout <= S * R1 - 1;   // statics used by the first step's sweeps

    // barrier wait accounting (the reference's per-block barrier_wait_ns,
    // _core.pyx:453-471; A.bar_cycles non-null for the parallel backend):
    // thread 0 of every CTA adds the SM cycles it waits at the inter-CTA
    // exchange barrier -- the reference's inter-block barrier; the phases'
    // CTA barriers stay untimed (a clock read around each sat on the chain)
    const bool btime = XF && t == 0 && A.bar_cycles != nullptr;
    unsigned long long bwait = 0;
    auto csync = [&]() { __syncthreads(); };
    auto csync_or = [&](int pred) -> int { return __syncthreads_or(pred); };
    auto xsync = [&]() {   // the step's exchange barrier
        const long long tb = btime ? clock64() : 0;
        if (ncl > 1) cluster_barrier();
        else __syncthreads();
        if (btime) bwait += (unsigned long long)(clock64() - tb);
    };

    // neighbours' thread index of a pushed point (same W everywhere)
    const bool has_l = rank > 0, has_r = rank + 1 < ncl;
    const int x0_l = has_l ? A.htask[rank - 1].x0 : 0;
    const int x0_r = has_r ? A.htask[rank + 1].x0 : 0;
    const int G = A.h_g;
    const bool push_l = own && has_l && i < tk.o0 + G;
    const bool push_r = own && has_r && i >= tk.o1 - G;
    Real* sm_l = sm;
    Real* sm_r = sm;
    if constexpr (!GX) {
        if (has_l) sm_l = cg::this_cluster().map_shared_rank(sm, rank - 1);
        if (has_r) sm_r = cg::this_cluster().map_shared_rank(sm, rank + 1);
    }
    // grid exchange: one side's record = NR x G points x 13 state words
    const size_t hrec = size_t(NR) * size_t(G) * HL_NSTATE;
    const int t_l = BIND ? 2 * (i - x0_l) + r : r * W + (i - x0_l);
    const int t_r = BIND ? 2 * (i - x0_r) + r : r * W + (i - x0_r);

    // ---- statics (written by host copies only) ----
    const uint32_t fl = A.pflags[pt];
    const bool pl = (fl & SF_PLOCK) != 0, flk = (fl & SF_FLOCK) != 0;
    const bool dist = (fl & SF_DIST) != 0, ext = (fl & SF_EXT) != 0;
    const Real m = A.mass[pt], rm = rcp_rn(m), im = A.invm[pt];
    const bool m_ok = in_window(m);
    // element i: w_sum = im_i + im_{i+1}; element i-1: im_{i-1} + im_i (the
    // same operands in the same order as the thread that owns it)
    const Real im_up = ev ? A.invm[pt + 1] : Real(0);
    const Real ws = im + im_up;
    const Real rws = rcp_rn(ws);
    const bool act = ev && dist && !(ws <= Real(0));
    OKC(1, !(m_ga0 & act & !in_window(ws)));
    const bool hl = pv && i > 0;   // element i-1 exists
    const uint32_t fl_l = hl ? A.pflags[pt - 1] : 0u;
    const Real ws_l = (hl ? A.invm[pt - 1] : Real(0)) + im;
    const Real rws_l = rcp_rn(ws_l);
    const bool act_l = hl && (fl_l & SF_DIST) && !(ws_l <= Real(0));
    OKC(1, !(m_ga0 & act_l & !in_window(ws_l)));
    // colour c: the element of colour c containing point i -- its own
    // (lower end) when i % 2 == c, the left one (upper end) otherwise
    const bool a_side[2] = {(i & 1) == 0, (i & 1) == 1};
    const int partner[2] = {(i & 1) ? t - ST : t + ST, (i & 1) ? t + ST : t - ST};
    Real wsP[2], rwsP[2];
    bool actP[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        wsP[c] = a_side[c] ? ws : ws_l;
        rwsP[c] = a_side[c] ? rws : rws_l;
        actP[c] = (a_side[c] ? act : act_l) && pv;
    }
    // ---- the previous launch's results from here on ----
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // an earlier launch of this group failed its vote: the host replays
    // the exact kernel from that launch's first step, this one does nothing
    if (*reinterpret_cast<volatile int64_t*>(A.hfail)) return;
    if (A.debug & 1) {   // poison shared memory: uninitialised reads become NaN
        const size_t words = halo_smem_bytes(T, sizeof(Real)) / 4;
        for (size_t x = size_t(t); x < words; x += size_t(T)) reinterpret_cast<uint32_t*>(smem_raw)[x] = 0xffffffffu;
        if (!GX && ncl > 1) cluster_barrier();   // (before any neighbour's DSMEM store)
        else __syncthreads();
    }
    Real p[3], v[3], q[4], w[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        p[k] = A.pos[3 * size_t(pt) + k];
        v[k] = A.vel[3 * size_t(pt) + k];
        w[k] = A.w[3 * size_t(el) + k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = A.q[4 * size_t(el) + k];
    // drivers (_core.pyx:866-875): the rod driving this point / this frame
    const int drp = pv ? A.hdrv[2 * pt] : -1, drf = ev ? A.hdrv[2 * pt + 1] : -1;
    Real dvel[3] = {Real(0), Real(0), Real(0)}, drot = Real(0);
    if (drp >= 0)
#pragma unroll
        for (int k = 0; k < 3; ++k) dvel[k] = A.drv_v[3 * drp + k];
    if (drf >= 0) drot = A.drv_rot[drf];
    // bindings: the point at the same local index of the other rod
    const int hb = (BIND && pv) ? A.hbind[pt] : -1;
    const bool bnd = hb >= 0;
    const bool b_is_a = (hb & 1) != 0;
    const int t_b = t ^ 1;   // (NR == 2)
    Real bw_own = Real(0), bws = Real(0), brws = Real(0);
    if constexpr (BIND) {
        const Real im_o = bnd ? A.invm[A.h_poff[1 - rr] + i] : Real(0);
        const bool bi = (hb & 2) != 0;
        const Real wa = bi ? (b_is_a ? im : im_o) : Real(0);
        const Real wb = b_is_a ? im_o : im;
        bws = wa + wb;
        brws = rcp_rn(bws);
        bw_own = b_is_a ? wa : wb;
    }
    const bool b_upd = bnd && (!b_is_a || bw_own > Real(0));   // one-way: a is never moved
    // grab anchors (_core.pyx:1002-1020): the world's grab slots that hold
    // this point (slot order is the reference's order for several on one
    // point); the phase exists when any slot is active
    bool grabs = XF && A.any_grabs != 0;
    uint32_t gmask = 0;
    if (grabs && pv)
        for (int gsl = 0; gsl < A.ngrab; ++gsl)
            if (A.g_act[gsl] && A.g_pt[gsl] == pt) gmask |= 1u << gsl;

    // Live launches (one cluster, S = 1; ph_boundary, _core.pyx:477-506):
    // the drainer (rank 0, thread 0) applies the ring rows it saw -- its read
    // of the ring's tail is issued a step ahead -- just before the cluster
    // barrier that ends a step, stamping the next step as their apply step,
    // and bumps a generation word in every CTA's shared memory; after the
    // barrier the CTAs reload their driver values and grab slots, so a command
    // takes effect at the same step everywhere.  Per-step snapshots
    // (ph_publish, _core.pyx:1045-1052): owned points written into the
    // unpublished buffer, published by the drainer after the barrier.
    const bool LIVE = XF && A.live != nullptr;
    const bool drainer = LIVE && rank == 0 && t == 0;
    volatile int32_t* ctl =
        reinterpret_cast<volatile int32_t*>(smem_raw + align16(size_t(HL_NF) * size_t(T) * sizeof(Real)) + 4);
    int64_t live_head = 0, live_seen = 0;
    int32_t my_gen = 0, live_gen = 0;
    auto reload = [&]() {
        if (drp >= 0)
#pragma unroll
            for (int k = 0; k < 3; ++k) dvel[k] = A.drv_v_live[3 * drp + k];
        if (drf >= 0) drot = A.drv_rot_live[drf];
        bool anyg = false;
        gmask = 0;
        for (int gsl = 0; gsl < A.ngrab; ++gsl) {
            const bool a = A.g_act[gsl] != 0;
            anyg = anyg || a;
            if (a && pv && A.g_pt[gsl] == pt) gmask |= 1u << gsl;
        }
        grabs = anyg;
    };
    // mesh contacts (_core.pyx:509-662 detection, 906-947 impulses): every
    // thread keeps its point's contact slot in registers (ghosts too, like
    // the rest of the state: detection reads the step-start position, the
    // impulse phase is radius 0); the slots travel with the ghost exchange
    // and the owners write them back
    const bool CONT = XF && A.contacts_on != 0;
    ContactSlot<Real> cs;
    cs.act = false;
    cs.depth = cs.acc_n = cs.acc_t = Real(0);
    cs.n[0] = cs.n[1] = cs.n[2] = Real(0);
    if (CONT && pv) {
        cs.act = A.cact[pt] != 0;
#pragma unroll
        for (int k = 0; k < 3; ++k) cs.n[k] = A.cnorm[3 * size_t(pt) + k];
        cs.depth = A.cdepth[pt];
        cs.acc_n = A.cacc_n[pt];
        cs.acc_t = A.cacc_t[pt];
    }
    if (LIVE) {   // the rows staged before the launch apply at its first step
        if (t == 0) *ctl = 0;
        if (drainer) {
            live_head = *reinterpret_cast<volatile int64_t*>(&A.live->head);
            live_seen = ld_acquire_sys(&A.live->tail);
            if (live_seen > live_head) live_head = live_drain(A, live_head, A.step0);
        }
        if (ncl > 1) cluster_barrier();
        else __syncthreads();
        reload();
    }

    int cur = 0;   // state buffer of this exchange period
    int jp = 0;    // step within the period
    int nx = 0;    // exchanges so far
    for (int step = 0; step < A.steps; ++step) {
        const int sb = cur * HL_NSTATE;
        const int B = (S - jp) * R1;
        const bool m_sc = pv && d_l <= B && d_r <= B - 1;   // scatter of element i
        const bool m_ga = pv && dout <= B - 1;              // gather of point / frame i
        const bool m_in = pv && dout <= B - R1;             // integrate (feeds the next step)
        if (!GX && step > 0 && jp == 0 && !own) {   // ghosts: the state the neighbours pushed
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                p[k] = HS(sb + HL_P + k, t);
                v[k] = HS(sb + HL_V + k, t);
                w[k] = HS(sb + HL_W + k, t);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) q[k] = HS(sb + HL_Q + k, t);
            if (CONT) {
                cs.act = HS(sb + HL_CA, t) != Real(0);
#pragma unroll
                for (int k = 0; k < 3; ++k) cs.n[k] = HS(sb + HL_CN + k, t);
                cs.depth = HS(sb + HL_CD, t);
            }
        }
        if (step == 0 || GX || jp > 0) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                HS(sb + HL_P + k, t) = p[k];
                HS(sb + HL_V + k, t) = v[k];
                HS(sb + HL_W + k, t) = w[k];
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) HS(sb + HL_Q + k, t) = q[k];
            csync();
        }

        int64_t live_next = 0;
        if (drainer) live_next = ld_relaxed_sys(&A.live->tail);   // used at this step's end
        if (CONT) {   // contact slots: reset, detection on collision steps (_core.pyx:730-741)
            cs.acc_n = Real(0);
            cs.acc_t = Real(0);
            if ((A.step0 + step) % A.coll_interval == 0) {
                cs.act = false;
                if (pv && A.has_mesh && A.cmask[pt]) OKC(512, !(mesh_detect(A, int64_t(pt), p, cs) & m_ga));
            }
        }

        // ============ scatter (_core.pyx:745-805): element i ============
        Real pb[3], vb[3], qb[4], wb[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            pb[k] = HS(sb + HL_P + k, t + ST);
            vb[k] = HS(sb + HL_V + k, t + ST);
            wb[k] = HS(sb + HL_W + k, t + ST);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) qb[k] = HS(sb + HL_Q + k, t + ST);
        Real d[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) d[k] = pb[k] - p[k];
        const Real dd = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
        const bool sc = m_sc & ev;
        const bool dd_ok = in_window(dd);
        OKC(2, (!sc | dd_ok));   // a degenerate segment: the exact kernel stamps it
        const Real len = sqrt_rn(dd);
        const Real rlen = rcp_rn(len);
        // the phase's quotients on the fast path; a lane that needs one
        // outside its range recomputes them all with IEEE divisions, behind
        // one warp-uniform test for the phase
        bool slow = false;
        auto fq = [&](Real a, Real b, Real rb, bool b_ok, bool need) -> Real {
            bool qok = b_ok;
            const Real x = hl_quot(a, b, rb, qok);
            slow = slow | (need & !qok);
            return x;
        };
        const Real bnum = beta * (len - A.u.l);
        Real bias = fq(bnum, dt, rdt, dt_ok, sc & dist);
        Real t3[3], nn[3], pair[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) t3[k] = fq(d[k], len, rlen, dd_ok, sc);
        Real kpl_len = fq(A.u.kpl, len, rlen, dd_ok, sc);
        Real v3 = Real(0);
        if constexpr (GEN) v3 = fq(len, A.u.l, A.u.il, l_ok, sc & ext);
        // binding constants of this step (start-of-step positions,
        // _core.pyx:981-1001): d = p_b - p_a on both threads of the column
        Real bd[3] = {Real(0), Real(0), Real(0)}, bnq[3] = {Real(0), Real(0), Real(0)};
        Real bdist = Real(0), bbias = Real(0);
        bool bact = false;
        if constexpr (BIND) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const Real po = HS(sb + HL_P + k, t_b);
                bd[k] = b_is_a ? po - p[k] : p[k] - po;
            }
            const Real bdd = bd[0] * bd[0] + bd[1] * bd[1] + bd[2] * bd[2];
            bact = bnd && !(bdd == Real(0)) && !(bws == Real(0));
            const bool bneed = bact && dout <= B - 3;   // the first binding phase's cone
            bdist = sqrt_rn(bdd);
            const Real rbd = rcp_rn(bdist);
            const bool bdd_ok = in_window(bdd);
            OKC(4, (!bneed | (bdd_ok & in_window(bws))));
#pragma unroll
            for (int k = 0; k < 3; ++k) bnq[k] = fq(bd[k], bdist, rbd, bdd_ok, bneed);
            bbias = fq(beta * bdist, dt, rdt, dt_ok, bneed);
        }
        if (__any_sync(0xffffffffu, slow)) {
            if (slow) {
                bias = div_ieee(bnum, dt);
#pragma unroll
                for (int k = 0; k < 3; ++k) t3[k] = div_ieee(d[k], len);
                kpl_len = div_ieee(A.u.kpl, len);
                if constexpr (GEN) v3 = div_ieee(len, A.u.l);
                if constexpr (BIND) {
#pragma unroll
                    for (int k = 0; k < 3; ++k) bnq[k] = div_ieee(bd[k], bdist);
                    bbias = div_ieee(beta * bdist, dt);
                }
            }
        }
        Real bn[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            pair[k] = Real(0);
            nn[k] = t3[k];
            bn[k] = b_is_a ? bnq[k] : -bnq[k];
        }
        if constexpr (GEN) {   // stretch, Eq. 2
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const Real g = pair[k] - A.u.ks * (v3 - Real(1.0)) * t3[k];
                pair[k] = ext ? g : pair[k];
            }
        }
        Real d3v[3], er[3], f4[4], fo[4], fn[4], ef[3], jt[3];
        dir3(q, d3v);
#pragma unroll
        for (int k = 0; k < 3; ++k) er[k] = t3[k] - d3v[k];
        Real dotp = er[0] * t3[0] + er[1] * t3[1] + er[2] * t3[2];
#pragma unroll
        for (int k = 0; k < 3; ++k) pair[k] = pair[k] - kpl_len * (er[k] - dotp * t3[k]);
        dir3_jt(q, er, f4);
#pragma unroll
        for (int k = 0; k < 4; ++k) fo[k] = A.u.kpl * f4[k];
#pragma unroll
        for (int k = 0; k < 3; ++k) ef[k] = -pair[k] + A.u.gt * (vb[k] - v[k]);
        const bool jv = i + 1 < ne;   // junction i|i+1 inside the rod
        {
            dotp = q[0] * qb[0] + q[1] * qb[1] + q[2] * qb[2] + q[3] * qb[3];
            const Real sgn = dotp < Real(0) ? Real(-1.0) : Real(1.0);
            const Real il = A.u.il;
            Real qnn[4], qp[4], u[3];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                qnn[k] = sgn * qb[k];
                qp[k] = (qnn[k] - q[k]) * il;
            }
            conj_prod_vec(q, qp, u);
#pragma unroll
            for (int k = 0; k < 3; ++k) u[k] = u[k] * Real(2.0);
            const Real two_il = Real(2.0) * il;
            const Real mtwo_il = Real(-2.0) * il;
            Real fob[4], fnb[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                fob[k] = fo[k];
                fnb[k] = Real(0);
            }
            auto bend = [&](auto kc) {
                constexpr int K = decltype(kc)::value;
                const Real du = u[K] - A.u.us[K];
                const Real coeff = A.u.kb[K] * du * A.u.l;
                Real bp[4], ba[4];
                bform<K>(qp, bp);
                bform<K>(q, ba);
                const Real sc = sgn * coeff;
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    const Real ga = Real(2.0) * bp[x] + two_il * ba[x];
                    const Real gn = mtwo_il * ba[x];
                    fob[x] = fob[x] - coeff * ga;
                    fnb[x] = fnb[x] - sc * gn;
                }
            };
            bend(std::integral_constant<int, 0>{});
            bend(std::integral_constant<int, 1>{});
            bend(std::integral_constant<int, 2>{});
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                fo[k] = jv ? fob[k] : fo[k];
                fn[k] = jv ? fnb[k] : Real(0);
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const Real j3 = A.u.gr * (wb[k] - w[k]);
                jt[k] = jv ? j3 : Real(0);
            }
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            HS(HL_EF + k, t) = ef[k];
            HS(HL_JT + k, t) = jt[k];
            HS(HL_NN + k, t) = nn[k];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) HS(HL_FN + k, t) = fn[k];
        HS(HL_B, t) = bias;
        csync();

        // ============ gather (_core.pyx:808-875): point i, frame i ============
        Real efl[3], fnl[4], jtl[3], nn_l[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            efl[k] = HS(HL_EF + k, t - ST);
            jtl[k] = HS(HL_JT + k, t - ST);
            nn_l[k] = HS(HL_NN + k, t - ST);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) fnl[k] = HS(HL_FN + k, t - ST);
        const Real bias_l = HS(HL_B, t - ST);
        Real a_v[3], dvv[3], a_w[3], dww[3];
        slow = false;
        {
            const bool hp = i > 0;
            Real f[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                f[k] = m * grav[k];
                f[k] = f[k] + ((GEN && A.has_fext) ? A.fext[3 * size_t(pt) + k] : Real(0));
                const Real g0 = f[k] + ef[k];   // the point's own element (not the last point)
                f[k] = ev ? g0 : f[k];
                const Real g = f[k] - efl[k];
                f[k] = hp ? g : f[k];
            }
            OKC(8, (!m_ga | (isfinite(f[0]) & isfinite(f[1]) & isfinite(f[2]))));
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                a_v[k] = dt * f[k];
                dvv[k] = fq(a_v[k], m, rm, m_ok, m_ga & !pl);
            }
        }
        {   // frame i
            const bool jp = i > 0;
            Real F[4], tau[3], iw[3], gy[3];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const Real g = fo[k] + fnl[k];
                F[k] = jp ? g : fo[k];
            }
            const Real dot = F[0] * q[0] + F[1] * q[1] + F[2] * q[2] + F[3] * q[3];
#pragma unroll
            for (int k = 0; k < 4; ++k) F[k] = F[k] - dot * q[k];
            conj_prod_vec(q, F, tau);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                tau[k] = tau[k] * Real(0.5);
                const Real g = tau[k] + jt[k];
                tau[k] = jv ? g : tau[k];
                const Real g2 = tau[k] - jtl[k];
                tau[k] = jp ? g2 : tau[k];
            }
            OKC(16, (!(m_ga & ev) | (isfinite(tau[0]) & isfinite(tau[1]) & isfinite(tau[2]))));
#pragma unroll
            for (int k = 0; k < 3; ++k) iw[k] = A.u.I[k] * w[k];
            gy[0] = w[1] * iw[2] - w[2] * iw[1];
            gy[1] = w[2] * iw[0] - w[0] * iw[2];
            gy[2] = w[0] * iw[1] - w[1] * iw[0];
#pragma unroll
            for (int k = 0; k < 3; ++k) {   // per-axis inertia
                a_w[k] = dt * (tau[k] - gy[k]);
                dww[k] = fq(a_w[k], A.u.I[k], A.u.rI[k], I_ok, m_ga & ev & !flk);
            }
        }
        if (__any_sync(0xffffffffu, slow)) {
            if (slow) {
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    dvv[k] = div_ieee(a_v[k], m);
                    dww[k] = div_ieee(a_w[k], A.u.I[k]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            add_if(!pl, v[k], dvv[k]);
            add_if(!flk, w[k], dww[k]);
        }
        // drivers overwrite after the update
        if (drp >= 0)
#pragma unroll
            for (int k = 0; k < 3; ++k) v[k] = dvel[k];
        if (drf >= 0) {
            w[0] = Real(0.0);
            w[1] = Real(0.0);
            w[2] = drot;
        }

        // ============ constraint iterations (_core.pyx:1069-1076) ============
        Real nP[2][3], bP[2];   // the phase's element tangent, negated on the b side
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            bP[c] = a_side[c] ? bias : bias_l;
#pragma unroll
            for (int k = 0; k < 3; ++k) nP[c][k] = a_side[c] ? nn[k] : -nn_l[k];
        }
        // (rods without distance-projected elements and bindings: no sweeps,
        // like the general kernel)
        // The sweeps run on the fast quotients; a lane whose result the
        // owned range needs and whose dividend left the window (rare: tiny
        // impulses early in a run) is noted, the notes ORed into the sweeps'
        // last barrier, and then this CTA alone replays its sweeps from the
        // post-gather velocities with the IEEE division for such lanes (one
        // warp-uniform test per phase) -- its neighbours are unaffected.
        const int iters = (BIND || grabs || CONT || A.any_dist) ? A.iters : 0;
        const Real v_g[3] = {v[0], v[1], v[2]};
        auto sweeps = [&](auto careful_c) -> int {
            constexpr bool CAREFUL = decltype(careful_c)::value;
            int vb_off = HL_VA;
            bool noted = false;
            int any_noted = 0;
#pragma unroll
            for (int k = 0; k < 3; ++k) HS(vb_off + k, t) = v[k];
            csync();
            int rem = B - 1;   // radius still to come after the current phase
            // one iteration; the fast sweeps' last phase ends at an OR-barrier
            // that collects the notes (the last iteration is peeled, so no
            // phase tests which barrier to take)
            auto iteration = [&](auto last_c) {
                constexpr bool LAST = decltype(last_c)::value;
                // the iteration's final phase: odd colour, binding or grab
                auto end_phase = [&](bool final_) {
                    if (!CAREFUL && LAST && final_) any_noted = csync_or(noted);
                    else csync();
                };
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    --rem;
                    const bool chk = pv && dout <= rem;
                    Real dv[3];
#pragma unroll
                    for (int k = 0; k < 3; ++k) dv[k] = HS(vb_off + k, partner[c]) - v[k];
                    Real x = dv[0] * nP[c][0];
                    x = x + dv[1] * nP[c][1];
                    x = x + dv[2] * nP[c][2];
                    x = x + bP[c];
                    const Real q0 = (-x) * rwsP[c];
                    Real lam = fma(fma(-q0, wsP[c], -x), rwsP[c], q0);
                    const bool z = is_zero(x);
                    if (z) lam = Real(-0.0);
                    const bool off = chk & actP[c] & !(in_window(x) | z);
                    if constexpr (CAREFUL) {
                        // the reference's -(((0 + p0) + p1) + p2 + bias) / w_sum
                        if (__any_sync(0xffffffffu, off))
                            if (off) lam = div_ieee(-(x + Real(0.0)), wsP[c]);
                    } else {
                        noted = noted | off;
                    }
#pragma unroll
                    for (int k = 0; k < 3; ++k) sub_if(actP[c], v[k], im * lam * nP[c][k]);
                    if (c == 1) {
                        // The iteration's central phases (_core.pyx:906-1020:
                        // contacts, bindings, grabs) are radius 0 along a rod
                        // and a binding's partner is the adjacent lane, so they
                        // run here, before the odd phase's one barrier.
                        if (CONT) {   // contact impulses, own point
                            if (cs.act && !pl) contact_impulse_r(A, m, v, cs);
                        }
                        if constexpr (BIND) {   // bindings: the partner's post-odd velocity by shuffle
                            Real vbp[3];
#pragma unroll
                            for (int k = 0; k < 3; ++k) vbp[k] = __shfl_xor_sync(0xffffffffu, v[k], 1);
                            Real vrel = Real(0.0);
#pragma unroll
                            for (int k = 0; k < 3; ++k) vrel = vrel + (vbp[k] - v[k]) * bn[k];
                            // the colour phases' quotient: vrel and bias are never
                            // -0 (vrel starts from +0, the bias is >= 0), so a zero
                            // dividend gives -0 like the reference's
                            // -(vrel + bias) / ws; outside the window: noted
                            const Real xb = vrel + bbias;
                            const Real qb0 = (-xb) * brws;
                            Real blam = fma(fma(-qb0, bws, -xb), brws, qb0);
                            const bool zb = is_zero(xb);
                            if (zb) blam = Real(-0.0);
                            const bool boff = bact & (dout <= rem) & !(in_window(xb) | zb);
                            if constexpr (CAREFUL) {
                                if (__any_sync(0xffffffffu, boff))
                                    if (boff) blam = div_ieee(-(vrel + bbias), bws);
                            } else {
                                noted = noted | boff;
                            }
#pragma unroll
                            for (int k = 0; k < 3; ++k) sub_if(bact & b_upd, v[k], bw_own * blam * bn[k]);
                        }
                        if (XF && grabs) {   // grab anchors, start-of-step positions, slot order
                            uint32_t gm = gmask;
                            while (gm) {
                                const int gsl = __ffs(gm) - 1;
                                gm &= gm - 1;
                                const Real wbv = im;
                                if (wbv == Real(0)) continue;
                                Real d[3], gn[3];
#pragma unroll
                                for (int k = 0; k < 3; ++k) d[k] = p[k] - A.g_tgt[3 * gsl + k];
                                const Real dist = norm3(d);
                                if (dist == Real(0)) continue;
                                Real gvrel = Real(0.0);
#pragma unroll
                                for (int k = 0; k < 3; ++k) {
                                    gn[k] = d[k] / dist;
                                    gvrel = gvrel + v[k] * gn[k];
                                }
                                const Real glam = -(gvrel + beta * dist / dt) / wbv;
#pragma unroll
                                for (int k = 0; k < 3; ++k) v[k] = v[k] + wbv * glam * gn[k];
                            }
                        }
                    }
                    vb_off = HL_VA + HL_VB - vb_off;
#pragma unroll
                    for (int k = 0; k < 3; ++k) HS(vb_off + k, t) = v[k];
                    end_phase(c == 1);
                }
            };
            if constexpr (CAREFUL) {
                for (int it = iters; it > 0; --it) iteration(std::false_type{});
            } else {
                for (int it = iters; it > 1; --it) iteration(std::false_type{});
                iteration(std::true_type{});
            }
            return any_noted;
        };
        if (iters > 0 && sweeps(std::false_type{})) {
            if (CONT) {   // (the step's accumulators start at zero)
                cs.acc_n = Real(0);
                cs.acc_t = Real(0);
            }
            if (A.debug & 4) why |= 256u | 32u;   // (debug: a careful replay happened)
#pragma unroll
            for (int k = 0; k < 3; ++k) v[k] = v_g[k];
            sweeps(std::true_type{});
        }

        // ================= integrate (_core.pyx:1023-1042) =================
#pragma unroll
        for (int k = 0; k < 3; ++k) p[k] = p[k] + dt * v[k];
        {
            Real dq[4];
            const Real om[4] = {Real(0.0), w[0], w[1], w[2]};
            hprod(q, om, dq);
            const Real h = dt * Real(0.5);
            Real qq4[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) qq4[k] = q[k] + h * dq[k];
            const Real qq = qq4[0] * qq4[0] + qq4[1] * qq4[1] + qq4[2] * qq4[2] + qq4[3] * qq4[3];
            const bool qq_ok = in_window(qq);
            OKC(128, (!(m_in & ev) | qq_ok));
            const Real nrm = sqrt_rn(qq);
            const Real rn = rcp_rn(nrm);
            Real qn[4];
            hl_div<4>(qq4, nrm, rn, qq_ok, m_in & ev, qn);
#pragma unroll
            for (int k = 0; k < 4; ++k) q[k] = qn[k];
        }

        if (LIVE) {
            if (A.snap && own) {   // this step's snapshot into the unpublished buffer
                const int64_t wbuf = (A.snap_base + step + 1) & 1;
                double* sp = A.snap_pos + wbuf * 3 * A.snap_P;
                double* sq = A.snap_q + wbuf * 4 * A.snap_E;
#pragma unroll
                for (int k = 0; k < 3; ++k) sp[3 * size_t(pt) + k] = double(p[k]);
                if (ev)
#pragma unroll
                    for (int k = 0; k < 4; ++k) sq[4 * size_t(el) + k] = double(q[k]);
            }
            if (drainer) {   // the next step's commands, before the barrier ending this one
                if (step + 1 < A.steps && live_seen > live_head) {
                    live_head = live_drain(A, live_head, A.step0 + step + 1);
                    ++live_gen;
                    for (unsigned c = 0; c < ncl; ++c)
                        *cg::this_cluster().map_shared_rank(const_cast<int32_t*>(ctl), c) = live_gen;
                }
                live_seen = live_next;
            }
        }

        // ===== exchange (every S steps): owned boundary state to the neighbours =====
        const bool xs = jp == S - 1 && step + 1 < A.steps;
        jp = xs ? 0 : jp + 1;
        if (GX && xs) {
            const int par = nx & 1;
            ++nx;
            Real* mine = A.halo + (size_t(par) * ncl + rank) * 2 * hrec;
            auto gput = [&](Real* b, int idx) {
                Real* x = b + (size_t(r) * G + idx) * HL_NSTATE;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    x[HL_P + k] = p[k];
                    x[HL_V + k] = v[k];
                    x[HL_W + k] = w[k];
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) x[HL_Q + k] = q[k];
                if (CONT) {
                    x[HL_CA] = cs.act ? Real(1) : Real(0);
#pragma unroll
                    for (int k = 0; k < 3; ++k) x[HL_CN + k] = cs.n[k];
                    x[HL_CD] = cs.depth;
                }
            };
            if (push_l) gput(mine, i - tk.o0);                    // side 0: for the left neighbour
            if (push_r) gput(mine + hrec, i - (tk.o1 - G));       // side 1: for the right one
            csync();
            if (t == 0) {
                __threadfence();
                st_release_gpu(A.flags + rank, nx);
                if (has_l)
                    while (ld_acquire_gpu(A.flags + rank - 1) < nx) {}
                if (has_r)
                    while (ld_acquire_gpu(A.flags + rank + 1) < nx) {}
            }
            csync();
            if (pv && !own) {
                const bool left = i < tk.o0;
                const Real* src = A.halo + (size_t(par) * ncl + (left ? rank - 1 : rank + 1)) * 2 * hrec +
                                  (left ? hrec : 0);
                const int idx = left ? i - (tk.o0 - G) : i - tk.o1;
                const Real* x = src + (size_t(r) * G + idx) * HL_NSTATE;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    p[k] = ld_halo(x + HL_P + k);
                    v[k] = ld_halo(x + HL_V + k);
                    w[k] = ld_halo(x + HL_W + k);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) q[k] = ld_halo(x + HL_Q + k);
                if (CONT) {
                    cs.act = ld_halo(x + HL_CA) != Real(0);
#pragma unroll
                    for (int k = 0; k < 3; ++k) cs.n[k] = ld_halo(x + HL_CN + k);
                    cs.depth = ld_halo(x + HL_CD);
                }
            }
        } else if (!GX && xs) {
            cur ^= 1;
            const int nb = cur * HL_NSTATE;
            auto put = [&](Real* base, int x) {
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    base[(nb + HL_P + k) * T + x] = p[k];
                    base[(nb + HL_V + k) * T + x] = v[k];
                    base[(nb + HL_W + k) * T + x] = w[k];
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) base[(nb + HL_Q + k) * T + x] = q[k];
                if (CONT) {
                    base[(nb + HL_CA) * T + x] = cs.act ? Real(1) : Real(0);
#pragma unroll
                    for (int k = 0; k < 3; ++k) base[(nb + HL_CN + k) * T + x] = cs.n[k];
                    base[(nb + HL_CD) * T + x] = cs.depth;
                }
            };
            if (own) put(sm, t);
            if (push_l) put(sm_l, t_l);
            if (push_r) put(sm_r, t_r);
            xsync();
        }
        if (LIVE && step + 1 < A.steps) {   // (live launches exchange every step)
            if (A.snap && drainer) {        // the step's snapshot: every CTA's writes are done
                const int64_t ver = A.snap_base + step + 1;
                *reinterpret_cast<volatile int64_t*>(&A.snap->step[ver & 1]) = A.step0 + step + 1;
                st_release_sys(&A.snap->pub, ver);
            }
            if (*ctl != my_gen) {   // commands applied for the next step
                my_gen = *ctl;
                reload();
            }
        }
    }

    // ---- the cluster's vote, then write-back (or the exact redo) ----
    int* vote = reinterpret_cast<int*>(smem_raw + align16(size_t(HL_NF) * size_t(T) * sizeof(Real)));
    const int bad = __syncthreads_or(!ok);   // (ok only collects results the owned range needs)
    int any = 0;
    if constexpr (GX) {
        // grid: OR into the redo word, then an arrival count over all CTAs
        // (co-resident) before anyone reads it
        if (t == 0) {   // flags[ncl]: arrivals, flags[ncl + 1]: the OR of the votes
            if (bad) atomicOr(A.flags + ncl + 1, 1);
            __threadfence();
            atomicAdd(A.flags + ncl, 1);
            while (ld_acquire_gpu(A.flags + ncl) < int(ncl)) {}
            *vote = ld_acquire_gpu(A.flags + ncl + 1);
        }
        __syncthreads();
        any = *vote;
    } else if (ncl == 1) {   // one CTA: its own vote
        any = bad;
    } else {
        if (t == 0) *vote = bad;
        cluster_barrier();
        if (t < int(ncl)) any = *cg::this_cluster().map_shared_rank(vote, t);
        any = __syncthreads_or(any);
        cluster_barrier();   // every remote read done before a CTA exits
    }
    if (LIVE && A.snap && drainer) {   // the last step's snapshot
        const int64_t ver = A.snap_base + A.steps;
        *reinterpret_cast<volatile int64_t*>(&A.snap->step[ver & 1]) = A.step0 + A.steps;
        st_release_sys(&A.snap->pub, ver);
    }
    if (btime && bwait) atomicAdd(A.bar_cycles, bwait);
    if ((A.debug & 4) && why && A.prof) atomicOr(A.prof + PROF_SLOTS - 1, (unsigned long long)why);
#undef OKC
    if (any) {   // nothing written back: the host replays this launch exactly
        if (rank == 0 && t == 0) *A.hfail = A.step0 + 1;
        return;
    }
    if (CONT && own) {   // the contact slots; epoch_results' count after the last step
        A.cact[pt] = cs.act ? 1 : 0;
#pragma unroll
        for (int k = 0; k < 3; ++k) A.cnorm[3 * size_t(pt) + k] = cs.n[k];
        A.cdepth[pt] = cs.depth;
        A.cacc_n[pt] = cs.acc_n;
        A.cacc_t[pt] = cs.acc_t;
        if (cs.act) atomicAdd(A.contacts, 1ull);
    }
    if (own) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            A.pos[3 * size_t(pt) + k] = p[k];
            A.vel[3 * size_t(pt) + k] = v[k];
        }
        if (ev) {
#pragma unroll
            for (int k = 0; k < 3; ++k) A.w[3 * size_t(el) + k] = w[k];
#pragma unroll
            for (int k = 0; k < 4; ++k) A.q[4 * size_t(el) + k] = q[k];
        }
    }
#undef HS
}

}  // namespace rsb
