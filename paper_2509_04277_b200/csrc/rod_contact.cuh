// rod_contact.cuh -- mesh contacts for the step kernel: per-point detection
// against the triangle mesh's AABB tree (broad phase: iterative traversal of
// the implicit heap with a 32-entry stack; narrow phase: Ericson's closest
// point; aggregation: penetration-weighted normal, maximum depth) and the
// per-point normal impulse with accumulator and box friction.
//
// Restated from the reference core (_core.pyx:509-662 detection, 906-947
// impulses) with the same operation order, so the fp64 mirror build rounds
// exactly like it; the traversal order (right child popped first) and the
// hit order inside a leaf fix the order of the weighted-normal sum.  Every
// point is independent: one thread per owned point, tree and mesh read
// through the read-only path (they are small and stay L2-resident).
#pragma once
#include <stdint.h>

#include "rod_common.h"

namespace rsb {

constexpr int CONTACT_STACK = 32;   // _core.pyx:55 STACK_CAP

template <typename Real>
__device__ __forceinline__ void closest_tri(const Real p[3], const Real a[3], const Real b[3], const Real c[3],
                                            Real out[3]) {
    Real ab[3], ac[3], ap[3];
    for (int k = 0; k < 3; ++k) {
        ab[k] = b[k] - a[k];
        ac[k] = c[k] - a[k];
        ap[k] = p[k] - a[k];
    }
    const Real d1 = ab[0] * ap[0] + ab[1] * ap[1] + ab[2] * ap[2];
    const Real d2 = ac[0] * ap[0] + ac[1] * ap[1] + ac[2] * ap[2];
    if (d1 <= Real(0) && d2 <= Real(0)) {
        for (int k = 0; k < 3; ++k) out[k] = a[k];
        return;
    }
    Real bp[3];
    for (int k = 0; k < 3; ++k) bp[k] = p[k] - b[k];
    const Real d3 = ab[0] * bp[0] + ab[1] * bp[1] + ab[2] * bp[2];
    const Real d4 = ac[0] * bp[0] + ac[1] * bp[1] + ac[2] * bp[2];
    if (d3 >= Real(0) && d4 <= d3) {
        for (int k = 0; k < 3; ++k) out[k] = b[k];
        return;
    }
    const Real vc = d1 * d4 - d3 * d2;
    if (vc <= Real(0) && d1 >= Real(0) && d3 <= Real(0)) {
        const Real t = d1 / (d1 - d3);
        for (int k = 0; k < 3; ++k) out[k] = a[k] + t * ab[k];
        return;
    }
    Real cp[3];
    for (int k = 0; k < 3; ++k) cp[k] = p[k] - c[k];
    const Real d5 = ab[0] * cp[0] + ab[1] * cp[1] + ab[2] * cp[2];
    const Real d6 = ac[0] * cp[0] + ac[1] * cp[1] + ac[2] * cp[2];
    if (d6 >= Real(0) && d5 <= d6) {
        for (int k = 0; k < 3; ++k) out[k] = c[k];
        return;
    }
    const Real vb = d5 * d2 - d1 * d6;
    if (vb <= Real(0) && d2 >= Real(0) && d6 <= Real(0)) {
        const Real t = d2 / (d2 - d6);
        for (int k = 0; k < 3; ++k) out[k] = a[k] + t * ac[k];
        return;
    }
    const Real va = d3 * d6 - d5 * d4;
    if (va <= Real(0) && (d4 - d3) >= Real(0) && (d5 - d6) >= Real(0)) {
        const Real t = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        for (int k = 0; k < 3; ++k) out[k] = b[k] + t * (c[k] - b[k]);
        return;
    }
    const Real denom = Real(1.0) / (va + vb + vc);
    for (int k = 0; k < 3; ++k) out[k] = a[k] + ab[k] * (vb * denom) + ac[k] * (vc * denom);
}

// A point's contact slot (_core.pyx:730-741) held in registers (the wide-halo
// kernel keeps one per thread; the general kernel's slots live in global
// memory, the wrappers below).
template <typename Real>
struct ContactSlot {
    Real n[3], depth, acc_n, acc_t;
    bool act;
};

// Detection for global point p with centre `center` (start-of-step position):
// on a hit the slot's normal and depth are set and act = true (a miss leaves
// the slot alone); returns true for a degenerate (zero-area) triangle met.
template <typename Real>
__device__ __noinline__ bool mesh_detect(const StepArgs<Real>& A, int64_t p, const Real center[3],
                                         ContactSlot<Real>& cs) {
    int stack[CONTACT_STACK];
    const Real radius = A.cradii[p] + A.coll_margin;
    Real lo[3], hi[3], wsum[3] = {Real(0), Real(0), Real(0)}, best[3] = {Real(0), Real(0), Real(0)};
    for (int k = 0; k < 3; ++k) {
        lo[k] = center[k] - radius;
        hi[k] = center[k] + radius;
    }
    bool degenerate = false;
    int nhits = 0, top = 1;
    Real maxd = Real(-1.0);
    stack[0] = 0;
    while (top) {
        const int node = stack[--top];
        if (node >= A.n_nodes) continue;
        const int cnt = __ldg(A.ncount + node);
        if (cnt < 0) continue;
        const Real* mn = A.nmin + 3 * node;
        const Real* mx = A.nmax + 3 * node;
        if (__ldg(mn) > hi[0] || __ldg(mn + 1) > hi[1] || __ldg(mn + 2) > hi[2] || __ldg(mx) < lo[0] ||
            __ldg(mx + 1) < lo[1] || __ldg(mx + 2) < lo[2])
            continue;
        if (cnt == 0) {
            stack[top] = 2 * node + 1;
            stack[top + 1] = 2 * node + 2;
            top += 2;
            continue;
        }
        const int first = __ldg(A.nstart + node);
        for (int t = first; t < first + cnt; ++t) {
            const int tri = __ldg(A.torder + t);
            Real a[3], b[3], c[3], e1[3], e2[3], face[3], cl[3], delta[3], n[3];
            const int ia = __ldg(A.tris + 3 * tri), ib = __ldg(A.tris + 3 * tri + 1), ic = __ldg(A.tris + 3 * tri + 2);
            for (int k = 0; k < 3; ++k) {
                a[k] = __ldg(A.verts + 3 * ia + k);
                b[k] = __ldg(A.verts + 3 * ib + k);
                c[k] = __ldg(A.verts + 3 * ic + k);
            }
            for (int k = 0; k < 3; ++k) {
                e1[k] = b[k] - a[k];
                e2[k] = c[k] - a[k];
            }
            face[0] = e1[1] * e2[2] - e1[2] * e2[1];
            face[1] = e1[2] * e2[0] - e1[0] * e2[2];
            face[2] = e1[0] * e2[1] - e1[1] * e2[0];
            const Real area2 = sqrt(face[0] * face[0] + face[1] * face[1] + face[2] * face[2]);
            if (area2 == Real(0)) {
                degenerate = true;
                continue;
            }
            closest_tri(center, a, b, c, cl);
            for (int k = 0; k < 3; ++k) delta[k] = center[k] - cl[k];
            const Real d = sqrt(delta[0] * delta[0] + delta[1] * delta[1] + delta[2] * delta[2]);
            if (d >= radius) continue;
            Real dot = Real(0);
            for (int k = 0; k < 3; ++k) {
                n[k] = face[k] / area2;
                dot = dot + n[k] * (center[k] - a[k]);
            }
            if (dot < Real(0))
                for (int k = 0; k < 3; ++k) n[k] = -n[k];
            const Real depth = radius - d;
            nhits += 1;
            for (int k = 0; k < 3; ++k) wsum[k] = wsum[k] + depth * n[k];
            if (depth > maxd) {
                maxd = depth;
                for (int k = 0; k < 3; ++k) best[k] = n[k];
            }
        }
    }
    if (nhits == 0) return degenerate;
    const Real norm = sqrt(wsum[0] * wsum[0] + wsum[1] * wsum[1] + wsum[2] * wsum[2]);
    if (norm < Real(1e-12) * (maxd > Real(1.0) ? maxd : Real(1.0))) {
        for (int k = 0; k < 3; ++k) cs.n[k] = best[k];
    } else {
        for (int k = 0; k < 3; ++k) cs.n[k] = wsum[k] / norm;
    }
    maxd = maxd - A.coll_margin;   // the margin inflates detection only
    if (maxd < Real(0)) maxd = Real(0);
    cs.depth = maxd;
    cs.act = true;
    return degenerate;
}

// The same writing the global slot of point p (cnorm, cdepth, cact = 1).
template <typename Real>
__device__ __noinline__ bool mesh_contact(const StepArgs<Real>& A, int64_t p, const Real center[3]) {
    ContactSlot<Real> cs;
    cs.act = false;
    const bool degenerate = mesh_detect(A, p, center, cs);
    if (cs.act) {
        for (int k = 0; k < 3; ++k) A.cnorm[3 * p + k] = cs.n[k];
        A.cdepth[p] = cs.depth;
        A.cact[p] = 1;
    }
    return degenerate;
}

// Normal impulse with accumulator, then box friction, on the velocity v of
// an unlocked point with an active contact (_core.pyx:906-947), slot in
// registers.
template <typename Real>
__device__ __forceinline__ void contact_impulse_r(const StepArgs<Real>& A, Real m, Real v[3], ContactSlot<Real>& cs) {
    Real n[3], vt[3];
    Real vn = Real(0);
    for (int k = 0; k < 3; ++k) {
        n[k] = cs.n[k];
        vn = vn + v[k] * n[k];
    }
    const Real raw = m * ((-vn) * (Real(1.0) + A.restitution) + (A.beta * cs.depth) / A.dt);
    const Real acc = cs.acc_n;
    Real new_acc = acc + raw;
    if (new_acc < Real(0)) new_acc = Real(0);
    const Real applied = new_acc - acc;
    for (int k = 0; k < 3; ++k) v[k] = v[k] + (applied / m) * n[k];
    cs.acc_n = new_acc;
    if (A.mu > Real(0)) {
        Real dot = Real(0), vt_norm = Real(0);
        for (int k = 0; k < 3; ++k) dot = dot + v[k] * n[k];
        for (int k = 0; k < 3; ++k) {
            vt[k] = v[k] - dot * n[k];
            vt_norm = vt_norm + vt[k] * vt[k];
        }
        vt_norm = sqrt(vt_norm);
        Real cap = A.mu * new_acc - cs.acc_t;
        if (cap < Real(0)) cap = Real(0);
        Real jt = m * vt_norm;
        if (jt > cap) jt = cap;
        if (vt_norm > Real(0)) {
            const Real scale = jt / (m * vt_norm);
            for (int k = 0; k < 3; ++k) v[k] = v[k] - scale * vt[k];
        }
        cs.acc_t = cs.acc_t + jt;
    }
}
// ... on point p's global slot
template <typename Real>
__device__ __forceinline__ void contact_impulse(const StepArgs<Real>& A, int64_t p, Real m, Real v[3]) {
    ContactSlot<Real> cs;
    for (int k = 0; k < 3; ++k) cs.n[k] = A.cnorm[3 * p + k];
    cs.depth = A.cdepth[p];
    cs.acc_n = A.cacc_n[p];
    cs.acc_t = A.cacc_t[p];
    cs.act = true;
    contact_impulse_r(A, m, v, cs);
    A.cacc_n[p] = cs.acc_n;
    if (A.mu > Real(0)) A.cacc_t[p] = cs.acc_t;
}

// The impulse on a velocity held in shared memory, out of line: the contact
// phase runs only for scenes with contacts, and inlining it would cost every
// step kernel registers.
template <typename Real>
__device__ __noinline__ void contact_impulse_at(const StepArgs<Real>& A, int64_t p, Real m, Real* vx, Real* vy,
                                                Real* vz) {
    Real v[3] = {*vx, *vy, *vz};
    contact_impulse(A, p, m, v);
    *vx = v[0];
    *vy = v[1];
    *vz = v[2];
}

}  // namespace rsb
