// rod_warp.cuh -- one-warp, register-resident step kernel for single rods of
// 32..63 elements; rod_warp1.cuh is the
// one-point-per-lane form for <= 31 elements.  (A 64-element rod does not
// fit: its last point would be a 65th on 32 x 2 slots, and carrying it as an
// extra point of lane 31 put selects on the colour chains -- measured 3.89
// us/step for cfg1 against 3.80 on the CTA kernel, so 64 stays there.)
//
// A single rod is latency-bound: 23 dependent phases per step, each a short
// fp64 chain.  The CTA kernel (rod_step.cuh) spends a bar.sync and a shared
// memory round trip on every phase.  Here one warp holds the whole rod in
// registers: lane L owns points 2L, 2L+1 and the elements starting there;
// the rod's last point n sits in that grid (lane n/2).  Neighbours come by
// shuffle:
//   * scatter: the upper point / element of slot 1 from lane L+1;
//   * gather: the left element of slot 0 from lane L-1;
//   * colour sweeps: the even element 2L is lane-local (computed once, both
//     halves applied); the odd element 2L+1 spans lanes L and L+1 and BOTH
//     lanes compute it -- identical inputs, identical operations, so the
//     halves are bit-identical to one computation.  A lane's b-side copy
//     holds the element's tangent negated (once per step), which makes its
//     chain the a side's instruction for instruction:
//       (v_a - v_b) . (-n) == (v_b - v_a) . n   term by term, and
//       v_b - (im_b lam)(-n) == v_b + (im_b lam) n,
//     both exact in IEEE arithmetic.  One shuffle round per odd phase, none
//     per even phase, no barrier and no select on the chains (updates of
//     inactive elements are predicated off).
//
// Arithmetic is the reference's expression by expression, shared with the
// batched kernel (rod_batch.cuh).  Speculative only: a rod whose operand
// checks fail is left to the exact CTA kernel (redo list).  The planner
// routes single-rod CTA-tier tasks here (launch-uniform material, no
// drivers, bindings, grabs, contacts).  A world of one such rod launches
// lazily at any epoch length (redo_mode 2): a failed vote writes nothing
// back and stamps the group's redo word, later launches return at once,
// and the host replays the exact kernel at its next synchronisation; a
// batch of them keeps the redo list and its consume launch (epochs of >=
// kSpecMinSteps steps).
#pragma once

#include "rod_warp1.cuh"

namespace rsb {

constexpr int RW_MAX_EL = 63;

template <typename Real, int MODE, bool GEN>
__global__ void __launch_bounds__(32, 1) rod_warp_kernel(const StepArgs<Real> A) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // lazy single-rod launches (redo_mode 2): an earlier launch failed its
    // vote and left its first step in the group's redo word; the host
    // replays the exact kernel from there, this launch does nothing
    if (A.redo_mode == 2 && *reinterpret_cast<volatile int64_t*>(A.hfail)) return;
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = int(threadIdx.x & 31u);
    const int ti = int(blockIdx.x);
    if (ti >= A.ntasks) return;
    const CtaTask task = A.tasks[ti];
    const int p0 = task.p0, e0 = task.e0;
    const int n = task.np - 1;          // elements
    const Real dt = A.dt, beta = A.beta;
    const Real rdt = Real(1.0) / dt;
    const bool dt_ok = in_window(dt);
    const Real grav[3] = {A.gx, A.gy, A.gz};
    const bool l_ok = in_window(A.u.l);
    const bool I_ok = in_window(A.u.I[0]) & in_window(A.u.I[1]) & in_window(A.u.I[2]);
    bool ok = true;

    // ---- load: slots j = 2L + s; pv: the point exists, ev: its element ----
    Real p[2][3], v[2][3], q[2][4], w[2][3], m[2], rm[2], im[2];
    bool pv[2], ev[2], pl[2], flk[2], dist[2], ext[2], m_ok[2];
    int pt[2], el[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const int j = 2 * lane + s;
        pv[s] = j <= n;
        ev[s] = j < n;
        pt[s] = p0 + (pv[s] ? j : 0);
        el[s] = e0 + (ev[s] ? j : 0);
        const uint32_t f = A.pflags[pt[s]];
        pl[s] = (f & SF_PLOCK) != 0;
        flk[s] = (f & SF_FLOCK) != 0;
        dist[s] = (f & SF_DIST) != 0;
        ext[s] = (f & SF_EXT) != 0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            p[s][k] = A.pos[3 * size_t(pt[s]) + k];
            v[s][k] = A.vel[3 * size_t(pt[s]) + k];
            w[s][k] = A.w[3 * size_t(el[s]) + k];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) q[s][k] = A.q[4 * size_t(el[s]) + k];
        m[s] = A.mass[pt[s]];
        rm[s] = rcp_rn(m[s]);   // used only behind m_ok
        im[s] = A.invm[pt[s]];
        m_ok[s] = in_window(m[s]);
    }
    // element statics (_core.pyx:886-900): w_sum of the two inverse masses
    Real imb[2], ws[2], rws[2];
    bool act[2];
    {
        const Real im_n0 = __shfl_down_sync(FULL, im[0], 1);
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            imb[s] = s == 0 ? im[1] : im_n0;
            ws[s] = im[s] + imb[s];
            rws[s] = rcp_rn(ws[s]);   // used only when act
            act[s] = ev[s] && dist[s] && !(ws[s] <= Real(0));
            ok = ok & !(act[s] & !in_window(ws[s]));
        }
    }
    // the odd element to the left (2L-1, lane L-1's slot 1): slot 0 is its b end
    const Real ws_l = __shfl_up_sync(FULL, ws[1], 1), rws_l = __shfl_up_sync(FULL, rws[1], 1);
    const bool act_l = __shfl_up_sync(FULL, act[1], 1) && lane > 0 && pv[0];

    for (int step = 0; step < A.steps; ++step) {
        // ============ scatter (_core.pyx:745-805) ============
        // upper neighbours of slot 1 from lane L+1
        Real pn[3], vn[3], qn1[4], wn1[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            pn[k] = __shfl_down_sync(FULL, p[0][k], 1);
            vn[k] = __shfl_down_sync(FULL, v[0][k], 1);
            wn1[k] = __shfl_down_sync(FULL, w[0][k], 1);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) qn1[k] = __shfl_down_sync(FULL, q[0][k], 1);
        Real ef[2][3], fo[2][4], fn[2][4], jt[2][3], nn[2][3], bias[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            Real vb[3], d[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                vb[k] = s == 0 ? v[1][k] : vn[k];
                d[k] = (s == 0 ? p[1][k] : pn[k]) - p[s][k];
            }
            const Real dd = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
            ok = ok & (!ev[s] | in_window(dd));
            const Real len = sqrt_rn(dd);
            const Real rlen = rcp_rn(len);
            {
                const Real c = len - A.u.l;
                const Real a1[1] = {beta * c};
                Real q1[1];
                const bool bok = bw_div<1>(a1, dt, rdt, dt_ok, q1);
                ok = ok & (!ev[s] | !dist[s] | bok);
                bias[s] = q1[0];
            }
            Real t[3], pair[3], kpl_len;
            {
                const Real num[4] = {d[0], d[1], d[2], A.u.kpl};
                Real quo[4];
                ok = ok & (!ev[s] | bw_div<4>(num, len, rlen, true, quo));
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    t[k] = quo[k];
                    pair[k] = Real(0);
                    nn[s][k] = t[k];
                }
                kpl_len = quo[3];
            }
            if constexpr (GEN) {   // stretch, Eq. 2
                const Real a1[1] = {len};
                Real q1[1];
                const bool vok = bw_div<1>(a1, A.u.l, A.u.il, l_ok, q1);
                ok = ok & (!ev[s] | !ext[s] | vok);
                const Real v3 = q1[0];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const Real g = pair[k] - A.u.ks * (v3 - Real(1.0)) * t[k];
                    pair[k] = ext[s] ? g : pair[k];
                }
            }
            Real d3v[3], er[3], f4[4];
            dir3(q[s], d3v);
#pragma unroll
            for (int k = 0; k < 3; ++k) er[k] = t[k] - d3v[k];
            Real dotp = er[0] * t[0] + er[1] * t[1] + er[2] * t[2];
#pragma unroll
            for (int k = 0; k < 3; ++k) pair[k] = pair[k] - kpl_len * (er[k] - dotp * t[k]);
            dir3_jt(q[s], er, f4);
#pragma unroll
            for (int k = 0; k < 4; ++k) fo[s][k] = A.u.kpl * f4[k];
#pragma unroll
            for (int k = 0; k < 3; ++k) ef[s][k] = -pair[k] + A.u.gt * (vb[k] - v[s][k]);
            // bend / twist (Eq. 5-6): junction j|j+1 inside the rod
            const bool jv = 2 * lane + s + 1 < n;
            Real qb[4], wb[3];
#pragma unroll
            for (int k = 0; k < 4; ++k) qb[k] = s == 0 ? q[1][k] : qn1[k];
#pragma unroll
            for (int k = 0; k < 3; ++k) wb[k] = s == 0 ? w[1][k] : wn1[k];
            dotp = q[s][0] * qb[0] + q[s][1] * qb[1] + q[s][2] * qb[2] + q[s][3] * qb[3];
            const Real sgn = dotp < Real(0) ? Real(-1.0) : Real(1.0);
            const Real il = A.u.il;
            Real qnn[4], qp[4], u[3];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                qnn[k] = sgn * qb[k];
                qp[k] = (qnn[k] - q[s][k]) * il;
            }
            conj_prod_vec(q[s], qp, u);
#pragma unroll
            for (int k = 0; k < 3; ++k) u[k] = u[k] * Real(2.0);
            const Real two_il = Real(2.0) * il;
            const Real mtwo_il = Real(-2.0) * il;
            Real fob[4], fnb[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                fob[k] = fo[s][k];
                fnb[k] = Real(0);
            }
            auto bend = [&](auto kc) {
                constexpr int K = decltype(kc)::value;
                const Real du = u[K] - A.u.us[K];
                const Real coeff = A.u.kb[K] * du * A.u.l;
                Real bp[4], ba[4];
                bform<K>(qp, bp);
                bform<K>(q[s], ba);
                const Real sc = sgn * coeff;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const Real ga = Real(2.0) * bp[i] + two_il * ba[i];
                    const Real gn = mtwo_il * ba[i];
                    fob[i] = fob[i] - coeff * ga;
                    fnb[i] = fnb[i] - sc * gn;
                }
            };
            bend(std::integral_constant<int, 0>{});
            bend(std::integral_constant<int, 1>{});
            bend(std::integral_constant<int, 2>{});
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                fo[s][k] = jv ? fob[k] : fo[s][k];
                fn[s][k] = jv ? fnb[k] : Real(0);
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const Real j3 = A.u.gr * (wb[k] - w[s][k]);
                jt[s][k] = jv ? j3 : Real(0);
            }
        }

        // ============ gather (_core.pyx:808-875) ============
        Real efl[3], fnl[4], jtl[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            efl[k] = __shfl_up_sync(FULL, ef[1][k], 1);
            jtl[k] = __shfl_up_sync(FULL, jt[1][k], 1);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) fnl[k] = __shfl_up_sync(FULL, fn[1][k], 1);
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int j = 2 * lane + s;
            const bool hp = j > 0;
            const Real* e_l = s == 0 ? efl : ef[0];
            const Real* n_l = s == 0 ? fnl : fn[0];
            const Real* j_l = s == 0 ? jtl : jt[0];
            Real f[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                f[k] = m[s] * grav[k];
                f[k] = f[k] + ((GEN && A.has_fext) ? A.fext[3 * size_t(pt[s]) + k] : Real(0));
                const Real g0 = f[k] + ef[s][k];   // the point's own element (not the last point)
                f[k] = ev[s] ? g0 : f[k];
                const Real g = f[k] - e_l[k];
                f[k] = hp ? g : f[k];
            }
            ok = ok & (!pv[s] | (isfinite(f[0]) & isfinite(f[1]) & isfinite(f[2])));
            {
                const Real a[3] = {dt * f[0], dt * f[1], dt * f[2]};
                Real dvv[3];
                const bool dok = bw_div<3>(a, m[s], rm[s], m_ok[s], dvv);
                ok = ok & (!pv[s] | pl[s] | dok);
#pragma unroll
                for (int k = 0; k < 3; ++k) add_if(!pl[s], v[s][k], dvv[k]);
            }
            const bool jp = hp;
            const bool jv = j + 1 < n;
            Real F[4], tau[3], iw[3], gy[3];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const Real g = fo[s][k] + n_l[k];
                F[k] = jp ? g : fo[s][k];
            }
            const Real dot = F[0] * q[s][0] + F[1] * q[s][1] + F[2] * q[s][2] + F[3] * q[s][3];
#pragma unroll
            for (int k = 0; k < 4; ++k) F[k] = F[k] - dot * q[s][k];
            conj_prod_vec(q[s], F, tau);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                tau[k] = tau[k] * Real(0.5);
                const Real g = tau[k] + jt[s][k];
                tau[k] = jv ? g : tau[k];
                const Real g2 = tau[k] - j_l[k];
                tau[k] = jp ? g2 : tau[k];
            }
            ok = ok & (!ev[s] | (isfinite(tau[0]) & isfinite(tau[1]) & isfinite(tau[2])));
#pragma unroll
            for (int k = 0; k < 3; ++k) iw[k] = A.u.I[k] * w[s][k];
            gy[0] = w[s][1] * iw[2] - w[s][2] * iw[1];
            gy[1] = w[s][2] * iw[0] - w[s][0] * iw[2];
            gy[2] = w[s][0] * iw[1] - w[s][1] * iw[0];
            {
                const Real a[3] = {dt * (tau[0] - gy[0]), dt * (tau[1] - gy[1]), dt * (tau[2] - gy[2])};
                bool dok = I_ok;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const Real dw = bw_quot(a[k], A.u.I[k], A.u.rI[k]);
                    dok = dok & dividend_ok(a[k]);
                    add_if(!flk[s], w[s][k], dw);
                }
                ok = ok & (!ev[s] | flk[s] | dok);
            }
        }
        // ============ constraint iterations (_core.pyx:1069-1076) ============
        // slot 0 as the b end of element 2L-1: its tangent (negated) and bias
        Real nl[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) nl[k] = -__shfl_up_sync(FULL, nn[1][k], 1);
        const Real bias_l = __shfl_up_sync(FULL, bias[1], 1);
        auto lam_of = [&](const Real (&dv)[3], const Real (&nv)[3], Real bs, Real wsv, Real rwsv, bool ac) -> Real {
            Real x = dv[0] * nv[0];
            x = x + dv[1] * nv[1];
            x = x + dv[2] * nv[2];
            x = x + bs;
            const Real q0 = (-x) * rwsv;
            Real lam = fma(fma(-q0, wsv, -x), rwsv, q0);
            const bool z = is_zero(x);
            if (z) lam = Real(-0.0);
            ok = ok & !(ac & !(in_window(x) | z));
            return lam;
        };
        for (int it = A.iters; it > 0; --it) {
            {   // even: element 2L, slot 0 -> slot 1 in the lane
                Real dv[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) dv[k] = v[1][k] - v[0][k];
                const Real lam = lam_of(dv, nn[0], bias[0], ws[0], rws[0], act[0]);
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    sub_if(act[0], v[0][k], im[0] * lam * nn[0][k]);
                    add_if(act[0], v[1][k], imb[0] * lam * nn[0][k]);
                }
            }
            {   // odd: element 2L+1 (slot 1, a end) and element 2L-1 (slot 0, b end)
                Real d1[3], d0[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    d1[k] = __shfl_down_sync(FULL, v[0][k], 1) - v[1][k];
                    d0[k] = __shfl_up_sync(FULL, v[1][k], 1) - v[0][k];
                }
                const Real lam1 = lam_of(d1, nn[1], bias[1], ws[1], rws[1], act[1]);
                const Real lam0 = lam_of(d0, nl, bias_l, ws_l, rws_l, act_l);
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    sub_if(act[1], v[1][k], im[1] * lam1 * nn[1][k]);
                    sub_if(act_l, v[0][k], im[0] * lam0 * nl[k]);
                }
            }
        }

        // ================= integrate (_core.pyx:1023-1042) =================
#pragma unroll
        for (int s = 0; s < 2; ++s) {
#pragma unroll
            for (int k = 0; k < 3; ++k) p[s][k] = p[s][k] + dt * v[s][k];
            Real dq[4];
            const Real om[4] = {Real(0.0), w[s][0], w[s][1], w[s][2]};
            hprod(q[s], om, dq);
            const Real h = dt * Real(0.5);
            Real qq4[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) qq4[k] = q[s][k] + h * dq[k];
            const Real qq = qq4[0] * qq4[0] + qq4[1] * qq4[1] + qq4[2] * qq4[2] + qq4[3] * qq4[3];
            ok = ok & (!ev[s] | in_window(qq));
            const Real nrm = sqrt_rn(qq);
            const Real rn = rcp_rn(nrm);
            Real qn[4];
            ok = ok & (!ev[s] | bw_div<4>(qq4, nrm, rn, true, qn));
#pragma unroll
            for (int k = 0; k < 4; ++k) q[s][k] = qn[k];
        }
    }

    // ---- write back, or leave the rod to the exact kernel ----
    if (__any_sync(FULL, !ok)) {
        if (lane == 0) {
            if (A.redo_mode == 2) *A.hfail = A.step0 + 1;   // lazy: nothing written back
            else A.redo_list[atomicAdd(A.redo_count, 1)] = ti;
        }
        return;
    }
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        if (pv[s]) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                A.pos[3 * size_t(pt[s]) + k] = p[s][k];
                A.vel[3 * size_t(pt[s]) + k] = v[s][k];
            }
        }
        if (ev[s]) {
#pragma unroll
            for (int k = 0; k < 3; ++k) A.w[3 * size_t(el[s]) + k] = w[s][k];
#pragma unroll
            for (int k = 0; k < 4; ++k) A.q[4 * size_t(el[s]) + k] = q[s][k];
        }
    }
}

}  // namespace rsb
