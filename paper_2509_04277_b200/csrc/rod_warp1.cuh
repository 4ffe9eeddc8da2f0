// rod_warp1.cuh -- one-warp, one-point-per-lane step kernel for single rods
// of <= 31 elements (the small end of the cfg4 sweep).
//
// Lane L owns point L and element L (points L, L+1); lane n owns the rod's
// last point.  Everything is in registers; neighbours come by shuffle.  In
// each colour phase every lane moves its own point: the lane whose element
// has the phase's parity is that element's lower end (a), the other lane of
// the pair its upper end (b), and both compute the element's impulse from the
// same inputs with the same operations, so the two halves are bit-identical
// to one computation.  The roles differ only in the sign of the tangent the
// lane holds for the phase (n on the a side, -n on the b side, negated once
// per step), and that sign carries through exactly:
//   (v_partner - v_own) . (+-n) == (v_b - v_a) . n     term by term (IEEE
//                                                      subtraction and
//                                                      negation are exact)
//   v_own - (im_own lam)(+-n) == v_a - (im_a lam) n  /  v_b + (im_b lam) n
// so both lanes run the identical instruction stream, with no select and no
// sign flip on the dependency chain.  Per-phase element constants (tangent,
// bias, w_sum) are formed once per step: a colour phase is one shuffle round
// and one dependency chain.
//
// Arithmetic as in rod_batch.cuh / rod_warp.cuh (the reference's expression
// order); speculative only, exact CTA kernel over the redo list otherwise
// (a single rod: lazily, through the group's redo word -- rod_warp.cuh).
#pragma once

#include "rod_batch.cuh"

namespace rsb {

constexpr int RW1_MAX_EL = 31;

// v += t under a predicate, as one predicated instruction (no select)
__device__ __forceinline__ void add_if(bool p, double& v, double t) {
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q add.rn.f64 %0, %0, %1;\n\t}" : "+d"(v) : "d"(t), "r"(int(p)));
}
__device__ __forceinline__ void add_if(bool p, float& v, float t) {
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q add.rn.f32 %0, %0, %1;\n\t}" : "+f"(v) : "f"(t), "r"(int(p)));
}
// v -= t under a predicate
__device__ __forceinline__ void sub_if(bool p, double& v, double t) {
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q sub.rn.f64 %0, %0, %1;\n\t}" : "+d"(v) : "d"(t), "r"(int(p)));
}
__device__ __forceinline__ void sub_if(bool p, float& v, float t) {
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q sub.rn.f32 %0, %0, %1;\n\t}" : "+f"(v) : "f"(t), "r"(int(p)));
}

template <typename Real, int MODE, bool GEN>
__global__ void __launch_bounds__(32, 1) rod_warp1_kernel(const StepArgs<Real> A) {
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
    const int n = task.np - 1;          // elements; points 0..n on lanes 0..n
    const bool pv = lane <= n;          // lane holds a point
    const bool ev = lane < n;           // ... and an element
    const Real dt = A.dt, beta = A.beta;
    const Real rdt = Real(1.0) / dt;
    const bool dt_ok = in_window(dt);
    const Real grav[3] = {A.gx, A.gy, A.gz};
    const bool l_ok = in_window(A.u.l);
    const bool I_ok = in_window(A.u.I[0]) & in_window(A.u.I[1]) & in_window(A.u.I[2]);
    bool ok = true;

    // ---- load (lanes past the rod read point 0 / element 0) ----
    const int pt = p0 + (pv ? lane : 0), el = e0 + (ev ? lane : 0);
    Real p[3], v[3], q[4], w[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        p[k] = A.pos[3 * size_t(pt) + k];
        v[k] = A.vel[3 * size_t(pt) + k];
        w[k] = A.w[3 * size_t(el) + k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = A.q[4 * size_t(el) + k];
    const uint32_t fl = A.pflags[pt];
    const bool pl = (fl & SF_PLOCK) != 0, flk = (fl & SF_FLOCK) != 0;
    const bool dist = (fl & SF_DIST) != 0, ext = (fl & SF_EXT) != 0;
    const Real m = A.mass[pt], rm = rcp_rn(m), im = A.invm[pt];
    const bool m_ok = in_window(m);
    // element statics: w_sum = im_a + im_b (_core.pyx:886-900)
    const Real im_up = __shfl_down_sync(FULL, im, 1);
    const Real ws = im + im_up;
    const Real rws = rcp_rn(ws);   // used only when act
    const bool act = ev && dist && !(ws <= Real(0));
    ok = ok & !(act & !in_window(ws));
    // per colour phase c: the element this lane's point takes part in (its
    // own, lower end, when lane % 2 == c; the left one, upper end,
    // otherwise), that element's w_sum / 1/w_sum / activity, the point's
    // own inverse mass, and the partner lane across the element
    const bool a_side[2] = {(lane & 1) == 0, (lane & 1) == 1};
    const int partner[2] = {lane ^ 1, (lane & 1) ? lane + 1 : lane - 1};
    const Real ws_l = __shfl_up_sync(FULL, ws, 1), rws_l = __shfl_up_sync(FULL, rws, 1);
    const bool act_l = __shfl_up_sync(FULL, act, 1) && lane > 0;
    Real wsP[2], rwsP[2];
    bool actP[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        wsP[c] = a_side[c] ? ws : ws_l;
        rwsP[c] = a_side[c] ? rws : rws_l;
        actP[c] = (a_side[c] ? act : act_l) && pv;
    }

    for (int step = 0; step < A.steps; ++step) {
        // ============ scatter (_core.pyx:745-805): element L ============
        Real pb[3], vb[3], qb[4], wb[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            pb[k] = __shfl_down_sync(FULL, p[k], 1);
            vb[k] = __shfl_down_sync(FULL, v[k], 1);
            wb[k] = __shfl_down_sync(FULL, w[k], 1);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) qb[k] = __shfl_down_sync(FULL, q[k], 1);
        Real d[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) d[k] = pb[k] - p[k];
        const Real dd = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
        ok = ok & (!ev | in_window(dd));
        const Real len = sqrt_rn(dd);
        const Real rlen = rcp_rn(len);
        Real nn[3], bias;
        {
            const Real c = len - A.u.l;
            const Real a1[1] = {beta * c};
            Real q1[1];
            const bool bok = bw_div<1>(a1, dt, rdt, dt_ok, q1);
            ok = ok & (!ev | !dist | bok);
            bias = q1[0];
        }
        Real t[3], pair[3], kpl_len;
        {
            const Real num[4] = {d[0], d[1], d[2], A.u.kpl};
            Real quo[4];
            ok = ok & (!ev | bw_div<4>(num, len, rlen, true, quo));
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                t[k] = quo[k];
                pair[k] = Real(0);
                nn[k] = t[k];
            }
            kpl_len = quo[3];
        }
        if constexpr (GEN) {   // stretch, Eq. 2
            const Real a1[1] = {len};
            Real q1[1];
            const bool vok = bw_div<1>(a1, A.u.l, A.u.il, l_ok, q1);
            ok = ok & (!ev | !ext | vok);
            const Real v3 = q1[0];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const Real g = pair[k] - A.u.ks * (v3 - Real(1.0)) * t[k];
                pair[k] = ext ? g : pair[k];
            }
        }
        Real d3v[3], er[3], f4[4], fo[4], fn[4], ef[3], jt[3];
        dir3(q, d3v);
#pragma unroll
        for (int k = 0; k < 3; ++k) er[k] = t[k] - d3v[k];
        Real dotp = er[0] * t[0] + er[1] * t[1] + er[2] * t[2];
#pragma unroll
        for (int k = 0; k < 3; ++k) pair[k] = pair[k] - kpl_len * (er[k] - dotp * t[k]);
        dir3_jt(q, er, f4);
#pragma unroll
        for (int k = 0; k < 4; ++k) fo[k] = A.u.kpl * f4[k];
#pragma unroll
        for (int k = 0; k < 3; ++k) ef[k] = -pair[k] + A.u.gt * (vb[k] - v[k]);
        const bool jv = lane + 1 < n;   // junction L|L+1 inside the rod
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
                fo[k] = jv ? fob[k] : fo[k];
                fn[k] = jv ? fnb[k] : Real(0);
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const Real j3 = A.u.gr * (wb[k] - w[k]);
                jt[k] = jv ? j3 : Real(0);
            }
        }

        // ============ gather (_core.pyx:808-875): point L, frame L ============
        Real efl[3], fnl[4], jtl[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            efl[k] = __shfl_up_sync(FULL, ef[k], 1);
            jtl[k] = __shfl_up_sync(FULL, jt[k], 1);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) fnl[k] = __shfl_up_sync(FULL, fn[k], 1);
        {
            const bool hp = lane > 0;
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
            ok = ok & (!pv | (isfinite(f[0]) & isfinite(f[1]) & isfinite(f[2])));
            const Real a[3] = {dt * f[0], dt * f[1], dt * f[2]};
            Real dvv[3];
            const bool dok = bw_div<3>(a, m, rm, m_ok, dvv);
            ok = ok & (!pv | pl | dok);
#pragma unroll
            for (int k = 0; k < 3; ++k) add_if(!pl, v[k], dvv[k]);
        }
        {   // frame L
            const bool jp = lane > 0;
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
            ok = ok & (!ev | (isfinite(tau[0]) & isfinite(tau[1]) & isfinite(tau[2])));
#pragma unroll
            for (int k = 0; k < 3; ++k) iw[k] = A.u.I[k] * w[k];
            gy[0] = w[1] * iw[2] - w[2] * iw[1];
            gy[1] = w[2] * iw[0] - w[0] * iw[2];
            gy[2] = w[0] * iw[1] - w[1] * iw[0];
            const Real a[3] = {dt * (tau[0] - gy[0]), dt * (tau[1] - gy[1]), dt * (tau[2] - gy[2])};
            bool dok = I_ok;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const Real dw = bw_quot(a[k], A.u.I[k], A.u.rI[k]);
                dok = dok & dividend_ok(a[k]);
                add_if(!flk, w[k], dw);
            }
            ok = ok & (!ev | flk | dok);
        }

        // ============ constraint iterations (_core.pyx:1069-1076) ============
        // per phase: the element's tangent and bias (own, or the left one)
        const Real nn_l[3] = {__shfl_up_sync(FULL, nn[0], 1), __shfl_up_sync(FULL, nn[1], 1),
                              __shfl_up_sync(FULL, nn[2], 1)};
        const Real bias_l = __shfl_up_sync(FULL, bias, 1);
        Real nP[2][3], bP[2];   // the phase's element tangent, negated on the b side
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            bP[c] = a_side[c] ? bias : bias_l;
#pragma unroll
            for (int k = 0; k < 3; ++k) nP[c][k] = a_side[c] ? nn[k] : -nn_l[k];
        }
        for (int it = A.iters; it > 0; --it) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                Real dv[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) dv[k] = __shfl_sync(FULL, v[k], partner[c]) - v[k];
                Real x = dv[0] * nP[c][0];
                x = x + dv[1] * nP[c][1];
                x = x + dv[2] * nP[c][2];
                x = x + bP[c];
                const Real q0 = (-x) * rwsP[c];
                Real lam = fma(fma(-q0, wsP[c], -x), rwsP[c], q0);
                const bool z = is_zero(x);
                if (z) lam = Real(-0.0);
                ok = ok & !(actP[c] & !(in_window(x) | z));
#pragma unroll
                for (int k = 0; k < 3; ++k) sub_if(actP[c], v[k], im * lam * nP[c][k]);
            }
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
            ok = ok & (!ev | in_window(qq));
            const Real nrm = sqrt_rn(qq);
            const Real rn = rcp_rn(nrm);
            Real qn[4];
            ok = ok & (!ev | bw_div<4>(qq4, nrm, rn, true, qn));
#pragma unroll
            for (int k = 0; k < 4; ++k) q[k] = qn[k];
        }
    }

    if (__any_sync(FULL, !ok)) {
        if (lane == 0) {
            if (A.redo_mode == 2) *A.hfail = A.step0 + 1;   // lazy: nothing written back
            else A.redo_list[atomicAdd(A.redo_count, 1)] = ti;
        }
        return;
    }
    if (pv) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            A.pos[3 * size_t(pt) + k] = p[k];
            A.vel[3 * size_t(pt) + k] = v[k];
        }
    }
    if (ev) {
#pragma unroll
        for (int k = 0; k < 3; ++k) A.w[3 * size_t(el) + k] = w[k];
#pragma unroll
        for (int k = 0; k < 4; ++k) A.q[4 * size_t(el) + k] = q[k];
    }
}

}  // namespace rsb
