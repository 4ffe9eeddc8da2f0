/*
 * rod_oracle.c -- CPU restatement of the reference CoRdE step.
 *
 * TEST INFRASTRUCTURE ONLY: used by tests/ as the parity checker and by
 * bench.py as the CPU baseline ("port").  Never linked into the product.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement bit-for-bit
 * against (a) the committed golden fixtures in tests/golden/ produced by the
 * reference package itself (tests/golden/make_golden.py) and (b) the
 * reference's own compiled core built from /root/reference into oracle/_ref/
 * by oracle/build_ref.sh, when that build is present.
 *
 * Build with plain IEEE double arithmetic and no contraction
 * (-ffp-contract=off, no -march): the reference core is compiled without FMA
 * (pkg/setup.py:11), and every expression below keeps the reference's
 * operation order (left-to-right sums, explicit divisions, sqrt).
 *
 * Phase semantics (per step, _core.pyx:1058-1080):
 *   scatter -> gather(+drivers) -> iters x [distance even, distance odd,
 *   (contacts: none in scope), central: bindings then grabs] -> integrate.
 */
#include "rod_oracle.h"

#include <math.h>
#include <stddef.h>

/* ---- quaternion helpers (_core.pyx:409-447; quat.py:12-119) ------------ */

/* Hamilton product o = a*b, scalar first. */
static void hprod(const double *a, const double *b, double *o)
{
    o[0] = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
    o[1] = a[0] * b[1] + b[0] * a[1] + a[2] * b[3] - a[3] * b[2];
    o[2] = a[0] * b[2] + b[0] * a[2] + a[3] * b[1] - a[1] * b[3];
    o[3] = a[0] * b[3] + b[0] * a[3] + a[1] * b[2] - a[2] * b[1];
}

/* vector part of conj(a)*b */
static void conj_prod_vec(const double *a, const double *b, double *v)
{
    double c[4] = {a[0], -a[1], -a[2], -a[3]};
    double t[4];
    hprod(c, b, t);
    v[0] = t[1];
    v[1] = t[2];
    v[2] = t[3];
}

/* B_k x for the three skew bilinear strain forms (quat.py:98-119) */
static void bform(int k, const double *x, double *o)
{
    if (k == 0) {
        o[0] = x[1]; o[1] = -x[0]; o[2] = -x[3]; o[3] = x[2];
    } else if (k == 1) {
        o[0] = x[2]; o[1] = x[3]; o[2] = -x[0]; o[3] = -x[1];
    } else {
        o[0] = x[3]; o[1] = -x[2]; o[2] = x[1]; o[3] = -x[0];
    }
}

/* third director, unnormalised polynomial form (quat.py:54-66) */
static void dir3(const double *q, double *d)
{
    d[0] = 2.0 * (q[1] * q[3] + q[0] * q[2]);
    d[1] = 2.0 * (q[2] * q[3] - q[0] * q[1]);
    d[2] = 1.0 - 2.0 * (q[1] * q[1] + q[2] * q[2]);
}

/* J(q)^T r with J = d dir3 / d q (quat.py:69-83) */
static void dir3_jt(const double *q, const double *r, double *o)
{
    const double qw = q[0], qx = q[1], qy = q[2], qz = q[3];
    o[0] = 2.0 * qy * r[0] - 2.0 * qx * r[1];
    o[1] = 2.0 * qz * r[0] - 2.0 * qw * r[1] - 4.0 * qx * r[2];
    o[2] = 2.0 * qw * r[0] + 2.0 * qz * r[1] - 4.0 * qy * r[2];
    o[3] = 2.0 * qx * r[0] + 2.0 * qy * r[1];
}

static double norm3(const double *d)
{
    return sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
}

void ro_prepare(ro_world *w)
{
    for (int64_t p = 0; p < w->P; ++p) {
        w->pt_elo[p] = -1;
        w->pt_ehi[p] = -1;
    }
    for (int64_t e = 0; e < w->E; ++e) {
        int64_t p = w->elem_point[e];
        w->pt_elo[p] = e;
        w->pt_ehi[p + 1] = e;
    }
}

/* ---- element / junction scatter (_core.pyx:745-805; Eq. 2-8) ----------- */

static void scatter_element(ro_world *w, int64_t e)
{
    const int64_t pa = w->elem_point[e], pb = pa + 1;
    const double l = w->rest[e];
    double *ef = w->ef + 3 * e, *fo = w->ff_own + 4 * e, *fn = w->ff_next + 4 * e;
    double d[3], t[3], pair[3], d3v[3], err[3], f4[4];

    for (int k = 0; k < 3; ++k)
        d[k] = w->pos[3 * pb + k] - w->pos[3 * pa + k];
    const double len = norm3(d);
    if (len == 0.0) {                       /* degenerate segment */
        w->err_step = w->step;
        for (int k = 0; k < 3; ++k) ef[k] = 0.0;
        for (int k = 0; k < 4; ++k) { fo[k] = 0.0; fn[k] = 0.0; }
        return;                             /* jtau left untouched */
    }
    for (int k = 0; k < 3; ++k) {
        t[k] = d[k] / len;
        pair[k] = 0.0;
    }
    if (w->ext[e] != 0.0) {                 /* stretch, Eq. 2 */
        const double v3 = len / l;
        for (int k = 0; k < 3; ++k)
            pair[k] = pair[k] - w->ks[e] * (v3 - 1.0) * t[k];
    }
    /* quaternion-tangent penalty (Eq. 7-8) */
    const double *qa = w->q + 4 * e;
    dir3(qa, d3v);
    for (int k = 0; k < 3; ++k) err[k] = t[k] - d3v[k];
    double dotp = err[0] * t[0] + err[1] * t[1] + err[2] * t[2];
    for (int k = 0; k < 3; ++k)
        pair[k] = pair[k] - (w->kp[e] * l / len) * (err[k] - dotp * t[k]);
    dir3_jt(qa, err, f4);
    for (int k = 0; k < 4; ++k) {
        fo[k] = w->kp[e] * l * f4[k];
        fn[k] = 0.0;
    }
    for (int k = 0; k < 3; ++k)
        ef[k] = -pair[k] + w->gt[e] * (w->vel[3 * pb + k] - w->vel[3 * pa + k]);

    if (!w->jvalid[e])
        return;
    /* bend/twist across junction e|e+1 from the Darboux vector (Eq. 5-6) */
    const double *qb = w->q + 4 * (e + 1);
    dotp = qa[0] * qb[0] + qa[1] * qb[1] + qa[2] * qb[2] + qa[3] * qb[3];
    const double sgn = dotp < 0.0 ? -1.0 : 1.0;
    const double il = 1.0 / l;
    double qn[4], qp[4], u[3], bp[4], ba[4];
    for (int k = 0; k < 4; ++k) {
        qn[k] = sgn * qb[k];
        qp[k] = (qn[k] - qa[k]) * il;
    }
    conj_prod_vec(qa, qp, u);
    for (int k = 0; k < 3; ++k) u[k] = u[k] * 2.0;
    for (int k = 0; k < 3; ++k) {
        const double du = u[k] - w->ustar[3 * e + k];
        const double coeff = w->kb[3 * e + k] * du * l;
        bform(k, qp, bp);
        bform(k, qa, ba);
        double ga[4], gn[4];
        for (int i = 0; i < 4; ++i) {
            ga[i] = 2.0 * bp[i] + 2.0 * il * ba[i];
            gn[i] = -2.0 * il * ba[i];
        }
        for (int i = 0; i < 4; ++i) {
            fo[i] = fo[i] - coeff * ga[i];
            fn[i] = fn[i] - sgn * coeff * gn[i];
        }
    }
    for (int k = 0; k < 3; ++k)
        w->jtau[3 * e + k] = w->gr[e] * (w->w[3 * (e + 1) + k] - w->w[3 * e + k]);
}

void ro_scatter(ro_world *w)
{
    for (int64_t e = 0; e < w->E; ++e)
        scatter_element(w, e);
}

/* ---- point / frame gather and velocity update (_core.pyx:808-875) ----- */

void ro_gather(ro_world *w)
{
    const double g[3] = {w->gx, w->gy, w->gz};
    for (int64_t i = 0; i < w->P; ++i) {
        double f[3];
        for (int k = 0; k < 3; ++k) {
            f[k] = w->mass[i] * g[k];
            f[k] = f[k] + w->fext[3 * i + k];
        }
        int64_t e = w->pt_elo[i];
        if (e >= 0)
            for (int k = 0; k < 3; ++k) f[k] = f[k] + w->ef[3 * e + k];
        e = w->pt_ehi[i];
        if (e >= 0)
            for (int k = 0; k < 3; ++k) f[k] = f[k] - w->ef[3 * e + k];
        if (!(isfinite(f[0]) && isfinite(f[1]) && isfinite(f[2])))
            w->err_step = w->step;
        if (!w->plock[i])
            for (int k = 0; k < 3; ++k)
                w->vel[3 * i + k] = w->vel[3 * i + k] + w->dt * f[k] / w->mass[i];
    }
    for (int64_t e = 0; e < w->E; ++e) {
        const double *q = w->q + 4 * e;
        double *om = w->w + 3 * e;
        const int prev = e > 0 && w->jvalid[e - 1];
        double F[4], tau[3], iw[3], gy[3];
        for (int k = 0; k < 4; ++k) F[k] = w->ff_own[4 * e + k];
        if (prev)
            for (int k = 0; k < 4; ++k) F[k] = F[k] + w->ff_next[4 * (e - 1) + k];
        const double dot = F[0] * q[0] + F[1] * q[1] + F[2] * q[2] + F[3] * q[3];
        for (int k = 0; k < 4; ++k) F[k] = F[k] - dot * q[k];
        conj_prod_vec(q, F, tau);
        for (int k = 0; k < 3; ++k) tau[k] = tau[k] * 0.5;
        if (w->jvalid[e])
            for (int k = 0; k < 3; ++k) tau[k] = tau[k] + w->jtau[3 * e + k];
        if (prev)
            for (int k = 0; k < 3; ++k) tau[k] = tau[k] - w->jtau[3 * (e - 1) + k];
        if (!(isfinite(tau[0]) && isfinite(tau[1]) && isfinite(tau[2])))
            w->err_step = w->step;
        for (int k = 0; k < 3; ++k) iw[k] = w->inert[3 * e + k] * om[k];
        gy[0] = om[1] * iw[2] - om[2] * iw[1];
        gy[1] = om[2] * iw[0] - om[0] * iw[2];
        gy[2] = om[0] * iw[1] - om[1] * iw[0];
        if (!w->flock[e])
            for (int k = 0; k < 3; ++k)
                om[k] = om[k] + w->dt * (tau[k] - gy[k]) / w->inert[3 * e + k];
    }
    /* drivers overwrite after the update, rod order (_core.pyx:866-875) */
    for (int64_t r = 0; r < w->R; ++r) {
        const int64_t p = w->drv_pt[r];
        if (p >= 0)
            for (int k = 0; k < 3; ++k) w->vel[3 * p + k] = w->drv_v[3 * r + k];
        const int64_t e = w->drv_fr[r];
        if (e >= 0) {
            w->w[3 * e] = 0.0;
            w->w[3 * e + 1] = 0.0;
            w->w[3 * e + 2] = w->drv_rot[r];
        }
    }
}

/* ---- inextensibility: red/black distance impulses (_core.pyx:878-903) - */

void ro_distance(ro_world *w, int64_t parity)
{
    for (int64_t e = 0; e < w->E; ++e) {
        if (w->elem_parity[e] != parity || w->ext[e] != 0.0)
            continue;
        const int64_t a = w->elem_point[e], b = a + 1;
        double d[3], n[3];
        for (int k = 0; k < 3; ++k) d[k] = w->pos[3 * b + k] - w->pos[3 * a + k];
        const double dist = norm3(d);
        const double wsum = w->invm[a] + w->invm[b];
        if (dist <= 0.0 || wsum <= 0.0)
            continue;
        for (int k = 0; k < 3; ++k) n[k] = d[k] / dist;
        const double c = dist - w->rest[e];
        double vrel = 0.0;
        for (int k = 0; k < 3; ++k)
            vrel = vrel + (w->vel[3 * b + k] - w->vel[3 * a + k]) * n[k];
        const double lam = -(vrel + w->beta * c / w->dt) / wsum;
        for (int k = 0; k < 3; ++k) {
            w->vel[3 * a + k] = w->vel[3 * a + k] - w->invm[a] * lam * n[k];
            w->vel[3 * b + k] = w->vel[3 * b + k] + w->invm[b] * lam * n[k];
        }
    }
}

/* ---- rod-rod bindings, then grab anchors (_core.pyx:981-1020) --------- */

void ro_central(ro_world *w)
{
    for (int64_t k = 0; k < w->nbind; ++k) {
        const int64_t a = w->bind_a[k], b = w->bind_b[k];
        const double wa = w->bind_mode[k] == 0 ? 0.0 : w->invm[a];
        const double wb = w->invm[b];
        double d[3], n[3];
        for (int i = 0; i < 3; ++i) d[i] = w->pos[3 * b + i] - w->pos[3 * a + i];
        const double dist = norm3(d);
        const double wsum = wa + wb;
        if (dist == 0.0 || wsum == 0.0)
            continue;
        double vrel = 0.0;
        for (int i = 0; i < 3; ++i) {
            n[i] = d[i] / dist;
            vrel = vrel + (w->vel[3 * b + i] - w->vel[3 * a + i]) * n[i];
        }
        const double lam = -(vrel + w->beta * dist / w->dt) / wsum;
        if (wa > 0.0)
            for (int i = 0; i < 3; ++i)
                w->vel[3 * a + i] = w->vel[3 * a + i] - wa * lam * n[i];
        for (int i = 0; i < 3; ++i)
            w->vel[3 * b + i] = w->vel[3 * b + i] + wb * lam * n[i];
    }
    for (int64_t k = 0; k < w->ngrab; ++k) {
        if (!w->g_act[k])
            continue;
        const int64_t b = w->g_pt[k];
        const double wb = w->invm[b];
        if (wb == 0.0)
            continue;
        double d[3], n[3];
        for (int i = 0; i < 3; ++i) d[i] = w->pos[3 * b + i] - w->g_tgt[3 * k + i];
        const double dist = norm3(d);
        if (dist == 0.0)
            continue;
        double vrel = 0.0;
        for (int i = 0; i < 3; ++i) {
            n[i] = d[i] / dist;
            vrel = vrel + w->vel[3 * b + i] * n[i];
        }
        const double lam = -(vrel + w->beta * dist / w->dt) / wb;
        for (int i = 0; i < 3; ++i)
            w->vel[3 * b + i] = w->vel[3 * b + i] + wb * lam * n[i];
    }
}

/* ---- explicit position / orientation update (_core.pyx:1023-1042) ----- */

void ro_integrate(ro_world *w)
{
    for (int64_t i = 0; i < 3 * w->P; ++i)
        w->pos[i] = w->pos[i] + w->dt * w->vel[i];
    for (int64_t e = 0; e < w->E; ++e) {
        double *q = w->q + 4 * e;
        const double om[4] = {0.0, w->w[3 * e], w->w[3 * e + 1], w->w[3 * e + 2]};
        double dq[4];
        hprod(q, om, dq);
        for (int k = 0; k < 4; ++k) q[k] = q[k] + w->dt * 0.5 * dq[k];
        const double nrm = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        for (int k = 0; k < 4; ++k) q[k] = q[k] / nrm;
    }
}

void ro_run(ro_world *w, int64_t steps)
{
    for (int64_t s = 0; s < steps; ++s) {
        ro_scatter(w);
        ro_gather(w);
        for (int64_t it = 0; it < w->iters; ++it) {
            ro_distance(w, 0);
            ro_distance(w, 1);
            ro_central(w);
        }
        ro_integrate(w);
        w->step += 1;
    }
}
