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

/* ---- mesh contacts: detection (_core.pyx:509-662) ----------------------- */

#define RO_STACK_CAP 32

/* Ericson's closest point of triangle abc to p (_core.pyx:509-559) */
static void closest_tri(const double *p, const double *a, const double *b, const double *c,
                        double *out)
{
    double ab[3], ac[3], ap[3], bp[3], cp[3];
    for (int k = 0; k < 3; ++k) {
        ab[k] = b[k] - a[k];
        ac[k] = c[k] - a[k];
        ap[k] = p[k] - a[k];
    }
    const double d1 = ab[0] * ap[0] + ab[1] * ap[1] + ab[2] * ap[2];
    const double d2 = ac[0] * ap[0] + ac[1] * ap[1] + ac[2] * ap[2];
    if (d1 <= 0.0 && d2 <= 0.0) {
        for (int k = 0; k < 3; ++k) out[k] = a[k];
        return;
    }
    for (int k = 0; k < 3; ++k) bp[k] = p[k] - b[k];
    const double d3 = ab[0] * bp[0] + ab[1] * bp[1] + ab[2] * bp[2];
    const double d4 = ac[0] * bp[0] + ac[1] * bp[1] + ac[2] * bp[2];
    if (d3 >= 0.0 && d4 <= d3) {
        for (int k = 0; k < 3; ++k) out[k] = b[k];
        return;
    }
    const double vc = d1 * d4 - d3 * d2;
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
        const double t = d1 / (d1 - d3);
        for (int k = 0; k < 3; ++k) out[k] = a[k] + t * ab[k];
        return;
    }
    for (int k = 0; k < 3; ++k) cp[k] = p[k] - c[k];
    const double d5 = ab[0] * cp[0] + ab[1] * cp[1] + ab[2] * cp[2];
    const double d6 = ac[0] * cp[0] + ac[1] * cp[1] + ac[2] * cp[2];
    if (d6 >= 0.0 && d5 <= d6) {
        for (int k = 0; k < 3; ++k) out[k] = c[k];
        return;
    }
    const double vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
        const double t = d2 / (d2 - d6);
        for (int k = 0; k < 3; ++k) out[k] = a[k] + t * ac[k];
        return;
    }
    const double va = d3 * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
        const double t = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        for (int k = 0; k < 3; ++k) out[k] = b[k] + t * (c[k] - b[k]);
        return;
    }
    const double denom = 1.0 / (va + vb + vc);
    for (int k = 0; k < 3; ++k) out[k] = a[k] + ab[k] * (vb * denom) + ac[k] * (vc * denom);
}

/* broad + narrow phase + aggregation for the sphere of point i */
static void mesh_contact(ro_world *w, int64_t i)
{
    int64_t stack[RO_STACK_CAP];
    const double *center = w->pos + 3 * i;
    const double radius = w->cradii[i] + w->coll_margin;
    double lo[3], hi[3], wsum[3] = {0.0, 0.0, 0.0}, best_n[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < 3; ++k) {
        lo[k] = center[k] - radius;
        hi[k] = center[k] + radius;
    }
    int64_t nhits = 0, top = 1;
    double maxd = -1.0;
    stack[0] = 0;
    while (top) {
        const int64_t node = stack[--top];
        if (node >= w->n_nodes || w->ncount[node] < 0)
            continue;
        const double *mn = w->nmin + 3 * node, *mx = w->nmax + 3 * node;
        if (mn[0] > hi[0] || mn[1] > hi[1] || mn[2] > hi[2] || mx[0] < lo[0] || mx[1] < lo[1] ||
            mx[2] < lo[2])
            continue;
        const int64_t cnt = w->ncount[node];
        if (cnt == 0) {
            stack[top] = 2 * node + 1;
            stack[top + 1] = 2 * node + 2;
            top += 2;
            continue;
        }
        for (int64_t t = w->nstart[node]; t < w->nstart[node] + cnt; ++t) {
            const int64_t tri = w->torder[t];
            const double *a = w->verts + 3 * w->tris[3 * tri];
            const double *b = w->verts + 3 * w->tris[3 * tri + 1];
            const double *c = w->verts + 3 * w->tris[3 * tri + 2];
            double e1[3], e2[3], face[3], closest[3], delta[3], n[3];
            for (int k = 0; k < 3; ++k) {
                e1[k] = b[k] - a[k];
                e2[k] = c[k] - a[k];
            }
            face[0] = e1[1] * e2[2] - e1[2] * e2[1];
            face[1] = e1[2] * e2[0] - e1[0] * e2[2];
            face[2] = e1[0] * e2[1] - e1[1] * e2[0];
            const double area2 = sqrt(face[0] * face[0] + face[1] * face[1] + face[2] * face[2]);
            if (area2 == 0.0) {
                w->err_step = w->step;
                continue;
            }
            closest_tri(center, a, b, c, closest);
            for (int k = 0; k < 3; ++k) delta[k] = center[k] - closest[k];
            const double d = sqrt(delta[0] * delta[0] + delta[1] * delta[1] + delta[2] * delta[2]);
            if (d >= radius)
                continue;
            double dot = 0.0;
            for (int k = 0; k < 3; ++k) {
                n[k] = face[k] / area2;
                dot += n[k] * (center[k] - a[k]);
            }
            if (dot < 0.0)
                for (int k = 0; k < 3; ++k) n[k] = -n[k];
            const double depth = radius - d;
            nhits += 1;
            for (int k = 0; k < 3; ++k) wsum[k] += depth * n[k];
            if (depth > maxd) {
                maxd = depth;
                for (int k = 0; k < 3; ++k) best_n[k] = n[k];
            }
        }
    }
    if (nhits == 0)
        return;
    const double norm = sqrt(wsum[0] * wsum[0] + wsum[1] * wsum[1] + wsum[2] * wsum[2]);
    if (norm < 1e-12 * (maxd > 1.0 ? maxd : 1.0)) {
        for (int k = 0; k < 3; ++k) w->cnorm[3 * i + k] = best_n[k];
    } else {
        for (int k = 0; k < 3; ++k) w->cnorm[3 * i + k] = wsum[k] / norm;
    }
    maxd -= w->coll_margin;               /* the margin inflates detection only */
    if (maxd < 0.0)
        maxd = 0.0;
    w->cdepth[i] = maxd;
    w->cact[i] = 1;
    w->contacts += 1;
}

/* contact slot reset + detection for every point (_core.pyx:730-741) */
static void detect_contacts(ro_world *w)
{
    const int detect = w->step % w->coll_interval == 0;
    w->contacts = 0;
    for (int64_t i = 0; i < w->P; ++i) {
        w->cacc_n[i] = 0.0;
        w->cacc_t[i] = 0.0;
        if (detect) {
            w->cact[i] = 0;
            if (w->has_mesh && w->cmask[i])
                mesh_contact(w, i);
        } else if (w->cact[i]) {
            w->contacts += 1;
        }
    }
}

void ro_scatter(ro_world *w)
{
    if (w->cact)
        detect_contacts(w);
    for (int64_t e = 0; e < w->E; ++e)
        scatter_element(w, e);
}

/* ---- self-collision broad phase (_core.pyx:665-708) ---------------------- */

void ro_selfpairs(ro_world *w)
{
    if (!w->has_self)
        return;
    if (w->step % w->coll_interval != 0) {   /* reuse the set, reset accumulators */
        for (int64_t k = 0; k < w->pairs; ++k) w->pair_acc[k] = 0.0;
        return;
    }
    for (int64_t g = 0; g < w->n_groups; ++g) {
        double *c = w->grp_c + 3 * g;
        c[0] = 0.0;
        c[1] = 0.0;
        c[2] = 0.0;
        for (int64_t i = w->grp_s[g]; i < w->grp_e[g]; ++i)
            for (int k = 0; k < 3; ++k) c[k] += w->pos[3 * i + k];
        const double inv = 1.0 / (double)(w->grp_e[g] - w->grp_s[g]);
        for (int k = 0; k < 3; ++k) c[k] *= inv;
    }
    int64_t cnt = 0;
    for (int64_t a = 0; a < w->n_groups; ++a) {
        for (int64_t b = a + 1; b < w->n_groups; ++b) {
            if (w->grp_rod[a] == w->grp_rod[b]) {
                const int64_t g = w->grp_gi[a] - w->grp_gi[b];
                if (-w->excl <= g && g <= w->excl)
                    continue;
            }
            const double *ca = w->grp_c + 3 * a, *cb = w->grp_c + 3 * b;
            double dx = cb[0] - ca[0], dy = cb[1] - ca[1], dz = cb[2] - ca[2];
            if (dx * dx + dy * dy + dz * dz >= w->broad * w->broad)
                continue;
            for (int64_t i = w->grp_s[a]; i < w->grp_e[a]; ++i) {
                for (int64_t j = w->grp_s[b]; j < w->grp_e[b]; ++j) {
                    dx = w->pos[3 * j] - w->pos[3 * i];
                    dy = w->pos[3 * j + 1] - w->pos[3 * i + 1];
                    dz = w->pos[3 * j + 2] - w->pos[3 * i + 2];
                    if (dx * dx + dy * dy + dz * dz < w->touch * w->touch && cnt < w->pair_cap) {
                        w->pair_a[cnt] = i;
                        w->pair_b[cnt] = j;
                        w->pair_md[cnt] = w->touch;
                        w->pair_acc[cnt] = 0.0;
                        cnt += 1;
                    }
                }
            }
        }
    }
    w->pairs = cnt;
}

/* ---- contact impulses with accumulator and box friction (_core.pyx:906-947) */

void ro_contacts(ro_world *w)
{
    if (!w->cact)
        return;
    for (int64_t i = 0; i < w->P; ++i) {
        if (w->cact[i] != 1 || w->plock[i])
            continue;
        double *v = w->vel + 3 * i, n[3], vt[3];
        const double m = w->mass[i];
        double vn = 0.0;
        for (int k = 0; k < 3; ++k) {
            n[k] = w->cnorm[3 * i + k];
            vn += v[k] * n[k];
        }
        const double raw = m * (-vn * (1.0 + w->restitution) + w->beta * w->cdepth[i] / w->dt);
        double new_acc = w->cacc_n[i] + raw;
        if (new_acc < 0.0)
            new_acc = 0.0;
        const double applied = new_acc - w->cacc_n[i];
        for (int k = 0; k < 3; ++k) v[k] += (applied / m) * n[k];
        w->cacc_n[i] = new_acc;
        if (w->mu > 0.0) {
            double dot = 0.0, vt_norm = 0.0;
            for (int k = 0; k < 3; ++k) dot += v[k] * n[k];
            for (int k = 0; k < 3; ++k) {
                vt[k] = v[k] - dot * n[k];
                vt_norm += vt[k] * vt[k];
            }
            vt_norm = sqrt(vt_norm);
            double cap = w->mu * new_acc - w->cacc_t[i];
            if (cap < 0.0)
                cap = 0.0;
            double jt = m * vt_norm;
            if (jt > cap)
                jt = cap;
            if (vt_norm > 0.0) {
                const double scale = jt / (m * vt_norm);
                for (int k = 0; k < 3; ++k) v[k] -= scale * vt[k];
            }
            w->cacc_t[i] += jt;
        }
    }
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
    /* self-collision pairs, in list order (_core.pyx:956-980) */
    for (int64_t k = 0; k < w->pairs; ++k) {
        const int64_t a = w->pair_a[k], b = w->pair_b[k];
        double d[3], n[3];
        for (int i = 0; i < 3; ++i) d[i] = w->pos[3 * b + i] - w->pos[3 * a + i];
        const double dist = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        const double wsum = w->invm[a] + w->invm[b];
        if (dist == 0.0 || wsum == 0.0)
            continue;
        double vrel = 0.0;
        for (int i = 0; i < 3; ++i) {
            n[i] = d[i] / dist;
            vrel += (w->vel[3 * b + i] - w->vel[3 * a + i]) * n[i];
        }
        double depth = w->pair_md[k] - dist;
        if (depth < 0.0)
            depth = 0.0;
        const double raw = (-vrel + w->beta * depth / w->dt) / wsum;
        double new_acc = w->pair_acc[k] + raw;
        if (new_acc < 0.0)
            new_acc = 0.0;
        const double lam = new_acc - w->pair_acc[k];
        w->pair_acc[k] = new_acc;
        for (int i = 0; i < 3; ++i) {
            w->vel[3 * a + i] -= w->invm[a] * lam * n[i];
            w->vel[3 * b + i] += w->invm[b] * lam * n[i];
        }
    }
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
        if (w->step % (w->coll_interval > 0 ? w->coll_interval : 1) == 0)
            w->pairs = 0;                   /* ph_boundary (_core.pyx:504-505) */
        ro_scatter(w);
        ro_selfpairs(w);
        ro_gather(w);
        for (int64_t it = 0; it < w->iters; ++it) {
            ro_distance(w, 0);
            ro_distance(w, 1);
            ro_contacts(w);
            ro_central(w);
        }
        ro_integrate(w);
        w->step += 1;
    }
}
