/*
 * rod_oracle.h -- CPU restatement of the reference CoRdE step (TEST
 * INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the timed CPU baseline -- never as the product path.
 *
 * The struct mirrors the reference's flat World arrays (world.py:77-182):
 * positions/velocities (P,3) f64 AoS, frames (E,4), angular velocities (E,3),
 * per-element material arrays, per-point/per-frame lock flags, drivers,
 * bindings and grab anchors.  The stepping semantics follow the reference's
 * compiled serial step (_core.pyx:1058-1080): elastic forces, constraints,
 * bindings, grabs, mesh contacts and self-collision pairs.
 */
#ifndef ROD_ORACLE_H
#define ROD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ro_world {
    int64_t P, E, R;            /* points, elements, rods */
    int64_t iters;              /* constraint iterations */
    double dt, beta;            /* step, Baumgarte position bias */
    double gx, gy, gz;          /* gravity */
    /* dynamic state (mutated in place) */
    double *pos, *vel, *q, *w;
    /* per-element constants */
    const double *rest, *ustar, *inert, *ks, *kp, *gt, *gr, *ext, *kb;
    /* per-point constants */
    const double *mass, *invm, *fext;
    const uint8_t *plock;       /* (P) point locked */
    const uint8_t *flock;       /* (E) frame locked */
    const int64_t *elem_point;  /* (E) lower point of element */
    const int64_t *elem_parity; /* (E) red/black colour */
    const uint8_t *jvalid;      /* (E) junction e <-> e+1 valid */
    /* drivers, one per rod, -1 when absent */
    const double *drv_v, *drv_rot;
    const int64_t *drv_pt, *drv_fr;
    /* bindings */
    int64_t nbind;
    const int64_t *bind_a, *bind_b, *bind_mode;
    /* grab anchors */
    int64_t ngrab;
    const uint8_t *g_act;
    const int64_t *g_pt;
    const double *g_tgt;
    /* scratch, caller-allocated and persistent like the reference ctx:
       ef (E,3), ff_own (E,4), ff_next (E,4), jtau (E,3), pt_elo/pt_ehi (P) */
    double *ef, *ff_own, *ff_next, *jtau;
    int64_t *pt_elo, *pt_ehi;
    /* counters: step counter and last error step (-1 if none) */
    int64_t step;
    int64_t err_step;
    /* mesh contacts (_core.pyx:509-662, 906-947); has_mesh 0: none.  The
       tree arrays follow bvh.TriMeshBvh, the contact slots world.py:157-161 */
    int64_t has_mesh, n_nodes;
    const double *nmin, *nmax, *verts;
    const int64_t *nstart, *ncount, *torder, *tris;
    const double *cradii;        /* (P) contact radius */
    const uint8_t *cmask;        /* (P) point collides with the mesh */
    uint8_t *cact;               /* (P) contact active */
    double *cnorm, *cdepth;      /* (P,3), (P) */
    double *cacc_n, *cacc_t;     /* (P) impulse accumulators */
    int64_t coll_interval;
    double coll_margin, restitution, mu;
    int64_t contacts;            /* active contacts after the last step */
    /* self-collision (_core.pyx:665-708, 956-980); has_self 0: none */
    int64_t has_self, n_groups, excl, pair_cap;
    const int64_t *grp_rod, *grp_gi, *grp_s, *grp_e;   /* (G) group table */
    double *grp_c;                                     /* (G,3) scratch */
    double touch, broad;
    int64_t *pair_a, *pair_b;    /* (pair_cap) world.pair_a / pair_b */
    double *pair_md, *pair_acc;  /* world.pair_min_dist / pair_acc */
    int64_t pairs;               /* CNT_PAIRS: pairs in the current set */
} ro_world;

/* Build pt_elo / pt_ehi from elem_point (make_context, _core.pyx:264-272). */
void ro_prepare(ro_world *w);
/* Advance `steps` time steps. */
void ro_run(ro_world *w, int64_t steps);
/* Single phases, exported for unit tests of the restatement. */
void ro_scatter(ro_world *w);
void ro_gather(ro_world *w);
void ro_distance(ro_world *w, int64_t parity);
void ro_central(ro_world *w);
void ro_contacts(ro_world *w);
void ro_selfpairs(ro_world *w);
void ro_integrate(ro_world *w);

#ifdef __cplusplus
}
#endif
#endif
