/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference hot path.
 * See kf_oracle.h for the contract. References are to /root/reference/proj.
 *
 * Arithmetic is written in the reference's evaluation order so that, built
 * with -ffp-contract=off (oracle/Makefile), results are bit-identical to the
 * reference; tests/test_oracle.py checks exactly that.
 */
#define _GNU_SOURCE
#include "kf_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define KG 1.4 /* kGamma, state.hpp:16 */
static const double kPi = 3.14159265358979323846;         /* kinetics.cpp:10 */
static const double kInvSqrtPi = 0.5641895835477562869;   /* tangent.cpp:13 */
static const double kSingularDetEps = 1e-12;              /* pointcloud.hpp:50 */

enum { K_REGULAR = 0, K_LINEX = 1, K_LINEY = 2, K_EMPTY = 3, K_SINGULAR = 4 };

typedef struct { double rho, u1, u2, p; } prim_t;

typedef struct {
    int* off; /* n+1 */
    int* idx;
    double* w;  /* split: own-direction weight; full: wx */
    double* w2; /* full only: wy */
    double* one;
    int* kind;
} list_t;

struct kfo_cloud {
    int n;
    double *x, *y, *nx, *ny;
    int* kind;
    list_t nbr, xpos, xneg, ypos, yneg;
    int* flagged;
    int n_flagged;
    int* empty_pts;
    int n_empty;
    int* singular_pts;
    int n_singular;
    int* color;
    int n_colors;
    int** groups;
    int* group_size;
    int *wall, *outer;
    int n_wall, n_outer;
};

static void set_err(kfo_err* e, int code, int point, const char* what)
{
    if (!e) return;
    e->code = code;
    e->point = point;
    if (point >= 0)
        snprintf(e->msg, sizeof e->msg, "%s at point %d", what, point);
    else
        snprintf(e->msg, sizeof e->msg, "%s", what);
}

/* ---------------- state algebra: state.cpp ---------------- */

/* primitives_from_conserved, state.cpp:5-16. Returns 0 ok, 1 density, 2 pressure. */
static int prim_from_cons(const double* U, prim_t* w)
{
    const double rho = U[0];
    if (!(rho > 0.0)) return 1;
    const double u1 = U[1] / rho;
    const double u2 = U[2] / rho;
    const double p = (KG - 1.0) * (U[3] - 0.5 * rho * (u1 * u1 + u2 * u2));
    if (!(p > 0.0)) return 2;
    w->rho = rho; w->u1 = u1; w->u2 = u2; w->p = p;
    return 0;
}

/* conserved_from_primitives, state.cpp:18-22 */
static void cons_from_prim(const prim_t* w, double* U)
{
    const double rho_e = w->p / (KG - 1.0) + 0.5 * w->rho * (w->u1 * w->u1 + w->u2 * w->u2);
    U[0] = w->rho;
    U[1] = w->rho * w->u1;
    U[2] = w->rho * w->u2;
    U[3] = rho_e;
}

/* q_from_primitives, state.cpp:24-30 (beta: state.hpp:89) */
static void q_from_prim(const prim_t* w, double* q)
{
    const double beta = 0.5 * w->rho / w->p;
    const double q1 = log(w->rho) + log(beta) / (KG - 1.0) - beta * (w->u1 * w->u1 + w->u2 * w->u2);
    q[0] = q1;
    q[1] = 2.0 * beta * w->u1;
    q[2] = 2.0 * beta * w->u2;
    q[3] = -2.0 * beta;
}

/* primitives_from_q, state.cpp:32-46. 0 ok, 1 q4>=0, 2 degenerate density. */
static int prim_from_q(const double* q, prim_t* w)
{
    if (!(q[3] < 0.0)) return 1;
    const double beta = -0.5 * q[3];
    const double u1 = q[1] / (2.0 * beta);
    const double u2 = q[2] / (2.0 * beta);
    const double ln_rho = q[0] - log(beta) / (KG - 1.0) + beta * (u1 * u1 + u2 * u2);
    const double rho = exp(ln_rho);
    const double p = 0.5 * rho / beta;
    if (!isfinite(rho) || !(rho > 0.0) || !(p > 0.0)) return 2;
    w->rho = rho; w->u1 = u1; w->u2 = u2; w->p = p;
    return 0;
}

static double sound_speed(const prim_t* w) { return sqrt(KG * w->p / w->rho); } /* state.hpp:88 */

static int all_finite4(const double* a)
{
    return isfinite(a[0]) && isfinite(a[1]) && isfinite(a[2]) && isfinite(a[3]);
}

/* ---------------- kinetics.cpp ---------------- */

/* flux_gx / flux_gy, kinetics.cpp:19-37 */
static void flux_full(const double* U, int axis, double* G)
{
    const double rho = U[0];
    const double u1 = U[1] / rho;
    const double u2 = U[2] / rho;
    const double pr = 0.4 * (U[3] - 0.5 * rho * (u1 * u1 + u2 * u2));
    if (axis == 0) {
        G[0] = rho * u1; G[1] = pr + rho * u1 * u1; G[2] = rho * u1 * u2; G[3] = (pr + U[3]) * u1;
    } else {
        G[0] = rho * u2; G[1] = rho * u1 * u2; G[2] = pr + rho * u2 * u2; G[3] = (pr + U[3]) * u2;
    }
}

/* split_flux(Primitives, axis, sign), kinetics.cpp:49-70 */
static void split_flux_prim(const prim_t* w, int axis, int sign, double* G)
{
    const double sg = (sign == 0) ? 1.0 : -1.0;
    const double un = (axis == 0) ? w->u1 : w->u2;
    const double ut = (axis == 0) ? w->u2 : w->u1;
    const double beta = 0.5 * w->rho / w->p;
    const double s = un * sqrt(beta);
    const double A = 0.5 * (1.0 + sg * erf(s));
    const double B = 0.5 * exp(-s * s) / sqrt(kPi * beta);
    const double ke = 0.5 * w->rho * (w->u1 * w->u1 + w->u2 * w->u2);
    const double mass = w->rho * (un * A + sg * B);
    const double mom_n = (w->p + w->rho * un * un) * A + sg * w->rho * un * B;
    const double mom_t = ut * mass;
    const double energy = (KG / (KG - 1.0) * w->p + ke) * un * A +
                          sg * ((KG + 1.0) / (2.0 * (KG - 1.0)) * w->p + ke) * B;
    G[0] = mass;
    G[1] = axis == 0 ? mom_n : mom_t;
    G[2] = axis == 0 ? mom_t : mom_n;
    G[3] = energy;
}

/* spectral radii, kinetics.cpp:87-110 */
static double srad_full(const prim_t* w, int axis)
{
    const double un = (axis == 0) ? w->u1 : w->u2;
    return fabs(un) + sound_speed(w);
}

static double srad_split(const prim_t* w, int axis, int sign)
{
    const double un = (axis == 0) ? w->u1 : w->u2;
    const double a = sound_speed(w);
    if (sign == 0) return 0.5 * fabs((un + a) + fabs(un + a));
    return 0.5 * fabs((un - a) - fabs(un - a));
}

/* ---------------- tangent.cpp ---------------- */

/* require_valid / require_valid_increment, tangent.cpp:15-37: 0 ok, 1 bad */
static int valid_u(const double* U)
{
    const double rho = U[0];
    if (!(rho > 0.0)) return 1;
    const double pr = 0.4 * (U[3] - 0.5 * (U[1] * U[1] + U[2] * U[2]) / rho);
    if (!(pr > 0.0)) return 1;
    return 0;
}

/* jvp_full, tangent.cpp:41-69 (caller has checked validity) */
static void jvp_full_exact(const double* U, const double* Ud, int axis, double* o)
{
    const double rhod = Ud[0];
    const double rho = U[0];
    double temp = U[1] / rho;
    const double u1d = (Ud[1] - temp * rhod) / rho;
    const double u1 = temp;
    temp = U[2] / rho;
    const double u2d = (Ud[2] - temp * rhod) / rho;
    const double u2 = temp;
    temp = u1 * u1 + u2 * u2;
    const double prd = 0.4 * (Ud[3] - 0.5 * (temp * rhod + rho * (2.0 * u1 * u1d + 2.0 * u2 * u2d)));
    const double pr = 0.4 * (U[3] - 0.5 * (rho * temp));
    if (axis == 0) {
        o[0] = u1 * rhod + rho * u1d;
        o[1] = prd + u1 * u1 * rhod + rho * 2.0 * u1 * u1d;
        o[2] = u2 * (u1 * rhod + rho * u1d) + rho * u1 * u2d;
        o[3] = u1 * (prd + Ud[3]) + (pr + U[3]) * u1d;
    } else {
        o[0] = u2 * rhod + rho * u2d;
        o[1] = u1 * (u2 * rhod + rho * u2d) + rho * u2 * u1d;
        o[2] = prd + u2 * u2 * rhod + rho * 2.0 * u2 * u2d;
        o[3] = u2 * (prd + Ud[3]) + (pr + U[3]) * u2d;
    }
}

/* jvp_split, tangent.cpp:71-137 (caller has checked validity) */
static void jvp_split_exact(const double* U, const double* Ud, int axis, int sign, double* o)
{
    const double sg = (sign == 0) ? 1.0 : -1.0;
    const double rhod = Ud[0];
    const double rho = U[0];
    double temp = U[1] / rho;
    const double u1d = (Ud[1] - temp * rhod) / rho;
    const double u1 = temp;
    temp = U[2] / rho;
    const double u2d = (Ud[2] - temp * rhod) / rho;
    const double u2 = temp;
    const double v2 = u1 * u1 + u2 * u2;
    const double v2d = 2.0 * u1 * u1d + 2.0 * u2 * u2d;
    const double prd = 0.4 * (Ud[3] - 0.5 * (v2 * rhod + rho * v2d));
    const double pr = 0.4 * (U[3] - 0.5 * rho * v2);

    const double un = (axis == 0) ? u1 : u2;
    const double und = (axis == 0) ? u1d : u2d;
    const double ut = (axis == 0) ? u2 : u1;
    const double utd = (axis == 0) ? u2d : u1d;

    const double beta = 0.5 * rho / pr;
    const double betad = 0.5 * (rhod * pr - rho * prd) / (pr * pr);
    const double sqb = sqrt(beta);
    const double sqbd = 0.5 * betad / sqb;
    const double s = un * sqb;
    const double sd = und * sqb + un * sqbd;

    const double ex = exp(-s * s);
    const double exd = -2.0 * s * sd * ex;
    const double A = 0.5 * (1.0 + sg * erf(s));
    const double Ad = sg * kInvSqrtPi * ex * sd;
    const double B = 0.5 * ex / sqrt(kPi * beta);
    const double Bd = 0.5 * exd / sqrt(kPi * beta) - 0.25 * kInvSqrtPi * ex * betad / (beta * sqb);

    const double ke = 0.5 * rho * v2;
    const double ked = 0.5 * (rhod * v2 + rho * v2d);

    const double mass = rho * (un * A + sg * B);
    const double massd = rhod * (un * A + sg * B) + rho * (und * A + un * Ad + sg * Bd);
    const double mom_nd = (prd + rhod * un * un + 2.0 * rho * un * und) * A +
                          (pr + rho * un * un) * Ad +
                          sg * ((rhod * un + rho * und) * B + rho * un * Bd);
    const double mom_td = utd * mass + ut * massd;

    const double ge = KG / (KG - 1.0);
    const double gb = (KG + 1.0) / (2.0 * (KG - 1.0));
    const double c1 = ge * pr + ke;
    const double c1d = ge * prd + ked;
    const double c2 = gb * pr + ke;
    const double c2d = gb * prd + ked;
    const double energyd = c1d * un * A + c1 * (und * A + un * Ad) + sg * (c2d * B + c2 * Bd);

    o[0] = massd;
    o[1] = axis == 0 ? mom_nd : mom_td;
    o[2] = axis == 0 ? mom_td : mom_nd;
    o[3] = energyd;
}

/* split_flux(Vec4 U, ...), kinetics.cpp:72-75; 1 if U invalid */
static int split_flux_cons(const double* U, int axis, int sign, double* G)
{
    prim_t w;
    if (prim_from_cons(U, &w)) return 1;
    split_flux_prim(&w, axis, sign, G);
    return 0;
}

/* mode_jvp_split, tangent.cpp:155-161 with incremental_jvp_split :147-153.
 * Returns 0 ok, 1 invalid base state, 2 invalid increment. */
static int mode_jvp_split(int exact, const double* U, const double* dU, int axis, int sign,
                          double* o)
{
    if (valid_u(U)) return 1;
    if (exact) {
        jvp_split_exact(U, dU, axis, sign, o);
        return 0;
    }
    double V[4], a[4], b[4];
    for (int k = 0; k < 4; ++k) V[k] = U[k] + dU[k];
    if (valid_u(V)) return 2;
    if (split_flux_cons(V, axis, sign, a)) return 2;
    if (split_flux_cons(U, axis, sign, b)) return 1;
    for (int k = 0; k < 4; ++k) o[k] = a[k] - b[k];
    return 0;
}

/* mode_jvp_full, tangent.cpp:163-168 with incremental_jvp_full :139-145 */
static int mode_jvp_full(int exact, const double* U, const double* dU, int axis, double* o)
{
    if (valid_u(U)) return 1;
    if (exact) {
        jvp_full_exact(U, dU, axis, o);
        return 0;
    }
    double V[4], a[4], b[4];
    for (int k = 0; k < 4; ++k) V[k] = U[k] + dU[k];
    if (valid_u(V)) return 2;
    flux_full(V, axis, a);
    flux_full(U, axis, b);
    for (int k = 0; k < 4; ++k) o[k] = a[k] - b[k];
    return 0;
}

/* ---------------- ingestion ---------------- */

static void list_alloc(list_t* L, int n, long nnz, int with_w2)
{
    memset(L, 0, sizeof *L);
    L->off = calloc((size_t)n + 1, sizeof(int));
    L->idx = calloc((size_t)(nnz > 0 ? nnz : 1), sizeof(int));
    L->w = calloc((size_t)(nnz > 0 ? nnz : 1), sizeof(double));
    if (with_w2) L->w2 = calloc((size_t)(nnz > 0 ? nnz : 1), sizeof(double));
    L->one = calloc((size_t)n, sizeof(double));
    L->kind = calloc((size_t)n, sizeof(int));
}

static void list_free(list_t* L)
{
    free(L->off); free(L->idx); free(L->w); free(L->w2); free(L->one); free(L->kind);
}

typedef struct { double mxx, myy, mxy; } moments_t;

/* stencil_moments, spatial.cpp:17-27 */
static moments_t moments(const kfo_cloud* c, int p, const int* st, int m)
{
    moments_t r = {0.0, 0.0, 0.0};
    for (int k = 0; k < m; ++k) {
        const double dx = c->x[st[k]] - c->x[p];
        const double dy = c->y[st[k]] - c->y[p];
        r.mxx += dx * dx;
        r.myy += dy * dy;
        r.mxy += dx * dy;
    }
    return r;
}

/* classify_moments, spatial.cpp:29-38 */
static int classify(moments_t m, int n)
{
    if (n == 0) return K_EMPTY;
    if (m.mxx == 0.0 && m.myy == 0.0) return K_SINGULAR;
    if (m.myy == 0.0) return K_LINEX;
    if (m.mxx == 0.0) return K_LINEY;
    const double det = m.mxx * m.myy - m.mxy * m.mxy;
    if (det < kSingularDetEps * m.mxx * m.myy) return K_SINGULAR;
    return K_REGULAR;
}

/* build_split_stencils' singular lambda, pointcloud.cpp:264-277 */
static int split_singular(const kfo_cloud* c, int p, const int* st, int m)
{
    if (m == 0) return 0;
    moments_t r = moments(c, p, st, m);
    if (r.mxx == 0.0 || r.myy == 0.0) return 0;
    const double det = r.mxx * r.myy - r.mxy * r.mxy;
    return det < kSingularDetEps * r.mxx * r.myy;
}

/* fill_split, spatial.cpp:40-76; axis 0 X 1 Y */
static void fill_split(const kfo_cloud* c, int p, list_t* L, int axis, int* flagged)
{
    const int b = L->off[p], m = L->off[p + 1] - b;
    const int* st = L->idx + b;
    double* w = L->w + b;
    for (int k = 0; k < m; ++k) w[k] = 0.0;
    const moments_t mo = moments(c, p, st, m);
    const int kind = classify(mo, m);
    L->kind[p] = kind;
    L->one[p] = 0.0;
    switch (kind) {
        case K_EMPTY: return;
        case K_SINGULAR: *flagged = 1; return;
        case K_LINEX:
            if (axis == 1) return;
            for (int k = 0; k < m; ++k) w[k] = (c->x[st[k]] - c->x[p]) / mo.mxx;
            break;
        case K_LINEY:
            if (axis == 0) return;
            for (int k = 0; k < m; ++k) w[k] = (c->y[st[k]] - c->y[p]) / mo.myy;
            break;
        default: {
            const double den = mo.mxx * mo.myy - mo.mxy * mo.mxy;
            for (int k = 0; k < m; ++k) {
                const double dx = c->x[st[k]] - c->x[p];
                const double dy = c->y[st[k]] - c->y[p];
                w[k] = (axis == 0) ? (mo.myy * dx - mo.mxy * dy) / den
                                   : (mo.mxx * dy - mo.mxy * dx) / den;
            }
        }
    }
    double s = 0.0;
    for (int k = 0; k < m; ++k) s += w[k];
    L->one[p] = s;
}

static int cmp_int(const void* a, const void* b)
{
    const int x = *(const int*)a, y = *(const int*)b;
    return (x > y) - (x < y);
}

/* symmetrized_connectivity + color_points + build_sweep_plan,
 * coloring.cpp:7-62 */
static void color_cloud(kfo_cloud* c)
{
    const int n = c->n;
    int* deg = calloc((size_t)n + 1, sizeof(int));
    for (int i = 0; i < n; ++i)
        for (int k = c->nbr.off[i]; k < c->nbr.off[i + 1]; ++k) {
            deg[i]++;
            deg[c->nbr.idx[k]]++;
        }
    int* aoff = calloc((size_t)n + 1, sizeof(int));
    for (int i = 0; i < n; ++i) aoff[i + 1] = aoff[i] + deg[i];
    int* adj = malloc(sizeof(int) * (size_t)(aoff[n] > 0 ? aoff[n] : 1));
    int* fill = calloc((size_t)n, sizeof(int));
    for (int i = 0; i < n; ++i)
        for (int k = c->nbr.off[i]; k < c->nbr.off[i + 1]; ++k) {
            const int q = c->nbr.idx[k];
            adj[aoff[i] + fill[i]++] = q;
            adj[aoff[q] + fill[q]++] = i;
        }
    /* sort + unique per row */
    int* asz = calloc((size_t)n, sizeof(int));
    for (int i = 0; i < n; ++i) {
        int* a = adj + aoff[i];
        const int m = aoff[i + 1] - aoff[i];
        qsort(a, (size_t)m, sizeof(int), cmp_int);
        int u = 0;
        for (int k = 0; k < m; ++k)
            if (u == 0 || a[k] != a[u - 1]) a[u++] = a[k];
        asz[i] = u;
    }
    c->color = calloc((size_t)(n > 0 ? n : 1), sizeof(int));
    if (n > 0) {
        c->color[0] = 1;
        char* used = NULL;
        size_t used_cap = 0;
        for (int i = 0; i < n; ++i) {
            for (int t = 0; t < asz[i]; ++t) {
                const int p = adj[aoff[i] + t];
                if (c->color[p] != 0) continue;
                const size_t us = (size_t)asz[p] + 2;
                if (us > used_cap) {
                    free(used);
                    used = malloc(us);
                    used_cap = us;
                }
                memset(used, 0, us);
                for (int s = 0; s < asz[p]; ++s) {
                    const int cq = c->color[adj[aoff[p] + s]];
                    if (cq > 0 && (size_t)cq < us) used[cq] = 1;
                }
                int k = 1;
                while (used[k]) ++k;
                c->color[p] = k;
            }
        }
        free(used);
        for (int i = 0; i < n; ++i)
            if (c->color[i] == 0) c->color[i] = 1;
    }
    int nc = 0;
    for (int i = 0; i < n; ++i)
        if (c->color[i] > nc) nc = c->color[i];
    c->n_colors = nc;
    c->group_size = calloc((size_t)(nc > 0 ? nc : 1), sizeof(int));
    c->groups = calloc((size_t)(nc > 0 ? nc : 1), sizeof(int*));
    for (int i = 0; i < n; ++i) c->group_size[c->color[i] - 1]++;
    for (int g = 0; g < nc; ++g) c->groups[g] = malloc(sizeof(int) * (size_t)(c->group_size[g] + 1));
    int* gf = calloc((size_t)(nc > 0 ? nc : 1), sizeof(int));
    for (int i = 0; i < n; ++i) {
        const int g = c->color[i] - 1;
        c->groups[g][gf[g]++] = i;
    }
    free(gf); free(deg); free(aoff); free(adj); free(fill); free(asz);
}

kfo_cloud* kfo_cloud_new(int n, const double* x, const double* y, const int* kind,
                         const double* nx, const double* ny, const int* off, const int* idx)
{
    kfo_cloud* c = calloc(1, sizeof *c);
    c->n = n;
    c->x = malloc(sizeof(double) * (size_t)n);
    c->y = malloc(sizeof(double) * (size_t)n);
    c->nx = malloc(sizeof(double) * (size_t)n);
    c->ny = malloc(sizeof(double) * (size_t)n);
    c->kind = malloc(sizeof(int) * (size_t)n);
    memcpy(c->x, x, sizeof(double) * (size_t)n);
    memcpy(c->y, y, sizeof(double) * (size_t)n);
    memcpy(c->nx, nx, sizeof(double) * (size_t)n);
    memcpy(c->ny, ny, sizeof(double) * (size_t)n);
    memcpy(c->kind, kind, sizeof(int) * (size_t)n);
    const long nnz = off[n];
    list_alloc(&c->nbr, n, nnz, 1);
    memcpy(c->nbr.off, off, sizeof(int) * ((size_t)n + 1));
    memcpy(c->nbr.idx, idx, sizeof(int) * (size_t)(nnz > 0 ? nnz : 0));

    c->wall = malloc(sizeof(int) * (size_t)(n + 1));
    c->outer = malloc(sizeof(int) * (size_t)(n + 1));
    for (int p = 0; p < n; ++p) {
        if (kind[p] == 0) c->wall[c->n_wall++] = p;
        if (kind[p] == 2) c->outer[c->n_outer++] = p;
    }

    /* build_split_stencils, pointcloud.cpp:257-299 */
    list_t* L[4] = {&c->xpos, &c->xneg, &c->ypos, &c->yneg};
    for (int s = 0; s < 4; ++s) list_alloc(L[s], n, nnz, 0);
    long fill[4] = {0, 0, 0, 0};
    c->empty_pts = malloc(sizeof(int) * (size_t)(n + 1));
    c->singular_pts = malloc(sizeof(int) * (size_t)(n + 1));
    for (int p = 0; p < n; ++p) {
        for (int s = 0; s < 4; ++s) L[s]->off[p] = (int)fill[s];
        for (int k = off[p]; k < off[p + 1]; ++k) {
            const int q = idx[k];
            const double dx = x[q] - x[p];
            const double dy = y[q] - y[p];
            if (dx >= 0.0) c->xpos.idx[fill[0]++] = q;
            if (dx <= 0.0) c->xneg.idx[fill[1]++] = q;
            if (dy >= 0.0) c->ypos.idx[fill[2]++] = q;
            if (dy <= 0.0) c->yneg.idx[fill[3]++] = q;
        }
        for (int s = 0; s < 4; ++s) L[s]->off[p + 1] = (int)fill[s];
        int empty = 0;
        for (int s = 0; s < 4; ++s) empty |= (L[s]->off[p + 1] == L[s]->off[p]);
        if (empty) c->empty_pts[c->n_empty++] = p;
        int sing = 0;
        for (int s = 0; s < 4; ++s)
            sing |= split_singular(c, p, L[s]->idx + L[s]->off[p], L[s]->off[p + 1] - L[s]->off[p]);
        sing |= split_singular(c, p, idx + off[p], off[p + 1] - off[p]);
        if (sing) c->singular_pts[c->n_singular++] = p;
    }

    /* build_ls_coefficients, spatial.cpp:80-128 */
    c->flagged = malloc(sizeof(int) * (size_t)(n + 1));
    for (int p = 0; p < n; ++p) {
        int flagged = 0;
        const int b = off[p], m = off[p + 1] - off[p];
        const moments_t mo = moments(c, p, idx + b, m);
        const int fk = classify(mo, m);
        c->nbr.kind[p] = fk;
        for (int k = 0; k < m; ++k) {
            c->nbr.w[b + k] = 0.0;
            c->nbr.w2[b + k] = 0.0;
        }
        if (fk == K_REGULAR) {
            const double den = mo.mxx * mo.myy - mo.mxy * mo.mxy;
            for (int k = 0; k < m; ++k) {
                const double dx = x[idx[b + k]] - x[p];
                const double dy = y[idx[b + k]] - y[p];
                c->nbr.w[b + k] = (mo.myy * dx - mo.mxy * dy) / den;
                c->nbr.w2[b + k] = (mo.mxx * dy - mo.mxy * dx) / den;
            }
        } else if (fk == K_LINEX) {
            for (int k = 0; k < m; ++k) c->nbr.w[b + k] = (x[idx[b + k]] - x[p]) / mo.mxx;
        } else if (fk == K_LINEY) {
            for (int k = 0; k < m; ++k) c->nbr.w2[b + k] = (y[idx[b + k]] - y[p]) / mo.myy;
        } else if (fk == K_SINGULAR) {
            flagged = 1;
        }
        fill_split(c, p, &c->xpos, 0, &flagged);
        fill_split(c, p, &c->xneg, 0, &flagged);
        fill_split(c, p, &c->ypos, 1, &flagged);
        fill_split(c, p, &c->yneg, 1, &flagged);
        if (flagged) c->flagged[c->n_flagged++] = p;
    }
    color_cloud(c);
    return c;
}

void kfo_cloud_free(kfo_cloud* c)
{
    if (!c) return;
    free(c->x); free(c->y); free(c->nx); free(c->ny); free(c->kind);
    list_free(&c->nbr); list_free(&c->xpos); list_free(&c->xneg); list_free(&c->ypos);
    list_free(&c->yneg);
    free(c->flagged); free(c->empty_pts); free(c->singular_pts); free(c->color);
    for (int g = 0; g < c->n_colors; ++g) free(c->groups[g]);
    free(c->groups); free(c->group_size); free(c->wall); free(c->outer);
    free(c);
}

int kfo_n(const kfo_cloud* c) { return c->n; }
int kfo_n_colors(const kfo_cloud* c) { return c->n_colors; }

static const list_t* list_of(const kfo_cloud* c, int which)
{
    switch (which) {
        case 1: return &c->xpos;
        case 2: return &c->xneg;
        case 3: return &c->ypos;
        case 4: return &c->yneg;
        default: return &c->nbr;
    }
}

long kfo_list_nnz(const kfo_cloud* c, int which) { return list_of(c, which)->off[c->n]; }

void kfo_list(const kfo_cloud* c, int which, int* off, int* idx)
{
    const list_t* L = list_of(c, which);
    memcpy(off, L->off, sizeof(int) * ((size_t)c->n + 1));
    memcpy(idx, L->idx, sizeof(int) * (size_t)L->off[c->n]);
}

void kfo_ls_full(const kfo_cloud* c, double* wx, double* wy, int* kinds)
{
    const long m = c->nbr.off[c->n];
    memcpy(wx, c->nbr.w, sizeof(double) * (size_t)m);
    memcpy(wy, c->nbr.w2, sizeof(double) * (size_t)m);
    memcpy(kinds, c->nbr.kind, sizeof(int) * (size_t)c->n);
}

void kfo_ls_split(const kfo_cloud* c, int which, double* w, double* one, int* kinds)
{
    const list_t* L = list_of(c, which);
    memcpy(w, L->w, sizeof(double) * (size_t)L->off[c->n]);
    memcpy(one, L->one, sizeof(double) * (size_t)c->n);
    memcpy(kinds, L->kind, sizeof(int) * (size_t)c->n);
}

int kfo_flagged(const kfo_cloud* c, int* out)
{
    if (out) memcpy(out, c->flagged, sizeof(int) * (size_t)c->n_flagged);
    return c->n_flagged;
}

void kfo_colors(const kfo_cloud* c, int* color) { memcpy(color, c->color, sizeof(int) * (size_t)c->n); }

int kfo_report(const kfo_cloud* c, int* empty, int* n_empty, int* singular, int* n_singular)
{
    *n_empty = c->n_empty;
    *n_singular = c->n_singular;
    if (empty) memcpy(empty, c->empty_pts, sizeof(int) * (size_t)c->n_empty);
    if (singular) memcpy(singular, c->singular_pts, sizeof(int) * (size_t)c->n_singular);
    return 0;
}

/* ---------------- stages ---------------- */

/* Freestream::make, driver.cpp:12-22 */
static void freestream(double mach, double aoa, prim_t* w, double* U)
{
    const double alpha = aoa * M_PI / 180.0;
    w->rho = 1.0;
    w->u1 = mach * cos(alpha);
    w->u2 = mach * sin(alpha);
    w->p = 1.0 / KG;
    cons_from_prim(w, U);
}

void kfo_freestream(double mach, double aoa, double* U4)
{
    prim_t w;
    freestream(mach, aoa, &w, U4);
}

/* q loop, driver.cpp:229-230 -> q_from_conserved state.cpp:53-56 (serial) */
int kfo_q(const kfo_cloud* c, const double* U, double* q, kfo_err* e)
{
    for (int p = 0; p < c->n; ++p) {
        prim_t w;
        const int r = prim_from_cons(U + 4 * p, &w);
        if (r) {
            set_err(e, 1, p, r == 1 ? "nonpositive density" : "nonpositive pressure");
            return 1;
        }
        q_from_prim(&w, q + 4 * p);
    }
    return 0;
}

/* q_derivatives, spatial.cpp:151-196 */
void kfo_grads(const kfo_cloud* c, const double* q, int n_inner, double* qx, double* qy)
{
    const int n = c->n;
    const int* off = c->nbr.off;
    const int* idx = c->nbr.idx;
#pragma omp parallel for schedule(static)
    for (int p = 0; p < n; ++p) {
        double gx[4] = {0, 0, 0, 0}, gy[4] = {0, 0, 0, 0};
        for (int k = off[p]; k < off[p + 1]; ++k) {
            const int i = idx[k];
            for (int j = 0; j < 4; ++j) {
                const double dq = q[4 * i + j] - q[4 * p + j];
                gx[j] += c->nbr.w[k] * dq;
                gy[j] += c->nbr.w2[k] * dq;
            }
        }
        for (int j = 0; j < 4; ++j) {
            qx[4 * p + j] = gx[j];
            qy[4 * p + j] = gy[j];
        }
    }
    if (n_inner < 2) return;
    double* px = malloc(sizeof(double) * 4 * (size_t)n);
    double* py = malloc(sizeof(double) * 4 * (size_t)n);
    for (int pass = 2; pass <= n_inner; ++pass) {
        memcpy(px, qx, sizeof(double) * 4 * (size_t)n);
        memcpy(py, qy, sizeof(double) * 4 * (size_t)n);
#pragma omp parallel for schedule(static)
        for (int p = 0; p < n; ++p) {
            double gx[4] = {0, 0, 0, 0}, gy[4] = {0, 0, 0, 0};
            for (int k = off[p]; k < off[p + 1]; ++k) {
                const int i = idx[k];
                const double dx = c->x[i] - c->x[p];
                const double dy = c->y[i] - c->y[p];
                for (int j = 0; j < 4; ++j) {
                    const double dqt = (q[4 * i + j] - q[4 * p + j]) -
                                       0.5 * (dx * (px[4 * i + j] - px[4 * p + j]) +
                                              dy * (py[4 * i + j] - py[4 * p + j]));
                    gx[j] += c->nbr.w[k] * dqt;
                    gy[j] += c->nbr.w2[k] * dqt;
                }
            }
            for (int j = 0; j < 4; ++j) {
                qx[4 * p + j] = gx[j];
                qy[4 * p + j] = gy[j];
            }
        }
    }
    free(px);
    free(py);
}

/* direction map, spatial.hpp:49-56 and spatial.cpp:204-209:
 * d=0 X+ on xneg, 1 X- on xpos, 2 Y+ on yneg, 3 Y- on ypos */
static const list_t* dir_list(const kfo_cloud* c, int d)
{
    switch (d) {
        case 0: return &c->xneg;
        case 1: return &c->xpos;
        case 2: return &c->yneg;
        default: return &c->ypos;
    }
}

/* accumulate_second_order, spatial.cpp:213-232; 0 ok, 1 demote */
static int acc_second(const kfo_cloud* c, const list_t* st, int p, int axis, int sign,
                      const double* q, const double* qx, const double* qy, double* R)
{
    for (int k = st->off[p]; k < st->off[p + 1]; ++k) {
        if (st->w[k] == 0.0) continue;
        const int i = st->idx[k];
        const double dx = c->x[i] - c->x[p];
        const double dy = c->y[i] - c->y[p];
        double qti[4], qt0[4];
        for (int j = 0; j < 4; ++j) {
            qti[j] = q[4 * i + j] - 0.5 * (dx * qx[4 * i + j] + dy * qy[4 * i + j]);
            qt0[j] = q[4 * p + j] - 0.5 * (dx * qx[4 * p + j] + dy * qy[4 * p + j]);
        }
        if (!(qti[3] < 0.0) || !(qt0[3] < 0.0) || !all_finite4(qti) || !all_finite4(qt0))
            return 1;
        prim_t wi, w0;
        if (prim_from_q(qti, &wi)) return 1;
        if (prim_from_q(qt0, &w0)) return 1;
        double Gi[4], G0[4];
        split_flux_prim(&wi, axis, sign, Gi);
        split_flux_prim(&w0, axis, sign, G0);
        for (int j = 0; j < 4; ++j) R[j] += st->w[k] * (Gi[j] - G0[j]);
    }
    return 0;
}

/* accumulate_first_order, spatial.cpp:234-245; 0 ok, 1 invalid base state */
static int acc_first(const list_t* st, int p, int axis, int sign, const double* q, double* R)
{
    double G0[4] = {0, 0, 0, 0};
    if (st->off[p + 1] > st->off[p]) {
        prim_t w;
        if (prim_from_q(q + 4 * p, &w)) return 1;
        split_flux_prim(&w, axis, sign, G0);
    }
    for (int k = st->off[p]; k < st->off[p + 1]; ++k) {
        if (st->w[k] == 0.0) continue;
        prim_t w;
        if (prim_from_q(q + 4 * st->idx[k], &w)) return 1;
        double Gi[4];
        split_flux_prim(&w, axis, sign, Gi);
        for (int j = 0; j < 4; ++j) R[j] += st->w[k] * (Gi[j] - G0[j]);
    }
    return 0;
}

/* flux_residual, spatial.cpp:249-298 */
int kfo_residual(const kfo_cloud* c, const double* q, const double* qx, const double* qy,
                 int first_order, double* R, int* demoted, kfo_err* e)
{
    const int n = c->n;
    int bad = -1;
#pragma omp parallel for schedule(static)
    for (int p = 0; p < n; ++p) {
        double acc[4] = {0, 0, 0, 0};
        int ok = !first_order;
        if (ok) {
            for (int d = 0; d < 4; ++d)
                if (acc_second(c, dir_list(c, d), p, d / 2, d % 2, q, qx, qy, acc)) {
                    ok = 0;
                    break;
                }
        }
        if (demoted) demoted[p] = 0;
        if (!ok) {
            for (int j = 0; j < 4; ++j) acc[j] = 0.0;
            if (!first_order && demoted) demoted[p] = 1;
            int fail = 0;
            for (int d = 0; d < 4 && !fail; ++d)
                fail = acc_first(dir_list(c, d), p, d / 2, d % 2, q, acc);
            if (fail) {
#pragma omp critical
                if (bad < 0 || p < bad) bad = p;
                continue;
            }
        }
        for (int j = 0; j < 4; ++j) R[4 * p + j] = acc[j];
    }
    if (bad >= 0) {
        set_err(e, 1, bad, "flux_residual: invalid base state");
        return 1;
    }
    return 0;
}

/* local_timestep, driver.cpp:24-47 */
int kfo_timestep(const kfo_cloud* c, const double* U, double cfl, double* dt, kfo_err* e)
{
    int bad = -1;
#pragma omp parallel for schedule(static)
    for (int p = 0; p < c->n; ++p) {
        double h = DBL_MAX;
        for (int k = c->nbr.off[p]; k < c->nbr.off[p + 1]; ++k) {
            const int q = c->nbr.idx[k];
            const double v = hypot(c->x[q] - c->x[p], c->y[q] - c->y[p]);
            h = (v < h) ? v : h; /* std::min(h, v) */
        }
        prim_t w;
        if (prim_from_cons(U + 4 * p, &w)) {
#pragma omp critical
            if (bad < 0 || p < bad) bad = p;
            continue;
        }
        const double speed = hypot(w.u1, w.u2) + sound_speed(&w);
        dt[p] = cfl * h / speed;
    }
    if (bad >= 0) {
        set_err(e, 1, bad, "local_timestep: invalid state");
        return 1;
    }
    return 0;
}

/* compute_s_term, implicit.cpp:96-134 */
int kfo_s_term(const kfo_cloud* c, const double* U, const double* dU_prev, int exact,
               double* S, int* n_fallback, kfo_err* e)
{
    int bad = -1, nf = 0;
#pragma omp parallel for schedule(static) reduction(+ : nf)
    for (int p = 0; p < c->n; ++p) {
        const double cx = c->xpos.one[p] + c->xneg.one[p];
        const double cy = c->ypos.one[p] + c->yneg.one[p];
        double ax[4], ay[4];
        int r = mode_jvp_full(exact, U + 4 * p, dU_prev + 4 * p, 0, ax);
        if (r == 0) r = mode_jvp_full(exact, U + 4 * p, dU_prev + 4 * p, 1, ay);
        if (r == 2) {
            nf++;
            r = mode_jvp_full(1, U + 4 * p, dU_prev + 4 * p, 0, ax);
            if (r == 0) r = mode_jvp_full(1, U + 4 * p, dU_prev + 4 * p, 1, ay);
        }
        if (r) {
#pragma omp critical
            if (bad < 0 || p < bad) bad = p;
            continue;
        }
        for (int j = 0; j < 4; ++j) S[4 * p + j] = (-0.5 * cx) * ax[j] + (-0.5 * cy) * ay[j];
    }
    if (n_fallback) *n_fallback = nf;
    if (bad >= 0) {
        set_err(e, 1, bad, "s-term: invalid base state");
        return 1;
    }
    return 0;
}

/* assemble_diagonal, implicit.cpp:39-94 */
int kfo_diagonal(const kfo_cloud* c, const double* U, const double* dt, int variant, double* d,
                 kfo_err* e)
{
    const int with_s = (variant == 3 || variant == 4);
    int bad = -1;
#pragma omp parallel for schedule(static)
    for (int p = 0; p < c->n; ++p) {
        prim_t w;
        if (!(dt[p] > 0.0) || prim_from_cons(U + 4 * p, &w)) {
#pragma omp critical
            if (bad < 0 || p < bad) bad = p;
            continue;
        }
        double v = 1.0 / dt[p];
        if (with_s) {
            v += 0.5 * srad_full(&w, 0) * (c->xpos.one[p] - c->xneg.one[p]);
            v += 0.5 * srad_full(&w, 1) * (c->ypos.one[p] - c->yneg.one[p]);
        } else {
            v -= srad_split(&w, 0, 0) * c->xneg.one[p];
            v += srad_split(&w, 0, 1) * c->xpos.one[p];
            v -= srad_split(&w, 1, 0) * c->yneg.one[p];
            v += srad_split(&w, 1, 1) * c->ypos.one[p];
        }
        d[p] = v;
        if (!(v > 0.0)) {
#pragma omp critical
            if (bad < 0 || p < bad) bad = p;
        }
    }
    if (bad >= 0) {
        if (e) {
            e->code = 1;
            e->point = bad;
            snprintf(e->msg, sizeof e->msg,
                     "implicit diagonal nonpositive at point %d (time step too large)", bad);
        }
        return 1;
    }
    return 0;
}

/* neighbour_products, implicit.cpp:153-170; 0 ok, else invalid */
static int nbr_products(const kfo_cloud* c, const double* U, const double* incr, int exact,
                        int p, int lower, double* acc)
{
    const int cp = c->color[p];
    for (int j = 0; j < 4; ++j) acc[j] = 0.0;
    for (int d = 0; d < 4; ++d) {
        const list_t* st = dir_list(c, d);
        for (int k = st->off[p]; k < st->off[p + 1]; ++k) {
            if (st->w[k] == 0.0) continue;
            const int i = st->idx[k];
            const int ci = c->color[i];
            if (lower ? (ci >= cp) : (ci <= cp)) continue;
            double J[4];
            if (mode_jvp_split(exact, U + 4 * i, incr + 4 * i, d / 2, d % 2, J)) return 1;
            for (int j = 0; j < 4; ++j) acc[j] += st->w[k] * J[j];
        }
    }
    return 0;
}

/* forward_sweep + backward_sweep, implicit.cpp:174-226 */
int kfo_sweeps(const kfo_cloud* c, const double* U, const double* R, const double* S,
               const double* d, int exact, double* dUs, double* dU, kfo_err* e)
{
    const int n = c->n;
    memset(dUs, 0, sizeof(double) * 4 * (size_t)n);
    for (int g = 0; g < c->n_colors; ++g) {
        const int* grp = c->groups[g];
        const int ng = c->group_size[g];
        int bad = -1;
#pragma omp parallel for schedule(static)
        for (int t = 0; t < ng; ++t) {
            const int p = grp[t];
            double rhs[4], acc[4];
            for (int j = 0; j < 4; ++j) rhs[j] = R[4 * p + j];
            if (S)
                for (int j = 0; j < 4; ++j) rhs[j] -= S[4 * p + j];
            if (nbr_products(c, U, dUs, exact, p, 1, acc)) {
#pragma omp critical
                if (bad < 0 || p < bad) bad = p;
                continue;
            }
            for (int j = 0; j < 4; ++j) rhs[j] += acc[j];
            const double f = -1.0 / d[p];
            for (int j = 0; j < 4; ++j) dUs[4 * p + j] = f * rhs[j];
        }
        if (bad >= 0) {
            set_err(e, 1, bad, "forward sweep: invalid state encountered");
            return 1;
        }
    }
    memset(dU, 0, sizeof(double) * 4 * (size_t)n);
    for (int g = c->n_colors - 1; g >= 0; --g) {
        const int* grp = c->groups[g];
        const int ng = c->group_size[g];
        int bad = -1;
#pragma omp parallel for schedule(static)
        for (int t = 0; t < ng; ++t) {
            const int p = grp[t];
            double up[4];
            if (nbr_products(c, U, dU, exact, p, 0, up)) {
#pragma omp critical
                if (bad < 0 || p < bad) bad = p;
                continue;
            }
            const double f = 1.0 / d[p];
            for (int j = 0; j < 4; ++j) dU[4 * p + j] = dUs[4 * p + j] - f * up[j];
        }
        if (bad >= 0) {
            set_err(e, 1, bad, "backward sweep: invalid state encountered");
            return 1;
        }
    }
    return 0;
}

/* nearest_interior_neighbour, driver.cpp:51-65 */
static int nearest_interior(const kfo_cloud* c, int p)
{
    int best = -1;
    double best_d = DBL_MAX;
    for (int k = c->nbr.off[p]; k < c->nbr.off[p + 1]; ++k) {
        const int q = c->nbr.idx[k];
        if (c->kind[q] != 1) continue;
        const double dd = hypot(c->x[q] - c->x[p], c->y[q] - c->y[p]);
        if (dd < best_d) {
            best_d = dd;
            best = q;
        }
    }
    return best;
}

/* apply_boundary_conditions, driver.cpp:69-95 */
int kfo_bc(const kfo_cloud* c, double* U, double mach, double aoa, int bc_mode, kfo_err* e)
{
    prim_t fw;
    double fU[4];
    freestream(mach, aoa, &fw, fU);
    if (bc_mode) {
        for (int t = 0; t < c->n_wall; ++t) memcpy(U + 4 * c->wall[t], fU, sizeof fU);
        for (int t = 0; t < c->n_outer; ++t) memcpy(U + 4 * c->outer[t], fU, sizeof fU);
        return 0;
    }
    for (int t = 0; t < c->n_wall; ++t) {
        const int p = c->wall[t];
        prim_t w;
        const int r = prim_from_cons(U + 4 * p, &w);
        if (r) {
            set_err(e, 1, p, r == 1 ? "nonpositive density" : "nonpositive pressure");
            return 1;
        }
        const double un = w.u1 * c->nx[p] + w.u2 * c->ny[p];
        w.u1 -= un * c->nx[p];
        w.u2 -= un * c->ny[p];
        cons_from_prim(&w, U + 4 * p);
    }
    for (int t = 0; t < c->n_outer; ++t) {
        const int p = c->outer[t];
        prim_t w;
        const int r = prim_from_cons(U + 4 * p, &w);
        if (r) {
            set_err(e, 1, p, r == 1 ? "nonpositive density" : "nonpositive pressure");
            return 1;
        }
        const double un = w.u1 * c->nx[p] + w.u2 * c->ny[p];
        if (un < 0.0) {
            memcpy(U + 4 * p, fU, sizeof fU);
        } else {
            const int q = nearest_interior(c, p);
            if (q >= 0)
                memcpy(U + 4 * p, U + 4 * q, 4 * sizeof(double));
            else
                memcpy(U + 4 * p, fU, sizeof fU);
        }
    }
    return 0;
}

/* compute_forces + surface_cp, driver.cpp:114-167 */
int kfo_forces(const kfo_cloud* c, const double* U, double mach, double aoa, double* cl,
               double* cd, kfo_err* e)
{
    const int W = c->n_wall;
    const int* wall = c->wall;
    if (W < 3) {
        set_err(e, 2, -1, "compute_forces: no usable wall loop");
        return 1;
    }
    for (int k = 0; k < W; ++k) {
        const int a = wall[k], b = wall[(k + 1) % W];
        if (hypot(c->x[b] - c->x[a], c->y[b] - c->y[a]) > 0.5) {
            set_err(e, 2, -1, "compute_forces: wall points are not ordered along the surface");
            return 1;
        }
    }
    prim_t fw;
    double fU[4];
    freestream(mach, aoa, &fw, fU);
    const double qdyn = 0.5 * fw.rho * mach * mach;
    double* cp = malloc(sizeof(double) * (size_t)W);
    for (int k = 0; k < W; ++k) {
        prim_t w;
        const int r = prim_from_cons(U + 4 * wall[k], &w);
        if (r) {
            set_err(e, 1, wall[k], r == 1 ? "nonpositive density" : "nonpositive pressure");
            free(cp);
            return 1;
        }
        cp[k] = (w.p - fw.p) / qdyn;
    }
    double area2 = 0.0;
    for (int k = 0; k < W; ++k) {
        const int a = wall[k], b = wall[(k + 1) % W];
        area2 += c->x[a] * c->y[b] - c->x[b] * c->y[a];
    }
    const double orient = (area2 >= 0.0) ? 1.0 : -1.0;
    double fx = 0.0, fy = 0.0;
    for (int k = 0; k < W; ++k) {
        const int a = wall[k], b = wall[(k + 1) % W];
        const double tx = c->x[b] - c->x[a];
        const double ty = c->y[b] - c->y[a];
        const double cpm = 0.5 * (cp[k] + cp[(k + 1) % W]);
        fx -= cpm * orient * ty;
        fy -= cpm * orient * (-tx);
    }
    free(cp);
    const double alpha = aoa * M_PI / 180.0;
    *cd = fx * cos(alpha) + fy * sin(alpha);
    *cl = -fx * sin(alpha) + fy * cos(alpha);
    return 0;
}

/* run_fixed_point, driver.cpp:188-282 (implicit and explicit variants) */
int kfo_run(const kfo_cloud* c, const kfo_config* cfg, int* n_done, double* residual,
            double* cl, double* cd, int* first_order, double* final_state, int* diverged,
            char* reason, int reason_len)
{
    const int n = c->n;
    *n_done = 0;
    *diverged = 0;
    if (reason_len > 0) reason[0] = 0;
    if (!(cfg->cfl > 0.0)) {
        snprintf(reason, (size_t)reason_len, "cfl must be positive");
        return 1;
    }
    if (cfg->n_iterations < 1) {
        snprintf(reason, (size_t)reason_len, "n_iterations must be >= 1");
        return 1;
    }
    for (int t = 0; t < c->n_flagged; ++t)
        if (c->kind[c->flagged[t]] == 1) {
            snprintf(reason, (size_t)reason_len,
                     "interior point %d has a singular least-squares stencil", c->flagged[t]);
            return 1;
        }
    if (!(cfg->mach > 0.0)) {
        snprintf(reason, (size_t)reason_len, "freestream Mach must be positive");
        return 1;
    }
    const int implicit = cfg->variant != 0;
    const int with_s = cfg->variant == 3 || cfg->variant == 4;
    const int exact = cfg->variant == 2 || cfg->variant == 4;
    prim_t fw;
    double fU[4];
    freestream(cfg->mach, cfg->aoa_deg, &fw, fU);

    double* state = malloc(sizeof(double) * 4 * (size_t)n);
    for (int p = 0; p < n; ++p) memcpy(state + 4 * p, fU, sizeof fU);
    kfo_err e = {0, -1, ""};
    kfo_bc(c, state, cfg->mach, cfg->aoa_deg, cfg->bc_mode, &e);

    double* dU_prev = calloc(4 * (size_t)n, sizeof(double));
    double* q = malloc(sizeof(double) * 4 * (size_t)n);
    double* qx = malloc(sizeof(double) * 4 * (size_t)n);
    double* qy = malloc(sizeof(double) * 4 * (size_t)n);
    double* R = malloc(sizeof(double) * 4 * (size_t)n);
    double* S = malloc(sizeof(double) * 4 * (size_t)n);
    double* dUs = malloc(sizeof(double) * 4 * (size_t)n);
    double* dU = malloc(sizeof(double) * 4 * (size_t)n);
    double* dt = malloc(sizeof(double) * (size_t)n);
    double* d = malloc(sizeof(double) * (size_t)n);
    int* dem = malloc(sizeof(int) * (size_t)n);
    double res0 = -1.0;
    int aborted = 0;

    for (int it = 1; it <= cfg->n_iterations; ++it) {
        double cfl = cfg->cfl;
        if (cfg->cfl_ramp_iters > 0 && it < cfg->cfl_ramp_iters) {
            const double c0 = (cfg->cfl_start > 0.0) ? cfg->cfl_start : 0.1 * cfg->cfl;
            cfl = c0 + (cfg->cfl - c0) * it / cfg->cfl_ramp_iters;
        }
        int fail = kfo_q(c, state, q, &e);
        if (!fail) {
            kfo_grads(c, q, cfg->n_inner, qx, qy);
            fail = kfo_residual(c, q, qx, qy, 0, R, dem, &e);
        }
        int nfo = 0;
        if (!fail)
            for (int p = 0; p < n; ++p) nfo += dem[p];
        if (!fail) fail = kfo_timestep(c, state, cfl, dt, &e);
        if (!fail) {
            if (implicit) {
                if (with_s) fail = kfo_s_term(c, state, dU_prev, exact, S, NULL, &e);
                if (!fail) fail = kfo_diagonal(c, state, dt, cfg->variant, d, &e);
                if (!fail) fail = kfo_sweeps(c, state, R, with_s ? S : NULL, d, exact, dUs, dU, &e);
                if (!fail) {
                    for (int p = 0; p < 4 * n; ++p) state[p] += dU[p];
                    for (int p = 0; p < n && !fail; ++p) {
                        prim_t w;
                        const int r = prim_from_cons(state + 4 * p, &w);
                        if (r) {
                            set_err(&e, 1, p, r == 1 ? "nonpositive density" : "nonpositive pressure");
                            fail = 1;
                        }
                    }
                }
                if (!fail) fail = kfo_bc(c, state, cfg->mach, cfg->aoa_deg, cfg->bc_mode, &e);
                if (!fail) memcpy(dU_prev, dU, sizeof(double) * 4 * (size_t)n);
            } else {
                /* explicit_update, driver.cpp:97-112 */
                for (int p = 0; p < n && !fail; ++p) {
                    for (int j = 0; j < 4; ++j) state[4 * p + j] -= dt[p] * R[4 * p + j];
                    prim_t w;
                    if (prim_from_cons(state + 4 * p, &w)) {
                        set_err(&e, 1, p,
                                "explicit update left the valid-state set (time step too large?)");
                        fail = 1;
                    }
                }
                if (!fail) fail = kfo_bc(c, state, cfg->mach, cfg->aoa_deg, cfg->bc_mode, &e);
            }
        }
        double rc = 0.0, rl = 0.0, rd = 0.0;
        if (!fail) {
            double ss = 0.0;
            for (int p = 0; p < n; ++p) ss += R[4 * p] * R[4 * p];
            rc = sqrt(ss / n);
            fail = kfo_forces(c, state, cfg->mach, cfg->aoa_deg, &rl, &rd, &e);
        }
        if (fail) {
            *diverged = 1;
            snprintf(reason, (size_t)reason_len, "%s", e.msg);
            aborted = 1;
            break;
        }
        const int k = (*n_done)++;
        residual[k] = rc;
        cl[k] = rl;
        cd[k] = rd;
        if (first_order) first_order[k] = nfo;
        if (it == 1) res0 = rc;
        if (rc > cfg->divergence_factor * (res0 > 1e-300 ? res0 : 1e-300)) {
            *diverged = 1;
            snprintf(reason, (size_t)reason_len, "residual diverged");
            break;
        }
        if (cfg->convergence_decades > 0.0 && res0 > 0.0 &&
            rc <= res0 * pow(10.0, -cfg->convergence_decades))
            break;
    }
    (void)aborted;
    if (final_state) memcpy(final_state, state, sizeof(double) * 4 * (size_t)n);
    free(state); free(dU_prev); free(q); free(qx); free(qy); free(R); free(S); free(dUs);
    free(dU); free(dt); free(d); free(dem);
    return 0;
}

/* ---------------- point physics probes ---------------- */

int kfo_split_flux(const double* U, int axis, int sign, double* G)
{
    return split_flux_cons(U, axis, sign, G);
}

int kfo_jvp_split(const double* U, const double* dU, int axis, int sign, int exact, double* out)
{
    return mode_jvp_split(exact, U, dU, axis, sign, out);
}

int kfo_jvp_full(const double* U, const double* dU, int axis, int exact, double* out)
{
    return mode_jvp_full(exact, U, dU, axis, out);
}
