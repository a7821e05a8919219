/*
 * biewos_patch.c — CPU ORACLE (test infrastructure only) for the local-BIE
 * collocation of the DtN path: patch mesh, sphere Green's functions, triangle
 * quadratures, second-kind assembly and the dense solve. Restates
 *   greens.cpp:21-89,165-192     (image terms, dG/dn_x, d2G/dn_x dn_y)
 *   quadrature.cpp:73-87, quadrature.hpp:48-98 (deg-5 rule, polar/split/refined)
 *   patch_solver.cpp:14-52      (frame, band mesh)
 *   patch_solver.cpp:62-121     (sphere / flat patch setup; generalised to an
 *                                interior-side sphere, any sphere centre and any
 *                                face normal — the BASELINE geometries)
 *   patch_solver.cpp:197-309    (assemble, second and first kind)
 *   patch_solver.cpp:311-324    (LU solve, residual, est_error)
 * with one deliberate change: the Gamma integral uses the
 * theta-Gauss-Legendre x phi-uniform WOS nodes directly (any node list with
 * weights is accepted) instead of bilinear interpolation of a uniform grid.
 * Only tests/, smoke() and bench.py's CPU legs load this file.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/biewos_b200.h"

#define PI 3.14159265358979323846
static const double kInv4Pi = 1.0 / (4.0 * PI); /* greens.cpp:9 */

typedef struct { double v[3]; } v3;
static inline v3 mk(double x, double y, double z) { v3 r = {{x, y, z}}; return r; }
static inline v3 add(v3 a, v3 b) { return mk(a.v[0] + b.v[0], a.v[1] + b.v[1], a.v[2] + b.v[2]); }
static inline v3 sub(v3 a, v3 b) { return mk(a.v[0] - b.v[0], a.v[1] - b.v[1], a.v[2] - b.v[2]); }
static inline v3 scl(double s, v3 a) { return mk(s * a.v[0], s * a.v[1], s * a.v[2]); }
static inline v3 dvs(v3 a, double s) { return mk(a.v[0] / s, a.v[1] / s, a.v[2] / s); }
static inline double dot(v3 a, v3 b) { return a.v[0] * b.v[0] + a.v[1] * b.v[1] + a.v[2] * b.v[2]; }
static inline double nrm(v3 a) { return sqrt(dot(a, a)); }
static inline v3 cross(v3 a, v3 b) {
    return mk(a.v[1] * b.v[2] - a.v[2] * b.v[1], a.v[2] * b.v[0] - a.v[0] * b.v[2],
              a.v[0] * b.v[1] - a.v[1] * b.v[0]);
}
static inline v3 ld(const double* p) { return mk(p[0], p[1], p[2]); }

int or_gauss_legendre(int n, double* nodes, double* weights); /* biewos_oracle.c */

/* ---------------- sphere Green's function (greens.cpp:21-39,165-192) ------- */
typedef struct {
    double c;
    v3 p, gradc;
    double jac[3][3];
} term;

/* returns 0 or BW_ERR_SINGULARITY; y relative to the sphere centre */
static int build_terms(double a, v3 y, term t[2]) {
    const double rho = nrm(y);
    if (rho < 1e-14 * a) return BW_ERR_SINGULARITY;
    const v3 yh = dvs(y, rho);
    const double k = a * a / (rho * rho);
    t[0].c = 1.0;
    t[0].p = y;
    t[0].gradc = mk(0, 0, 0);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) t[0].jac[i][j] = i == j ? 1.0 : 0.0;
    t[1].c = -a / rho;
    t[1].p = scl(k, y);
    t[1].gradc = scl(a / (rho * rho), yh);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            t[1].jac[i][j] = k * ((i == j ? 1.0 : 0.0) - 2.0 * yh.v[i] * yh.v[j]);
    return 0;
}

static v3 jmul(const double J[3][3], v3 v) {
    return mk(J[0][0] * v.v[0] + J[0][1] * v.v[1] + J[0][2] * v.v[2],
              J[1][0] * v.v[0] + J[1][1] * v.v[1] + J[1][2] * v.v[2],
              J[2][0] * v.v[0] + J[2][1] * v.v[1] + J[2][2] * v.v[2]);
}

/* sphere_dg_dnx (greens.cpp:79-89,177-181): x, y absolute */
double or_sphere_dg_dnx(const double* c, double a, const double* x, const double* nx,
                        const double* y, int* err) {
    term t[2];
    if (build_terms(a, sub(ld(y), ld(c)), t)) { *err = BW_ERR_SINGULARITY; return NAN; }
    const v3 xl = sub(ld(x), ld(c));
    double s = 0;
    for (int i = 0; i < 2; ++i) {
        const v3 r = sub(xl, t[i].p);
        const double d = nrm(r);
        if (i == 0 && d < 1e-12 * a) { *err = BW_ERR_SINGULARITY; return NAN; }
        s += -t[i].c * dot(r, ld(nx)) / (d * d * d);
    }
    return kInv4Pi * s;
}

/* sphere_d2g (greens.cpp:51-65,185-190) */
double or_sphere_d2g(const double* c, double a, const double* x, const double* nx,
                     const double* y, const double* ny, int* err) {
    term t[2];
    if (build_terms(a, sub(ld(y), ld(c)), t)) { *err = BW_ERR_SINGULARITY; return NAN; }
    const v3 xl = sub(ld(x), ld(c));
    const v3 NX = ld(nx), NY = ld(ny);
    double s = 0;
    for (int i = 0; i < 2; ++i) {
        const v3 r = sub(xl, t[i].p);
        const double d = nrm(r);
        if (i == 0 && d < 1e-12 * a) { *err = BW_ERR_SINGULARITY; return NAN; }
        const double d3 = d * d * d;
        const v3 dp = jmul(t[i].jac, NY);
        const double rnx = dot(r, NX);
        s += -(dot(t[i].gradc, NY)) * rnx / d3 + t[i].c * dot(dp, NX) / d3 -
             3.0 * t[i].c * rnx * dot(r, dp) / (d3 * d * d);
    }
    return kInv4Pi * s;
}

/* sphere_g (greens.cpp:41-49 eval_g, first-kind A entries) */
double or_sphere_g(const double* c, double a, const double* x, const double* y, int* err) {
    term t[2];
    if (build_terms(a, sub(ld(y), ld(c)), t)) { *err = BW_ERR_SINGULARITY; return NAN; }
    const v3 xl = sub(ld(x), ld(c));
    double s = 0;
    for (int i = 0; i < 2; ++i) {
        const double d = nrm(sub(xl, t[i].p));
        if (i == 0 && d < 1e-12 * a) { *err = BW_ERR_SINGULARITY; return NAN; }
        s += t[i].c / d;
    }
    return kInv4Pi * s;
}

/* sphere_dg_dny (greens.cpp:67-77 eval_dg_dny, first-kind b and Gamma terms) */
double or_sphere_dg_dny(const double* c, double a, const double* x, const double* y,
                        const double* ny, int* err) {
    term t[2];
    if (build_terms(a, sub(ld(y), ld(c)), t)) { *err = BW_ERR_SINGULARITY; return NAN; }
    const v3 xl = sub(ld(x), ld(c));
    const v3 NY = ld(ny);
    double s = 0;
    for (int i = 0; i < 2; ++i) {
        const v3 r = sub(xl, t[i].p);
        const double d = nrm(r);
        if (i == 0 && d < 1e-12 * a) { *err = BW_ERR_SINGULARITY; return NAN; }
        s += dot(t[i].gradc, NY) / d + t[i].c * dot(r, jmul(t[i].jac, NY)) / (d * d * d);
    }
    return kInv4Pi * s;
}

/* ---------------- triangle quadrature (quadrature.cpp:73-87, .hpp:48-98) --- */
static const double kTriW[7] = {0.225, 0.132394152788506, 0.132394152788506, 0.132394152788506,
                                0.125939180544827, 0.125939180544827, 0.125939180544827};
static const double kTriB[7][3] = {{1.0 / 3, 1.0 / 3, 1.0 / 3},
                                   {0.059715871789770, 0.470142064105115, 0.470142064105115},
                                   {0.470142064105115, 0.059715871789770, 0.470142064105115},
                                   {0.470142064105115, 0.470142064105115, 0.059715871789770},
                                   {0.797426985353087, 0.101286507323456, 0.101286507323456},
                                   {0.101286507323456, 0.797426985353087, 0.101286507323456},
                                   {0.101286507323456, 0.101286507323456, 0.797426985353087}};

typedef struct {
    int kind;         /* 0: dG/dn_x, 1: d2G (b-term, times (phi(y) - u_i)),
                         2: G, 3: dG/dn_y (first-kind b-term, times (phi(y) - u_i)) */
    const double* c;  /* Green sphere centre */
    double a;
    v3 x, nx, ny;
    /* surface for eval_dirichlet of quadrature points */
    const bw_scene* scene;
    int surf;         /* 0 sphere (centre sc, radius R), 1 plane (point sp, normal sn) */
    v3 sc;
    double R;
    v3 sn;
    double ui;
    int err;
} kctx;

double or_eval_phi(const bw_scene* s, const double y[3], int feature);

/* eval_dirichlet (geometry.cpp:198-220) at a quadrature point of the patch:
 * project onto the patch's own surface and evaluate the closed-form data. */
static double dirichlet_on_patch(const kctx* k, v3 y) {
    v3 p;
    if (k->surf == 0) {
        const v3 q = sub(y, k->sc);
        p = add(k->sc, scl(k->R / nrm(q), q));
    } else {
        p = sub(y, scl(dot(sub(y, k->sc), k->sn), k->sn));
    }
    return or_eval_phi(k->scene, p.v, 0);
}

static double kern(kctx* k, v3 y) {
    int err = 0;
    double v;
    if (k->kind == 0) {
        v = or_sphere_dg_dnx(k->c, k->a, k->x.v, k->nx.v, y.v, &err);
    } else if (k->kind == 1) {
        v = or_sphere_d2g(k->c, k->a, k->x.v, k->nx.v, y.v, k->ny.v, &err) *
            (dirichlet_on_patch(k, y) - k->ui);
    } else if (k->kind == 2) {
        v = or_sphere_g(k->c, k->a, k->x.v, y.v, &err);
    } else {
        v = or_sphere_dg_dny(k->c, k->a, k->x.v, y.v, k->ny.v, &err) *
            (dirichlet_on_patch(k, y) - k->ui);
    }
    if (err) k->err = err;
    return v;
}

static double integrate_triangle(v3 v0, v3 v1, v3 v2, kctx* k) {
    const double area = 0.5 * nrm(cross(sub(v1, v0), sub(v2, v0)));
    double s = 0;
    for (int i = 0; i < 7; ++i) {
        const v3 p = add(add(scl(kTriB[i][0], v0), scl(kTriB[i][1], v1)), scl(kTriB[i][2], v2));
        s += kTriW[i] * kern(k, p);
    }
    return area * s;
}

static double integrate_polar(v3 v0, v3 v1, v3 v2, int n, const double* gx, const double* gw,
                              kctx* k) {
    const double area2 = nrm(cross(sub(v1, v0), sub(v2, v0)));
    double sum = 0;
    for (int i = 0; i < n; ++i) {
        const double s = 0.5 * (gx[i] + 1.0);
        const v3 w = add(v1, scl(s, sub(v2, v1)));
        double inner = 0;
        for (int j = 0; j < n; ++j) {
            const double t = 0.5 * (gx[j] + 1.0);
            inner += 0.25 * gw[j] * t * kern(k, add(v0, scl(t, sub(w, v0))));
        }
        sum += gw[i] * inner;
    }
    return area2 * sum;
}

static double integrate_split(v3 v0, v3 v1, v3 v2, v3 x, int n, const double* gx,
                              const double* gw, kctx* k) {
    return integrate_polar(x, v0, v1, n, gx, gw, k) + integrate_polar(x, v1, v2, n, gx, gw, k) +
           integrate_polar(x, v2, v0, n, gx, gw, k);
}

static double integrate_refined(v3 v0, v3 v1, v3 v2, int depth, kctx* k) {
    if (depth <= 0) return integrate_triangle(v0, v1, v2, k);
    const v3 m01 = scl(0.5, add(v0, v1)), m12 = scl(0.5, add(v1, v2)), m20 = scl(0.5, add(v2, v0));
    return integrate_refined(v0, m01, m20, depth - 1, k) +
           integrate_refined(m01, v1, m12, depth - 1, k) +
           integrate_refined(m20, m12, v2, depth - 1, k) +
           integrate_refined(m01, m12, m20, depth - 1, k);
}

/* ---------------- patch setup + mesh (patch_solver.cpp:14-121) ------------ */
/* Patch description (one boundary point):
 *   o[3]     patch centre on the boundary
 *   axis[3]  unit normal INTO the solution domain (Gamma pole)
 *   a        sphere radius
 *   surf     0: the boundary near o is the sphere |y - sc| = R
 *            1: the boundary near o is the plane through o with normal axis
 * The mesh is the reference's fan + band triangulation: ring k (1..bands) at
 * geodesic angle alpha_max k / bands (sphere, alpha_max = acos(1 - a^2/2R^2))
 * or radius a k / bands (plane), azimuth 2 pi j / azimuth, in the frame of the
 * RADIAL direction (sphere) or of the axis (plane); normals oriented into the
 * solution domain. m = azimuth (2 bands - 1) panels. */
typedef struct {
    int m, nv;
    double* verts;    /* nv x 3 */
    int* tris;        /* m x 3 */
    double* cen;      /* m x 3 */
    double* nrm;      /* m x 3 */
    double* area;     /* m */
    double* diam;     /* m */
} or_mesh;

static void frame_rows(v3 ax, v3* e1, v3* e2) { /* patch_solver.cpp:14-23 */
    const v3 ref = fabs(ax.v[0]) < 0.9 ? mk(1, 0, 0) : mk(0, 1, 0);
    v3 c = cross(ax, ref);
    *e1 = dvs(c, nrm(c));
    *e2 = cross(ax, *e1);
}

int or_patch_mesh_size(int bands, int azimuth, int* m, int* nv) {
    *m = azimuth * (2 * bands - 1);
    *nv = 1 + bands * azimuth;
    return 0;
}

/* Fills caller-allocated arrays (sizes from or_patch_mesh_size). */
int or_patch_mesh(const double* o_, const double* axis_, int surf, const double* sc_, double R,
                  double a, int bands, int azimuth, double* verts, int* tris, double* cen,
                  double* nrm_, double* area, double* diam) {
    const v3 o = ld(o_), axis = ld(axis_);
    v3 e1, e2, rad;
    if (surf == 0) {
        rad = dvs(sub(o, ld(sc_)), nrm(sub(o, ld(sc_))));
        frame_rows(rad, &e1, &e2);
    } else {
        rad = axis;
        frame_rows(axis, &e1, &e2);
    }
    const int M = azimuth;
    memcpy(verts, o.v, sizeof o.v);
    const double alpha_max = surf == 0 ? acos(1.0 - a * a / (2.0 * R * R)) : 0.0;
    for (int k = 1; k <= bands; ++k) {
        for (int j = 0; j < M; ++j) {
            const double beta = 2.0 * PI * j / M;
            v3 v;
            if (surf == 0) {
                const double al = alpha_max * k / bands;
                const v3 loc = mk(sin(al) * cos(beta), sin(al) * sin(beta), cos(al));
                /* R * (rot^T * local) + centre (patch_solver.cpp:80-83) */
                const v3 w = add(add(scl(loc.v[0], e1), scl(loc.v[1], e2)), scl(loc.v[2], rad));
                v = add(ld(sc_), scl(R, w));
            } else {
                const double r = a * k / bands;
                v = add(o, add(scl(r * cos(beta), e1), scl(r * sin(beta), e2)));
            }
            memcpy(verts + 3 * (1 + (k - 1) * M + j), v.v, sizeof v.v);
        }
    }
#define VID(ring, j) (1 + (ring) * M + ((j) % M))
    int t = 0;
    for (int j = 0; j < M; ++j) { /* fan (patch_solver.cpp:31) */
        tris[3 * t] = 0; tris[3 * t + 1] = VID(0, j); tris[3 * t + 2] = VID(0, j + 1); ++t;
    }
    for (int k = 0; k + 1 < bands; ++k)
        for (int j = 0; j < M; ++j) { /* bands (patch_solver.cpp:32-36) */
            tris[3 * t] = VID(k, j); tris[3 * t + 1] = VID(k + 1, j); tris[3 * t + 2] = VID(k + 1, j + 1); ++t;
            tris[3 * t] = VID(k, j); tris[3 * t + 1] = VID(k + 1, j + 1); tris[3 * t + 2] = VID(k, j + 1); ++t;
        }
#undef VID
    const double side = dot(axis, rad) >= 0 ? 1.0 : -1.0; /* interior sphere: flip */
    for (int i = 0; i < t; ++i) { /* patch_solver.cpp:37-50 */
        const v3 v0 = ld(verts + 3 * tris[3 * i]), v1 = ld(verts + 3 * tris[3 * i + 1]),
                 v2 = ld(verts + 3 * tris[3 * i + 2]);
        const v3 c = dvs(add(add(v0, v1), v2), 3.0);
        v3 n = cross(sub(v1, v0), sub(v2, v0));
        const double a2 = nrm(n);
        n = dvs(n, a2);
        const v3 outward = surf == 0 ? dvs(sub(c, ld(sc_)), nrm(sub(c, ld(sc_)))) : axis;
        if (dot(n, outward) < 0) n = scl(-1.0, n);
        n = scl(side, n);
        memcpy(cen + 3 * i, c.v, sizeof c.v);
        memcpy(nrm_ + 3 * i, n.v, sizeof n.v);
        area[i] = 0.5 * a2;
        double dm = nrm(sub(v1, v0));
        if (nrm(sub(v2, v1)) > dm) dm = nrm(sub(v2, v1));
        if (nrm(sub(v0, v2)) > dm) dm = nrm(sub(v0, v2));
        diam[i] = dm;
    }
    return 0;
}

/* ---------------- second-kind assembly (patch_solver.cpp:197-309) --------- */
/* Gamma: n_g nodes y (n_g x 3), full weights w (surface element included),
 * node means um and variances-of-the-mean uv (Estimate.variance / n).
 * Outputs A (m x m row-major), b (m), b_se (m). Returns 0 or an error. */
/* bie_kind: 0 second kind (the default, runner.cpp:192-193), 1 first kind
 * (A_ij = int G, b with dG/dn_y; patch_solver.cpp:285-305). */
int or_assemble_kind(const bw_scene* scene, const double* o, const double* axis, int surf,
                     const double* sc, double R, double a, int bands, int azimuth,
                     int gauss_polar, int near_depth, const double* gy, const double* gw_,
                     const double* um, const double* uv, int n_g, int bie_kind, double* A,
                     double* b, double* b_se) {
    const int ka = bie_kind == 1 ? 2 : 0, kb = bie_kind == 1 ? 3 : 1;
    const double diag = bie_kind == 1 ? 0.0 : 0.5;
    int m, nv;
    or_patch_mesh_size(bands, azimuth, &m, &nv);
    double* verts = malloc(sizeof(double) * 3 * nv);
    int* tris = malloc(sizeof(int) * 3 * m);
    double* cen = malloc(sizeof(double) * 3 * m);
    double* nr = malloc(sizeof(double) * 3 * m);
    double* area = malloc(sizeof(double) * m);
    double* diam = malloc(sizeof(double) * m);
    or_patch_mesh(o, axis, surf, sc, R, a, bands, azimuth, verts, tris, cen, nr, area, diam);
    double gx[64], gwt[64];
    or_gauss_legendre(gauss_polar, gx, gwt);

    kctx k;
    memset(&k, 0, sizeof k);
    k.c = o;
    k.a = a;
    k.scene = scene;
    k.surf = surf;
    k.sc = surf == 0 ? ld(sc) : ld(o);
    k.R = R;
    k.sn = ld(axis);
    int err = 0;
    for (int i = 0; i < m; ++i) {
        const v3 xi = ld(cen + 3 * i), ni = ld(nr + 3 * i);
        k.x = xi;
        k.nx = ni;
        k.ui = dirichlet_on_patch(&k, xi); /* eval_dirichlet at the centroid */
        double bg = 0, vg = 0;
        for (int g = 0; g < n_g; ++g) { /* Gamma term (patch_solver.cpp:253-262) */
            const v3 y = ld(gy + 3 * g);
            const v3 ny = dvs(sub(y, ld(o)), a);
            int e = 0;
            const double kk = bie_kind == 1 ? or_sphere_dg_dny(o, a, xi.v, y.v, ny.v, &e)
                                            : or_sphere_d2g(o, a, xi.v, ni.v, y.v, ny.v, &e);
            if (e) err = e;
            bg += gw_[g] * kk * (um[g] - k.ui);
            vg += gw_[g] * kk * gw_[g] * kk * uv[g];
        }
        b[i] = -bg;
        b_se[i] = sqrt(vg);
        for (int j = 0; j < m; ++j) { /* panel terms (patch_solver.cpp:264-306) */
            const v3 v0 = ld(verts + 3 * tris[3 * j]), v1 = ld(verts + 3 * tris[3 * j + 1]),
                     v2 = ld(verts + 3 * tris[3 * j + 2]);
            k.ny = ld(nr + 3 * j);
            const double dist = nrm(sub(xi, ld(cen + 3 * j)));
            double aij, bij;
            if (j == i) {
                k.kind = ka;
                aij = diag + integrate_split(v0, v1, v2, xi, gauss_polar, gx, gwt, &k);
                k.kind = kb;
                bij = integrate_split(v0, v1, v2, xi, gauss_polar, gx, gwt, &k);
            } else if (dist < 2.0 * diam[j]) {
                k.kind = ka;
                aij = integrate_refined(v0, v1, v2, near_depth, &k);
                k.kind = kb;
                bij = integrate_refined(v0, v1, v2, near_depth, &k);
            } else {
                k.kind = ka;
                aij = integrate_triangle(v0, v1, v2, &k);
                k.kind = kb;
                bij = integrate_triangle(v0, v1, v2, &k);
            }
            A[i * m + j] = aij;
            b[i] += bij;
        }
    }
    if (k.err) err = k.err;
    free(verts); free(tris); free(cen); free(nr); free(area); free(diam);
    return err;
}

int or_assemble(const bw_scene* scene, const double* o, const double* axis, int surf,
                const double* sc, double R, double a, int bands, int azimuth, int gauss_polar,
                int near_depth, const double* gy, const double* gw_, const double* um,
                const double* uv, int n_g, double* A, double* b, double* b_se) {
    return or_assemble_kind(scene, o, axis, surf, sc, R, a, bands, azimuth, gauss_polar,
                            near_depth, gy, gw_, um, uv, n_g, 0, A, b, b_se);
}

int or_lu_solve(int m, const double* A_in, const double* B, int nrhs, double* X, double* resid);

/* solve_patch + the point value (patch_solver.cpp:311-324): x = A^-1 b,
 * residual gate, est_error = |A^-1 b_se|; the Neumann value at o is the
 * area-weighted mean over the `azimuth` fan panels around the apex, with its
 * error from est_error. Returns 0, BW_ERR_SOLVER or an assembly error. */
int or_solve_patch_point_kind(const bw_scene* scene, const double* o, const double* axis,
                              int surf, const double* sc, double R, double a, int bands,
                              int azimuth, int gauss_polar, int near_depth, const double* gy,
                              const double* gw_, const double* um, const double* uv, int n_g,
                              int bie_kind, double* dudn, double* dudn_err, double* x_out,
                              double* resid_out) {
    int m, nv;
    or_patch_mesh_size(bands, azimuth, &m, &nv);
    double* A = malloc(sizeof(double) * m * m);
    double* B = malloc(sizeof(double) * 2 * m);
    double* X = malloc(sizeof(double) * 2 * m);
    int st = or_assemble_kind(scene, o, axis, surf, sc, R, a, bands, azimuth, gauss_polar,
                              near_depth, gy, gw_, um, uv, n_g, bie_kind, A, B, B + m);
    double resid = 0;
    if (!st) {
        const int info = or_lu_solve(m, A, B, 2, X, &resid);
        int finite = 1;
        for (int i = 0; i < m; ++i) finite &= isfinite(X[i]);
        if (info || !finite || resid > 1e-10) st = BW_ERR_SOLVER;
    }
    /* fan panels: indices 0..azimuth-1; areas recomputed */
    double* verts = malloc(sizeof(double) * 3 * nv);
    int* tris = malloc(sizeof(int) * 3 * m);
    double* cen = malloc(sizeof(double) * 3 * m);
    double* nr = malloc(sizeof(double) * 3 * m);
    double* area = malloc(sizeof(double) * m);
    double* diam = malloc(sizeof(double) * m);
    or_patch_mesh(o, axis, surf, sc, R, a, bands, azimuth, verts, tris, cen, nr, area, diam);
    double s = 0, se = 0, at = 0;
    for (int j = 0; j < azimuth; ++j) {
        s += area[j] * X[j];
        se += area[j] * fabs(X[m + j]);
        at += area[j];
    }
    *dudn = s / at;
    *dudn_err = se / at;
    if (x_out) memcpy(x_out, X, sizeof(double) * m);
    if (resid_out) *resid_out = resid;
    free(A); free(B); free(X); free(verts); free(tris); free(cen); free(nr); free(area); free(diam);
    return st;
}

int or_solve_patch_point(const bw_scene* scene, const double* o, const double* axis, int surf,
                         const double* sc, double R, double a, int bands, int azimuth,
                         int gauss_polar, int near_depth, const double* gy, const double* gw_,
                         const double* um, const double* uv, int n_g, double* dudn,
                         double* dudn_err, double* x_out, double* resid_out) {
    return or_solve_patch_point_kind(scene, o, axis, surf, sc, R, a, bands, azimuth, gauss_polar,
                                     near_depth, gy, gw_, um, uv, n_g, 0, dudn, dudn_err, x_out,
                                     resid_out);
}
