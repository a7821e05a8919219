// bw_patch_common.cuh — shared device pieces of the local-BIE collocation
// (K4 generic assembly in bw_patch.cu, the congruence-class DtN in
// bw_dtn_class.cu): vector helpers, the triangle rules, the sphere Green's
// function pair and the patch mesh (patch_solver.cpp:26-52, 62-121).
#pragma once

#include <cmath>

#include "bw_internal.h"

namespace bw {
namespace {

constexpr double kInv4Pi = 0.079577471545947667884441881686257181;
constexpr double kPi = 3.14159265358979323846;

__constant__ double kTriW[7] = {0.225, 0.132394152788506, 0.132394152788506, 0.132394152788506,
                                0.125939180544827, 0.125939180544827, 0.125939180544827};
__constant__ double kTriB[7][3] = {{1.0 / 3, 1.0 / 3, 1.0 / 3},
                                   {0.059715871789770, 0.470142064105115, 0.470142064105115},
                                   {0.470142064105115, 0.059715871789770, 0.470142064105115},
                                   {0.470142064105115, 0.470142064105115, 0.059715871789770},
                                   {0.797426985353087, 0.101286507323456, 0.101286507323456},
                                   {0.101286507323456, 0.797426985353087, 0.101286507323456},
                                   {0.101286507323456, 0.101286507323456, 0.797426985353087}};

struct V3 {
    double x, y, z;
};
__device__ __forceinline__ V3 v3(double x, double y, double z) { return V3{x, y, z}; }
__device__ __forceinline__ V3 operator+(V3 a, V3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ V3 operator-(V3 a, V3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ V3 operator*(double s, V3 a) { return v3(s * a.x, s * a.y, s * a.z); }
__device__ __forceinline__ double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ double len(V3 a) { return sqrt(dot(a, a)); }
__device__ __forceinline__ V3 cross(V3 a, V3 b) {
    return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ V3 ldv(const double* p) { return v3(p[0], p[1], p[2]); }
__device__ __forceinline__ void stv(double* p, V3 v) {
    p[0] = v.x;
    p[1] = v.y;
    p[2] = v.z;
}

// sphere Green's function of B(o, a) (greens.cpp:21-39,79-89,51-65), both
// derivatives the collocation needs at one quadrature point y, sharing the
// image construction: source term (c = 1, p = y, grad c = 0, J = I) and Kelvin
// image (c = -a/rho, p = k y, grad c = (a/rho^2) yh, J = k (I - 2 yh yh^T),
// k = a^2/rho^2). Reciprocal square roots replace the reference's divisions
// (same algebra; differences are rounding, checked at 1e-10).
struct Kernels {
    double dgdnx; // dG/dn_x (x, y)             (greens.cpp:79-89)
    double d2g;   // d2G/dn_x dn_y (x, y; n_y)  (greens.cpp:51-65)
};

__device__ __forceinline__ Kernels green_pair(double a, V3 xl, V3 nx, V3 yl, V3 ny) {
    const double ri = rsqrt(dot(yl, yl));
    const V3 yh = ri * yl;
    const double k = a * a * (ri * ri);
    const double c = -a * ri;
    const V3 p = k * yl;
    const double yn = dot(yh, ny);
    const double gny = a * (ri * ri) * yn; // grad c . n_y
    const V3 dp = k * (ny - (2.0 * yn) * yh);
    const V3 r0 = xl - yl;
    const double i0 = rsqrt(dot(r0, r0));
    const double i03 = i0 * i0 * i0;
    const V3 r1 = xl - p;
    const double i1 = rsqrt(dot(r1, r1));
    const double i13 = i1 * i1 * i1;
    const double rnx0 = dot(r0, nx), rnx1 = dot(r1, nx);
    Kernels K;
    K.dgdnx = kInv4Pi * (-rnx0 * i03 - c * rnx1 * i13);
    K.d2g = kInv4Pi * (dot(ny, nx) * i03 - 3.0 * rnx0 * dot(r0, ny) * (i03 * i0 * i0) -
                       gny * rnx1 * i13 + c * dot(dp, nx) * i13 -
                       3.0 * c * rnx1 * dot(r1, dp) * (i13 * i1 * i1));
    return K;
}

__device__ __forceinline__ double d2g(double a, V3 xl, V3 nx, V3 yl, V3 ny) {
    return green_pair(a, xl, nx, yl, ny).d2g;
}

// The first-kind pair (greens.cpp:41-49 eval_g, :67-77 eval_dg_dny) on the same
// image construction: G(x, y) and dG/dn_y(x, y; n_y).
struct KernelsFirst {
    double g;
    double dgdny;
};

__device__ __forceinline__ KernelsFirst green_first(double a, V3 xl, V3 yl, V3 ny) {
    const double ri = rsqrt(dot(yl, yl));
    const V3 yh = ri * yl;
    const double k = a * a * (ri * ri);
    const double c = -a * ri;
    const V3 p = k * yl;
    const double yn = dot(yh, ny);
    const double gny = a * (ri * ri) * yn; // grad c . n_y
    const V3 dp = k * (ny - (2.0 * yn) * yh);
    const V3 r0 = xl - yl;
    const double i0 = rsqrt(dot(r0, r0));
    const V3 r1 = xl - p;
    const double i1 = rsqrt(dot(r1, r1));
    KernelsFirst K;
    K.g = kInv4Pi * (i0 + c * i1);
    K.dgdny = kInv4Pi * (dot(r0, ny) * (i0 * i0 * i0) + gny * i1 + c * dot(r1, dp) * (i1 * i1 * i1));
    return K;
}

// The collocation kernels of one BIE kind (patch_solver.cpp:264-306): the
// A-kernel (second: dG/dn_x, first: G) and the b-kernel multiplying
// (phi(y) - u_i) and the Gamma data (second: d2G/dn_x dn_y, first: dG/dn_y).
__device__ __forceinline__ void bie_kernels(int kind, double a, V3 xl, V3 nx, V3 yl, V3 ny,
                                            double& ka, double& kb) {
    if (kind == BW_BIE_FIRST) {
        const KernelsFirst K = green_first(a, xl, yl, ny);
        ka = K.g;
        kb = K.dgdny;
    } else {
        const Kernels K = green_pair(a, xl, nx, yl, ny);
        ka = K.dgdnx;
        kb = K.d2g;
    }
}

struct PatchGeo {
    int surf;  // 0 sphere (centre sc, radius R), 1 plane (through o, normal axis)
    V3 sc, o, axis;
    double R, a;
};

// eval_dirichlet on the patch surface (geometry.cpp:198-220): projection
// onto the patch's own sphere / plane, then the closed-form data.
template <int PHI>
__device__ __forceinline__ double phi_on_patch(const DevScene& S, const PatchGeo& g, V3 y) {
    V3 p;
    if (g.surf == 0) {
        const V3 q = y - g.sc;
        p = g.sc + (g.R * rsqrt(dot(q, q))) * q;
    } else {
        p = y - dot(y - g.o, g.axis) * g.axis;
    }
    return eval_phi<PHI>(S, p.x, p.y, p.z, 0);
}

// Patch mesh (fan + bands, patch_solver.cpp:26-52, 62-121) in shared memory:
// vertices, triangles, centroids, normals (into the solution domain), areas
// and diameters. Called by all threads of the block; ends with a barrier.
struct Mesh {
    double verts[65][3];
    int tris[64][3];
    double cen[64][3], nrm[64][3], area[64], diam[64];
};

// The same arrays for any panel count (the large-patch path keeps them in
// dynamic shared memory).
struct MeshView {
    double (*verts)[3];
    int (*tris)[3];
    double (*cen)[3];
    double (*nrm)[3];
    double* area;
    double* diam;
};

__device__ __forceinline__ MeshView view(Mesh& M) {
    return MeshView{M.verts, M.tris, M.cen, M.nrm, M.area, M.diam};
}

__device__ __forceinline__ void mesh_frame(const PatchGeo& g, V3& rad, V3& e1, V3& e2) {
    rad = g.axis;
    if (g.surf == 0) {
        const V3 q = g.o - g.sc;
        rad = (1.0 / len(q)) * q;
    }
    const V3 ref = fabs(rad.x) < 0.9 ? v3(1, 0, 0) : v3(0, 1, 0);
    e1 = cross(rad, ref);
    e1 = (1.0 / len(e1)) * e1;
    e2 = cross(rad, e1);
}

__device__ void build_mesh(const PatchGeo& g, int bands, int az, MeshView M, int tid, int nthr) {
    const int m = az * (2 * bands - 1);
    const int nv = 1 + bands * az;
    V3 rad, e1, e2;
    mesh_frame(g, rad, e1, e2);
    const double alpha_max = g.surf == 0 ? acos(1.0 - g.a * g.a / (2.0 * g.R * g.R)) : 0.0;
    for (int v = tid; v < nv; v += nthr) {
        V3 p = g.o;
        if (v > 0) {
            const int k = (v - 1) / az + 1, j = (v - 1) % az;
            const double beta = 2.0 * kPi * j / az;
            double sb, cb;
            sincos(beta, &sb, &cb);
            if (g.surf == 0) {
                double sa, ca;
                sincos(alpha_max * k / bands, &sa, &ca);
                p = g.sc + g.R * ((sa * cb) * e1 + (sa * sb) * e2 + ca * rad);
            } else {
                const double r = g.a * k / bands;
                p = g.o + (r * cb) * e1 + (r * sb) * e2;
            }
        }
        stv(M.verts[v], p);
    }
    for (int t = tid; t < m; t += nthr) {
        int a0, a1, a2;
        if (t < az) {
            a0 = 0;
            a1 = 1 + t;
            a2 = 1 + (t + 1) % az;
        } else {
            const int u = t - az, kk = u / (2 * az), rem = u % (2 * az), j = rem >> 1;
            const int va = 1 + kk * az + j, vb = 1 + (kk + 1) * az + j;
            const int vb1 = 1 + (kk + 1) * az + (j + 1) % az, va1 = 1 + kk * az + (j + 1) % az;
            if ((rem & 1) == 0) {
                a0 = va; a1 = vb; a2 = vb1;
            } else {
                a0 = va; a1 = vb1; a2 = va1;
            }
        }
        M.tris[t][0] = a0;
        M.tris[t][1] = a1;
        M.tris[t][2] = a2;
    }
    __syncthreads();
    const double side = dot(g.axis, rad) >= 0 ? 1.0 : -1.0;
    for (int t = tid; t < m; t += nthr) {
        const V3 v0 = ldv(M.verts[M.tris[t][0]]), v1 = ldv(M.verts[M.tris[t][1]]),
                 v2 = ldv(M.verts[M.tris[t][2]]);
        const V3 c = (1.0 / 3.0) * (v0 + v1 + v2);
        V3 n = cross(v1 - v0, v2 - v0);
        const double a2 = len(n);
        n = (1.0 / a2) * n;
        V3 out = g.axis;
        if (g.surf == 0) {
            const V3 q = c - g.sc;
            out = (1.0 / len(q)) * q;
        }
        if (dot(n, out) < 0) n = -1.0 * n;
        n = side * n;
        stv(M.cen[t], c);
        stv(M.nrm[t], n);
        M.area[t] = 0.5 * a2;
        M.diam[t] = fmax(fmax(len(v1 - v0), len(v2 - v1)), len(v0 - v2));
    }
    __syncthreads();
}

// Leaf `leaf` of the depth-`depth` midpoint subdivision of (v0, v1, v2)
// (integrate_triangle_refined, quadrature.hpp:80-98), child order 0..3.
__device__ __forceinline__ void refine_leaf(V3& a0, V3& a1, V3& a2, int leaf, int depth) {
    for (int lv = depth - 1; lv >= 0; --lv) {
        const int ch = (leaf >> (2 * lv)) & 3;
        const V3 m01 = 0.5 * (a0 + a1), m12 = 0.5 * (a1 + a2), m20 = 0.5 * (a2 + a0);
        if (ch == 0) { a1 = m01; a2 = m20; }
        else if (ch == 1) { a0 = m01; a2 = m12; }
        else if (ch == 2) { a0 = m20; a1 = m12; }
        else { a0 = m01; a1 = m12; a2 = m20; }
    }
}

__device__ __forceinline__ PatchGeo patch_geo(const bw_patch& P) {
    PatchGeo g;
    g.surf = P.surf;
    g.sc = ldv(P.sc);
    g.o = ldv(P.o);
    g.axis = ldv(P.axis);
    g.R = P.R;
    g.a = P.a;
    return g;
}

} // namespace
} // namespace bw
