// bw_dtn_class.cu — K7: the local DtN through congruence-class tables.
//
// The second-kind patch system of a boundary point (patch_solver.cpp:197-309)
// depends on the point only through (i) a rigid motion of its patch and (ii)
// the data: the sphere Green's function of the hemisphere ball is invariant
// under rigid motions, so A, the quadrature weights and every kernel value
// are the same for all patches with equal (surface, R, a, side, Gamma class).
// Linear algebra then collapses the per-point work:
//
//   b_i   = -sum_k Kg_ik (u_k - u_i) + sum_q D_iq (phi(y_q) - u_i)
//   dudn  = f^T A^-1 b = g . b,          g = A^-T f,  f_j = -area_j / area_fan
//         = sum_k hK_k u_k + sum_i hU_i u_i + sum_q hQ_q phi(y_q)
//   hK_k  = -sum_i g_i Kg_ik,  hU_i = g_i (sum_k Kg_ik - sum_q D_iq),
//   hQ_q  = sum_i g_i D_iq
//   err   = sum_fan (area_j / area_fan) |(A^-1 b_se)_j|,
//   b_se_i = sqrt(sum_k Kg_ik^2 var_k)
//
// with Kg_ik = w_k d2G(x_i, y_k) on the Gamma nodes and D_iq = W_q d2G(x_i, y_q)
// (first kind, BW_BIE_FIRST: A from G, Kg and D from dG/dn_y, no 1/2 on the diagonal)
// over the panel quadrature points q of row i (self: polar split; near:
// refined; far: degree-5 rule — exactly the point sets of K4, bw_patch.cu).
// A constant shift phi0 of all data leaves b unchanged (hK + hU + hQ sum to 0)
// and is applied to keep the long sums well-conditioned; the self points of
// row i (the singular, polar-split part) keep K4's own form phi(y_q) - u_i, so
// hU_i carries only the near/far row sum of D.
//
// Per class (one canonical patch per key, built from the key alone, so the
// tables — and therefore every point's result — do not depend on how points
// are sharded or batched):
//   class_geom_kernel  mesh, A (transposed for K2), Kg, row sums of Kg and D,
//                      local coordinates of every data point (projected onto
//                      the patch surface as phi_on_patch does), fan weights
//   K2 (bw_lu.cu)      A^T [g | F^T] = [f | e_0 .. e_az-1], residual gate on g
//   class_h_kernel     hQ (thread per point, rows in order), hU, hK
// Per boundary point:
//   class_apply_kernel phi at the class's points mapped by the point's frame,
//                      dot products with hQ/hU/hK, b_se, err, status.
// Gamma nodes outside the domain (est.n == 0) drop out of b exactly as in K4
// (their Kg column is removed from hK and from the u_i coefficients).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "bw_patch_common.cuh"

namespace bw {

namespace {

constexpr int kGeomThreads = 128;
constexpr int kGeomWarps = kGeomThreads / 32;
constexpr int kHThreads = 256;
constexpr int kApplyThreads = 256;
constexpr int kApplyWarps = kApplyThreads / 32;
constexpr int kGroup = kApplyWarps; // patches per apply CTA (one warp each in the epilogue)

// Sizes of one class's tables (all classes of a call share them).
struct ClassDims {
    int m, az, nv, n_nodes, np, depth;
    int kind;    // BW_BIE_SECOND / BW_BIE_FIRST
    int L7;      // refined points per panel: 4^depth x 7
    int P3;      // self points per row: 3 np^2
    int Q;       // panel data points: m (L7 + 7) + m P3
    int Qt;      // + m centroids
    // per-class strides (doubles)
    size_t sA, sKg, sLq, sH;
};

ClassDims class_dims(int bands, int az, int n_nodes, int np, int depth, int kind) {
    ClassDims d;
    d.kind = kind;
    d.m = az * (2 * bands - 1);
    d.az = az;
    d.nv = 1 + bands * az;
    d.n_nodes = n_nodes;
    d.np = np;
    d.depth = depth;
    d.L7 = (1 << (2 * depth)) * 7;
    d.P3 = 3 * np * np;
    d.Q = d.m * (d.L7 + 7) + d.m * d.P3;
    d.Qt = d.Q + d.m;
    d.sA = (size_t)d.m * d.m;
    d.sKg = (size_t)d.m * n_nodes;
    d.sLq = 3 * (size_t)d.Qt;
    d.sH = (size_t)d.Qt;
    return d;
}

// Device views of one chunk of classes.
struct ClassTables {
    const bw_patch* canon; // nc canonical patches
    Mesh* mesh;            // nc
    double* At;            // nc x m x m  (A transposed: K2 solves A^T z = r)
    double* R;             // nc x (az+1) x m right-hand sides
    double* Z;             // nc x (az+1) x m solutions: g, then rows of A^-1 at the fan
    double* Kg;            // nc x m x n_nodes
    double* rowKg;         // nc x m
    double* rowD;          // nc x m
    double* wfan;          // nc x az  (area_j / area_fan)
    double* lq;            // nc x 3 x Qt local coordinates (SoA)
    double* H;             // nc x Qt   (hQ, then hU at the centroid entries)
    double* hK;            // nc x n_nodes
    int32_t* info;         // nc
    double* resid;         // nc
};

// One data point of a class, in the canonical patch's coordinates.
// kind 0: refined point of panel j (rows i != j near j); 1: far point of
// panel j (rows i != j not near j); 2: self point of row j; 3: centroid j.
struct QPoint {
    V3 y;
    double W;
    int j, kind;
};

__device__ __forceinline__ QPoint decode_point(int q, const Mesh& M, const ClassDims& d,
                                               const double* ps, const double* pt,
                                               const double* pw) {
    QPoint r;
    const int nref = d.m * d.L7, nfar = 7 * d.m, nself = d.m * d.P3;
    if (q < nref) {
        const int j = q / d.L7, rem = q % d.L7, leaf = rem / 7, p = rem % 7;
        V3 a0 = ldv(M.verts[M.tris[j][0]]), a1 = ldv(M.verts[M.tris[j][1]]),
           a2 = ldv(M.verts[M.tris[j][2]]);
        refine_leaf(a0, a1, a2, leaf, d.depth);
        const double area = 0.5 * len(cross(a1 - a0, a2 - a0));
        r.y = kTriB[p][0] * a0 + kTriB[p][1] * a1 + kTriB[p][2] * a2;
        r.W = area * kTriW[p];
        r.j = j;
        r.kind = 0;
        return r;
    }
    q -= nref;
    if (q < nfar) {
        const int j = q / 7, p = q % 7;
        const V3 v0 = ldv(M.verts[M.tris[j][0]]), v1 = ldv(M.verts[M.tris[j][1]]),
                 v2 = ldv(M.verts[M.tris[j][2]]);
        const double area = 0.5 * len(cross(v1 - v0, v2 - v0));
        r.y = kTriB[p][0] * v0 + kTriB[p][1] * v1 + kTriB[p][2] * v2;
        r.W = area * kTriW[p];
        r.j = j;
        r.kind = 1;
        return r;
    }
    q -= nfar;
    if (q < nself) {
        const int per = d.np * d.np;
        const int i = q / d.P3, rem = q % d.P3, sub = rem / per, qq = rem % per;
        const V3 v0 = ldv(M.verts[M.tris[i][0]]), v1 = ldv(M.verts[M.tris[i][1]]),
                 v2 = ldv(M.verts[M.tris[i][2]]);
        const V3 xi = ldv(M.cen[i]);
        const V3 a0 = sub == 0 ? v0 : (sub == 1 ? v1 : v2);
        const V3 a1 = sub == 0 ? v1 : (sub == 1 ? v2 : v0);
        const double area2 = len(cross(a0 - xi, a1 - xi));
        const V3 w = a0 + ps[qq] * (a1 - a0);
        r.y = xi + pt[qq] * (w - xi);
        r.W = area2 * pw[qq];
        r.j = i;
        r.kind = 2;
        return r;
    }
    q -= nself;
    r.y = ldv(M.cen[q]);
    r.W = 0.0;
    r.j = q;
    r.kind = 3;
    return r;
}

// point projected onto the patch surface (phi_on_patch, bw_patch_common.cuh)
__device__ __forceinline__ V3 project_patch(const PatchGeo& g, V3 y) {
    if (g.surf == 0) {
        const V3 q = y - g.sc;
        return g.sc + (g.R * rsqrt(dot(q, q))) * q;
    }
    return y - dot(y - g.o, g.axis) * g.axis;
}

// polar rule table (integrate_triangle_polar, quadrature.hpp:60-78)
__device__ __forceinline__ void polar_table(const double* gl, int np, double* ps, double* pt,
                                            double* pw, int tid, int nthr) {
    for (int q = tid; q < np * np; q += nthr) {
        const int i = q / np, j = q % np;
        const double t = 0.5 * (gl[j] + 1.0);
        ps[q] = 0.5 * (gl[i] + 1.0);
        pt[q] = t;
        pw[q] = gl[32 + i] * (0.25 * gl[32 + j] * t);
    }
}

struct GeomSmem {
    Mesh mesh;
    double B[64][65];
};

// ---- pass 1: per class geometry, A, Kg, row sums, point coordinates ----
__global__ void __launch_bounds__(kGeomThreads)
    class_geom_kernel(ClassTables T, ClassDims d, int bands, const double* __restrict__ dirs,
                      const double* __restrict__ wts, const double* __restrict__ gl) {
    __shared__ GeomSmem sm;
    extern __shared__ __align__(16) double dyn[];
    double* gy = dyn;                 // 3 n_nodes
    double* gw = gy + 3 * d.n_nodes;  // n_nodes
    double* ps = gw + d.n_nodes;      // np^2
    double* pt_ = ps + d.np * d.np;
    double* pw = pt_ + d.np * d.np;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int m = d.m, c = blockIdx.x;
    const bw_patch P = T.canon[c];
    const PatchGeo g = patch_geo(P);
    polar_table(gl, d.np, ps, pt_, pw, tid, kGeomThreads);
    build_mesh(g, bands, d.az, view(sm.mesh), tid, kGeomThreads);
    const Mesh& M = sm.mesh;
    for (int j = tid; j < d.n_nodes; j += kGeomThreads) {
        double x, y, z;
        patch_node_local(P.o, P.axis, P.a, dirs + ((int64_t)P.cls * d.n_nodes + j) * 3, x, y, z);
        gy[3 * j] = x;
        gy[3 * j + 1] = y;
        gy[3 * j + 2] = z;
        gw[j] = wts[(int64_t)P.cls * d.n_nodes + j] * (P.a * P.a);
    }
    __syncthreads();
    // Kg and its row sums: warp per row
    double* Kg = T.Kg + c * d.sKg;
    for (int i = warp; i < m; i += kGeomWarps) {
        const V3 xl = ldv(M.cen[i]) - g.o, ni = ldv(M.nrm[i]);
        double s = 0.0;
        for (int k = lane; k < d.n_nodes; k += 32) {
            const V3 yl = ldv(gy + 3 * k) - g.o;
            const V3 ny = (1.0 / g.a) * yl;
            double ka, kb;
            bie_kernels(d.kind, g.a, xl, ni, yl, ny, ka, kb);
            const double v = gw[k] * kb;
            Kg[(size_t)i * d.n_nodes + k] = v;
            s += v;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
        if (lane == 0) T.rowKg[c * m + i] = s;
    }
    // A and D row sums: self + near panels, warp-cooperative (as K4)
    double* At = T.At + c * d.sA;
    const int np = d.np;
    for (int i = warp; i < m; i += kGeomWarps) {
        const V3 xi = ldv(M.cen[i]);
        const V3 xl = xi - g.o, nx = ldv(M.nrm[i]);
        for (int j = 0; j < m; ++j) {
            const double dist = len(xi - ldv(M.cen[j]));
            const bool self = j == i;
            if (!self && !(dist < 2.0 * M.diam[j])) continue;
            const V3 ny = ldv(M.nrm[j]);
            const V3 v0 = ldv(M.verts[M.tris[j][0]]), v1 = ldv(M.verts[M.tris[j][1]]),
                     v2 = ldv(M.verts[M.tris[j][2]]);
            double sa = 0.0, sb = 0.0;
            if (self) {
                const int per = np * np;
#pragma unroll 1
                for (int sub = 0; sub < 3; ++sub) {
                    const V3 a0 = sub == 0 ? v0 : (sub == 1 ? v1 : v2);
                    const V3 a1 = sub == 0 ? v1 : (sub == 1 ? v2 : v0);
                    const double area2 = len(cross(a0 - xi, a1 - xi));
                    for (int q = lane; q < per; q += 32) {
                        const V3 w = a0 + ps[q] * (a1 - a0);
                        const double wq = area2 * pw[q];
                        double ka, kb;
                        bie_kernels(d.kind, g.a, xl, nx, (xi + pt_[q] * (w - xi)) - g.o, ny, ka, kb);
                        sa = fma(wq, ka, sa);
                        sb = fma(wq, kb, sb);
                    }
                }
            } else {
                const int leaves = 1 << (2 * d.depth);
                for (int q = lane; q < leaves * 7; q += 32) {
                    const int leaf = q / 7, p = q % 7;
                    V3 a0 = v0, a1 = v1, a2 = v2;
                    refine_leaf(a0, a1, a2, leaf, d.depth);
                    const double area = 0.5 * len(cross(a1 - a0, a2 - a0));
                    const V3 y = kTriB[p][0] * a0 + kTriB[p][1] * a1 + kTriB[p][2] * a2;
                    double ka, kb;
                    bie_kernels(d.kind, g.a, xl, nx, y - g.o, ny, ka, kb);
                    sa = fma(area * kTriW[p], ka, sa);
                    sb = fma(area * kTriW[p], kb, sb);
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                sa += __shfl_down_sync(0xffffffffu, sa, off);
                sb += __shfl_down_sync(0xffffffffu, sb, off);
            }
            if (lane == 0) {
                At[(size_t)j * m + i] = self && d.kind == BW_BIE_SECOND ? 0.5 + sa : sa;
                sm.B[i][j] = sb;
            }
        }
    }
    // far panels: thread per pair, degree-5 rule
    for (int pq = tid; pq < m * m; pq += kGeomThreads) {
        const int i = pq / m, j = pq % m;
        const V3 xi = ldv(M.cen[i]);
        const double dist = len(xi - ldv(M.cen[j]));
        if (i == j || dist < 2.0 * M.diam[j]) continue;
        const V3 xl = xi - g.o, nx = ldv(M.nrm[i]), ny = ldv(M.nrm[j]);
        const V3 v0 = ldv(M.verts[M.tris[j][0]]), v1 = ldv(M.verts[M.tris[j][1]]),
                 v2 = ldv(M.verts[M.tris[j][2]]);
        const double area = 0.5 * len(cross(v1 - v0, v2 - v0));
        double sa = 0.0, sb = 0.0;
#pragma unroll
        for (int p = 0; p < 7; ++p) {
            const V3 y = kTriB[p][0] * v0 + kTriB[p][1] * v1 + kTriB[p][2] * v2;
            double ka, kb;
            bie_kernels(d.kind, g.a, xl, nx, y - g.o, ny, ka, kb);
            sa = fma(kTriW[p], ka, sa);
            sb = fma(area * kTriW[p], kb, sb);
        }
        At[(size_t)j * m + i] = area * sa;
        sm.B[i][j] = sb;
    }
    // point coordinates (projected, in the canonical mesh frame)
    V3 rad, e1, e2;
    mesh_frame(g, rad, e1, e2);
    double* lq = T.lq + c * d.sLq;
    for (int q = tid; q < d.Qt; q += kGeomThreads) {
        const QPoint p = decode_point(q, M, d, ps, pt_, pw);
        const V3 u = project_patch(g, p.y) - g.o;
        lq[q] = dot(u, e1);
        lq[d.Qt + q] = dot(u, e2);
        lq[2 * (size_t)d.Qt + q] = dot(u, rad);
    }
    if (tid == 0) T.mesh[c] = sm.mesh;
    __syncthreads();
    for (int i = tid; i < m; i += kGeomThreads) {
        double s = 0.0;
        for (int j = 0; j < m; ++j)
            if (j != i) s += sm.B[i][j]; // self points carry their own shift (apply)
        T.rowD[c * m + i] = s;
    }
    // right-hand sides: f (fan-weighted point value) and unit vectors e_j, j < az
    double at = 0.0;
    for (int j = 0; j < d.az; ++j) at += M.area[j];
    const int nr = d.az + 1;
    double* R = T.R + (size_t)c * nr * m;
    for (int e = tid; e < nr * m; e += kGeomThreads) {
        const int r = e / m, j = e % m;
        double v = 0.0;
        if (r == 0) v = j < d.az ? -M.area[j] / at : 0.0;
        else v = (j == r - 1) ? 1.0 : 0.0;
        R[e] = v;
    }
    for (int j = tid; j < d.az; j += kGeomThreads) T.wfan[c * d.az + j] = M.area[j] / at;
}

// ---- pass 2: hQ (thread per point), hU, hK ----
__global__ void __launch_bounds__(kHThreads)
    class_h_kernel(ClassTables T, ClassDims d, const double* __restrict__ gl) {
    __shared__ Mesh M;
    __shared__ double gv[64];
    extern __shared__ __align__(16) double dyn[];
    double* ps = dyn;
    double* pt_ = ps + d.np * d.np;
    double* pw = pt_ + d.np * d.np;
    const int tid = threadIdx.x, c = blockIdx.y, m = d.m;
    {
        const double* src = reinterpret_cast<const double*>(T.mesh + c);
        double* dst = reinterpret_cast<double*>(&M);
        for (int e = tid; e < (int)(sizeof(Mesh) / sizeof(double)); e += kHThreads) dst[e] = src[e];
    }
    const double* Zc = T.Z + (size_t)c * (d.az + 1) * m;
    for (int i = tid; i < m; i += kHThreads) gv[i] = Zc[i];
    polar_table(gl, d.np, ps, pt_, pw, tid, kHThreads);
    __syncthreads();
    const PatchGeo g = patch_geo(T.canon[c]);
    const int q = blockIdx.x * kHThreads + tid;
    double* H = T.H + c * d.sH;
    if (q < d.Q) {
        const QPoint p = decode_point(q, M, d, ps, pt_, pw);
        const V3 yl = p.y - g.o, ny = ldv(M.nrm[p.j]);
        const V3 cj = ldv(M.cen[p.j]);
        const double dj = 2.0 * M.diam[p.j];
        double h = 0.0;
        double ka, kb;
        if (p.kind == 2) {
            bie_kernels(d.kind, g.a, cj - g.o, ny, yl, ny, ka, kb);
            h = gv[p.j] * (p.W * kb);
        } else {
            for (int i = 0; i < m; ++i) {
                if (i == p.j) continue;
                const V3 xi = ldv(M.cen[i]);
                const bool near = len(xi - cj) < dj;
                if (near != (p.kind == 0)) continue;
                bie_kernels(d.kind, g.a, xi - g.o, ldv(M.nrm[i]), yl, ny, ka, kb);
                h = fma(gv[i], p.W * kb, h);
            }
        }
        H[q] = h;
    } else if (q < d.Qt) {
        const int i = q - d.Q;
        H[q] = gv[i] * (T.rowKg[c * m + i] - T.rowD[c * m + i]);
    }
    if (blockIdx.x == 0) {
        const double* Kg = T.Kg + c * d.sKg;
        for (int k = tid; k < d.n_nodes; k += kHThreads) {
            double s = 0.0;
            for (int i = 0; i < m; ++i) s = fma(gv[i], Kg[(size_t)i * d.n_nodes + k], s);
            T.hK[c * d.n_nodes + k] = -s;
        }
    }
}

// ---- per boundary point: apply the class tables ----
// Compensated accumulation (TwoSum + the FMA product error): the point value
// is a sum of ~7e4 terms that cancel to a few digits, so the running error is
// carried alongside the sum (s, c) and folded in once at the end.
__device__ __forceinline__ void acc2(double& s, double& c, double h, double v) {
    const double p = __dmul_rn(h, v); // _rn: no contraction into the TwoSum
    const double pe = fma(h, v, -p);
    const double t = __dadd_rn(s, p);
    const double z = __dsub_rn(t, s);
    c += __dadd_rn(__dsub_rn(s, __dsub_rn(t, z)), __dsub_rn(p, z)) + pe;
    s = t;
}

__device__ __forceinline__ void merge2(double& s, double& c, double s2, double c2) {
    const double t = __dadd_rn(s, s2);
    const double z = __dsub_rn(t, s);
    c += __dadd_rn(__dsub_rn(s, __dsub_rn(t, z)), __dsub_rn(s2, z)) + c2;
    s = t;
}

struct ApplySmem {
    double o[kGroup][3], E[kGroup][9], phi0[kGroup];
    double red[kApplyWarps][kGroup], redc[kApplyWarps][kGroup];
    double accT[kGroup][kApplyThreads];
    double accC[kGroup][kApplyThreads];
    double acc[kGroup];
    double bse[kGroup][64];
    double u[kGroup][64]; // phi at the centroids (u_i of K4)
    double gv[64], F[8][64];
    int bad[kGroup];
};

template <int PHI>
__global__ void __launch_bounds__(kApplyThreads)
    class_apply_kernel(const DevScene S, ClassTables T, ClassDims d, int cbase,
                       const bw_patch* __restrict__ patches, const int64_t* __restrict__ perm,
                       const int64_t* __restrict__ groups, const bw_estimate* __restrict__ est,
                       double* __restrict__ dudn, double* __restrict__ err,
                       int32_t* __restrict__ status) {
    __shared__ ApplySmem sm;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, m = d.m;
    // group = (class, first index into perm, count)
    const int64_t* G = groups + 3 * (int64_t)blockIdx.x;
    const int c = (int)G[0] - cbase;
    const int64_t first = G[1];
    const int np_ = (int)G[2];
    if (tid < np_) {
        BW_CHECK(perm[first + tid] >= 0 && c >= 0);
        const bw_patch P = patches[perm[first + tid]];
        const PatchGeo g = patch_geo(P);
        V3 rad, e1, e2;
        mesh_frame(g, rad, e1, e2);
        sm.o[tid][0] = g.o.x; sm.o[tid][1] = g.o.y; sm.o[tid][2] = g.o.z;
        sm.E[tid][0] = e1.x; sm.E[tid][1] = e1.y; sm.E[tid][2] = e1.z;
        sm.E[tid][3] = e2.x; sm.E[tid][4] = e2.y; sm.E[tid][5] = e2.z;
        sm.E[tid][6] = rad.x; sm.E[tid][7] = rad.y; sm.E[tid][8] = rad.z;
        sm.phi0[tid] = eval_phi<PHI>(S, g.o.x, g.o.y, g.o.z, 0);
        sm.bad[tid] = 0;
    }
    const int nr = d.az + 1;
    const double* Zc = T.Z + (size_t)c * nr * m;
    for (int e = tid; e < m; e += kApplyThreads) sm.gv[e] = Zc[e];
    for (int e = tid; e < d.az * m; e += kApplyThreads) sm.F[e / m][e % m] = Zc[m + e];
    __syncthreads();
    // per-thread partial sums live in shared memory (acc[p][tid]): the patch
    // loop stays rolled, so the frames are not hoisted into registers
    double* acc = sm.accT[0] + tid;
    double* cmp = sm.accC[0] + tid;
#pragma unroll
    for (int p = 0; p < kGroup; ++p) acc[p * kApplyThreads] = cmp[p * kApplyThreads] = 0.0;
#define BW_ACC(p, h, v) acc2(acc[(p) * kApplyThreads], cmp[(p) * kApplyThreads], (h), (v))
    const double* lx = T.lq + c * d.sLq;
    const double* ly = lx + d.Qt;
    const double* lz = ly + d.Qt;
    const double* H = T.H + c * d.sH;
    auto phi_at = [&](int p, double a, double b, double z) {
        const double* E = sm.E[p];
        const double x = sm.o[p][0] + (a * E[0] + b * E[3] + z * E[6]);
        const double y = sm.o[p][1] + (a * E[1] + b * E[4] + z * E[7]);
        const double w = sm.o[p][2] + (a * E[2] + b * E[5] + z * E[8]);
        return eval_phi<PHI>(S, x, y, w, 0);
    };
    // u_i (centroids) and their terms hU_i (u_i - phi0)
    // (thread i takes row i for every patch of the group: a patch's sums never
    // depend on which other patches share the block)
    for (int i = tid; i < m; i += kApplyThreads) {
        const int q = d.Q + i;
#pragma unroll 1
        for (int p = 0; p < np_; ++p) {
            const double u = phi_at(p, lx[q], ly[q], lz[q]);
            sm.u[p][i] = u;
            BW_ACC(p, H[q], u - sm.phi0[p]);
        }
    }
    __syncthreads();
    // refined + far points: phi - phi0
    const int q_self = d.m * (d.L7 + 7);
    for (int q = tid; q < q_self; q += kApplyThreads) {
        const double a = lx[q], b = ly[q], z = lz[q], h = H[q];
#pragma unroll 1
        for (int p = 0; p < np_; ++p)
            BW_ACC(p, h, phi_at(p, a, b, z) - sm.phi0[p]);
    }
    // self points of row i: phi - u_i, as K4 forms it (the singular part)
    for (int q = q_self + tid; q < d.Q; q += kApplyThreads) {
        const double a = lx[q], b = ly[q], z = lz[q], h = H[q];
        const int i = (q - q_self) / d.P3;
#pragma unroll 1
        for (int p = 0; p < np_; ++p)
            BW_ACC(p, h, phi_at(p, a, b, z) - sm.u[p][i]);
    }
    // Gamma nodes
    const double* hK = T.hK + c * d.n_nodes;
    for (int k = tid; k < d.n_nodes; k += kApplyThreads) {
        const double hk = hK[k];
#pragma unroll 1
        for (int p = 0; p < np_; ++p) {
            const bw_estimate e = est[perm[first + p] * d.n_nodes + k];
            if (e.n > 0) BW_ACC(p, hk, e.mean - sm.phi0[p]);
            else sm.bad[p] = 1;
        }
    }
#pragma unroll
    for (int p = 0; p < kGroup; ++p) {
        double v = acc[p * kApplyThreads], vc = cmp[p * kApplyThreads];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double o = __shfl_down_sync(0xffffffffu, v, off);
            const double oc = __shfl_down_sync(0xffffffffu, vc, off);
            merge2(v, vc, o, oc);
        }
        if (lane == 0) {
            sm.red[warp][p] = v;
            sm.redc[warp][p] = vc;
        }
    }
#undef BW_ACC
    __syncthreads();
    if (tid < kGroup) {
        double v = 0.0, vc = 0.0;
        for (int w = 0; w < kApplyWarps; ++w) merge2(v, vc, sm.red[w][tid], sm.redc[w][tid]);
        sm.acc[tid] = v + vc;
    }
    __syncthreads();
    // epilogue: warp p finishes patch p
    if (warp < np_) {
        const int p = warp;
        const int64_t bp = perm[first + p];
        const bw_estimate* E = est + bp * d.n_nodes;
        const double* Kg = T.Kg + c * d.sKg;
        for (int i = 0; i < m; ++i) {
            double s = 0.0;
            for (int k = lane; k < d.n_nodes; k += 32) {
                const bw_estimate e = E[k];
                const double var = e.n > 0 ? e.variance / (double)e.n : 0.0;
                const double kk = Kg[(size_t)i * d.n_nodes + k];
                s = fma(kk * kk, var, s);
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
            if (lane == 0) sm.bse[p][i] = sqrt(s);
        }
        double corr = 0.0;
        if (sm.bad[p]) {
            // remove the Kg columns of the invalid nodes from the u_i terms
            for (int k = lane; k < d.n_nodes; k += 32) {
                if (E[k].n > 0) continue;
                double s = 0.0;
                for (int i = 0; i < m; ++i)
                    s = fma(sm.gv[i] * (sm.u[p][i] - sm.phi0[p]), Kg[(size_t)i * d.n_nodes + k], s);
                corr -= s;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) corr += __shfl_down_sync(0xffffffffu, corr, off);
        }
        __syncwarp();
        double e_sum = 0.0;
        for (int j = lane; j < d.az; j += 32) {
            double x = 0.0;
            for (int i = 0; i < m; ++i) x = fma(sm.F[j][i], sm.bse[p][i], x);
            e_sum += T.wfan[c * d.az + j] * fabs(x);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) e_sum += __shfl_down_sync(0xffffffffu, e_sum, off);
        if (lane == 0) {
            dudn[bp] = sm.acc[p] + corr;
            err[bp] = e_sum;
            status[bp] = (T.info[c] ? 2 : 0) | (sm.bad[p] ? 1 : 0);
        }
    }
}

// ---- host: congruence classes ----

struct ClassKey {
    int32_t surf, cls, side;
    uint64_t a, R;
    int64_t self; // -1: canonical class; else the patch index (own exemplar)
    bool operator==(const ClassKey& o) const {
        return surf == o.surf && cls == o.cls && side == o.side && a == o.a && R == o.R &&
               self == o.self;
    }
};
struct ClassKeyHash {
    size_t operator()(const ClassKey& k) const {
        uint64_t h = 1469598103934665603ull;
        auto mix = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
        mix((uint64_t)k.surf);
        mix((uint64_t)k.cls);
        mix((uint64_t)k.side);
        mix(k.a);
        mix(k.R);
        mix((uint64_t)k.self);
        return (size_t)h;
    }
};

uint64_t bits(double v) {
    uint64_t u;
    std::memcpy(&u, &v, 8);
    return u;
}

// Class of one patch and, for a new class, its exemplar: canonical when the
// patch is a clean rigid image of the canonical one (unit axis, o on its
// sphere, axis = +-radial, frame completion unambiguous), else the patch itself.
ClassKey class_of(const bw_patch& p, int64_t idx, bw_patch& exemplar) {
    ClassKey k{p.surf, p.cls, 1, bits(p.a), 0, -1};
    const double an = std::sqrt(p.axis[0] * p.axis[0] + p.axis[1] * p.axis[1] + p.axis[2] * p.axis[2]);
    bool clean = std::fabs(an - 1.0) < 1e-12 && p.a > 0 && (p.surf == 0 || p.surf == 1);
    if (clean && p.surf == 0) {
        const double q[3] = {p.o[0] - p.sc[0], p.o[1] - p.sc[1], p.o[2] - p.sc[2]};
        const double r = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2]);
        const double rad[3] = {q[0] / r, q[1] / r, q[2] / r};
        const double s = rad[0] * p.axis[0] + rad[1] * p.axis[1] + rad[2] * p.axis[2] >= 0 ? 1.0 : -1.0;
        double dev = 0.0;
        for (int t = 0; t < 3; ++t) dev = std::max(dev, std::fabs(p.axis[t] - s * rad[t]));
        clean = std::fabs(r - p.R) < 1e-12 * p.R && dev < 1e-9 &&
                std::fabs(std::fabs(rad[0]) - 0.9) > 1e-9;
        k.side = (int)s;
        k.R = bits(p.R);
    } else if (clean) {
        clean = std::fabs(std::fabs(p.axis[0]) - 0.9) > 1e-9;
    }
    std::memset(&exemplar, 0, sizeof(exemplar));
    if (!clean) {
        k.self = idx;
        exemplar = p;
        return k;
    }
    exemplar.surf = p.surf;
    exemplar.cls = p.cls;
    exemplar.a = p.a;
    if (p.surf == 0) {
        exemplar.R = p.R;
        exemplar.o[2] = p.R;
        exemplar.axis[2] = (double)k.side;
    } else {
        exemplar.axis[2] = 1.0;
    }
    return k;
}

template <int PHI>
cudaError_t launch_apply_t(bw_ctx* ctx, const DevScene& S, const ClassTables& T, const ClassDims& d,
                           int cbase, const bw_patch* patches, const int64_t* perm,
                           const int64_t* groups, int64_t n_groups, const bw_estimate* est,
                           double* dudn, double* err, int32_t* status) {
    if (n_groups <= 0) return cudaSuccess;
    ++ctx->launches;
    class_apply_kernel<PHI><<<(unsigned)n_groups, kApplyThreads, 0, ctx->stream>>>(
        S, T, d, cbase, patches, perm, groups, est, dudn, err, status);
    return cudaGetLastError();
}

// Order-independent 2 x 64-bit checksum of a word array (position mixed into
// every word; two multiplier pairs), accumulated with atomics into out[0..1].
__global__ void hash_words_kernel(const uint64_t* __restrict__ w, int64_t n, uint64_t salt,
                                  unsigned long long* __restrict__ out) {
    uint64_t a = 0, b = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t v = w[i];
        uint64_t x = (v ^ ((uint64_t)i * 0x9E3779B97F4A7C15ull) ^ salt) * 0xD2E7470EE14C6C93ull;
        x ^= x >> 29;
        a += x * 0xCA5A826395121157ull;
        uint64_t y = (v + (uint64_t)i * 0xBB67AE8584CAA73Bull + salt) * 0x94D049BB133111EBull;
        y ^= y >> 31;
        b += y * 0xBF58476D1CE4E5B9ull;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, off);
        b += __shfl_down_sync(0xffffffffu, b, off);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&out[0], (unsigned long long)a);
        atomicAdd(&out[1], (unsigned long long)b);
    }
}

} // namespace

// The whole Neumann stage for n_bp patches whose Gamma node estimates are in
// `est`, through congruence-class tables. Returns BW_OK, BW_ERR_SOLVER (some
// class failed the residual gate) or an error; `applicable` = false when the
// configuration is outside what the class path covers (caller uses K4).
bw_status dtn_neumann_classes(bw_ctx* ctx, const DevScene& S, const bw_patch* d_patches,
                              int64_t n_bp, const double* d_dirs, const double* d_weights,
                              int32_t n_rule, int32_t n_nodes, const bw_estimate* d_est, int bands, int az,
                              int np, int depth, int kind, double tol, const double* d_gl,
                              double* d_dudn,
                              double* d_err, int32_t* d_status, bool* applicable) {
    *applicable = false;
    const ClassDims d = class_dims(bands, az, n_nodes, np, depth, kind);
    if (az + 1 > 8 || d.m > 64 || n_bp <= 0) return BW_OK;
    *applicable = true;
    bw_status st = BW_OK;
    cudaError_t ce;
    // 0. the cache key: checksums of the patches and of the Gamma rule (device),
    // read back with one 64-byte copy
    static_assert(sizeof(bw_patch) % 8 == 0, "patches hash as 64-bit words");
    unsigned long long* d_hash =
        (unsigned long long*)scratch(ctx, kSlotClsHash, sizeof(unsigned long long) * 8, &st);
    if (st) return st;
    ce = cudaMemsetAsync(d_hash, 0, sizeof(unsigned long long) * 8, ctx->stream);
    if ((st = cuda_check(ctx, ce, "class hash memset"))) return st;
    {
        const int hb = (int)std::min<int64_t>((n_bp * (int64_t)(sizeof(bw_patch) / 8) + 255) / 256,
                                              (int64_t)ctx->sm_count * 8);
        ctx->launches += 4;
        hash_words_kernel<<<hb, 256, 0, ctx->stream>>>((const uint64_t*)d_patches,
                                                       n_bp * (int64_t)(sizeof(bw_patch) / 8), 1, d_hash);
        hash_words_kernel<<<8, 256, 0, ctx->stream>>>((const uint64_t*)d_dirs,
                                                      (int64_t)n_rule * n_nodes * 3, 2, d_hash + 2);
        hash_words_kernel<<<8, 256, 0, ctx->stream>>>((const uint64_t*)d_weights,
                                                      (int64_t)n_rule * n_nodes, 3, d_hash + 4);
        hash_words_kernel<<<1, 64, 0, ctx->stream>>>((const uint64_t*)d_gl, 64, 4, d_hash + 6);
    }
    uint64_t hkey[8];
    ce = cudaMemcpyAsync(hkey, d_hash, sizeof hkey, cudaMemcpyDeviceToHost, ctx->stream);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(ctx->stream);
    if ((st = cuda_check(ctx, ce, "class hash d2h"))) return st;
    bw_ctx::ClassCache& C = ctx->cls;
    const bool hit = C.valid && C.n_bp == n_bp && C.bands == bands && C.az == az && C.np == np &&
                     C.depth == depth && C.kind == kind && C.n_nodes == n_nodes &&
                     C.n_rule == n_rule && C.tol == tol &&
                     std::memcmp(C.hash, hkey, sizeof hkey) == 0 &&
                     ctx->scratch[kSlotClsPerm] && ctx->scratch[kSlotClsGroups];
    int64_t* d_perm = nullptr;
    int64_t* d_groups = nullptr;
    if (hit) {
        ++C.hits;
        d_perm = (int64_t*)ctx->scratch[kSlotClsPerm];
        d_groups = (int64_t*)ctx->scratch[kSlotClsGroups];
    } else {
    C.valid = false;
    C.tables_valid = false;
    // 1. classes (host): patches -> keys, canonical exemplars, points sorted by class
    std::vector<bw_patch> hp((size_t)n_bp);
    ce = cudaMemcpyAsync(hp.data(), d_patches, sizeof(bw_patch) * n_bp, cudaMemcpyDeviceToHost,
                         ctx->stream);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(ctx->stream);
    if ((st = cuda_check(ctx, ce, "class patches d2h"))) return st;
    std::unordered_map<ClassKey, int, ClassKeyHash> index;
    std::vector<bw_patch> canon;
    std::vector<int> cls_of((size_t)n_bp);
    for (int64_t i = 0; i < n_bp; ++i) {
        bw_patch ex;
        const ClassKey k = class_of(hp[i], i, ex);
        auto it = index.find(k);
        if (it == index.end()) {
            it = index.emplace(k, (int)canon.size()).first;
            canon.push_back(ex);
        }
        cls_of[i] = it->second;
    }
    const int n_cls = (int)canon.size();
    std::vector<int64_t> count(n_cls + 1, 0);
    for (int64_t i = 0; i < n_bp; ++i) ++count[cls_of[i] + 1];
    for (int c = 0; c < n_cls; ++c) count[c + 1] += count[c];
    std::vector<int64_t> perm((size_t)n_bp);
    {
        std::vector<int64_t> pos(count.begin(), count.end() - 1);
        for (int64_t i = 0; i < n_bp; ++i) perm[pos[cls_of[i]]++] = i;
    }
    std::vector<int64_t> groups;       // (class, first, count) triples
    std::vector<int64_t> group_start;  // first group of each class
    for (int c = 0; c < n_cls; ++c) {
        group_start.push_back((int64_t)groups.size() / 3);
        for (int64_t f = count[c]; f < count[c + 1]; f += kGroup) {
            groups.push_back(c);
            groups.push_back(f);
            groups.push_back(std::min<int64_t>(kGroup, count[c + 1] - f));
        }
    }
    group_start.push_back((int64_t)groups.size() / 3);
    // 2. device copies of the class bookkeeping
    d_perm = (int64_t*)scratch(ctx, kSlotClsPerm, sizeof(int64_t) * n_bp, &st);
    d_groups = (int64_t*)scratch(ctx, kSlotClsGroups, sizeof(int64_t) * groups.size(), &st);
    if (st) return st;
    ce = cudaMemcpyAsync(d_perm, perm.data(), sizeof(int64_t) * n_bp, cudaMemcpyHostToDevice,
                         ctx->stream);
    if (ce == cudaSuccess)
        ce = cudaMemcpyAsync(d_groups, groups.data(), sizeof(int64_t) * groups.size(),
                             cudaMemcpyHostToDevice, ctx->stream);
    // perm / groups are pageable host vectors of this scope: the copies must
    // have left them before they go away
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(ctx->stream);
    if ((st = cuda_check(ctx, ce, "class tables h2d"))) return st;
    C.n_bp = n_bp; C.bands = bands; C.az = az; C.np = np; C.depth = depth; C.kind = kind;
    C.n_nodes = n_nodes; C.n_rule = n_rule; C.tol = tol;
    std::memcpy(C.hash, hkey, sizeof hkey);
    C.n_cls = n_cls;
    C.canon = std::move(canon);
    C.group_start = std::move(group_start);
    C.n_group_words = groups.size();
    C.solver_fail = false;
    C.valid = true;
    }
    const int n_cls = C.n_cls;
    const std::vector<bw_patch>& canon = C.canon;
    const std::vector<int64_t>& group_start = C.group_start;
    // 3. classes in chunks bounded by table memory (~1 GiB)
    const size_t per_class = sizeof(double) * (d.sA + (size_t)2 * (az + 1) * d.m + d.sKg +
                                               3 * (size_t)d.m + az + d.sLq + d.sH + n_nodes + 1) +
                             sizeof(Mesh) + sizeof(bw_patch) + sizeof(int32_t) + 64;
    int chunk = (int)std::max<size_t>(1, ((size_t)1 << 30) / per_class);
    chunk = std::min(chunk, n_cls);
    ClassTables T;
    {
        const size_t nc = (size_t)chunk;
        T.canon = (const bw_patch*)scratch(ctx, kSlotClsCanon, sizeof(bw_patch) * nc, &st);
        T.mesh = (Mesh*)scratch(ctx, kSlotClsMesh, sizeof(Mesh) * nc, &st);
        T.At = (double*)scratch(ctx, kSlotClsA, sizeof(double) * nc * d.sA, &st);
        T.R = (double*)scratch(ctx, kSlotClsR, sizeof(double) * nc * (az + 1) * d.m, &st);
        T.Z = (double*)scratch(ctx, kSlotClsZ, sizeof(double) * nc * (az + 1) * d.m, &st);
        T.Kg = (double*)scratch(ctx, kSlotClsKg, sizeof(double) * nc * d.sKg, &st);
        double* rows = (double*)scratch(ctx, kSlotClsRows, sizeof(double) * nc * (2 * d.m + az), &st);
        T.lq = (double*)scratch(ctx, kSlotClsLq, sizeof(double) * nc * d.sLq, &st);
        T.H = (double*)scratch(ctx, kSlotClsH, sizeof(double) * nc * d.sH, &st);
        T.hK = (double*)scratch(ctx, kSlotClsHK, sizeof(double) * nc * n_nodes, &st);
        T.info = (int32_t*)scratch(ctx, kSlotClsInfo, sizeof(int32_t) * nc, &st);
        T.resid = (double*)scratch(ctx, kSlotClsResid, sizeof(double) * nc, &st);
        if (st) return st;
        T.rowKg = rows;
        T.rowD = rows + nc * d.m;
        T.wfan = rows + 2 * nc * d.m;
    }
    const size_t geom_dyn = sizeof(double) * (4 * (size_t)n_nodes + 3 * (size_t)np * np);
    const size_t h_dyn = sizeof(double) * 3 * (size_t)np * np;
    ce = cudaFuncSetAttribute(class_geom_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)geom_dyn);
    if ((st = cuda_check(ctx, ce, "class geom attr"))) return st;
    // all classes in one chunk and the key unchanged: the tables of the previous
    // call are still in their scratch slots (only this function writes them)
    const bool reuse_tables = hit && C.tables_valid && chunk >= n_cls && C.chunk == chunk;
    bool solver_fail = reuse_tables ? C.solver_fail : false;
    if (!reuse_tables) C.tables_valid = false; // until this build completes
    std::vector<int32_t> hinfo;
    for (int c0 = 0; c0 < n_cls; c0 += chunk) {
        const int nc = std::min(chunk, n_cls - c0);
        if (!reuse_tables) {
            ce = cudaMemcpyAsync((void*)T.canon, canon.data() + c0, sizeof(bw_patch) * nc,
                                 cudaMemcpyHostToDevice, ctx->stream);
            if ((st = cuda_check(ctx, ce, "class canon h2d"))) return st;
            ++ctx->launches;
            class_geom_kernel<<<nc, kGeomThreads, geom_dyn, ctx->stream>>>(T, d, bands, d_dirs,
                                                                           d_weights, d_gl);
            if ((st = cuda_check(ctx, cudaGetLastError(), "class geom launch"))) return st;
            ce = launch_lu(ctx, d.m, nc, T.At, T.R, az + 1, tol, T.Z, T.resid, T.info);
            if ((st = cuda_check(ctx, ce, "class lu launch"))) return st;
            const dim3 hgrid((unsigned)((d.Qt + kHThreads - 1) / kHThreads), (unsigned)nc);
            ++ctx->launches;
            class_h_kernel<<<hgrid, kHThreads, h_dyn, ctx->stream>>>(T, d, d_gl);
            if ((st = cuda_check(ctx, cudaGetLastError(), "class h launch"))) return st;
        }
        const int64_t g0 = group_start[c0], g1 = group_start[c0 + nc];
        const int64_t* dg = d_groups + 3 * g0;
#define BW_APPLY(P) launch_apply_t<P>(ctx, S, T, d, c0, d_patches, d_perm, dg, g1 - g0, d_est, \
                                      d_dudn, d_err, d_status)
        switch (S.phi_kind) {
            case BW_PHI_FEATURE_CONST: ce = BW_APPLY(BW_PHI_FEATURE_CONST); break;
            case BW_PHI_QUADRATIC: ce = BW_APPLY(BW_PHI_QUADRATIC); break;
            case BW_PHI_EXP_SIN_SIN: ce = BW_APPLY(BW_PHI_EXP_SIN_SIN); break;
            case BW_PHI_SIN_SIN: ce = BW_APPLY(BW_PHI_SIN_SIN); break;
            default: ce = BW_APPLY(BW_PHI_POINT_SOURCE); break;
        }
#undef BW_APPLY
        if ((st = cuda_check(ctx, ce, "class apply launch"))) return st;
        if (reuse_tables) continue; // the residual gate ran when the tables were built
        hinfo.resize(nc);
        ce = cudaMemcpyAsync(hinfo.data(), T.info, sizeof(int32_t) * nc, cudaMemcpyDeviceToHost,
                             ctx->stream);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(ctx->stream);
        if ((st = cuda_check(ctx, ce, "class info d2h"))) return st;
        for (int c = 0; c < nc; ++c) solver_fail |= hinfo[c] != 0;
    }
    C.chunk = chunk;
    C.tables_valid = chunk >= n_cls;
    C.solver_fail = solver_fail;
    if (solver_fail) return fail(ctx, BW_ERR_SOLVER, "patch solve residual above tolerance (SolverError)");
    return BW_OK;
}

} // namespace bw
