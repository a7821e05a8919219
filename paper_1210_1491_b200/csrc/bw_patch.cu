// bw_patch.cu — K4: per-patch local-BIE collocation assembly on the device,
// and K5: the Neumann value at each boundary point from the solved patch.
//
// Replaces, per boundary point, the reference's host loop
//   make_*_patch_setup (patch_solver.cpp:62-121) -> assemble (:197-309)
// (second kind, or first kind: BW_BIE_FIRST) with one CTA per patch:
//   mesh     fan + band triangulation (patch_solver.cpp:26-52), normals into
//            the solution domain; sphere or plane surface (BASELINE geometries)
//   Gamma    the K1 node estimates at the theta-GL x phi-uniform nodes,
//            positions recomputed bit-identically to K1
//   b_i      -sum_k w_k d2G(x_i,n_i,y_k,ny_k)(u_k - u_i)   (warp per row)
//   A_ij, +b self/near panels: warp-cooperative polar-split / depth-2 refined
//            rules (quadrature.hpp:60-98); far panels: thread per pair, deg-5
//   b_se_i   sqrt(sum (w_k K)^2 var_k)
// Every sum has a fixed order, so results are deterministic; they differ from
// the sequential CPU oracle only by rounding (parity gate 1e-10).
#include <cmath>

#include "bw_patch_common.cuh"

namespace bw {

namespace {

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;

struct PairCtx {
    V3 xl, nx, ny; // collocation point (relative to o), its normal, panel normal
    double ui;
    int kind;      // BW_BIE_SECOND / BW_BIE_FIRST
};

// one quadrature point at y (absolute): the A-kernel and the b-kernel times
// (phi(y) - u_i) of the BIE kind (second: dG/dn_x, d2G; first: G, dG/dn_y)
template <int PHI>
__device__ __forceinline__ void pair_kernels(const DevScene& S, const PatchGeo& g,
                                             const PairCtx& c, V3 y, double& ka, double& kb) {
    double k2;
    bie_kernels(c.kind, g.a, c.xl, c.nx, y - g.o, c.ny, ka, k2);
    kb = k2 * (phi_on_patch<PHI>(S, g, y) - c.ui);
}

struct Smem {
    Mesh mesh;
    double ucoll[64];
    double bg[64], vg[64];
    double B[64][65]; // panel contributions to b, summed in panel order
    double gl_x[32], gl_w[32];
    int clipped;
};

// The Gamma node arrays are dynamic shared memory: y[n][3], w[n], um[n], uv[n]
template <int PHI>
__global__ void __launch_bounds__(kThreads, 4)
    assemble_kernel(const DevScene S, const bw_patch* __restrict__ patches, int64_t n_bp,
                    const double* __restrict__ dirs, const double* __restrict__ wts, int n_nodes,
                    const bw_estimate* __restrict__ est, int bands, int az, int gauss_polar,
                    int near_depth, int kind, const double* __restrict__ gl,
                    double* __restrict__ A_out,
                    double* __restrict__ b_out, double* __restrict__ area_out,
                    double* __restrict__ cen_out,
                    int32_t* __restrict__ flags) {
    __shared__ Smem sm;
    extern __shared__ __align__(16) double gam[];
    double* gy = gam;
    double* gw = gy + 3 * n_nodes;
    double* gum = gw + n_nodes;
    double* guv = gum + n_nodes;
    // polar rule table (integrate_triangle_polar, quadrature.hpp:60-78):
    // point q = (i, j): s = (x_i + 1)/2, t = (x_j + 1)/2, weight w_i (w_j t / 4)
    double* ps = guv + n_nodes;
    double* pt_ = ps + gauss_polar * gauss_polar;
    double* pw = pt_ + gauss_polar * gauss_polar;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int m = az * (2 * bands - 1);
    if (tid < gauss_polar) {
        sm.gl_x[tid] = gl[tid];
        sm.gl_w[tid] = gl[32 + tid];
    }
    for (int q = tid; q < gauss_polar * gauss_polar; q += kThreads) {
        const int i = q / gauss_polar, j = q % gauss_polar;
        const double t = 0.5 * (gl[j] + 1.0);
        ps[q] = 0.5 * (gl[i] + 1.0);
        pt_[q] = t;
        pw[q] = gl[32 + i] * (0.25 * gl[32 + j] * t);
    }

    for (int64_t bp = blockIdx.x; bp < n_bp; bp += gridDim.x) {
        const bw_patch P = patches[bp];
        const PatchGeo g = patch_geo(P);
        if (tid == 0) sm.clipped = 0;
        // ---- mesh (patch_solver.cpp:26-52, 62-121) ----
        build_mesh(g, bands, az, view(sm.mesh), tid, kThreads);
        for (int t = tid; t < m; t += kThreads) {
            area_out[bp * m + t] = sm.mesh.area[t];
            if (cen_out) stv(cen_out + 3 * (bp * m + t), ldv(sm.mesh.cen[t]));
            sm.ucoll[t] = phi_on_patch<PHI>(S, g, ldv(sm.mesh.cen[t]));
        }
        // ---- Gamma nodes: K1's node formula (bit-identical positions) ----
        {
            for (int j = tid; j < n_nodes; j += kThreads) {
                double x, y, z;
                patch_node_local(P.o, P.axis, P.a, dirs + ((int64_t)P.cls * n_nodes + j) * 3, x, y,
                                 z);
                gy[3 * j] = x;
                gy[3 * j + 1] = y;
                gy[3 * j + 2] = z;
                const bw_estimate e = est[bp * n_nodes + j];
                const bool ok = e.n > 0;
                gw[j] = ok ? wts[(int64_t)P.cls * n_nodes + j] * (P.a * P.a) : 0.0;
                gum[j] = ok ? e.mean : 0.0;
                guv[j] = ok ? e.variance / (double)e.n : 0.0;
                if (!ok) atomicOr(&sm.clipped, 1);
            }
        }
        __syncthreads();
        // ---- Gamma part of b (patch_solver.cpp:253-262): warp per row ----
        for (int i = warp; i < m; i += kWarps) {
            const V3 xl = ldv(sm.mesh.cen[i]) - g.o, ni = ldv(sm.mesh.nrm[i]);
            const double ui = sm.ucoll[i];
            double bg = 0.0, vg = 0.0;
            for (int k = lane; k < n_nodes; k += 32) {
                const V3 yl = ldv(gy + 3 * k) - g.o;
                const V3 ny = (1.0 / g.a) * yl;
                double ka_unused, kk;
                bie_kernels(kind, g.a, xl, ni, yl, ny, ka_unused, kk);
                const double wk = gw[k] * kk;
                bg = fma(wk, gum[k] - ui, bg);
                vg = fma(wk * wk, guv[k], vg);
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                bg += __shfl_down_sync(0xffffffffu, bg, off);
                vg += __shfl_down_sync(0xffffffffu, vg, off);
            }
            if (lane == 0) {
                sm.bg[i] = bg;
                sm.vg[i] = vg;
            }
        }
        // ---- panel integrals: self + near, warp-cooperative ----
        const int np = gauss_polar;
        for (int i = warp; i < m; i += kWarps) {
            PairCtx c;
            c.kind = kind;
            c.xl = ldv(sm.mesh.cen[i]) - g.o;
            c.nx = ldv(sm.mesh.nrm[i]);
            c.ui = sm.ucoll[i];
            const V3 xi = ldv(sm.mesh.cen[i]);
            for (int j = 0; j < m; ++j) {
                const double dist = len(xi - ldv(sm.mesh.cen[j]));
                const bool self = j == i;
                if (!self && !(dist < 2.0 * sm.mesh.diam[j])) continue; // far: phase B
                c.ny = ldv(sm.mesh.nrm[j]);
                const V3 v0 = ldv(sm.mesh.verts[sm.mesh.tris[j][0]]), v1 = ldv(sm.mesh.verts[sm.mesh.tris[j][1]]),
                         v2 = ldv(sm.mesh.verts[sm.mesh.tris[j][2]]);
                double sa = 0.0, sb = 0.0;
                if (self) {
                    // integrate_triangle_split: 3 polar sub-triangles about xi
                    // (s, t, w) of the n x n polar rule come from a shared table
                    const int per = np * np;
#pragma unroll 1
                    for (int sub = 0; sub < 3; ++sub) {
                        const V3 a0 = sub == 0 ? v0 : (sub == 1 ? v1 : v2);
                        const V3 a1 = sub == 0 ? v1 : (sub == 1 ? v2 : v0);
                        const double area2 = len(cross(a0 - xi, a1 - xi));
                        for (int q = lane; q < per; q += 32) {
                            const double s = ps[q], t = pt_[q];
                            const V3 w = a0 + s * (a1 - a0);
                            const double wq = area2 * pw[q];
                            double ka, kb;
                            pair_kernels<PHI>(S, g, c, xi + t * (w - xi), ka, kb);
                            sa = fma(wq, ka, sa);
                            sb = fma(wq, kb, sb);
                        }
                    }
                } else {
                    // integrate_triangle_refined, depth near_depth (4^depth leaves x 7)
                    const int leaves = 1 << (2 * near_depth);
                    for (int q = lane; q < leaves * 7; q += 32) {
                        const int leaf = q / 7;
                        const int pt = q % 7;
                        V3 a0 = v0, a1 = v1, a2 = v2;
                        refine_leaf(a0, a1, a2, leaf, near_depth);
                        const double area = 0.5 * len(cross(a1 - a0, a2 - a0));
                        const V3 y = kTriB[pt][0] * a0 + kTriB[pt][1] * a1 + kTriB[pt][2] * a2;
                        double ka, kb;
                        pair_kernels<PHI>(S, g, c, y, ka, kb);
                        sa = fma(area * kTriW[pt], ka, sa);
                        sb = fma(area * kTriW[pt], kb, sb);
                    }
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    sa += __shfl_down_sync(0xffffffffu, sa, off);
                    sb += __shfl_down_sync(0xffffffffu, sb, off);
                }
                if (lane == 0) {
                    A_out[(bp * m + i) * m + j] = self && kind == BW_BIE_SECOND ? 0.5 + sa : sa;
                    sm.B[i][j] = sb;
                }
            }
        }
        // ---- far panels: thread per pair, degree-5 rule ----
        for (int pq = tid; pq < m * m; pq += kThreads) {
            const int i = pq / m, j = pq % m;
            const V3 xi = ldv(sm.mesh.cen[i]);
            const double dist = len(xi - ldv(sm.mesh.cen[j]));
            if (i == j || dist < 2.0 * sm.mesh.diam[j]) continue;
            PairCtx c;
            c.kind = kind;
            c.xl = xi - g.o;
            c.nx = ldv(sm.mesh.nrm[i]);
            c.ny = ldv(sm.mesh.nrm[j]);
            c.ui = sm.ucoll[i];
            const V3 v0 = ldv(sm.mesh.verts[sm.mesh.tris[j][0]]), v1 = ldv(sm.mesh.verts[sm.mesh.tris[j][1]]),
                     v2 = ldv(sm.mesh.verts[sm.mesh.tris[j][2]]);
            const double area = 0.5 * len(cross(v1 - v0, v2 - v0));
            double sa = 0.0, sb = 0.0;
#pragma unroll
            for (int pt = 0; pt < 7; ++pt) {
                const V3 y = kTriB[pt][0] * v0 + kTriB[pt][1] * v1 + kTriB[pt][2] * v2;
                double ka, kb;
                pair_kernels<PHI>(S, g, c, y, ka, kb);
                sa = fma(kTriW[pt], ka, sa);
                sb = fma(kTriW[pt], kb, sb);
            }
            A_out[(bp * m + i) * m + j] = area * sa;
            sm.B[i][j] = area * sb;
        }
        __syncthreads();
        // ---- b = -Gamma part + panel contributions in panel order ----
        for (int i = tid; i < m; i += kThreads) {
            double b = -sm.bg[i];
            for (int j = 0; j < m; ++j) b += sm.B[i][j];
            b_out[(bp * 2 + 0) * m + i] = b;
            b_out[(bp * 2 + 1) * m + i] = sqrt(sm.vg[i]);
        }
        if (tid == 0) flags[bp] = sm.clipped;
        __syncthreads();
    }
}

// K5: Neumann value at the boundary point = area-weighted mean of du/dn over
// the `az` fan panels around the apex (their normals point into the domain);
// reported along the domain-OUTWARD normal (sign flip), with the propagated
// WOS error sum(area |A^-1 b_se|) / sum(area).
__global__ void point_value_kernel(int64_t n_bp, int m, int az, const double* __restrict__ X,
                                   const double* __restrict__ area,
                                   const int32_t* __restrict__ info,
                                   const int32_t* __restrict__ flags, double* __restrict__ dudn,
                                   double* __restrict__ err, int32_t* __restrict__ status) {
    const int64_t bp = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (bp >= n_bp) return;
    double s = 0.0, se = 0.0, at = 0.0;
    for (int j = 0; j < az; ++j) { // fan panels 0..az-1 (patch_solver.cpp:31)
        const double w = area[bp * m + j];
        s += w * X[(bp * 2 + 0) * m + j];
        se += w * fabs(X[(bp * 2 + 1) * m + j]);
        at += w;
    }
    dudn[bp] = -s / at;
    err[bp] = se / at;
    status[bp] = (info[bp] ? 2 : 0) | (flags[bp] ? 1 : 0);
}

// solve_patch's NeumannField (patch_solver.cpp:311-335, patch_solver.hpp:78-82)
// per panel: du/dn along the panel normal (into the domain), r = |centroid - o|,
// est_error = |A^-1 b_se|.
__global__ void patch_field_kernel(int64_t n_bp, int m, const bw_patch* __restrict__ patches,
                                   const double* __restrict__ X, const double* __restrict__ cen,
                                   double* __restrict__ dudn, double* __restrict__ r,
                                   double* __restrict__ est_error) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_bp * m) return;
    const int64_t bp = e / m;
    const int i = (int)(e - bp * m);
    const bw_patch P = patches[bp];
    dudn[e] = X[(bp * 2 + 0) * m + i];
    est_error[e] = fabs(X[(bp * 2 + 1) * m + i]);
    const double dx = cen[3 * e] - P.o[0], dy = cen[3 * e + 1] - P.o[1], dz = cen[3 * e + 2] - P.o[2];
    r[e] = sqrt(dx * dx + dy * dy + dz * dz);
}

__global__ void unpack_kernel(const bw_patch* __restrict__ p, int64_t n, double* __restrict__ c,
                              double* __restrict__ ax, double* __restrict__ r,
                              int32_t* __restrict__ cls) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bw_patch q = p[i];
    for (int k = 0; k < 3; ++k) {
        c[3 * i + k] = q.o[k];
        ax[3 * i + k] = q.axis[k];
    }
    r[i] = q.a;
    cls[i] = q.cls;
}

__global__ void check_classes_kernel(const bw_patch* __restrict__ p, int64_t n, int32_t n_cls,
                                     unsigned long long* __restrict__ ctr) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && (p[i].cls < 0 || p[i].cls >= n_cls)) atomicAdd(&ctr[kCtrBadClass], 1ull);
}

template <int PHI>
cudaError_t launch_assemble_t(bw_ctx* ctx, const DevScene& S, const bw_patch* patches,
                              int64_t n_bp, const double* dirs, const double* wts, int n_nodes,
                              const bw_estimate* est, int bands, int az, int gauss_polar,
                              int near_depth, int kind, const double* d_gl, double* A, double* b,
                              double* area, double* cen, int32_t* flags) {
    const size_t dyn = sizeof(double) * (6 * (size_t)n_nodes + 3 * (size_t)gauss_polar * gauss_polar);
    auto kern = assemble_kernel<PHI>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, dyn);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    int64_t blocks = (int64_t)ctx->sm_count * per_sm;
    if (blocks > n_bp) blocks = n_bp;
    ++ctx->launches;
    kern<<<(unsigned)blocks, kThreads, dyn, ctx->stream>>>(S, patches, n_bp, dirs, wts, n_nodes, est,
                                                          bands, az, gauss_polar, near_depth, kind,
                                                          d_gl, A, b, area, cen, flags);
    return cudaGetLastError();
}

} // namespace

cudaError_t launch_unpack_patches(bw_ctx* ctx, const bw_patch* patches, int64_t n, double* centers,
                                  double* axes, double* radii, int32_t* cls) {
    if (n <= 0) return cudaSuccess;
    ++ctx->launches;
    unpack_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(patches, n, centers, axes,
                                                                        radii, cls);
    return cudaGetLastError();
}

cudaError_t launch_check_classes(bw_ctx* ctx, const bw_patch* patches, int64_t n, int32_t n_cls) {
    if (n <= 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(ctx->d_counters + kCtrBadClass, 0, sizeof(unsigned long long),
                                    ctx->stream);
    if (e != cudaSuccess) return e;
    ++ctx->launches;
    check_classes_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(patches, n, n_cls,
                                                                              ctx->d_counters);
    return cudaGetLastError();
}

cudaError_t launch_assemble(bw_ctx* ctx, const DevScene& S, const bw_patch* patches, int64_t n_bp,
                            const double* dirs, const double* wts, int n_nodes,
                            const bw_estimate* est, int bands, int az, int gauss_polar,
                            int near_depth, int kind, const double* d_gl, double* A, double* b,
                            double* area, double* cen, int32_t* flags) {
    if (n_bp <= 0) return cudaSuccess;
#define BW_ASM(P) launch_assemble_t<P>(ctx, S, patches, n_bp, dirs, wts, n_nodes, est, bands, az, \
                                       gauss_polar, near_depth, kind, d_gl, A, b, area, cen, flags)
    switch (S.phi_kind) {
        case BW_PHI_FEATURE_CONST: return BW_ASM(BW_PHI_FEATURE_CONST);
        case BW_PHI_QUADRATIC: return BW_ASM(BW_PHI_QUADRATIC);
        case BW_PHI_EXP_SIN_SIN: return BW_ASM(BW_PHI_EXP_SIN_SIN);
        case BW_PHI_SIN_SIN: return BW_ASM(BW_PHI_SIN_SIN);
        default: return BW_ASM(BW_PHI_POINT_SOURCE);
    }
#undef BW_ASM
}

cudaError_t launch_patch_field(bw_ctx* ctx, int64_t n_bp, int m, const bw_patch* patches,
                               const double* X, const double* cen, double* dudn, double* r,
                               double* est_error) {
    if (n_bp <= 0) return cudaSuccess;
    const int64_t n = n_bp * m;
    ++ctx->launches;
    patch_field_kernel<<<(unsigned)((n + 127) / 128), 128, 0, ctx->stream>>>(n_bp, m, patches, X, cen,
                                                                           dudn, r, est_error);
    return cudaGetLastError();
}

cudaError_t launch_point_values(bw_ctx* ctx, int64_t n_bp, int m, int az, const double* X,
                                const double* area, const int32_t* info, const int32_t* flags,
                                double* dudn, double* err, int32_t* status) {
    if (n_bp <= 0) return cudaSuccess;
    ++ctx->launches;
    point_value_kernel<<<(unsigned)((n_bp + 127) / 128), 128, 0, ctx->stream>>>(
        n_bp, m, az, X, area, info, flags, dudn, err, status);
    return cudaGetLastError();
}

} // namespace bw
