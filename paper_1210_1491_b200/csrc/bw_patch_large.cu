// bw_patch_large.cu — solve_patch for meshes beyond the warp-per-system path:
// the reference's biewos_patch default (16 bands x 36 azimuth = 1116 panels,
// 64 x 128 Gamma nodes, patch_solver.cpp:62-121, 197-335).
//
//   gamma_nodes_kernel     Gamma nodes of every patch (K1's node formula), their
//                          weights and node data (zero weight outside the domain)
//                          as SoA in HBM
//   assemble_large_kernel  grid (row blocks, patch): the mesh lives in dynamic
//                          shared memory (~100 B per panel), a warp per row i:
//                          Gamma sum over lanes, far panels lane-parallel (degree-5
//                          rule), self / near panels warp-cooperative (polar split /
//                          refined), both BIE kinds; rows straight to HBM
//   lu_large_kernel        one CTA per system: right-looking LU with first-max
//                          partial pivoting (Eigen's PartialPivLU choice) on the
//                          system in HBM, forward elimination of both right-hand
//                          sides fused, back substitution, the 1e-10 residual gate
//                          against the original matrix (patch_solver.cpp:314-324)
// The per-panel field then comes from patch_field_kernel (bw_patch.cu).
#include <cmath>

#include "bw_patch_common.cuh"

namespace bw {

namespace {

constexpr int kLThreads = 128;
constexpr int kLWarps = kLThreads / 32;
constexpr int kLuThreads = 1024;

__global__ void gamma_nodes_kernel(const bw_patch* __restrict__ patches, int64_t n_bp,
                                   const double* __restrict__ dirs, const double* __restrict__ wts,
                                   int n_nodes, const bw_estimate* __restrict__ est,
                                   double* __restrict__ gam, int32_t* __restrict__ flags) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_bp * n_nodes) return;
    const int64_t bp = e / n_nodes;
    const int k = (int)(e - bp * n_nodes);
    const bw_patch P = patches[bp];
    double x, y, z;
    patch_node_local(P.o, P.axis, P.a, dirs + ((int64_t)P.cls * n_nodes + k) * 3, x, y, z);
    double* G = gam + bp * 6 * (int64_t)n_nodes; // SoA: x, y, z, w, mean, var/n
    G[k] = x;
    G[n_nodes + k] = y;
    G[2 * n_nodes + k] = z;
    const bw_estimate s = est[e];
    const bool ok = s.n > 0;
    G[3 * n_nodes + k] = ok ? wts[(int64_t)P.cls * n_nodes + k] * (P.a * P.a) : 0.0;
    G[4 * n_nodes + k] = ok ? s.mean : 0.0;
    G[5 * n_nodes + k] = ok ? s.variance / (double)s.n : 0.0;
    if (!ok) atomicOr(&flags[bp], 1);
}

template <int PHI>
__global__ void __launch_bounds__(kLThreads)
    assemble_large_kernel(const DevScene S, const bw_patch* __restrict__ patches,
                          const double* __restrict__ gam, int n_nodes, int bands, int az, int np,
                          int depth, int kind, const double* __restrict__ gl, int rows_per_block,
                          double* __restrict__ A_out, double* __restrict__ b_out,
                          double* __restrict__ cen_out) {
    extern __shared__ __align__(16) double dyn[];
    const int m = az * (2 * bands - 1), nv = 1 + bands * az;
    MeshView M;
    M.verts = reinterpret_cast<double(*)[3]>(dyn);
    M.cen = reinterpret_cast<double(*)[3]>(dyn + 3 * nv);
    M.nrm = reinterpret_cast<double(*)[3]>(dyn + 3 * nv + 3 * m);
    M.area = dyn + 3 * nv + 6 * m;
    M.diam = M.area + m;
    double* ucoll = M.diam + m;
    double* ps = ucoll + m;
    double* pt_ = ps + np * np;
    double* pw = pt_ + np * np;
    M.tris = reinterpret_cast<int(*)[3]>(pw + np * np);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t bp = blockIdx.y;
    const bw_patch P = patches[bp];
    const PatchGeo g = patch_geo(P);
    for (int q = tid; q < np * np; q += kLThreads) {
        const int i = q / np, j = q % np;
        const double t = 0.5 * (gl[j] + 1.0);
        ps[q] = 0.5 * (gl[i] + 1.0);
        pt_[q] = t;
        pw[q] = gl[32 + i] * (0.25 * gl[32 + j] * t);
    }
    build_mesh(g, bands, az, M, tid, kLThreads);
    for (int t = tid; t < m; t += kLThreads) ucoll[t] = phi_on_patch<PHI>(S, g, ldv(M.cen[t]));
    if (blockIdx.x == 0 && cen_out)
        for (int t = tid; t < m; t += kLThreads) stv(cen_out + 3 * (bp * m + t), ldv(M.cen[t]));
    __syncthreads();
    const double* G = gam + bp * 6 * (int64_t)n_nodes;
    const int i0 = blockIdx.x * rows_per_block;
    const int i1 = min(m, i0 + rows_per_block);
    for (int i = i0 + warp; i < i1; i += kLWarps) {
        const V3 xi = ldv(M.cen[i]);
        const V3 xl = xi - g.o, nx = ldv(M.nrm[i]);
        const double ui = ucoll[i];
        // Gamma part of b (patch_solver.cpp:253-262)
        double bg = 0.0, vg = 0.0;
        for (int k = lane; k < n_nodes; k += 32) {
            const V3 yl = v3(G[k], G[n_nodes + k], G[2 * n_nodes + k]) - g.o;
            const V3 ny = (1.0 / g.a) * yl;
            double ka_unused, kk;
            bie_kernels(kind, g.a, xl, nx, yl, ny, ka_unused, kk);
            const double wk = G[3 * n_nodes + k] * kk;
            bg = fma(wk, G[4 * n_nodes + k] - ui, bg);
            vg = fma(wk * wk, G[5 * n_nodes + k], vg);
        }
        // panel integrals (patch_solver.cpp:264-306), 32 panels per chunk
        double bs = 0.0;
        double* Arow = A_out + (bp * m + i) * (int64_t)m;
        for (int j0 = 0; j0 < m; j0 += 32) {
            const int j = j0 + lane;
            bool far = false;
            if (j < m) {
                const double dist = len(xi - ldv(M.cen[j]));
                far = j != i && !(dist < 2.0 * M.diam[j]);
            }
            if (far) { // degree-5 rule on the whole panel
                const V3 ny = ldv(M.nrm[j]);
                const V3 v0 = ldv(M.verts[M.tris[j][0]]), v1 = ldv(M.verts[M.tris[j][1]]),
                         v2 = ldv(M.verts[M.tris[j][2]]);
                const double area = 0.5 * len(cross(v1 - v0, v2 - v0));
                double sa = 0.0, sb = 0.0;
#pragma unroll
                for (int p = 0; p < 7; ++p) {
                    const V3 y = kTriB[p][0] * v0 + kTriB[p][1] * v1 + kTriB[p][2] * v2;
                    double ka, kb;
                    bie_kernels(kind, g.a, xl, nx, y - g.o, ny, ka, kb);
                    sa = fma(kTriW[p], ka, sa);
                    sb = fma(kTriW[p], kb * (phi_on_patch<PHI>(S, g, y) - ui), sb);
                }
                Arow[j] = area * sa;
                bs += area * sb;
            }
            unsigned near = __ballot_sync(0xffffffffu, j < m && !far);
            while (near) {
                const int jj = j0 + __ffs(near) - 1;
                near &= near - 1;
                const bool self = jj == i;
                const V3 ny = ldv(M.nrm[jj]);
                const V3 v0 = ldv(M.verts[M.tris[jj][0]]), v1 = ldv(M.verts[M.tris[jj][1]]),
                         v2 = ldv(M.verts[M.tris[jj][2]]);
                double sa = 0.0, sb = 0.0;
                if (self) { // polar split about x_i
                    const int per = np * np;
#pragma unroll 1
                    for (int sub = 0; sub < 3; ++sub) {
                        const V3 a0 = sub == 0 ? v0 : (sub == 1 ? v1 : v2);
                        const V3 a1 = sub == 0 ? v1 : (sub == 1 ? v2 : v0);
                        const double area2 = len(cross(a0 - xi, a1 - xi));
                        for (int q = lane; q < per; q += 32) {
                            const V3 w = a0 + ps[q] * (a1 - a0);
                            const V3 y = xi + pt_[q] * (w - xi);
                            const double wq = area2 * pw[q];
                            double ka, kb;
                            bie_kernels(kind, g.a, xl, nx, y - g.o, ny, ka, kb);
                            sa = fma(wq, ka, sa);
                            sb = fma(wq, kb * (phi_on_patch<PHI>(S, g, y) - ui), sb);
                        }
                    }
                } else { // refined, 4^depth leaves x 7 points
                    const int leaves = 1 << (2 * depth);
                    for (int q = lane; q < leaves * 7; q += 32) {
                        const int leaf = q / 7, p = q % 7;
                        V3 a0 = v0, a1 = v1, a2 = v2;
                        refine_leaf(a0, a1, a2, leaf, depth);
                        const double area = 0.5 * len(cross(a1 - a0, a2 - a0));
                        const V3 y = kTriB[p][0] * a0 + kTriB[p][1] * a1 + kTriB[p][2] * a2;
                        double ka, kb;
                        bie_kernels(kind, g.a, xl, nx, y - g.o, ny, ka, kb);
                        sa = fma(area * kTriW[p], ka, sa);
                        sb = fma(area * kTriW[p], kb * (phi_on_patch<PHI>(S, g, y) - ui), sb);
                    }
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    sa += __shfl_down_sync(0xffffffffu, sa, off);
                    sb += __shfl_down_sync(0xffffffffu, sb, off);
                }
                if (lane == 0) {
                    Arow[jj] = self && kind == BW_BIE_SECOND ? 0.5 + sa : sa;
                    bs += sb;
                }
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            bg += __shfl_down_sync(0xffffffffu, bg, off);
            vg += __shfl_down_sync(0xffffffffu, vg, off);
            bs += __shfl_down_sync(0xffffffffu, bs, off);
        }
        if (lane == 0) {
            b_out[(bp * 2 + 0) * m + i] = bs - bg;
            b_out[(bp * 2 + 1) * m + i] = sqrt(vg);
        }
    }
}

// block-wide argmax of |v| with the lowest index on ties
__device__ __forceinline__ void block_argmax(double v, int idx, double* sv, int* si, double& best,
                                             int& bi) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, off);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, off);
        if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
    }
    if (lane == 0) { sv[warp] = v; si[warp] = idx; }
    __syncthreads();
    if (warp == 0) {
        v = lane < (int)(blockDim.x >> 5) ? sv[lane] : -1.0;
        idx = lane < (int)(blockDim.x >> 5) ? si[lane] : 0x7fffffff;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, off);
            const int oi = __shfl_xor_sync(0xffffffffu, idx, off);
            if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
        }
        if (lane == 0) { sv[0] = v; si[0] = idx; }
    }
    __syncthreads();
    best = sv[0];
    bi = si[0];
    __syncthreads();
}

__device__ __forceinline__ double block_sum(double v, double* sv) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if (lane == 0) sv[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sv[w];
        sv[0] = s;
    }
    __syncthreads();
    s = sv[0];
    __syncthreads();
    return s;
}

// One CTA per system: A (m x m, overwritten by its LU), B (2 x m, overwritten),
// A0 / B0 untouched copies for the residual; X (2 x m).
__global__ void __launch_bounds__(kLuThreads)
    lu_large_kernel(int m, double* __restrict__ A, double* __restrict__ B,
                    const double* __restrict__ A0, const double* __restrict__ B0, double tol,
                    double* __restrict__ X, double* __restrict__ resid, int32_t* __restrict__ info) {
    __shared__ double sv[32];
    __shared__ int si[32];
    const int64_t s = blockIdx.x;
    double* a = A + s * (int64_t)m * m;
    double* b = B + s * 2 * (int64_t)m;
    const double* a0 = A0 + s * (int64_t)m * m;
    const double* b0 = B0 + s * 2 * (int64_t)m;
    double* x = X + s * 2 * (int64_t)m;
    const int tid = threadIdx.x, nt = blockDim.x;
    int sing = 0;
    for (int k = 0; k < m; ++k) {
        double v = -1.0;
        int bi = 0x7fffffff;
        for (int r = k + tid; r < m; r += nt) {
            const double av = fabs(a[(int64_t)r * m + k]);
            if (av > v) { v = av; bi = r; }
        }
        double best;
        int p;
        block_argmax(v, bi, sv, si, best, p);
        if (!(best > 0.0)) { sing = 1; continue; }
        if (p != k) {
            for (int c = tid; c < m; c += nt) {
                const double t = a[(int64_t)k * m + c];
                a[(int64_t)k * m + c] = a[(int64_t)p * m + c];
                a[(int64_t)p * m + c] = t;
            }
            if (tid < 2) {
                const double t = b[tid * m + k];
                b[tid * m + k] = b[tid * m + p];
                b[tid * m + p] = t;
            }
        }
        __syncthreads();
        const double piv = a[(int64_t)k * m + k];
        for (int r = k + 1 + tid; r < m; r += nt) a[(int64_t)r * m + k] /= piv;
        __syncthreads();
        // trailing update and the fused forward elimination of both rhs
        const int rows = m - k - 1;
        for (int e = tid; e < rows * (m - k); e += nt) {
            const int r = k + 1 + e / (m - k), c = k + e % (m - k);
            const double l = a[(int64_t)r * m + k];
            if (c == k) {
                b[r] -= l * b[k];
                b[m + r] -= l * b[m + k];
            } else {
                a[(int64_t)r * m + c] -= l * a[(int64_t)k * m + c];
            }
        }
        __syncthreads();
    }
    // back substitution, column-oriented: x_i for both rhs
    for (int i = m - 1; i >= 0; --i) {
        if (tid < 2) {
            const double xi = b[tid * m + i] / a[(int64_t)i * m + i];
            b[tid * m + i] = xi;
            x[tid * m + i] = xi;
        }
        __syncthreads();
        for (int r = tid; r < i; r += nt) {
            const double arc = a[(int64_t)r * m + i];
            b[r] -= arc * b[i];
            b[m + r] -= arc * b[m + i];
        }
        __syncthreads();
    }
    // residual ||A0 x - b0|| / ||b0|| (first rhs), as the reference's gate
    double rr = 0.0, bb = 0.0;
    for (int r = tid; r < m; r += nt) {
        double acc = 0.0;
        for (int c = 0; c < m; ++c) acc = fma(a0[(int64_t)r * m + c], x[c], acc);
        const double d = acc - b0[r];
        rr += d * d;
        bb += b0[r] * b0[r];
    }
    rr = block_sum(rr, sv);
    bb = block_sum(bb, sv);
    if (tid == 0) {
        const double res = sqrt(rr) / fmax(sqrt(bb), 1e-300);
        resid[s] = res;
        info[s] = (sing || !(res <= tol)) ? 1 : 0;
    }
}

template <int PHI>
cudaError_t launch_large_t(bw_ctx* ctx, const DevScene& S, const bw_patch* patches, int64_t n_bp,
                           const double* gam, int n_nodes, int bands, int az, int np, int depth,
                           int kind, const double* gl, double* A, double* b, double* cen) {
    const int m = az * (2 * bands - 1), nv = 1 + bands * az;
    const size_t dyn = sizeof(double) * ((size_t)3 * nv + 9 * (size_t)m + 3 * (size_t)np * np) +
                       sizeof(int) * 3 * (size_t)m;
    auto kern = assemble_large_kernel<PHI>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return e;
    const int rows_per_block = 32;
    const dim3 grid((unsigned)((m + rows_per_block - 1) / rows_per_block), (unsigned)n_bp);
    ++ctx->launches;
    kern<<<grid, kLThreads, dyn, ctx->stream>>>(S, patches, gam, n_nodes, bands, az, np, depth, kind,
                                                gl, rows_per_block, A, b, cen);
    return cudaGetLastError();
}

} // namespace

size_t large_patch_smem(int bands, int az, int np) {
    const int m = az * (2 * bands - 1), nv = 1 + bands * az;
    return sizeof(double) * ((size_t)3 * nv + 9 * (size_t)m + 3 * (size_t)np * np) +
           sizeof(int) * 3 * (size_t)m;
}

cudaError_t launch_gamma_nodes(bw_ctx* ctx, const bw_patch* patches, int64_t n_bp,
                               const double* dirs, const double* wts, int n_nodes,
                               const bw_estimate* est, double* gam, int32_t* flags) {
    cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int32_t) * n_bp, ctx->stream);
    if (e != cudaSuccess) return e;
    const int64_t n = n_bp * n_nodes;
    ++ctx->launches;
    gamma_nodes_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(patches, n_bp, dirs, wts,
                                                                           n_nodes, est, gam, flags);
    return cudaGetLastError();
}

cudaError_t launch_assemble_large(bw_ctx* ctx, const DevScene& S, const bw_patch* patches,
                                  int64_t n_bp, const double* gam, int n_nodes, int bands, int az,
                                  int np, int depth, int kind, const double* gl, double* A,
                                  double* b, double* cen) {
    if (n_bp <= 0) return cudaSuccess;
#define BW_LG(P) launch_large_t<P>(ctx, S, patches, n_bp, gam, n_nodes, bands, az, np, depth, kind, \
                                   gl, A, b, cen)
    switch (S.phi_kind) {
        case BW_PHI_FEATURE_CONST: return BW_LG(BW_PHI_FEATURE_CONST);
        case BW_PHI_QUADRATIC: return BW_LG(BW_PHI_QUADRATIC);
        case BW_PHI_EXP_SIN_SIN: return BW_LG(BW_PHI_EXP_SIN_SIN);
        case BW_PHI_SIN_SIN: return BW_LG(BW_PHI_SIN_SIN);
        default: return BW_LG(BW_PHI_POINT_SOURCE);
    }
#undef BW_LG
}

cudaError_t launch_lu_large(bw_ctx* ctx, int m, int64_t n_sys, double* A, double* B,
                            const double* A0, const double* B0, double tol, double* X,
                            double* resid, int32_t* info) {
    if (n_sys <= 0) return cudaSuccess;
    ++ctx->launches;
    lu_large_kernel<<<(unsigned)n_sys, kLuThreads, 0, ctx->stream>>>(m, A, B, A0, B0, tol, X, resid,
                                                                     info);
    return cudaGetLastError();
}

} // namespace bw
