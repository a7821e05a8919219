// bw_point.cu — K6: the flat-boundary point formula of the reference,
//   du/dn(x) = Sigma1' + Sigma2'          (point_solver.hpp:8-38, along -axis)
// for many boundary points at once, one warp per point:
//   Sigma1' = -sum_i w_i h(y_i) (u_i - phi(x)),  h = 3 cos(theta) / (2 pi a^3)
//             over the WOS node estimates u_i at the cap-rule nodes
//             (sigma1_prime, point_solver.cpp:143-174; h_kernel, greens.cpp:155-163)
//   Sigma2' = -(1/2pi) sum_k w_k (1/rho^3 - 1/a^3) (phi(y_k) - phi(x))
//             on the ring rule over delta <= rho <= a (sigma2_prime,
//             point_solver.cpp:119-141; ring_rule, quadrature.cpp:55-71)
// Piecewise-constant plate data take the reference's exact finite-part path
// instead (sigma2_plates_exact, point_solver.cpp:43-114). The reference's
// checks raise per point: GeometryError (axis / centre, :14-22),
// ClassificationError (x or a ring node off every feature, geometry.cpp:211),
// DomainError (disk S_a not covered, :112, :124), SingularityError (data jump
// at x, :104) — counted in ctx->d_counters and returned by bw_point_formula.
// Lane-strided partial sums + fixed shuffle tree (deterministic).
#include <cmath>

#include "bw_internal.h"

namespace bw {

namespace {

constexpr double kPi = 3.14159265358979323846;

// Dirichlet data evaluated without FMA contraction, in the reference's
// operation order: Sigma2' sums (1/rho^3 - 1/a^3)(phi(y) - phi(x)) with
// cancellation ~1/delta, so ulp-level differences matter at the 1e-9 level of
// the reference's frozen values.
template <int PHI>
__device__ __forceinline__ double phi_rn(const DevScene& S, double x, double y, double z) {
    const double* c = S.phi;
    if (PHI == BW_PHI_FEATURE_CONST) return S.fpot[0];
    if (PHI == BW_PHI_QUADRATIC) {
        double v = __dadd_rn(c[0], __dmul_rn(c[1], x));
        v = __dadd_rn(v, __dmul_rn(c[2], y));
        v = __dadd_rn(v, __dmul_rn(c[3], z));
        v = __dadd_rn(v, __dmul_rn(__dmul_rn(c[4], x), x));
        v = __dadd_rn(v, __dmul_rn(__dmul_rn(c[5], y), y));
        v = __dadd_rn(v, __dmul_rn(__dmul_rn(c[6], z), z));
        v = __dadd_rn(v, __dmul_rn(__dmul_rn(c[7], x), y));
        v = __dadd_rn(v, __dmul_rn(__dmul_rn(c[8], x), z));
        return __dadd_rn(v, __dmul_rn(__dmul_rn(c[9], y), z));
    }
    if (PHI == BW_PHI_POINT_SOURCE) {
        const double dx = __dsub_rn(x, c[1]), dy = __dsub_rn(y, c[2]), dz = __dsub_rn(z, c[3]);
        const double n = __dsqrt_rn(
            __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
        return __dadd_rn(c[4], __ddiv_rn(c[0], n));
    }
    return eval_phi<PHI>(S, x, y, z, 0);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    return v;
}

// Scene::scale (geometry.cpp:101-113)
__device__ double scene_scale(const DevScene& S) {
    if (S.kind == BW_SCENE_THINDISK) return S.disk_r;
    if (S.kind == BW_SCENE_SPHERE) return S.R;
    if (S.kind == BW_SCENE_PLATESET) {
        double m = 0.0;
        for (int i = 0; i < S.n_cav; ++i) {
            const double4 pl = S.cav[i];
            m = fmax(m, fmax(fmax(fabs(pl.x), fabs(pl.y)), fmax(fabs(pl.z), fabs(pl.w))));
        }
        return m;
    }
    if (S.kind == BW_SCENE_BOX || S.kind == BW_SCENE_BOX_CAVITIES) { // box faces (extension)
        double m = 0.0;
        for (int k = 0; k < 3; ++k) m = fmax(m, fmax(fabs(S.lo[k]), fabs(S.hi[k])));
        return m;
    }
    return 1.0;
}

// eval_dirichlet's feature search (geometry.cpp:198-216) on the flat scenes:
// nearest feature (lowest index on ties), its distance and the projection.
__device__ int flat_feature(const DevScene& S, double x, double y, double z, double& dist,
                            double& px, double& py, double& pz) {
    int best = -1;
    dist = __longlong_as_double(0x7ff0000000000000LL);
    const int nf = feature_count<-1>(S);
    for (int f = 0; f < nf; ++f) {
        double qx, qy, qz;
        project<-1>(S, S.cav, x, y, z, f, qx, qy, qz);
        const double d = norm3(x - qx, y - qy, z - qz);
        if (d < dist) {
            dist = d;
            best = f;
            px = qx; py = qy; pz = qz;
        }
    }
    return best;
}

// clip_ray (point_solver.cpp:24-41): [t0, t1] of x + t (dx, dy) inside the plate
__device__ __forceinline__ bool clip_ray(double4 pl, double x, double y, double dx, double dy,
                                         double& t0, double& t1) {
    t0 = 0.0;
    t1 = __longlong_as_double(0x7ff0000000000000LL);
    const double ps[2] = {x, y}, ds[2] = {dx, dy};
    const double lo[2] = {pl.x, pl.z}, hi[2] = {pl.y, pl.w};
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        if (fabs(ds[i]) < 1e-15) {
            if (ps[i] < lo[i] || ps[i] > hi[i]) return false;
        } else {
            double ta = (lo[i] - ps[i]) / ds[i];
            double tb = (hi[i] - ps[i]) / ds[i];
            if (ta > tb) { const double t = ta; ta = tb; tb = t; }
            t0 = fmax(t0, ta);
            t1 = fmin(t1, tb);
        }
    }
    return t1 > t0;
}

// sigma2_plates_exact (point_solver.cpp:43-114) for piecewise-constant plate
// data, one warp: lane 0 builds and sorts the angular breakpoints in shared
// memory, the lanes share the (segment, Gauss node) pairs.
__device__ double sigma2_plates_exact(const DevScene& S, double cx, double cy, double a,
                                      double phix, const double* gl20, double* cuts, int* ncut,
                                      int lane, unsigned long long* ctr) {
    const double two_pi = 2.0 * kPi;
    if (lane == 0) {
        int n = 0;
        auto add = [&](double ang) {
            ang = fmod(ang, two_pi);
            if (ang < 0) ang += two_pi;
            cuts[n++] = ang;
        };
        cuts[n++] = 0.0;
        cuts[n++] = two_pi;
        for (int k = 0; k < S.n_cav; ++k) {
            const double4 pl = S.cav[k];
            const double xs[2] = {pl.x, pl.y}, ys[2] = {pl.z, pl.w};
            for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 2; ++j) add(atan2(ys[j] - cy, xs[i] - cx));
            for (int i = 0; i < 2; ++i) {
                const double u = (xs[i] - cx) / a;
                if (fabs(u) <= 1.0) {
                    add(acos(u));
                    add(-acos(u));
                }
            }
            for (int j = 0; j < 2; ++j) {
                const double u = (ys[j] - cy) / a;
                if (fabs(u) <= 1.0) {
                    add(asin(u));
                    add(kPi - asin(u));
                }
            }
        }
        for (int k = 0; k < 4; ++k) cuts[n++] = k * kPi / 2.0;
        for (int i = 1; i < n; ++i) { // insertion sort (std::sort order)
            const double v = cuts[i];
            int j = i - 1;
            while (j >= 0 && cuts[j] > v) {
                cuts[j + 1] = cuts[j];
                --j;
            }
            cuts[j + 1] = v;
        }
        int m = 1; // std::unique with |u - v| < 1e-13 against the last kept cut
        for (int i = 1; i < n; ++i)
            if (!(fabs(cuts[m - 1] - cuts[i]) < 1e-13)) cuts[m++] = cuts[i];
        *ncut = m;
    }
    __syncwarp();
    const int items = (*ncut - 1) * 20;
    double tot = 0.0, cov = 0.0;
    bool singular = false;
    for (int it = lane; it < items; it += 32) {
        const int sg = it / 20, i = it % 20;
        const double th0 = cuts[sg], th1 = cuts[sg + 1];
        if (th1 - th0 < 1e-14) continue;
        const double th = th0 + (th1 - th0) * 0.5 * (gl20[i] + 1.0);
        const double w = gl20[32 + i] * 0.5 * (th1 - th0);
        const double dx = cos(th), dy = sin(th);
        for (int k = 0; k < S.n_cav; ++k) {
            double t0, t1;
            if (!clip_ray(S.cav[k], cx, cy, dx, dy, t0, t1)) continue;
            const double r0 = fmax(t0, 0.0), r1 = fmin(t1, a);
            if (r1 <= r0) continue;
            cov += w * 0.5 * (r1 * r1 - r0 * r0);
            const double dphi = S.fpot[k] - phix;
            if (dphi == 0) continue;
            if (r0 < 1e-14) singular = true;
            const double radial = (1.0 / r0 - 1.0 / r1) - (r1 * r1 - r0 * r0) / (2.0 * a * a * a);
            tot += w * dphi * radial;
        }
    }
    tot = warp_sum(tot);
    cov = warp_sum(cov);
    if (__any_sync(0xffffffffu, singular) && lane == 0) atomicAdd(&ctr[kCtrSingular], 1ull);
    if (lane == 0 && fabs(cov - kPi * a * a) > 1e-8 * kPi * a * a) atomicAdd(&ctr[kCtrDomain], 1ull);
    __syncwarp();
    return -tot / two_pi;
}

template <int PHI>
__global__ void point_kernel(const DevScene S, const bw_patch* __restrict__ patches, int64_t n_bp,
                             const double* __restrict__ cap_dirs,
                             const double* __restrict__ cap_w, int n_cap,
                             const bw_estimate* __restrict__ est, const double* __restrict__ ring,
                             int n_ring, const double* __restrict__ gl20,
                             double* __restrict__ total, double* __restrict__ s1_out,
                             double* __restrict__ s2_out, double* __restrict__ se_out,
                             unsigned long long* __restrict__ ctr, int cut_cap) {
    extern __shared__ __align__(16) double cut_smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double* cuts = cut_smem + (size_t)wib * (cut_cap + 1);
    int* ncut = reinterpret_cast<int*>(cuts + cut_cap);
    const bool plates_exact = PHI == BW_PHI_FEATURE_CONST && S.kind == BW_SCENE_PLATESET;
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    const double scale = scene_scale(S);
    const double plane = S.kind == BW_SCENE_HALFSPACE ? S.plane_z : 0.0;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t bp = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; bp < n_bp; bp += warps) {
        const bw_patch P = patches[bp];
        const double a = P.a;
        // check_flat_frame (point_solver.cpp:14-22); on box faces (an extension
        // of the reference) the axis must be normal to the face holding o
        bool bad_frame;
        if (S.kind == BW_SCENE_BOX || S.kind == BW_SCENE_BOX_CAVITIES) {
            double dd, qx, qy, qz;
            const int ff = flat_feature(S, P.o[0], P.o[1], P.o[2], dd, qx, qy, qz);
            bad_frame = ff < 0 || ff >= 6 || fabs(fabs(P.axis[ff >> 1]) - 1.0) > 1e-12;
        } else {
            bad_frame = fabs(fabs(P.axis[2]) - 1.0) > 1e-12 ||
                        fabs(P.o[2] - plane) > 1e-9 * fmax(1.0, scale);
        }
        if (bad_frame) {
            if (lane == 0) {
                atomicAdd(&ctr[kCtrGeometry], 1ull);
                total[bp] = nan;
                if (s1_out) s1_out[bp] = nan;
                if (s2_out) s2_out[bp] = nan;
                if (se_out) se_out[bp] = nan;
            }
            continue;
        }
        // phi(x) = eval_dirichlet(scene, x) (geometry.cpp:198-220)
        double dist, px, py, pz;
        const int f = flat_feature(S, P.o[0], P.o[1], P.o[2], dist, px, py, pz);
        if (f < 0 || dist > 1e-6 * scale) {
            if (lane == 0) {
                atomicAdd(&ctr[kCtrClassify], 1ull);
                total[bp] = nan;
                if (s1_out) s1_out[bp] = nan;
                if (s2_out) s2_out[bp] = nan;
                if (se_out) se_out[bp] = nan;
            }
            continue;
        }
        const double phix = PHI == BW_PHI_FEATURE_CONST ? S.fpot[f] : eval_phi<PHI>(S, px, py, pz, 0);
        // Sigma1': cap nodes (positions as K1 generates them)
        double v1 = 0.0, var = 0.0;
        for (int i = lane; i < n_cap; i += 32) {
            double x, y, z;
            patch_node_local(P.o, P.axis, a, cap_dirs + 3 * i, x, y, z);
            const double rx = x - P.o[0], ry = y - P.o[1], rz = z - P.o[2];
            const double r = sqrt(rx * rx + ry * ry + rz * rz);
            const double ct = (P.axis[0] * rx + P.axis[1] * ry + P.axis[2] * rz) / r;
            const double h = 3.0 / (2.0 * kPi * a * a * a) * ct;
            const double coeff = cap_w[i] * (a * a) * h;
            const bw_estimate e = est[bp * n_cap + i];
            v1 -= coeff * (e.mean - phix);
            if (e.n > 0) var += coeff * coeff * e.variance / (double)e.n;
        }
        v1 = warp_sum(v1);
        var = warp_sum(var);
        double s2;
        if (plates_exact) {
            s2 = sigma2_plates_exact(S, P.o[0], P.o[1], a, phix, gl20, cuts, ncut, lane, ctr);
        } else {
            if (S.kind == BW_SCENE_THINDISK && hypot(P.o[0], P.o[1]) + a > S.disk_r + 1e-12) {
                if (lane == 0) atomicAdd(&ctr[kCtrDomain], 1ull);
            }
            // Sigma2': ring rule in the plane through o normal to axis; the
            // table holds {rho/a, cos psi, sin psi, w/a^2} (host libm, as the
            // reference)
            double e10, e11, e12, e20, e21, e22;
            {
                const double ax0 = P.axis[0], ax1 = P.axis[1], ax2 = P.axis[2];
                const bool use_x = fabs(ax0) < 0.9;
                const double r0 = use_x ? 1.0 : 0.0, r1 = use_x ? 0.0 : 1.0;
                const double c0 = __dsub_rn(__dmul_rn(ax1, 0.0), __dmul_rn(ax2, r1));
                const double c1 = __dsub_rn(__dmul_rn(ax2, r0), __dmul_rn(ax0, 0.0));
                const double c2 = __dsub_rn(__dmul_rn(ax0, r1), __dmul_rn(ax1, r0));
                const double n = __dsqrt_rn(dot3_rn(c0, c1, c2, c0, c1, c2));
                e10 = __ddiv_rn(c0, n); e11 = __ddiv_rn(c1, n); e12 = __ddiv_rn(c2, n);
                e20 = __dsub_rn(__dmul_rn(ax1, e12), __dmul_rn(ax2, e11));
                e21 = __dsub_rn(__dmul_rn(ax2, e10), __dmul_rn(ax0, e12));
                e22 = __dsub_rn(__dmul_rn(ax0, e11), __dmul_rn(ax1, e10));
            }
            const double phix_rn = PHI == BW_PHI_FEATURE_CONST ? phix : phi_rn<PHI>(S, px, py, pz);
            const double tol = 1e-6 * fmax(1.0, scale);
            double v2 = 0.0;
            bool off = false;
            const double a3 = __dmul_rn(__dmul_rn(a, a), a);
            for (int k = lane; k < n_ring; k += 32) {
                const double rho = __dmul_rn(ring[4 * k], a), cp = ring[4 * k + 1],
                             sp = ring[4 * k + 2], w = __dmul_rn(__dmul_rn(ring[4 * k + 3], a), a);
                // y = c + rho (cos psi e1 + sin psi e2)   (point_solver.cpp:133)
                const double x = __dadd_rn(P.o[0], __dmul_rn(rho, __dadd_rn(__dmul_rn(cp, e10), __dmul_rn(sp, e20))));
                const double y = __dadd_rn(P.o[1], __dmul_rn(rho, __dadd_rn(__dmul_rn(cp, e11), __dmul_rn(sp, e21))));
                const double z = __dadd_rn(P.o[2], __dmul_rn(rho, __dadd_rn(__dmul_rn(cp, e12), __dmul_rn(sp, e22))));
                // eval_dirichlet(scene, y, tol): data at the projection on the
                // nearest feature; off every feature -> ClassificationError
                double dy, qx, qy, qz;
                const int fy = flat_feature(S, x, y, z, dy, qx, qy, qz);
                if (fy < 0 || dy > tol) off = true;
                const double phiy = PHI == BW_PHI_FEATURE_CONST ? S.fpot[fy < 0 ? 0 : fy]
                                                                : phi_rn<PHI>(S, qx, qy, qz);
                const double r3 = __dmul_rn(__dmul_rn(rho, rho), rho);
                const double kern = __dsub_rn(__ddiv_rn(1.0, r3), __ddiv_rn(1.0, a3));
                v2 = __dadd_rn(v2, __dmul_rn(__dmul_rn(w, kern), __dsub_rn(phiy, phix_rn)));
            }
            if (__any_sync(0xffffffffu, off) && lane == 0) atomicAdd(&ctr[kCtrClassify], 1ull);
            v2 = warp_sum(v2);
            s2 = -v2 / (2.0 * kPi);
        }
        if (lane == 0) {
            total[bp] = v1 + s2;
            if (s1_out) s1_out[bp] = v1;
            if (s2_out) s2_out[bp] = s2;
            if (se_out) se_out[bp] = sqrt(var);
        }
    }
}

template <int PHI>
cudaError_t launch_point_t(bw_ctx* ctx, const DevScene& S, const bw_patch* patches, int64_t n_bp,
                           const double* cap_dirs, const double* cap_w, int n_cap,
                           const bw_estimate* est, const double* ring, int n_ring,
                           const double* gl20, double* total, double* s1, double* s2, double* se) {
    cudaError_t e = cudaMemsetAsync(ctx->d_counters, 0, sizeof(unsigned long long) * kCtrCount,
                                    ctx->stream);
    if (e != cudaSuccess) return e;
    // the exact plate path needs a breakpoint buffer per warp: one warp per block
    const bool exact = PHI == BW_PHI_FEATURE_CONST && S.kind == BW_SCENE_PLATESET;
    const int cut_cap = exact ? 12 * S.n_cav + 8 : 0;
    const int threads = exact ? 32 : 128;
    const size_t dyn = exact ? sizeof(double) * (size_t)(cut_cap + 1) : 0;
    if (dyn > 48 * 1024) {
        e = cudaFuncSetAttribute(point_kernel<PHI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)dyn);
        if (e != cudaSuccess) return e;
    }
    const int per_block = threads / 32;
    int64_t blocks = (n_bp + per_block - 1) / per_block;
    if (blocks > (int64_t)ctx->sm_count * 16) blocks = (int64_t)ctx->sm_count * 16;
    ++ctx->launches;
    point_kernel<PHI><<<(unsigned)blocks, threads, dyn, ctx->stream>>>(
        S, patches, n_bp, cap_dirs, cap_w, n_cap, est, ring, n_ring, gl20, total, s1, s2, se,
        ctx->d_counters, cut_cap);
    return cudaGetLastError();
}

} // namespace

cudaError_t launch_point_formula(bw_ctx* ctx, const DevScene& S, const bw_patch* patches,
                                 int64_t n_bp, const double* cap_dirs, const double* cap_w,
                                 int n_cap, const bw_estimate* est, const double* ring,
                                 int n_ring, const double* gl20, double* total, double* s1,
                                 double* s2, double* se) {
    if (n_bp <= 0) return cudaSuccess;
#define BW_PT(P) launch_point_t<P>(ctx, S, patches, n_bp, cap_dirs, cap_w, n_cap, est, ring, n_ring, \
                                   gl20, total, s1, s2, se)
    switch (S.phi_kind) {
        case BW_PHI_FEATURE_CONST: return BW_PT(BW_PHI_FEATURE_CONST);
        case BW_PHI_QUADRATIC: return BW_PT(BW_PHI_QUADRATIC);
        case BW_PHI_EXP_SIN_SIN: return BW_PT(BW_PHI_EXP_SIN_SIN);
        case BW_PHI_SIN_SIN: return BW_PT(BW_PHI_SIN_SIN);
        default: return BW_PT(BW_PHI_POINT_SOURCE);
    }
#undef BW_PT
}

} // namespace bw
