// bw_point.cu — K6: the flat-boundary point formula of the reference,
//   du/dn(x) = Sigma1' + Sigma2'          (point_solver.hpp:8-38, along -axis)
// for many boundary points at once, one warp per point:
//   Sigma1' = -sum_i w_i h(y_i) (u_i - phi(x)),  h = 3 cos(theta) / (2 pi a^3)
//             over the WOS node estimates u_i at the cap-rule nodes
//             (sigma1_prime, point_solver.cpp:143-174; h_kernel, greens.cpp:155-163)
//   Sigma2' = -(1/2pi) sum_k w_k (1/rho^3 - 1/a^3) (phi(y_k) - phi(x))
//             on the ring rule over delta <= rho <= a (sigma2_prime,
//             point_solver.cpp:119-141; ring_rule, quadrature.cpp:55-71)
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

template <int PHI>
__global__ void point_kernel(const DevScene S, const bw_patch* __restrict__ patches, int64_t n_bp,
                             const double* __restrict__ cap_dirs,
                             const double* __restrict__ cap_w, int n_cap,
                             const bw_estimate* __restrict__ est, const double* __restrict__ ring,
                             int n_ring, double* __restrict__ total, double* __restrict__ s1_out,
                             double* __restrict__ s2_out, double* __restrict__ se_out) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t bp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); bp < n_bp;
         bp += warps) {
        const bw_patch P = patches[bp];
        const double a = P.a;
        const double phix = eval_phi<PHI>(S, P.o[0], P.o[1], P.o[2], 0);
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
        // Sigma2': ring rule in the plane through o normal to axis; the table
        // holds {rho/a, cos psi, sin psi, w/a^2} (host libm, as the reference)
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
        const double phix_rn = phi_rn<PHI>(S, P.o[0], P.o[1], P.o[2]);
        double v2 = 0.0;
        const double a3 = __dmul_rn(__dmul_rn(a, a), a);
        for (int k = lane; k < n_ring; k += 32) {
            const double rho = __dmul_rn(ring[4 * k], a), cp = ring[4 * k + 1],
                         sp = ring[4 * k + 2], w = __dmul_rn(__dmul_rn(ring[4 * k + 3], a), a);
            // y = c + rho (cos psi e1 + sin psi e2)   (point_solver.cpp:133)
            const double x = __dadd_rn(P.o[0], __dmul_rn(rho, __dadd_rn(__dmul_rn(cp, e10), __dmul_rn(sp, e20))));
            const double y = __dadd_rn(P.o[1], __dmul_rn(rho, __dadd_rn(__dmul_rn(cp, e11), __dmul_rn(sp, e21))));
            const double z = __dadd_rn(P.o[2], __dmul_rn(rho, __dadd_rn(__dmul_rn(cp, e12), __dmul_rn(sp, e22))));
            const double phiy = phi_rn<PHI>(S, x, y, z);
            const double r3 = __dmul_rn(__dmul_rn(rho, rho), rho);
            const double kern = __dsub_rn(__ddiv_rn(1.0, r3), __ddiv_rn(1.0, a3));
            v2 = __dadd_rn(v2, __dmul_rn(__dmul_rn(w, kern), __dsub_rn(phiy, phix_rn)));
        }
        v1 = warp_sum(v1);
        var = warp_sum(var);
        v2 = warp_sum(v2);
        if (lane == 0) {
            const double s2 = -v2 / (2.0 * kPi);
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
                           const bw_estimate* est, const double* ring, int n_ring, double* total,
                           double* s1, double* s2, double* se) {
    const int threads = 128;
    int64_t blocks = (n_bp + 3) / 4;
    if (blocks > (int64_t)ctx->sm_count * 16) blocks = (int64_t)ctx->sm_count * 16;
    ++ctx->launches;
    point_kernel<PHI><<<(unsigned)blocks, threads, 0, ctx->stream>>>(
        S, patches, n_bp, cap_dirs, cap_w, n_cap, est, ring, n_ring, total, s1, s2, se);
    return cudaGetLastError();
}

} // namespace

cudaError_t launch_point_formula(bw_ctx* ctx, const DevScene& S, const bw_patch* patches,
                                 int64_t n_bp, const double* cap_dirs, const double* cap_w,
                                 int n_cap, const bw_estimate* est, const double* ring,
                                 int n_ring, double* total, double* s1, double* s2, double* se) {
    if (n_bp <= 0) return cudaSuccess;
#define BW_PT(P) launch_point_t<P>(ctx, S, patches, n_bp, cap_dirs, cap_w, n_cap, est, ring, n_ring, \
                                   total, s1, s2, se)
    switch (S.phi_kind) {
        case BW_PHI_FEATURE_CONST: return BW_PT(BW_PHI_FEATURE_CONST);
        case BW_PHI_QUADRATIC: return BW_PT(BW_PHI_QUADRATIC);
        case BW_PHI_EXP_SIN_SIN: return BW_PT(BW_PHI_EXP_SIN_SIN);
        default: return BW_PT(BW_PHI_POINT_SOURCE);
    }
#undef BW_PT
}

} // namespace bw
