// bw_lu.cu — K2: batched dense LU with partial pivoting + multi-RHS solve +
// residual, one CTA of four warps per system (sm_100a, fp64).
//
// Replaces the per-patch Eigen::PartialPivLU / solve / residual gate of
// patch_solver.cpp:314-324. The reference solves one m x m system per patch
// on the host; the DtN pipeline has one per boundary point (1e3..2e5), each
// small (m <= 64). A system lives in shared memory as the augmented matrix
// [A | B^T] (row-major, odd row stride), so row swaps and the elimination
// carry the right-hand sides along (the forward substitution is fused into
// the factorisation). Shared memory bounds an SM at 8 systems of m = 54, so a
// system gets four warps: one warp per system (round 1) left 9 warps per SM
// and ran on shared-memory latency (issue 27 %).
//
//   panel  : right-looking LU in panels of kNB columns. Per column: warp 0
//            finds the pivot (arg-max of |a_ik| over rows i >= k, first index
//            on ties like Eigen's maxCoeff, three REDUX on the bit pattern),
//            the row swap runs over the columns, threads over rows form
//            l_i = a_ik / pivot and update the panel's remaining columns
//   U12    : thread per column right of the panel (right-hand sides included):
//            the panel's unit-lower triangle applied to its kNB rows
//   update : warps over rows, lanes over columns; the kNB multipliers of a row
//            come as two broadcast 16-byte loads, the panel's U rows sit in
//            registers: a_ij = fma(-l_it, u_tj, a_ij) for t ascending
//   back   : column-oriented back substitution, a half-warp per right-hand side
//   resid  : ||A x0 - b0|| / max(||b0||, 1e-300) against the original A, b
//
// Every element sees the same fused multiply-adds in the same (pivot-ascending)
// order as the unblocked elimination, so the factors, solutions and residuals
// are bitwise those of the round-1 kernel.
#include "bw_internal.h"

namespace bw {

namespace {

constexpr int kThreads = 128;
constexpr int kNB = 4;

__device__ __forceinline__ int lu_ld(int m, int nrhs) { return (m + nrhs) | 1; }

__global__ void __launch_bounds__(kThreads, 8)
    lu_kernel(int m, int64_t n_sys, const double* __restrict__ A, const double* __restrict__ B,
              int nrhs, double tol, double* __restrict__ X, double* __restrict__ resid,
              int32_t* __restrict__ info, unsigned long long* __restrict__ ctr) {
    extern __shared__ __align__(16) double sm[];
    __shared__ int piv_sh[2]; // pivot row, 1 when the column is exactly zero
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int W = m + nrhs, ld = lu_ld(m, nrhs);
    constexpr int kWarps = kThreads / 32;
    double* const As = sm;                                        // m x ld
    double* const Lp = sm + (((size_t)m * ld + 1) & ~(size_t)1);  // m x kNB, 16-byte aligned
    const bool col0 = lane < m, col1 = lane + 32 < m; // the lane's columns of a row of A
    for (int64_t s = blockIdx.x; s < n_sys; s += gridDim.x) {
        const double* Ag = A + (size_t)s * m * m;
        const double* Bg = B + (size_t)s * nrhs * m;
        {
            const double* g = Ag + warp * m + lane;
            double* a = As + warp * ld + lane;
            for (int r = warp; r < m; r += kWarps, g += kWarps * m, a += kWarps * ld) {
                if (col0) a[0] = g[0];
                if (col1) a[32] = g[32];
            }
        }
        for (int r = 0; r < nrhs; ++r)
            for (int i = tid; i < m; i += kThreads) As[i * ld + m + r] = Bg[r * m + i];
        __syncthreads();
        int sing = 0;
        for (int k0 = 0; k0 < m; k0 += kNB) {
            const int nb = min(kNB, m - k0);
            for (int k = k0; k < k0 + nb; ++k) {
                double* const rk = As + k * ld; // pivot row (after the swap)
                if (warp == 0) {
                    // arg-max of |a_ik| over i >= k on the bit pattern (monotonic
                    // for non-negative doubles), first index on ties
                    const int i0 = k + lane, i1 = i0 + 32;
                    const double* ck = rk + lane * ld + k;
                    unsigned long long b0 = 0ull, b1 = 0ull;
                    if (i0 < m) b0 = (unsigned long long)__double_as_longlong(fabs(ck[0]));
                    if (i1 < m) b1 = (unsigned long long)__double_as_longlong(fabs(ck[32 * ld]));
                    const bool second = b1 > b0;
                    const unsigned long long bb = second ? b1 : b0;
                    const int bi = i0 < m ? (second ? i1 : i0) : 0x7fffffff;
                    const unsigned hi = (unsigned)(bb >> 32), lo = (unsigned)bb;
                    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
                    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
                    const bool cand = hi == mh && lo == ml;
                    const int p = (int)__reduce_min_sync(0xffffffffu, cand ? (unsigned)bi : 0x7fffffffu);
                    if (lane == 0) {
                        piv_sh[0] = p;
                        piv_sh[1] = (mh | ml) == 0u;
                    }
                }
                __syncthreads();
                const int p = piv_sh[0];
                const bool zero = piv_sh[1] != 0;
                if (p != k) {
                    if (tid < W) {
                        double* rp = As + p * ld;
                        const double t = rk[tid];
                        rk[tid] = rp[tid];
                        rp[tid] = t;
                    }
                    __syncthreads();
                }
                if (zero) { // singular column: no elimination step (info = 1)
                    sing = 1;
                    __syncthreads(); // piv_sh is rewritten by the next column
                    continue;
                }
                if (k + 1 + tid < m) {
                    const double piv = rk[k];
                    double* ri = rk + (1 + tid) * ld;
                    const double l = ri[k] / piv;
                    ri[k] = l;
                    for (int c = k + 1; c < k0 + nb; ++c) ri[c] = fma(-l, rk[c], ri[c]);
                }
                __syncthreads();
            }
            const int c0 = k0 + nb; // first row and column right of / below the panel
            double* const P = As + k0 * ld; // the panel's first row
            // U12: the panel's unit-lower triangle applied to the panel rows of
            // every column to the right (thread per column; W - c0 <= 72 < 128),
            // and the panel's multipliers of the rows below copied to Lp
            if (c0 + tid < W) {
                double* pc = P + c0 + tid;
                double u[kNB];
#pragma unroll
                for (int t = 0; t < kNB; ++t) u[t] = t < nb ? pc[t * ld] : 0.0;
#pragma unroll
                for (int a = 1; a < kNB; ++a)
#pragma unroll
                    for (int b = 0; b < a; ++b)
                        if (a < nb) u[a] = fma(-P[a * ld + k0 + b], u[b], u[a]);
#pragma unroll
                for (int t = 1; t < kNB; ++t)
                    if (t < nb) pc[t * ld] = u[t];
            }
            if (c0 + tid < m) {
                const double* src = P + (nb + tid) * ld + k0;
                double* dst = Lp + (c0 + tid) * kNB;
#pragma unroll
                for (int t = 0; t < kNB; ++t) dst[t] = t < nb ? src[t] : 0.0;
            }
            __syncthreads();
            // trailing update: rows below the panel over the warps, two columns
            // per lane, the panel's U rows in registers, the row's multipliers
            // as two broadcast 16-byte loads
            const int ncol = W - c0;
            if (c0 < m) {
                for (int cb = 0; cb + lane < ncol; cb += 64) {
                    const bool v1 = cb + 32 + lane < ncol;
                    const double* pu = P + c0 + cb + lane;
                    double u[kNB], w[kNB];
#pragma unroll
                    for (int t = 0; t < kNB; ++t) {
                        u[t] = pu[t * ld];
                        w[t] = v1 ? pu[t * ld + 32] : 0.0;
                    }
                    double* pa = P + (nb + warp) * ld + c0 + cb + lane;
                    const double2* pl = reinterpret_cast<const double2*>(Lp + (c0 + warp) * kNB);
                    for (int i = c0 + warp; i < m; i += kWarps, pa += kWarps * ld, pl += kWarps * kNB / 2) {
                        const double2 l01 = pl[0], l23 = pl[1];
                        double a = pa[0];
                        a = fma(-l01.x, u[0], a);
                        a = fma(-l01.y, u[1], a);
                        a = fma(-l23.x, u[2], a);
                        a = fma(-l23.y, u[3], a);
                        pa[0] = a;
                        if (v1) {
                            double a1 = pa[32];
                            a1 = fma(-l01.x, w[0], a1);
                            a1 = fma(-l01.y, w[1], a1);
                            a1 = fma(-l23.x, w[2], a1);
                            a1 = fma(-l23.y, w[3], a1);
                            pa[32] = a1;
                        }
                    }
                }
            }
            __syncthreads();
        }
        // back substitution: a half-warp per right-hand side, lanes over rows
        {
            const int r = tid >> 4, q = tid & 15;
            const unsigned hmask = 0xffffu << (lane & 16);
            if (r < nrhs) {
                double* bj = As + (m - 1) * ld + m + r; // b_j
                const double* dj = As + (m - 1) * ld + (m - 1); // a_jj
                for (int j = m - 1; j >= 0; --j, bj -= ld, dj -= ld + 1) {
                    const double xj = bj[0] / dj[0];
                    __syncwarp(hmask);
                    const double* aij = As + q * ld + j;
                    double* bi = As + q * ld + m + r;
                    for (int i = q; i < j; i += 16, aij += 16 * ld, bi += 16 * ld)
                        bi[0] = fma(-aij[0], xj, bi[0]);
                    if (q == 0) bj[0] = xj;
                    __syncwarp(hmask);
                }
            }
        }
        __syncthreads();
        double* Xg = X + (size_t)s * nrhs * m;
        bool finite = true;
        for (int r = 0; r < nrhs; ++r)
            for (int i = tid; i < m; i += kThreads) {
                const double x = As[i * ld + m + r];
                Xg[r * m + i] = x;
                finite = finite && isfinite(x);
                if (r == 0) Lp[i] = x; // x of rhs 0 for the residual
            }
        finite = __syncthreads_and(finite);
        // residual of rhs 0 against the original system (patch_solver.cpp:317-318):
        // A again from global memory (coalesced), then lanes over rows
        {
            const double* g = Ag + warp * m + lane;
            double* a = As + warp * ld + lane;
            for (int r = warp; r < m; r += kWarps, g += kWarps * m, a += kWarps * ld) {
                if (col0) a[0] = g[0];
                if (col1) a[32] = g[32];
            }
        }
        __syncthreads();
        if (warp == 0) {
            double rn = 0.0, bn = 0.0;
            for (int i = lane; i < m; i += 32) {
                const double* ai = As + i * ld;
                double acc = 0.0;
                for (int j = 0; j < m; ++j) acc = fma(ai[j], Lp[j], acc);
                const double bi = Bg[i];
                const double r = acc - bi;
                rn += r * r;
                bn += bi * bi;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                rn += __shfl_xor_sync(0xffffffffu, rn, off);
                bn += __shfl_xor_sync(0xffffffffu, bn, off);
            }
            if (lane == 0) {
                const double b = sqrt(bn);
                const double rr = sqrt(rn) / (b > 1e-300 ? b : 1e-300);
                resid[s] = rr;
                const int inf = sing ? 1 : ((!finite || !(rr <= tol)) ? 2 : 0);
                info[s] = inf;
                if (inf) atomicAdd(&ctr[kCtrReliability], 1ull);
            }
        }
        __syncthreads();
    }
}

} // namespace

cudaError_t launch_lu(bw_ctx* ctx, int m, int64_t n_sys, const double* A, const double* B,
                      int nrhs, double tol, double* X, double* resid, int32_t* info) {
    cudaError_t e =
        cudaMemsetAsync(ctx->d_counters, 0, sizeof(unsigned long long) * kCtrCount, ctx->stream);
    if (e != cudaSuccess || n_sys <= 0) return e;
    const int ld = (m + nrhs) | 1;
    const size_t smem = sizeof(double) * ((((size_t)m * ld + 1) & ~(size_t)1) + (size_t)m * kNB);
    if (smem > 48 * 1024) {
        e = cudaFuncSetAttribute(lu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lu_kernel, kThreads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    int64_t blocks = (int64_t)ctx->sm_count * per_sm;
    if (blocks > n_sys) blocks = n_sys;
    ++ctx->launches;
    lu_kernel<<<(unsigned)blocks, kThreads, smem, ctx->stream>>>(m, n_sys, A, B, nrhs, tol, X,
                                                                 resid, info, ctx->d_counters);
    return cudaGetLastError();
}

} // namespace bw
