// bw_lu.cu — K2: batched dense LU with partial pivoting + multi-RHS solve +
// residual, one warp per system (sm_100a, fp64).
//
// Replaces the per-patch Eigen::PartialPivLU / solve / residual gate of
// patch_solver.cpp:314-324. The reference solves one m x m system per patch
// on the host; the DtN pipeline has one per boundary point (1e3..2e5), each
// small (m <= 64), so a warp owns one system in shared memory:
//   pivot  : warp arg-max of |a_ik| over rows i >= k, first index on ties
//            (Eigen's maxCoeff picks the first maximum)
//   swap   : lanes over columns (A) and right-hand sides (B)
//   update : lanes over rows i > k; the same sweep applies L to B, so the
//            forward substitution is fused into the factorisation
//   back   : column-oriented back substitution, lanes over rows
//   resid  : ||A x0 - b0|| / max(||b0||, 1e-300) against the original A, b
#include "bw_internal.h"

namespace bw {

namespace {

constexpr int kWarps = 4;

__global__ void __launch_bounds__(kWarps * 32)
    lu_kernel(int m, int64_t n_sys, const double* __restrict__ A, const double* __restrict__ B,
              int nrhs, double tol, double* __restrict__ X, double* __restrict__ resid,
              int32_t* __restrict__ info, unsigned long long* __restrict__ ctr) {
    extern __shared__ __align__(16) double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ld = m + 1; // padded row stride: lanes over rows hit distinct banks
    double* As = sm + (size_t)warp * (m * ld + nrhs * m);
    double* Bs = As + m * ld;
    for (int64_t s = (int64_t)blockIdx.x * kWarps + warp; s < n_sys;
         s += (int64_t)gridDim.x * kWarps) {
        const double* Ag = A + (size_t)s * m * m;
        const double* Bg = B + (size_t)s * nrhs * m;
        for (int e = lane; e < m * m; e += 32) As[(e / m) * ld + (e % m)] = Ag[e];
        for (int e = lane; e < nrhs * m; e += 32) Bs[e] = Bg[e];
        __syncwarp();
        int sing = 0;
        for (int k = 0; k < m; ++k) {
            double best = -1.0;
            int bi = m;
            for (int i = k + lane; i < m; i += 32) {
                const double v = fabs(As[i * ld + k]);
                if (v > best) { best = v; bi = i; }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, best, off);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
                if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
            }
            const int p = bi;
            if (p != k) {
                for (int j = lane; j < m; j += 32) {
                    const double t = As[k * ld + j];
                    As[k * ld + j] = As[p * ld + j];
                    As[p * ld + j] = t;
                }
                for (int r = lane; r < nrhs; r += 32) {
                    const double t = Bs[r * m + k];
                    Bs[r * m + k] = Bs[r * m + p];
                    Bs[r * m + p] = t;
                }
            }
            __syncwarp();
            if (best == 0.0) { sing = 1; continue; }
            const double piv = As[k * ld + k];
            const double* rk = As + k * ld;
            // lanes over rows i > k. The sweep over the columns of a row is
            // staged 8 columns at a time, all loads before the FMAs and the
            // stores: the compiler cannot prove that a store to row i misses
            // the pivot row, so an unstaged loop serialises load -> FMA ->
            // store per element on shared-memory latency (<= 9 systems per SM
            // leave too few warps to hide it). Same operations, same order of
            // rounding per element, as a plain loop.
            double l0 = 0.0, l1 = 0.0;
            const int i0 = k + 1 + lane, i1 = i0 + 32;
            for (int i = i0; i < m; i += 32) {
                double* ri = As + i * ld;
                const double l = ri[k] / piv;
                ri[k] = l;
                if (i == i0) l0 = l; else l1 = l;
                int j = k + 1;
                for (; j + 8 <= m; j += 8) {
                    double a[8], x[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) {
                        a[t] = rk[j + t];
                        x[t] = ri[j + t];
                    }
#pragma unroll
                    for (int t = 0; t < 8; ++t) ri[j + t] = x[t] - l * a[t];
                }
                for (; j < m; ++j) ri[j] -= l * rk[j];
            }
            const bool h0 = i0 < m, h1 = i1 < m;
            for (int r = 0; r < nrhs; ++r) {
                const double bk = Bs[r * m + k];
                if (h0) Bs[r * m + i0] -= l0 * bk;
                if (h1) Bs[r * m + i1] -= l1 * bk;
            }
            __syncwarp();
        }
        for (int j = m - 1; j >= 0; --j) {
            for (int r = 0; r < nrhs; ++r) {
                const double xj = Bs[r * m + j] / As[j * ld + j];
                __syncwarp();
                for (int i = lane; i < j; i += 32) Bs[r * m + i] -= As[i * ld + j] * xj;
                if (lane == 0) Bs[r * m + j] = xj;
                __syncwarp();
            }
        }
        double* Xg = X + (size_t)s * nrhs * m;
        for (int e = lane; e < nrhs * m; e += 32) Xg[e] = Bs[e];
        // residual of rhs 0 against the original system (patch_solver.cpp:317-318)
        double rn = 0.0, bn = 0.0;
        bool finite = true;
        for (int i = lane; i < m; i += 32) {
            double acc = 0.0;
            for (int j = 0; j < m; ++j) acc = fma(Ag[(size_t)i * m + j], Bs[j], acc);
            const double r = acc - Bg[i];
            rn += r * r;
            bn += Bg[i] * Bg[i];
        }
        for (int e = lane; e < nrhs * m; e += 32) finite = finite && isfinite(Bs[e]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            rn += __shfl_xor_sync(0xffffffffu, rn, off);
            bn += __shfl_xor_sync(0xffffffffu, bn, off);
        }
        finite = __all_sync(0xffffffffu, finite);
        if (lane == 0) {
            const double b = sqrt(bn);
            const double rr = sqrt(rn) / (b > 1e-300 ? b : 1e-300);
            resid[s] = rr;
            const int inf = sing ? 1 : ((!finite || !(rr <= tol)) ? 2 : 0);
            info[s] = inf;
            if (inf) atomicAdd(&ctr[kCtrReliability], 1ull);
        }
        __syncwarp();
    }
}

} // namespace

cudaError_t launch_lu(bw_ctx* ctx, int m, int64_t n_sys, const double* A, const double* B,
                      int nrhs, double tol, double* X, double* resid, int32_t* info) {
    cudaError_t e =
        cudaMemsetAsync(ctx->d_counters, 0, sizeof(unsigned long long) * kCtrCount, ctx->stream);
    if (e != cudaSuccess || n_sys <= 0) return e;
    const size_t smem = sizeof(double) * kWarps * ((size_t)m * (m + 1) + (size_t)nrhs * m);
    if (smem > 48 * 1024) {
        e = cudaFuncSetAttribute(lu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lu_kernel, kWarps * 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    int64_t blocks = (int64_t)ctx->sm_count * per_sm;
    const int64_t need = (n_sys + kWarps - 1) / kWarps;
    if (blocks > need) blocks = need;
    ++ctx->launches;
    lu_kernel<<<(unsigned)blocks, kWarps * 32, smem, ctx->stream>>>(m, n_sys, A, B, nrhs, tol, X,
                                                                    resid, info, ctx->d_counters);
    return cudaGetLastError();
}

} // namespace bw
