// bw_potential.cu — K3: integral-representation potential sum (sm_100a, fp64).
//
// Replaces biewos::evaluate (field_eval.cpp:7-19):
//   u(x) = sum_j area_j [ (n_j . r) / (4 pi d^3) u_j - dudn_j / (4 pi d) ],  r = x - p_j
// for many targets at once. Panels are tiled through shared memory as SoA with
// the 1/(4 pi) and area folded into two weights (w_u = area u / 4pi,
// w_n = area dudn / 4pi), so a pair costs: 3 sub, 3 fma (d^2), rsqrt,
// 2 mul, 3 fma (n.r), 2 fma (accumulate). Each thread owns kT targets and
// reuses every broadcast panel load kT times. Panel ranges are split over
// gridDim.y so small target counts still fill 148 SMs; the partial sums are
// reduced in fixed order by a second kernel (deterministic).
// Near-field targets (d^2 < area for some panel; the reference throws
// NearFieldError, field_eval.cpp:12-13) are flagged and get NaN.
#include "bw_internal.h"

namespace bw {

namespace {

constexpr int kThreads = 256;
constexpr int kT = 4;        // targets per thread
constexpr int kTile = 256;   // panels per shared-memory tile
constexpr double kInv4Pi = 0.079577471545947667884441881686257181; // 1/(4 pi)

__global__ void __launch_bounds__(kThreads)
    potential_kernel(const double* __restrict__ panels, int64_t n_panels, int64_t chunk,
                     const double* __restrict__ targets, int64_t n_t,
                     double* __restrict__ partial, uint8_t* __restrict__ near_part) {
    __shared__ double sp[8][kTile]; // px py pz nx ny nz wu wn
    __shared__ double sa[kTile];    // area (near-field test)
    const int64_t t0 = ((int64_t)blockIdx.x * kThreads + threadIdx.x) * kT;
    const int64_t p_begin = (int64_t)blockIdx.y * chunk;
    int64_t p_end = p_begin + chunk;
    if (p_end > n_panels) p_end = n_panels;

    double tx[kT], ty[kT], tz[kT], acc[kT];
    bool nf[kT];
#pragma unroll
    for (int q = 0; q < kT; ++q) {
        const int64_t t = t0 + q;
        const bool ok = t < n_t;
        tx[q] = ok ? targets[3 * t] : 0.0;
        ty[q] = ok ? targets[3 * t + 1] : 0.0;
        tz[q] = ok ? targets[3 * t + 2] : 0.0;
        acc[q] = 0.0;
        nf[q] = false;
    }
    for (int64_t base = p_begin; base < p_end; base += kTile) {
        const int nt = (int)((p_end - base) < kTile ? (p_end - base) : kTile);
        __syncthreads();
        for (int i = threadIdx.x; i < nt; i += kThreads) {
            const double* P = panels + 9 * (base + i);
            sp[0][i] = P[0];
            sp[1][i] = P[1];
            sp[2][i] = P[2];
            sp[3][i] = P[3];
            sp[4][i] = P[4];
            sp[5][i] = P[5];
            sp[6][i] = P[6] * P[7] * kInv4Pi;
            sp[7][i] = P[6] * P[8] * kInv4Pi;
            sa[i] = P[6];
        }
        __syncthreads();
#pragma unroll 2
        for (int i = 0; i < nt; ++i) {
            const double px = sp[0][i], py = sp[1][i], pz = sp[2][i];
            const double nx = sp[3][i], ny = sp[4][i], nz = sp[5][i];
            const double wu = sp[6][i], wn = sp[7][i], area = sa[i];
#pragma unroll
            for (int q = 0; q < kT; ++q) {
                const double rx = tx[q] - px, ry = ty[q] - py, rz = tz[q] - pz;
                const double d2 = fma(rx, rx, fma(ry, ry, rz * rz));
                nf[q] |= d2 < area;
                const double ri = rsqrt(d2);
                const double nr = fma(nx, rx, fma(ny, ry, nz * rz));
                acc[q] = fma(wu * nr, ri * ri * ri, acc[q]);
                acc[q] = fma(-wn, ri, acc[q]);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < kT; ++q) {
        const int64_t t = t0 + q;
        if (t < n_t) {
            partial[(int64_t)blockIdx.y * n_t + t] = acc[q];
            near_part[(int64_t)blockIdx.y * n_t + t] = nf[q] ? 1 : 0;
        }
    }
}

__global__ void potential_reduce(const double* __restrict__ partial,
                                 const uint8_t* __restrict__ near_part, int splits, int64_t n_t,
                                 double* __restrict__ u, uint8_t* __restrict__ near,
                                 unsigned long long* __restrict__ ctr) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_t) return;
    double s = 0.0;
    uint8_t f = 0;
    for (int k = 0; k < splits; ++k) {
        s += partial[(int64_t)k * n_t + t];
        f |= near_part[(int64_t)k * n_t + t];
    }
    u[t] = f ? __longlong_as_double(0x7ff8000000000000LL) : s;
    if (near) near[t] = f;
    if (f) atomicAdd(&ctr[kCtrNear], 1ull);
}

} // namespace

cudaError_t launch_potential(bw_ctx* ctx, const double* panels, int64_t n_panels,
                             const double* targets, int64_t n_t, double* u, uint8_t* near,
                             int64_t* near_count) {
    (void)near_count;
    cudaError_t e =
        cudaMemsetAsync(ctx->d_counters, 0, sizeof(unsigned long long) * kCtrCount, ctx->stream);
    if (e != cudaSuccess || n_t <= 0) return e;
    const int64_t per_block = (int64_t)kThreads * kT;
    const int64_t bx = (n_t + per_block - 1) / per_block;
    // enough blocks for ~4 waves of 148 SMs, panel chunks a multiple of the tile
    int64_t splits = (4 * (int64_t)ctx->sm_count + bx - 1) / bx;
    const int64_t max_splits = (n_panels + kTile - 1) / kTile;
    if (splits > max_splits) splits = max_splits;
    if (splits < 1) splits = 1;
    if (splits > 65535) splits = 65535;
    int64_t chunk = (n_panels + splits - 1) / splits;
    chunk = ((chunk + kTile - 1) / kTile) * kTile;
    splits = chunk > 0 ? (n_panels + chunk - 1) / chunk : 1;
    if (splits < 1) splits = 1;
    bw_status st = BW_OK;
    double* partial = (double*)scratch(ctx, kSlotTmp0, sizeof(double) * splits * n_t, &st);
    uint8_t* np = (uint8_t*)scratch(ctx, kSlotTmp1, (size_t)splits * n_t, &st);
    if (st != BW_OK) return cudaErrorMemoryAllocation;
    dim3 grid((unsigned)bx, (unsigned)splits);
    ++ctx->launches;
    potential_kernel<<<grid, kThreads, 0, ctx->stream>>>(panels, n_panels, chunk, targets, n_t,
                                                         partial, np);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ++ctx->launches;
    potential_reduce<<<(unsigned)((n_t + 255) / 256), 256, 0, ctx->stream>>>(
        partial, np, (int)splits, n_t, u, near, ctx->d_counters);
    return cudaGetLastError();
}

} // namespace bw
