// bw_potential.cu — K3: integral-representation potential sum (sm_100a, fp64).
//
// Replaces biewos::evaluate (field_eval.cpp:7-19):
//   u(x) = sum_j area_j [ (n_j . r) / (4 pi d^3) u_j - dudn_j / (4 pi d) ],  r = x - p_j
// for many targets at once. The panel set streams through shared memory in
// tiles: a tile of the caller's AoS records (72 B each, contiguous) is copied
// with coalesced 16-byte loads, then folded once per panel into 8 doubles,
// p, w_u n and w_n (w_u = area u / 4 pi, w_n = area dudn / 4 pi) plus the area
// for the near-field test, stored as two double4 per panel so the inner loop
// reads a panel with four broadcast LDS.128. Per pair:
//   r = x - p (3), d^2 (3), 1/d by MUFU.RSQ64H + one cubic Newton step (5,
//   relative error ~2^-60), (w_u n).r (3), acc += (1/d)((w_u n.r)/d^2 - w_n) (3)
// = 17 fp64 instructions. Each thread owns kT targets and reuses every panel
// kT times. Panel ranges are split over gridDim.y so small target counts still
// fill 148 SMs; the partial sums are reduced in fixed order by a second kernel
// (deterministic). Near-field targets (d^2 < area for some panel; the
// reference throws NearFieldError, field_eval.cpp:12-13) are flagged and NaN.
#include "bw_internal.h"

namespace bw {

namespace {

constexpr int kThreads = 128;
constexpr int kT = 8;        // targets per thread
constexpr int kTile = 256;   // panels per shared-memory tile
constexpr double kInv4Pi = 0.079577471545947667884441881686257181; // 1/(4 pi)

// 1/sqrt(a) for a > 0: rsqrt.approx + one cubic Newton step (as sqrt_fast)
__device__ __forceinline__ double rsqrt_nr(double a) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    const double e = fma(a, -(y * y), 1.0);
    return fma(fma(e, 0.375, 0.5), y * e, y);
}

__global__ void __launch_bounds__(kThreads)
    potential_kernel(const double* __restrict__ panels, int64_t n_panels, int64_t chunk,
                     const double* __restrict__ targets, int64_t n_t,
                     double* __restrict__ partial, uint8_t* __restrict__ near_part) {
    __shared__ __align__(16) double raw[9 * kTile];   // the tile's records as given
    __shared__ double4 sp[2 * kTile];                 // {p, w_n}, {w_u n, area}
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
        // coalesced copy of 9 nt contiguous doubles (16-byte loads when aligned)
        const double* src = panels + 9 * base;
        const int ne = 9 * nt;
        if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            const double2* s2 = reinterpret_cast<const double2*>(src);
            double2* r2 = reinterpret_cast<double2*>(raw);
            for (int i = threadIdx.x; i < ne / 2; i += kThreads) r2[i] = s2[i];
            if ((ne & 1) && threadIdx.x == 0) raw[ne - 1] = src[ne - 1];
        } else {
            for (int i = threadIdx.x; i < ne; i += kThreads) raw[i] = src[i];
        }
        __syncthreads();
        for (int i = threadIdx.x; i < nt; i += kThreads) {
            const double* P = raw + 9 * i;
            const double wu = P[6] * P[7] * kInv4Pi;
            const double wn = P[6] * P[8] * kInv4Pi;
            sp[2 * i] = make_double4(P[0], P[1], P[2], wn);
            sp[2 * i + 1] = make_double4(wu * P[3], wu * P[4], wu * P[5], P[6]);
        }
        __syncthreads();
#pragma unroll 2
        for (int i = 0; i < nt; ++i) {
            const double4 a = sp[2 * i], b = sp[2 * i + 1];
#pragma unroll
            for (int q = 0; q < kT; ++q) {
                const double rx = tx[q] - a.x, ry = ty[q] - a.y, rz = tz[q] - a.z;
                const double d2 = fma(rx, rx, fma(ry, ry, rz * rz));
                nf[q] |= d2 < b.w;
                const double ri = rsqrt_nr(d2);
                const double wnr = fma(b.x, rx, fma(b.y, ry, b.z * rz)); // w_u (n . r)
                acc[q] = fma(ri, fma(wnr, ri * ri, -a.w), acc[q]);
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
