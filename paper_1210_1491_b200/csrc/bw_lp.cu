// bw_lp.cu — the last-passage estimator of the reference (next-row f3,
// last_passage.cpp:47-121) on the device:
//   path k: stream (seed, point 0, path k, domain 1); start on the cap with
//   theta = asin(sqrt(U1)), phi = 2 pi U2 (sample_start_point, :47-51), then
//   the WOS walk continues on the same stream (:77-79); value phi(x) for
//   paths lost to infinity, phi(x) - exit value otherwise; per-feature counts.
// K_lp_walk runs one path per thread and stores each path's value and
// outcome; K_lp_reduce then reproduces the reference's statistics exactly:
// Welford over 4096-path chunks in path order, Chan merge in chunk order
// (:15-43, :68-97).
#include <cmath>

#include <algorithm>

#include "bw_internal.h"

namespace bw {

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr int kChunk = 4096;

template <int KIND>
__device__ __forceinline__ double lp_nearest(const DevScene& S, const double4* cav, double x,
                                             double y, double z) {
    if (KIND == BW_SCENE_HALFSPACE) return fabs(z - S.plane_z);
    if (KIND == BW_SCENE_SPHERE) return fabs(norm3(x, y, z) - S.R);
    if (KIND == BW_SCENE_THINDISK) {
        const double rho = hypot(x, y);
        return rho <= S.disk_r ? fabs(z) : hypot(rho - S.disk_r, z);
    }
    double best = __longlong_as_double(0x7ff0000000000000LL);
    for (int i = 0; i < S.n_cav; ++i) { // PLATESET
        const double4 pl = cav[i];
        const double dx = fmax(fmax(pl.x - x, 0.0), x - pl.y);
        const double dy = fmax(fmax(pl.z - y, 0.0), y - pl.w);
        best = fmin(best, sqrt(dx * dx + dy * dy + z * z));
    }
    return best;
}

// one Philox word of the LP stream: word w of block w / 4
__device__ __forceinline__ void lp_words(const PhiloxKeys& K, uint32_t blk, uint64_t path,
                                         uint64_t w[4]) {
    philox_block(K, blk, path, 0, 1, w); // ctr {blk, path, point 0, domain 1}
}

template <int KIND, int PHI>
__global__ void lp_walk_kernel(const DevScene S, const DevWos W, const PhiloxKeys K1,
                               double cx, double cy, double cz, double a, double e10, double e11,
                               double e12, double e20, double e21, double e22, double ax0,
                               double ax1, double ax2, double phix, int64_t n_paths,
                               double* __restrict__ val, int32_t* __restrict__ feat,
                               unsigned long long* __restrict__ counts,
                               unsigned long long* __restrict__ ctr) {
    extern __shared__ __align__(16) unsigned char smem[];
    double4* cav = reinterpret_cast<double4*>(smem);
    for (int i = threadIdx.x; i < S.n_cav; i += blockDim.x) cav[i] = S.cav[i];
    __syncthreads();
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_paths;
         k += (int64_t)gridDim.x * blockDim.x) {
        uint64_t w[4];
        lp_words(K1, 0, (uint64_t)k, w);
        // sample_start_point: theta = asin(sqrt(U)), phi = 2 pi U; cap_point
        const double u1 = (double)(w[0] >> 11) * 0x1.0p-53;
        const double u2 = (double)(w[1] >> 11) * 0x1.0p-53;
        const double th = asin(sqrt(u1)), ph = 2.0 * kPi * u2;
        double st, ct, sp, cp;
        sincos(th, &st, &ct);
        sincos(ph, &sp, &cp);
        const double lx = a * st * cp, ly = a * st * sp, lz = a * ct;
        double x = cx + (e10 * lx + e20 * ly + ax0 * lz);
        double y = cy + (e11 * lx + e21 * ly + ax1 * lz);
        double z = cz + (e12 * lx + e22 * ly + ax2 * lz);
        // the walk (wos.cpp:64-78) on words 2, 3, 4, ... of the same stream
        int steps = 0, f = -2;
        uint32_t blk = 0;
        int pos = 2;
        for (;;) {
            if (norm3(x, y, z) > W.trunc) { f = -1; break; }
            const double d = lp_nearest<KIND>(S, cav, x, y, z);
            if (d <= W.eps) {
                double px = x, py = y, pz = z;
                f = classify<KIND>(S, cav, W.eps, x, y, z, px, py, pz);
                if (f < 0) {
                    atomicAdd(&ctr[kCtrClassify], 1ull);
                } else {
                    x = px; y = py; z = pz;
                }
                break;
            }
            if (steps >= W.max_steps) { f = -2; break; }
            if (pos == 4) {
                lp_words(K1, ++blk, (uint64_t)k, w);
                pos = 0;
            }
            const double zz = 2.0 * ((double)(w[pos] >> 11) * 0x1.0p-53) - 1.0;
            const double az = 2.0 * kPi * ((double)(w[pos + 1] >> 11) * 0x1.0p-53);
            pos += 2;
            const double r = sqrt(fmax(1.0 - zz * zz, 0.0));
            double s, c;
            sincos(az, &s, &c);
            x = fma(d, r * c, x);
            y = fma(d, r * s, y);
            z = fma(d, zz, z);
            ++steps;
        }
        feat[k] = f;
        double v = 0.0;
        if (f == -1) v = phix;
        else if (f >= 0) {
            v = phix - eval_phi<PHI>(S, x, y, z, f);
            atomicAdd(&counts[f], 1ull);
        }
        val[k] = v;
    }
}

// Chunk statistics exactly as LpChunk (last_passage.cpp:15-43): thread c owns
// chunk c and pushes its paths in order into global scratch (5 doubles per
// chunk: n, n_inf, n_failed, mean, m2), then one thread merges the chunks in
// chunk order. No size limit beyond the path arrays themselves.
__global__ void lp_chunk_kernel(const double* __restrict__ val, const int32_t* __restrict__ feat,
                                int64_t n_paths, double* __restrict__ chunks) {
    const int64_t n_chunks = (n_paths + kChunk - 1) / kChunk;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_chunks;
         c += (int64_t)gridDim.x * blockDim.x) {
        double n = 0, ninf = 0, nfail = 0, mean = 0, m2 = 0;
        const int64_t hi = min((c + 1) * (int64_t)kChunk, n_paths);
        for (int64_t k = c * kChunk; k < hi; ++k) {
            const int f = feat[k];
            if (f == -2) { nfail += 1; continue; }
            if (f == -1) ninf += 1;
            n += 1;
            const double v = val[k];
            const double d = v - mean;
            mean += d / n;
            m2 += d * (v - mean);
        }
        double* r = chunks + 5 * c;
        r[0] = n; r[1] = ninf; r[2] = nfail; r[3] = mean; r[4] = m2;
    }
}

__global__ void lp_merge_kernel(const double* __restrict__ chunks, int64_t n_chunks,
                                double* __restrict__ out) {
    double n = 0, ninf = 0, nfail = 0, mean = 0, m2 = 0;
    for (int64_t c = 0; c < n_chunks; ++c) {
        const double* r = chunks + 5 * c;
        const double on = r[0], omean = r[3], om2 = r[4];
        ninf += r[1];
        nfail += r[2];
        if (on == 0) continue;
        if (n == 0) { n = on; mean = omean; m2 = om2; continue; }
        const double d = omean - mean;
        const double nt = n + on;
        mean += d * on / nt;
        m2 += om2 + d * d * n * on / nt;
        n = nt;
    }
    out[0] = n; out[1] = ninf; out[2] = nfail; out[3] = mean; out[4] = m2;
}

// eval_dirichlet (geometry.cpp:198-220) of one point on the device: value and
// feature, feature -3 when no feature lies within tol.
template <int KIND, int PHI>
__global__ void dirichlet_kernel(const DevScene S, double x, double y, double z, double tol,
                                 double* out) {
    extern __shared__ __align__(16) unsigned char smem[];
    double4* cav = reinterpret_cast<double4*>(smem);
    for (int i = threadIdx.x; i < S.n_cav; i += blockDim.x) cav[i] = S.cav[i];
    __syncthreads();
    if (threadIdx.x) return;
    double px = x, py = y, pz = z;
    const int f = classify<KIND>(S, cav, tol, x, y, z, px, py, pz);
    out[0] = f < 0 ? __longlong_as_double(0x7ff8000000000000LL) : eval_phi<PHI>(S, px, py, pz, f);
    out[1] = (double)f;
}

template <int KIND, int PHI>
cudaError_t launch_dirichlet_t(bw_ctx* ctx, const DevScene& S, size_t smem, const double* x,
                               double tol, double* d_out) {
    ++ctx->launches;
    dirichlet_kernel<KIND, PHI><<<1, 32, smem, ctx->stream>>>(S, x[0], x[1], x[2], tol, d_out);
    return cudaGetLastError();
}

template <int KIND, int PHI>
cudaError_t launch_lp_t(bw_ctx* ctx, const DevScene& S, size_t smem, const DevWos& W,
                        const double* c, double a, const double* ax, int64_t n_paths,
                        double phix, double* val, int32_t* feat, unsigned long long* counts,
                        double* red_out) {
    cudaError_t e;
    // frame (greens.cpp:98-105)
    const bool use_x = std::fabs(ax[0]) < 0.9;
    const double r0 = use_x ? 1.0 : 0.0, r1 = use_x ? 0.0 : 1.0;
    double c0 = ax[1] * 0.0 - ax[2] * r1, c1 = ax[2] * r0 - ax[0] * 0.0, c2 = ax[0] * r1 - ax[1] * r0;
    const double n = std::sqrt(c0 * c0 + c1 * c1 + c2 * c2);
    c0 /= n; c1 /= n; c2 /= n;
    const double e20 = ax[1] * c2 - ax[2] * c1, e21 = ax[2] * c0 - ax[0] * c2,
                 e22 = ax[0] * c1 - ax[1] * c0;
    const PhiloxKeys K1 = make_keys(W.keys.k0[0], 1);
    const int threads = 128;
    int64_t blocks = (n_paths + threads - 1) / threads;
    if (blocks > (int64_t)ctx->sm_count * 32) blocks = (int64_t)ctx->sm_count * 32;
    if (blocks < 1) blocks = 1;
    ++ctx->launches;
    lp_walk_kernel<KIND, PHI><<<(unsigned)blocks, threads, smem, ctx->stream>>>(
        S, W, K1, c[0], c[1], c[2], a, c0, c1, c2, e20, e21, e22, ax[0], ax[1], ax[2], phix, n_paths,
        val, feat, counts, ctx->d_counters);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int64_t n_chunks = (n_paths + kChunk - 1) / kChunk;
    bw_status st = BW_OK;
    double* chunks = (double*)scratch(ctx, kSlotTmp0, sizeof(double) * 5 * (size_t)std::max<int64_t>(n_chunks, 1), &st);
    if (st != BW_OK) return cudaErrorMemoryAllocation;
    ++ctx->launches;
    lp_chunk_kernel<<<(unsigned)std::min<int64_t>((n_chunks + 127) / 128 + 1, 4096), 128, 0, ctx->stream>>>(
        val, feat, n_paths, chunks);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ++ctx->launches;
    lp_merge_kernel<<<1, 1, 0, ctx->stream>>>(chunks, n_chunks, red_out);
    return cudaGetLastError();
}

#define BW_PHI_SWITCH(CALL)                                         \
    switch (S.phi_kind) {                                           \
        case BW_PHI_FEATURE_CONST: { constexpr int P = 0; CALL; }  \
        case BW_PHI_QUADRATIC: { constexpr int P = 1; CALL; }      \
        case BW_PHI_EXP_SIN_SIN: { constexpr int P = 2; CALL; }    \
        case BW_PHI_SIN_SIN: { constexpr int P = 4; CALL; }        \
        default: { constexpr int P = 3; CALL; }                     \
    }
#define BW_KIND_SWITCH(CALL)                                        \
    switch (S.kind) {                                               \
        case BW_SCENE_HALFSPACE: { constexpr int K = 0; BW_PHI_SWITCH(CALL) } \
        case BW_SCENE_PLATESET: { constexpr int K = 1; BW_PHI_SWITCH(CALL) }  \
        case BW_SCENE_THINDISK: { constexpr int K = 2; BW_PHI_SWITCH(CALL) }  \
        case BW_SCENE_SPHERE: { constexpr int K = 3; BW_PHI_SWITCH(CALL) }    \
        default: return cudaErrorNotSupported;                      \
    }

} // namespace

cudaError_t launch_dirichlet(bw_ctx* ctx, const DevScene& S, size_t smem, const double* x,
                             double tol, double* d_out) {
    BW_KIND_SWITCH(return (launch_dirichlet_t<K, P>(ctx, S, smem, x, tol, d_out)))
}

cudaError_t launch_lp(bw_ctx* ctx, const DevScene& S, size_t smem, const DevWos& W,
                      const double* c, double a, const double* ax, int64_t n_paths, double phix,
                      double* val, int32_t* feat, unsigned long long* counts, double* red) {
    BW_KIND_SWITCH(return (launch_lp_t<K, P>(ctx, S, smem, W, c, a, ax, n_paths, phix, val, feat,
                                             counts, red)))
}

} // namespace bw
