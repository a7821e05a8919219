// bw_diag.cu — FP64 pipe microbenchmark: the measured roofline denominator.
#include "bw_internal.h"

namespace bw {
namespace {

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void __launch_bounds__(256) dfma_kernel(double* out, double a, double b) {
    double acc[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += acc[c];
    if (s == 1.2345) out[0] = s; // keep the chains alive
}

__global__ void sqrt_kernel(const double* __restrict__ a, int64_t n, double* __restrict__ fast,
                            double* __restrict__ rn) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        fast[i] = sqrt_fast(a[i]);
        rn[i] = __dsqrt_rn(a[i]);
    }
}

} // namespace

cudaError_t launch_dfma(bw_ctx* ctx, double* tflops, double* ms_out) {
    double* d = nullptr;
    cudaError_t e = cudaMalloc(&d, sizeof(double));
    if (e != cudaSuccess) return e;
    const int blocks = ctx->sm_count * 8, threads = 256;
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    ++ctx->launches;
    dfma_kernel<<<blocks, threads, 0, ctx->stream>>>(d, 0.999999, 1e-7); // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(t0, ctx->stream);
        ++ctx->launches;
        dfma_kernel<<<blocks, threads, 0, ctx->stream>>>(d, 0.999999, 1e-7);
        cudaEventRecord(t1, ctx->stream);
        cudaEventSynchronize(t1);
        float ms = 0;
        cudaEventElapsedTime(&ms, t0, t1);
        if (ms < best) best = ms;
    }
    e = cudaGetLastError();
    const double flops = 2.0 * kChains * kIters * (double)blocks * threads;
    *tflops = flops / (best * 1e-3) / 1e12;
    *ms_out = best;
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    cudaFree(d);
    return e;
}

// The WOS stream of one (point, walk) as K1 forms it: per-node table (rounds
// 0-1 block words, round-2 M0 products), per-walk round-1 product, then
// philox_wos_nt; one warp, blocks b = lane, lane + 32, ...
__global__ void wos_stream_kernel(PhiloxKeys K, uint64_t point, uint64_t path, int n_blocks,
                                  uint64_t* __restrict__ out) {
    __shared__ ulonglong2 nt[2 * kBlkTab];
    const int lane = threadIdx.x;
    const uint64_t lo1p = kM1 * point;
    const uint64_t hi1p = __umul64hi(kM1, point);
    node_tab_fill(K, lo1p, nt, lane);
    __syncwarp();
    uint64_t wh, wl;
    walk_prod(K, path, hi1p, wh, wl);
    for (int b = lane; b < n_blocks; b += 32) {
        uint64_t w[4];
        philox_wos_nt(K, nt, (uint32_t)b, wh, wl, lo1p, w);
        for (int j = 0; j < 4; ++j) out[4 * (int64_t)b + j] = w[j];
    }
}

// The BW_RNG_PHILOX4X32 stream of one (point, walk) as K1 forms it (per-node
// uint4 table, per-walk round-1 product, p32_wos_block); one warp.
__global__ void wos_stream32_kernel(Philox32Keys K, uint64_t point, uint32_t path, int n_blocks,
                                    uint64_t* __restrict__ out) {
    __shared__ uint4 tab[kBlkTab32 + 1];
    const int lane = threadIdx.x;
    const P32Node N = p32_node(point);
    for (int b = lane; b < kBlkTab32; b += 32) tab[b] = p32_tab_entry(K, N, (uint32_t)b);
    if (lane == 0) tab[kBlkTab32] = make_uint4(K.kk[1], K.kk[2], 0u, 0u);
    __syncwarp();
    uint32_t wh, wl;
    p32_walk(K, N, path, wh, wl);
    for (int b = lane; b < n_blocks; b += 32) {
        uint32_t o0, o1, o2, o3;
        p32_wos_block_s(K, N, (uint32_t)__cvta_generic_to_shared(tab), (uint32_t)b, wh, wl, o0, o1,
                        o2, o3);
        p32_words(o0, o1, o2, o3, out[2 * (int64_t)b], out[2 * (int64_t)b + 1]);
    }
}

__global__ void philox32_kernel(const uint32_t* __restrict__ ctr, const uint32_t* __restrict__ key,
                                int64_t n, uint32_t* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    Philox32Keys K;
    uint32_t a = key[2 * i], b = key[2 * i + 1];
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) {
            a += kP32W0;
            b += kP32W1;
        }
        K.kk[2 * r] = a;
        K.kk[2 * r + 1] = b;
    }
    uint32_t c[4] = {ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]};
    philox4x32_block(K, c);
    for (int j = 0; j < 4; ++j) out[4 * i + j] = c[j];
}

} // namespace bw

extern "C" bw_status bw_diag_wos_stream32(bw_ctx* ctx, uint64_t seed, uint64_t point_id,
                                          uint64_t path_id, int32_t n_blocks, uint64_t* out) {
    if (!ctx || n_blocks < 0 || (n_blocks > 0 && !out)) return BW_ERR_INVALID;
    if (n_blocks == 0) return BW_OK;
    cudaSetDevice(ctx->device);
    uint64_t* d = nullptr;
    cudaError_t e = cudaMalloc(&d, 2 * (size_t)n_blocks * sizeof(uint64_t));
    if (e == cudaSuccess) {
        ++ctx->launches;
        bw::wos_stream32_kernel<<<1, 32, 0, ctx->stream>>>(bw::make_keys32(seed, 0), point_id,
                                                           (uint32_t)path_id, n_blocks, d);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, 2 * (size_t)n_blocks * sizeof(uint64_t),
                                              cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    cudaFree(d);
    return bw::cuda_check(ctx, e, "diag_wos_stream32");
}

extern "C" bw_status bw_philox4x32_blocks(bw_ctx* ctx, const uint32_t* ctr, const uint32_t* key,
                                          int64_t n, uint32_t* out) {
    if (!ctx || n < 0 || (n > 0 && (!ctr || !key || !out))) return BW_ERR_INVALID;
    if (n == 0) return BW_OK;
    cudaSetDevice(ctx->device);
    uint32_t* d = nullptr;
    const size_t bytes = (size_t)n * 10 * sizeof(uint32_t);
    cudaError_t e = cudaMalloc(&d, bytes);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d, ctr, 4 * n * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d + 4 * n, key, 2 * n * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) {
        ++ctx->launches;
        bw::philox32_kernel<<<(unsigned)((n + 127) / 128), 128, 0, ctx->stream>>>(d, d + 4 * n, n, d + 6 * n);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, d + 6 * n, 4 * n * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    cudaFree(d);
    return bw::cuda_check(ctx, e, "philox4x32_blocks");
}

extern "C" bw_status bw_diag_wos_stream(bw_ctx* ctx, uint64_t seed, uint64_t point_id,
                                        uint64_t path_id, int32_t n_blocks, uint64_t* out) {
    if (!ctx || n_blocks < 0 || (n_blocks > 0 && !out)) return BW_ERR_INVALID;
    if (n_blocks == 0) return BW_OK;
    cudaSetDevice(ctx->device);
    uint64_t* d = nullptr;
    cudaError_t e = cudaMalloc(&d, 4 * (size_t)n_blocks * sizeof(uint64_t));
    if (e == cudaSuccess) {
        ++ctx->launches;
        bw::wos_stream_kernel<<<1, 32, 0, ctx->stream>>>(bw::make_keys(seed, 0), point_id, path_id,
                                                         n_blocks, d);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, 4 * (size_t)n_blocks * sizeof(uint64_t),
                                              cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    cudaFree(d);
    return bw::cuda_check(ctx, e, "diag_wos_stream");
}

extern "C" bw_status bw_measure_fp64_peak(bw_ctx* ctx, double* tflops, double* kernel_ms) {
    if (!ctx || !tflops) return BW_ERR_INVALID;
    cudaSetDevice(ctx->device);
    double ms = 0;
    bw_status st = bw::cuda_check(ctx, bw::launch_dfma(ctx, tflops, &ms), "dfma");
    if (kernel_ms) *kernel_ms = ms;
    return st;
}

extern "C" bw_status bw_diag_sqrt(bw_ctx* ctx, const double* a, int64_t n, double* fast,
                                  double* rn) {
    if (!ctx || n < 0 || (n > 0 && (!a || !fast || !rn))) return BW_ERR_INVALID;
    if (n == 0) return BW_OK;
    cudaSetDevice(ctx->device);
    double *d = nullptr;
    cudaError_t e = cudaMalloc(&d, 3 * n * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpyAsync(d, a, n * sizeof(double), cudaMemcpyHostToDevice,
                                              ctx->stream);
    if (e == cudaSuccess) {
        ++ctx->launches;
        bw::sqrt_kernel<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(d, n, d + n, d + 2 * n);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(fast, d + n, n * sizeof(double),
                                              cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(rn, d + 2 * n, n * sizeof(double),
                                              cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    cudaFree(d);
    return bw::cuda_check(ctx, e, "diag_sqrt");
}

extern "C" bw_status bw_diag_stat_math(bw_ctx* ctx, const double* a, const uint32_t* u, int64_t n,
                                       double* root, double* sn, double* cs) {
    if (!ctx || n < 0 || (n > 0 && (!a || !u || !root || !sn || !cs))) return BW_ERR_INVALID;
    if (n == 0) return BW_OK;
    cudaSetDevice(ctx->device);
    double* d = nullptr;
    uint32_t* du = nullptr;
    cudaError_t e = cudaMalloc(&d, 4 * n * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&du, n * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemcpyAsync(d, a, n * sizeof(double), cudaMemcpyHostToDevice,
                                              ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(du, u, n * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                              ctx->stream);
    if (e == cudaSuccess) e = bw::launch_stat_math(ctx, d, du, n, d + n, d + 2 * n, d + 3 * n);
    if (e == cudaSuccess) e = cudaMemcpyAsync(root, d + n, n * sizeof(double),
                                              cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(sn, d + 2 * n, n * sizeof(double),
                                              cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(cs, d + 3 * n, n * sizeof(double),
                                              cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    cudaFree(d);
    cudaFree(du);
    return bw::cuda_check(ctx, e, "diag_stat_math");
}
