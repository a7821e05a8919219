// Throughput microbenchmark of the integer multiply forms Philox4x64 compiles to
// (IMAD.WIDE.U32, IMAD.HI.U32, IMAD) and of DFMA on one B200, in warp-instructions
// per SM-cycle. Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a int_pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kChains = 8, kIters = 2048;

template <int OP>
__global__ void __launch_bounds__(256) kern(uint32_t* out, uint32_t m, uint32_t seed, long long* clk) {
    uint32_t a[kChains], b[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) { a[c] = seed * (threadIdx.x + c); b[c] = c; }
    long long t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if (OP == 0) { // IMAD.WIDE.U32: 64-bit accumulate
                uint64_t w = (uint64_t)a[c] * m + b[c];
                a[c] = (uint32_t)w; b[c] = (uint32_t)(w >> 32);
            } else if (OP == 1) { // IMAD.HI.U32
                a[c] = __umulhi(a[c], m) + b[c];
            } else if (OP == 2) { // IMAD (lo)
                a[c] = a[c] * m + b[c];
            } else if (OP == 4) { // full 64x64->128 product by a constant (Philox mulhilo)
                uint64_t x = ((uint64_t)b[c] << 32) | a[c];
                uint64_t lo = x * 0xD2E7470EE14C6C93ULL, hi = __umul64hi(x, 0xD2E7470EE14C6C93ULL);
                a[c] = (uint32_t)(hi ^ lo); b[c] = (uint32_t)((hi >> 32) ^ (lo >> 32)) ^ m;
            } else if (OP == 3) { // LOP3
                a[c] = (a[c] ^ m) ^ b[c]; b[c] = a[c] ^ (b[c] + 1);
            }
        }
    }
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s ^= a[c] ^ b[c];
    if (s == 0x12345u) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) clk[0] = t1 - t0;
}

__global__ void __launch_bounds__(256) dk(double* out, double m, long long* clk) {
    double a[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) a[c] = threadIdx.x * 1e-3 + c;
    long long t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) a[c] = fma(a[c], m, 1e-7);
    }
    long long t1 = clock64();
    double s = 0;
    for (int c = 0; c < kChains; ++c) s += a[c];
    if (s == 1.2345) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) clk[0] = t1 - t0;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* o; double* od; long long* clk;
    cudaMalloc(&o, 4); cudaMalloc(&od, 8); cudaMalloc(&clk, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char* names[] = {"IMAD.WIDE.U32 op", "IMAD.HI.U32 op", "IMAD op", "LOP3 op", "mulhilo64", "DFMA"};
    const double ghz = 1.965;
    for (int op = 0; op < 6; ++op) {
        for (int wps : {4, 8, 16, 24, 32, 48}) {
            const int thr = 128, blocks = sms * (wps / 4);
            auto launch = [&] {
                if (op == 0) kern<0><<<blocks, thr>>>(o, 0x9E3779B9u, 7, clk);
                if (op == 1) kern<1><<<blocks, thr>>>(o, 0x9E3779B9u, 7, clk);
                if (op == 2) kern<2><<<blocks, thr>>>(o, 0x9E3779B9u, 7, clk);
                if (op == 3) kern<3><<<blocks, thr>>>(o, 0x9E3779B9u, 7, clk);
                if (op == 4) kern<4><<<blocks, thr>>>(o, 0x9E3779B9u, 7, clk);
                if (op == 5) dk<<<blocks, thr>>>(od, 0.999999, clk);
            };
            launch(); cudaDeviceSynchronize();
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            const double ops = (double)kChains * kIters * blocks * thr / 32.0; // warp-level ops
            printf("%-18s warps/SM %2d: %.3f warp-ops per SM-cycle at %.3f GHz (%.3f ms)\n", names[op], wps,
                   ops / sms / (ms * 1e-3 * ghz * 1e9), ghz, ms);
        }
    }
    return 0;
}
