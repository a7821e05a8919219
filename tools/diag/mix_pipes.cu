// Do IMAD.WIDE (fmaheavy) and DFMA (fp64) share issue capacity on B200?
// Times N_W wide-multiply chains and N_D DFMA chains per thread, alone and mixed.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int kIters = 2048;
template <int NW, int ND>
__global__ void __launch_bounds__(128) mix(uint32_t* o, double* od, uint32_t m, double dm) {
    uint32_t a[NW > 0 ? NW : 1], b[NW > 0 ? NW : 1];
    double d[ND > 0 ? ND : 1];
#pragma unroll
    for (int c = 0; c < NW; ++c) { a[c] = threadIdx.x + c; b[c] = c; }
#pragma unroll
    for (int c = 0; c < ND; ++c) d[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < NW; ++c) {
            uint64_t w = (uint64_t)a[c] * m + ((uint64_t)b[c] << 32 | b[c]);
            a[c] = (uint32_t)w; b[c] = (uint32_t)(w >> 32);
        }
#pragma unroll
        for (int c = 0; c < ND; ++c) d[c] = fma(d[c], dm, 1e-7);
    }
    uint32_t s = 0; double t = 0;
#pragma unroll
    for (int c = 0; c < NW; ++c) s ^= a[c] ^ b[c];
#pragma unroll
    for (int c = 0; c < ND; ++c) t += d[c];
    if (s == 0x12345u) o[0] = s;
    if (t == 1.2345) od[0] = t;
}
template <int NW, int ND>
void run(int sms, uint32_t* o, double* od) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = sms * 8;
    mix<NW, ND><<<blocks, 128>>>(o, od, 0x9E3779B9u, 0.999999);
    cudaEventRecord(e0);
    mix<NW, ND><<<blocks, 128>>>(o, od, 0x9E3779B9u, 0.999999);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double cyc = ms * 1e-3 * 1.965e9;
    const double warps = blocks * 4.0 / sms / 4.0; // per SMSP
    printf("wide chains %d, dfma chains %d: %.3f ms, per SMSP-cycle: %.3f wide-ops, %.3f dfma\n", NW, ND, ms,
           NW * kIters * warps / cyc, ND * kIters * warps / cyc);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* o; double* od; cudaMalloc(&o, 4); cudaMalloc(&od, 8);
    run<8, 0>(sms, o, od); run<0, 8>(sms, o, od); run<8, 8>(sms, o, od);
    run<8, 4>(sms, o, od); run<4, 8>(sms, o, od);
    return 0;
}
