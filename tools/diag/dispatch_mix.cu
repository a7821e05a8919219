// Does an fp64 instruction hold the SMSP's dispatch port for two cycles on
// B200? Times ND independent DFMA chains and NA independent 32-bit ALU chains
// (LOP3 / IADD3 alternating) per thread, alone and mixed, 8 warps per SMSP.
// If the port is shared, the mixed time is the SUM of the two alone times
// (2 cycles per DFMA + 1 per ALU op); if fp64 only occupied its own pipe, the
// mixed time would be the MAX. Diagnostic, not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int kIters = 4096;
template <int ND, int NA>
__global__ void __launch_bounds__(128) mix(uint32_t* o, double* od, uint32_t m, double dm) {
    uint32_t a[NA > 0 ? NA : 1];
    double d[ND > 0 ? ND : 1];
#pragma unroll
    for (int c = 0; c < NA; ++c) a[c] = threadIdx.x * 2654435761u + c;
#pragma unroll
    for (int c = 0; c < ND; ++c) d[c] = threadIdx.x * 1e-3 + c;
#pragma unroll 1
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < (ND > NA ? ND : NA); ++c) {
            if (c < ND) d[c] = fma(d[c], dm, 1e-7);
            if (c < NA) a[c] = (c & 1) ? (a[c] ^ m ^ (uint32_t)i) : (a[c] + m + (uint32_t)i);
            if (c + ND < NA) a[c + ND] = ((c + ND) & 1) ? (a[c + ND] ^ m ^ (uint32_t)i) : (a[c + ND] + m + (uint32_t)i);
        }
    }
    uint32_t s = 0; double t = 0;
#pragma unroll
    for (int c = 0; c < NA; ++c) s ^= a[c];
#pragma unroll
    for (int c = 0; c < ND; ++c) t += d[c];
    if (s == 0x12345u) o[0] = s;
    if (t == 1.2345) od[0] = t;
}
template <int ND, int NA>
void run(int sms, uint32_t* o, double* od, double ghz) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = sms * 8; // 8 warps per SMSP
    mix<ND, NA><<<blocks, 128>>>(o, od, 0x9E3779B9u, 0.999999);
    cudaEventRecord(e0);
    mix<ND, NA><<<blocks, 128>>>(o, od, 0x9E3779B9u, 0.999999);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double cyc = ms * 1e-3 * ghz * 1e9;
    const double per_iter = cyc / kIters / 8.0; // SMSP cycles per warp-iteration
    printf("dfma %2d, alu %2d: %.3f ms, %.2f SMSP-cycles per warp-iteration (2 ND + NA = %d, max = %d)\n",
           ND, NA, ms, per_iter, 2 * ND + NA, 2 * ND > NA ? 2 * ND : NA);
}
int main() {
    int sms, khz; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double ghz = khz * 1e-6;
    printf("SMs %d, clock %.3f GHz\n", sms, ghz);
    uint32_t* o; double* od; cudaMalloc(&o, 4); cudaMalloc(&od, 8);
    run<8, 0>(sms, o, od, ghz); run<0, 8>(sms, o, od, ghz); run<0, 16>(sms, o, od, ghz);
    run<8, 8>(sms, o, od, ghz); run<8, 16>(sms, o, od, ghz); run<4, 16>(sms, o, od, ghz);
    run<6, 12>(sms, o, od, ghz);
    return 0;
}
