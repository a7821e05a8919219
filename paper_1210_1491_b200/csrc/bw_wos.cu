// bw_wos.cu — K1: the walk-on-spheres kernels (sm_100a, fp64).
//
// Replaces the reference's estimate_u_batch -> walk -> nearest_feature ->
// classify_exit -> exit_value chain (wos.cpp:61-132, geometry.cpp:131-239).
//
// Design:
//  * Persistent warps. A warp takes one node (= one start point) from a
//    global queue and runs ALL of that node's n_paths walks: lane l starts
//    walk l; a lane whose walk ends takes the next walk index (ballot +
//    popc, lane order), so a warp stays full until the node's walks run out.
//    Which walks a lane runs depends only on the node's own trajectories, so
//    per-node results are bitwise independent of the grid, the queue order
//    and the number of GPUs (the guarantee of wos.hpp:43-44).
//  * Philox4x64-10 streams keyed exactly as the reference's RngStream
//    (seed, point_id, path_id, domain 0). One block per loop trip feeds two
//    jumps, so every lane needs a block on every trip (no divergent RNG).
//  * Per-lane Welford (wos.cpp:18-23), then a fixed shuffle tree of Chan
//    merges (wos.cpp:24-39). The reference merges 4096-walk chunks in path
//    order instead; both are exact Welford/Chan algebra, so results agree to
//    rounding (statistical parity).
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "bw_internal.h"

#ifndef BW_GRID_MAGIC
#define BW_GRID_MAGIC 1
#endif
#ifndef BW_SINCOS_XOR
#define BW_SINCOS_XOR 1
#endif
#ifndef BW_SINCOS_HI
#define BW_SINCOS_HI 1
#endif
#ifndef BW_CAND_INT
#define BW_CAND_INT 1
#endif
#ifndef BW_FACE_NOSQRT
#define BW_FACE_NOSQRT 1
#endif

namespace bw {

namespace {

constexpr int kWarpsPerBlock = 4;


struct SmemScene {
    const double4* cav;
    const uint16_t* cstart;
    const uint16_t* clist;
    // 32-bit shared-window addresses of the same arrays (stage<true>), held in
    // registers: the candidate loop then addresses shared memory directly
    // instead of re-deriving the window base and the list offset every entry
    uint32_t cav_s, cs_s, cl_s;
};

__device__ __forceinline__ uint32_t shared_addr(const void* p) {
    // volatile: the address stays in a register (no per-use rematerialisation)
    uint32_t a;
    asm volatile("mov.b32 %0, %1;" : "=r"(a) : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return a;
}
__device__ __forceinline__ unsigned lds_u16(uint32_t a) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double4 lds_d4(uint32_t a) {
    double4 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+16];" : "=d"(v.z), "=d"(v.w) : "r"(a));
    return v;
}

// nearest_feature (geometry.cpp:131-155) for the compiled scene kind. SH: the
// candidate grid and the cavities are staged in shared memory (stage<true>).
// Rp: the sphere's radius from a register the caller pins (K1's statistical
// loop; ptxas otherwise reloads S.R from the parameter bank on every block).
template <int KIND, bool SH = false, bool FAST = false>
__device__ __forceinline__ double nearest(const DevScene& S, const SmemScene& M, double x,
                                          double y, double z, double Rp) {
    if (KIND == BW_SCENE_HALFSPACE) return fabs(z - S.plane_z);
    if (KIND == BW_SCENE_PLATESET) { // plate_distance (geometry.cpp:11-15), lowest index wins
        double best = __longlong_as_double(0x7ff0000000000000LL);
        for (int i = 0; i < S.n_cav; ++i) {
            const double4 pl = M.cav[i];
            const double dx = fmax(fmax(pl.x - x, 0.0), x - pl.y);
            const double dy = fmax(fmax(pl.z - y, 0.0), y - pl.w);
            best = fmin(best, sqrt(dx * dx + dy * dy + z * z));
        }
        return best;
    }
    if (KIND == BW_SCENE_THINDISK) { // geometry.cpp:143-149
        const double rho = hypot(x, y);
        return rho <= S.disk_r ? fabs(z) : hypot(rho - S.disk_r, z);
    }
    // FAST (K1's statistical mode): the signed value; every consumer there
    // takes |d| as an operand modifier (post, the jump's three fma), which
    // saves the DADD that forms fabs on the fp64 pipe
    if (KIND == BW_SCENE_SPHERE) {
        // (a walk position exactly at the centre, |p|^2 = 0, would make this NaN:
        // the walk then runs out its step budget and counts as failed, like any
        // walk the reference gives up on; node starts take the exact root)
        if (FAST && BW_SQRT_Q) return sqrt_q_minus(x * x + y * y + z * z, Rp);
        const double dr = sqrt_walk<FAST>(x * x + y * y + z * z) - S.R;
        return FAST ? dr : fabs(dr);
    }
    double best = box_face_distance<FAST>(S, x, y, z);
    if (KIND == BW_SCENE_BOX_CAVITIES) {
        if (S.gn > 0) {
            // candidate list of the cell holding p: contains every cavity that
            // can be nearest anywhere in the cell (bw_capi.cu build_grid), so the
            // min equals the brute-force min (up to the rounding of the pruning
            // test below, i.e. within an ulp, in rare near-ties).
            const int gn = S.gn;
#if BW_GRID_MAGIC
            const int ix = grid_axis(x, S.ginv, S.gc0[0], gn);
            const int iy = grid_axis(y, S.ginv, S.gc0[1], gn);
            const int iz = grid_axis(z, S.ginv, S.gc0[2], gn);
#else
            int ix = (int)floor((x - S.gorig[0]) * S.ginv);
            int iy = (int)floor((y - S.gorig[1]) * S.ginv);
            int iz = (int)floor((z - S.gorig[2]) * S.ginv);
            ix = min(max(ix, 0), gn - 1);
            iy = min(max(iy, 0), gn - 1);
            iz = min(max(iz, 0), gn - 1);
#endif
            const int cell = (iz * gn + iy) * gn + ix;
            BW_CHECK(cell >= 0 && cell < gn * gn * gn);
            const int b = SH ? (int)lds_u16(M.cs_s + 2u * cell) : M.cstart[cell];
            const int e = SH ? (int)lds_u16(M.cs_s + 2u * cell + 2u) : M.cstart[cell + 1];
            BW_CHECK(b <= e);
            // candidates come by lower bound L_i over the cell, ascending
            // (bw_capi.cu build_grid): once L_i >= best no later one can be
            // nearer (packed lists carry L_i); one whose squared centre
            // distance is >= (best + r)^2 cannot be either, so its root is skipped
#if BW_CAND_INT
            if (S.lpacked) {
                // the L_i test on the raw entry: with q = ceil(best / lstep)
                // (linv is rounded up), Lq >= q gives Lq lstep >= best, i.e. stop
                // at entry >= q << 8. Every entry the product test
                // (Lq lstep < best) visits is still visited, and an entry only
                // this test visits has distance >= best, so the minimum is
                // bitwise the same. best <= 0 (a rounding error outside the
                // box) gives q <= 0: nothing is visited.
                int thr = min(__double2int_ru(best * S.linv), 256) << 8;
                for (int t = b; t < e; ++t) {
                    const int ent = (int)(SH ? lds_u16(M.cl_s + 2u * t) : M.clist[t]);
                    if (ent >= thr) break;
                    BW_CHECK((ent & 0xff) < S.n_cav);
                    const double4 c = SH ? lds_d4(M.cav_s + 32u * (ent & 0xff)) : M.cav[ent & 0xff];
                    const double qx = x - c.x, qy = y - c.y, qz = z - c.z;
                    const double d2 = qx * qx + qy * qy + qz * qz;
                    const double lim = best + c.w;
#ifndef BW_CAND_NOPRE
#define BW_CAND_NOPRE 1 // statistical mode: no d2 < (best + r)^2 pretest before the 4-fp64 root (+2.2 % cfg3)
#endif
                    if ((FAST && BW_CAND_NOPRE) || d2 < lim * lim) {
                        best = dmin_nn(FAST && BW_SQRT_Q ? fabs(sqrt_q_minus(d2, c.w)) : fabs(sqrt_walk<FAST>(d2) - c.w), best);
                        thr = min(__double2int_ru(best * S.linv), 256) << 8;
                    }
                }
                return best;
            }
#endif
            const unsigned imask = S.lpacked ? 0xffu : 0xffffu;
            for (int t = b; t < e; ++t) {
                const unsigned ent = SH ? lds_u16(M.cl_s + 2u * t) : M.clist[t];
                if (S.lpacked && (double)(ent >> 8) * S.lstep >= best) break;
                BW_CHECK((int)(ent & imask) < S.n_cav);
                const double4 c = SH ? lds_d4(M.cav_s + 32u * (ent & imask)) : M.cav[ent & imask];
                const double qx = x - c.x, qy = y - c.y, qz = z - c.z;
                const double d2 = qx * qx + qy * qy + qz * qz;
                const double lim = best + c.w;
                if (d2 < lim * lim) best = dmin_nn(FAST && BW_SQRT_Q ? fabs(sqrt_q_minus(d2, c.w)) : fabs(sqrt_walk<FAST>(d2) - c.w), best);
            }
        } else {
            for (int i = 0; i < S.n_cav; ++i) {
                const double4 c = M.cav[i];
                best = fmin(best, fabs(norm3(x - c.x, y - c.y, z - c.z) - c.w));
            }
        }
    }
    return best;
}

// (sin, cos)(2 pi U) for U = (w >> 11) 2^-53, without a generic range
// reduction: with m = w >> 11, 4U = m 2^-51 splits EXACTLY into the nearest
// integer q (integer arithmetic) and r = 4U - q in [-1/2, 1/2], so
// 2 pi U = (pi/2)(q + r): one polynomial pair in r on |pi r / 2| <= pi/4 and a
// quadrant swap/sign by q. sin(pi r/2) = r P(r^2), cos(pi r/2) = Q(r^2) with P
// (degree 6) and Q (degree 7) Chebyshev fits on r^2 in [0, 1/4] (fit error
// 3e-18 and 3e-20 relative; tools/fit_sincos.py): <= 0.82 / 0.59 ulp after
// rounding, as accurate as the 9-term Taylor pair they replace, 3 DFMA fewer.
__constant__ double kSinC[7] = {0x1.921fb54442d18p+0,  -0x1.4abbce625be41p-1, 0x1.466bc677587f8p-4,
                                -0x1.32d2cce2e5b19p-8, 0x1.50782fda12d96p-13, -0x1.e30071afc3e59p-19,
                                0x1.e3f38399551bfp-25};
__constant__ double kCosC[8] = {0x1.0000000000000p+0,  -0x1.3bd3cc9be45dep+0, 0x1.03c1f081b5aacp-2,
                                -0x1.55d3c7e3c90f8p-6, 0x1.e1f5068355e15p-11, -0x1.a6d1ec7906c20p-16,
                                0x1.f9cc41140bb60p-22, -0x1.b264ba152378ap-28};

// FAST (RNG = 1 only): degree-5 / degree-6 fits of the same functions (fit
// error 6.7e-15 / 4.7e-17; |sin| within 3.4e-15 absolute), 2 DFMA fewer.
__constant__ double kSinC5[6] = {0x1.921fb54442cfap+0, -0x1.4abbce6257a2ap-1, 0x1.466bc67123fa1p-4,
                                 -0x1.32d2c644adc0bp-8, 0x1.5071ce4b47930p-13, -0x1.dd54805f3f706p-19};
__constant__ double kCosC6[7] = {0x1.0000000000000p+0,  -0x1.3bd3cc9be458bp+0, 0x1.03c1f081b0780p-2,
                                 -0x1.55d3c7dbfd139p-6, 0x1.e1f4fb60281f6p-11, -0x1.a6c9c1be9eb49p-16,
                                 0x1.f3dbcea61b1a4p-22};

// FAST + BW_SINCOS_TAB (RNG = 1): (sin, cos) of the stream's azimuth
// az = 2 pi (u + 1/2) 2^-32 from its 32-bit word u, by a table of the centre
// angles a_k = (k + 1/2) 2 pi / kTrigTab (filled from long-double sinl / cosl
// at bw_init, staged in shared memory per CTA) and the angle addition rule
// with short series in the remainder: with B = kTrigBits, u = k 2^(32-B) + f,
// k the top B bits (one shift, one mask -> the table's byte offset) and f the
// low 32-B bits (one mask),
//   delta = (f + 1/2 - 2^(31-B)) 2 pi 2^-32, |delta| <= pi / kTrigTab,
//   sin delta = delta (1 - delta^2/6 + delta^4/120)
//   cos delta = 1 - delta^2/2 + delta^4/24 (- delta^6/720 for B = 8)
// (B = 9: truncation <= 7e-20 / 8e-17, B = 8: 1e-17 / 2e-20), so the result is
// within ~2 ulp of sin / cos(az): 11 (B = 9) or 12 fp64 + 1 LDS.128 per sincos
// against 19 fp64 and the quadrant logic of the polynomial pair.
#ifndef BW_SINCOS_TAB
#define BW_SINCOS_TAB 1
#endif
#ifndef BW_TRIG_BITS
#define BW_TRIG_BITS 9
#endif
constexpr int kTrigBits = BW_TRIG_BITS;
constexpr int kTrigTab = 1 << kTrigBits;
__constant__ double2 kTrig[kTrigTab]; // {sin a_k, cos a_k}

// stage kTrig into the CTA's table (256 entries measured -0.7 % on the cavity
// box and -3 % on the sphere against 512: profiles/r2/ab_u32.log)
__device__ __forceinline__ void stage_trig(double2* trig) {
    for (int i = threadIdx.x; i < kTrigTab; i += blockDim.x) trig[i] = kTrig[i];
}

// The loop's fp64 literals with a non-zero low word (DFMA takes a 32-bit
// immediate for the high word only; the others ptxas re-materialises with two
// moves each on every trip). PIN keeps them in registers across the loop by
// passing them through shared memory with volatile loads, which ptxas cannot
// re-materialise: +1.7 % on the sphere, +0.4 % on the cavity box, -3.8 % on
// the plain box (80 registers, no room), so the box kernels do not pin
// (profiles/r2/ab_u32_pin.log).
#ifndef BW_PIN_CONST
#define BW_PIN_CONST(KIND) ((KIND) != BW_SCENE_BOX)
#endif
struct JumpConst {
    double k, kh, c3, c5, c4, z31;
};
template <int B, bool PIN, bool PINZ = false>
__device__ __forceinline__ JumpConst jump_const() {
    // kh = (1/2 - 2^(31-B)) k: the remainder's offset from the entry's centre
    // angle, exact in a double before the one rounding of the product
    JumpConst J{0x1.921fb54442d18p-30, (0.5 - (double)(1u << (B > 0 ? 31 - B : 22))) * 0x1.921fb54442d18p-30,
                -0x1.5555555555555p-3, 0x1.1111111111111p-7, 0x1.5555555555555p-5, 0x1.0p-31};
    if constexpr (PIN) {
    __shared__ double kc[6];
    if (threadIdx.x == 0) {
        kc[0] = J.k; kc[1] = J.kh; kc[2] = J.c3; kc[3] = J.c5; kc[4] = J.c4; kc[5] = J.z31;
    }
    __syncthreads();
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(kc);
    asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(J.k) : "r"(a));
    asm volatile("ld.volatile.shared.f64 %0, [%1+8];" : "=d"(J.kh) : "r"(a));
    asm volatile("ld.volatile.shared.f64 %0, [%1+16];" : "=d"(J.c3) : "r"(a));
    asm volatile("ld.volatile.shared.f64 %0, [%1+24];" : "=d"(J.c5) : "r"(a));
    asm volatile("ld.volatile.shared.f64 %0, [%1+32];" : "=d"(J.c4) : "r"(a));
    // 2^-31 (z's scale; a high-word immediate, but the fma already carries one):
    // pinned on the sphere only (+1.0 %; -0.9 % on the cavity box)
    if (PINZ) asm volatile("ld.volatile.shared.f64 %0, [%1+40];" : "=d"(J.z31) : "r"(a));
    }
    return J;
}

template <int B>
__device__ __forceinline__ void sincos32_tab(uint32_t u, uint32_t trig_s, const JumpConst& J,
                                             double& s, double& c) {
    static_assert(B == 8 || B == 9, "series lengths are set for 256 / 512 entries");
    // byte offset of entry k = u >> (32 - B), and f = the low 32 - B bits
    const uint32_t k16 = (u >> (28 - B)) & (uint32_t)(((1 << B) - 1) << 4);
    const uint32_t f = u & ((1u << (32 - B)) - 1u);
    const double delta = fma((double)f, J.k, J.kh); // (f + 1/2 - 2^(31-B)) 2 pi 2^-32
    double s0, c0;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(s0), "=d"(c0) : "r"(trig_s + k16));
    const double d2 = delta * delta;
    // with the ~1e-12 roots (BW_SQRT_Q) the delta^5/120 term (<= 7e-14 at
    // B = 9) is below the direction's own error: sin delta = delta - delta^3/6
    const double sd = BW_SQRT_Q && B >= 9 ? fma(delta * d2, J.c3, delta)
                                          : fma(delta, d2 * fma(d2, J.c5, J.c3), delta);
    const double cd = B >= 9
        ? fma(d2, fma(d2, J.c4, -0.5), 1.0)
        : fma(d2, fma(d2, fma(d2, -0x1.6c16c16c16c17p-10, J.c4), -0.5), 1.0);
    s = fma(s0, cd, c0 * sd);
    c = fma(c0, cd, -(s0 * sd));
}

// The same azimuth without the table (the kernels that cannot spare its
// shared memory): 4 (u + 1/2) 2^-32 = q + r with q = round(u 2^-30) mod 4 and
// r = (t + 1/2) 2^-30, t the sign-extended low 30 bits of u; then the FAST
// polynomial pair in r and the quadrant swap / signs of sincos_2pi_u.
__device__ __forceinline__ void sincos32_poly(uint32_t u, double& s, double& c);

template <bool XOR = (BW_SINCOS_XOR != 0), bool FAST = false>
__device__ __forceinline__ void sincos_2pi_u(uint64_t w, double& s, double& c) {
#if BW_SINCOS_HI
    // the same q and r from 32-bit ops on the word: with v = w & ~0x7FF
    // (= m 2^11), q = (v + 2^61) >> 62 (mod 4 suffices) sits in the top two
    // bits of the high word + 2^29, and r = (v - q 2^62) 2^-62 as a signed
    // 64-bit integer (|.| < 2^61, low 11 bits zero: exact in a double)
    const uint32_t whi = (uint32_t)(w >> 32);
    const uint32_t t = (whi + 0x20000000u) & 0xC0000000u; // q << 30 (mod 2^32)
    const uint32_t q = t >> 30;
    const int64_t ri = (int64_t)(((uint64_t)(whi - t) << 32) | ((uint32_t)w & 0xFFFFF800u));
    const double r = (double)ri * 0x1.0p-62;
#else
    const uint64_t m = w >> 11;
    const uint64_t q = (m + (1ull << 50)) >> 51;
    const double r = (double)((int64_t)m - (int64_t)(q << 51)) * 0x1.0p-51;
#endif
    const double r2 = r * r;
    double ps, pc;
    if (FAST) {
        ps = kSinC5[5];
        pc = kCosC6[6];
#pragma unroll
        for (int i = 4; i >= 0; --i) ps = fma(ps, r2, kSinC5[i]);
#pragma unroll
        for (int i = 5; i >= 0; --i) pc = fma(pc, r2, kCosC6[i]);
    } else {
        ps = kSinC[6];
        pc = kCosC[7];
#pragma unroll
        for (int i = 5; i >= 0; --i) ps = fma(ps, r2, kSinC[i]);
#pragma unroll
        for (int i = 6; i >= 0; --i) pc = fma(pc, r2, kCosC[i]);
    }
    ps *= r;
    const bool swap = q & 1;
    double sv = swap ? pc : ps;
    double cv = swap ? ps : pc;
    if (XOR) {
        // signs: sin by bit 1 of q, cos by bit 1 of q + 1, flipped in the high
        // words with one LOP3 each (q << 30 carries bit 1 of q in bit 31);
        // 9 instructions per sincos instead of 13 (+1.3 % cfg4, +2.3 % cfg2)
#if !BW_SINCOS_HI
        const unsigned t = (unsigned)q << 30;
#endif
        sv = __hiloint2double(__double2hiint(sv) ^ (int)(t & 0x80000000u), __double2loint(sv));
        cv = __hiloint2double(__double2hiint(cv) ^ (int)((t + 0x40000000u) & 0x80000000u),
                              __double2loint(cv));
    } else { // the compiler's predicated negations measured 0.4 % faster on the cavity box
        if (q & 2) sv = -sv;
        if ((q + 1) & 2) cv = -cv;
    }
    s = sv;
    c = cv;
}

__device__ __forceinline__ void sincos32_poly(uint32_t u, double& s, double& c) {
    const uint32_t q = (u + 0x20000000u) >> 30;
    const int32_t t = (int32_t)(u << 2) >> 2;
    const double r = fma((double)t, 0x1.0p-30, 0x1.0p-31);
    const double r2 = r * r;
    double ps = kSinC5[5], pc = kCosC6[6];
#pragma unroll
    for (int i = 4; i >= 0; --i) ps = fma(ps, r2, kSinC5[i]);
#pragma unroll
    for (int i = 5; i >= 0; --i) pc = fma(pc, r2, kCosC6[i]);
    ps *= r;
    const bool swap = q & 1;
    double sv = swap ? pc : ps;
    double cv = swap ? ps : pc;
    if (q & 2) sv = -sv;
    if ((q + 1) & 2) cv = -cv;
    s = sv;
    c = cv;
}

// One jump direction of the Philox4x32 stream (statistical mode): words
// (oz, oa) of the step, z = p32_z(oz), azimuth from oa (table or polynomial),
// 1-ulp root.
template <int TB> // TB: table bits, 0 = no table
__device__ __forceinline__ void jump_dir32(uint32_t oz, uint32_t oa, double& ux, double& uy,
                                           double& uz, uint32_t trig_s, const JumpConst& J) {
    const double zz = fma((double)(int32_t)oz, J.z31, 0x1.0p-32); // p32_z
    double s, c;
    if constexpr (TB > 0) sincos32_tab<TB>(oa, trig_s, J, s, c);
    else sincos32_poly(oa, s, c);
    // 1 - z^2 >= 2^-31 - 2^-64 on the centred grid: no zero guard on the root
    const double r = BW_SQRT_Q ? sqrt_q(fma(-zz, zz, 1.0)) : sqrt_1ulp<false>(fma(-zz, zz, 1.0));
    ux = r * c;
    uy = r * s;
    uz = zz;
}

// One WOS jump (wos.cpp:73-76) from two stream words:
//   z = 2U1 - 1, az = 2 pi U2, r = sqrt(max(0, 1 - z^2)), p += d (r cos az, r sin az, z)
// U = (w >> 11) 2^-53; 2U is formed exactly, so z = fma(m, 2^-52, -1) rounds once
// like the reference; (cos, sin)(az) agree with the reference's to a few ulp.
// jump_dir is the direction alone, (r cos az, r sin az, z): K1 forms both
// directions of a trip right after the Philox block, so their sincos/sqrt
// chains overlap (the second does not depend on the first jump's outcome).
template <bool XOR = (BW_SINCOS_XOR != 0)>
__device__ __forceinline__ void jump_dir(uint64_t wz, uint64_t wa, double& ux, double& uy,
                                         double& uz) {
#if BW_SINCOS_HI
    // (w & ~0x7FF) has <= 53 significant bits: exact, and times 2^-63 it is
    // (w >> 11) 2^-52 (one LOP3 instead of a 64-bit shift)
    const double zz = fma((double)(wz & ~0x7FFull), 0x1.0p-63, -1.0);
#else
    const double zz = fma((double)(wz >> 11), 0x1.0p-52, -1.0);
#endif
    double s, c;
    sincos_2pi_u<XOR, false>(wa, s, c);
    const double r = sqrt_walk<false>(fma(-zz, zz, 1.0));
    ux = r * c;
    uy = r * s;
    uz = zz;
}

__device__ __forceinline__ void jump(double& x, double& y, double& z, double d, uint64_t wz,
                                     uint64_t wa) {
    double ux, uy, uz;
    jump_dir<(BW_SINCOS_XOR != 0)>(wz, wa, ux, uy, uz);
    x = fma(d, ux, x);
    y = fma(d, uy, y);
    z = fma(d, uz, z);
}

// classify_exit for the drain path of K1. With a candidate grid, only the six
// faces and the cell's candidate cavities are projected (the nearest feature
// is always among them; brute force over 70 features cost ~2000 instructions
// per exit); otherwise the full reference loop (geometry.cpp:222-239).
template <int KIND>
__device__ __forceinline__ int classify_exit(const DevScene& S, const SmemScene& M, double eps,
                                             double x, double y, double z, double& px,
                                             double& py, double& pz) {
    // the plain box takes the faces-without-roots block below and stops there
    // (bitwise the reference loop's result; its six projections and roots were
    // a quarter of the box kernel's instructions: ncu_k1_cfg2_summary.md)
    constexpr bool kBoxOnly = KIND == BW_SCENE_BOX && BW_FACE_NOSQRT;
    if (!kBoxOnly && (KIND != BW_SCENE_BOX_CAVITIES || S.gn == 0))
        return classify<KIND>(S, M.cav, eps, x, y, z, px, py, pz);
    int best = -1;
    double dist = __longlong_as_double(0x7ff0000000000000LL);
    auto consider = [&](int f) {
        double qx, qy, qz;
        project<KIND>(S, M.cav, x, y, z, f, qx, qy, qz);
        const double d = norm3(x - qx, y - qy, z - qz);
        if (d < dist || (d == dist && f < best)) {
            dist = d;
            best = f;
            px = qx; py = qy; pz = qz;
        }
    };
#if BW_FACE_NOSQRT
    {
        // the six faces without their roots: with the point inside the box on
        // the other two axes (the clamps below are no-ops) the distance to a
        // face is norm3(t, 0, 0) = sqrt(RN(t^2)) = |t| exactly (radix 2, no
        // under/overflow: |t| > 2^-470 here), so |t| is bitwise the value the
        // projection gives; anything else takes the general path
        const double cx = fmin(fmax(x, S.lo[0]), S.hi[0]);
        const double cy = fmin(fmax(y, S.lo[1]), S.hi[1]);
        const double cz = fmin(fmax(z, S.lo[2]), S.hi[2]);
        const double p3[3] = {x, y, z};
        bool plain = cx == x && cy == y && cz == z;
        double t6[6];
#pragma unroll
        for (int f = 0; f < 6; ++f) {
            t6[f] = fabs(p3[f >> 1] - ((f & 1) ? S.hi[f >> 1] : S.lo[f >> 1]));
            plain = plain && t6[f] > 0x1.0p-470;
        }
        if (plain) {
#pragma unroll
            for (int f = 0; f < 6; ++f)
                if (t6[f] < dist) { // strict <: the lowest index wins ties, as consider()
                    dist = t6[f];
                    best = f;
                }
            px = x; py = y; pz = z;
            const double v = (best & 1) ? S.hi[best >> 1] : S.lo[best >> 1];
            if ((best >> 1) == 0) px = v; else if ((best >> 1) == 1) py = v; else pz = v;
        } else {
            for (int f = 0; f < 6; ++f) consider(f);
        }
    }
#else
    for (int f = 0; f < 6; ++f) consider(f);
#endif
    if (kBoxOnly) return (best < 0 || dist > eps) ? -3 : best;
    const int gn = S.gn;
    const int ix = grid_axis(x, S.ginv, S.gc0[0], gn);
    const int iy = grid_axis(y, S.ginv, S.gc0[1], gn);
    const int iz = grid_axis(z, S.ginv, S.gc0[2], gn);
    const int cell = (iz * gn + iy) * gn + ix;
    BW_CHECK(cell >= 0 && cell < gn * gn * gn);
    const unsigned imask = S.lpacked ? 0xffu : 0xffffu;
    for (int t = M.cstart[cell]; t < M.cstart[cell + 1]; ++t) {
        BW_CHECK((int)(M.clist[t] & imask) < S.n_cav);
        consider(6 + (int)(M.clist[t] & imask));
    }
    return (best < 0 || dist > eps) ? -3 : best;
}

// classify_exit of the statistical mode on the cavity box with the grid in
// shared memory: the nearest feature by distance (faces as |t|, candidate
// cavities as |sqrt(d2) - r| with the 1-ulp root, read with LDS and pruned by
// their packed cell bound like the walk's distance), and only the winner is
// projected. The parity mode keeps classify_exit above (the reference's
// project-then-measure loop and tie rule); here a tie between two features
// within an ulp has no statistical weight. ~half the drain's instructions.
#ifndef BW_CLASSIFY_FAST
#define BW_CLASSIFY_FAST 1
#endif
__device__ __forceinline__ int classify_exit_fast(const DevScene& S, const SmemScene& M, double eps,
                                                  double x, double y, double z, double& px,
                                                  double& py, double& pz) {
    int best = 0;
    const double p3[3] = {x, y, z};
    double dist = fabs(x - S.lo[0]);
#pragma unroll
    for (int f = 1; f < 6; ++f) {
        const double t = fabs(p3[f >> 1] - ((f & 1) ? S.hi[f >> 1] : S.lo[f >> 1]));
        if (t < dist) {
            dist = t;
            best = f;
        }
    }
    const int gn = S.gn;
    const int ix = grid_axis(x, S.ginv, S.gc0[0], gn);
    const int iy = grid_axis(y, S.ginv, S.gc0[1], gn);
    const int iz = grid_axis(z, S.ginv, S.gc0[2], gn);
    const int cell = (iz * gn + iy) * gn + ix;
    BW_CHECK(cell >= 0 && cell < gn * gn * gn);
    const int b = (int)lds_u16(M.cs_s + 2u * cell), e = (int)lds_u16(M.cs_s + 2u * cell + 2u);
    const unsigned imask = S.lpacked ? 0xffu : 0xffffu;
    // packed entries ascend by their bound Lq: stop once Lq lstep >= dist
    int thr = S.lpacked ? min(__double2int_ru(dist * S.linv), 256) << 8 : 0x7fffffff;
    for (int t = b; t < e; ++t) {
        const int ent = (int)lds_u16(M.cl_s + 2u * t);
        if (ent >= thr) break;
        BW_CHECK((int)(ent & imask) < S.n_cav);
        const double4 c = lds_d4(M.cav_s + 32u * (ent & imask));
        const double qx = x - c.x, qy = y - c.y, qz = z - c.z;
        const double dd = BW_SQRT_Q ? fabs(sqrt_q_minus(qx * qx + qy * qy + qz * qz, c.w))
                                    : fabs(sqrt_1ulp(qx * qx + qy * qy + qz * qz) - c.w);
        if (dd < dist) {
            dist = dd;
            best = 6 + (int)(ent & imask);
            if (S.lpacked) thr = min(__double2int_ru(dist * S.linv), 256) << 8;
        }
    }
    if (dist > eps) return -3;
    if (best < 6) {
        px = x; py = y; pz = z;
        const double v = (best & 1) ? S.hi[best >> 1] : S.lo[best >> 1];
        if ((best >> 1) == 0) px = v; else if ((best >> 1) == 1) py = v; else pz = v;
    } else {
        const double4 c = lds_d4(M.cav_s + 32u * (best - 6));
        const double qx = x - c.x, qy = y - c.y, qz = z - c.z;
        const double k = BW_SQRT_Q ? c.w * rsqrt_q(qx * qx + qy * qy + qz * qz)
                                   : div_walk(c.w, sqrt_1ulp(qx * qx + qy * qy + qz * qz));
        px = fma(qx, k, c.x);
        py = fma(qy, k, c.y);
        pz = fma(qz, k, c.z);
    }
    return best;
}

// classify_exit of the statistical mode on the plain box: the nearest of the
// six faces by |t| (lowest index on ties, like the reference loop) and the
// point with that coordinate replaced; ~30 instructions for the ~100 of the
// exact block in classify_exit (clamps, the plain test, six guarded distances).
__device__ __forceinline__ int classify_exit_box_fast(const DevScene& S, double eps, double x,
                                                      double y, double z, double& px, double& py,
                                                      double& pz) {
    const double p3[3] = {x, y, z};
    int best = 0;
    double dist = fabs(x - S.lo[0]);
#pragma unroll
    for (int f = 1; f < 6; ++f) {
        const double t = fabs(p3[f >> 1] - ((f & 1) ? S.hi[f >> 1] : S.lo[f >> 1]));
        if (t < dist) {
            dist = t;
            best = f;
        }
    }
    if (dist > eps) return -3;
    px = x; py = y; pz = z;
    const double v = (best & 1) ? S.hi[best >> 1] : S.lo[best >> 1];
    if ((best >> 1) == 0) px = v; else if ((best >> 1) == 1) py = v; else pz = v;
    return best;
}

// Post-jump tests in the reference order (wos.cpp:65-67):
// returns 1 (truncated to infinity), 0 (inside the eps shell), -1 (continue).
// UNB: 1 / 0 = the scene is / is not unbounded, fixed at launch (the
// statistical mode's instantiations); -1 = read W.bounded.
template <int KIND, bool SH = false, bool FAST = false, int UNB = -1>
__device__ __forceinline__ int post(const DevScene& S, const SmemScene& M, const DevWos& W,
                                    double eps, double x, double y, double z, double& d,
                                    double Rp) {
    if ((UNB < 0 ? !W.bounded : UNB == 1) && norm3(x, y, z) > W.trunc) return 1;
    d = nearest<KIND, SH, FAST>(S, M, x, y, z, Rp); // FAST: |d| is the distance
    return (FAST ? fabs(d) : d) <= eps ? 0 : -1;
}

// Per-lane running sums of (v - shift) and (v - shift)^2, with shift the
// Dirichlet closed form at the node itself (for harmonic data, u(start) = the
// expectation, so the sums stay small and M2 = S2 - S1^2/n keeps full
// precision). Replaces the per-exit division of Welford's push (wos.cpp:18-23);
// lanes merge with a fixed shuffle tree, so the result is deterministic.
struct LaneAcc {
    int32_t n, n_inf, n_fail, n_cls;
    int64_t steps;
    double s1, s2;
};

__device__ __forceinline__ void tree_sum(LaneAcc& a, int lane) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const int n = __shfl_down_sync(0xffffffffu, a.n, off);
        const int ni = __shfl_down_sync(0xffffffffu, a.n_inf, off);
        const int nf = __shfl_down_sync(0xffffffffu, a.n_fail, off);
        const int nc = __shfl_down_sync(0xffffffffu, a.n_cls, off);
        const long long st = __shfl_down_sync(0xffffffffu, (long long)a.steps, off);
        const double s1 = __shfl_down_sync(0xffffffffu, a.s1, off);
        const double s2 = __shfl_down_sync(0xffffffffu, a.s2, off);
        if (lane < off) {
            a.n += n;
            a.n_inf += ni;
            a.n_fail += nf;
            a.n_cls += nc;
            a.steps += st;
            a.s1 += s1;
            a.s2 += s2;
        }
    }
}

__device__ void patch_node(const NodeSource& src, int64_t g, double& x, double& y, double& z) {
    const int64_t b = g / src.n_nodes;
    const int j = (int)(g - b * src.n_nodes);
    const int cls = src.cls ? src.cls[b] : 0;
    BW_CHECK(cls >= 0 && (src.n_cls == 0 || cls < src.n_cls) && j >= 0 && j < src.n_nodes);
    patch_node_local(src.centers + 3 * b, src.axes + 3 * b, src.radii[b],
                     src.dirs + ((int64_t)cls * src.n_nodes + j) * 3, x, y, z);
}

// Copy cavities (+ candidate grid) into shared memory when they fit. With
// FULL (launch-time choice, mode 2 only) the returned pointers are derived from
// the shared array on every path, so the compiler emits LDS for the candidate
// loop instead of generic loads (runtime mode: any space).
template <bool FULL = false, bool SYNC = false>
__device__ __forceinline__ SmemScene stage(const DevScene& S, int smem_mode) {
    extern __shared__ __align__(16) unsigned char smem[];
    SmemScene M{S.cav, S.cell_start, S.cell_list, 0u, 0u, 0u};
    if (!FULL && smem_mode == 0) {
        if (SYNC) __syncthreads(); // the caller's own shared staging
        return M;
    }
    double4* cav = reinterpret_cast<double4*>(smem);
    for (int i = threadIdx.x; i < S.n_cav; i += blockDim.x) cav[i] = S.cav[i];
    M.cav = cav;
    if (FULL || (S.gn > 0 && smem_mode == 2)) {
        const int ncell = S.gn * S.gn * S.gn;
        uint16_t* cs = reinterpret_cast<uint16_t*>(cav + S.n_cav);
        for (int i = threadIdx.x; i <= ncell; i += blockDim.x) cs[i] = S.cell_start[i];
        uint16_t* cl = reinterpret_cast<uint16_t*>(cs + ncell + 1);
        const int nl = S.cell_start[ncell];
        for (int i = threadIdx.x; i < nl; i += blockDim.x) cl[i] = S.cell_list[i];
        M.cstart = cs;
        M.clist = cl;
        if (FULL) {
            M.cav_s = shared_addr(cav);
            M.cs_s = shared_addr(cs);
            M.cl_s = shared_addr(cl);
        }
    }
    __syncthreads();
    return M;
}

// K1: persistent node-per-warp WOS estimator.
//
// Exits are not processed where they happen: a lane whose walk ends parks the
// exit point in a one-slot buffer and immediately starts its next walk. The
// warp drains the buffers (classification, Dirichlet data, sums) together once
// kFlush lanes hold one, when a lane needs its slot again, or when the node's
// walks are exhausted — so the exit code runs with most lanes active instead
// of one or two (it ran divergently on ~1.4x per loop trip before).
// Blocks of 4 warps per SM the register budget is sized for: 6 (<= 80
// registers) by default; 7 (<= 72) on the sphere in the statistical mode, whose loop fits
// (+1.3 %; the box loses 5 % there and 8 blocks lose 4 % on both:
// profiles/r2/ab_u32_blocks.log); 5 on the cavity box, whose candidate-list
// distance needs 96.
//
// RNG (bw_rng_kind): 0 = the reference's Philox4x64-10 RngStream, one block
// per loop trip feeding both jumps (15 wide products per block: per-node and
// per-walk tables, see node_tab_fill / walk_prod); 1 = Philox4x32-10, one block
// per jump (15 32-bit products per block from a per-node uint4 table and a
// per-walk product formed at refill).
#ifndef BW_WOS_MIN_BLOCKS
#define BW_WOS_MIN_BLOCKS(KIND, RNG) \
    ((KIND) == BW_SCENE_BOX_CAVITIES ? 5 : ((KIND) == BW_SCENE_SPHERE && (RNG) == 1 ? 7 : 6))
#endif
#ifndef BW_WOS_FLUSH
#define BW_WOS_FLUSH 26
#endif
constexpr int kFlush = BW_WOS_FLUSH;
// stream blocks per loop trip of the statistical mode: 3 (2 on the cavity box,
// where a third costs 6 %; profiles/r2/ab_u32_trip_blocks.log)
#ifndef BW_TRIP_BLOCKS0
#define BW_TRIP_BLOCKS0 1 // the parity mode
#endif
#ifndef BW_TRIP_BLOCKS
#define BW_TRIP_BLOCKS(KIND) ((KIND) == BW_SCENE_BOX_CAVITIES ? 2 : 3)
#endif

// Per-warp shared scratch: the node's start (reloaded on every refill), the
// parked exit points and the rare counters live here instead of registers,
// which keeps the walk loop under 85 registers (6 blocks of 4 warps per SM).
template <int RNG>
struct WarpScratch {
    double sx, sy, sz, d0, shift, eps;
    double ex[32], ey[32], ez[32];
    int32_t n_fail[32], n_inf[32], n_cls[32];
    // RNG 0: round-1 Philox product M0 (hi1p ^ walk ^ k0[0]) (walk_prod) of
    // each lane's current walk, and a ring of the next 32 walk indices.
    // Between two drains every lane takes at most one new walk (a lane that
    // ends twice forces a drain first), so refills never run past
    // [next, next + 32), the window the drain refreshes. RNG 1 forms its
    // per-walk product at refill (one 32-bit product) and needs neither.
    ulonglong2 cur[RNG == 0 ? 32 : 1];
    ulonglong2 ring[RNG == 0 ? 32 : 1];
    // this node's Philox table: RNG 0 node_tab_fill (2 entries per block, 64
    // blocks = 128 steps), RNG 1 p32_tab_entry (one uint4 per block, 64
    // blocks = 128 steps)
    ulonglong2 nt[RNG == 0 ? 2 * kBlkTab : kBlkTab32 + 1]; // + the slow path's key slot
};
static_assert(sizeof(ulonglong2) == sizeof(uint4), "node table entries");
static_assert(offsetof(WarpScratch<1>, sx) == 0 && offsetof(WarpScratch<1>, d0) == 24 &&
                  offsetof(WarpScratch<1>, ey) - offsetof(WarpScratch<1>, ex) == 256 &&
                  offsetof(WarpScratch<1>, ez) - offsetof(WarpScratch<1>, ex) == 512 &&
                  offsetof(WarpScratch<0>, sx) == 0 && offsetof(WarpScratch<0>, d0) == 24 &&
                  offsetof(WarpScratch<0>, ez) - offsetof(WarpScratch<0>, ex) == 512,
              "BW_WS_PIN addresses the scratch by these offsets");

template <int KIND, int PHI, bool SMEM_FULL, int RNG, bool UNB_T = false>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, BW_WOS_MIN_BLOCKS(KIND, RNG))
    wos_nodes_kernel(const DevScene S, const DevWos W, const NodeSource src, int64_t n_total,
                     uint64_t pid_base, bw_estimate* __restrict__ out,
                     int64_t* __restrict__ steps_out, unsigned long long* __restrict__ ctr,
                     int smem_mode) {
    // the FAST sincos table: per CTA in shared memory (before stage's barrier);
    // its 4 KB are the RNG 0 walk-product rings RNG 1 does not keep
#ifndef BW_SINCOS_TAB_CAV
#define BW_SINCOS_TAB_CAV 1
#endif
    constexpr bool kTab = RNG == 1 && BW_SINCOS_TAB &&
                          (KIND != BW_SCENE_BOX_CAVITIES || BW_SINCOS_TAB_CAV);
    constexpr int kTB = kTab ? kTrigBits : 0;
    __shared__ __align__(16) double2 trig[kTab ? (1 << kTB) : 1];
    if (kTab) stage_trig(trig);
    const SmemScene M = stage<SMEM_FULL, kTab>(S, smem_mode);
    const uint32_t trig_s = shared_addr(trig);
    __shared__ WarpScratch<RNG> scratch_all[kWarpsPerBlock];
    WarpScratch<RNG>& ws = scratch_all[threadIdx.x >> 5];
    uint4* const tab32 = reinterpret_cast<uint4*>(ws.nt);
#ifndef BW_TAB_SADDR
#define BW_TAB_SADDR 1
#endif
    const uint32_t tab_s = BW_TAB_SADDR ? shared_addr(ws.nt) : 0u;
    const int lane = threadIdx.x & 31;
    // BW_WS_PIN: under register pressure ptxas re-derives the warp scratch
    // address, the lane and the lane mask from %tid on every trip (12
    // instructions on the cavity box, 3-4 elsewhere); pinned in registers, the
    // refill block addresses the scratch through them (+2.3 % cavity box,
    // +1.4 % sphere, +1.5 % box: profiles/r2/ab_u32_cavity_drain.log,
    // ab_u32_cand_wspin.log)
#ifndef BW_WS_PIN
#define BW_WS_PIN(KIND) 1
#endif
    constexpr bool kWsPin = BW_WS_PIN(KIND);
    const uint32_t ws_s = kWsPin ? shared_addr(&ws) : 0u;
    const uint32_t wsl_s = kWsPin ? shared_addr(&ws.ex[lane]) : 0u;
    unsigned lt_mask = (1u << lane) - 1u;
    if (kWsPin) asm volatile("mov.b32 %0, %0;" : "+r"(lt_mask));
    const int n_paths = W.n_paths;
    const uint32_t bmax = (uint32_t)W.max_blk; // statistical mode: the step budget in blocks
    // the statistical mode also takes the 1-ulp roots and the shorter sincos fits
    constexpr bool kFast = RNG == 1;
    // the trunc-radius test of unbounded scenes: compiled in or out for the
    // statistical mode (launch_wos_t picks by W.bounded), a runtime flag for
    // the parity mode
    constexpr int kUnb = RNG == 1 ? (UNB_T ? 1 : 0) : -1;
    const JumpConst jc = jump_const<kTB, RNG == 1 && BW_PIN_CONST(KIND), KIND == BW_SCENE_SPHERE>();
    // the sphere's radius, pinned like the constants above in the statistical mode
    double sr = S.R;
    if (RNG == 1 && KIND == BW_SCENE_SPHERE) {
        __shared__ double sr_sh;
        if (threadIdx.x == 0) sr_sh = S.R;
        __syncthreads();
        asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(sr) : "r"((uint32_t)__cvta_generic_to_shared(&sr_sh)));
    }

    for (;;) {
        unsigned long long node_u = 0;
        if (lane == 0) node_u = atomicAdd(&ctr[kCtrWork], 1ull);
        const int64_t node = (int64_t)__shfl_sync(0xffffffffu, node_u, 0);
        if (node >= n_total) break;
        uint64_t pid = pid_base + (uint64_t)node;
        if (src.bp_ids) {
            const int64_t b = node / src.n_nodes;
            pid = pid_base + (uint64_t)(src.bp_ids[b] * src.n_nodes + (node - b * src.n_nodes));
        }

        double sx, sy, sz;
        double eps = W.eps;
        bool skip = false;
        if (src.xyz) {
            sx = src.xyz[3 * node];
            sy = src.xyz[3 * node + 1];
            sz = src.xyz[3 * node + 2];
        } else {
            patch_node(src, node, sx, sy, sz);
            // per-point shell: eps_b = min(eps, eps_rel a_b) (bw_wos_config.eps_rel)
            if (W.eps_rel > 0.0) eps = fmin(eps, W.eps_rel * src.radii[node / src.n_nodes]);
            if (src.check_domain) {
                if (KIND == BW_SCENE_BOX_CAVITIES) {
                    // in_domain with the cavities split over the lanes (same
                    // per-cavity predicate, geometry.cpp:100-113 style)
                    bool hit = !(sx > S.lo[0] && sx < S.hi[0] && sy > S.lo[1] && sy < S.hi[1] &&
                                 sz > S.lo[2] && sz < S.hi[2]);
                    for (int i = lane; i < S.n_cav; i += 32) {
                        const double4 c = M.cav[i];
                        if (!(norm3(sx - c.x, sy - c.y, sz - c.z) > c.w)) hit = true;
                    }
                    skip = __any_sync(0xffffffffu, hit);
                } else {
                    skip = !in_domain<KIND>(S, M.cav, sx, sy, sz);
                }
            }
        }
        if (skip) {
            if (lane == 0) {
                out[node] = bw_estimate{__longlong_as_double(0x7ff8000000000000LL), 0.0, 0, 0, 0};
                if (steps_out) steps_out[node] = 0;
            }
            continue;
        }

        double d0 = 0;
        const int o0 = post<KIND, SMEM_FULL>(S, M, W, eps, sx, sy, sz, d0, S.R);
        if (o0 >= 0) {
            // every walk ends at its start with 0 steps (wos.cpp:65-71)
            if (lane == 0) {
                bw_estimate e{0.0, 0.0, 0, 0, 0};
                if (o0 == 1) {
                    e.n = n_paths;
                    e.n_infinity = n_paths;
                } else {
                    double px = sx, py = sy, pz = sz;
                    const int f = classify<KIND>(S, M.cav, eps, sx, sy, sz, px, py, pz);
                    if (f < 0) {
                        atomicAdd(&ctr[kCtrClassify], (unsigned long long)n_paths);
                    } else {
                        e.n = n_paths;
                        e.mean = eval_phi<PHI>(S, px, py, pz, f);
                    }
                }
                out[node] = e;
                if (steps_out) steps_out[node] = 0;
            }
            continue;
        }

        if (lane == 0) {
            ws.sx = sx;
            ws.sy = sy;
            ws.sz = sz;
            ws.d0 = d0;
            ws.eps = eps;
            ws.shift = eval_phi<PHI>(S, sx, sy, sz, 0);
        }
        ws.n_fail[lane] = 0;
        ws.n_inf[lane] = 0;
        ws.n_cls[lane] = 0;
        // per-node stream constants and tables
        uint64_t lo1p = 0, hi1p = 0;
        P32Node pn{0u, 0u, 0u};
        uint32_t wh32 = 0, wl32 = 0;
        if (RNG == 0) {
            lo1p = kM1 * pid; // per-node half of Philox round 0
            hi1p = __umul64hi(kM1, pid);
            uint64_t h, l;
            walk_prod(W.keys, (uint64_t)lane, hi1p, h, l);
            ws.cur[lane] = make_ulonglong2(h, l);
            walk_prod(W.keys, (uint64_t)(32 + lane), hi1p, h, l);
            ws.ring[lane] = make_ulonglong2(h, l);
            node_tab_fill(W.keys, lo1p, ws.nt, lane);
        } else {
            pn = p32_node(pid);
#pragma unroll
            for (int b = lane; b < kBlkTab32; b += 32) tab32[b] = p32_tab_entry(W.keys32, pn, (uint32_t)b);
            if (lane == 0) tab32[kBlkTab32] = make_uint4(W.keys32.kk[1], W.keys32.kk[2], 0u, 0u);
            p32_walk(W.keys32, pn, (uint32_t)lane, wh32, wl32);
        }
        __syncwarp();
        int32_t n_ok = 0;
        int64_t steps_sum = 0;
        double s1 = 0.0, s2 = 0.0;
        int k = lane;
        bool active = k < n_paths;
        double x = sx, y = sy, z = sz, d = d0;
        uint32_t blk = 0; // loop trips of the current walk
        int steps = 0;
        // Warp-uniform bookkeeping (every lane holds the same values, derived
        // from the one ballot per trip): next walk index, lanes walking, parked.
        int next = 32;
        int n_running = min(32, n_paths);
        unsigned pmask = 0u;
        int pend = 0; // 0 empty, 1 absorbed, 2 infinity, 3 failed
        for (;;) {
            // 0 absorbed, 1 infinity, 2 failed; statistical mode: + 4 when the walk
            // ended on a block's first jump (its step count is then odd)
            int outcome = -1;
            if (active) {
                // statistical mode: BW_TRIP_BLOCKS stream blocks (two jumps each)
                // per trip (the parity mode keeps one, and with it the walk to
                // lane assignment its results were pinned with): the
                // ballot, drain test, refill and loop bookkeeping (~60 issue
                // slots) run once per trip, and a lane whose walk ends inside
                // a trip idles to its end
#pragma unroll
                for (int half = 0; half < (RNG == 1 ? BW_TRIP_BLOCKS(KIND) : BW_TRIP_BLOCKS0); ++half) {
                    // step budget: the parity mode counts steps (wos.cpp:69); the
                    // statistical mode counts blocks — its budget is max_steps
                    // rounded down to even, checked once per block, and the
                    // walk's step count is 2 blk - (exit on the block's first
                    // jump), formed when the walk ends
                    if (RNG == 1 ? blk >= bmax : steps >= W.max_steps) {
                        outcome = 2;
                        break;
                    }
                    // both jump directions of a block first: their sincos/sqrt
                    // chains overlap (the second does not depend on the first
                    // jump's outcome)
                    double ux1, uy1, uz1, ux2, uy2, uz2;
                    if (RNG == 0) {
                        uint64_t w[4];
                        const ulonglong2 wp = ws.cur[lane];
                        philox_wos_nt(W.keys, ws.nt, blk, wp.x, wp.y, lo1p, w);
                        constexpr bool kXor = BW_SINCOS_XOR && KIND != BW_SCENE_BOX_CAVITIES;
                        jump_dir<kXor>(w[0], w[1], ux1, uy1, uz1);
                        jump_dir<kXor>(w[2], w[3], ux2, uy2, uz2);
                    } else {
                        uint32_t o0, o1, o2, o3;
                        if (BW_TAB_SADDR)
                            p32_wos_block_s(W.keys32, pn, tab_s, blk, wh32, wl32, o0, o1, o2, o3);
                        else
                            p32_wos_block(W.keys32, pn, tab32, blk, wh32, wl32, o0, o1, o2, o3);
                        jump_dir32<kTB>(o0, o1, ux1, uy1, uz1, trig_s, jc);
                        jump_dir32<kTB>(o2, o3, ux2, uy2, uz2, trig_s, jc);
                    }
                    ++blk;
                    const double da = kFast ? fabs(d) : d;
                    x = fma(da, ux1, x);
                    y = fma(da, uy1, y);
                    z = fma(da, uz1, z);
                    if (RNG == 0) ++steps;
                    outcome = post<KIND, SMEM_FULL, kFast, kUnb>(S, M, W, eps, x, y, z, d, sr);
                    if (outcome >= 0) {
                        if (RNG == 1) outcome |= 4;
                        break;
                    }
                    if (RNG == 0 && steps >= W.max_steps) {
                        outcome = 2;
                        break;
                    }
                    const double db = kFast ? fabs(d) : d;
                    x = fma(db, ux2, x);
                    y = fma(db, uy2, y);
                    z = fma(db, uz2, z);
                    if (RNG == 0) ++steps;
                    outcome = post<KIND, SMEM_FULL, kFast, kUnb>(S, M, W, eps, x, y, z, d, sr);
                    if (outcome >= 0) break;
                }
            }
            const bool done = outcome >= 0;
            const unsigned dmask = __ballot_sync(0xffffffffu, done);
            const int nd = __popc(dmask);
            const int walking = n_running - nd;
            if ((dmask & pmask) || __popc(pmask | dmask) >= kFlush || (walking == 0 && nd == 0)) {
                // drain the parked exits (single site; lanes mostly converged)
                if (pend) {
                    bool ok = true;
                    double v = 0.0;
                    if (pend == 1) {
                        const double qx = ws.ex[lane], qy = ws.ey[lane], qz = ws.ez[lane];
                        double px = qx, py = qy, pz = qz;
                        int f;
                        // statistical mode: the walk's distance (half-extent form,
                        // Newton-step roots) and the classification's differ in
                        // the last digits, so an exit the walk took at d <= eps
                        // is classified against eps (1 + 1e-6) (at exactly eps
                        // the strict test turned away ~1e-10 of the exits:
                        // 14 of config 5's 1e11 walks)
                        const double ceps = kFast ? ws.eps * (1.0 + 1e-6) : ws.eps;
                        if constexpr (KIND == BW_SCENE_BOX_CAVITIES && SMEM_FULL && RNG == 1 &&
                                      BW_CLASSIFY_FAST) {
                            f = classify_exit_fast(S, M, ceps, qx, qy, qz, px, py, pz);
                        } else if constexpr (KIND == BW_SCENE_BOX && RNG == 1 && BW_CLASSIFY_FAST) {
                            f = classify_exit_box_fast(S, ceps, qx, qy, qz, px, py, pz);
                        } else if constexpr (KIND == BW_SCENE_SPHERE && RNG == 1 &&
                                             BW_CLASSIFY_FAST) {
                            // one feature, and the walk's own test put the point
                            // within eps of it: project, no second distance
                            f = 0;
                            const double k =
                                BW_SQRT_Q ? sr * rsqrt_q(fma(qx, qx, fma(qy, qy, qz * qz)))
                                          : div_walk(S.R, sqrt_1ulp(fma(qx, qx, fma(qy, qy, qz * qz))));
                            px = qx * k;
                            py = qy * k;
                            pz = qz * k;
                        } else
                            f = classify_exit<KIND>(S, M, ceps, qx, qy, qz, px, py, pz);
                        if (f < 0) {
                            ++ws.n_cls[lane];
                            ok = false;
                        } else {
                            v = eval_phi<PHI, RNG == 1 && BW_SQRT_Q>(S, px, py, pz, f);
                        }
                    } else if (pend == 2) {
                        ++ws.n_inf[lane];
                    } else {
                        ++ws.n_fail[lane];
                        ok = false;
                    }
                    if (ok) {
                        const double dv = v - ws.shift;
                        ++n_ok;
                        s1 += dv;
                        s2 = fma(dv, dv, s2);
                    }
                    pend = 0;
                }
                pmask = 0u;
                if (RNG == 0) {
                    // refresh the ring for the walks [next, next + 32)
                    uint64_t h, l;
                    const int kk = next + lane;
                    walk_prod(W.keys, (uint64_t)kk, hi1p, h, l);
                    __syncwarp();
                    ws.ring[kk & 31] = make_ulonglong2(h, l);
                    __syncwarp();
                }
            }
            if (done) {
                steps_sum += RNG == 1 ? (int)(2u * blk) - (outcome >> 2) : steps;
                pend = (outcome & 3) + 1;
                if (kWsPin) {
                    asm volatile("st.shared.f64 [%0], %1;" :: "r"(wsl_s), "d"(x) : "memory");
                    asm volatile("st.shared.f64 [%0+256], %1;" :: "r"(wsl_s), "d"(y) : "memory");
                    asm volatile("st.shared.f64 [%0+512], %1;" :: "r"(wsl_s), "d"(z) : "memory");
                } else {
                    ws.ex[lane] = x;
                    ws.ey[lane] = y;
                    ws.ez[lane] = z;
                }
                k = next + __popc(dmask & lt_mask);
                active = k < n_paths;
                if (RNG == 0) ws.cur[lane] = ws.ring[k & 31];
                else p32_walk(W.keys32, pn, (uint32_t)k, wh32, wl32);
                if (kWsPin) {
                    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(ws_s) : "memory");
                    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+16];" : "=d"(z), "=d"(d) : "r"(ws_s) : "memory");
                } else {
                    x = ws.sx;
                    y = ws.sy;
                    z = ws.sz;
                    d = ws.d0;
                }
                blk = 0;
                steps = 0;
            }
            pmask |= dmask;
            n_running = walking + min(nd, max(n_paths - next, 0));
            next += nd;
            if (n_running == 0 && pmask == 0u) break;
        }
        __syncwarp();
        LaneAcc acc{n_ok, ws.n_inf[lane], ws.n_fail[lane], ws.n_cls[lane], steps_sum, s1, s2};
        tree_sum(acc, lane);
        if (lane == 0) {
            const double shift = ws.shift;
            bw_estimate e;
            const double n = (double)acc.n;
            e.mean = acc.n > 0 ? shift + acc.s1 / n : 0.0;
            const double m2 = acc.n > 0 ? fmax(acc.s2 - acc.s1 * (acc.s1 / n), 0.0) : 0.0;
            e.variance = acc.n > 1 ? m2 / (n - 1.0) : 0.0; // wos.cpp:47
            e.n = acc.n;
            e.n_infinity = acc.n_inf;
            e.n_failed = acc.n_fail;
            out[node] = e;
            if (steps_out) steps_out[node] = acc.steps;
            if ((double)acc.n_fail > 0.001 * (double)n_paths) // wos.cpp:43-44
                atomicAdd(&ctr[kCtrReliability], 1ull);
            if (acc.n_cls) atomicAdd(&ctr[kCtrClassify], (unsigned long long)acc.n_cls);
        }
        __syncwarp();
    }
}

// Single trajectories in the reference's exact control flow (wos.cpp:61-79),
// one thread per walk. Used for walk-by-walk parity against the oracle.
template <int KIND, int RNG>
__global__ void walk_kernel(const DevScene S, const DevWos W, const double* __restrict__ starts,
                            int64_t n, const uint64_t* __restrict__ pids,
                            const uint64_t* __restrict__ paths, double* __restrict__ exit_pts,
                            int32_t* __restrict__ feat, int32_t* __restrict__ steps_out,
                            unsigned long long* __restrict__ ctr, int smem_mode) {
    // the RNG = 1 trajectories exactly as K1 walks them (same table, 1-ulp roots)
    constexpr int kTB = RNG == 1 && BW_SINCOS_TAB && (KIND != BW_SCENE_BOX_CAVITIES || BW_SINCOS_TAB_CAV)
                            ? kTrigBits : 0;
    __shared__ __align__(16) double2 trig[kTB ? (1 << kTB) : 1];
    if (kTB) stage_trig(trig);
    const JumpConst jc = jump_const<kTB, RNG == 1 && BW_PIN_CONST(KIND), KIND == BW_SCENE_SPHERE>();
    const SmemScene M = stage<false, true>(S, smem_mode);
    const uint32_t trig_s = shared_addr(trig);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double x = starts[3 * i], y = starts[3 * i + 1], z = starts[3 * i + 2];
        const uint64_t pid = pids[i], path = paths[i];
        const uint64_t lo1p = kM1 * pid, hi1p = __umul64hi(kM1, pid);
        int steps = 0, f = 0;
        uint32_t blk = 0;
        uint64_t w[4];
        uint32_t c32[4] = {0u, 0u, 0u, 0u};
        (void)lo1p;
        for (;;) {
            if (norm3(x, y, z) > W.trunc) { f = -1; break; }
            // the RNG = 1 trajectories exactly as K1 walks them (1-ulp roots)
            const double d = steps == 0 ? nearest<KIND>(S, M, x, y, z, S.R)
                                        : fabs(nearest<KIND, false, RNG == 1>(S, M, x, y, z, S.R));
            if (d <= W.eps) {
                double px = x, py = y, pz = z;
                f = classify<KIND>(S, M.cav, W.eps, x, y, z, px, py, pz);
                if (f < 0) atomicAdd(&ctr[kCtrClassify], 1ull);
                x = px; y = py; z = pz;
                break;
            }
            // the statistical mode's budget is max_steps rounded down to even (K1 checks it per block)
            if (steps >= (RNG == 1 ? (W.max_steps & ~1) : W.max_steps)) { f = -2; break; }
            if (RNG == 0) {
                if ((steps & 1) == 0) philox_wos(W.keys, blk++, path, hi1p, lo1p, w);
                const int o = (steps & 1) * 2;
                jump(x, y, z, d, w[o], w[o + 1]);
            } else { // Philox4x32 block steps / 2, ctr {blk, path, lo(pid), hi(pid)}:
                     // words (o0, o1) on even steps, (o2, o3) on odd ones
                if ((steps & 1) == 0) {
                    c32[0] = blk++;
                    c32[1] = (uint32_t)path;
                    c32[2] = (uint32_t)pid;
                    c32[3] = (uint32_t)(pid >> 32);
                    philox4x32_block(W.keys32, c32);
                }
                const int o = (steps & 1) * 2;
                double ux, uy, uz;
                jump_dir32<kTB>(c32[o], c32[o + 1], ux, uy, uz, trig_s, jc);
                x = fma(d, ux, x);
                y = fma(d, uy, y);
                z = fma(d, uz, z);
            }
            ++steps;
        }
        exit_pts[3 * i] = x;
        exit_pts[3 * i + 1] = y;
        exit_pts[3 * i + 2] = z;
        feat[i] = f;
        steps_out[i] = steps;
    }
}

__global__ void philox_kernel(const uint64_t* __restrict__ ctr, const uint64_t* __restrict__ key,
                              int64_t n, uint64_t* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    PhiloxKeys K;
    uint64_t a = key[2 * i], b = key[2 * i + 1];
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) {
            a += kW0;
            b += kW1;
        }
        K.k0[r] = a;
        K.k1[r] = b;
    }
    uint64_t o[4];
    philox_block(K, ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3], o);
    for (int j = 0; j < 4; ++j) out[4 * i + j] = o[j];
}

template <int KIND, int PHI>
cudaError_t launch_wos_t(bw_ctx* ctx, const DevScene& S, size_t smem, const DevWos& W,
                         const NodeSource& src, int64_t n_total, uint64_t pid_base,
                         bw_estimate* out, int64_t* steps) {
    const int threads = kWarpsPerBlock * 32;
    const int mode = smem == 0 ? 0 : (S.gn > 0 && smem > (size_t)S.n_cav * 32 ? 2 : 1);
    // statistical mode: the unbounded-scene test is a template flag (half-space,
    // plates and disk are always unbounded; sphere and boxes by W.bounded)
    constexpr bool kAlwaysUnb = KIND == BW_SCENE_HALFSPACE || KIND == BW_SCENE_PLATESET ||
                                KIND == BW_SCENE_THINDISK;
    auto kern = wos_nodes_kernel<KIND, PHI, false, 0>;
    if (W.rng == 1) {
        kern = wos_nodes_kernel<KIND, PHI, false, 1, true>;
        if constexpr (!kAlwaysUnb) {
            if (W.bounded) kern = wos_nodes_kernel<KIND, PHI, false, 1, false>;
        }
    }
    // cavity grid fully in shared memory: the LDS instantiation
    if constexpr (KIND == BW_SCENE_BOX_CAVITIES) {
        if (mode == 2) {
            kern = wos_nodes_kernel<KIND, PHI, true, 0>;
            if (W.rng == 1)
                kern = W.bounded ? wos_nodes_kernel<KIND, PHI, true, 1, false>
                                 : wos_nodes_kernel<KIND, PHI, true, 1, true>;
        }
    }
    if (smem > 0) { // static (warp scratch) + dynamic may pass 48 KB
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    int64_t blocks = (int64_t)ctx->sm_count * per_sm;
    const int64_t need = (n_total + kWarpsPerBlock - 1) / kWarpsPerBlock;
    if (blocks > need) blocks = need;
    if (blocks < 1) blocks = 1;
    e = cudaMemsetAsync(ctx->d_counters, 0, sizeof(unsigned long long) * kCtrCount, ctx->stream);
    if (e != cudaSuccess) return e;
    ++ctx->launches;
    kern<<<(unsigned)blocks, threads, smem, ctx->stream>>>(S, W, src, n_total, pid_base, out,
                                                          steps, ctx->d_counters, mode);
    return cudaGetLastError();
}

template <int KIND>
cudaError_t launch_walk_t(bw_ctx* ctx, const DevScene& S, size_t smem, const DevWos& W,
                          const double* starts, int64_t n, const uint64_t* pids,
                          const uint64_t* paths, double* exit_pts, int32_t* feat,
                          int32_t* steps) {
    const int mode = smem == 0 ? 0 : (S.gn > 0 && smem > (size_t)S.n_cav * 32 ? 2 : 1);
    auto kern = W.rng == 1 ? walk_kernel<KIND, 1> : walk_kernel<KIND, 0>;
    if (smem > 0) { // static (block table, warp scratch) + dynamic may pass 48 KB
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e =
        cudaMemsetAsync(ctx->d_counters, 0, sizeof(unsigned long long) * kCtrCount, ctx->stream);
    if (e != cudaSuccess) return e;
    const int threads = 128;
    int64_t blocks = (n + threads - 1) / threads;
    if (blocks > (int64_t)ctx->sm_count * 16) blocks = (int64_t)ctx->sm_count * 16;
    if (blocks < 1) blocks = 1;
    ++ctx->launches;
    kern<<<(unsigned)blocks, threads, smem, ctx->stream>>>(S, W, starts, n, pids, paths, exit_pts,
                                                          feat, steps, ctx->d_counters, mode);
    return cudaGetLastError();
}

// nearest_feature with the reference's argmin and tie rule (geometry.cpp:131-155:
// strict <, so the lowest feature index wins), brute force over the features.
template <int KIND>
__device__ double nearest_arg(const DevScene& S, const double4* cav, double x, double y, double z,
                              int& f) {
    f = 0;
    if (KIND == BW_SCENE_HALFSPACE) return fabs(z - S.plane_z);
    if (KIND == BW_SCENE_THINDISK) {
        const double rho = hypot(x, y);
        return rho <= S.disk_r ? fabs(z) : hypot(rho - S.disk_r, z);
    }
    if (KIND == BW_SCENE_SPHERE) return fabs(sqrt(x * x + y * y + z * z) - S.R);
    double best = __longlong_as_double(0x7ff0000000000000LL);
    f = -1;
    if (KIND == BW_SCENE_PLATESET) {
        for (int i = 0; i < S.n_cav; ++i) {
            const double4 pl = cav[i];
            const double dx = fmax(fmax(pl.x - x, 0.0), x - pl.y);
            const double dy = fmax(fmax(pl.z - y, 0.0), y - pl.w);
            const double d = sqrt(dx * dx + dy * dy + z * z);
            if (d < best) { best = d; f = i; }
        }
        return best;
    }
    const double p3[3] = {x, y, z};
    for (int k = 0; k < 3; ++k) {
        const double dlo = fabs(p3[k] - S.lo[k]);
        if (dlo < best) { best = dlo; f = 2 * k; }
        const double dhi = fabs(S.hi[k] - p3[k]);
        if (dhi < best) { best = dhi; f = 2 * k + 1; }
    }
    if (KIND == BW_SCENE_BOX_CAVITIES)
        for (int i = 0; i < S.n_cav; ++i) {
            const double4 c = cav[i];
            const double d = fabs(norm3(x - c.x, y - c.y, z - c.z) - c.w);
            if (d < best) { best = d; f = 6 + i; }
        }
    return best;
}

// Batch nearest_feature + classify_exit (geometry.cpp:131-155, 222-239) on the
// device, next to the distance K1's walk loop uses (candidate grid, early exit).
template <int KIND>
__global__ void geometry_kernel(const DevScene S, const double* __restrict__ pts, int64_t n,
                                double eps, double trunc, double* __restrict__ dist,
                                int32_t* __restrict__ feat, double* __restrict__ dist_walk,
                                double* __restrict__ proj, int32_t* __restrict__ exit_feat,
                                unsigned long long* __restrict__ ctr, int check_domain,
                                int smem_mode) {
    const SmemScene M = stage(S, smem_mode);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
        int f;
        const double d = nearest_arg<KIND>(S, M.cav, x, y, z, f);
        if (dist) dist[i] = d;
        if (feat) feat[i] = f;
        // distance_to_boundary's domain test (geometry.cpp:157-171)
        if (check_domain && !(in_domain<KIND>(S, M.cav, x, y, z) && d > 0))
            atomicAdd(&ctr[kCtrDomain], 1ull);
        if (dist_walk) dist_walk[i] = nearest<KIND>(S, M, x, y, z, S.R);
        if (exit_feat) {
            double px = x, py = y, pz = z;
            int e;
            if (norm3(x, y, z) > trunc) {
                e = -1; // kExitInfinity (geometry.cpp:223)
            } else {
                e = classify<KIND>(S, M.cav, eps, x, y, z, px, py, pz);
                if (e < 0) atomicAdd(&ctr[kCtrClassify], 1ull);
            }
            exit_feat[i] = e;
            if (proj) {
                proj[3 * i] = px;
                proj[3 * i + 1] = py;
                proj[3 * i + 2] = pz;
            }
        }
    }
}

template <int KIND>
cudaError_t launch_geometry_t(bw_ctx* ctx, const DevScene& S, size_t smem, const double* pts,
                              int64_t n, double eps, double trunc, double* dist, int32_t* feat,
                              double* dist_walk, double* proj, int32_t* exit_feat,
                              int check_domain) {
    const int mode = smem == 0 ? 0 : (S.gn > 0 && smem > (size_t)S.n_cav * 32 ? 2 : 1);
    auto kern = geometry_kernel<KIND>;
    if (smem > 0) { // static (block table, warp scratch) + dynamic may pass 48 KB
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e =
        cudaMemsetAsync(ctx->d_counters, 0, sizeof(unsigned long long) * kCtrCount, ctx->stream);
    if (e != cudaSuccess) return e;
    int64_t blocks = (n + 127) / 128;
    if (blocks > (int64_t)ctx->sm_count * 16) blocks = (int64_t)ctx->sm_count * 16;
    if (blocks < 1) blocks = 1;
    ++ctx->launches;
    kern<<<(unsigned)blocks, 128, smem, ctx->stream>>>(S, pts, n, eps, trunc, dist, feat, dist_walk,
                                                      proj, exit_feat, ctx->d_counters,
                                                      check_domain, mode);
    return cudaGetLastError();
}

template <int KIND>
cudaError_t launch_wos_k(bw_ctx* ctx, const DevScene& S, size_t smem, const DevWos& W,
                         const NodeSource& src, int64_t n_total, uint64_t pid_base,
                         bw_estimate* out, int64_t* steps) {
    switch (S.phi_kind) {
        case BW_PHI_FEATURE_CONST:
            return launch_wos_t<KIND, BW_PHI_FEATURE_CONST>(ctx, S, smem, W, src, n_total, pid_base, out, steps);
        case BW_PHI_QUADRATIC:
            return launch_wos_t<KIND, BW_PHI_QUADRATIC>(ctx, S, smem, W, src, n_total, pid_base, out, steps);
        case BW_PHI_EXP_SIN_SIN:
            return launch_wos_t<KIND, BW_PHI_EXP_SIN_SIN>(ctx, S, smem, W, src, n_total, pid_base, out, steps);
        case BW_PHI_SIN_SIN:
            return launch_wos_t<KIND, BW_PHI_SIN_SIN>(ctx, S, smem, W, src, n_total, pid_base, out, steps);
        default:
            return launch_wos_t<KIND, BW_PHI_POINT_SOURCE>(ctx, S, smem, W, src, n_total, pid_base, out, steps);
    }
}

} // namespace

// Diagnostic (bw_diag_stat_math): the statistical mode's root and table sincos
// as K1 evaluates them, for the accuracy tests.
namespace {
__global__ void stat_math_kernel(const double* __restrict__ a, const uint32_t* __restrict__ u,
                                 int64_t n, double* __restrict__ root, double* __restrict__ sn,
                                 double* __restrict__ cs) {
    __shared__ __align__(16) double2 trig[kTrigTab];
    stage_trig(trig);
    const JumpConst jc = jump_const<kTrigBits, false>();
    __syncthreads();
    const uint32_t trig_s = shared_addr(trig);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        root[i] = BW_SQRT_Q ? sqrt_q(a[i]) : sqrt_1ulp<false>(a[i]);
        double s, c;
        sincos32_tab<kTrigBits>(u[i], trig_s, jc, s, c);
        sn[i] = s;
        cs[i] = c;
    }
}
} // namespace

cudaError_t launch_stat_math(bw_ctx* ctx, const double* a, const uint32_t* u, int64_t n,
                             double* root, double* sn, double* cs) {
    ++ctx->launches;
    stat_math_kernel<<<ctx->sm_count * 2, 256, 0, ctx->stream>>>(a, u, n, root, sn, cs);
    return cudaGetLastError();
}

// The FAST sincos table (kTrig) of the current device, from long-double
// sinl / cosl of the centre angles (called by bw_init once per device).
cudaError_t init_trig_table() {
    double2 t[kTrigTab];
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int k = 0; k < kTrigTab; ++k) {
        const long double a = (2.0L * k + 1.0L) * pi / (long double)kTrigTab;
        t[k] = make_double2((double)sinl(a), (double)cosl(a));
    }
    return cudaMemcpyToSymbol(kTrig, t, sizeof t);
}

cudaError_t launch_wos(bw_ctx* ctx, const DevScene& S, size_t smem, const DevWos& W,
                       const NodeSource& src, int64_t n_total, uint64_t pid_base,
                       bw_estimate* out, int64_t* steps) {
    switch (S.kind) {
        case BW_SCENE_HALFSPACE:
            return launch_wos_k<BW_SCENE_HALFSPACE>(ctx, S, smem, W, src, n_total, pid_base, out, steps);
        case BW_SCENE_PLATESET:
            return launch_wos_k<BW_SCENE_PLATESET>(ctx, S, smem, W, src, n_total, pid_base, out, steps);
        case BW_SCENE_THINDISK:
            return launch_wos_k<BW_SCENE_THINDISK>(ctx, S, smem, W, src, n_total, pid_base, out, steps);
        case BW_SCENE_SPHERE:
            return launch_wos_k<BW_SCENE_SPHERE>(ctx, S, smem, W, src, n_total, pid_base, out, steps);
        case BW_SCENE_BOX:
            return launch_wos_k<BW_SCENE_BOX>(ctx, S, smem, W, src, n_total, pid_base, out, steps);
        default:
            return launch_wos_k<BW_SCENE_BOX_CAVITIES>(ctx, S, smem, W, src, n_total, pid_base, out, steps);
    }
}

cudaError_t launch_geometry(bw_ctx* ctx, const DevScene& S, size_t smem, const double* pts,
                            int64_t n, double eps, double trunc, double* dist, int32_t* feat,
                            double* dist_walk, double* proj, int32_t* exit_feat,
                            int check_domain) {
#define BW_GEO(K) launch_geometry_t<K>(ctx, S, smem, pts, n, eps, trunc, dist, feat, dist_walk, \
                                       proj, exit_feat, check_domain)
    switch (S.kind) {
        case BW_SCENE_HALFSPACE: return BW_GEO(BW_SCENE_HALFSPACE);
        case BW_SCENE_PLATESET: return BW_GEO(BW_SCENE_PLATESET);
        case BW_SCENE_THINDISK: return BW_GEO(BW_SCENE_THINDISK);
        case BW_SCENE_SPHERE: return BW_GEO(BW_SCENE_SPHERE);
        case BW_SCENE_BOX: return BW_GEO(BW_SCENE_BOX);
        default: return BW_GEO(BW_SCENE_BOX_CAVITIES);
    }
#undef BW_GEO
}

cudaError_t launch_walk(bw_ctx* ctx, const DevScene& S, size_t smem, const DevWos& W,
                        const double* starts, int64_t n, const uint64_t* pids,
                        const uint64_t* paths, double* exit_pts, int32_t* feat, int32_t* steps) {
    switch (S.kind) {
        case BW_SCENE_HALFSPACE:
            return launch_walk_t<BW_SCENE_HALFSPACE>(ctx, S, smem, W, starts, n, pids, paths, exit_pts, feat, steps);
        case BW_SCENE_PLATESET:
            return launch_walk_t<BW_SCENE_PLATESET>(ctx, S, smem, W, starts, n, pids, paths, exit_pts, feat, steps);
        case BW_SCENE_THINDISK:
            return launch_walk_t<BW_SCENE_THINDISK>(ctx, S, smem, W, starts, n, pids, paths, exit_pts, feat, steps);
        case BW_SCENE_SPHERE:
            return launch_walk_t<BW_SCENE_SPHERE>(ctx, S, smem, W, starts, n, pids, paths, exit_pts, feat, steps);
        case BW_SCENE_BOX:
            return launch_walk_t<BW_SCENE_BOX>(ctx, S, smem, W, starts, n, pids, paths, exit_pts, feat, steps);
        default:
            return launch_walk_t<BW_SCENE_BOX_CAVITIES>(ctx, S, smem, W, starts, n, pids, paths, exit_pts, feat, steps);
    }
}

cudaError_t launch_philox(bw_ctx* ctx, const uint64_t* ctr, const uint64_t* key, int64_t n,
                          uint64_t* out) {
    if (n <= 0) return cudaSuccess;
    ++ctx->launches;
    philox_kernel<<<(unsigned)((n + 127) / 128), 128, 0, ctx->stream>>>(ctr, key, n, out);
    return cudaGetLastError();
}

} // namespace bw
