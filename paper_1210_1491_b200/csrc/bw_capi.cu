// bw_capi.cu — the C-ABI (include/biewos_b200.h): context, scene upload,
// candidate-grid build, and the host/device entry points. Host code only.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "bw_internal.h"

namespace bw {

bw_status fail(bw_ctx* ctx, bw_status st, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return st;
}

bw_status cuda_check(bw_ctx* ctx, cudaError_t e, const char* what) {
    if (e == cudaSuccess) return BW_OK;
    return fail(ctx, BW_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void* scratch(bw_ctx* ctx, int slot, size_t bytes, bw_status* st) {
    if (bytes == 0) bytes = 16;
    if (ctx->scratch_bytes[slot] >= bytes) return ctx->scratch[slot];
    if (ctx->scratch[slot]) {
        cudaStreamSynchronize(ctx->stream);
        cudaFree(ctx->scratch[slot]);
        ctx->scratch[slot] = nullptr;
        ctx->scratch_bytes[slot] = 0;
    }
    const size_t alloc = bytes + bytes / 8; // headroom for slowly growing calls
    if (cudaMalloc(&ctx->scratch[slot], alloc) != cudaSuccess) {
        *st = fail(ctx, BW_ERR_CUDA, "cudaMalloc of " + std::to_string(alloc) + " bytes failed");
        return nullptr;
    }
    ctx->scratch_bytes[slot] = alloc;
    return ctx->scratch[slot];
}

namespace {

// Uniform grid of candidate cavities. For a cell C,
//   U  = min over features f of max_{p in C} dist_f(p)   (an upper bound of the
//        nearest distance anywhere in C)
//   L_i = min_{p in C} | |p - c_i| - r_i |                (a lower bound)
// cavity i is listed iff L_i <= U (+ rounding margin). A feature that is the
// nearest at some p in C has L_i <= dist_i(p) <= U, so the minimum over the
// list (plus the 6 faces) equals the brute-force minimum. Lists are sorted by
// L_i (nearest first) so the kernel's squared-distance test prunes most roots.
struct CandGrid {
    int gn = 0;
    double orig[3] = {0, 0, 0};
    double h = 0;
    std::vector<uint16_t> start; // list offsets: the whole list stays below 2^16 entries
    std::vector<uint16_t> list;
    std::vector<double> lower; // L_i of each list entry
};

CandGrid build_grid(const bw_scene* s, int gn) {
    CandGrid g;
    g.gn = gn;
    double ext = 0;
    for (int k = 0; k < 3; ++k) {
        g.orig[k] = s->box_lo[k];
        ext = std::max(ext, s->box_hi[k] - s->box_lo[k]);
    }
    g.h = ext / gn;
    const int ncell = gn * gn * gn;
    g.start.resize((size_t)ncell + 1);
    const double pad = 1e-9 * g.h;
    for (int iz = 0; iz < gn; ++iz)
        for (int iy = 0; iy < gn; ++iy)
            for (int ix = 0; ix < gn; ++ix) {
                const int cell = (iz * gn + iy) * gn + ix;
                double a[3], b[3];
                const int idx[3] = {ix, iy, iz};
                for (int k = 0; k < 3; ++k) {
                    a[k] = g.orig[k] + idx[k] * g.h - pad;
                    b[k] = g.orig[k] + (idx[k] + 1) * g.h + pad;
                }
                double U = INFINITY;
                for (int k = 0; k < 3; ++k) {
                    U = std::min(U, std::max(std::fabs(a[k] - s->box_lo[k]), std::fabs(b[k] - s->box_lo[k])));
                    U = std::min(U, std::max(std::fabs(s->box_hi[k] - a[k]), std::fabs(s->box_hi[k] - b[k])));
                }
                std::vector<double> L((size_t)s->n_cavities);
                for (int i = 0; i < s->n_cavities; ++i) {
                    const double* c = s->cavities + 4 * i;
                    double mn2 = 0, mx2 = 0;
                    for (int k = 0; k < 3; ++k) {
                        const double dn = c[k] < a[k] ? a[k] - c[k] : (c[k] > b[k] ? c[k] - b[k] : 0.0);
                        const double dx = std::max(std::fabs(c[k] - a[k]), std::fabs(c[k] - b[k]));
                        mn2 += dn * dn;
                        mx2 += dx * dx;
                    }
                    const double mind = std::sqrt(mn2), maxd = std::sqrt(mx2), r = c[3];
                    U = std::min(U, std::max(maxd - r, r - mind));
                    L[(size_t)i] = std::max({0.0, mind - r, r - maxd});
                }
                g.start[(size_t)cell] = (uint16_t)std::min<size_t>(g.list.size(), 0xffff);
                const double lim = U * (1.0 + 1e-9) + 1e-12;
                std::vector<std::pair<double, int>> cand;
                for (int i = 0; i < s->n_cavities; ++i)
                    if (L[(size_t)i] <= lim) cand.push_back({L[(size_t)i], i});
                std::stable_sort(cand.begin(), cand.end());
                for (const auto& c : cand) {
                    g.list.push_back((uint16_t)c.second);
                    g.lower.push_back(c.first);
                }
            }
    g.start[(size_t)ncell] = (uint16_t)std::min<size_t>(g.list.size(), 0xffff);
    return g;
}

int grid_n_from_env() {
    const char* e = std::getenv("BW_CAVITY_GRID");
    if (!e) return -1;
    return std::atoi(e);
}

} // namespace

bw_status upload_scene(bw_ctx* ctx, const bw_scene* s, DevScene& S, size_t& smem) {
    std::memset(&S, 0, sizeof S);
    smem = 0;
    if (!s) return fail(ctx, BW_ERR_INVALID, "scene is NULL");
    S.kind = s->kind;
    S.side = s->side;
    S.phi_kind = s->phi_kind;
    S.plane_z = s->plane_z;
    S.R = s->sphere_radius;
    S.mid_exact = 1;
    for (int k = 0; k < 3; ++k) {
        S.lo[k] = s->box_lo[k];
        S.hi[k] = s->box_hi[k];
        // TwoSum: lo + hi exact (and its half normal) -> the midpoint test of
        // box_face_distance is exact
        const volatile double sum = s->box_lo[k] + s->box_hi[k];
        const double bv = sum - s->box_lo[k];
        const double err = (s->box_lo[k] - (sum - bv)) + (s->box_hi[k] - bv);
        S.mid[k] = 0.5 * sum;
        S.half[k] = 0.5 * (s->box_hi[k] - s->box_lo[k]);
        if (err != 0.0 || !std::isfinite(sum) || (sum != 0.0 && std::fabs(sum) < 0x1.0p-1020))
            S.mid_exact = 0;
    }
    std::memcpy(S.phi, s->phi, sizeof S.phi);
    switch (s->kind) {
        case BW_SCENE_HALFSPACE:
        case BW_SCENE_SPHERE:
            break;
        case BW_SCENE_PLATESET:
            if (s->n_plates < 1 || s->n_plates > 1024 || !s->plates)
                return fail(ctx, BW_ERR_INVALID, "plate count must be in [1,1024] with data");
            for (int i = 0; i < s->n_plates; ++i) { // check_plates_disjoint (geometry.cpp:17-30)
                const double* a = s->plates + 4 * i;
                if (a[1] <= a[0] || a[3] <= a[2]) return fail(ctx, BW_ERR_GEOMETRY, "degenerate plate rectangle");
                for (int j = i + 1; j < s->n_plates; ++j) {
                    const double* b = s->plates + 4 * j;
                    const double ox = std::min(a[1], b[1]) - std::max(a[0], b[0]);
                    const double oy = std::min(a[3], b[3]) - std::max(a[2], b[2]);
                    if (ox > 1e-12 && oy > 1e-12) return fail(ctx, BW_ERR_GEOMETRY, "overlapping plates");
                }
            }
            break;
        case BW_SCENE_THINDISK:
            if (!(s->disk_radius > 0)) return fail(ctx, BW_ERR_GEOMETRY, "disk radius must be positive");
            break;
        case BW_SCENE_BOX:
        case BW_SCENE_BOX_CAVITIES:
            if (s->side != BW_INTERIOR)
                return fail(ctx, BW_ERR_APPLICABILITY, "box scenes are interior problems");
            for (int k = 0; k < 3; ++k)
                if (!(s->box_hi[k] > s->box_lo[k]))
                    return fail(ctx, BW_ERR_GEOMETRY, "degenerate box");
            break;
        default:
            return fail(ctx, BW_ERR_APPLICABILITY, "unknown scene kind");
    }
    if (s->kind == BW_SCENE_SPHERE && !(s->sphere_radius > 0))
        return fail(ctx, BW_ERR_GEOMETRY, "sphere radius must be positive");
    if (s->phi_kind < BW_PHI_FEATURE_CONST || s->phi_kind > BW_PHI_SIN_SIN)
        return fail(ctx, BW_ERR_APPLICABILITY,
                    "Dirichlet data has no closed form the device can evaluate");
    const bool plates = s->kind == BW_SCENE_PLATESET;
    const int ncav = s->kind == BW_SCENE_BOX_CAVITIES ? s->n_cavities : (plates ? s->n_plates : 0);
    if (ncav < 0 || ncav > 1024 || (ncav > 0 && !(plates ? s->plates : s->cavities)))
        return fail(ctx, BW_ERR_INVALID, "cavity count must be in [0,1024] with data");
    S.disk_r = s->disk_radius;
    const int nf = s->kind == BW_SCENE_BOX ? 6
                   : (s->kind == BW_SCENE_BOX_CAVITIES ? 6 + ncav : (plates ? ncav : 1));
    bw_status st = BW_OK;
    if (s->phi_kind == BW_PHI_FEATURE_CONST) {
        if (!s->feature_potential)
            return fail(ctx, BW_ERR_INVALID, "FEATURE_CONST data needs feature_potential");
        double* fp = (double*)scratch(ctx, kSlotFpot, sizeof(double) * nf, &st);
        if (st) return st;
        if ((st = cuda_check(ctx, cudaMemcpyAsync(fp, s->feature_potential, sizeof(double) * nf,
                                                  cudaMemcpyHostToDevice, ctx->stream), "fpot")))
            return st;
        S.fpot = fp;
    }
    S.n_cav = ncav;
    if (ncav > 0) {
        double* cav = (double*)scratch(ctx, kSlotCavities, sizeof(double) * 4 * ncav, &st);
        if (st) return st;
        if ((st = cuda_check(ctx, cudaMemcpyAsync(cav, plates ? s->plates : s->cavities,
                                                  sizeof(double) * 4 * ncav, cudaMemcpyHostToDevice,
                                                  ctx->stream), "cav")))
            return st;
        S.cav = reinterpret_cast<const double4*>(cav);
        smem = sizeof(double4) * ncav;
        int gn = plates ? 0 : grid_n_from_env();
        if (gn < 0) gn = ncav >= 8 ? 16 : 0;
        // the same geometry as the last call: reuse its device grid (no host
        // build, no copy, no stream sync)
        uint64_t key = 1469598103934665603ull; // FNV-1a over the grid's inputs
        auto mix = [&key](const void* p, size_t n) {
            const unsigned char* b = static_cast<const unsigned char*>(p);
            for (size_t i = 0; i < n; ++i) key = (key ^ b[i]) * 1099511628211ull;
        };
        mix(&gn, sizeof gn);
        mix(&ncav, sizeof ncav);
        mix(s->box_lo, sizeof s->box_lo);
        mix(s->box_hi, sizeof s->box_hi);
        if (!plates) mix(s->cavities, sizeof(double) * 4 * ncav);
        if (!plates && gn > 0 && ctx->grid.valid && ctx->grid.key == key) {
            const auto& G = ctx->grid;
            S.cell_start = (const uint16_t*)ctx->scratch[kSlotCellStart];
            S.cell_list = (const uint16_t*)ctx->scratch[kSlotCellList];
            S.gn = G.gn;
            S.lpacked = G.lpacked;
            S.lstep = G.lstep;
            S.linv = G.lstep > 0 ? (1.0 / G.lstep) * (1.0 + 1e-15) : 0.0;
            for (int k = 0; k < 3; ++k) {
                S.gorig[k] = G.orig[k];
                S.gc0[k] = -G.orig[k] * G.ginv - 0.5;
            }
            S.ginv = G.ginv;
            if (smem + G.bytes + 64 <= ctx->smem_optin - 16 * 1024) smem += G.bytes + 64;
            return BW_OK;
        }
        ctx->grid.valid = false;
        CandGrid g;
        // 16-bit offsets: coarsen the grid until the lists fit (else brute force)
        while (gn > 0) {
            g = build_grid(s, gn);
            if (g.list.size() <= 0xffff) break;
            gn = gn >= 8 ? gn * 3 / 4 : 0;
        }
        if (gn > 0) {
            // <= 256 cavities: pack each entry as (Lq << 8) | index with Lq a
            // conservative 8-bit lower bound (Lq * lstep <= L_i), so the kernel
            // can stop at the first candidate that cannot beat the best so far
            S.lpacked = 0;
            S.lstep = 0.0;
            if (ncav <= 256 && !g.list.empty()) {
                double lmax = 0.0;
                for (double L : g.lower) lmax = std::max(lmax, L);
                const double step = lmax > 0 ? lmax / 255.0 : 1.0;
                for (size_t t = 0; t < g.list.size(); ++t) {
                    int q = (int)std::floor(g.lower[t] / step);
                    q = std::min(std::max(q, 0), 255);
                    while (q > 0 && (double)q * step > g.lower[t]) --q;
                    g.list[t] = (uint16_t)((q << 8) | g.list[t]);
                }
                S.lpacked = 1;
                S.lstep = step;
                S.linv = (1.0 / step) * (1.0 + 1e-15);
            }
            uint16_t* cs = (uint16_t*)scratch(ctx, kSlotCellStart, sizeof(uint16_t) * g.start.size(), &st);
            if (st) return st;
            uint16_t* cl = (uint16_t*)scratch(ctx, kSlotCellList, sizeof(uint16_t) * (g.list.size() + 1), &st);
            if (st) return st;
            if ((st = cuda_check(ctx, cudaMemcpyAsync(cs, g.start.data(), sizeof(uint16_t) * g.start.size(),
                                                      cudaMemcpyHostToDevice, ctx->stream), "grid")))
                return st;
            if (!g.list.empty() &&
                (st = cuda_check(ctx, cudaMemcpyAsync(cl, g.list.data(), sizeof(uint16_t) * g.list.size(),
                                                      cudaMemcpyHostToDevice, ctx->stream), "grid")))
                return st;
            // the host vectors die here: make the async copies complete first
            if ((st = cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "grid sync"))) return st;
            S.cell_start = cs;
            S.cell_list = cl;
            S.gn = gn;
            S.gorig[0] = g.orig[0];
            S.gorig[1] = g.orig[1];
            S.gorig[2] = g.orig[2];
            S.ginv = 1.0 / g.h;
            for (int k = 0; k < 3; ++k) S.gc0[k] = -g.orig[k] * S.ginv - 0.5;
            const size_t grid_bytes = sizeof(uint16_t) * (g.start.size() + g.list.size());
            // K1's static shared memory (block table, warp scratch) is ~15 KB
            if (smem + grid_bytes + 64 <= ctx->smem_optin - 16 * 1024) smem += grid_bytes + 64;
            auto& G = ctx->grid;
            G.valid = true;
            G.key = key;
            G.gn = gn;
            G.lpacked = S.lpacked;
            G.lstep = S.lstep;
            for (int k = 0; k < 3; ++k) G.orig[k] = g.orig[k];
            G.ginv = S.ginv;
            G.bytes = grid_bytes;
        }
    }
    return BW_OK;
}

bw_status make_wos(bw_ctx* ctx, const bw_scene* s, const bw_wos_config* c, DevWos& W) {
    if (!c) return fail(ctx, BW_ERR_INVALID, "config is NULL");
    if (c->n_paths < 0) return fail(ctx, BW_ERR_INVALID, "n_paths must be >= 0");
    // K1 counts walks and walk indices in 32-bit registers (the lane refill
    // adds up to 32 past the last index)
    if (c->n_paths > (int64_t)INT32_MAX - 64)
        return fail(ctx, BW_ERR_INVALID, "n_paths must be <= 2^31 - 65 on the device");
    if (c->max_steps < 0) return fail(ctx, BW_ERR_INVALID, "max_steps must be >= 0");
    if (c->rng != BW_RNG_PHILOX4X64 && c->rng != BW_RNG_PHILOX4X32)
        return fail(ctx, BW_ERR_INVALID, "rng must be BW_RNG_PHILOX4X64 or BW_RNG_PHILOX4X32");
    if (!(c->eps_rel >= 0.0)) return fail(ctx, BW_ERR_INVALID, "eps_rel must be >= 0");
    W.eps = c->eps_shell;
    W.eps_rel = c->eps_rel;
    W.trunc = c->trunc_radius;
    W.max_steps = c->max_steps;
    W.max_blk = c->max_steps >> 1;
    W.n_paths = (int32_t)c->n_paths;
    W.rng = c->rng;
    W.keys = make_keys(c->seed, 0);
    W.keys32 = make_keys32(c->seed, 0);
    // |p| can only exceed trunc_radius on unbounded domains: skip the test
    // when the closed domain lies strictly inside the truncation sphere.
    double rmax = INFINITY; // half-space, plates, disk, exterior sphere: unbounded
    if (s->kind == BW_SCENE_SPHERE && s->side == BW_INTERIOR) rmax = s->sphere_radius;
    if (s->kind == BW_SCENE_BOX || s->kind == BW_SCENE_BOX_CAVITIES) {
        double q = 0;
        for (int k = 0; k < 3; ++k) {
            const double m = std::max(std::fabs(s->box_lo[k]), std::fabs(s->box_hi[k]));
            q += m * m;
        }
        rmax = std::sqrt(q);
    }
    W.bounded = rmax * (1.0 + 1e-9) < c->trunc_radius ? 1 : 0;
    // The statistical mode resolves distances to ~3e-12 of the boundary's size
    // (Newton-step roots, bw_device.cuh sqrt_q), so its shell must stay well
    // above that; the parity mode has no such limit.
    if (c->rng == BW_RNG_PHILOX4X32) {
        double scale = 1.0;
        if (s->kind == BW_SCENE_SPHERE) scale = s->sphere_radius;
        else if (s->kind == BW_SCENE_THINDISK) scale = s->disk_radius;
        else if (std::isfinite(rmax)) scale = rmax;
        if (!(c->eps_shell >= 1e-9 * scale))
            return fail(ctx, BW_ERR_INVALID,
                        "BW_RNG_PHILOX4X32 (statistical mode) needs eps_shell >= 1e-9 x the boundary's "
                        "size; use BW_RNG_PHILOX4X64 for thinner shells");
    }
    return BW_OK;
}

} // namespace bw

using namespace bw;

namespace {

bw_status finish(bw_ctx* ctx, const char* what) {
    bw_status st = cuda_check(ctx, cudaStreamSynchronize(ctx->stream), what);
    return st;
}

bw_status read_counters(bw_ctx* ctx, unsigned long long* h) {
    bw_status st = cuda_check(ctx, cudaMemcpyAsync(h, ctx->d_counters, sizeof(unsigned long long) * kCtrCount,
                                                   cudaMemcpyDeviceToHost, ctx->stream), "counters");
    if (st) return st;
    return finish(ctx, "counters sync");
}

bw_status wos_status(bw_ctx* ctx) {
    unsigned long long h[kCtrCount];
    bw_status st = read_counters(ctx, h);
    if (st) return st;
    if (h[kCtrClassify])
        return fail(ctx, BW_ERR_CLASSIFICATION,
                    std::to_string(h[kCtrClassify]) + " walks ended neither near the boundary nor truncated");
    if (h[kCtrReliability])
        return fail(ctx, BW_ERR_RELIABILITY,
                    std::to_string(h[kCtrReliability]) + " points: more than 0.1% of walks exceeded max_steps");
    return BW_OK;
}

template <class T>
bw_status h2d(bw_ctx* ctx, int slot, const T* h, size_t count, T** d) {
    bw_status st = BW_OK;
    *d = (T*)scratch(ctx, slot, sizeof(T) * count, &st);
    if (st) return st;
    if (count == 0) return BW_OK;
    return cuda_check(ctx, cudaMemcpyAsync(*d, h, sizeof(T) * count, cudaMemcpyHostToDevice, ctx->stream), "H2D");
}

template <class T>
bw_status d2h(bw_ctx* ctx, T* h, const T* d, size_t count) {
    if (count == 0 || !h) return BW_OK;
    return cuda_check(ctx, cudaMemcpyAsync(h, d, sizeof(T) * count, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
}

} // namespace

extern "C" {

int32_t bw_abi_version(void) { return BW_ABI_VERSION; }

bw_status bw_init(int device, bw_ctx** out) {
    if (!out) return BW_ERR_INVALID;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return BW_ERR_CUDA;
    if (device < 0 || device >= n) return BW_ERR_INVALID;
    if (cudaSetDevice(device) != cudaSuccess) return BW_ERR_CUDA;
    bw_ctx* ctx = new bw_ctx;
    ctx->device = device;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
        delete ctx;
        return BW_ERR_CUDA;
    }
    ctx->sm_count = prop.multiProcessorCount;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device);
    ctx->clock_khz = clk;
    ctx->smem_optin = prop.sharedMemPerBlockOptin;
    if (prop.major < 10) {
        delete ctx;
        return BW_ERR_CUDA; // sm_100a code only
    }
    if (init_trig_table() != cudaSuccess ||
        cudaMalloc(&ctx->d_counters, sizeof(unsigned long long) * kCtrAlloc) != cudaSuccess ||
        cudaMemset(ctx->d_counters, 0, sizeof(unsigned long long) * kCtrAlloc) != cudaSuccess) {
        delete ctx;
        return BW_ERR_CUDA;
    }
    *out = ctx;
    return BW_OK;
}

bw_status bw_finalize(bw_ctx* ctx) {
    if (!ctx) return BW_OK;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    for (int i = 0; i < kSlotCount; ++i)
        if (ctx->scratch[i]) cudaFree(ctx->scratch[i]);
    cudaFree(ctx->d_counters);
    delete ctx;
    return BW_OK;
}

bw_status bw_launch_count(const bw_ctx* ctx, uint64_t* count) {
    if (!ctx || !count) return BW_ERR_INVALID;
    *count = ctx->launches;
    return BW_OK;
}

const char* bw_last_error(const bw_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }

bw_status bw_set_stream(bw_ctx* ctx, void* stream) {
    if (!ctx) return BW_ERR_INVALID;
    ctx->stream = (cudaStream_t)stream;
    return BW_OK;
}

bw_status bw_synchronize(bw_ctx* ctx) {
    if (!ctx) return BW_ERR_INVALID;
    return finish(ctx, "synchronize");
}

bw_status bw_device_info(bw_ctx* ctx, int32_t* sm_count, int32_t* clock_khz) {
    if (!ctx) return BW_ERR_INVALID;
    if (sm_count) *sm_count = ctx->sm_count;
    if (clock_khz) *clock_khz = ctx->clock_khz;
    return BW_OK;
}

bw_status bw_philox_blocks(bw_ctx* ctx, const uint64_t* ctr, const uint64_t* key, int64_t n,
                           uint64_t* out) {
    if (!ctx || n < 0 || (n > 0 && (!ctr || !key || !out))) return fail(ctx, BW_ERR_INVALID, "bad arguments");
    cudaSetDevice(ctx->device);
    uint64_t *dc, *dk, *dout;
    bw_status st;
    if ((st = h2d(ctx, kSlotIn0, ctr, 4 * (size_t)n, &dc))) return st;
    if ((st = h2d(ctx, kSlotIn1, key, 2 * (size_t)n, &dk))) return st;
    dout = (uint64_t*)scratch(ctx, kSlotOut0, sizeof(uint64_t) * 4 * n, &st);
    if (st) return st;
    if ((st = cuda_check(ctx, launch_philox(ctx, dc, dk, n, dout), "philox launch"))) return st;
    if ((st = d2h(ctx, out, dout, 4 * (size_t)n))) return st;
    return finish(ctx, "philox");
}

namespace {
bw_status nearest_impl(bw_ctx* ctx, const bw_scene* scene, const double* points, int64_t n,
                       double* dist, int32_t* feature, double* dist_walk, int check_domain) {
    if (!ctx) return BW_ERR_INVALID;
    if (n < 0 || (n > 0 && (!points || !dist || !feature)))
        return fail(ctx, BW_ERR_INVALID, "bad arguments");
    cudaSetDevice(ctx->device);
    DevScene S;
    size_t smem;
    bw_status st;
    if ((st = upload_scene(ctx, scene, S, smem))) return st;
    if (n == 0) return BW_OK;
    double *dp, *dd, *dw = nullptr;
    int32_t* df;
    if ((st = h2d(ctx, kSlotIn0, points, 3 * (size_t)n, &dp))) return st;
    dd = (double*)scratch(ctx, kSlotOut0, sizeof(double) * 2 * n, &st);
    df = (int32_t*)scratch(ctx, kSlotOut1, sizeof(int32_t) * n, &st);
    if (st) return st;
    if (dist_walk) dw = dd + n;
    if ((st = cuda_check(ctx, launch_geometry(ctx, S, smem, dp, n, 0.0, INFINITY, dd, df, dw,
                                              nullptr, nullptr, check_domain), "geometry launch")))
        return st;
    if ((st = d2h(ctx, dist, dd, (size_t)n))) return st;
    if ((st = d2h(ctx, feature, df, (size_t)n))) return st;
    if (dist_walk && (st = d2h(ctx, dist_walk, dw, (size_t)n))) return st;
    unsigned long long h[kCtrCount];
    if ((st = read_counters(ctx, h))) return st;
    if (check_domain && h[kCtrDomain])
        return fail(ctx, BW_ERR_DOMAIN, "point on or outside the solution domain");
    return BW_OK;
}
} // namespace

bw_status bw_nearest_feature(bw_ctx* ctx, const bw_scene* scene, const double* points,
                             int64_t n, double* dist, int32_t* feature, double* dist_walk) {
    return nearest_impl(ctx, scene, points, n, dist, feature, dist_walk, 0);
}

bw_status bw_distance_to_boundary(bw_ctx* ctx, const bw_scene* scene, const double* points,
                                  int64_t n, double* dist, int32_t* feature) {
    return nearest_impl(ctx, scene, points, n, dist, feature, nullptr, 1);
}

bw_status bw_classify_exit(bw_ctx* ctx, const bw_scene* scene, const double* points, int64_t n,
                           double eps, double trunc_radius, double* projected, int32_t* feature) {
    if (!ctx) return BW_ERR_INVALID;
    if (n < 0 || (n > 0 && (!points || !projected || !feature)))
        return fail(ctx, BW_ERR_INVALID, "bad arguments");
    cudaSetDevice(ctx->device);
    DevScene S;
    size_t smem;
    bw_status st;
    if ((st = upload_scene(ctx, scene, S, smem))) return st;
    if (n == 0) return BW_OK;
    double *dp, *dq;
    int32_t* df;
    if ((st = h2d(ctx, kSlotIn0, points, 3 * (size_t)n, &dp))) return st;
    dq = (double*)scratch(ctx, kSlotOut0, sizeof(double) * 3 * n, &st);
    df = (int32_t*)scratch(ctx, kSlotOut1, sizeof(int32_t) * n, &st);
    if (st) return st;
    if ((st = cuda_check(ctx, launch_geometry(ctx, S, smem, dp, n, eps, trunc_radius, nullptr,
                                              nullptr, nullptr, dq, df, 0), "geometry launch")))
        return st;
    if ((st = d2h(ctx, projected, dq, 3 * (size_t)n))) return st;
    if ((st = d2h(ctx, feature, df, (size_t)n))) return st;
    unsigned long long h[kCtrCount];
    if ((st = read_counters(ctx, h))) return st;
    if (h[kCtrClassify])
        return fail(ctx, BW_ERR_CLASSIFICATION, "point is neither near the boundary nor truncated");
    return BW_OK;
}

bw_status bw_walk(bw_ctx* ctx, const bw_scene* scene, const bw_wos_config* cfg,
                  const double* starts, int64_t n, const uint64_t* point_ids,
                  const uint64_t* path_ids, double* exit_points, int32_t* features,
                  int32_t* steps) {
    if (!ctx) return BW_ERR_INVALID;
    if (n < 0 || (n > 0 && (!starts || !point_ids || !path_ids || !exit_points || !features || !steps)))
        return fail(ctx, BW_ERR_INVALID, "bad arguments");
    cudaSetDevice(ctx->device);
    DevScene S;
    size_t smem;
    DevWos W;
    bw_status st;
    if ((st = upload_scene(ctx, scene, S, smem))) return st;
    if ((st = make_wos(ctx, scene, cfg, W))) return st;
    if (n == 0) return BW_OK;
    double *ds, *dx;
    uint64_t *dp, *dq;
    int32_t *df, *dn;
    if ((st = h2d(ctx, kSlotIn0, starts, 3 * (size_t)n, &ds))) return st;
    if ((st = h2d(ctx, kSlotIn1, point_ids, (size_t)n, &dp))) return st;
    if ((st = h2d(ctx, kSlotIn2, path_ids, (size_t)n, &dq))) return st;
    dx = (double*)scratch(ctx, kSlotOut0, sizeof(double) * 3 * n, &st);
    if (st) return st;
    df = (int32_t*)scratch(ctx, kSlotOut1, sizeof(int32_t) * n, &st);
    if (st) return st;
    dn = (int32_t*)scratch(ctx, kSlotOut2, sizeof(int32_t) * n, &st);
    if (st) return st;
    if ((st = cuda_check(ctx, launch_walk(ctx, S, smem, W, ds, n, dp, dq, dx, df, dn), "walk launch")))
        return st;
    if ((st = d2h(ctx, exit_points, dx, 3 * (size_t)n))) return st;
    if ((st = d2h(ctx, features, df, (size_t)n))) return st;
    if ((st = d2h(ctx, steps, dn, (size_t)n))) return st;
    if ((st = finish(ctx, "walk"))) return st;
    return wos_status(ctx);
}

bw_status bw_wos_estimate_d(bw_ctx* ctx, const bw_scene* scene, const bw_wos_config* cfg,
                            const double* d_points, int64_t n, uint64_t point_id_base,
                            bw_estimate* d_out, int64_t* d_steps) {
    BW_RANGE("bw_wos_estimate_d (K1)");
    if (!ctx) return BW_ERR_INVALID;
    if (n < 0 || (n > 0 && (!d_points || !d_out))) return fail(ctx, BW_ERR_INVALID, "bad arguments");
    cudaSetDevice(ctx->device);
    DevScene S;
    size_t smem;
    DevWos W;
    bw_status st;
    if ((st = upload_scene(ctx, scene, S, smem))) return st;
    if ((st = make_wos(ctx, scene, cfg, W))) return st;
    if (n == 0) return BW_OK;
    NodeSource src{};
    src.xyz = d_points;
    if ((st = cuda_check(ctx, launch_wos(ctx, S, smem, W, src, n, point_id_base, d_out, d_steps), "wos launch")))
        return st;
    return wos_status(ctx);
}

bw_status bw_wos_estimate(bw_ctx* ctx, const bw_scene* scene, const bw_wos_config* cfg,
                          const double* points, int64_t n, uint64_t point_id_base,
                          bw_estimate* out, int64_t* steps_out) {
    if (!ctx) return BW_ERR_INVALID;
    if (n < 0 || (n > 0 && (!points || !out))) return fail(ctx, BW_ERR_INVALID, "bad arguments");
    if (n == 0) return BW_OK;
    cudaSetDevice(ctx->device);
    double* dp;
    bw_status st;
    if ((st = h2d(ctx, kSlotIn0, points, 3 * (size_t)n, &dp))) return st;
    bw_estimate* dout = (bw_estimate*)scratch(ctx, kSlotOut0, sizeof(bw_estimate) * n, &st);
    if (st) return st;
    int64_t* dsteps = (int64_t*)scratch(ctx, kSlotOut1, sizeof(int64_t) * n, &st);
    if (st) return st;
    const bw_status run = bw_wos_estimate_d(ctx, scene, cfg, dp, n, point_id_base, dout, dsteps);
    if (run != BW_OK && run != BW_ERR_RELIABILITY && run != BW_ERR_CLASSIFICATION) return run;
    if ((st = d2h(ctx, out, dout, (size_t)n))) return st;
    if ((st = d2h(ctx, steps_out, dsteps, (size_t)n))) return st;
    if ((st = finish(ctx, "estimate"))) return st;
    return run;
}

bw_status bw_wos_patch_nodes_d(bw_ctx* ctx, const bw_scene* scene, const bw_wos_config* cfg,
                               const double* d_centers, const double* d_axes,
                               const double* d_radii, const int32_t* d_cls,
                               const int64_t* d_bp_ids, int64_t n_bp,
                               const double* d_local_dirs, int32_t n_cls, int32_t n_nodes,
                               uint64_t point_id_base, bw_estimate* d_out, int64_t* d_steps) {
    BW_RANGE("bw_wos_patch_nodes_d (K1)");
    if (!ctx) return BW_ERR_INVALID;
    if (n_bp < 0 || n_nodes < 0 || n_cls < 1 ||
        (n_bp > 0 && (!d_centers || !d_axes || !d_radii || !d_local_dirs || !d_out)))
        return fail(ctx, BW_ERR_INVALID, "bad arguments");
    cudaSetDevice(ctx->device);
    DevScene S;
    size_t smem;
    DevWos W;
    bw_status st;
    if ((st = upload_scene(ctx, scene, S, smem))) return st;
    if ((st = make_wos(ctx, scene, cfg, W))) return st;
    if (n_bp == 0 || n_nodes == 0) return BW_OK;
    NodeSource src{};
    src.centers = d_centers;
    src.axes = d_axes;
    src.radii = d_radii;
    src.cls = d_cls;
    src.bp_ids = d_bp_ids;
    src.dirs = d_local_dirs;
    src.n_nodes = n_nodes;
    src.n_cls = n_cls;
    src.check_domain = 1;
    if ((st = cuda_check(ctx, launch_wos(ctx, S, smem, W, src, n_bp * (int64_t)n_nodes, point_id_base,
                                         d_out, d_steps), "wos launch")))
        return st;
    return wos_status(ctx);
}

bw_status bw_wos_patch_nodes(bw_ctx* ctx, const bw_scene* scene, const bw_wos_config* cfg,
                             const double* centers, const double* axes, const double* radii,
                             const int32_t* cls, const int64_t* bp_ids, int64_t n_bp,
                             const double* local_dirs, int32_t n_cls, int32_t n_nodes,
                             uint64_t point_id_base, bw_estimate* out, int64_t* steps_out) {
    if (!ctx) return BW_ERR_INVALID;
    if (n_bp < 0 || n_nodes < 0 || n_cls < 1 || (n_bp > 0 && (!centers || !axes || !radii || !local_dirs || !out)))
        return fail(ctx, BW_ERR_INVALID, "bad arguments");
    if (n_bp == 0 || n_nodes == 0) return BW_OK;
    cudaSetDevice(ctx->device);
    bw_status st;
    if (cls)
        for (int64_t i = 0; i < n_bp; ++i)
            if (cls[i] < 0 || cls[i] >= n_cls)
                return fail(ctx, BW_ERR_INVALID, "cls outside [0, n_cls)");
    double *dc, *da, *dr, *dl;
    int32_t* dk = nullptr;
    int64_t* dids = nullptr;
    if ((st = h2d(ctx, kSlotIn0, centers, 3 * (size_t)n_bp, &dc))) return st;
    if (bp_ids && (st = h2d(ctx, kSlotIn5, bp_ids, (size_t)n_bp, &dids))) return st;
    if ((st = h2d(ctx, kSlotIn1, axes, 3 * (size_t)n_bp, &da))) return st;
    if ((st = h2d(ctx, kSlotIn2, radii, (size_t)n_bp, &dr))) return st;
    if ((st = h2d(ctx, kSlotIn3, local_dirs, 3 * (size_t)n_cls * n_nodes, &dl))) return st;
    if (cls && (st = h2d(ctx, kSlotIn4, cls, (size_t)n_bp, &dk))) return st;
    const size_t nn = (size_t)n_bp * n_nodes;
    bw_estimate* dout = (bw_estimate*)scratch(ctx, kSlotOut0, sizeof(bw_estimate) * nn, &st);
    if (st) return st;
    int64_t* dsteps = (int64_t*)scratch(ctx, kSlotOut1, sizeof(int64_t) * nn, &st);
    if (st) return st;
    const bw_status run = bw_wos_patch_nodes_d(ctx, scene, cfg, dc, da, dr, dk, dids, n_bp, dl, n_cls,
                                               n_nodes, point_id_base, dout, dsteps);
    if (run != BW_OK && run != BW_ERR_RELIABILITY && run != BW_ERR_CLASSIFICATION) return run;
    if ((st = d2h(ctx, out, dout, nn))) return st;
    if ((st = d2h(ctx, steps_out, dsteps, nn))) return st;
    if ((st = finish(ctx, "patch nodes"))) return st;
    return run;
}

bw_status bw_potential_d(bw_ctx* ctx, const double* d_panels, int64_t n_panels,
                         const double* d_targets, int64_t n_t, double* d_u, uint8_t* d_near,
                         int64_t* near_count) {
    BW_RANGE("bw_potential_d (K3)");
    if (!ctx) return BW_ERR_INVALID;
    if (n_panels < 0 || n_t < 0 || (n_t > 0 && (!d_targets || !d_u)) || (n_panels > 0 && !d_panels))
        return fail(ctx, BW_ERR_INVALID, "bad arguments");
    cudaSetDevice(ctx->device);
    bw_status st;
    if ((st = cuda_check(ctx, launch_potential(ctx, d_panels, n_panels, d_targets, n_t, d_u, d_near, nullptr),
                         "potential launch")))
        return st;
    unsigned long long h[kCtrCount];
    if ((st = read_counters(ctx, h))) return st;
    if (near_count) *near_count = (int64_t)h[kCtrNear];
    if (h[kCtrNear] && !d_near)
        return fail(ctx, BW_ERR_NEARFIELD, "evaluation point within one panel diameter of the boundary");
    return BW_OK;
}

bw_status bw_potential(bw_ctx* ctx, const double* panels, int64_t n_panels, const double* targets,
                       int64_t n_t, double* u, uint8_t* near) {
    if (!ctx) return BW_ERR_INVALID;
    if (n_panels < 0 || n_t < 0 || (n_t > 0 && (!targets || !u)) || (n_panels > 0 && !panels))
        return fail(ctx, BW_ERR_INVALID, "bad arguments");
    if (n_t == 0) return BW_OK;
    cudaSetDevice(ctx->device);
    bw_status st;
    double *dp, *dt;
    if ((st = h2d(ctx, kSlotIn0, panels, 9 * (size_t)n_panels, &dp))) return st;
    if ((st = h2d(ctx, kSlotIn1, targets, 3 * (size_t)n_t, &dt))) return st;
    double* du = (double*)scratch(ctx, kSlotOut0, sizeof(double) * n_t, &st);
    if (st) return st;
    uint8_t* dn = (uint8_t*)scratch(ctx, kSlotOut1, (size_t)n_t, &st);
    if (st) return st;
    int64_t nc = 0;
    if ((st = bw_potential_d(ctx, dp, n_panels, dt, n_t, du, dn, &nc))) return st;
    if ((st = d2h(ctx, u, du, (size_t)n_t))) return st;
    if (near && (st = d2h(ctx, near, dn, (size_t)n_t))) return st;
    if ((st = finish(ctx, "potential"))) return st;
    if (nc && !near)
        return fail(ctx, BW_ERR_NEARFIELD, "evaluation point within one panel diameter of the boundary");
    return BW_OK;
}

bw_status bw_lu_solve_batched_d(bw_ctx* ctx, int32_t m, int64_t n_sys, const double* d_A,
                                const double* d_B, int32_t nrhs, double tol, double* d_X,
                                double* d_resid, int32_t* d_info) {
    BW_RANGE("bw_lu_solve_batched_d (K2)");
    if (!ctx) return BW_ERR_INVALID;
    if (m < 1 || m > 64 || nrhs < 1 || nrhs > 8 || n_sys < 0 ||
        (n_sys > 0 && (!d_A || !d_B || !d_X || !d_resid || !d_info)))
        return fail(ctx, BW_ERR_INVALID, "bad arguments (1 <= m <= 64, 1 <= nrhs <= 8)");
    cudaSetDevice(ctx->device);
    bw_status st;
    if ((st = cuda_check(ctx, launch_lu(ctx, m, n_sys, d_A, d_B, nrhs, tol, d_X, d_resid, d_info), "lu launch")))
        return st;
    unsigned long long h[kCtrCount];
    if ((st = read_counters(ctx, h))) return st;
    if (h[kCtrReliability])
        return fail(ctx, BW_ERR_SOLVER, std::to_string(h[kCtrReliability]) +
                                            " systems: singular or residual exceeds tolerance");
    return BW_OK;
}

bw_status bw_lu_solve_batched(bw_ctx* ctx, int32_t m, int64_t n_sys, const double* A,
                              const double* B, int32_t nrhs, double tol, double* X, double* resid,
                              int32_t* info) {
    if (!ctx) return BW_ERR_INVALID;
    if (m < 1 || m > 64 || nrhs < 1 || nrhs > 8 || n_sys < 0 ||
        (n_sys > 0 && (!A || !B || !X || !resid || !info)))
        return fail(ctx, BW_ERR_INVALID, "bad arguments (1 <= m <= 64, 1 <= nrhs <= 8)");
    if (n_sys == 0) return BW_OK;
    cudaSetDevice(ctx->device);
    bw_status st;
    double *dA, *dB;
    const size_t na = (size_t)n_sys * m * m, nb = (size_t)n_sys * nrhs * m;
    if ((st = h2d(ctx, kSlotIn0, A, na, &dA))) return st;
    if ((st = h2d(ctx, kSlotIn1, B, nb, &dB))) return st;
    double* dX = (double*)scratch(ctx, kSlotOut0, sizeof(double) * nb, &st);
    if (st) return st;
    double* dR = (double*)scratch(ctx, kSlotOut1, sizeof(double) * n_sys, &st);
    if (st) return st;
    int32_t* dI = (int32_t*)scratch(ctx, kSlotOut2, sizeof(int32_t) * n_sys, &st);
    if (st) return st;
    const bw_status run = bw_lu_solve_batched_d(ctx, m, n_sys, dA, dB, nrhs, tol, dX, dR, dI);
    if (run != BW_OK && run != BW_ERR_SOLVER) return run;
    if ((st = d2h(ctx, X, dX, nb))) return st;
    if ((st = d2h(ctx, resid, dR, (size_t)n_sys))) return st;
    if ((st = d2h(ctx, info, dI, (size_t)n_sys))) return st;
    if ((st = finish(ctx, "lu"))) return st;
    return run;
}

// ---- local DtN path ----

static_assert(bw::kSlotCount <= 96, "scratch slot table");

namespace {

// gauss_legendre (quadrature.cpp:7-35): Newton on P_n from cos(pi(i-1/4)/(n+1/2))
void host_gauss_legendre(int n, double* x, double* w) {
    const int m = (n + 1) / 2;
    for (int i = 1; i <= m; ++i) {
        double z = std::cos(3.14159265358979323846 * (i - 0.25) / (n + 0.5));
        double pp = 0, z1;
        do {
            double p1 = 1.0, p2 = 0.0;
            for (int j = 1; j <= n; ++j) {
                const double p3 = p2;
                p2 = p1;
                p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
            }
            pp = n * (z * p1 - p2) / (z * z - 1.0);
            z1 = z;
            z = z1 - p1 / pp;
        } while (std::fabs(z - z1) > 1e-15);
        x[i - 1] = -z;
        x[n - i] = z;
        w[i - 1] = 2.0 / ((1.0 - z * z) * pp * pp);
        w[n - i] = w[i - 1];
    }
    if (n % 2 == 1) x[n / 2] = 0.0;
}

// Patch classes index the Gamma rule tables on the device: reject cls outside
// [0, n_cls) before any kernel reads them (host arrays: here; device arrays:
// one check kernel and a read of its sticky counter).
bw_status check_classes_h(bw_ctx* ctx, const bw_patch* p, int64_t n, int32_t n_cls) {
    for (int64_t i = 0; i < n; ++i)
        if (p[i].cls < 0 || p[i].cls >= n_cls)
            return fail(ctx, BW_ERR_INVALID, "patch " + std::to_string(i) + ": cls " +
                                                 std::to_string(p[i].cls) + " outside [0, n_cls)");
    return BW_OK;
}

bw_status check_classes_d(bw_ctx* ctx, const bw_patch* d_p, int64_t n, int32_t n_cls) {
    bw_status st = cuda_check(ctx, launch_check_classes(ctx, d_p, n, n_cls), "class check");
    if (st) return st;
    unsigned long long bad = 0;
    st = cuda_check(ctx, cudaMemcpyAsync(&bad, ctx->d_counters + kCtrBadClass, sizeof bad,
                                         cudaMemcpyDeviceToHost, ctx->stream), "class check");
    if (st) return st;
    if ((st = cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "class check"))) return st;
    if (bad) return fail(ctx, BW_ERR_INVALID, std::to_string(bad) + " patches with cls outside [0, n_cls)");
    return BW_OK;
}

bw_status check_dtn_cfg(bw_ctx* ctx, const bw_dtn_config* cfg, int max_m = 64) {
    if (!cfg) return fail(ctx, BW_ERR_INVALID, "dtn config is NULL");
    const int m = cfg->azimuth * (2 * cfg->bands - 1);
    if (cfg->bands < 1 || cfg->azimuth < 3 || m > max_m)
        return fail(ctx, BW_ERR_INVALID, "need bands >= 1, azimuth >= 3, azimuth (2 bands - 1) <= " +
                                             std::to_string(max_m));
    if (cfg->gauss_polar < 1 || cfg->gauss_polar > 32 || cfg->near_depth < 0 || cfg->near_depth > 4)
        return fail(ctx, BW_ERR_INVALID, "need 1 <= gauss_polar <= 32, 0 <= near_depth <= 4");
    if (cfg->kind != BW_BIE_SECOND && cfg->kind != BW_BIE_FIRST)
        return fail(ctx, BW_ERR_INVALID, "kind must be BW_BIE_SECOND or BW_BIE_FIRST");
    return BW_OK;
}

} // namespace

bw_status bw_dtn_assemble_d(bw_ctx* ctx, const bw_scene* scene, const bw_patch* d_patches,
                            int64_t n_bp, const double* d_local_dirs, const double* d_weights,
                            int32_t n_cls, int32_t n_nodes, const bw_estimate* d_est,
                            const bw_dtn_config* cfg, double* d_A, double* d_b,
                            double* d_panel_area, int32_t* d_flags) {
    if (!ctx) return BW_ERR_INVALID;
    bw_status st;
    if ((st = check_dtn_cfg(ctx, cfg))) return st;
    if (n_bp < 0 || n_nodes < 1 || n_nodes > 2048 || n_cls < 1 ||
        (n_bp > 0 && (!d_patches || !d_local_dirs || !d_weights || !d_est || !d_A || !d_b ||
                      !d_panel_area || !d_flags)))
        return fail(ctx, BW_ERR_INVALID, "bad arguments");
    cudaSetDevice(ctx->device);
    DevScene S;
    size_t smem;
    if ((st = upload_scene(ctx, scene, S, smem))) return st;
    double gl[64] = {0};
    host_gauss_legendre(cfg->gauss_polar, gl, gl + 32);
    double* d_gl;
    if ((st = h2d(ctx, kSlotDtnGl, gl, 64, &d_gl))) return st;
    if ((st = cuda_check(ctx, launch_assemble(ctx, S, d_patches, n_bp, d_local_dirs, d_weights,
                                              n_nodes, d_est, cfg->bands, cfg->azimuth,
                                              cfg->gauss_polar, cfg->near_depth, cfg->kind, d_gl,
                                              d_A, d_b, d_panel_area, nullptr, d_flags),
                         "assemble launch")))
        return st;
    return finish(ctx, "assemble");
}

bw_status bw_dtn_point_values_d(bw_ctx* ctx, int64_t n_bp, const bw_dtn_config* cfg,
                                const double* d_X, const double* d_panel_area,
                                const int32_t* d_info, const int32_t* d_flags, double* d_dudn,
                                double* d_err, int32_t* d_status) {
    if (!ctx) return BW_ERR_INVALID;
    bw_status st;
    if ((st = check_dtn_cfg(ctx, cfg))) return st;
    cudaSetDevice(ctx->device);
    const int m = cfg->azimuth * (2 * cfg->bands - 1);
    if ((st = cuda_check(ctx, launch_point_values(ctx, n_bp, m, cfg->azimuth, d_X, d_panel_area,
                                                  d_info, d_flags, d_dudn, d_err, d_status),
                         "point values launch")))
        return st;
    return finish(ctx, "point values");
}

bw_status bw_dtn_solve_d(bw_ctx* ctx, const bw_scene* scene, const bw_wos_config* wos,
                         const bw_dtn_config* cfg, const bw_patch* d_patches,
                         const int64_t* d_bp_ids, int64_t n_bp, const double* d_local_dirs,
                         const double* d_weights, int32_t n_cls, int32_t n_nodes,
                         uint64_t point_id_base, double* d_dudn, double* d_err,
                         int32_t* d_status, bw_estimate* d_node_est, int64_t* d_steps) {
    BW_RANGE("bw_dtn_solve_d");
    if (!ctx) return BW_ERR_INVALID;
    bw_status st;
    if ((st = check_dtn_cfg(ctx, cfg))) return st;
    if (n_bp < 0 || n_nodes < 1 || n_nodes > 2048 || n_cls < 1 ||
        (n_bp > 0 && (!d_patches || !d_local_dirs || !d_weights || !d_dudn || !d_err || !d_status)))
        return fail(ctx, BW_ERR_INVALID, "bad arguments");
    if (n_bp == 0) return BW_OK;
    cudaSetDevice(ctx->device);
    if ((st = check_classes_d(ctx, d_patches, n_bp, n_cls))) return st;
    const size_t nn = (size_t)n_bp * n_nodes;
    double* c = (double*)scratch(ctx, kSlotDtnCenters, sizeof(double) * 3 * n_bp, &st);
    double* ax = (double*)scratch(ctx, kSlotDtnAxes, sizeof(double) * 3 * n_bp, &st);
    double* r = (double*)scratch(ctx, kSlotDtnRadii, sizeof(double) * n_bp, &st);
    int32_t* cls = (int32_t*)scratch(ctx, kSlotDtnCls, sizeof(int32_t) * n_bp, &st);
    bw_estimate* est = d_node_est ? d_node_est
                                  : (bw_estimate*)scratch(ctx, kSlotDtnEst, sizeof(bw_estimate) * nn, &st);
    if (st) return st;
    // K1 over every Gamma node
    if ((st = cuda_check(ctx, launch_unpack_patches(ctx, d_patches, n_bp, c, ax, r, cls), "unpack")))
        return st;
    const bw_status wos_st = bw_wos_patch_nodes_d(ctx, scene, wos, c, ax, r, cls, d_bp_ids, n_bp,
                                                  d_local_dirs, n_cls, n_nodes, point_id_base, est,
                                                  d_steps);
    if (wos_st != BW_OK && wos_st != BW_ERR_RELIABILITY) return wos_st;
    // Neumann stage: congruence-class tables (K7), else K4 -> K2 -> K5
    const bw_status nm_st = bw_dtn_neumann_d(ctx, scene, cfg, d_patches, n_bp, d_local_dirs,
                                             d_weights, n_cls, n_nodes, est, BW_DTN_CLASSES,
                                             d_dudn, d_err, d_status);
    if (nm_st != BW_OK && nm_st != BW_ERR_SOLVER) return nm_st;
    if (wos_st != BW_OK) return wos_st;
    return nm_st;
}

bw_status bw_dtn_neumann_d(bw_ctx* ctx, const bw_scene* scene, const bw_dtn_config* cfg,
                           const bw_patch* d_patches, int64_t n_bp, const double* d_local_dirs,
                           const double* d_weights, int32_t n_cls, int32_t n_nodes,
                           const bw_estimate* d_est, int32_t method, double* d_dudn,
                           double* d_err, int32_t* d_status) {
    BW_RANGE("bw_dtn_neumann_d (K7 | K4-K2-K5)");
    if (!ctx) return BW_ERR_INVALID;
    bw_status st;
    if ((st = check_dtn_cfg(ctx, cfg))) return st;
    if (n_bp < 0 || n_nodes < 1 || n_nodes > 2048 || n_cls < 1 ||
        (method != BW_DTN_CLASSES && method != BW_DTN_PER_PATCH) ||
        (n_bp > 0 && (!d_patches || !d_local_dirs || !d_weights || !d_est || !d_dudn || !d_err ||
                      !d_status)))
        return fail(ctx, BW_ERR_INVALID, "bad arguments");
    if (n_bp == 0) return BW_OK;
    cudaSetDevice(ctx->device);
    if ((st = check_classes_d(ctx, d_patches, n_bp, n_cls))) return st;
    const int m = cfg->azimuth * (2 * cfg->bands - 1);
    if (method == BW_DTN_CLASSES) {
        DevScene S;
        size_t smem;
        if ((st = upload_scene(ctx, scene, S, smem))) return st;
        double gl[64] = {0};
        host_gauss_legendre(cfg->gauss_polar, gl, gl + 32);
        double* d_gl;
        if ((st = h2d(ctx, kSlotDtnGl, gl, 64, &d_gl))) return st;
        bool applicable = false;
        const bw_status cs = dtn_neumann_classes(ctx, S, d_patches, n_bp, d_local_dirs, d_weights,
                                                 n_cls, n_nodes, d_est, cfg->bands, cfg->azimuth,
                                                 cfg->gauss_polar, cfg->near_depth, cfg->kind,
                                                 cfg->solve_tol, d_gl, d_dudn, d_err, d_status,
                                                 &applicable);
        if (applicable) {
            if (cs != BW_OK && cs != BW_ERR_SOLVER) return cs;
            if ((st = finish(ctx, "dtn classes"))) return st;
            return cs;
        }
    }
    double* A = (double*)scratch(ctx, kSlotDtnA, sizeof(double) * (size_t)n_bp * m * m, &st);
    double* b = (double*)scratch(ctx, kSlotDtnB, sizeof(double) * (size_t)n_bp * 2 * m, &st);
    double* X = (double*)scratch(ctx, kSlotDtnX, sizeof(double) * (size_t)n_bp * 2 * m, &st);
    double* res = (double*)scratch(ctx, kSlotDtnResid, sizeof(double) * n_bp, &st);
    int32_t* info = (int32_t*)scratch(ctx, kSlotDtnInfo, sizeof(int32_t) * n_bp, &st);
    double* area = (double*)scratch(ctx, kSlotDtnArea, sizeof(double) * (size_t)n_bp * m, &st);
    int32_t* flags = (int32_t*)scratch(ctx, kSlotDtnFlags, sizeof(int32_t) * n_bp, &st);
    if (st) return st;
    if ((st = bw_dtn_assemble_d(ctx, scene, d_patches, n_bp, d_local_dirs, d_weights, n_cls,
                                n_nodes, d_est, cfg, A, b, area, flags)))
        return st;
    const bw_status lu_st = bw_lu_solve_batched_d(ctx, m, n_bp, A, b, 2, cfg->solve_tol, X, res, info);
    if (lu_st != BW_OK && lu_st != BW_ERR_SOLVER) return lu_st;
    if ((st = bw_dtn_point_values_d(ctx, n_bp, cfg, X, area, info, flags, d_dudn, d_err, d_status)))
        return st;
    return lu_st;
}

bw_status bw_dtn_neumann(bw_ctx* ctx, const bw_scene* scene, const bw_dtn_config* cfg,
                         const bw_patch* patches, int64_t n_bp, const double* local_dirs,
                         const double* weights, int32_t n_cls, int32_t n_nodes,
                         const bw_estimate* est, int32_t method, double* dudn, double* err,
                         int32_t* status) {
    if (!ctx) return BW_ERR_INVALID;
    if (n_bp < 0 || n_nodes < 1 || n_cls < 1 ||
        (n_bp > 0 && (!patches || !local_dirs || !weights || !est || !dudn || !err || !status)))
        return fail(ctx, BW_ERR_INVALID, "bad arguments");
    if (n_bp == 0) return BW_OK;
    cudaSetDevice(ctx->device);
    bw_status st;
    if ((st = check_classes_h(ctx, patches, n_bp, n_cls))) return st;
    bw_patch* dp;
    double *dd, *dw;
    bw_estimate* de;
    if ((st = h2d(ctx, kSlotHostIn0, patches, (size_t)n_bp, &dp))) return st;
    if ((st = h2d(ctx, kSlotHostIn1, local_dirs, 3 * (size_t)n_cls * n_nodes, &dd))) return st;
    if ((st = h2d(ctx, kSlotHostIn2, weights, (size_t)n_cls * n_nodes, &dw))) return st;
    if ((st = h2d(ctx, kSlotHostIn3, est, (size_t)n_bp * n_nodes, &de))) return st;
    double* du = (double*)scratch(ctx, kSlotHostOut0, sizeof(double) * 2 * n_bp, &st);
    int32_t* ds = (int32_t*)scratch(ctx, kSlotHostOut1, sizeof(int32_t) * n_bp, &st);
    if (st) return st;
    const bw_status run = bw_dtn_neumann_d(ctx, scene, cfg, dp, n_bp, dd, dw, n_cls, n_nodes, de,
                                           method, du, du + n_bp, ds);
    if (run != BW_OK && run != BW_ERR_SOLVER) return run;
    if ((st = d2h(ctx, dudn, du, (size_t)n_bp))) return st;
    if ((st = d2h(ctx, err, du + n_bp, (size_t)n_bp))) return st;
    if ((st = d2h(ctx, status, ds, (size_t)n_bp))) return st;
    if ((st = finish(ctx, "dtn neumann"))) return st;
    return run;
}

namespace {
// solve_patch for meshes beyond the warp-per-system path (bw_patch_large.cu)
bw_status solve_patch_large(bw_ctx* ctx, const DevScene& S, const bw_dtn_config* cfg,
                            const bw_patch* dp, int64_t n_bp, const double* dd, const double* dw,
                            int32_t n_nodes, const bw_estimate* de, const double* d_gl,
                            double* out, int32_t* info, int32_t* flags) {
    bw_status st = BW_OK;
    const int m = cfg->azimuth * (2 * cfg->bands - 1);
    const size_t nm = (size_t)n_bp * m;
    if (large_patch_smem(cfg->bands, cfg->azimuth, cfg->gauss_polar) + 1024 > ctx->smem_optin)
        return fail(ctx, BW_ERR_INVALID, "patch mesh too large for one CTA's shared memory");
    double* gam = (double*)scratch(ctx, kSlotPfGam, sizeof(double) * 6 * (size_t)n_bp * n_nodes, &st);
    double* A = (double*)scratch(ctx, kSlotDtnA, sizeof(double) * nm * m, &st);
    double* A0 = (double*)scratch(ctx, kSlotPfA0, sizeof(double) * nm * m, &st);
    double* b = (double*)scratch(ctx, kSlotDtnB, sizeof(double) * 2 * nm, &st);
    double* b0 = (double*)scratch(ctx, kSlotPfB0, sizeof(double) * 2 * nm, &st);
    double* X = (double*)scratch(ctx, kSlotDtnX, sizeof(double) * 2 * nm, &st);
    double* res = (double*)scratch(ctx, kSlotDtnResid, sizeof(double) * n_bp, &st);
    double* cen = (double*)scratch(ctx, kSlotPfCen, sizeof(double) * 3 * nm, &st);
    if (st) return st;
    if ((st = cuda_check(ctx, launch_gamma_nodes(ctx, dp, n_bp, dd, dw, n_nodes, de, gam, flags),
                         "gamma nodes launch")))
        return st;
    if ((st = cuda_check(ctx, launch_assemble_large(ctx, S, dp, n_bp, gam, n_nodes, cfg->bands,
                                                    cfg->azimuth, cfg->gauss_polar, cfg->near_depth,
                                                    cfg->kind, d_gl, A, b, cen),
                         "large assemble launch")))
        return st;
    cudaError_t ce = cudaMemcpyAsync(A0, A, sizeof(double) * nm * m, cudaMemcpyDeviceToDevice,
                                     ctx->stream);
    if (ce == cudaSuccess)
        ce = cudaMemcpyAsync(b0, b, sizeof(double) * 2 * nm, cudaMemcpyDeviceToDevice, ctx->stream);
    if ((st = cuda_check(ctx, ce, "system copy"))) return st;
    if ((st = cuda_check(ctx, launch_lu_large(ctx, m, n_bp, A, b, A0, b0, cfg->solve_tol, X, res,
                                              info),
                         "large lu launch")))
        return st;
    return cuda_check(ctx, launch_patch_field(ctx, n_bp, m, dp, X, cen, out, out + nm, out + 2 * nm),
                      "patch field launch");
}
} // namespace

bw_status bw_solve_patch(bw_ctx* ctx, const bw_scene* scene, const bw_dtn_config* cfg,
                         const bw_patch* patches, int64_t n_bp, const double* local_dirs,
                         const double* weights, int32_t n_cls, int32_t n_nodes,
                         const bw_estimate* est, double* dudn, double* r, double* est_error,
                         int32_t* status) {
    BW_RANGE("bw_solve_patch");
    if (!ctx) return BW_ERR_INVALID;
    bw_status st;
    if ((st = check_dtn_cfg(ctx, cfg, 4096))) return st;
    const bool large = cfg->azimuth * (2 * cfg->bands - 1) > 64 || n_nodes > 2048 ||
                       std::getenv("BW_FORCE_LARGE_PATCH") != nullptr;
    if (n_bp < 0 || n_nodes < 1 || (!large && n_nodes > 2048) || n_cls < 1 ||
        (n_bp > 0 && (!patches || !local_dirs || !weights || !est || !dudn || !r || !est_error ||
                      !status)))
        return fail(ctx, BW_ERR_INVALID, "bad arguments");
    if (n_bp == 0) return BW_OK;
    cudaSetDevice(ctx->device);
    if ((st = check_classes_h(ctx, patches, n_bp, n_cls))) return st;
    const int m = cfg->azimuth * (2 * cfg->bands - 1);
    const size_t nm = (size_t)n_bp * m;
    bw_patch* dp;
    double *dd, *dw;
    bw_estimate* de;
    if ((st = h2d(ctx, kSlotHostIn0, patches, (size_t)n_bp, &dp))) return st;
    if ((st = h2d(ctx, kSlotHostIn1, local_dirs, 3 * (size_t)n_cls * n_nodes, &dd))) return st;
    if ((st = h2d(ctx, kSlotHostIn2, weights, (size_t)n_cls * n_nodes, &dw))) return st;
    if ((st = h2d(ctx, kSlotHostIn3, est, (size_t)n_bp * n_nodes, &de))) return st;
    double* A = (double*)scratch(ctx, kSlotDtnA, sizeof(double) * nm * m, &st);
    double* b = (double*)scratch(ctx, kSlotDtnB, sizeof(double) * 2 * nm, &st);
    double* X = (double*)scratch(ctx, kSlotDtnX, sizeof(double) * 2 * nm, &st);
    double* res = (double*)scratch(ctx, kSlotDtnResid, sizeof(double) * n_bp, &st);
    int32_t* info = (int32_t*)scratch(ctx, kSlotDtnInfo, sizeof(int32_t) * n_bp, &st);
    double* area = (double*)scratch(ctx, kSlotDtnArea, sizeof(double) * nm, &st);
    int32_t* flags = (int32_t*)scratch(ctx, kSlotDtnFlags, sizeof(int32_t) * n_bp, &st);
    double* cen = (double*)scratch(ctx, kSlotPfCen, sizeof(double) * 3 * nm, &st);
    double* out = (double*)scratch(ctx, kSlotHostOut0, sizeof(double) * 3 * nm, &st);
    if (st) return st;
    DevScene S;
    size_t smem;
    if ((st = upload_scene(ctx, scene, S, smem))) return st;
    double gl[64] = {0};
    host_gauss_legendre(cfg->gauss_polar, gl, gl + 32);
    double* d_gl;
    if ((st = h2d(ctx, kSlotDtnGl, gl, 64, &d_gl))) return st;
    bw_status lu_st = BW_OK;
    if (large) {
        if ((st = solve_patch_large(ctx, S, cfg, dp, n_bp, dd, dw, n_nodes, de, d_gl, out, info,
                                    flags)))
            return st;
    } else {
        if ((st = cuda_check(ctx, launch_assemble(ctx, S, dp, n_bp, dd, dw, n_nodes, de, cfg->bands,
                                                  cfg->azimuth, cfg->gauss_polar, cfg->near_depth,
                                                  cfg->kind, d_gl, A, b, area, cen, flags),
                             "assemble launch")))
            return st;
        lu_st = bw_lu_solve_batched_d(ctx, m, n_bp, A, b, 2, cfg->solve_tol, X, res, info);
        if (lu_st != BW_OK && lu_st != BW_ERR_SOLVER) return lu_st;
        if ((st = cuda_check(ctx, launch_patch_field(ctx, n_bp, m, dp, X, cen, out, out + nm,
                                                     out + 2 * nm),
                             "patch field launch")))
            return st;
    }
    if ((st = d2h(ctx, dudn, out, nm))) return st;
    if ((st = d2h(ctx, r, out + nm, nm))) return st;
    if ((st = d2h(ctx, est_error, out + 2 * nm, nm))) return st;
    std::vector<int32_t> hi((size_t)n_bp), hf((size_t)n_bp);
    if ((st = d2h(ctx, hi.data(), info, (size_t)n_bp))) return st;
    if ((st = d2h(ctx, hf.data(), flags, (size_t)n_bp))) return st;
    if ((st = finish(ctx, "solve patch"))) return st;
    bool any_fail = false;
    for (int64_t i = 0; i < n_bp; ++i) {
        status[i] = (hi[(size_t)i] ? 2 : 0) | (hf[(size_t)i] ? 1 : 0);
        any_fail |= hi[(size_t)i] != 0;
    }
    if (any_fail) return fail(ctx, BW_ERR_SOLVER, "patch solve residual above tolerance (SolverError)");
    return lu_st;
}

bw_status bw_dtn_solve(bw_ctx* ctx, const bw_scene* scene, const bw_wos_config* wos,
                       const bw_dtn_config* cfg, const bw_patch* patches, const int64_t* bp_ids,
                       int64_t n_bp, const double* local_dirs, const double* weights,
                       int32_t n_cls, int32_t n_nodes, uint64_t point_id_base, double* dudn,
                       double* err, int32_t* status, bw_estimate* node_est, int64_t* steps) {
    BW_RANGE("bw_dtn_solve");
    if (!ctx) return BW_ERR_INVALID;
    if (n_bp < 0 || n_nodes < 1 || n_cls < 1 ||
        (n_bp > 0 && (!patches || !local_dirs || !weights || !dudn || !err || !status)))
        return fail(ctx, BW_ERR_INVALID, "bad arguments");
    if (n_bp == 0) return BW_OK;
    cudaSetDevice(ctx->device);
    bw_status st;
    if ((st = check_classes_h(ctx, patches, n_bp, n_cls))) return st;
    bw_patch* dp;
    double *dd, *dw;
    int64_t* dids = nullptr;
    if ((st = h2d(ctx, kSlotHostIn0, patches, (size_t)n_bp, &dp))) return st;
    if ((st = h2d(ctx, kSlotHostIn1, local_dirs, 3 * (size_t)n_cls * n_nodes, &dd))) return st;
    if ((st = h2d(ctx, kSlotHostIn2, weights, (size_t)n_cls * n_nodes, &dw))) return st;
    if (bp_ids && (st = h2d(ctx, kSlotHostIn3, bp_ids, (size_t)n_bp, &dids))) return st;
    double* du = (double*)scratch(ctx, kSlotHostOut0, sizeof(double) * 2 * n_bp, &st);
    int32_t* ds = (int32_t*)scratch(ctx, kSlotHostOut1, sizeof(int32_t) * n_bp, &st);
    int64_t* dst = steps ? (int64_t*)scratch(ctx, kSlotHostOut2, sizeof(int64_t) * n_bp * n_nodes, &st)
                         : nullptr;
    if (st) return st;
    const bw_status run = bw_dtn_solve_d(ctx, scene, wos, cfg, dp, dids, n_bp, dd, dw, n_cls, n_nodes,
                                         point_id_base, du, du + n_bp, ds, nullptr, dst);
    if (run != BW_OK && run != BW_ERR_RELIABILITY && run != BW_ERR_SOLVER) return run;
    if ((st = d2h(ctx, dudn, du, (size_t)n_bp))) return st;
    if ((st = d2h(ctx, err, du + n_bp, (size_t)n_bp))) return st;
    if ((st = d2h(ctx, status, ds, (size_t)n_bp))) return st;
    if (node_est) {
        const bw_estimate* de = (const bw_estimate*)ctx->scratch[kSlotDtnEst];
        if ((st = d2h(ctx, node_est, de, (size_t)n_bp * n_nodes))) return st;
    }
    if (steps && (st = d2h(ctx, steps, dst, (size_t)n_bp * n_nodes))) return st;
    if ((st = finish(ctx, "dtn"))) return st;
    return run;
}

// ---- flat-boundary point formula ----

bw_status bw_point_formula_d(bw_ctx* ctx, const bw_scene* scene, const bw_patch* d_patches,
                             int64_t n_bp, const double* d_cap_dirs, const double* d_cap_weights,
                             int32_t n_cap, const bw_estimate* d_est, const double* d_ring,
                             int32_t n_ring, double* d_total, double* d_sigma1,
                             double* d_sigma2, double* d_std_error) {
    BW_RANGE("bw_point_formula_d (K6)");
    if (!ctx) return BW_ERR_INVALID;
    if (n_bp < 0 || n_cap < 1 || n_ring < 1 ||
        (n_bp > 0 && (!d_patches || !d_cap_dirs || !d_cap_weights || !d_est || !d_ring || !d_total)))
        return fail(ctx, BW_ERR_INVALID, "bad arguments");
    if (scene && scene->kind == BW_SCENE_SPHERE)
        return fail(ctx, BW_ERR_APPLICABILITY, "point solver requires a flat boundary scene");
    cudaSetDevice(ctx->device);
    DevScene S;
    size_t smem;
    bw_status st;
    if ((st = upload_scene(ctx, scene, S, smem))) return st;
    double gl[64] = {0}; // gauss_legendre(20) of sigma2_plates_exact (point_solver.cpp:84)
    host_gauss_legendre(20, gl, gl + 32);
    double* d_gl;
    if ((st = h2d(ctx, kSlotPtGl, gl, 64, &d_gl))) return st;
    if ((st = cuda_check(ctx, launch_point_formula(ctx, S, d_patches, n_bp, d_cap_dirs, d_cap_weights,
                                                   n_cap, d_est, d_ring, n_ring, d_gl, d_total,
                                                   d_sigma1, d_sigma2, d_std_error),
                         "point formula launch")))
        return st;
    unsigned long long h[kCtrCount];
    if ((st = read_counters(ctx, h))) return st;
    if (h[kCtrGeometry])
        return fail(ctx, BW_ERR_GEOMETRY, "hemisphere axis must be normal to the boundary plane "
                                          "and its centre on it (GeometryError)");
    if (h[kCtrClassify])
        return fail(ctx, BW_ERR_CLASSIFICATION, "point is not on a boundary feature (ClassificationError)");
    if (h[kCtrDomain])
        return fail(ctx, BW_ERR_DOMAIN, "disk S_a is not covered by the boundary feature (DomainError)");
    if (h[kCtrSingular])
        return fail(ctx, BW_ERR_SINGULARITY, "nonzero data jump at the collocation point (SingularityError)");
    return BW_OK;
}

bw_status bw_point_formula(bw_ctx* ctx, const bw_scene* scene, const bw_patch* patches,
                           int64_t n_bp, const double* cap_dirs, const double* cap_weights,
                           int32_t n_cap, const bw_estimate* est, const double* ring,
                           int32_t n_ring, double* total, double* sigma1, double* sigma2,
                           double* std_error) {
    if (!ctx) return BW_ERR_INVALID;
    if (n_bp < 0 || n_cap < 1 || n_ring < 1 ||
        (n_bp > 0 && (!patches || !cap_dirs || !cap_weights || !est || !ring || !total)))
        return fail(ctx, BW_ERR_INVALID, "bad arguments");
    if (n_bp == 0) return BW_OK;
    cudaSetDevice(ctx->device);
    bw_status st;
    bw_patch* dp;
    double *dd, *dw, *dr;
    bw_estimate* de;
    if ((st = h2d(ctx, kSlotPt0, patches, (size_t)n_bp, &dp))) return st;
    if ((st = h2d(ctx, kSlotPt1, cap_dirs, 3 * (size_t)n_cap, &dd))) return st;
    if ((st = h2d(ctx, kSlotPt2, cap_weights, (size_t)n_cap, &dw))) return st;
    if ((st = h2d(ctx, kSlotPt3, est, (size_t)n_bp * n_cap, &de))) return st;
    if ((st = h2d(ctx, kSlotPt4, ring, 4 * (size_t)n_ring, &dr))) return st;
    double* out = (double*)scratch(ctx, kSlotPt5, sizeof(double) * 4 * n_bp, &st);
    if (st) return st;
    if ((st = bw_point_formula_d(ctx, scene, dp, n_bp, dd, dw, n_cap, de, dr, n_ring, out,
                                 out + n_bp, out + 2 * n_bp, out + 3 * n_bp)))
        return st;
    if ((st = d2h(ctx, total, out, (size_t)n_bp))) return st;
    if (sigma1 && (st = d2h(ctx, sigma1, out + n_bp, (size_t)n_bp))) return st;
    if (sigma2 && (st = d2h(ctx, sigma2, out + 2 * n_bp, (size_t)n_bp))) return st;
    if (std_error && (st = d2h(ctx, std_error, out + 3 * n_bp, (size_t)n_bp))) return st;
    return finish(ctx, "point formula");
}

// ---- last-passage estimator ----

bw_status bw_estimate_lp(bw_ctx* ctx, const bw_scene* scene, const bw_wos_config* cfg,
                         const double* center, double radius, const double* axis,
                         int64_t n_paths, int32_t allow_general_data, bw_lp_result* out,
                         int64_t* feature_counts) {
    BW_RANGE("bw_estimate_lp");
    if (!ctx) return BW_ERR_INVALID;
    if (!scene || !center || !axis || !out || n_paths < 0) return fail(ctx, BW_ERR_INVALID, "bad arguments");
    if (!(radius > 0)) return fail(ctx, BW_ERR_GEOMETRY, "hemisphere radius must be positive");
    if (std::fabs(std::sqrt(axis[0] * axis[0] + axis[1] * axis[1] + axis[2] * axis[2]) - 1.0) > 1e-12)
        return fail(ctx, BW_ERR_GEOMETRY, "hemisphere axis must be unit length");
    cudaSetDevice(ctx->device);
    DevScene S;
    size_t smem;
    DevWos W;
    bw_status st;
    if ((st = upload_scene(ctx, scene, S, smem))) return st;
    if ((st = make_wos(ctx, scene, cfg, W))) return st;
    const int nf = scene->kind == BW_SCENE_PLATESET ? scene->n_plates : 1;
    if (scene->kind == BW_SCENE_BOX || scene->kind == BW_SCENE_BOX_CAVITIES)
        return fail(ctx, BW_ERR_APPLICABILITY, "last-passage walks need an unbounded (exterior) scene");
    // phi(x) at the centre (eval_dirichlet, tol 1e-6 * scale, geometry.cpp:218-220)
    double scale = 1.0;
    if (scene->kind == BW_SCENE_THINDISK) scale = scene->disk_radius;
    if (scene->kind == BW_SCENE_SPHERE) scale = scene->sphere_radius;
    if (scene->kind == BW_SCENE_PLATESET) {
        scale = 0;
        for (int i = 0; i < 4 * scene->n_plates; ++i) scale = std::max(scale, std::fabs(scene->plates[i]));
    }
    double* red = (double*)scratch(ctx, kSlotLpRed, sizeof(double) * 8, &st);
    if (st) return st;
    if ((st = cuda_check(ctx, launch_dirichlet(ctx, S, smem, center, 1e-6 * scale, red), "dirichlet")))
        return st;
    double h[5];
    if ((st = d2h(ctx, h, red, 2)) || (st = finish(ctx, "dirichlet"))) return st;
    if (!(h[1] >= 0)) return fail(ctx, BW_ERR_CLASSIFICATION, "point is not on a boundary feature");
    const double phix = h[0];
    if (!allow_general_data) { // last_passage.cpp:56-64
        if (scene->phi_kind != BW_PHI_FEATURE_CONST)
            return fail(ctx, BW_ERR_APPLICABILITY, "last-passage requires piecewise-constant Dirichlet data");
        for (int i = 0; i < nf; ++i) {
            const double v = scene->feature_potential[i];
            if (std::fabs(v) > 1e-12 && std::fabs(v - 1.0) > 1e-12)
                return fail(ctx, BW_ERR_APPLICABILITY, "last-passage requires a {0,1} potential level set");
        }
        if (std::fabs(phix - 1.0) > 1e-12)
            return fail(ctx, BW_ERR_APPLICABILITY, "hemisphere base must sit on the unit-potential feature");
    }
    double* val = (double*)scratch(ctx, kSlotLpVal, sizeof(double) * (size_t)std::max<int64_t>(n_paths, 1), &st);
    int32_t* feat = (int32_t*)scratch(ctx, kSlotLpFeat, sizeof(int32_t) * (size_t)std::max<int64_t>(n_paths, 1), &st);
    unsigned long long* cnt = (unsigned long long*)scratch(ctx, kSlotLpCounts, sizeof(unsigned long long) * nf, &st);
    if (st) return st;
    if ((st = cuda_check(ctx, cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * nf, ctx->stream), "memset")))
        return st;
    if ((st = cuda_check(ctx, cudaMemsetAsync(ctx->d_counters, 0, sizeof(unsigned long long) * kCtrCount, ctx->stream), "memset")))
        return st;
    if ((st = cuda_check(ctx, launch_lp(ctx, S, smem, W, center, radius, axis, n_paths, phix, val, feat, cnt, red),
                         "lp launch")))
        return st;
    std::vector<unsigned long long> hc((size_t)nf);
    if ((st = d2h(ctx, h, red, 5))) return st;
    if ((st = d2h(ctx, hc.data(), cnt, (size_t)nf))) return st;
    if ((st = finish(ctx, "lp"))) return st;
    unsigned long long hctr[kCtrCount];
    if ((st = read_counters(ctx, hctr))) return st;
    const double n = h[0], mean = h[3], m2 = h[4];
    const double pref = 3.0 / (2.0 * radius); // last_passage.cpp:102-106
    out->sigma_lp = pref * mean;
    const double var = n > 1 ? m2 / (n - 1) : 0.0;
    out->std_error = pref * std::sqrt(var / std::max(n, 1.0));
    out->n_paths = (int64_t)n;
    out->n_infinity = (int64_t)h[1];
    out->n_failed = (int64_t)h[2];
    if (feature_counts)
        for (int i = 0; i < nf; ++i) feature_counts[i] = (int64_t)hc[(size_t)i];
    if (hctr[kCtrClassify])
        return fail(ctx, BW_ERR_CLASSIFICATION, "walks ended neither near the boundary nor truncated");
    if (h[2] > 0.001 * (double)n_paths)
        return fail(ctx, BW_ERR_RELIABILITY, "more than 0.1% of last-passage walks exceeded max_steps");
    return BW_OK;
}

} // extern "C"

extern "C" bw_status bw_dtn_class_cache_hits(bw_ctx* ctx, uint64_t* hits) {
    if (!ctx || !hits) return BW_ERR_INVALID;
    *hits = ctx->cls.hits;
    return BW_OK;
}
