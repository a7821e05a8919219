/*
 * biewos_oracle.c — CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference's BIE-WOS hot path, used ONLY by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs as the checker. It is never linked into, called by, or a
 * fallback for the product library (paper_1210_1491_b200/).
 *
 * Every function cites the reference file:line it restates (paths relative to
 * the reference's proj/ directory). Scene kinds the reference lacks (BOX,
 * BOX_CAVITIES) are restated in the reference's style:
 * unsigned nearest distance + lowest-index argmin (geometry.cpp:131-155),
 * projection + classification loop (geometry.cpp:175-196, 222-239).
 *
 * Pinning: Philox KATs of tests/test_rng.cpp:11-34,
 * the reference's statistical/known-answer WOS tests (tests/test_wos.cpp),
 * and walk-by-walk comparison against the reference sources themselves
 * compiled under oracle/_ref (oracle/Makefile).
 *
 * Build: gcc -O2 -ffp-contract=off (no FMA contraction, like the reference's
 * default x86-64 build) -> oracle/_build/liboracle.so
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/biewos_b200.h"

#define OR_PI 3.14159265358979323846 /* types.hpp:16 kPi */

/* ------------------------------------------------------------------ */
/* C1 Philox4x64-10 (rng.hpp:14-38)                                    */
/* ------------------------------------------------------------------ */
static const uint64_t kM0 = 0xD2E7470EE14C6C93ULL; /* rng.hpp:20 */
static const uint64_t kM1 = 0xCA5A826395121157ULL; /* rng.hpp:21 */
static const uint64_t kW0 = 0x9E3779B97F4A7C15ULL; /* rng.hpp:22 */
static const uint64_t kW1 = 0xBB67AE8584CAA73BULL; /* rng.hpp:23 */

static inline void mulhilo(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
    unsigned __int128 p = (unsigned __int128)a * b; /* rng.hpp:14-18 */
    *hi = (uint64_t)(p >> 64);
    *lo = (uint64_t)p;
}

void or_philox_block(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
    uint64_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint64_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) { /* rng.hpp:27-36 */
        if (round > 0) {
            k0 += kW0;
            k1 += kW1;
        }
        uint64_t hi0, lo0, hi1, lo1;
        mulhilo(kM0, c[0], &hi0, &lo0);
        mulhilo(kM1, c[2], &hi1, &lo1);
        uint64_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    }
    memcpy(out, c, sizeof c);
}

void or_philox_blocks(const uint64_t* ctr, const uint64_t* key, int64_t n, uint64_t* out) {
    for (int64_t i = 0; i < n; ++i) or_philox_block(ctr + 4 * i, key + 2 * i, out + 4 * i);
}

/* Philox4x32-10 (the device's BW_RNG_PHILOX4X32 block; Random123 constants,
 * the same round structure as rng.hpp:25-38 on 32-bit words). Not part of
 * the reference: its own KATs (Random123's) pin it in tests/test_oracle.py. */
void or_philox4x32_block(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = (uint32_t)p1;
        c[2] = n2;
        c[3] = (uint32_t)p0;
    }
    memcpy(out, c, sizeof c);
}

void or_philox4x32_blocks(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out) {
    for (int64_t i = 0; i < n; ++i) or_philox4x32_block(ctr + 4 * i, key + 2 * i, out + 4 * i);
}

/* RngStream (rng.hpp:44-67): key {seed, 0x1BD11BDAA9FC1A22 ^ domain},
 * ctr {0, path_id, point_id, domain}; only ctr[0] advances.
 * kind 1 (BW_RNG_PHILOX4X32, the device's statistical mode; not a reference
 * stream): key {lo(seed), hi(seed) ^ 0x1BD11BDA ^ domain}, ctr {blk, path,
 * lo(point), hi(point)}; a block yields four 32-bit words o0..o3 in order,
 * one per uniform: U = (o + 1/2) 2^-32, so a block feeds two walk steps
 * (z from o0 / o2, azimuth from o1 / o3). As 64-bit words (tests of the
 * block layout) it reads (o0 << 32 | o1), (o2 << 32 | o3). */
typedef struct {
    uint64_t key[2];
    uint64_t ctr[4];
    uint64_t buf[4];
    uint32_t buf32[4];
    int pos, kind;
} or_rng;

static void rng_init_kind(or_rng* s, uint64_t seed, uint64_t point_id, uint64_t path_id,
                          uint64_t domain, int kind) {
    s->kind = kind;
    s->key[0] = seed;
    s->key[1] = 0x1BD11BDAA9FC1A22ULL ^ domain;
    s->ctr[0] = 0;
    s->ctr[1] = path_id;
    s->ctr[2] = point_id;
    s->ctr[3] = domain;
    s->pos = 4;
}

static void rng_init(or_rng* s, uint64_t seed, uint64_t point_id, uint64_t path_id,
                     uint64_t domain) {
    rng_init_kind(s, seed, point_id, path_id, domain, 0);
}

static inline uint32_t rng32_next(or_rng* s) { /* kind 1 only */
    if (s->pos == 4) {
        const uint32_t key[2] = {(uint32_t)s->key[0], (uint32_t)(s->key[0] >> 32) ^ 0x1BD11BDAu ^
                                                          (uint32_t)s->ctr[3]};
        const uint32_t ctr[4] = {(uint32_t)s->ctr[0], (uint32_t)s->ctr[1], (uint32_t)s->ctr[2],
                                 (uint32_t)(s->ctr[2] >> 32)};
        or_philox4x32_block(ctr, key, s->buf32);
        ++s->ctr[0];
        s->pos = 0;
    }
    return s->buf32[s->pos++];
}

static inline uint64_t rng_u64(or_rng* s) { /* rng.hpp:50-57 */
    if (s->kind == 1) {
        const uint64_t hi = rng32_next(s);
        return (hi << 32) | rng32_next(s);
    }
    if (s->pos == 4) {
        or_philox_block(s->ctr, s->key, s->buf);
        ++s->ctr[0];
        s->pos = 0;
    }
    return s->buf[s->pos++];
}

static inline double rng_double(or_rng* s) { /* rng.hpp:60 */
    if (s->kind == 1) return ((double)rng32_next(s) + 0.5) * 0x1.0p-32;
    return (double)(rng_u64(s) >> 11) * 0x1.0p-53;
}

/* exported for tests: first n doubles of stream (seed, point, path, domain) */
void or_rng_doubles(uint64_t seed, uint64_t point_id, uint64_t path_id, uint64_t domain,
                    int64_t n, double* out) {
    or_rng s;
    rng_init(&s, seed, point_id, path_id, domain);
    for (int64_t i = 0; i < n; ++i) out[i] = rng_double(&s);
}

void or_rng_u64s(uint64_t seed, uint64_t point_id, uint64_t path_id, uint64_t domain,
                 int64_t n, uint64_t* out) {
    or_rng s;
    rng_init(&s, seed, point_id, path_id, domain);
    for (int64_t i = 0; i < n; ++i) out[i] = rng_u64(&s);
}

/* the BW_RNG_PHILOX4X32 stream's uniforms in draw order: (o + 1/2) 2^-32 */
void or_rng32_doubles(uint64_t seed, uint64_t point_id, uint64_t path_id, int64_t n, double* out) {
    or_rng s;
    rng_init_kind(&s, seed, point_id, path_id, 0, 1);
    for (int64_t i = 0; i < n; ++i) out[i] = rng_double(&s);
}

/* the BW_RNG_PHILOX4X32 WOS stream (domain 0) as 64-bit words */
void or_rng32_u64s(uint64_t seed, uint64_t point_id, uint64_t path_id, int64_t n, uint64_t* out) {
    or_rng s;
    rng_init_kind(&s, seed, point_id, path_id, 0, 1);
    for (int64_t i = 0; i < n; ++i) out[i] = rng_u64(&s);
}

/* ------------------------------------------------------------------ */
/* C4 geometry (geometry.cpp)                                          */
/* ------------------------------------------------------------------ */
static inline double norm3(const double p[3]) { /* Eigen norm: sqrt(squaredNorm) */
    return sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
}

int or_feature_count(const bw_scene* s) { /* geometry.cpp:94-100 (+ new kinds) */
    switch (s->kind) {
        case BW_SCENE_PLATESET: return s->n_plates;
        case BW_SCENE_BOX: return 6;
        case BW_SCENE_BOX_CAVITIES: return 6 + s->n_cavities;
        default: return 1;
    }
}

/* nearest_feature (geometry.cpp:131-155): unsigned distance + argmin, ties
 * to the lowest index (strict <). BOX faces use the unsigned plane distance,
 * which equals the distance to the face rectangle for any point of the
 * closed box; cavities use |‖p-c‖ - r| like the sphere (geometry.cpp:150). */
double or_nearest_feature(const bw_scene* s, const double p[3], int* feature) {
    double best = INFINITY;
    int f = -1;
    switch (s->kind) {
        case BW_SCENE_HALFSPACE:
            best = fabs(p[2] - s->plane_z);
            f = 0;
            break;
        case BW_SCENE_PLATESET: /* geometry.cpp:137-141, plate_distance :11-15 */
            for (int i = 0; i < s->n_plates; ++i) {
                const double* pl = s->plates + 4 * i;
                double dx = pl[0] - p[0];
                if (0.0 > dx) dx = 0.0;
                if (p[0] - pl[1] > dx) dx = p[0] - pl[1];
                double dy = pl[2] - p[1];
                if (0.0 > dy) dy = 0.0;
                if (p[1] - pl[3] > dy) dy = p[1] - pl[3];
                const double d = sqrt(dx * dx + dy * dy + p[2] * p[2]);
                if (d < best) { best = d; f = i; }
            }
            break;
        case BW_SCENE_THINDISK: { /* geometry.cpp:143-149 */
            const double rho = hypot(p[0], p[1]);
            best = rho <= s->disk_radius ? fabs(p[2]) : hypot(rho - s->disk_radius, p[2]);
            f = 0;
            break;
        }
        case BW_SCENE_SPHERE:
            best = fabs(norm3(p) - s->sphere_radius);
            f = 0;
            break;
        case BW_SCENE_BOX:
        case BW_SCENE_BOX_CAVITIES: {
            for (int k = 0; k < 3; ++k) {
                const double dlo = fabs(p[k] - s->box_lo[k]);
                if (dlo < best) { best = dlo; f = 2 * k; }
                const double dhi = fabs(s->box_hi[k] - p[k]);
                if (dhi < best) { best = dhi; f = 2 * k + 1; }
            }
            if (s->kind == BW_SCENE_BOX_CAVITIES) {
                for (int i = 0; i < s->n_cavities; ++i) {
                    const double* c = s->cavities + 4 * i;
                    const double q[3] = {p[0] - c[0], p[1] - c[1], p[2] - c[2]};
                    const double d = fabs(norm3(q) - c[3]);
                    if (d < best) { best = d; f = 6 + i; }
                }
            }
            break;
        }
    }
    if (feature) *feature = f;
    return best;
}

/* Scene::in_domain (geometry.cpp:100-113 style) */
int or_in_domain(const bw_scene* s, const double p[3]) {
    switch (s->kind) {
        case BW_SCENE_HALFSPACE: return p[2] > s->plane_z;
        case BW_SCENE_PLATESET:
        case BW_SCENE_THINDISK: return or_nearest_feature(s, p, NULL) > 0; /* geometry.cpp:110-112 */
        case BW_SCENE_SPHERE: {
            const double r = norm3(p);
            return s->side == BW_INTERIOR ? r < s->sphere_radius : r > s->sphere_radius;
        }
        case BW_SCENE_BOX:
        case BW_SCENE_BOX_CAVITIES: {
            for (int k = 0; k < 3; ++k)
                if (!(p[k] > s->box_lo[k] && p[k] < s->box_hi[k])) return 0;
            if (s->kind == BW_SCENE_BOX_CAVITIES)
                for (int i = 0; i < s->n_cavities; ++i) {
                    const double* c = s->cavities + 4 * i;
                    const double q[3] = {p[0] - c[0], p[1] - c[1], p[2] - c[2]};
                    if (!(norm3(q) > c[3])) return 0;
                }
            return 1;
        }
    }
    return 0;
}

static inline double clampd(double v, double lo, double hi) {
    return v < lo ? lo : (hi < v ? hi : v); /* std::clamp */
}

/* project_to_feature (geometry.cpp:175-196) */
void or_project_to_feature(const bw_scene* s, const double p[3], int f, double out[3]) {
    switch (s->kind) {
        case BW_SCENE_HALFSPACE:
            out[0] = p[0]; out[1] = p[1]; out[2] = s->plane_z;
            return;
        case BW_SCENE_PLATESET: { /* geometry.cpp:180-183 */
            const double* pl = s->plates + 4 * f;
            out[0] = clampd(p[0], pl[0], pl[1]); out[1] = clampd(p[1], pl[2], pl[3]); out[2] = 0.0;
            return;
        }
        case BW_SCENE_THINDISK: { /* geometry.cpp:184-189 */
            const double rho = hypot(p[0], p[1]);
            if (rho <= s->disk_radius) { out[0] = p[0]; out[1] = p[1]; out[2] = 0.0; return; }
            const double k = s->disk_radius / rho;
            out[0] = p[0] * k; out[1] = p[1] * k; out[2] = 0.0;
            return;
        }
        case BW_SCENE_SPHERE: {
            const double r = norm3(p);
            if (r == 0) { out[0] = 0; out[1] = 0; out[2] = s->sphere_radius; return; }
            const double k = s->sphere_radius / r;
            out[0] = p[0] * k; out[1] = p[1] * k; out[2] = p[2] * k;
            return;
        }
        default: {
            if (f < 6) {
                const int ax = f / 2;
                for (int k = 0; k < 3; ++k) out[k] = clampd(p[k], s->box_lo[k], s->box_hi[k]);
                out[ax] = (f & 1) ? s->box_hi[ax] : s->box_lo[ax];
                return;
            }
            const double* c = s->cavities + 4 * (f - 6);
            const double q[3] = {p[0] - c[0], p[1] - c[1], p[2] - c[2]};
            const double r = norm3(q);
            if (r == 0) { out[0] = c[0]; out[1] = c[1]; out[2] = c[2] + c[3]; return; }
            const double k = c[3] / r;
            out[0] = c[0] + q[0] * k; out[1] = c[1] + q[1] * k; out[2] = c[2] + q[2] * k;
            return;
        }
    }
}

/* Dirichlet data at an on-boundary point (the closed forms of bw_phi_kind) */
double or_eval_phi(const bw_scene* s, const double y[3], int feature) {
    const double* c = s->phi;
    switch (s->phi_kind) {
        case BW_PHI_FEATURE_CONST: return s->feature_potential[feature];
        case BW_PHI_QUADRATIC:
            return c[0] + c[1] * y[0] + c[2] * y[1] + c[3] * y[2] + c[4] * y[0] * y[0] +
                   c[5] * y[1] * y[1] + c[6] * y[2] * y[2] + c[7] * y[0] * y[1] +
                   c[8] * y[0] * y[2] + c[9] * y[1] * y[2];
        case BW_PHI_EXP_SIN_SIN:
            return c[0] * exp(c[1] * (y[0] - c[4])) * sin(c[2] * (y[1] - c[5])) *
                   sin(c[3] * (y[2] - c[6]));
        case BW_PHI_POINT_SOURCE: {
            const double q[3] = {y[0] - c[1], y[1] - c[2], y[2] - c[3]};
            return c[4] + c[0] / norm3(q);
        }
        case BW_PHI_SIN_SIN: /* runner.cpp:318-324 */
            return c[0] * sin(c[1] * (y[0] - c[3])) * sin(c[2] * (y[1] - c[4]));
    }
    return NAN;
}

/* classify_exit (geometry.cpp:222-239). Returns 0 or BW_ERR_CLASSIFICATION. */
int or_classify_exit(const bw_scene* s, const double p[3], double eps, double trunc,
                     double proj[3], int* feature) {
    if (norm3(p) > trunc) {
        memcpy(proj, p, 3 * sizeof(double));
        *feature = -1;
        return 0;
    }
    int best = -1;
    double dist = INFINITY;
    const int nf = or_feature_count(s);
    for (int f = 0; f < nf; ++f) {
        double pr[3];
        or_project_to_feature(s, p, f, pr);
        const double q[3] = {p[0] - pr[0], p[1] - pr[1], p[2] - pr[2]};
        const double d = norm3(q);
        if (d < dist) {
            dist = d;
            best = f;
            memcpy(proj, pr, sizeof pr);
        }
    }
    if (best < 0 || dist > eps) return BW_ERR_CLASSIFICATION;
    *feature = best;
    return 0;
}

/* ------------------------------------------------------------------ */
/* C5 walk-on-spheres (wos.cpp:61-93)                                  */
/* ------------------------------------------------------------------ */
typedef struct {
    double point[3];
    int feature; /* >=0, -1 infinity, -2 failed (geometry.hpp:25-26) */
    int steps;
} or_exit;

static int walk_stream(const bw_scene* s, const double start[3], const bw_wos_config* cfg,
                       or_rng* rng, or_exit* ex) {
    double p[3] = {start[0], start[1], start[2]};
    int steps = 0;
    for (;;) { /* wos.cpp:64-78 */
        if (norm3(p) > cfg->trunc_radius) {
            memcpy(ex->point, p, sizeof p);
            ex->feature = -1;
            ex->steps = steps;
            return 0;
        }
        const double d = or_nearest_feature(s, p, NULL);
        if (d <= cfg->eps_shell) {
            const int st = or_classify_exit(s, p, cfg->eps_shell, cfg->trunc_radius, ex->point,
                                            &ex->feature);
            ex->steps = steps;
            return st;
        }
        /* kind 1 (the device's statistical mode): budget rounded down to even,
         * which the device checks once per stream block of two steps */
        if (steps >= (rng->kind == 1 ? (cfg->max_steps & ~1) : cfg->max_steps)) {
            memcpy(ex->point, p, sizeof p);
            ex->feature = -2;
            ex->steps = steps;
            return 0;
        }
        /* kind 1: z on the centred signed grid, (int32(o) + 1/2) 2^-31 (the
         * device's p32_z); azimuth 2 pi (o + 1/2) 2^-32 */
        const double z = rng->kind == 1 ? ((double)(int32_t)rng32_next(rng) + 0.5) * 0x1.0p-31
                                        : 2.0 * rng_double(rng) - 1.0;
        const double az = 2.0 * OR_PI * rng_double(rng);
        const double t = 1.0 - z * z;
        const double r = sqrt(t > 0.0 ? t : 0.0);
        const double v[3] = {r * cos(az), r * sin(az), z};
        p[0] = p[0] + d * v[0];
        p[1] = p[1] + d * v[1];
        p[2] = p[2] + d * v[2];
        ++steps;
    }
}

/* walk(scene, start, cfg, point_id, path_id) (wos.cpp:81-85) */
int or_walk(const bw_scene* s, const bw_wos_config* cfg, const double* starts, int64_t n,
            const uint64_t* point_ids, const uint64_t* path_ids, double* exit_points,
            int32_t* features, int32_t* steps) {
    int status = 0;
    for (int64_t i = 0; i < n; ++i) {
        or_rng rng;
        rng_init_kind(&rng, cfg->seed, point_ids[i], path_ids[i], 0, cfg->rng);
        or_exit ex;
        const int st = walk_stream(s, starts + 3 * i, cfg, &rng, &ex);
        if (st) {
            status = st;
            ex.feature = -3;
        }
        memcpy(exit_points + 3 * i, ex.point, 3 * sizeof(double));
        features[i] = ex.feature;
        steps[i] = ex.steps;
    }
    return status;
}

/* exit_value (wos.cpp:87-93) */
static double exit_value(const bw_scene* s, const or_exit* ex) {
    if (ex->feature == -1) return 0.0;
    return or_eval_phi(s, ex->point, ex->feature);
}

/* ChunkStat (wos.cpp:14-40) */
typedef struct {
    int64_t n, n_inf, n_failed;
    double mean, m2;
    int64_t steps; /* extra: ExitRecord.steps summed (geometry.hpp:31) */
    int err;
} chunk_stat;

static void cs_push(chunk_stat* c, double v) { /* wos.cpp:18-23 */
    ++c->n;
    const double d = v - c->mean;
    c->mean += d / (double)c->n;
    c->m2 += d * (v - c->mean);
}

static void cs_merge(chunk_stat* a, const chunk_stat* o) { /* wos.cpp:24-39 */
    a->n_inf += o->n_inf;
    a->n_failed += o->n_failed;
    a->steps += o->steps;
    if (!a->err) a->err = o->err;
    if (o->n == 0) return;
    if (a->n == 0) {
        a->n = o->n;
        a->mean = o->mean;
        a->m2 = o->m2;
        return;
    }
    const double d = o->mean - a->mean;
    const int64_t nt = a->n + o->n;
    a->mean += d * (double)o->n / (double)nt;
    a->m2 += o->m2 + d * d * (double)a->n * (double)o->n / (double)nt;
    a->n = nt;
}

#define OR_CHUNK 4096 /* wos.cpp:11 */

typedef struct {
    const bw_scene* s;
    const bw_wos_config* cfg;
    const double* pts;
    uint64_t base;
    int64_t chunks_per_point;
    chunk_stat* stats;
    int64_t lo, hi;
} task_range;

static void run_task(const task_range* tr, int64_t task) { /* wos.cpp:99-121 */
    const int64_t pt = task / tr->chunks_per_point;
    const int64_t chunk = task % tr->chunks_per_point;
    const int64_t lo = chunk * OR_CHUNK;
    const int64_t hi = tr->cfg->n_paths < lo + OR_CHUNK ? tr->cfg->n_paths : lo + OR_CHUNK;
    chunk_stat c;
    memset(&c, 0, sizeof c);
    for (int64_t k = lo; k < hi; ++k) {
        or_rng rng;
        rng_init_kind(&rng, tr->cfg->seed, tr->base + (uint64_t)pt, (uint64_t)k, 0, tr->cfg->rng);
        or_exit ex;
        const int st = walk_stream(tr->s, tr->pts + 3 * pt, tr->cfg, &rng, &ex);
        c.steps += ex.steps;
        if (st) {
            c.err = st;
            break;
        }
        if (ex.feature == -2) {
            ++c.n_failed;
            continue;
        }
        if (ex.feature == -1) ++c.n_inf;
        cs_push(&c, exit_value(tr->s, &ex));
    }
    tr->stats[task] = c;
}

static void* worker(void* arg) {
    const task_range* tr = (const task_range*)arg;
    for (int64_t t = tr->lo; t < tr->hi; ++t) run_task(tr, t);
    return NULL;
}

/* estimate_u_batch (wos.cpp:95-132) with parallel_for's static block
 * partition over `workers` threads (parallel.hpp:14-40). Returns 0,
 * BW_ERR_RELIABILITY (wos.cpp:43-44; outputs still filled) or
 * BW_ERR_CLASSIFICATION. steps_out (optional): walk steps per point. */
int or_estimate_u_batch(const bw_scene* s, const bw_wos_config* cfg, const double* pts,
                        int64_t npts, uint64_t point_id_base, int workers, bw_estimate* out,
                        int64_t* steps_out) {
    if (npts <= 0) return 0;
    const int64_t cpp = (cfg->n_paths + OR_CHUNK - 1) / OR_CHUNK;
    const int64_t n_tasks = npts * cpp;
    chunk_stat* stats = (chunk_stat*)calloc((size_t)n_tasks, sizeof(chunk_stat));
    if (workers < 1) workers = 1;
    int w = workers;
    if (w > n_tasks) w = (int)n_tasks;
    task_range* tr = (task_range*)calloc((size_t)w, sizeof(task_range));
    pthread_t* th = (pthread_t*)calloc((size_t)w, sizeof(pthread_t));
    for (int t = 0; t < w; ++t) {
        tr[t] = (task_range){s, cfg, pts, point_id_base, cpp, stats,
                             n_tasks * t / w, n_tasks * (t + 1) / w};
        if (w == 1)
            worker(&tr[t]);
        else
            pthread_create(&th[t], NULL, worker, &tr[t]);
    }
    if (w > 1)
        for (int t = 0; t < w; ++t) pthread_join(th[t], NULL);
    int status = 0;
    for (int64_t pt = 0; pt < npts; ++pt) { /* ordered merge, wos.cpp:123-131 */
        chunk_stat tot;
        memset(&tot, 0, sizeof tot);
        for (int64_t c = 0; c < cpp; ++c) cs_merge(&tot, &stats[pt * cpp + c]);
        if (tot.err) status = tot.err;
        if (!status && (double)tot.n_failed > 0.001 * (double)cfg->n_paths)
            status = BW_ERR_RELIABILITY;
        out[pt].mean = tot.mean; /* finalize, wos.cpp:42-53 */
        out[pt].variance = tot.n > 1 ? tot.m2 / (double)(tot.n - 1) : 0.0;
        out[pt].n = tot.n;
        out[pt].n_infinity = tot.n_inf;
        out[pt].n_failed = tot.n_failed;
        if (steps_out) steps_out[pt] = tot.steps;
    }
    free(stats);
    free(tr);
    free(th);
    return status;
}

/* ------------------------------------------------------------------ */
/* Frames, quadrature, node and boundary-point generators              */
/* ------------------------------------------------------------------ */

/* orthonormal completion (greens.cpp:98-105, patch_solver.cpp:14-23):
 * ref = X if |axis.x| < 0.9 else Y; e1 = normalize(axis x ref); e2 = axis x e1 */
void or_frame(const double ax[3], double e1[3], double e2[3]) {
    const double ref[3] = {fabs(ax[0]) < 0.9 ? 1.0 : 0.0, fabs(ax[0]) < 0.9 ? 0.0 : 1.0, 0.0};
    double c[3] = {ax[1] * ref[2] - ax[2] * ref[1], ax[2] * ref[0] - ax[0] * ref[2],
                   ax[0] * ref[1] - ax[1] * ref[0]};
    const double n = norm3(c);
    for (int k = 0; k < 3; ++k) e1[k] = c[k] / n;
    e2[0] = ax[1] * e1[2] - ax[2] * e1[1];
    e2[1] = ax[2] * e1[0] - ax[0] * e1[2];
    e2[2] = ax[0] * e1[1] - ax[1] * e1[0];
}

/* node = c + a * ((l.x e1 + l.y e2) + l.z axis), evaluated in this order
 * (no contraction) on host and device alike. */
void or_patch_nodes(const double* centers, const double* axes, const double* radii,
                    const int32_t* cls, int64_t n_bp, const double* local_dirs, int32_t n_nodes,
                    double* out) {
    for (int64_t b = 0; b < n_bp; ++b) {
        double e1[3], e2[3];
        const double* ax = axes + 3 * b;
        or_frame(ax, e1, e2);
        const double* L = local_dirs + (size_t)(cls ? cls[b] : 0) * n_nodes * 3;
        for (int j = 0; j < n_nodes; ++j) {
            const double* l = L + 3 * j;
            for (int k = 0; k < 3; ++k) {
                double w = l[0] * e1[k] + l[1] * e2[k];
                w = w + l[2] * ax[k];
                out[(b * n_nodes + j) * 3 + k] = centers[3 * b + k] + radii[b] * w;
            }
        }
    }
}

/* gauss_legendre (quadrature.cpp:7-35): Newton on P_n from cos(pi(i-1/4)/(n+1/2)) */
int or_gauss_legendre(int n, double* nodes, double* weights) {
    if (n < 1 || n > 64) return BW_ERR_GEOMETRY;
    const int m = (n + 1) / 2;
    for (int i = 1; i <= m; ++i) {
        double z = cos(OR_PI * (i - 0.25) / (n + 0.5));
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
        } while (fabs(z - z1) > 1e-15);
        nodes[i - 1] = -z;
        nodes[n - i] = z;
        weights[i - 1] = 2.0 / ((1.0 - z * z) * pp * pp);
        weights[n - i] = weights[i - 1];
    }
    if (n % 2 == 1) nodes[n / 2] = 0.0;
    return 0;
}

/* Gamma node rule of the BASELINE configs: theta Gauss-Legendre
 * on (0, theta_max) x phi uniform 2 pi j / n_phi. dirs: n_theta*n_phi x 3
 * local unit vectors (sin t cos p, sin t sin p, cos t), row-major [i][j];
 * weights: GL weight x (theta_max/2) x (2 pi / n_phi) x sin(theta) (unit sphere
 * surface element; multiply by a^2 for radius a). */
int or_gamma_rule(int n_theta, int n_phi, double theta_max, double* dirs, double* weights) {
    double x[64], w[64];
    const int st = or_gauss_legendre(n_theta, x, w);
    if (st) return st;
    for (int i = 0; i < n_theta; ++i) {
        const double th = theta_max * 0.5 * (x[i] + 1.0);
        const double st_ = sin(th), ct = cos(th);
        for (int j = 0; j < n_phi; ++j) {
            const double ph = 2.0 * OR_PI * j / n_phi;
            double* d = dirs + 3 * (i * n_phi + j);
            d[0] = st_ * cos(ph);
            d[1] = st_ * sin(ph);
            d[2] = ct;
            if (weights) weights[i * n_phi + j] = w[i] * 0.5 * theta_max * (2.0 * OR_PI / n_phi) * st_;
        }
    }
    return 0;
}

/* Fibonacci lattice on the unit sphere:
 * z_i = 1 - (2i+1)/N, phi_i = i * pi (3 - sqrt 5) */
void or_fibonacci_sphere(int64_t n, double radius, double* out) {
    const double ga = OR_PI * (3.0 - sqrt(5.0));
    for (int64_t i = 0; i < n; ++i) {
        const double z = 1.0 - (2.0 * (double)i + 1.0) / (double)n;
        const double r = sqrt(1.0 - z * z);
        const double ph = (double)i * ga;
        out[3 * i] = radius * r * cos(ph);
        out[3 * i + 1] = radius * r * sin(ph);
        out[3 * i + 2] = radius * z;
    }
}

/* ------------------------------------------------------------------ */
/* C10 potential sum (field_eval.cpp:7-19)                             */
/* ------------------------------------------------------------------ */
/* Plain restatement: sequential sum in panel order. near[i] set when some
 * panel has d^2 < area (the reference throws NearFieldError there). */
void or_potential(const double* panels, int64_t n_panels, const double* targets, int64_t n_t,
                  double* u, uint8_t* near) {
    for (int64_t t = 0; t < n_t; ++t) {
        const double* x = targets + 3 * t;
        double sum = 0;
        int nf = 0;
        for (int64_t j = 0; j < n_panels; ++j) {
            const double* P = panels + 9 * j;
            const double r[3] = {x[0] - P[0], x[1] - P[1], x[2] - P[2]};
            const double d = norm3(r);
            if (d * d < P[6]) { nf = 1; break; }
            const double g = 1.0 / (4.0 * OR_PI * d);
            const double dg = (P[3] * r[0] + P[4] * r[1] + P[5] * r[2]) / (4.0 * OR_PI * d * d * d);
            sum += P[6] * (dg * P[7] - g * P[8]);
        }
        u[t] = nf ? NAN : sum;
        if (near) near[t] = (uint8_t)nf;
    }
}

/* Same sum with every term and the accumulator in long double (x87 64-bit
 * mantissa): the accuracy reference for the 1e-10 parity gate (SURVEY.md
 * 8(d): measure the GPU error, not the naive sequential-sum error). */
void or_potential_ld(const double* panels, int64_t n_panels, const double* targets, int64_t n_t,
                     double* u, uint8_t* near) {
    const long double inv4pi = 1.0L / (4.0L * 3.141592653589793238462643383279502884L);
    for (int64_t t = 0; t < n_t; ++t) {
        const double* x = targets + 3 * t;
        long double sum = 0;
        int nf = 0;
        for (int64_t j = 0; j < n_panels; ++j) {
            const double* P = panels + 9 * j;
            const long double r0 = (long double)x[0] - P[0], r1 = (long double)x[1] - P[1],
                              r2 = (long double)x[2] - P[2];
            const long double d2 = r0 * r0 + r1 * r1 + r2 * r2;
            if (d2 < P[6]) { nf = 1; break; }
            const long double d = sqrtl(d2);
            const long double nr = P[3] * r0 + P[4] * r1 + P[5] * r2;
            sum += (long double)P[6] * inv4pi * (nr / (d2 * d) * P[7] - P[8] / d);
        }
        u[t] = nf ? NAN : (double)sum;
        if (near) near[t] = (uint8_t)nf;
    }
}

/* ------------------------------------------------------------------ */
/* C9 dense LU with partial pivoting (Eigen::PartialPivLU as used at     */
/* patch_solver.cpp:314-324): pivot = first max |a| in the column.       */
/* ------------------------------------------------------------------ */
int or_lu_solve(int m, const double* A_in, const double* B, int nrhs, double* X, double* resid) {
    double* A = (double*)malloc(sizeof(double) * m * m);
    int* piv = (int*)malloc(sizeof(int) * m);
    memcpy(A, A_in, sizeof(double) * m * m);
    int info = 0;
    for (int k = 0; k < m; ++k) {
        int p = k;
        double best = fabs(A[k * m + k]);
        for (int i = k + 1; i < m; ++i)
            if (fabs(A[i * m + k]) > best) { best = fabs(A[i * m + k]); p = i; }
        piv[k] = p;
        if (best == 0.0) { info = 1; continue; }
        if (p != k)
            for (int j = 0; j < m; ++j) {
                const double t = A[k * m + j];
                A[k * m + j] = A[p * m + j];
                A[p * m + j] = t;
            }
        for (int i = k + 1; i < m; ++i) {
            const double l = A[i * m + k] / A[k * m + k];
            A[i * m + k] = l;
            for (int j = k + 1; j < m; ++j) A[i * m + j] -= l * A[k * m + j];
        }
    }
    for (int r = 0; r < nrhs; ++r) {
        double* x = X + (size_t)r * m;
        memcpy(x, B + (size_t)r * m, sizeof(double) * m);
        for (int k = 0; k < m; ++k) {
            const double t = x[k];
            x[k] = x[piv[k]];
            x[piv[k]] = t;
        }
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < i; ++j) x[i] -= A[i * m + j] * x[j];
        for (int i = m - 1; i >= 0; --i) {
            for (int j = i + 1; j < m; ++j) x[i] -= A[i * m + j] * x[j];
            x[i] /= A[i * m + i];
        }
    }
    if (resid) { /* ||A x0 - b0|| / max(||b0||, 1e-300), patch_solver.cpp:317-318 */
        double rn = 0, bn = 0;
        for (int i = 0; i < m; ++i) {
            double s = 0;
            for (int j = 0; j < m; ++j) s += A_in[i * m + j] * X[j];
            s -= B[i];
            rn += s * s;
            bn += B[i] * B[i];
        }
        bn = sqrt(bn);
        *resid = sqrt(rn) / (bn > 1e-300 ? bn : 1e-300);
    }
    free(A);
    free(piv);
    return info;
}

int or_lu_solve_batched(int m, int64_t n_sys, const double* A, const double* B, int nrhs,
                        double* X, double* resid, int32_t* info) {
    int any = 0;
    for (int64_t s = 0; s < n_sys; ++s) {
        info[s] = or_lu_solve(m, A + (size_t)s * m * m, B + (size_t)s * nrhs * m, nrhs,
                              X + (size_t)s * nrhs * m, resid + s);
        any |= info[s];
    }
    return any;
}
