/*
 * biewos_b200.h — C-ABI of the B200-native BIE-WOS / local-DtN hot path.
 *
 * This is the drop-in boundary. Every entry point replaces one function of the
 * reference's public C++ API (proj/include/biewos/ headers under the reference
 * tree); the citation on each declaration names the function it replaces.
 * Plain pointers and sizes only: no torch, Eigen or std:: types cross it.
 *
 * Conventions
 *  - Every call is synchronous with respect to the host unless its name ends
 *    in `_d` (device-pointer variant, enqueued on the context stream).
 *  - Host-pointer variants copy inputs to HBM, run, and copy results back.
 *  - Errors: every call returns a bw_status. Non-OK codes map 1:1 onto the
 *    reference's exception classes (proj/include/biewos/types.hpp:22-45); the
 *    message is available from bw_last_error(ctx). There is no CPU fallback:
 *    a missing device is BW_ERR_CUDA.
 *  - Results are bitwise identical for any number of devices / launch
 *    geometry (mirrors the worker-count guarantee of wos.hpp:43-44).
 */
#ifndef BIEWOS_B200_H
#define BIEWOS_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BW_ABI_VERSION 3

/* ---- status codes: reference exception classes (types.hpp:22-45) ---- */
typedef enum bw_status {
    BW_OK = 0,
    BW_ERR_DOMAIN = 1,          /* DomainError          types.hpp:25 */
    BW_ERR_CLASSIFICATION = 2,  /* ClassificationError  types.hpp:27 */
    BW_ERR_SINGULARITY = 3,     /* SingularityError     types.hpp:29 */
    BW_ERR_GEOMETRY = 4,        /* GeometryError        types.hpp:31 */
    BW_ERR_RELIABILITY = 5,     /* ReliabilityError     types.hpp:33 */
    BW_ERR_APPLICABILITY = 6,   /* ApplicabilityError   types.hpp:35 */
    BW_ERR_EXTRAPOLATION = 7,   /* ExtrapolationError   types.hpp:37 */
    BW_ERR_NEARFIELD = 8,       /* NearFieldError       types.hpp:39 */
    BW_ERR_CONFIG = 9,          /* ConfigError          types.hpp:41 */
    BW_ERR_SOLVER = 10,         /* SolverError          types.hpp:43 */
    BW_ERR_CUDA = 64,           /* device/runtime failure (no fallback) */
    BW_ERR_INVALID = 65         /* bad argument at the C boundary */
} bw_status;

/* ---- scene: POD image of biewos::Scene (geometry.hpp:38-64) ---- */
typedef enum bw_scene_kind {
    BW_SCENE_HALFSPACE = 0,     /* z > plane_z; feature 0                    */
    BW_SCENE_PLATESET = 1,      /* zero-thickness rectangles on z = 0,
                                   feature i = plate i (geometry.hpp:14-18)  */
    BW_SCENE_THINDISK = 2,      /* disk of radius disk_radius on z = 0       */
    BW_SCENE_SPHERE = 3,        /* origin-centred sphere (geometry.hpp:45)  */
    BW_SCENE_BOX = 4,           /* interior of [lo,hi]; faces 0..5 =
                                   x=lo,x=hi,y=lo,y=hi,z=lo,z=hi             */
    BW_SCENE_BOX_CAVITIES = 5   /* box minus spherical holes; features 0..5
                                   faces, 6+i cavity i                       */
} bw_scene_kind;

typedef enum bw_side { BW_EXTERIOR = 0, BW_INTERIOR = 1 } bw_side; /* geometry.hpp:12 */

/* Closed-form Dirichlet data. The reference carries std::function phi
 * (geometry.hpp:34,49), which cannot run on a device; a scene whose data is
 * not one of these is refused with BW_ERR_APPLICABILITY (no CPU fallback). */
typedef enum bw_phi_kind {
    BW_PHI_FEATURE_CONST = 0,   /* piecewise_const: feature_potential[f]     */
    BW_PHI_QUADRATIC = 1,       /* c + g.x + Qxx x^2 + Qyy y^2 + Qzz z^2
                                   + Qxy xy + Qxz xz + Qyz yz
                                   phi = {c, gx,gy,gz, Qxx,Qyy,Qzz,Qxy,Qxz,Qyz} */
    BW_PHI_EXP_SIN_SIN = 2,     /* A exp(kx(x-x0)) sin(ky(y-y0)) sin(kz(z-z0))
                                   phi = {A, kx, ky, kz, x0, y0, z0}         */
    BW_PHI_POINT_SOURCE = 3,    /* c + q / |x - s|   phi = {q, sx,sy,sz, c}   */
    BW_PHI_SIN_SIN = 4          /* A sin(kx(x-x0)) sin(ky(y-y0))
                                   phi = {A, kx, ky, x0, y0}
                                   (runner.cpp:318-324 four_plates_sine)     */
} bw_phi_kind;

#define BW_MAX_FEATURES 1030    /* 6 faces + up to 1024 cavities */

typedef struct bw_scene {
    int32_t kind;               /* bw_scene_kind */
    int32_t side;               /* bw_side */
    double plane_z;             /* HALFSPACE */
    double sphere_radius;       /* SPHERE */
    double box_lo[3];           /* BOX, BOX_CAVITIES */
    double box_hi[3];
    int32_t n_cavities;         /* BOX_CAVITIES: <= 1024 */
    int32_t phi_kind;           /* bw_phi_kind */
    const double* cavities;     /* host: n_cavities x {cx,cy,cz,r} */
    const double* feature_potential; /* host: feature_count entries, FEATURE_CONST */
    double phi[16];
    int32_t n_plates;           /* PLATESET: <= 1024 */
    int32_t reserved;
    const double* plates;       /* host: n_plates x {x0, x1, y0, y1} */
    double disk_radius;         /* THINDISK */
} bw_scene;

/* ---- WosConfig (wos.hpp:13-20); `workers` has no meaning on device ----
 * Two additive fields (zero = the reference's behaviour):
 *  rng      BW_RNG_PHILOX4X64: the reference's RngStream (rng.hpp:44-67), bit
 *           for bit — the parity mode and the default. BW_RNG_PHILOX4X32:
 *           Philox4x32-10 (Random123 constants) keyed by (seed, point_id,
 *           path_id): counter {blk, path, lo(point), hi(point)}, one 32-bit
 *           word per uniform on the centred 2^-32 grid, so a block feeds two
 *           walk steps (and max_steps counts in whole blocks: an odd value
 *           acts as the even one below it; eps_shell must be >= 1e-9 x the
 *           boundary's size, the mode's roots carry ~3e-12); statistically
 *           equivalent, not the reference stream.
 *  eps_rel  patch nodes only (bw_wos_patch_nodes*, bw_dtn_solve*): boundary
 *           point b walks with eps_b = min(eps_shell, eps_rel * a_b), so a
 *           hemisphere shrunk near an edge keeps eps_b / a_b <= eps_rel. */
typedef enum bw_rng_kind { BW_RNG_PHILOX4X64 = 0, BW_RNG_PHILOX4X32 = 1 } bw_rng_kind;

typedef struct bw_wos_config {
    double eps_shell;           /* default 1e-5 */
    double trunc_radius;        /* default 1e5  */
    int64_t n_paths;            /* default 1000; <= 2^31 - 65 on the device */
    int32_t max_steps;          /* default 10000 */
    int32_t rng;                /* bw_rng_kind, default BW_RNG_PHILOX4X64 */
    uint64_t seed;              /* default 0 */
    double eps_rel;             /* default 0 (off) */
} bw_wos_config;

/* ---- Estimate (wos.hpp:22-29), identical field order and widths ---- */
typedef struct bw_estimate {
    double mean;
    double variance;            /* sample variance (n-1) of per-path values */
    int64_t n;
    int64_t n_infinity;
    int64_t n_failed;
} bw_estimate;

typedef struct bw_ctx bw_ctx;

/* ---- context: one per process per GPU ---- */
bw_status bw_init(int device, bw_ctx** out);
bw_status bw_finalize(bw_ctx* ctx);
/* number of kernels this context has launched (instrumentation for benches) */
bw_status bw_launch_count(const bw_ctx* ctx, uint64_t* count);
const char* bw_last_error(const bw_ctx* ctx);
/* Enqueue subsequent _d calls on this cudaStream_t (NULL = legacy default). */
bw_status bw_set_stream(bw_ctx* ctx, void* cuda_stream);
bw_status bw_synchronize(bw_ctx* ctx);
/* device properties used by the host side: SM count, clock (kHz) */
bw_status bw_device_info(bw_ctx* ctx, int32_t* sm_count, int32_t* clock_khz);
int32_t bw_abi_version(void);

/* ---- C1: Philox4x64-10 block function on device (rng.hpp:25-38) ----
 * ctr: n x 4, key: n x 2, out: n x 4 (host pointers). */
bw_status bw_philox_blocks(bw_ctx* ctx, const uint64_t* ctr, const uint64_t* key, int64_t n,
                           uint64_t* out);

/* Philox4x32-10 blocks (the BW_RNG_PHILOX4X32 block function): ctr n x 4,
 * key n x 2, out n x 4 32-bit words (host pointers; Random123 KATs). */
bw_status bw_philox4x32_blocks(bw_ctx* ctx, const uint32_t* ctr, const uint32_t* key, int64_t n,
                               uint32_t* out);

/* ---- C3/C4: geometry on the device (geometry.hpp:66-75) ----
 * nearest_feature (geometry.cpp:131-155): unsigned distance to the nearest
 * feature and its index (lowest index on ties) for n points. dist_walk
 * (optional) = the distance K1's walk loop computes for the same point
 * (cavity scenes: through the candidate grid); equal to dist up to an ulp. */
bw_status bw_nearest_feature(bw_ctx* ctx, const bw_scene* scene, const double* points,
                             int64_t n, double* dist, int32_t* feature, double* dist_walk);
/* distance_to_boundary (geometry.cpp:157-171): nearest_feature plus the domain
 * test; BW_ERR_DOMAIN (DomainError) when some point is on or outside the
 * solution domain (outputs are still written). */
bw_status bw_distance_to_boundary(bw_ctx* ctx, const bw_scene* scene, const double* points,
                                  int64_t n, double* dist, int32_t* feature);
/* classify_exit (geometry.cpp:222-239): feature -1 (kExitInfinity) beyond
 * trunc_radius, else the nearest feature and the projection onto it; a point
 * farther than eps from every feature gets -3 and the call returns
 * BW_ERR_CLASSIFICATION (ClassificationError). */
bw_status bw_classify_exit(bw_ctx* ctx, const bw_scene* scene, const double* points, int64_t n,
                           double eps, double trunc_radius, double* projected, int32_t* feature);

/* ---- C5: single trajectories (wos.hpp:32-34, wos.cpp:61-85) ----
 * One walk per entry with stream (cfg.seed, point_ids[i], path_ids[i], 0).
 * feature: >=0 feature, -1 infinity, -2 failed (geometry.hpp:25-26). */
bw_status bw_walk(bw_ctx* ctx, const bw_scene* scene, const bw_wos_config* cfg,
                  const double* starts, int64_t n, const uint64_t* point_ids,
                  const uint64_t* path_ids, double* exit_points, int32_t* features,
                  int32_t* steps);

/* ---- C5: estimate_u_batch (wos.hpp:45-46, wos.cpp:95-132) ----
 * points: n x 3 (host); out: n estimates; steps_out (optional): total WOS
 * steps per point. Point i uses point id point_id_base + i.
 * Returns BW_ERR_RELIABILITY when any point has > 0.1% failed walks
 * (wos.cpp:43-44) — `out` is still filled. */
bw_status bw_wos_estimate(bw_ctx* ctx, const bw_scene* scene, const bw_wos_config* cfg,
                          const double* points, int64_t n, uint64_t point_id_base,
                          bw_estimate* out, int64_t* steps_out);
/* device-pointer variant: d_points n x 3, d_out n estimates, d_steps (may be NULL) */
bw_status bw_wos_estimate_d(bw_ctx* ctx, const bw_scene* scene, const bw_wos_config* cfg,
                            const double* d_points, int64_t n, uint64_t point_id_base,
                            bw_estimate* d_out, int64_t* d_steps);

/* ---- hemisphere / Gamma nodes of many boundary points (sample_gamma_grid,
 * patch_solver.cpp:123-137, generalised to per-point frames) ----
 * For boundary point b with centre c_b, unit axis n_b and radius a_b the
 * node j is  y = c_b + a_b * (l.x e1 + l.y e2 + l.z n_b), l = local_dirs[cls_b][j],
 * with (e1, e2) the orthonormal completion of greens.cpp:98-105.
 * Node (b, j) uses point id point_id_base + B * n_nodes + j with B = bp_ids[b]
 * (the global index of a sharded boundary point; bp_ids == NULL means B = b),
 * so a point's streams, hence its results, do not depend on the sharding.
 * Nodes outside the solution domain are not walked: their estimate has n = 0
 * and mean = NaN. out/steps: n_bp * n_nodes, row-major [b][j]. */
bw_status bw_wos_patch_nodes(bw_ctx* ctx, const bw_scene* scene, const bw_wos_config* cfg,
                             const double* centers, const double* axes, const double* radii,
                             const int32_t* cls, const int64_t* bp_ids, int64_t n_bp,
                             const double* local_dirs, int32_t n_cls, int32_t n_nodes,
                             uint64_t point_id_base, bw_estimate* out, int64_t* steps_out);
bw_status bw_wos_patch_nodes_d(bw_ctx* ctx, const bw_scene* scene, const bw_wos_config* cfg,
                               const double* d_centers, const double* d_axes,
                               const double* d_radii, const int32_t* d_cls,
                               const int64_t* d_bp_ids, int64_t n_bp,
                               const double* d_local_dirs, int32_t n_cls, int32_t n_nodes,
                               uint64_t point_id_base, bw_estimate* d_out, int64_t* d_steps);

/* ---- C10: potential sum (field_eval.hpp:27, field_eval.cpp:7-19) ----
 * panels: n_panels x 9 doubles {px,py,pz, nx,ny,nz, area, u, dudn}
 * (BoundaryPanel field order, field_eval.hpp:12-18); targets n_t x 3.
 * A target with d^2 < area for some panel is near-field: with near != NULL
 * it is flagged (near[i] = 1, u[i] = NaN) and the call succeeds; with
 * near == NULL the call fails with BW_ERR_NEARFIELD (the reference throws). */
bw_status bw_potential(bw_ctx* ctx, const double* panels, int64_t n_panels,
                       const double* targets, int64_t n_t, double* u, uint8_t* near);
bw_status bw_potential_d(bw_ctx* ctx, const double* d_panels, int64_t n_panels,
                         const double* d_targets, int64_t n_t, double* d_u, uint8_t* d_near,
                         int64_t* d_near_count);

/* ---- C9: batched dense LU with partial pivoting + solve + residual
 * (patch_solver.cpp:314-324, Eigen::PartialPivLU) ----
 * A: n_sys x m x m row-major; B: n_sys x nrhs x m; X: same shape as B.
 * resid[s] = ||A x0 - b0|| / max(||b0||, 1e-300) for right-hand side 0.
 * info[s]: 0 ok, 1 singular pivot, 2 residual > tol or non-finite.
 * Returns BW_ERR_SOLVER when any system has info != 0 (outputs still
 * written). m <= 64. */
bw_status bw_lu_solve_batched(bw_ctx* ctx, int32_t m, int64_t n_sys, const double* A,
                              const double* B, int32_t nrhs, double tol, double* X,
                              double* resid, int32_t* info);
bw_status bw_lu_solve_batched_d(bw_ctx* ctx, int32_t m, int64_t n_sys, const double* d_A,
                                const double* d_B, int32_t nrhs, double tol, double* d_X,
                                double* d_resid, int32_t* d_info);

/* ---- local DtN: per-patch collocation (patch_solver.hpp:41-87) ----
 * One patch per boundary point (the reference builds one with
 * make_sphere_patch_setup / make_flat_patch_setup, patch_solver.cpp:62-121).
 *   o     point on the boundary (patch centre, Gamma sphere centre)
 *   axis  unit normal INTO the solution domain (the reference's
 *         "object-outward" normal, patch_solver.hpp:16,27; Gamma pole)
 *   a     Gamma sphere radius
 *   surf  0: boundary near o is the sphere |y - sc| = R (either side)
 *         1: boundary near o is the plane through o normal to axis
 *   cls   node class: row of local_dirs / weights (per-class theta_max) */
typedef struct bw_patch {
    double o[3];
    double axis[3];
    double sc[3];
    double a;
    double R;
    int32_t surf;
    int32_t cls;
} bw_patch;

/* BIE formulation of the local patch system (patch_solver.hpp:61 BieKind) */
enum { BW_BIE_SECOND = 0 /* default, runner.cpp:192-193 */, BW_BIE_FIRST = 1 };

typedef struct bw_dtn_config {
    int32_t bands;       /* mesh rings (patch_solver.hpp:41 n_bands)          */
    int32_t azimuth;     /* panels per ring; m = azimuth (2 bands - 1) <= 64   */
    int32_t gauss_polar; /* polar rule order of self panels (default 20)       */
    int32_t near_depth;  /* refinement depth of near panels (default 2)        */
    double solve_tol;    /* residual gate (patch_solver.cpp:319, 1e-10)        */
    int32_t kind;        /* BW_BIE_SECOND (default) or BW_BIE_FIRST            */
    int32_t reserved;
} bw_dtn_config;

/* Second-kind assembly (patch_solver.cpp:197-309) of all patches from the
 * Gamma node estimates of bw_wos_patch_nodes (est: n_bp x n_nodes, same
 * local_dirs; weights: n_cls x n_nodes unit-sphere weights, times a^2).
 * A: n_bp x m x m; b: n_bp x 2 x m (b, b_se); panel_area: n_bp x m;
 * flags[b] = 1 when some Gamma node lies outside the domain (clipped patch). */
bw_status bw_dtn_assemble_d(bw_ctx* ctx, const bw_scene* scene, const bw_patch* d_patches,
                            int64_t n_bp, const double* d_local_dirs, const double* d_weights,
                            int32_t n_cls, int32_t n_nodes, const bw_estimate* d_est,
                            const bw_dtn_config* cfg, double* d_A, double* d_b,
                            double* d_panel_area, int32_t* d_flags);

/* Neumann value at each boundary point from the solved patches: area-weighted
 * mean of du/dn over the fan panels around o, returned along the domain-
 * OUTWARD normal (-axis), with its WOS error |A^-1 b_se| averaged the same
 * way (solve_patch est_error, patch_solver.cpp:324).
 * status[b]: bit0 clipped patch, bit1 solver failure. */
bw_status bw_dtn_point_values_d(bw_ctx* ctx, int64_t n_bp, const bw_dtn_config* cfg,
                                const double* d_X, const double* d_panel_area,
                                const int32_t* d_info, const int32_t* d_flags, double* d_dudn,
                                double* d_err, int32_t* d_status);

/* solve_patch (patch_solver.cpp:311-335): the NeumannField of each patch
 * (patch_solver.hpp:78-82) from given Gamma node estimates — per panel du/dn
 * along the panel normal (into the solution domain), r = |centroid - o| and
 * est_error = |A^-1 b_se|; n_bp x m outputs, m = azimuth (2 bands - 1) <= 4096.
 * m <= 64 and <= 2048 nodes: K4 assembly (cfg->kind) + K2 LU; larger meshes
 * (the reference's 16 x 36 biewos_patch default): bw_patch_large.cu (the
 * environment variable BW_FORCE_LARGE_PATCH=1 routes every mesh there; a
 * test hook). Both apply the residual gate. status[b]: bit0
 * Gamma nodes outside the domain, bit1 SolverError (the call then returns
 * BW_ERR_SOLVER with the outputs written). Host pointers. */
bw_status bw_solve_patch(bw_ctx* ctx, const bw_scene* scene, const bw_dtn_config* cfg,
                         const bw_patch* patches, int64_t n_bp, const double* local_dirs,
                         const double* weights, int32_t n_cls, int32_t n_nodes,
                         const bw_estimate* est, double* dudn, double* r, double* est_error,
                         int32_t* status);

/* The whole DtN path for n_bp boundary points in one call (additive batch
 * API; the reference composes sample_gamma_grid + solve_patch per point,
 * patch_solver.cpp:123-137, 311-335): K1 WOS over every Gamma node, then the
 * Neumann stage of bw_dtn_neumann_d with BW_DTN_CLASSES (congruence-class
 * tables; BW_DTN_PER_PATCH = K4 assembly, K2 batched LU, K5 point values is
 * available through bw_dtn_neumann_d). bp_ids: global indices of the
 * points (stream ids, see bw_wos_patch_nodes) or NULL. Host pointers;
 * node_est (n_bp x n_nodes) and steps (n_bp x n_nodes) are optional. */
bw_status bw_dtn_solve(bw_ctx* ctx, const bw_scene* scene, const bw_wos_config* wos,
                       const bw_dtn_config* cfg, const bw_patch* patches, const int64_t* bp_ids,
                       int64_t n_bp, const double* local_dirs, const double* weights,
                       int32_t n_cls, int32_t n_nodes, uint64_t point_id_base, double* dudn,
                       double* err, int32_t* status, bw_estimate* node_est, int64_t* steps);
/* device-pointer variant; work buffers are owned by the context */
bw_status bw_dtn_solve_d(bw_ctx* ctx, const bw_scene* scene, const bw_wos_config* wos,
                         const bw_dtn_config* cfg, const bw_patch* d_patches,
                         const int64_t* d_bp_ids, int64_t n_bp, const double* d_local_dirs,
                         const double* d_weights, int32_t n_cls, int32_t n_nodes,
                         uint64_t point_id_base, double* d_dudn, double* d_err,
                         int32_t* d_status, bw_estimate* d_node_est, int64_t* d_steps);

/* The Neumann stage alone, from Gamma node estimates already in HBM (est:
 * n_bp x n_nodes, as bw_wos_patch_nodes_d writes them): dudn, err, status as
 * bw_dtn_point_values_d. Two methods with the same result up to rounding:
 *   BW_DTN_CLASSES    congruence-class tables: A, its LU and every quadrature
 *                     kernel value are computed once per class of rigidly
 *                     congruent patches (same surface, R, a, side, Gamma
 *                     class); per point only the data enter (K7). The residual
 *                     gate (patch_solver.cpp:317-323) is applied per class.
 *                     Falls back to BW_DTN_PER_PATCH when azimuth > 7.
 *   BW_DTN_PER_PATCH  assemble every patch (K4), batched LU (K2), point
 *                     values (K5): the reference's per-point structure,
 *                     patch_solver.cpp:197-335.
 * bw_dtn_solve / bw_dtn_solve_d use BW_DTN_CLASSES. */
enum { BW_DTN_CLASSES = 0, BW_DTN_PER_PATCH = 1 };
bw_status bw_dtn_neumann_d(bw_ctx* ctx, const bw_scene* scene, const bw_dtn_config* cfg,
                           const bw_patch* d_patches, int64_t n_bp, const double* d_local_dirs,
                           const double* d_weights, int32_t n_cls, int32_t n_nodes,
                           const bw_estimate* d_est, int32_t method, double* d_dudn,
                           double* d_err, int32_t* d_status);
/* host-array variant */
bw_status bw_dtn_neumann(bw_ctx* ctx, const bw_scene* scene, const bw_dtn_config* cfg,
                         const bw_patch* patches, int64_t n_bp, const double* local_dirs,
                         const double* weights, int32_t n_cls, int32_t n_nodes,
                         const bw_estimate* est, int32_t method, double* dudn, double* err,
                         int32_t* status);

/* ---- flat-boundary point formula (point_solver.hpp:25-38) ----
 * For each point (bw_patch o on a flat boundary piece, axis into the domain,
 * a = hemisphere radius): Sigma1' from node estimates at the cap-rule nodes
 * (cap_dirs: n_cap x 3 local unit vectors, cap_weights: n_cap unit-sphere
 * weights incl. sin(theta), est: n_bp x n_cap, e.g. from bw_wos_patch_nodes
 * with the same cap_dirs) and Sigma2' on the ring rule (ring: n_ring x
 * {rho/a, cos psi, sin psi, weight/a^2}, quadrature.cpp:55-71). total = Sigma1' + Sigma2'
 * is du/dn along -axis (the reference's convention, point_solver.hpp:8-10);
 * std_error is Sigma1's propagated WOS error (point_solver.cpp:168-172).
 * Piecewise-constant plate data use the reference's exact finite part
 * (sigma2_plates_exact, point_solver.cpp:43-114) instead of the ring rule.
 * The reference's per-point checks map to: BW_ERR_GEOMETRY (axis not normal
 * to the plane / centre off it, :14-22), BW_ERR_CLASSIFICATION (x or a ring
 * node off every feature), BW_ERR_DOMAIN (disk S_a not covered, :112/:124),
 * BW_ERR_SINGULARITY (data jump at x, :104); such points return NaN.
 * sigma1, sigma2, std_error may be NULL. */
bw_status bw_point_formula(bw_ctx* ctx, const bw_scene* scene, const bw_patch* patches,
                           int64_t n_bp, const double* cap_dirs, const double* cap_weights,
                           int32_t n_cap, const bw_estimate* est, const double* ring,
                           int32_t n_ring, double* total, double* sigma1, double* sigma2,
                           double* std_error);
bw_status bw_point_formula_d(bw_ctx* ctx, const bw_scene* scene, const bw_patch* d_patches,
                             int64_t n_bp, const double* d_cap_dirs, const double* d_cap_weights,
                             int32_t n_cap, const bw_estimate* d_est, const double* d_ring,
                             int32_t n_ring, double* d_total, double* d_sigma1,
                             double* d_sigma2, double* d_std_error);

/* ---- last-passage estimator (last_passage.hpp:10-35) ----
 * Charge density at the hemisphere centre from n_paths walks started on the
 * cap with cos-weighted density (stream domain 1, last_passage.cpp:12,77).
 * Strict mode (allow_general_data = 0) requires {0,1} piecewise-constant data
 * with the centre on a unit-potential feature (last_passage.cpp:56-64) and
 * fails with BW_ERR_APPLICABILITY otherwise. feature_counts (optional):
 * scene feature count entries. Statistics reproduce the reference's 4096-path
 * chunks and chunk-order merge exactly. */
typedef struct bw_lp_result {
    double sigma_lp;
    double std_error;
    int64_t n_paths;
    int64_t n_infinity;
    int64_t n_failed;
} bw_lp_result;

bw_status bw_estimate_lp(bw_ctx* ctx, const bw_scene* scene, const bw_wos_config* cfg,
                         const double* center, double radius, const double* axis,
                         int64_t n_paths, int32_t allow_general_data, bw_lp_result* out,
                         int64_t* feature_counts);

/* ---- diagnostics (no reference counterpart) ----
 * Measured FP64 FMA throughput of this device: a DFMA-only kernel over all
 * SMs, timed with CUDA events. The roofline denominator of the fp64 kernels
 * (MEASURED_PEAKS.json has no fp64 entry). */
bw_status bw_measure_fp64_peak(bw_ctx* ctx, double* tflops, double* kernel_ms);

/* The square root the WOS kernels use in the walk loop (sqrt_fast in
 * bw_device.cuh) beside the device's correctly rounded __dsqrt_rn, for n host
 * values (a >= 0): fast[i], rn[i]. Bitwise equal for a >= 2^-947. */
bw_status bw_diag_sqrt(bw_ctx* ctx, const double* a, int64_t n, double* fast, double* rn);

/* How often the Neumann stage (bw_dtn_solve*, bw_dtn_neumann*) found the
 * congruence classes of its patch set already built on this context: the
 * library keeps the classes (and, when they fit one table chunk, their tables)
 * of the last patch set and reuses them while the patches, the Gamma rule and
 * the mesh parameters are unchanged (compared by a device-side checksum), so
 * repeated solves on one geometry skip the patch read-back, the host
 * classification and the table build. Diagnostic. */
bw_status bw_dtn_class_cache_hits(bw_ctx* ctx, uint64_t* hits);

/* The statistical mode's (BW_RNG_PHILOX4X32) own arithmetic as K1 evaluates it:
 * root[i] = its square root of a[i] > 0 (one Newton step from the hardware
 * estimate, relative error <= 3e-12) and (sn, cs)[i] = sin, cos of the
 * azimuth 2 pi (u[i] + 1/2) 2^-32 by the table rule (absolute error <= 2e-13).
 * Host arrays; for the accuracy tests. */
bw_status bw_diag_stat_math(bw_ctx* ctx, const double* a, const uint32_t* u, int64_t n,
                            double* root, double* sn, double* cs);

/* The WOS stream blocks 0..n_blocks-1 of RngStream(seed, point_id, path_id)
 * (domain 0) as the WOS kernels form them (block table, per-walk and per-node
 * product tables, philox_wos_nt in bw_device.cuh): out n_blocks x 4. Equal to
 * bw_philox_blocks on ctr {blk, path_id, point_id, 0}, key {seed,
 * 0x1BD11BDAA9FC1A22} for every block. */
bw_status bw_diag_wos_stream(bw_ctx* ctx, uint64_t seed, uint64_t point_id, uint64_t path_id,
                             int32_t n_blocks, uint64_t* out);

/* ---- several GPUs in one process (the reference's worker-count invariance,
 * wos.hpp:19,43-44 / parallel.hpp:14-40, across devices) ----
 * A group holds one context per device and an NCCL communicator over them
 * (ncclCommInitAll; a repeated device id — one GPU standing in for several,
 * tests only — replaces NCCL by device-to-device copies). Boundary point b of
 * a batch runs on device b mod n with its global stream ids, each device's
 * shard from its own host thread; results are bitwise identical to the
 * single-device calls for any n. Status: the first hard error of any device,
 * else BW_ERR_RELIABILITY / BW_ERR_SOLVER with every output written (all
 * devices always reach the collective: a soft error on one cannot hang it). */
typedef struct bw_group bw_group;
bw_status bw_group_init(int32_t n_dev, const int32_t* devices, bw_group** out);
bw_status bw_group_finalize(bw_group* g);
bw_status bw_group_size(const bw_group* g, int32_t* n_dev, int32_t* uses_nccl);
/* the per-device context i (single-device entry points on one device) */
bw_ctx* bw_group_context(bw_group* g, int32_t i);
const char* bw_group_last_error(const bw_group* g);
bw_status bw_group_launch_count(const bw_group* g, uint64_t* count);

/* bw_dtn_solve sharded over the group (host arrays). walk_steps (optional):
 * total WOS steps; device_ms (optional): max over devices of the device time
 * of their shard (H2D, K1, K7, D2H). */
bw_status bw_group_dtn_solve(bw_group* g, const bw_scene* scene, const bw_wos_config* wos,
                             const bw_dtn_config* cfg, const bw_patch* patches,
                             const int64_t* bp_ids, int64_t n_bp, const double* local_dirs,
                             const double* weights, int32_t n_cls, int32_t n_nodes,
                             uint64_t point_id_base, double* dudn, double* err, int32_t* status,
                             int64_t* walk_steps, double* device_ms);

/* The whole BASELINE config-5 pipeline (the reference composes solve_patch
 * per point and evaluate per target, patch_solver.cpp:311-335,
 * field_eval.cpp:7-19): DtN of every boundary point (sharded as above), the
 * panel record {p, axis, area, u, -dudn} of each point (BoundaryPanel,
 * field_eval.hpp:12-18; normal and dudn into the domain; area and u_bp are the
 * caller's boundary discretisation), ncclAllGather of the records, targets
 * sharded strided and the potential K3 on each device over all panels in the
 * global order, results gathered to the host. near[i] flags near-field
 * targets (u[i] = NaN). dudn/err/status (optional): the Neumann data.
 * phase_ms (optional, 3 entries): max over devices of DtN, exchange
 * (D2H of the Neumann data, all-gather, reorder, target H2D), potential. */
bw_status bw_group_pipeline(bw_group* g, const bw_scene* scene, const bw_wos_config* wos,
                            const bw_dtn_config* cfg, const bw_patch* patches, int64_t n_bp,
                            const double* local_dirs, const double* weights, int32_t n_cls,
                            int32_t n_nodes, uint64_t point_id_base, const double* area,
                            const double* u_bp, const double* targets, int64_t n_t, double* u,
                            uint8_t* near, double* dudn, double* err, int32_t* status,
                            int64_t* walk_steps, double* phase_ms);

/* The BW_RNG_PHILOX4X32 WOS stream of (seed, point_id, path_id) as K1 forms
 * it (per-node table, per-walk product, p32_wos_block_s): out n_blocks x 2
 * 64-bit words (o0 << 32 | o1, o2 << 32 | o3) of block b, i.e. the (z,
 * azimuth) words of walk steps 2b and 2b + 1. */
bw_status bw_diag_wos_stream32(bw_ctx* ctx, uint64_t seed, uint64_t point_id, uint64_t path_id,
                               int32_t n_blocks, uint64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* BIEWOS_B200_H */
