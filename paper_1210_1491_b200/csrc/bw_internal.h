// bw_internal.h — host-side internals shared by the .cu translation units.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "bw_device.cuh"

// NVTX ranges around the phases of every entry point (header-only nvtx3: no
// link dependency; free when no tool is attached). Nsight Systems / ncu
// --nvtx show K1, the Neumann stage, the potential and the group's phases.
#include <nvtx3/nvToolsExt.h>
namespace bw {
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
} // namespace bw
#define BW_RANGE_CAT2(a, b) a##b
#define BW_RANGE_CAT(a, b) BW_RANGE_CAT2(a, b)
#define BW_RANGE(name) ::bw::NvtxRange BW_RANGE_CAT(bw_nvtx_, __LINE__)(name)

struct bw_ctx {
    int device = 0;
    int sm_count = 0;
    int clock_khz = 0;
    size_t smem_optin = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    // grow-only device scratch, one slot per purpose
    void* scratch[96] = {nullptr};
    size_t scratch_bytes[96] = {0};
    unsigned long long* d_counters = nullptr; // work counters + error flags
    unsigned long long launches = 0;          // kernels launched (bw_launch_count)
    // the cavity candidate grid of the last box scene (upload_scene): rebuilt
    // (host build, H2D, stream sync) only when the scene's geometry changes
    struct GridCache {
        bool valid = false;
        uint64_t key = 0;
        int32_t gn = 0, lpacked = 0;
        double lstep = 0, orig[3] = {0, 0, 0}, ginv = 0;
        size_t bytes = 0;
    } grid;
    // K7's congruence classes of the last patch set (dtn_neumann_classes): the
    // class keys, permutation and groups — and, when all classes fit one table
    // chunk, the class tables themselves — are reused while the patches, the
    // Gamma rule and the mesh parameters hash to the same key, so a repeated
    // solve on the same geometry does no patch D2H, no host hashing and no
    // table rebuild (one 64-byte checksum read instead)
    struct ClassCache {
        bool valid = false;
        int64_t n_bp = 0;
        int32_t bands = 0, az = 0, np = 0, depth = 0, kind = 0, n_nodes = 0, n_rule = 0;
        double tol = 0;
        uint64_t hash[8] = {0};
        int32_t n_cls = 0, chunk = 0;
        bool tables_valid = false, solver_fail = false;
        std::vector<bw_patch> canon;
        std::vector<int64_t> group_start;
        size_t n_group_words = 0;
        unsigned long long hits = 0; // diagnostic (bw_dtn_class_cache_hits)
    } cls;
};

namespace bw {

enum ScratchSlot {
    kSlotCavities = 0,
    kSlotFpot,
    kSlotCellStart,
    kSlotCellList,
    kSlotIn0,
    kSlotIn1,
    kSlotIn2,
    kSlotIn3,
    kSlotIn4,
    kSlotOut0,
    kSlotOut1,
    kSlotOut2,
    kSlotOut3,
    kSlotTmp0,
    kSlotTmp1,
    kSlotIn5,
    kSlotDtnCenters,
    kSlotDtnAxes,
    kSlotDtnRadii,
    kSlotDtnCls,
    kSlotDtnEst,
    kSlotDtnSteps,
    kSlotDtnA,
    kSlotDtnB,
    kSlotDtnX,
    kSlotDtnResid,
    kSlotDtnInfo,
    kSlotDtnArea,
    kSlotDtnFlags,
    kSlotDtnGl,
    kSlotHostIn0,
    kSlotHostIn1,
    kSlotHostIn2,
    kSlotHostIn3,
    kSlotHostOut0,
    kSlotHostOut1,
    kSlotHostOut2,
    kSlotPt0,
    kSlotPt1,
    kSlotPt2,
    kSlotPt3,
    kSlotPt4,
    kSlotPt5,
    kSlotPt6,
    kSlotPt7,
    kSlotPt8,
    kSlotLpVal,
    kSlotLpFeat,
    kSlotLpCounts,
    kSlotLpRed,
    kSlotClsPerm,
    kSlotClsGroups,
    kSlotClsCanon,
    kSlotClsMesh,
    kSlotClsA,
    kSlotClsR,
    kSlotClsZ,
    kSlotClsKg,
    kSlotClsRows,
    kSlotClsLq,
    kSlotClsH,
    kSlotClsHK,
    kSlotClsInfo,
    kSlotClsResid,
    kSlotClsHash,
    kSlotPtGl,
    kSlotPfCen,
    kSlotPfGam,
    kSlotPfA0,
    kSlotPfB0,
    kSlotCount
};

// counters layout in ctx->d_counters
enum CounterIdx {
    kCtrWork = 0,        // dynamic node queue
    kCtrReliability = 1, // nodes with > 0.1% failed walks
    kCtrClassify = 2,    // walks with a ClassificationError
    kCtrNear = 3,        // near-field targets
    kCtrGeometry = 4,    // point formula: GeometryError (point_solver.cpp:14-22)
    kCtrDomain = 5,      // point formula: DomainError (disk S_a not on the feature)
    kCtrSingular = 6,    // point formula: SingularityError (data jump at x)
    kCtrCount = 8,       // counters the launches reset
    kCtrBadClass = 8,    // sticky: patches whose cls is outside [0, n_cls) (check_classes_d)
    kCtrAlloc = 16
};

bw_status fail(bw_ctx* ctx, bw_status st, const std::string& msg);
bw_status cuda_check(bw_ctx* ctx, cudaError_t e, const char* what);
void* scratch(bw_ctx* ctx, int slot, size_t bytes, bw_status* st);

// Scene upload + candidate grid (bw_scene.cpp)
bw_status upload_scene(bw_ctx* ctx, const bw_scene* s, DevScene& out, size_t& smem_bytes);
bw_status make_wos(bw_ctx* ctx, const bw_scene* s, const bw_wos_config* c, DevWos& out);

// Kernel launchers (bw_wos.cu, bw_potential.cu, bw_lu.cu)
struct NodeSource {
    const double* xyz;     // explicit points (n x 3) or nullptr
    const double* centers; // patch mode: n_bp x 3
    const double* axes;    // n_bp x 3
    const double* radii;   // n_bp
    const int32_t* cls;    // n_bp (or nullptr -> class 0)
    const int64_t* bp_ids; // n_bp global indices (or nullptr -> identity)
    const double* dirs;    // n_cls x n_nodes x 3
    int32_t n_nodes;       // nodes per boundary point (patch mode)
    int32_t check_domain;  // skip nodes outside the domain (patch mode)
    int32_t n_cls;         // rows of dirs (bounds checks; 0 = unknown)
};

cudaError_t init_trig_table(); // bw_wos.cu: FAST sincos table of the current device
cudaError_t launch_stat_math(bw_ctx* ctx, const double* a, const uint32_t* u, int64_t n,
                             double* root, double* sn, double* cs); // bw_wos.cu (diagnostic)
cudaError_t launch_wos(bw_ctx* ctx, const DevScene& S, size_t smem_scene, const DevWos& W,
                       const NodeSource& src, int64_t n_nodes_total, uint64_t pid_base,
                       bw_estimate* out, int64_t* steps);
cudaError_t launch_geometry(bw_ctx* ctx, const DevScene& S, size_t smem, const double* pts,
                            int64_t n, double eps, double trunc, double* dist, int32_t* feat,
                            double* dist_walk, double* proj, int32_t* exit_feat,
                            int check_domain);
cudaError_t launch_walk(bw_ctx* ctx, const DevScene& S, size_t smem_scene, const DevWos& W,
                        const double* starts, int64_t n, const uint64_t* pids,
                        const uint64_t* paths, double* exit_pts, int32_t* feat, int32_t* steps);
cudaError_t launch_philox(bw_ctx* ctx, const uint64_t* ctr, const uint64_t* key, int64_t n,
                          uint64_t* out);
cudaError_t launch_potential(bw_ctx* ctx, const double* panels, int64_t n_panels,
                             const double* targets, int64_t n_t, double* u, uint8_t* near,
                             int64_t* near_count);
cudaError_t launch_dfma(bw_ctx* ctx, double* tflops, double* ms);
cudaError_t launch_unpack_patches(bw_ctx* ctx, const bw_patch* patches, int64_t n, double* centers,
                                  double* axes, double* radii, int32_t* cls);
// counts patches with cls outside [0, n_cls) into d_counters[kCtrBadClass]
cudaError_t launch_check_classes(bw_ctx* ctx, const bw_patch* patches, int64_t n, int32_t n_cls);
cudaError_t launch_assemble(bw_ctx* ctx, const DevScene& S, const bw_patch* patches, int64_t n_bp,
                            const double* dirs, const double* wts, int n_nodes,
                            const bw_estimate* est, int bands, int az, int gauss_polar,
                            int near_depth, int kind, const double* d_gl, double* A, double* b,
                            double* area, double* cen, int32_t* flags);
// large-patch solve_patch path (bw_patch_large.cu)
size_t large_patch_smem(int bands, int az, int np);
cudaError_t launch_gamma_nodes(bw_ctx* ctx, const bw_patch* patches, int64_t n_bp,
                               const double* dirs, const double* wts, int n_nodes,
                               const bw_estimate* est, double* gam, int32_t* flags);
cudaError_t launch_assemble_large(bw_ctx* ctx, const DevScene& S, const bw_patch* patches,
                                  int64_t n_bp, const double* gam, int n_nodes, int bands, int az,
                                  int np, int depth, int kind, const double* gl, double* A,
                                  double* b, double* cen);
cudaError_t launch_lu_large(bw_ctx* ctx, int m, int64_t n_sys, double* A, double* B,
                            const double* A0, const double* B0, double tol, double* X,
                            double* resid, int32_t* info);
cudaError_t launch_patch_field(bw_ctx* ctx, int64_t n_bp, int m, const bw_patch* patches,
                               const double* X, const double* cen, double* dudn, double* r,
                               double* est_error);
cudaError_t launch_point_formula(bw_ctx* ctx, const DevScene& S, const bw_patch* patches,
                                 int64_t n_bp, const double* cap_dirs, const double* cap_w,
                                 int n_cap, const bw_estimate* est, const double* ring,
                                 int n_ring, const double* gl20, double* total, double* s1,
                                 double* s2, double* se);
cudaError_t launch_dirichlet(bw_ctx* ctx, const DevScene& S, size_t smem, const double* x,
                             double tol, double* d_out);
cudaError_t launch_lp(bw_ctx* ctx, const DevScene& S, size_t smem, const DevWos& W,
                      const double* c, double a, const double* ax, int64_t n_paths, double phix,
                      double* val, int32_t* feat, unsigned long long* counts, double* red);
cudaError_t launch_point_values(bw_ctx* ctx, int64_t n_bp, int m, int az, const double* X,
                                const double* area, const int32_t* info, const int32_t* flags,
                                double* dudn, double* err, int32_t* status);
cudaError_t launch_lu(bw_ctx* ctx, int m, int64_t n_sys, const double* A, const double* B,
                      int nrhs, double tol, double* X, double* resid, int32_t* info);

// Neumann stage through congruence-class tables (bw_dtn_class.cu)
bw_status dtn_neumann_classes(bw_ctx* ctx, const DevScene& S, const bw_patch* d_patches,
                              int64_t n_bp, const double* d_dirs, const double* d_weights,
                              int32_t n_rule, int32_t n_nodes, const bw_estimate* d_est, int bands, int az,
                              int np, int depth, int kind, double tol, const double* d_gl,
                              double* d_dudn,
                              double* d_err, int32_t* d_status, bool* applicable);

} // namespace bw
