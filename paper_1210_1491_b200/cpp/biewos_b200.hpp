// biewos_b200.hpp — C++ host mirror of the reference's public API
// (proj/include/biewos/{types,geometry,wos,field_eval,patch_solver}.hpp) over the
// C-ABI of include/biewos_b200.h. Same names, argument meaning and exception
// classes as the reference; Eigen-free value types (Vec3) so it needs nothing
// but the library. Header-only; link with -lbiewos_b200.
//
//   biewos_b200::estimate_u_batch(scene, points, cfg, base)   wos.hpp:45-46
//   biewos_b200::estimate_u / walk / exit_value / wos_sampler  wos.hpp:32-50
//   biewos_b200::evaluate(data, x), evaluate_batch             field_eval.hpp:27
//   biewos_b200::lu_solve_batched                              patch_solver.cpp:314-324
//   biewos_b200::dtn_solve                                     solve_patch per point
//
// There is no CPU fallback: a missing device throws CudaError.
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/biewos_b200.h"

namespace biewos_b200 {

using Real = double;
inline constexpr Real kPi = 3.14159265358979323846; // types.hpp:16

struct Vec3 {
    Real x = 0, y = 0, z = 0;
    Vec3() = default;
    Vec3(Real a, Real b, Real c) : x(a), y(b), z(c) {}
    Real norm() const { return std::sqrt(x * x + y * y + z * z); }
    Vec3 operator-(const Vec3& o) const { return {x - o.x, y - o.y, z - o.z}; }
    Vec3 operator+(const Vec3& o) const { return {x + o.x, y + o.y, z + o.z}; }
    Vec3 operator*(Real s) const { return {x * s, y * s, z * s}; }
    Real dot(const Vec3& o) const { return x * o.x + y * o.y + z * o.z; }
};

// ---- exceptions (types.hpp:22-45) ----
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct DomainError : Error { using Error::Error; };
struct ClassificationError : Error { using Error::Error; };
struct SingularityError : Error { using Error::Error; };
struct GeometryError : Error { using Error::Error; };
struct ReliabilityError : Error { using Error::Error; };
struct ApplicabilityError : Error { using Error::Error; };
struct ExtrapolationError : Error { using Error::Error; };
struct NearFieldError : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
struct SolverError : Error { using Error::Error; };
struct CudaError : Error { using Error::Error; };

[[noreturn]] inline void throw_status(bw_status s, const std::string& msg) {
    switch (s) {
        case BW_ERR_DOMAIN: throw DomainError(msg);
        case BW_ERR_CLASSIFICATION: throw ClassificationError(msg);
        case BW_ERR_SINGULARITY: throw SingularityError(msg);
        case BW_ERR_GEOMETRY: throw GeometryError(msg);
        case BW_ERR_RELIABILITY: throw ReliabilityError(msg);
        case BW_ERR_APPLICABILITY: throw ApplicabilityError(msg);
        case BW_ERR_EXTRAPOLATION: throw ExtrapolationError(msg);
        case BW_ERR_NEARFIELD: throw NearFieldError(msg);
        case BW_ERR_CONFIG: throw ConfigError(msg);
        case BW_ERR_SOLVER: throw SolverError(msg);
        case BW_ERR_CUDA: throw CudaError(msg);
        default: throw Error(msg);
    }
}

// ---- one context per process (device 0 unless set_device is called first) ----
class Device {
public:
    static Device& get() {
        static Device d;
        return d;
    }
    bw_ctx* ctx() {
        std::call_once(once_, [this] {
            if (bw_init(device_, &ctx_) != BW_OK)
                throw CudaError("no usable sm_100 device (there is no CPU fallback)");
        });
        return ctx_;
    }
    void check(bw_status s) {
        if (s != BW_OK) throw_status(s, bw_last_error(ctx_));
    }
    static void set_device(int d) { get().device_ = d; }
    std::mutex& mutex() { return mu_; }

private:
    Device() = default;
    ~Device() {
        if (ctx_) bw_finalize(ctx_);
    }
    int device_ = 0;
    bw_ctx* ctx_ = nullptr;
    std::once_flag once_;
    std::mutex mu_; // the reference API is synchronous
};

// ---- geometry (geometry.hpp:11-64) ----
enum class SceneKind { HalfSpace = BW_SCENE_HALFSPACE, PlateSet = BW_SCENE_PLATESET,
                       ThinDisk = BW_SCENE_THINDISK, Sphere = BW_SCENE_SPHERE, Box = BW_SCENE_BOX,
                       BoxCavities = BW_SCENE_BOX_CAVITIES };

struct Plate { // geometry.hpp:14-18
    Real x0, x1, y0, y1;
    Real potential = 0.0;
};
enum class DomainSide { Exterior = BW_EXTERIOR, Interior = BW_INTERIOR };

inline constexpr int kExitInfinity = -1; // geometry.hpp:25
inline constexpr int kExitFailed = -2;   // geometry.hpp:26

// Closed-form Dirichlet data (the device cannot run a std::function).
struct Dirichlet {
    int kind = BW_PHI_FEATURE_CONST;
    Real p[16] = {0};
    static Dirichlet quadratic(Real c, Vec3 g, Real qxx, Real qyy, Real qzz, Real qxy = 0,
                               Real qxz = 0, Real qyz = 0) {
        Dirichlet d;
        d.kind = BW_PHI_QUADRATIC;
        const Real v[10] = {c, g.x, g.y, g.z, qxx, qyy, qzz, qxy, qxz, qyz};
        for (int i = 0; i < 10; ++i) d.p[i] = v[i];
        return d;
    }
    static Dirichlet point_source(Real q, Vec3 s, Real c = 0) {
        Dirichlet d;
        d.kind = BW_PHI_POINT_SOURCE;
        const Real v[5] = {q, s.x, s.y, s.z, c};
        for (int i = 0; i < 5; ++i) d.p[i] = v[i];
        return d;
    }
    static Dirichlet exp_sin_sin(Real A, Vec3 k, Vec3 origin = {}) {
        Dirichlet d;
        d.kind = BW_PHI_EXP_SIN_SIN;
        const Real v[7] = {A, k.x, k.y, k.z, origin.x, origin.y, origin.z};
        for (int i = 0; i < 7; ++i) d.p[i] = v[i];
        return d;
    }
    // A sin(m (x - x0)) sin(n (y - y0)): the four_plates_sine data (runner.cpp:318-324)
    static Dirichlet sin_sin(Real A, Real m, Real n, Real x0 = 0, Real y0 = 0) {
        Dirichlet d;
        d.kind = BW_PHI_SIN_SIN;
        const Real v[5] = {A, m, n, x0, y0};
        for (int i = 0; i < 5; ++i) d.p[i] = v[i];
        return d;
    }
    Real operator()(const Vec3& y) const {
        switch (kind) {
            case BW_PHI_SIN_SIN: return p[0] * std::sin(p[1] * (y.x - p[3])) * std::sin(p[2] * (y.y - p[4]));
            case BW_PHI_QUADRATIC:
                return p[0] + p[1] * y.x + p[2] * y.y + p[3] * y.z + p[4] * y.x * y.x +
                       p[5] * y.y * y.y + p[6] * y.z * y.z + p[7] * y.x * y.y + p[8] * y.x * y.z +
                       p[9] * y.y * y.z;
            case BW_PHI_EXP_SIN_SIN:
                return p[0] * std::exp(p[1] * (y.x - p[4])) * std::sin(p[2] * (y.y - p[5])) *
                       std::sin(p[3] * (y.z - p[6]));
            case BW_PHI_POINT_SOURCE: return p[4] + p[0] / (y - Vec3(p[1], p[2], p[3])).norm();
        }
        return std::nan("");
    }
};

struct Scene {
    SceneKind kind = SceneKind::HalfSpace;
    DomainSide side = DomainSide::Exterior;
    Real plane_z = 0, sphere_radius = 0;
    Vec3 lo, hi;
    std::vector<Real> cavities; // n x {cx, cy, cz, r}
    std::vector<Real> plates;   // n x {x0, x1, y0, y1}
    Real disk_radius = 0;
    bool piecewise_const = false;
    std::vector<Real> feature_potential;
    Dirichlet dirichlet;

    static Scene half_space(Real plane_z, Dirichlet phi) {
        Scene s;
        s.plane_z = plane_z;
        s.dirichlet = phi;
        return s;
    }
    static Scene plate_set(const std::vector<Plate>& pl) { // geometry.cpp:42-50
        Scene s;
        s.kind = SceneKind::PlateSet;
        s.piecewise_const = true;
        for (const Plate& p : pl) {
            s.plates.insert(s.plates.end(), {p.x0, p.x1, p.y0, p.y1});
            s.feature_potential.push_back(p.potential);
        }
        return s;
    }
    static Scene four_plates(const Real (&v)[4]) { // geometry.cpp:61-64
        return plate_set({Plate{0, 1, 0, 1, v[0]}, Plate{-1, 0, 0, 1, v[1]},
                          Plate{-1, 0, -1, 0, v[2]}, Plate{0, 1, -1, 0, v[3]}});
    }
    static Scene thin_disk(Real radius, Real potential) { // geometry.cpp:66-73
        Scene s;
        s.kind = SceneKind::ThinDisk;
        s.disk_radius = radius;
        s.piecewise_const = true;
        s.feature_potential = {potential};
        return s;
    }
    static Scene sphere(Real radius, DomainSide side, Real potential) {
        Scene s;
        s.kind = SceneKind::Sphere;
        s.side = side;
        s.sphere_radius = radius;
        s.piecewise_const = true;
        s.feature_potential = {potential};
        return s;
    }
    static Scene sphere(Real radius, DomainSide side, Dirichlet phi) {
        Scene s;
        s.kind = SceneKind::Sphere;
        s.side = side;
        s.sphere_radius = radius;
        s.dirichlet = phi;
        return s;
    }
    static Scene box(Vec3 lo, Vec3 hi, Dirichlet phi) {
        Scene s;
        s.kind = SceneKind::Box;
        s.side = DomainSide::Interior;
        s.lo = lo;
        s.hi = hi;
        s.dirichlet = phi;
        return s;
    }
    static Scene box_with_cavities(Vec3 lo, Vec3 hi, std::vector<Real> cav, Dirichlet phi) {
        Scene s = box(lo, hi, phi);
        s.kind = SceneKind::BoxCavities;
        s.cavities = std::move(cav);
        return s;
    }
    int feature_count() const {
        if (kind == SceneKind::Box) return 6;
        if (kind == SceneKind::BoxCavities) return 6 + (int)cavities.size() / 4;
        if (kind == SceneKind::PlateSet) return (int)plates.size() / 4;
        return 1;
    }
    bw_scene to_c() const {
        bw_scene c{};
        c.kind = (int32_t)kind;
        c.side = (int32_t)side;
        c.plane_z = plane_z;
        c.sphere_radius = sphere_radius;
        c.box_lo[0] = lo.x; c.box_lo[1] = lo.y; c.box_lo[2] = lo.z;
        c.box_hi[0] = hi.x; c.box_hi[1] = hi.y; c.box_hi[2] = hi.z;
        c.n_cavities = (int32_t)(cavities.size() / 4);
        c.cavities = cavities.empty() ? nullptr : cavities.data();
        c.n_plates = (int32_t)(plates.size() / 4);
        c.plates = plates.empty() ? nullptr : plates.data();
        c.disk_radius = disk_radius;
        if (piecewise_const) {
            c.phi_kind = BW_PHI_FEATURE_CONST;
            c.feature_potential = feature_potential.data();
        } else {
            c.phi_kind = dirichlet.kind;
            for (int i = 0; i < 16; ++i) c.phi[i] = dirichlet.p[i];
        }
        return c;
    }
};

// ---- WOS (wos.hpp:13-50) ----
struct WosConfig {
    Real eps_shell = 1e-5;
    Real trunc_radius = 1e5;
    std::int64_t n_paths = 1000;
    int max_steps = 10000;
    std::uint64_t seed = 0;
    int workers = 1; // speed only, never results (no meaning on the device)
    bw_wos_config to_c() const { return {eps_shell, trunc_radius, n_paths, max_steps, 0, seed}; }
};

struct Estimate { // identical layout to bw_estimate (wos.hpp:22-29)
    Real mean = 0;
    Real variance = 0;
    std::int64_t n = 0;
    std::int64_t n_infinity = 0;
    std::int64_t n_failed = 0;
    Real std_error() const { return n > 0 ? std::sqrt(variance / (Real)n) : 0.0; }
};
static_assert(sizeof(Estimate) == sizeof(bw_estimate), "Estimate must mirror bw_estimate");

struct ExitRecord {
    Vec3 point;
    int feature;
    int steps;
};

inline ExitRecord walk(const Scene& scene, const Vec3& start, const WosConfig& cfg,
                       std::uint64_t point_id, std::uint64_t path_id) {
    auto& d = Device::get();
    std::lock_guard<std::mutex> lk(d.mutex());
    const bw_scene sc = scene.to_c();
    const bw_wos_config c = cfg.to_c();
    double in[3] = {start.x, start.y, start.z}, out[3];
    int32_t f = 0, st = 0;
    d.check(bw_walk(d.ctx(), &sc, &c, in, 1, &point_id, &path_id, out, &f, &st));
    return {Vec3(out[0], out[1], out[2]), f, st};
}

inline Real exit_value(const Scene& scene, const ExitRecord& rec) { // wos.cpp:87-93
    if (rec.feature == kExitInfinity) return 0.0;
    if (rec.feature == kExitFailed) throw ReliabilityError("no boundary value for a failed path");
    if (scene.piecewise_const) return scene.feature_potential[(size_t)rec.feature];
    return scene.dirichlet(rec.point);
}

inline std::vector<Estimate> estimate_u_batch(const Scene& scene, const std::vector<Vec3>& points,
                                              const WosConfig& cfg,
                                              std::uint64_t point_id_base = 0) {
    std::vector<Estimate> out(points.size());
    if (points.empty()) return out;
    auto& d = Device::get();
    std::lock_guard<std::mutex> lk(d.mutex());
    const bw_scene sc = scene.to_c();
    const bw_wos_config c = cfg.to_c();
    std::vector<double> xyz(3 * points.size());
    for (size_t i = 0; i < points.size(); ++i) {
        xyz[3 * i] = points[i].x;
        xyz[3 * i + 1] = points[i].y;
        xyz[3 * i + 2] = points[i].z;
    }
    d.check(bw_wos_estimate(d.ctx(), &sc, &c, xyz.data(), (int64_t)points.size(), point_id_base,
                            reinterpret_cast<bw_estimate*>(out.data()), nullptr));
    return out;
}

inline Estimate estimate_u(const Scene& scene, const Vec3& p, const WosConfig& cfg,
                           std::uint64_t point_id = 0) {
    return estimate_u_batch(scene, {p}, cfg, point_id).front();
}

using PotentialSampler = std::function<Estimate(const Vec3& y, std::uint64_t point_id)>;
inline PotentialSampler wos_sampler(const Scene& scene, const WosConfig& cfg) {
    return [scene, cfg](const Vec3& y, std::uint64_t id) { return estimate_u(scene, y, cfg, id); };
}

// ---- potential (field_eval.hpp:12-27) ----
struct BoundaryPanel {
    Vec3 point, normal;
    Real area, u, dudn;
};
struct BoundaryData {
    std::vector<BoundaryPanel> panels;
};

inline std::vector<Real> evaluate_batch(const BoundaryData& data, const std::vector<Vec3>& x,
                                        std::vector<uint8_t>* near = nullptr) {
    auto& d = Device::get();
    std::lock_guard<std::mutex> lk(d.mutex());
    std::vector<double> P(9 * data.panels.size()), T(3 * x.size());
    for (size_t j = 0; j < data.panels.size(); ++j) {
        const auto& p = data.panels[j];
        const double v[9] = {p.point.x, p.point.y, p.point.z, p.normal.x, p.normal.y,
                             p.normal.z, p.area, p.u, p.dudn};
        for (int k = 0; k < 9; ++k) P[9 * j + k] = v[k];
    }
    for (size_t i = 0; i < x.size(); ++i) {
        T[3 * i] = x[i].x;
        T[3 * i + 1] = x[i].y;
        T[3 * i + 2] = x[i].z;
    }
    std::vector<Real> u(x.size());
    if (near) near->assign(x.size(), 0);
    d.check(bw_potential(d.ctx(), P.data(), (int64_t)data.panels.size(), T.data(),
                         (int64_t)x.size(), u.data(), near ? near->data() : nullptr));
    return u;
}

inline Real evaluate(const BoundaryData& data, const Vec3& x) { // field_eval.cpp:7-19
    return evaluate_batch(data, {x}).front();
}

// ---- dense solves (patch_solver.cpp:314-324), many systems per call ----
// A: n x m x m row-major, B: n x nrhs x m. Throws SolverError like the reference
// when any system is singular or misses the residual gate (outputs still set).
inline void lu_solve_batched(int m, int64_t n, const std::vector<Real>& A,
                             const std::vector<Real>& B, int nrhs, std::vector<Real>& X,
                             std::vector<Real>& resid, std::vector<int32_t>& info,
                             Real tol = 1e-10) {
    auto& d = Device::get();
    std::lock_guard<std::mutex> lk(d.mutex());
    X.assign(B.size(), 0.0);
    resid.assign((size_t)n, 0.0);
    info.assign((size_t)n, 0);
    d.check(bw_lu_solve_batched(d.ctx(), m, n, A.data(), B.data(), nrhs, tol, X.data(),
                                resid.data(), info.data()));
}

} // namespace biewos_b200
