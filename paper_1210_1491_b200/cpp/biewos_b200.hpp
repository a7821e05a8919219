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
    int rng = BW_RNG_PHILOX4X64; // additive: BW_RNG_PHILOX4X32 (statistical parity only)
    Real eps_rel = 0;            // additive: patch nodes use min(eps_shell, eps_rel a_b)
    bw_wos_config to_c() const {
        return {eps_shell, trunc_radius, n_paths, max_steps, rng, seed, eps_rel};
    }
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

// ---- quadrature (quadrature.cpp:7-71): host tables, as the reference builds them ----
// gauss_legendre: Newton on P_n from cos(pi (i - 1/4)/(n + 1/2)) (quadrature.cpp:7-35)
inline void gauss_legendre(int n, std::vector<Real>& x, std::vector<Real>& w) {
    if (n < 1 || n > 64) throw GeometryError("gauss_legendre: order must be in [1,64]");
    x.assign((size_t)n, 0.0);
    w.assign((size_t)n, 0.0);
    const int m = (n + 1) / 2;
    for (int i = 1; i <= m; ++i) {
        Real z = std::cos(kPi * (i - 0.25) / (n + 0.5)), pp = 0, z1;
        do {
            Real p1 = 1.0, p2 = 0.0;
            for (int j = 1; j <= n; ++j) {
                const Real p3 = p2;
                p2 = p1;
                p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
            }
            pp = n * (z * p1 - p2) / (z * z - 1.0);
            z1 = z;
            z = z1 - p1 / pp;
        } while (std::fabs(z - z1) > 1e-15);
        x[(size_t)(i - 1)] = -z;
        x[(size_t)(n - i)] = z;
        w[(size_t)(i - 1)] = 2.0 / ((1.0 - z * z) * pp * pp);
        w[(size_t)(n - i)] = w[(size_t)(i - 1)];
    }
    if (n % 2 == 1) x[(size_t)(n / 2)] = 0.0;
}

// A node rule on the unit hemisphere: local directions (n x 3) and weights.
struct NodeRule {
    std::vector<Real> dirs, weights;
    int size() const { return (int)weights.size(); }
};

// cap_rule (quadrature.cpp:37-53) for a unit radius: theta = (pi/4)(x_i + 1),
// phi = pi (x_j + 1), weight w_i w_j (pi^2/4) sin theta (times a^2 per point)
inline NodeRule cap_rule_unit(int n) {
    if (n < 2) throw GeometryError("cap_rule: need n >= 2");
    std::vector<Real> x, w;
    gauss_legendre(n, x, w);
    NodeRule r;
    for (int i = 0; i < n; ++i) {
        const Real th = kPi / 4.0 * (x[(size_t)i] + 1.0);
        const Real elem = (kPi * kPi / 4.0) * std::sin(th);
        for (int j = 0; j < n; ++j) {
            const Real ph = kPi * (x[(size_t)j] + 1.0);
            r.dirs.insert(r.dirs.end(), {std::sin(th) * std::cos(ph), std::sin(th) * std::sin(ph),
                                         std::cos(th)});
            r.weights.push_back(w[(size_t)i] * w[(size_t)j] * elem);
        }
    }
    return r;
}

// ring_rule (quadrature.cpp:55-71) in units of a: rows {rho/a, cos psi, sin psi, weight/a^2}
inline std::vector<Real> ring_rule_unit(int n, Real delta_frac) {
    if (!(delta_frac > 0) || delta_frac >= 1.0) throw GeometryError("ring_rule: need 0 < delta < a");
    std::vector<Real> x, w, out;
    gauss_legendre(n, x, w);
    for (int i = 0; i < n; ++i) {
        const Real rho = delta_frac + (1.0 - delta_frac) * 0.5 * (x[(size_t)i] + 1.0);
        const Real wr = w[(size_t)i] * 0.5 * (1.0 - delta_frac);
        for (int j = 0; j < n; ++j) {
            const Real psi = kPi * (x[(size_t)j] + 1.0);
            out.insert(out.end(), {rho, std::cos(psi), std::sin(psi), wr * w[(size_t)j] * kPi * rho});
        }
    }
    return out;
}

// The DtN Gamma rule: theta Gauss-Legendre on [0, theta_max] x uniform phi,
// unit-sphere weights (GL weight x theta_max/2 x 2 pi/n_phi x sin theta).
inline NodeRule gamma_rule(int n_theta, int n_phi, Real theta_max) {
    std::vector<Real> x, w;
    gauss_legendre(n_theta, x, w);
    NodeRule r;
    for (int i = 0; i < n_theta; ++i) {
        const Real th = theta_max * 0.5 * (x[(size_t)i] + 1.0);
        for (int j = 0; j < n_phi; ++j) {
            const Real ph = 2.0 * kPi * j / n_phi;
            r.dirs.insert(r.dirs.end(), {std::sin(th) * std::cos(ph), std::sin(th) * std::sin(ph),
                                         std::cos(th)});
            r.weights.push_back(w[(size_t)i] * (theta_max * 0.5) * (2.0 * kPi / n_phi) * std::sin(th));
        }
    }
    return r;
}

// ---- hemisphere frame (greens.hpp:11-24) and node positions ----
struct HemisphereFrame {
    Vec3 center;
    Real radius;
    Vec3 axis{0, 0, 1};
};

// y = c + a ((l.x e1 + l.y e2) + l.z axis) with (e1, e2) the completion of
// greens.cpp:98-105, in the operation order K1 uses (bit-identical nodes).
inline Vec3 node_position(const Vec3& c, const Vec3& ax, Real a, const Real* l) {
    const bool use_x = std::fabs(ax.x) < 0.9;
    const Real r0 = use_x ? 1.0 : 0.0, r1 = use_x ? 0.0 : 1.0, r2 = 0.0;
    const Real c0 = ax.y * r2 - ax.z * r1, c1 = ax.z * r0 - ax.x * r2, c2 = ax.x * r1 - ax.y * r0;
    const Real n = std::sqrt((c0 * c0 + c1 * c1) + c2 * c2);
    const Real e10 = c0 / n, e11 = c1 / n, e12 = c2 / n;
    const Real e20 = ax.y * e12 - ax.z * e11, e21 = ax.z * e10 - ax.x * e12,
               e22 = ax.x * e11 - ax.y * e10;
    return Vec3(c.x + a * ((l[0] * e10 + l[1] * e20) + l[2] * ax.x),
                c.y + a * ((l[0] * e11 + l[1] * e21) + l[2] * ax.y),
                c.z + a * ((l[0] * e12 + l[1] * e22) + l[2] * ax.z));
}

inline bw_patch flat_patch(const HemisphereFrame& f) {
    bw_patch p{};
    p.o[0] = f.center.x; p.o[1] = f.center.y; p.o[2] = f.center.z;
    p.axis[0] = f.axis.x; p.axis[1] = f.axis.y; p.axis[2] = f.axis.z;
    p.a = f.radius;
    p.surf = 1;
    return p;
}

// ---- geometry on the device (geometry.hpp:66-75, geometry.cpp:131-239) ----
struct DistanceQuery {
    Real distance;
    int feature;
};

inline DistanceQuery nearest_feature(const Scene& scene, const Vec3& p) {
    auto& d = Device::get();
    std::lock_guard<std::mutex> lk(d.mutex());
    const bw_scene sc = scene.to_c();
    const double in[3] = {p.x, p.y, p.z};
    double dist = 0;
    int32_t f = -1;
    d.check(bw_nearest_feature(d.ctx(), &sc, in, 1, &dist, &f, nullptr));
    return {dist, f};
}

inline DistanceQuery distance_to_boundary(const Scene& scene, const Vec3& p) {
    auto& d = Device::get();
    std::lock_guard<std::mutex> lk(d.mutex());
    const bw_scene sc = scene.to_c();
    const double in[3] = {p.x, p.y, p.z};
    double dist = 0;
    int32_t f = -1;
    d.check(bw_distance_to_boundary(d.ctx(), &sc, in, 1, &dist, &f));
    return {dist, f};
}

inline ExitRecord classify_exit(const Scene& scene, const Vec3& p, Real eps, Real trunc_radius) {
    auto& d = Device::get();
    std::lock_guard<std::mutex> lk(d.mutex());
    const bw_scene sc = scene.to_c();
    const double in[3] = {p.x, p.y, p.z};
    double q[3];
    int32_t f = -1;
    d.check(bw_classify_exit(d.ctx(), &sc, in, 1, eps, trunc_radius, q, &f));
    return {Vec3(q[0], q[1], q[2]), f, 0};
}

// ---- flat-boundary point formula (point_solver.hpp:8-38) ----
struct PointNeumannResult {
    Real sigma1 = 0, sigma2 = 0, total = 0, std_error = 0;
    Real a = 0, delta = 0;
    int n_g1 = 0, n_g2 = 0;
    WosConfig wos;
};

namespace detail {
inline PointNeumannResult point_formula(const Scene& scene, const HemisphereFrame& f, int n_g1,
                                        int n_g2, Real delta, const WosConfig& cfg,
                                        const NodeRule& cap, const std::vector<Estimate>& est) {
    auto& d = Device::get();
    const bw_scene sc = scene.to_c();
    const bw_patch P = flat_patch(f);
    const std::vector<Real> ring = ring_rule_unit(n_g2, delta / f.radius);
    PointNeumannResult r;
    d.check(bw_point_formula(d.ctx(), &sc, &P, 1, cap.dirs.data(), cap.weights.data(), cap.size(),
                             reinterpret_cast<const bw_estimate*>(est.data()), ring.data(),
                             (int32_t)(ring.size() / 4), &r.total, &r.sigma1, &r.sigma2,
                             &r.std_error));
    r.a = f.radius;
    r.delta = delta;
    r.n_g1 = n_g1;
    r.n_g2 = n_g2;
    r.wos = cfg;
    return r;
}
} // namespace detail

// solve_point (point_solver.cpp:195-201): K1 at the cap nodes (point ids =
// node index, as sigma1_prime's estimate_u_batch), then K6.
inline PointNeumannResult solve_point(const Scene& scene, const HemisphereFrame& f, int n_g1,
                                      int n_g2, Real delta, const WosConfig& cfg) {
    if (scene.kind == SceneKind::Sphere)
        throw ApplicabilityError("point solver requires a flat boundary scene");
    const NodeRule cap = cap_rule_unit(n_g1);
    auto& d = Device::get();
    std::lock_guard<std::mutex> lk(d.mutex());
    const bw_scene sc = scene.to_c();
    const bw_wos_config c = cfg.to_c();
    const double ctr[3] = {f.center.x, f.center.y, f.center.z};
    const double ax[3] = {f.axis.x, f.axis.y, f.axis.z};
    const double rad = f.radius;
    std::vector<Estimate> est((size_t)cap.size());
    d.check(bw_wos_patch_nodes(d.ctx(), &sc, &c, ctr, ax, &rad, nullptr, nullptr, 1,
                               cap.dirs.data(), 1, cap.size(), 0,
                               reinterpret_cast<bw_estimate*>(est.data()), nullptr));
    return detail::point_formula(scene, f, n_g1, n_g2, delta, cfg, cap, est);
}

// solve_point with a PotentialSampler (point_solver.cpp:202-208)
inline PointNeumannResult solve_point(const Scene& scene, const HemisphereFrame& f, int n_g1,
                                      int n_g2, Real delta, const WosConfig& cfg,
                                      const PotentialSampler& sampler) {
    if (scene.kind == SceneKind::Sphere)
        throw ApplicabilityError("point solver requires a flat boundary scene");
    const NodeRule cap = cap_rule_unit(n_g1);
    std::vector<Estimate> est((size_t)cap.size());
    for (int i = 0; i < cap.size(); ++i)
        est[(size_t)i] = sampler(node_position(f.center, f.axis, f.radius, &cap.dirs[3 * (size_t)i]),
                                 (std::uint64_t)i);
    auto& d = Device::get();
    std::lock_guard<std::mutex> lk(d.mutex());
    return detail::point_formula(scene, f, n_g1, n_g2, delta, cfg, cap, est);
}

// ---- last-passage estimator (last_passage.hpp:10-35) ----
struct LastPassageResult {
    Real sigma_lp = 0, std_error = 0;
    std::int64_t n_paths = 0, n_infinity = 0, n_failed = 0;
    std::vector<std::int64_t> feature_counts;
};

inline LastPassageResult estimate_lp(const Scene& scene, const HemisphereFrame& f,
                                     std::int64_t n_paths, const WosConfig& cfg,
                                     bool allow_general_data = false) {
    auto& d = Device::get();
    std::lock_guard<std::mutex> lk(d.mutex());
    const bw_scene sc = scene.to_c();
    const bw_wos_config c = cfg.to_c();
    const double ctr[3] = {f.center.x, f.center.y, f.center.z};
    const double ax[3] = {f.axis.x, f.axis.y, f.axis.z};
    LastPassageResult r;
    r.feature_counts.assign((size_t)scene.feature_count(), 0);
    bw_lp_result o{};
    d.check(bw_estimate_lp(d.ctx(), &sc, &c, ctr, f.radius, ax, n_paths, allow_general_data ? 1 : 0,
                           &o, r.feature_counts.data()));
    r.sigma_lp = o.sigma_lp;
    r.std_error = o.std_error;
    r.n_paths = o.n_paths;
    r.n_infinity = o.n_infinity;
    r.n_failed = o.n_failed;
    return r;
}

// ---- the local DtN map over many boundary points (the additive batch API) ----
enum class BieKind { FirstKind, SecondKind }; // patch_solver.hpp:61

struct DtnConfig {
    int bands = 5, azimuth = 6, gauss_polar = 20, near_depth = 2;
    Real solve_tol = 1e-10;
    BieKind kind = BieKind::SecondKind; // runner.cpp:192-193 default
    bw_dtn_config to_c() const {
        return {bands, azimuth, gauss_polar, near_depth, solve_tol,
                kind == BieKind::FirstKind ? BW_BIE_FIRST : BW_BIE_SECOND, 0};
    }
};

struct NeumannPoint {
    Real dudn;  // along the domain-outward normal (-axis)
    Real err;   // propagated WOS error
    int status; // bit0 patch nodes outside the domain, bit1 solver failure
};

// patches: one bw_patch per boundary point (o, axis into the domain, a, its
// sphere or plane, Gamma class); gamma: one node rule per class. Throws
// ReliabilityError / SolverError like the reference (results still returned
// through `out` when given).
inline std::vector<NeumannPoint> dtn_solve(const Scene& scene, const WosConfig& cfg,
                                           const DtnConfig& dtn, const std::vector<bw_patch>& patches,
                                           const std::vector<NodeRule>& gamma,
                                           std::uint64_t point_id_base = 0) {
    std::vector<NeumannPoint> out(patches.size());
    if (patches.empty()) return out;
    const int n_nodes = gamma.at(0).size();
    std::vector<Real> dirs, wts;
    for (const NodeRule& g : gamma) {
        if (g.size() != n_nodes) throw GeometryError("all Gamma classes need the same node count");
        dirs.insert(dirs.end(), g.dirs.begin(), g.dirs.end());
        wts.insert(wts.end(), g.weights.begin(), g.weights.end());
    }
    auto& d = Device::get();
    std::lock_guard<std::mutex> lk(d.mutex());
    const bw_scene sc = scene.to_c();
    const bw_wos_config c = cfg.to_c();
    const bw_dtn_config dc = dtn.to_c();
    const size_t n = patches.size();
    std::vector<Real> dudn(n), err(n);
    std::vector<int32_t> status(n);
    d.check(bw_dtn_solve(d.ctx(), &sc, &c, &dc, patches.data(), nullptr, (int64_t)n, dirs.data(),
                         wts.data(), (int32_t)gamma.size(), n_nodes, point_id_base, dudn.data(),
                         err.data(), status.data(), nullptr, nullptr));
    for (size_t i = 0; i < n; ++i) out[i] = {dudn[i], err[i], status[i]};
    return out;
}

// solve_patch (patch_solver.cpp:311-335): the per-panel Neumann field of one
// patch from its Gamma node estimates (est: one per node of `gamma`).
struct NeumannField { // patch_solver.hpp:78-82
    std::vector<Real> dudn, r, est_error; // per panel; dudn along the panel normal
    int status = 0;                       // bit0 nodes outside the domain, bit1 solver
};

inline NeumannField solve_patch(const Scene& scene, const DtnConfig& dtn, const bw_patch& patch,
                                const NodeRule& gamma, const std::vector<Estimate>& est) {
    if ((int)est.size() != gamma.size()) throw GeometryError("one estimate per Gamma node");
    auto& d = Device::get();
    std::lock_guard<std::mutex> lk(d.mutex());
    const bw_scene sc = scene.to_c();
    const bw_dtn_config dc = dtn.to_c();
    const int m = dtn.azimuth * (2 * dtn.bands - 1);
    NeumannField f;
    f.dudn.assign((size_t)m, 0.0);
    f.r.assign((size_t)m, 0.0);
    f.est_error.assign((size_t)m, 0.0);
    int32_t status = 0;
    d.check(bw_solve_patch(d.ctx(), &sc, &dc, &patch, 1, gamma.dirs.data(), gamma.weights.data(), 1,
                           gamma.size(), reinterpret_cast<const bw_estimate*>(est.data()),
                           f.dudn.data(), f.r.data(), f.est_error.data(), &status));
    f.status = status;
    return f;
}

} // namespace biewos_b200
