// bridge_b200.cpp — Scene -> bw_scene, the closed-form side table, the device
// context and the status -> exception mapping (biewos_b200_bridge.hpp).
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "biewos/types.hpp"
#include "biewos_b200_bridge.hpp"

namespace biewos::b200 {

namespace {

struct ClosedForm {
    int kind;
    double c[16];
};

std::mutex g_mu;
std::unordered_map<const Scene*, ClosedForm>& table() {
    static std::unordered_map<const Scene*, ClosedForm> t;
    return t;
}

} // namespace

void set_dirichlet(const Scene& scene, int kind, const double* coeffs16) {
    ClosedForm f{kind, {}};
    std::memcpy(f.c, coeffs16, sizeof f.c);
    std::lock_guard<std::mutex> lk(g_mu);
    table()[&scene] = f;
}

void clear_dirichlet(const Scene& scene) {
    std::lock_guard<std::mutex> lk(g_mu);
    table().erase(&scene);
}

bw_scene to_bw(const Scene& s, std::vector<double>& storage) {
    bw_scene c{};
    c.side = s.side == DomainSide::Interior ? BW_INTERIOR : BW_EXTERIOR;
    storage.clear();
    switch (s.kind) {
        case SceneKind::HalfSpace:
            c.kind = BW_SCENE_HALFSPACE;
            c.plane_z = s.plane_z;
            break;
        case SceneKind::PlateSet:
            c.kind = BW_SCENE_PLATESET;
            c.n_plates = static_cast<int32_t>(s.plates.size());
            for (const Plate& p : s.plates) storage.insert(storage.end(), {p.x0, p.x1, p.y0, p.y1});
            break;
        case SceneKind::ThinDisk:
            c.kind = BW_SCENE_THINDISK;
            c.disk_radius = s.disk_radius;
            break;
        case SceneKind::Sphere:
            c.kind = BW_SCENE_SPHERE;
            c.sphere_radius = s.sphere_radius;
            break;
    }
    const size_t n_geo = storage.size();
    if (s.piecewise_const) {
        c.phi_kind = BW_PHI_FEATURE_CONST;
        storage.insert(storage.end(), s.feature_potential.begin(), s.feature_potential.end());
    } else {
        std::lock_guard<std::mutex> lk(g_mu);
        const auto it = table().find(&s);
        if (it == table().end())
            throw ApplicabilityError(
                "B200 path: the scene's Dirichlet data is an opaque std::function; declare its "
                "closed form with biewos::b200::set_dirichlet (no CPU fallback)");
        c.phi_kind = it->second.kind;
        std::memcpy(c.phi, it->second.c, sizeof c.phi);
    }
    // pointers last: storage no longer grows
    if (s.kind == SceneKind::PlateSet) c.plates = storage.data();
    if (s.piecewise_const) c.feature_potential = storage.data() + n_geo;
    return c;
}

bw_ctx* context() {
    static bw_ctx* ctx = [] {
        const char* e = std::getenv("BW_DEVICE");
        bw_ctx* c = nullptr;
        const bw_status st = bw_init(e ? std::atoi(e) : 0, &c);
        if (st != BW_OK) check(st);
        return c;
    }();
    return ctx;
}

void check(bw_status st) {
    if (st == BW_OK) return;
    const std::string m = std::string("B200: ") + bw_last_error(context());
    switch (st) {
        case BW_ERR_DOMAIN: throw DomainError(m);
        case BW_ERR_CLASSIFICATION: throw ClassificationError(m);
        case BW_ERR_SINGULARITY: throw SingularityError(m);
        case BW_ERR_GEOMETRY: throw GeometryError(m);
        case BW_ERR_RELIABILITY: throw ReliabilityError(m);
        case BW_ERR_APPLICABILITY: throw ApplicabilityError(m);
        case BW_ERR_EXTRAPOLATION: throw ExtrapolationError(m);
        case BW_ERR_NEARFIELD: throw NearFieldError(m);
        case BW_ERR_CONFIG: throw ConfigError(m);
        case BW_ERR_SOLVER: throw SolverError(m);
        default: throw Error(m + " (status " + std::to_string(static_cast<int>(st)) + ")");
    }
}

} // namespace biewos::b200
