// wos_b200.cpp — the reference's wos.hpp entry points on the B200 library.
// Links in place of proj/src/wos.cpp; every estimate runs K1 (bw_wos_estimate)
// on the reference's own Philox4x64 streams (seed, point_id, path_id), so the
// reference's call sites (point_solver.cpp:166, patch_solver.cpp:135) get the
// same walks as wos.cpp would run, with results independent of `workers`
// (wos.hpp:19,43-44).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "biewos/wos.hpp"
#include "biewos_b200_bridge.hpp"

namespace biewos {

namespace {

std::mutex g_call; // the reference's API is synchronous; one device call at a time

bw_wos_config to_bw(const WosConfig& c) {
    bw_wos_config w{};
    w.eps_shell = c.eps_shell;
    w.trunc_radius = c.trunc_radius;
    w.n_paths = c.n_paths;
    w.max_steps = c.max_steps;
    // the reference's RngStream, walk for walk; BW_RNG=philox4x32 in the
    // environment selects the library's statistical mode instead (the same
    // estimator on independent Philox4x32-10 streams, ~2.3x the rate; parity
    // with wos.cpp is then statistical)
    const char* r = std::getenv("BW_RNG");
    w.rng = (r && std::strcmp(r, "philox4x32") == 0) ? BW_RNG_PHILOX4X32 : BW_RNG_PHILOX4X64;
    w.seed = c.seed;
    w.eps_rel = 0.0;
    return w;
}

} // namespace

Real Estimate::std_error() const { // wos.hpp:28
    return n > 0 ? std::sqrt(variance / static_cast<Real>(n)) : 0.0;
}

ExitRecord walk(const Scene&, const Vec3&, const WosConfig&, RngStream&) {
    // a caller-owned stream object has no device image; the keyed overload
    // below is the one the reference's estimators use
    throw ApplicabilityError("B200 path: walk() with a caller-owned RngStream is not available; "
                             "use walk(scene, start, cfg, point_id, path_id)");
}

ExitRecord walk(const Scene& scene, const Vec3& start, const WosConfig& cfg,
                std::uint64_t point_id, std::uint64_t path_id) {
    std::vector<double> store;
    const bw_scene s = b200::to_bw(scene, store);
    const bw_wos_config w = to_bw(cfg);
    const double p[3] = {start.x(), start.y(), start.z()};
    double ex[3];
    int32_t f = 0, steps = 0;
    std::lock_guard<std::mutex> lk(g_call);
    b200::check(bw_walk(b200::context(), &s, &w, p, 1, &point_id, &path_id, ex, &f, &steps));
    return ExitRecord{Vec3(ex[0], ex[1], ex[2]), f, steps};
}

Real exit_value(const Scene& scene, const ExitRecord& rec) { // wos.hpp:37 semantics
    if (rec.feature == kExitInfinity) return 0.0;
    if (rec.feature == kExitFailed) throw ReliabilityError("no boundary value for a failed path");
    return scene.piecewise_const ? scene.feature_potential[static_cast<size_t>(rec.feature)]
                                 : scene.dirichlet(rec.point);
}

std::vector<Estimate> estimate_u_batch(const Scene& scene, const std::vector<Vec3>& points,
                                       const WosConfig& cfg, std::uint64_t point_id_base) {
    std::vector<double> store;
    const bw_scene s = b200::to_bw(scene, store);
    const bw_wos_config w = to_bw(cfg);
    std::vector<double> xyz;
    xyz.reserve(3 * points.size());
    for (const Vec3& p : points) xyz.insert(xyz.end(), {p.x(), p.y(), p.z()});
    std::vector<bw_estimate> out(points.size());
    bw_status st;
    {
        std::lock_guard<std::mutex> lk(g_call);
        st = bw_wos_estimate(b200::context(), &s, &w, xyz.data(), static_cast<int64_t>(points.size()),
                             point_id_base, out.data(), nullptr);
    }
    b200::check(st); // ReliabilityError as wos.cpp's finalize throws it
    std::vector<Estimate> est(points.size());
    for (size_t i = 0; i < points.size(); ++i) {
        est[i].mean = out[i].mean;
        est[i].variance = out[i].variance;
        est[i].n = out[i].n;
        est[i].n_infinity = out[i].n_infinity;
        est[i].n_failed = out[i].n_failed;
    }
    return est;
}

Estimate estimate_u(const Scene& scene, const Vec3& p, const WosConfig& cfg,
                    std::uint64_t point_id) {
    return estimate_u_batch(scene, {p}, cfg, point_id).front();
}

PotentialSampler wos_sampler(const Scene& scene, const WosConfig& cfg) {
    return [&scene, cfg](const Vec3& y, std::uint64_t point_id) {
        return estimate_u(scene, y, cfg, point_id);
    };
}

} // namespace biewos
