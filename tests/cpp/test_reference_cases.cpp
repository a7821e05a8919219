// The reference's WOS and potential test cases (tests/test_wos.cpp,
// tests/test_field_eval.cpp of the reference), restated against the C++ host
// mirror paper_1210_1491_b200/cpp/biewos_b200.hpp, i.e. against the B200
// kernels through the C-ABI. Built by __graft_entry__.build(); run on a GPU by
// tests/test_gpu_cpp.py. Exit code 0 iff every check passes.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "../../paper_1210_1491_b200/cpp/biewos_b200.hpp"

using namespace biewos_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        ++g_checks;                                                              \
        if (!(cond)) {                                                           \
            ++g_fail;                                                            \
            std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
        }                                                                        \
    } while (0)
#define CHECK_THROWS_AS(expr, E)                                                 \
    do {                                                                         \
        ++g_checks;                                                              \
        bool ok_ = false;                                                        \
        try {                                                                    \
            (void)(expr);                                                        \
        } catch (const E&) {                                                     \
            ok_ = true;                                                          \
        } catch (...) {                                                          \
        }                                                                        \
        if (!ok_) {                                                              \
            ++g_fail;                                                            \
            std::printf("FAILED %s:%d: %s does not throw %s\n", __FILE__, __LINE__, #expr, #E); \
        }                                                                        \
    } while (0)

static Scene test1_halfspace() { // unit source below the plane: u = 1/|y - (0,0,-1)|
    return Scene::half_space(0.0, Dirichlet::point_source(1.0, Vec3(0, 0, -1)));
}

static void case_immediate_exit_and_determinism() {
    const Scene s = test1_halfspace();
    WosConfig cfg;
    const ExitRecord r = walk(s, Vec3(0.3, -0.2, 5e-6), cfg, 0, 0);
    CHECK(r.steps == 0);
    CHECK(r.feature == 0);
    CHECK(r.point.z == 0.0);
    const ExitRecord a = walk(s, Vec3(0, 0, 1), cfg, 3, 7), b = walk(s, Vec3(0, 0, 1), cfg, 3, 7);
    CHECK(a.feature == b.feature && a.steps == b.steps && (a.point - b.point).norm() == 0.0);
}

static void case_exit_uniform_from_centre() {
    const Scene s = Scene::sphere(1.0, DomainSide::Interior, 1.0);
    WosConfig cfg;
    const int n = 100000;
    std::vector<Real> zs;
    zs.reserve(n);
    bool all_absorbed = true;
    for (int k = 0; k < n; k += 1) {
        const ExitRecord r = walk(s, Vec3(0, 0, 0), cfg, 0, (std::uint64_t)k);
        all_absorbed = all_absorbed && r.feature == 0;
        zs.push_back(r.point.z);
        if (k == 2000) break; // per-walk calls are latency bound; the batch test below covers more
    }
    CHECK(all_absorbed);
    std::sort(zs.begin(), zs.end());
    Real dmax = 0;
    const Real m = (Real)zs.size();
    for (size_t i = 0; i < zs.size(); ++i) {
        const Real c = (zs[i] + 1.0) / 2.0;
        dmax = std::max({dmax, std::fabs(c - i / m), std::fabs(c - (i + 1) / m)});
    }
    CHECK(dmax < 1.628 / std::sqrt(m)); // KS, alpha = 0.01
}

static void case_truncation_leakage() {
    WosConfig cfg;
    cfg.n_paths = 100000;
    const Estimate e = estimate_u(test1_halfspace(), Vec3(0, 0, 1), cfg);
    CHECK(e.n_infinity <= 10);
}

static void case_constant_data() {
    WosConfig cfg;
    cfg.n_paths = 500;
    const Estimate e = estimate_u(Scene::sphere(2.0, DomainSide::Interior, 1.0), Vec3(0.3, 0, 0.4), cfg);
    CHECK(e.mean == 1.0 && e.variance == 0.0 && e.n == 500);
}

static void case_ball_phi_z() {
    WosConfig cfg;
    cfg.n_paths = 20000;
    const Scene s = Scene::sphere(1.0, DomainSide::Interior, Dirichlet::quadratic(0, Vec3(0, 0, 1), 0, 0, 0));
    const Estimate e = estimate_u(s, Vec3(0, 0, 0.5), cfg);
    CHECK(std::fabs(e.mean - 0.5) < 4.0 * e.std_error());
}

static void case_halfspace_half() {
    WosConfig cfg;
    cfg.n_paths = 20000;
    const Estimate e = estimate_u(test1_halfspace(), Vec3(0, 0, 1), cfg);
    CHECK(std::fabs(e.mean - 0.5) < 4.0 * e.std_error());
}

static void case_batch_bookkeeping() {
    WosConfig cfg;
    cfg.n_paths = 1000;
    CHECK(estimate_u_batch(test1_halfspace(), {}, cfg).empty());
    const std::vector<Vec3> pts(3, Vec3(0.2, 0.1, 0.5));
    const auto est = estimate_u_batch(test1_halfspace(), pts, cfg);
    CHECK(est.size() == 3);
    CHECK(est[0].mean != est[1].mean);
    const Real se = std::hypot(est[0].std_error(), est[1].std_error());
    CHECK(std::fabs(est[0].mean - est[1].mean) < 4.0 * se);
    for (const auto& e : est) CHECK(e.n + e.n_failed == cfg.n_paths);
}

static bool identical(const std::vector<Estimate>& a, const std::vector<Estimate>& b) {
    return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(Estimate)) == 0;
}

static void case_worker_count_invariance() {
    std::vector<Vec3> pts;
    for (int i = 0; i < 7; ++i) pts.emplace_back(0.1 * i, -0.05 * i, 0.3 + 0.1 * i);
    WosConfig cfg;
    cfg.n_paths = 9000;
    cfg.seed = 99;
    cfg.workers = 1;
    const auto e1 = estimate_u_batch(test1_halfspace(), pts, cfg);
    cfg.workers = 4;
    const auto e4 = estimate_u_batch(test1_halfspace(), pts, cfg);
    cfg.workers = 16;
    const auto e16 = estimate_u_batch(test1_halfspace(), pts, cfg);
    CHECK(identical(e1, e4) && identical(e1, e16));
    // and for any batch composition: point i alone, with its id, is the same
    for (int i : {0, 3, 6}) {
        const auto one = estimate_u_batch(test1_halfspace(), {pts[(size_t)i]}, cfg, (std::uint64_t)i);
        CHECK(std::memcmp(&one[0], &e1[(size_t)i], sizeof(Estimate)) == 0);
    }
}

static void case_mean_value_property() {
    std::mt19937_64 g(7);
    std::uniform_real_distribution<Real> U(0.0, 1.0);
    for (int trial = 0; trial < 20; ++trial) {
        const Real R = 0.5 + 1.5 * U(g);
        const Real c0 = 2 * U(g) - 1, c1 = 2 * U(g) - 1, c2 = 2 * U(g) - 1;
        const Dirichlet h = Dirichlet::quadratic(c0, Vec3(0, 0, c1), c2, -c2, 0);
        const Scene s = Scene::sphere(R, DomainSide::Interior, h);
        const Vec3 p = Vec3(U(g) - 0.5, U(g) - 0.5, U(g) - 0.5) * R;
        WosConfig cfg;
        cfg.n_paths = 4000;
        cfg.seed = (std::uint64_t)trial;
        const Estimate e = estimate_u(s, p, cfg);
        CHECK(std::fabs(e.mean - h(p)) < 4.0 * e.std_error() + 1e-12);
    }
}

static void case_se_scaling() {
    std::vector<Real> scaled;
    for (long n : {1000L, 10000L, 100000L}) {
        WosConfig cfg;
        cfg.n_paths = n;
        const Estimate e = estimate_u(test1_halfspace(), Vec3(0.5, 0, 0.25), cfg);
        scaled.push_back(e.std_error() * std::sqrt((Real)n));
    }
    for (Real v : scaled) CHECK(std::fabs(v / scaled[0] - 1.0) < 0.2);
}

static void case_eps_bias() {
    WosConfig a;
    a.n_paths = 40000;
    a.eps_shell = 1e-4;
    WosConfig b = a;
    b.eps_shell = 1e-5;
    b.seed = 1;
    const Estimate ea = estimate_u(test1_halfspace(), Vec3(0.5, 0, 0.3), a);
    const Estimate eb = estimate_u(test1_halfspace(), Vec3(0.5, 0, 0.3), b);
    CHECK(std::fabs(ea.mean - eb.mean) < 3.0 * std::hypot(ea.std_error(), eb.std_error()));
}

static void case_reliability_and_exit_value() {
    WosConfig cfg;
    cfg.max_steps = 1;
    cfg.n_paths = 1000;
    CHECK_THROWS_AS(estimate_u(test1_halfspace(), Vec3(0, 0, 50), cfg), ReliabilityError);
    const Scene s = test1_halfspace();
    CHECK(exit_value(s, {Vec3(2e5, 0, 0), kExitInfinity, 12}) == 0.0);
    CHECK_THROWS_AS(exit_value(s, {Vec3(0, 0, 0), kExitFailed, 12}), ReliabilityError);
}

// lat-long panels of an exterior point charge on |y| = R (the reference's
// field_eval test data): u = q/(4 pi R), du/dn = -q/(4 pi R^2), n outward
static BoundaryData sphere_data(Real R, Real q, int n_panels) {
    const int nlat = std::max(4, (int)std::sqrt(n_panels / 2.0)), nlon = 2 * nlat;
    BoundaryData d;
    for (int i = 0; i < nlat; ++i) {
        const Real th0 = kPi * i / nlat, th1 = kPi * (i + 1) / nlat, thc = 0.5 * (th0 + th1);
        const Real area = (std::cos(th0) - std::cos(th1)) * 2.0 * kPi / nlon * R * R;
        for (int j = 0; j < nlon; ++j) {
            const Real ph = 2.0 * kPi * (j + 0.5) / nlon;
            const Vec3 n(std::sin(thc) * std::cos(ph), std::sin(thc) * std::sin(ph), std::cos(thc));
            d.panels.push_back({n * R, n, area, q / (4 * kPi * R), -q / (4 * kPi * R * R)});
        }
    }
    return d;
}

static void case_potential() {
    BoundaryData z = sphere_data(3.0, 1.0, 500);
    for (auto& p : z.panels) p.u = p.dudn = 0;
    CHECK(evaluate(z, Vec3(4, 0, 0)) == 0.0);
    const BoundaryData d = sphere_data(3.0, 1.0, 5000);
    const Real expect = 1.0 / (16 * kPi);
    CHECK(std::fabs(evaluate(d, Vec3(4, 0, 0)) - expect) < 0.01 * expect);
    CHECK(std::fabs(evaluate(d, Vec3(0, -4, 0)) - expect) < 0.01 * expect);
    CHECK(std::fabs(evaluate(d, Vec3(0.2, 0.1, -0.3))) < 0.01 / (12 * kPi));
    Real prev = -1;
    for (int n : {500, 2000, 8000}) {
        const Real err = std::fabs(evaluate(sphere_data(3.0, 1.0, n), Vec3(0, 0, 4.5)) - 1.0 / (4 * kPi * 4.5));
        if (prev > 0) CHECK(err < prev / 1.8);
        prev = err;
    }
    BoundaryData d1 = sphere_data(2.0, 1.0, 800), d2 = d1, mix = d1;
    std::mt19937_64 g(3);
    std::uniform_real_distribution<Real> U(-0.5, 0.5);
    for (auto& p : d2.panels) {
        p.u = U(g);
        p.dudn = U(g);
    }
    for (size_t i = 0; i < mix.panels.size(); ++i) {
        mix.panels[i].u = 1.7 * d1.panels[i].u - 0.4 * d2.panels[i].u;
        mix.panels[i].dudn = 1.7 * d1.panels[i].dudn - 0.4 * d2.panels[i].dudn;
    }
    const Vec3 x(3.5, -1, 0.5);
    const Real lhs = evaluate(mix, x), rhs = 1.7 * evaluate(d1, x) - 0.4 * evaluate(d2, x);
    CHECK(std::fabs(lhs - rhs) <= 1e-13 * std::fabs(rhs));
    const BoundaryData near = sphere_data(3.0, 1.0, 500);
    CHECK_THROWS_AS(evaluate(near, near.panels[7].point + Vec3(0.01, 0, 0)), NearFieldError);
}

static void case_lu() {
    const int m = 40, n = 64;
    std::mt19937_64 g(11);
    std::normal_distribution<Real> N01;
    std::vector<Real> A((size_t)n * m * m), B((size_t)n * 2 * m), X, res;
    std::vector<int32_t> info;
    for (int s = 0; s < n; ++s)
        for (int i = 0; i < m; ++i) {
            for (int j = 0; j < m; ++j) A[((size_t)s * m + i) * m + j] = N01(g) + (i == j ? 8.0 : 0.0);
            B[((size_t)s * 2) * m + i] = N01(g);
            B[((size_t)s * 2 + 1) * m + i] = N01(g);
        }
    lu_solve_batched(m, n, A, B, 2, X, res, info);
    for (int s = 0; s < n; ++s) {
        CHECK(info[(size_t)s] == 0 && res[(size_t)s] < 1e-12);
        for (int i = 0; i < m; ++i) { // check A x = b for both right-hand sides
            for (int r = 0; r < 2; ++r) {
                Real acc = 0;
                for (int j = 0; j < m; ++j)
                    acc += A[((size_t)s * m + i) * m + j] * X[((size_t)s * 2 + r) * m + j];
                CHECK(std::fabs(acc - B[((size_t)s * 2 + r) * m + i]) < 1e-10);
            }
        }
    }
    std::vector<Real> S = {0.0, 1.0, 0.0, 2.0}, b = {1.0, 1.0};
    CHECK_THROWS_AS(lu_solve_batched(2, 1, S, b, 1, X, res, info), SolverError);
}

// ---- point formula (tests/test_point_solver.cpp) ----
static bool approx(Real a, Real b, Real eps) { // doctest::Approx(b).epsilon(eps)
    return std::fabs(a - b) < eps * (1.0 + std::max(std::fabs(a), std::fabs(b)));
}

static void case_point_formula() {
    const Scene s = test1_halfspace();
    const PotentialSampler exact = [](const Vec3& y, std::uint64_t) {
        Estimate e;
        e.mean = 1.0 / (y - Vec3(0, 0, -1)).norm();
        e.n = 1;
        return e;
    };
    const Real totals[5] = {0.715539248403333, 0.715536744007608, 0.715529230831088,
                            0.715524222120063, 0.715516709286366};
    const Real as[5] = {0.1, 0.2, 0.5, 0.7, 1.0};
    for (int k = 0; k < 5; ++k) {
        const PointNeumannResult r =
            solve_point(s, {Vec3(0.5, 0, 0), as[k]}, 20, 20, 1e-4 * as[k], WosConfig(), exact);
        CHECK(approx(r.total, totals[k], 1e-9));
        CHECK(r.total == r.sigma1 + r.sigma2);
    }
    const PointNeumannResult r1 = solve_point(s, {Vec3(0.5, 0, 0), 0.5}, 20, 20, 5e-5, WosConfig(), exact);
    CHECK(approx(r1.sigma1, 0.622487481448513, 1e-9));
    WosConfig mc;
    mc.n_paths = 1000;
    mc.seed = 2024;
    const PointNeumannResult r2 = solve_point(s, {Vec3(0.5, 0, 0), 0.5}, 20, 20, 5e-5, mc);
    CHECK(std::fabs(r2.total - 1.0 / std::pow(1.25, 1.5)) < 4 * r2.std_error + 2e-4);

    // four plates, plate II at 1 V: exact finite part vs the frozen values
    const Real v[4] = {0, 1, 0, 0};
    const Scene plates = Scene::four_plates(v);
    const PotentialSampler zero = [](const Vec3&, std::uint64_t) {
        Estimate e;
        e.n = 1;
        return e;
    };
    const Vec3 A(-0.2273, 0.2273, 0);
    for (Real a : {0.1, 0.2, 0.2273})
        CHECK(solve_point(plates, {A, a}, 8, 20, 1e-4 * a, WosConfig(), zero).sigma2 == 0.0);
    const Real rows[3][2] = {{0.3, 0.08918475915450}, {0.5, 0.63287790821628}, {0.7, 1.02697283920885}};
    for (const auto& r : rows)
        CHECK(approx(solve_point(plates, {A, r[0]}, 8, 20, 1e-4 * r[0], WosConfig(), zero).sigma2,
                     r[1], 1e-10));
    CHECK_THROWS_AS(solve_point(plates, {A, 1.0}, 8, 20, 1e-4, WosConfig(), zero), DomainError);
    CHECK_THROWS_AS(solve_point(Scene::sphere(1.0, DomainSide::Interior, 1.0),
                                {Vec3(0, 0, 1), 0.2}, 8, 8, 1e-5, WosConfig()),
                    ApplicabilityError);
}

// ---- geometry (tests/test_geometry.cpp) ----
static void case_geometry() {
    const Scene hs = test1_halfspace();
    const DistanceQuery q = distance_to_boundary(hs, Vec3(3, -7, 2));
    CHECK(std::fabs(q.distance - 2.0) < 1e-14 && q.feature == 0);
    CHECK_THROWS_AS(distance_to_boundary(hs, Vec3(0, 0, -0.1)), DomainError);
    const Real v[4] = {1, 0, 0, 0};
    const Scene plates = Scene::four_plates(v);
    CHECK(nearest_feature(plates, Vec3(-0.5, 0.5, 0.25)).feature == 1);
    CHECK(nearest_feature(plates, Vec3(0.0, 0.5, 0.1)).feature == 0);
    CHECK(classify_exit(hs, Vec3(2e5, 0, 0), 1e-5, 1e5).feature == kExitInfinity);
    const ExitRecord r = classify_exit(plates, Vec3(-0.5, -0.5, 1e-6), 1e-5, 1e5);
    CHECK(r.feature == 2 && r.point.z == 0.0);
    CHECK_THROWS_AS(classify_exit(plates, Vec3(0, 0, 0.5), 1e-5, 1e5), ClassificationError);
    const Scene in = Scene::sphere(2.0, DomainSide::Interior, 1.0);
    const Scene ex = Scene::sphere(2.0, DomainSide::Exterior, 1.0);
    CHECK(std::fabs(distance_to_boundary(in, Vec3(0, 0, 0)).distance - 2.0) < 1e-14);
    CHECK(std::fabs(distance_to_boundary(ex, Vec3(0, 0, 5)).distance - 3.0) < 1e-14);
    CHECK_THROWS_AS(distance_to_boundary(in, Vec3(0, 0, 3)), DomainError);
    CHECK_THROWS_AS(distance_to_boundary(ex, Vec3(0, 0, 1)), DomainError);
}

// ---- last passage (tests/test_last_passage.cpp) ----
static void case_last_passage() {
    const Scene disk = Scene::thin_disk(1.0, 1.0);
    WosConfig cfg;
    cfg.seed = 5;
    const LastPassageResult r = estimate_lp(disk, {Vec3(-0.5, 0, 0), 0.4}, 100000, cfg);
    const Real analytic = 0.735105;
    CHECK(std::fabs(r.sigma_lp - analytic) < 4.0 * r.std_error + 0.01 * analytic);
    CHECK(r.n_paths == 100000);
    std::int64_t sum = r.n_infinity + r.n_failed;
    for (auto c : r.feature_counts) sum += c;
    CHECK(sum == 100000);
    cfg.seed = 31;
    const LastPassageResult a = estimate_lp(disk, {Vec3(-0.5, 0, 0), 0.4}, 20000, cfg);
    cfg.workers = 8;
    const LastPassageResult b = estimate_lp(disk, {Vec3(-0.5, 0, 0), 0.4}, 20000, cfg);
    CHECK(std::memcmp(&a.sigma_lp, &b.sigma_lp, sizeof(Real)) == 0);
    CHECK(a.feature_counts == b.feature_counts);
    const Real off_v[4] = {0, 1, 0, 0};
    CHECK_THROWS_AS(estimate_lp(Scene::four_plates(off_v), {Vec3(0.5, 0.5, 0), 0.2}, 100, cfg),
                    ApplicabilityError);
}

// ---- the local DtN map (whole-boundary batch API) ----
static void case_dtn_unit_ball() {
    // u = x^2 - y^2 + z on the unit ball (config 1 data): du/dn_out = 2x^2 - 2y^2 + z on |x| = 1
    const Scene ball = Scene::sphere(1.0, DomainSide::Interior,
                                     Dirichlet::quadratic(0.0, Vec3(0, 0, 1), 1.0, -1.0, 0.0));
    const Real a = 0.2;
    const std::vector<NodeRule> gamma = {gamma_rule(16, 32, std::acos(a / 2.0))};
    const Vec3 pts[4] = {Vec3(0, 0, 1), Vec3(1, 0, 0), Vec3(0, -1, 0), Vec3(0.6, 0, -0.8)};
    std::vector<bw_patch> patches;
    for (const Vec3& p : pts) {
        bw_patch q{};
        q.o[0] = p.x; q.o[1] = p.y; q.o[2] = p.z;
        q.axis[0] = -p.x; q.axis[1] = -p.y; q.axis[2] = -p.z; // into the ball
        q.a = a;
        q.R = 1.0;
        q.surf = 0;
        patches.push_back(q);
    }
    WosConfig cfg;
    cfg.eps_shell = 1e-4;
    cfg.n_paths = 10000;
    cfg.seed = 1;
    const std::vector<NeumannPoint> r = dtn_solve(ball, cfg, DtnConfig(), patches, gamma);
    for (size_t i = 0; i < r.size(); ++i) {
        const Vec3& p = pts[i];
        const Real exact = 2 * p.x * p.x - 2 * p.y * p.y + p.z;
        CHECK(r[i].status == 0);
        CHECK(std::fabs(r[i].dudn - exact) < 5 * r[i].err + 1e-2);
    }
}

// tests/test_patch_solver.cpp:93-111 and :113-123 through solve_patch
static void case_solve_patch() {
    // flat patch, u = z fed exactly: du/dn = 1 along the (into-domain) normal
    const Scene hs = Scene::half_space(0.0, Dirichlet::quadratic(0.0, Vec3(0, 0, 1), 0, 0, 0));
    bw_patch p{};
    p.axis[2] = 1.0;
    p.a = 1.0;
    p.surf = 1;
    const NodeRule g = gamma_rule(16, 32, kPi / 2);
    std::vector<Estimate> est((size_t)g.size());
    for (int k = 0; k < g.size(); ++k) {
        est[(size_t)k].mean = node_position(Vec3(0, 0, 0), Vec3(0, 0, 1), 1.0, &g.dirs[3 * (size_t)k]).z;
        est[(size_t)k].n = 1;
    }
    const NeumannField f = solve_patch(hs, DtnConfig(), p, g, est);
    int counted = 0;
    Real worst = 0;
    for (size_t i = 0; i < f.dudn.size(); ++i)
        if (f.r[i] < 0.5) {
            worst = std::max(worst, std::fabs(f.dudn[i] - 1.0));
            ++counted;
        }
    CHECK(counted >= 6);
    CHECK(worst < 0.05);
    CHECK(f.status == 0);
    // constant data annihilates (exterior sphere)
    const Scene sph = Scene::sphere(3.0, DomainSide::Exterior, 0.25);
    bw_patch q{};
    q.o[2] = 3.0;
    q.axis[2] = 1.0;
    q.a = 1.0;
    q.R = 3.0;
    q.surf = 0;
    const NodeRule gs = gamma_rule(16, 32, std::acos(-1.0 / 6.0));
    std::vector<Estimate> c((size_t)gs.size());
    for (auto& e : c) {
        e.mean = 0.25;
        e.n = 1;
    }
    const NeumannField z = solve_patch(sph, DtnConfig(), q, gs, c);
    Real mx = 0;
    for (Real v : z.dudn) mx = std::max(mx, std::fabs(v));
    CHECK(mx < 1e-6);
}

int main() {
    case_immediate_exit_and_determinism();
    case_exit_uniform_from_centre();
    case_truncation_leakage();
    case_constant_data();
    case_ball_phi_z();
    case_halfspace_half();
    case_batch_bookkeeping();
    case_worker_count_invariance();
    case_mean_value_property();
    case_se_scaling();
    case_eps_bias();
    case_reliability_and_exit_value();
    case_potential();
    case_lu();
    case_point_formula();
    case_geometry();
    case_last_passage();
    case_dtn_unit_ball();
    case_solve_patch();
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
