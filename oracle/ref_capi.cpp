// ref_capi.cpp — TEST INFRASTRUCTURE. A C shim over the reference's own,
// unmodified C++ sources (compiled from /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/libbiewos_ref.so). It lets the tests and the
// `--impl reference` bench arm call the reference implementation itself:
//   biewos::walk              (wos.cpp:81-85)
//   biewos::estimate_u_batch  (wos.cpp:95-132)
//   biewos::evaluate          (field_eval.cpp:7-19)
//   biewos::philox::block     (rng.hpp:25-38)
//   biewos::gauss_legendre    (quadrature.cpp:7-35)
// Exceptions are mapped to the bw_status codes of include/biewos_b200.h.
#include <cmath>
#include <cstring>
#include <exception>
#include <vector>

#include "biewos/field_eval.hpp"
#include "biewos/geometry.hpp"
#include "biewos/greens.hpp"
#include "biewos/patch_solver.hpp"
#include "biewos/point_solver.hpp"
#include "biewos/quadrature.hpp"
#include "biewos/rng.hpp"
#include "biewos/wos.hpp"

#include "../include/biewos_b200.h"
#ifdef BW_INTEGRATED
// integration/Makefile builds this shim a second time against the reference's
// sources with wos.cpp / field_eval.cpp replaced by the B200 binding: the
// closed form of the data is declared to the bridge (geometry.hpp:34,49)
#include "../integration/biewos_b200_bridge.hpp"
#endif

using namespace biewos;

namespace {

int map_exc() {
    try {
        throw;
    } catch (const DomainError&) {
        return BW_ERR_DOMAIN;
    } catch (const ClassificationError&) {
        return BW_ERR_CLASSIFICATION;
    } catch (const SingularityError&) {
        return BW_ERR_SINGULARITY;
    } catch (const GeometryError&) {
        return BW_ERR_GEOMETRY;
    } catch (const ReliabilityError&) {
        return BW_ERR_RELIABILITY;
    } catch (const ApplicabilityError&) {
        return BW_ERR_APPLICABILITY;
    } catch (const NearFieldError&) {
        return BW_ERR_NEARFIELD;
    } catch (const SolverError&) {
        return BW_ERR_SOLVER;
    } catch (...) {
        return BW_ERR_INVALID;
    }
}

// The closed-form data of bw_phi_kind as the std::function the reference takes.
DirichletFn phi_fn(const bw_scene& s) {
    double c[16];
    std::memcpy(c, s.phi, sizeof c);
    std::vector<double> c16(c, c + 16);
    switch (s.phi_kind) {
        case BW_PHI_QUADRATIC:
            return [c16](const Vec3& y) {
                const double* k = c16.data();
                return k[0] + k[1] * y.x() + k[2] * y.y() + k[3] * y.z() + k[4] * y.x() * y.x() +
                       k[5] * y.y() * y.y() + k[6] * y.z() * y.z() + k[7] * y.x() * y.y() +
                       k[8] * y.x() * y.z() + k[9] * y.y() * y.z();
            };
        case BW_PHI_EXP_SIN_SIN:
            return [c16](const Vec3& y) {
                const double* k = c16.data();
                return k[0] * std::exp(k[1] * (y.x() - k[4])) * std::sin(k[2] * (y.y() - k[5])) *
                       std::sin(k[3] * (y.z() - k[6]));
            };
        case BW_PHI_POINT_SOURCE:
            return [c16](const Vec3& y) {
                const double* k = c16.data();
                return k[4] + k[0] / (y - Vec3(k[1], k[2], k[3])).norm();
            };
        case BW_PHI_SIN_SIN: // runner.cpp:318-324 (four_plates_sine)
            return [c16](const Vec3& y) {
                const double* k = c16.data();
                return k[0] * std::sin(k[1] * (y.x() - k[3])) * std::sin(k[2] * (y.y() - k[4]));
            };
    }
    return {};
}

// Scene factories of geometry.cpp:34-92 for the kinds the reference has.
bool make_scene_impl(const bw_scene* s, Scene& out);

bool make_scene(const bw_scene* s, Scene& out) {
    if (!make_scene_impl(s, out)) return false;
#ifdef BW_INTEGRATED
    if (!out.piecewise_const) biewos::b200::set_dirichlet(out, s->phi_kind, s->phi);
#endif
    return true;
}

bool make_scene_impl(const bw_scene* s, Scene& out) {
    const DomainSide side = s->side == BW_INTERIOR ? DomainSide::Interior : DomainSide::Exterior;
    if (s->kind == BW_SCENE_SPHERE) {
        out = s->phi_kind == BW_PHI_FEATURE_CONST
                  ? Scene::sphere(s->sphere_radius, side, s->feature_potential[0])
                  : Scene::sphere(s->sphere_radius, side, phi_fn(*s));
        return true;
    }
    if (s->kind == BW_SCENE_HALFSPACE && s->phi_kind != BW_PHI_FEATURE_CONST) {
        out = Scene::half_space(s->plane_z, phi_fn(*s));
        return true;
    }
    if (s->kind == BW_SCENE_PLATESET) {
        std::vector<Plate> pl;
        for (int i = 0; i < s->n_plates; ++i) {
            const double* r = s->plates + 4 * i;
            pl.push_back(Plate{r[0], r[1], r[2], r[3],
                               s->phi_kind == BW_PHI_FEATURE_CONST ? s->feature_potential[i] : 0.0});
        }
        out = s->phi_kind == BW_PHI_FEATURE_CONST ? Scene::plate_set(pl) : Scene::plate_set(pl, phi_fn(*s));
        return true;
    }
    if (s->kind == BW_SCENE_THINDISK && s->phi_kind == BW_PHI_FEATURE_CONST) {
        out = Scene::thin_disk(s->disk_radius, s->feature_potential[0]);
        return true;
    }
    return false;
}

WosConfig make_cfg(const bw_wos_config* c, int workers) {
    WosConfig w;
    w.eps_shell = c->eps_shell;
    w.trunc_radius = c->trunc_radius;
    w.n_paths = c->n_paths;
    w.max_steps = c->max_steps;
    w.seed = c->seed;
    w.workers = workers;
    return w;
}

} // namespace

extern "C" {

void ref_philox_block(const uint64_t* ctr, const uint64_t* key, uint64_t* out) {
    const auto r = philox::block({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
    for (int i = 0; i < 4; ++i) out[i] = r[static_cast<size_t>(i)];
}

void ref_rng_doubles(uint64_t seed, uint64_t point_id, uint64_t path_id, uint64_t domain,
                     int64_t n, double* out) {
    RngStream s(seed, point_id, path_id, domain);
    for (int64_t i = 0; i < n; ++i) out[i] = s.next_double();
}

int ref_walk(const bw_scene* scene, const bw_wos_config* cfg, const double* starts, int64_t n,
             const uint64_t* point_ids, const uint64_t* path_ids, double* exit_points,
             int32_t* features, int32_t* steps) {
    try {
        Scene s;
        if (!make_scene(scene, s)) return BW_ERR_APPLICABILITY;
        const WosConfig w = make_cfg(cfg, 1);
        for (int64_t i = 0; i < n; ++i) {
            const Vec3 p(starts[3 * i], starts[3 * i + 1], starts[3 * i + 2]);
            const ExitRecord r = walk(s, p, w, point_ids[i], path_ids[i]);
            exit_points[3 * i] = r.point.x();
            exit_points[3 * i + 1] = r.point.y();
            exit_points[3 * i + 2] = r.point.z();
            features[i] = r.feature;
            steps[i] = r.steps;
        }
        return BW_OK;
    } catch (...) {
        return map_exc();
    }
}

int ref_estimate_u_batch(const bw_scene* scene, const bw_wos_config* cfg, const double* pts,
                         int64_t n, uint64_t point_id_base, int workers, bw_estimate* out) {
    try {
        Scene s;
        if (!make_scene(scene, s)) return BW_ERR_APPLICABILITY;
        std::vector<Vec3> p;
        p.reserve(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) p.emplace_back(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
        const auto est = estimate_u_batch(s, p, make_cfg(cfg, workers), point_id_base);
        for (size_t i = 0; i < est.size(); ++i) {
            out[i].mean = est[i].mean;
            out[i].variance = est[i].variance;
            out[i].n = est[i].n;
            out[i].n_infinity = est[i].n_infinity;
            out[i].n_failed = est[i].n_failed;
        }
        return BW_OK;
    } catch (...) {
        return map_exc();
    }
}

// evaluate() per target; near[i] = 1 where the reference throws NearFieldError.
int ref_evaluate(const double* panels, int64_t n_panels, const double* targets, int64_t n_t,
                 double* u, uint8_t* near) {
    BoundaryData d;
    d.panels.reserve(static_cast<size_t>(n_panels));
    for (int64_t j = 0; j < n_panels; ++j) {
        const double* P = panels + 9 * j;
        d.panels.push_back({Vec3(P[0], P[1], P[2]), Vec3(P[3], P[4], P[5]), P[6], P[7], P[8]});
    }
    int status = BW_OK;
    for (int64_t t = 0; t < n_t; ++t) {
        try {
            u[t] = evaluate(d, Vec3(targets[3 * t], targets[3 * t + 1], targets[3 * t + 2]));
            if (near) near[t] = 0;
        } catch (...) {
            status = map_exc();
            u[t] = NAN;
            if (near) near[t] = 1;
        }
    }
    return status;
}

int ref_gauss_legendre(int n, double* nodes, double* weights) {
    try {
        const GaussRule1D g = gauss_legendre(n);
        for (int i = 0; i < n; ++i) {
            nodes[i] = g.nodes[i];
            weights[i] = g.weights[i];
        }
        return BW_OK;
    } catch (...) {
        return map_exc();
    }
}

int ref_sphere_kernels(const double* c, double a, const double* x, const double* nx,
                       const double* y, const double* ny, double* dg_dnx, double* d2g) {
    try {
        const SphereFrame f{Vec3(c[0], c[1], c[2]), a};
        const Vec3 X(x[0], x[1], x[2]), NX(nx[0], nx[1], nx[2]), Y(y[0], y[1], y[2]),
            NY(ny[0], ny[1], ny[2]);
        *dg_dnx = sphere_dg_dnx(f, X, NX, Y);
        *d2g = sphere_d2g(f, X, NX, Y, NY);
        return BW_OK;
    } catch (...) {
        return map_exc();
    }
}

// Exterior sphere patch of the reference (make_sphere_patch_setup +
// sample_gamma_grid with exact data + assemble; bie_kind 0 second, 1 first), and the Gamma
// node list its assemble integrates (patch_solver.cpp:206-233 loop, rebuilt
// from the public gauss_legendre / gamma_point / interp_gamma). A: m x m,
// b, b_se: m; gy: n_g x 3, gw, gu: n_g (n_g = 5 * gauss_gamma^2).
int ref_sphere_patch_assemble_kind(const bw_scene* scene, const double* o, double a, int bands,
                                   int azimuth, int n_theta, int n_phi, int bie_kind, double* A,
                                   double* b, double* b_se, double* gy, double* gw, double* gu,
                                   int* m_out, int* ng_out) {
    try {
        Scene s;
        if (!make_scene(scene, s)) return BW_ERR_APPLICABILITY;
        const DirichletFn u = s.piecewise_const ? DirichletFn([&](const Vec3&) {
            return s.feature_potential[0];
        }) : s.dirichlet;
        const PatchSetup setup = make_sphere_patch_setup(s, Vec3(o[0], o[1], o[2]), a, bands,
                                                         azimuth, n_theta, n_phi);
        const GammaGrid grid = sample_gamma_grid(setup, [&](const Vec3& y, std::uint64_t) {
            Estimate e;
            e.mean = u(y);
            e.n = 1;
            return e;
        });
        const DenseSystem sys =
            assemble(s, setup, bie_kind == 1 ? BieKind::FirstKind : BieKind::SecondKind, grid);
        const int m = setup.mesh.n_panels();
        *m_out = m;
        if (A) {
            for (int i = 0; i < m; ++i) {
                b[i] = sys.b[i];
                b_se[i] = sys.b_se[i];
                for (int j = 0; j < m; ++j) A[i * m + j] = sys.A(i, j);
            }
        }
        const GaussRule1D g = gauss_legendre(setup.gauss_gamma);
        const double breaks[6] = {0.0, 0.5, 0.75, 0.875, 0.9375, 1.0};
        int n = 0;
        for (int seg = 0; seg < 5; ++seg) {
            const double t0 = breaks[seg] * setup.theta_grid_max, t1 = breaks[seg + 1] * setup.theta_grid_max;
            for (int i = 0; i < g.order; ++i) {
                const double theta = t0 + (t1 - t0) * 0.5 * (g.nodes[i] + 1.0);
                const double wt = g.weights[i] * 0.5 * (t1 - t0);
                for (int j = 0; j < g.order; ++j) {
                    const double phi = kPi * (g.nodes[j] + 1.0);
                    const Vec3 y = setup.gamma_point(theta, phi);
                    if (gy) {
                        gy[3 * n] = y.x();
                        gy[3 * n + 1] = y.y();
                        gy[3 * n + 2] = y.z();
                        gw[n] = wt * g.weights[j] * kPi * a * a * std::sin(theta);
                        gu[n] = interp_gamma(grid, setup, y);
                    }
                    ++n;
                }
            }
        }
        *ng_out = n;
        return BW_OK;
    } catch (...) {
        return map_exc();
    }
}

// solve_point (point_solver.hpp:33-35) with WOS values: the reference's
// sigma1_prime -> estimate_u_batch call chain (point_solver.cpp:166).
int ref_solve_point_wos(const bw_scene* scene, const bw_wos_config* cfg, const double* c,
                        double a, const double* axis, int n_g1, int n_g2, double delta,
                        int workers, double* out4) {
    try {
        Scene s;
        if (!make_scene(scene, s)) return BW_ERR_APPLICABILITY;
        const HemisphereFrame f(Vec3(c[0], c[1], c[2]), a, Vec3(axis[0], axis[1], axis[2]));
        const PointNeumannResult r = solve_point(s, f, n_g1, n_g2, delta, make_cfg(cfg, workers));
        out4[0] = r.sigma1;
        out4[1] = r.sigma2;
        out4[2] = r.total;
        out4[3] = r.std_error;
        return BW_OK;
    } catch (...) {
        return map_exc();
    }
}

// solve_patch (patch_solver.hpp:84-85) with a WOS-sampled Gamma grid: the
// reference's sample_gamma_grid -> estimate_u_batch call chain
// (patch_solver.cpp:123-137) on its sphere patch (flat patch for a half-space).
int ref_solve_patch_wos(const bw_scene* scene, const bw_wos_config* cfg, const double* o,
                        double a, int bands, int azimuth, int n_theta, int n_phi, int bie_kind,
                        int workers, double* dudn, double* r, double* est_error, int* m_out) {
    try {
        Scene s;
        if (!make_scene(scene, s)) return BW_ERR_APPLICABILITY;
        const Vec3 O(o[0], o[1], o[2]);
        const PatchSetup setup = s.kind == SceneKind::HalfSpace
                                     ? make_flat_patch_setup(O, a, bands, azimuth, n_theta, n_phi)
                                     : make_sphere_patch_setup(s, O, a, bands, azimuth, n_theta,
                                                               n_phi);
        const NeumannField nf = solve_patch(
            s, setup, bie_kind == 1 ? BieKind::FirstKind : BieKind::SecondKind,
            make_cfg(cfg, workers));
        const int m = setup.mesh.n_panels();
        *m_out = m;
        if (dudn)
            for (int i = 0; i < m; ++i) {
                dudn[i] = nf.dudn[i];
                r[i] = nf.r[i];
                est_error[i] = nf.est_error[i];
            }
        return BW_OK;
    } catch (...) {
        return map_exc();
    }
}

int ref_sphere_patch_assemble(const bw_scene* scene, const double* o, double a, int bands,
                              int azimuth, int n_theta, int n_phi, double* A, double* b,
                              double* b_se, double* gy, double* gw, double* gu, int* m_out,
                              int* ng_out) {
    return ref_sphere_patch_assemble_kind(scene, o, a, bands, azimuth, n_theta, n_phi, 0, A, b,
                                          b_se, gy, gw, gu, m_out, ng_out);
}

} // extern "C"
