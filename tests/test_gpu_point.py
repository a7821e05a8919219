"""GPU: the flat-boundary point formula (K6) against the reference's frozen
values (tests/test_point_solver.cpp of the reference: Sigma2' ring values at
1e-9, Sigma1' with the exact sampler 0.622487481448513 at 1e-9, solve_point
totals, the Monte-Carlo run near the analytic density)."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import paper_1210_1491_b200 as bw
from paper_1210_1491_b200 import point_solver as ps
from paper_1210_1491_b200.geometry import PointSource, Scene

pytestmark = pytest.mark.gpu
CFG = Path(__file__).resolve().parents[1] / "configs"
ANALYTIC = 1.0 / 1.25 ** 1.5  # 0.71554...


def approx(a, b, eps):
    """doctest::Approx(b).epsilon(eps) semantics (scale 1): the reference's own tolerance."""
    return abs(a - b) < eps * (1.0 + max(abs(a), abs(b)))


def _halfspace_test1():
    return Scene.half_space(0.0, PointSource(q=1.0, s=(0, 0, -1.0)))


def exact_sampler(y, pid):
    return bw.Estimate(mean=1.0 / np.linalg.norm(np.asarray(y) - [0, 0, -1.0]), variance=0.0, n=1)


def test_sigma2_frozen_ring_values(gpu):
    rows = [(0.1, 0.018774176765485), (0.2, 0.037509938413963), (0.5, 0.093041749382575),
            (0.7, 0.128953220225998), (1.0, 0.179947714623269)]
    for a, expect in rows:
        r = ps.solve_point(_halfspace_test1(), ps.HemisphereFrame((0.5, 0, 0), a), 20, 20,
                           1e-4 * a, bw.WosConfig(), sampler=exact_sampler)
        assert approx(r.sigma2, expect, 1e-9)


def test_sigma1_exact_sampler_frozen(gpu):
    r = ps.solve_point(_halfspace_test1(), ps.HemisphereFrame((0.5, 0, 0), 0.5), 20, 20, 5e-5,
                       bw.WosConfig(), sampler=exact_sampler)
    assert approx(r.sigma1, 0.622487481448513, 1e-9)
    assert r.std_error == 0.0


def test_solve_point_exact_sampler_totals(gpu):
    totals = [0.715539248403333, 0.715536744007608, 0.715529230831088, 0.715524222120063,
              0.715516709286366]
    for a, t in zip([0.1, 0.2, 0.5, 0.7, 1.0], totals):
        r = ps.solve_point(_halfspace_test1(), ps.HemisphereFrame((0.5, 0, 0), a), 20, 20,
                           1e-4 * a, bw.WosConfig(), sampler=exact_sampler)
        assert approx(r.total, t, 1e-9)
        assert r.total == r.sigma1 + r.sigma2
        assert abs(r.total / ANALYTIC - 1) < 1e-4


def test_solve_point_monte_carlo(gpu):
    r = ps.solve_point(_halfspace_test1(), ps.HemisphereFrame((0.5, 0, 0), 0.5), 20, 20, 5e-5,
                       bw.WosConfig(n_paths=1000, seed=2024))
    assert abs(r.total - ANALYTIC) < 4 * r.std_error + 2e-4
    assert 0 < r.std_error < 0.01


def test_point_formula_rejects_curved_scenes(gpu):
    s = Scene.sphere(1.0, bw.DomainSide.Interior, 1.0)
    with pytest.raises(bw.ApplicabilityError):
        ps.solve_point(s, ps.HemisphereFrame((0, 0, 1.0), 0.2), 8, 8, 1e-5, bw.WosConfig())


def test_point_formula_on_cube_faces(gpu):
    """Batch: interior face points of config 2 (cube), vs the analytic data."""
    from paper_1210_1491_b200 import workloads

    w = workloads.config2()
    far = np.where(w.radii == w.a)[0][::200]
    total, s1, s2, se = ps.solve_points(w.scene, w.points[far], w.axes[far], w.radii[far], 16,
                                        20, 1e-4, bw.WosConfig(eps_shell=1e-5, n_paths=4096,
                                                               seed=2))
    exact = w.exact_dudn_outward()[far]
    scale = np.abs(w.exact_grad(w.points[far])).max(axis=1) + 1
    assert (np.abs(total - exact) < 5 * se + 2e-2 * scale).mean() > 0.95


def _zero_sampler(y, pid):
    return bw.Estimate(mean=0.0, variance=0.0, n=1)


def _s2(scene, center, a, delta, n_g2=20):
    return ps.solve_point(scene, ps.HemisphereFrame(center, a), 8, n_g2, delta, bw.WosConfig(),
                          sampler=_zero_sampler).sigma2


def test_sigma2_zero_for_constant_disk_data(gpu):  # test_point_solver.cpp:66-70
    assert _s2(Scene.thin_disk(1.0, 1.0), (-0.5, 0, 0), 0.4, 1e-4 * 0.4) == 0.0


def test_sigma2_four_plates_exact_frozen(gpu):  # test_point_solver.cpp:72-92
    """Piecewise-constant plate data: the exact finite part (angular breakpoints
    + Gauss segments, point_solver.cpp:43-114) against the frozen values."""
    s = Scene.four_plates([0, 1, 0, 0])  # plate II at 1 V
    A = (-0.2273, 0.2273, 0.0)
    for a in (0.1, 0.2, 0.2273):
        assert _s2(s, A, a, 1e-4 * a) == 0.0
    for a, expect in ((0.3, 0.08918475915450), (0.5, 0.63287790821628), (0.7, 1.02697283920885)):
        assert approx(_s2(s, A, a, 1e-4 * a), expect, 1e-10)
    assert abs(_s2(s, A, 0.5, 1e-4) - 0.6330) < 2e-4  # the paper's table value
    with pytest.raises(bw.DomainError):
        _s2(s, A, 1.0, 1e-4)  # disk poking past the plate union


def test_point_formula_frame_and_feature_checks(gpu):  # point_solver.cpp:14-22
    s = Scene.four_plates([0, 1, 0, 0])
    with pytest.raises(bw.GeometryError):
        ps.solve_point(s, ps.HemisphereFrame((-0.3, 0.3, 0.0), 0.1, (0.0, 0.6, 0.8)), 8, 8, 1e-5,
                       bw.WosConfig(), sampler=_zero_sampler)
    with pytest.raises(bw.GeometryError):
        ps.solve_point(s, ps.HemisphereFrame((-0.3, 0.3, 0.01), 0.1), 8, 8, 1e-5,
                       bw.WosConfig(), sampler=_zero_sampler)
    with pytest.raises(bw.ClassificationError):  # centre off the plates
        ps.solve_point(s, ps.HemisphereFrame((-1.5, 0.3, 0.0), 0.1), 8, 8, 1e-5,
                       bw.WosConfig(), sampler=_zero_sampler)


def test_four_plates_sine_runner(gpu):
    """runner.cpp:318-324 four_plates_sine (sin(x) sin(y) on the four plates,
    the reference's configs/four_plates_sine.cfg parameters): the density at
    (-0.5, 0.5) is a-independent within the propagated error, and the CSV is
    identical for any worker count."""
    from paper_1210_1491_b200 import runner

    c = runner.parse_config_file(str(CFG / "four_plates_sine_b200.cfg"))
    rec = runner.run(c)
    r = np.array(rec.rows, dtype=float)
    total, se = r[:, 8], r[:, 9]
    assert np.isfinite(total).all() and (se > 0).all()
    mid = np.median(total)
    assert (np.abs(total - mid) < 4 * np.hypot(se, np.median(se)) + 5e-3).all()
    again = runner.run(runner.parse_config_file(str(CFG / "four_plates_sine_b200.cfg")), workers=5)
    assert again.csv_text == rec.csv_text
