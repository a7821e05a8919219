"""Host-side pieces of the reference API that need no device (CPU suite)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1210_1491_b200 as bw
from paper_1210_1491_b200.geometry import PointSource, Scene


def test_exit_value_infinity_and_failed():  # test_wos.cpp:192-196
    s = Scene.half_space(0.0, PointSource(q=1.0, s=(0, 0, -1.0)))
    assert bw.exit_value(s, bw.ExitRecord(np.array([2e5, 0, 0]), bw.kExitInfinity, 12)) == 0.0
    with pytest.raises(bw.ReliabilityError):
        bw.exit_value(s, bw.ExitRecord(np.zeros(3), bw.kExitFailed, 12))


def test_exit_value_feature_data():  # wos.cpp:87-93
    plates = Scene.four_plates([0, 1, 0, 0])
    assert bw.exit_value(plates, bw.ExitRecord(np.array([-0.5, 0.5, 0]), 1, 3)) == 1.0
    s = Scene.half_space(0.0, PointSource(q=1.0, s=(0, 0, -1.0)))
    assert bw.exit_value(s, bw.ExitRecord(np.array([0.0, 0, 0]), 0, 3)) == 1.0


def test_gauss_legendre_orders():  # test_quadrature.cpp:11-44
    from paper_1210_1491_b200.nodes import gauss_legendre

    for n in (1, 2, 5, 20, 64):
        x, w = gauss_legendre(n)
        assert abs(w.sum() - 2.0) < 1e-13
        for k in range(2 * n):  # degree 2n-1 exactness
            exact = 0.0 if k % 2 else 2.0 / (k + 1)
            assert abs((w * x ** k).sum() - exact) < 1e-12
    for n in (0, 65):
        with pytest.raises(bw.GeometryError):
            gauss_legendre(n)


def test_cap_rule_area_and_normalisation():  # test_quadrature.cpp:46-60
    from paper_1210_1491_b200.point_solver import cap_rule

    _, w = cap_rule(20)
    assert abs(w.sum() - 2 * np.pi) < 1e-8 * 2 * np.pi
    d, w = cap_rule(30)
    a = 0.5
    ct = d[:, 2]
    w = w * a * a
    assert abs((w * 3.0 / (2 * np.pi * a ** 3) * ct).sum() - 3.0) < 1e-8 * 3
    assert abs((w * ct).sum() - np.pi * a * a) < 1e-8 * np.pi * a * a
    with pytest.raises(bw.GeometryError):
        cap_rule(1)


def test_ring_rule_weight_and_domain():  # test_quadrature.cpp:62-73
    from paper_1210_1491_b200.point_solver import ring_rule_unit

    a = 0.5
    for doa in (1e-1, 1e-3, 1e-6):
        r = ring_rule_unit(20, doa)
        w = r[:, 3] * a * a
        assert abs(w.sum() - np.pi * (a * a - (doa * a) ** 2)) < 1e-10 * np.pi * a * a
        assert (r[:, 0] * a >= doa * a).all()
    for dfrac in (1.0, 1.4):
        with pytest.raises(bw.GeometryError):
            ring_rule_unit(8, dfrac)
