"""Pin the collocation oracle (oracle/biewos_patch.c) against the reference's
own assemble (patch_solver.cpp:197-309) on the reference's exterior sphere
patch with identical Gamma nodes: A and b must be bit-identical. CPU only."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import oracle_lib as O
from paper_1210_1491_b200.geometry import DomainSide, PointSource, Quadratic, Scene

_P = C.c_void_p


def _ref_assemble(reflib, sc, o, a, bands, az, nt, nphi, kind=0):
    f = reflib.ref_sphere_patch_assemble_kind
    f.argtypes = [_P, _P, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int] + [_P] * 8
    m, ng = C.c_int(), C.c_int()
    assert f(C.byref(sc), O.p(o), a, bands, az, nt, nphi, kind, *([None] * 6), C.byref(m),
             C.byref(ng)) == 0
    m, ng = m.value, ng.value
    A, b, bse = np.zeros((m, m)), np.zeros(m), np.zeros(m)
    gy, gw, gu = np.zeros((ng, 3)), np.zeros(ng), np.zeros(ng)
    assert f(C.byref(sc), O.p(o), a, bands, az, nt, nphi, kind, O.p(A), O.p(b), O.p(bse),
             O.p(gy), O.p(gw), O.p(gu), C.byref(C.c_int()), C.byref(C.c_int())) == 0
    return A, b, bse, gy, gw, gu


def _or_assemble(orc, sc, o, axis, surf, cen, R, a, bands, az, gy, gw, gu, guv, kind=0):
    f = orc.or_assemble_kind
    f.argtypes = [_P, _P, _P, C.c_int, _P, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                  C.c_int, _P, _P, _P, _P, C.c_int, C.c_int, _P, _P, _P]
    m = az * (2 * bands - 1)
    A, b, bse = np.zeros((m, m)), np.zeros(m), np.zeros(m)
    st = f(C.byref(sc), O.p(o), O.p(axis), surf, O.p(cen), R, a, bands, az, 20, 2, O.p(gy),
           O.p(gw), O.p(gu), O.p(guv), len(gu), kind, O.p(A), O.p(b), O.p(bse))
    return st, A, b, bse


@pytest.mark.parametrize("kind", [0, 1])  # second kind (default), first kind
@pytest.mark.parametrize("o,a,bands,az", [((0, 0, 3.0), 1.0, 6, 16),
                                          ((1.2, -2.0, 1.9), 0.7, 4, 9)])
def test_assemble_bit_identical_to_reference(orc, reflib, o, a, bands, az, kind):
    R = float(np.linalg.norm(o))
    sc = Scene.sphere(R, DomainSide.Exterior, PointSource(q=1 / (4 * np.pi), s=(0, 0, 0))).to_c()
    o = np.array(o, float)
    A, b, bse, gy, gw, gu = _ref_assemble(reflib, sc, o, a, bands, az, 32, 64, kind)
    st, A2, b2, _ = _or_assemble(orc, sc, o, o / np.linalg.norm(o), 0, np.zeros(3), R, a, bands,
                                 az, gy, gw, gu, np.zeros(len(gu)), kind)
    assert st == 0
    assert np.array_equal(A, A2) and np.array_equal(b, b2)


def test_first_and_second_kind_agree_reference(orc, reflib):
    """tests/test_patch_solver.cpp:125-143: the two kinds agree within 2%."""
    R, a = 3.0, 1.0
    sc = Scene.sphere(R, DomainSide.Exterior, PointSource(q=1 / (4 * np.pi), s=(0, 0, 0))).to_c()
    o = np.array([0, 0, 3.0])
    A2, b2, *_ = _ref_assemble(reflib, sc, o, a, 8, 20, 48, 96, 0)
    A1, b1, *_ = _ref_assemble(reflib, sc, o, a, 8, 20, 48, 96, 1)
    x2, x1 = np.linalg.solve(A2, b2)[:20].mean(), np.linalg.solve(A1, b1)[:20].mean()
    target = -1 / (36 * np.pi)
    assert abs(x2 / target - 1) < 0.02 and abs(x1 - x2) / abs(target) < 0.02


def test_sphere_patch_accuracy_reference_test(orc, reflib):
    """tests/test_patch_solver.cpp:125-143: exterior sphere, exact Gamma data,
    2% within 0.7a (here: the fan value at the patch centre)."""
    R, a = 3.0, 1.0
    sc = Scene.sphere(R, DomainSide.Exterior, PointSource(q=1 / (4 * np.pi), s=(0, 0, 0))).to_c()
    o = np.array([0, 0, 3.0])
    A, b, *_ = _ref_assemble(reflib, sc, o, a, 8, 20, 48, 96)
    x = np.linalg.solve(A, b)
    assert abs(x[:20].mean() / (-1 / (36 * np.pi)) - 1) < 0.02


def test_interior_ball_patch_exact_data(orc):
    """The interior-side patch the reference lacks: u = x^2 - y^2 + z on the
    unit ball with exact Gamma data (GL x uniform nodes) -> analytic du/dn."""
    from paper_1210_1491_b200 import dtn, workloads

    w = workloads.config1()
    sc = w.scene.to_c()
    P = dtn.patches_for(w)
    for b in (0, 400, 999):
        gy = O.or_patch_nodes(orc, w.points[b:b + 1], w.axes[b:b + 1], w.a, None, w.dirs[0])[0]
        d, e, st = O.or_patch_point(orc, sc, P[b], gy, w.weights[0] * w.a ** 2, w.exact_u(gy),
                                    np.zeros(len(gy)))
        assert st == 0
        exact = -w.exact_dudn_outward()[b]
        assert abs(d - exact) < 5e-3 * np.abs(w.exact_grad(w.points[b])).max()
