"""The reference's own collocation and WOS test cases (tests/test_patch_solver.cpp,
tests/test_wos.cpp) restated on the device path: the Neumann stage (both
methods, bw_dtn_neumann) fed exact Gamma data, the Gamma nodes sampled by K1,
and the statistical WOS properties. The device reads du/dn at the patch
centre along the domain-OUTWARD normal (-axis), so the reference's targets
change sign where its field is quoted along +axis."""
from __future__ import annotations

import math

import numpy as np
import pytest

import paper_1210_1491_b200 as bw
from paper_1210_1491_b200 import dtn, nodes
from paper_1210_1491_b200.geometry import DomainSide, PointSource, Quadratic, Scene

pytestmark = pytest.mark.gpu
METHODS = [dtn.DTN_CLASSES, dtn.DTN_PER_PATCH]


def _patch(o, axis, a, surf, R=0.0):
    p = np.zeros(1, dtn.PATCH_DTYPE)
    p["o"], p["axis"], p["a"], p["surf"], p["R"] = o, axis, a, surf, R
    return p


def _exact_nodes(p, dirs, u):
    pos = nodes.patch_node_positions(p["o"], p["axis"], p["a"], None, dirs)[0]
    est = np.zeros((1, len(pos)), bw.ESTIMATE_DTYPE)
    est["mean"][0] = u(pos)
    est["n"] = 1
    return est


@pytest.mark.parametrize("method", METHODS)
def test_flat_patch_u_equals_z(gpu, method):  # test_patch_solver.cpp:93-111
    scene = Scene.half_space(0.0, Quadratic(g=(0.0, 0.0, 1.0)))
    p = _patch((0, 0, 0), (0, 0, 1.0), 1.0, 1)
    dirs, w = nodes.gamma_rule(16, 32, math.pi / 2)
    est = _exact_nodes(p, dirs, lambda y: y[:, 2])
    r = dtn.dtn_neumann(scene, p, dirs, w, est, method=method)
    assert r.status[0] == 0
    assert abs(r.dudn[0] - (-1.0)) < 0.01  # du/dn_out = -du/dz


@pytest.mark.parametrize("method", METHODS)
def test_constant_data_annihilates(gpu, method):  # test_patch_solver.cpp:113-123
    scene = Scene.sphere(3.0, DomainSide.Exterior, 0.25)
    p = _patch((0, 0, 3.0), (0, 0, 1.0), 1.0, 0, R=3.0)
    dirs, w = nodes.gamma_rule(16, 32, math.acos(-1.0 / 6.0))
    est = _exact_nodes(p, dirs, lambda y: np.full(len(y), 0.25))
    r = dtn.dtn_neumann(scene, p, dirs, w, est, method=method)
    assert abs(r.dudn[0]) < 1e-6


@pytest.mark.parametrize("method", METHODS)
def test_sphere_patch_exact_gamma_data(gpu, method):  # test_patch_solver.cpp:125-143
    """Exterior sphere R = 3 at potential 1/(12 pi): u = 1/(4 pi |y|); the
    patch of radius 1 at the pole gives du/dn_out = 1/(36 pi) within 2 %."""
    scene = Scene.sphere(3.0, DomainSide.Exterior, 1.0 / (12 * math.pi))
    p = _patch((0, 0, 3.0), (0, 0, 1.0), 1.0, 0, R=3.0)
    dirs, w = nodes.gamma_rule(16, 32, math.acos(-1.0 / 6.0))
    est = _exact_nodes(p, dirs, lambda y: 1.0 / (4 * math.pi * np.linalg.norm(y, axis=1)))
    r = dtn.dtn_neumann(scene, p, dirs, w, est, method=method)
    target = 1.0 / (36 * math.pi)
    assert r.status[0] == 0
    assert abs(r.dudn[0] / target - 1.0) < 0.02


def test_gamma_nodes_sampled_by_wos(gpu):  # test_patch_solver.cpp:193-209
    scene = Scene.sphere(3.0, DomainSide.Exterior, 1.0 / (12 * math.pi))
    dirs, _ = nodes.gamma_rule(8, 16, math.acos(-1.0 / 6.0))
    est, _ = nodes.wos_patch_nodes(scene, bw.WosConfig(n_paths=2000), np.array([[0, 0, 3.0]]),
                                   np.array([[0, 0, 1.0]]), 1.0, dirs)
    pos = nodes.patch_node_positions([[0, 0, 3.0]], [[0, 0, 1.0]], 1.0, None, dirs)[0]
    exact = 1.0 / (4 * math.pi * np.linalg.norm(pos, axis=1))
    se = np.sqrt(est["variance"][0] / est["n"][0])
    assert (np.abs(est["mean"][0] - exact) > 4 * se).sum() <= 3


def _test1():
    return Scene.half_space(0.0, PointSource(q=1.0, s=(0, 0, -1.0)))


def test_standard_error_scales_like_inverse_sqrt_n(gpu):  # test_wos.cpp:156-167
    scaled = []
    for n in (1000, 10000, 100000):
        e = bw.estimate_u(_test1(), (0.5, 0, 0.25), bw.WosConfig(n_paths=n))
        scaled.append(e.std_error() * math.sqrt(n))
    assert all(abs(v / scaled[0] - 1.0) < 0.2 for v in scaled)


def test_eps_shell_bias_below_resolution(gpu):  # test_wos.cpp:169-182
    ea = bw.estimate_u(_test1(), (0.5, 0, 0.3), bw.WosConfig(n_paths=40000, eps_shell=1e-4))
    eb = bw.estimate_u(_test1(), (0.5, 0, 0.3), bw.WosConfig(n_paths=40000, eps_shell=1e-5,
                                                              seed=1))
    se = math.hypot(ea.std_error(), eb.std_error())
    assert abs(ea.mean - eb.mean) < 3 * se
