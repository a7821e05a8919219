"""The drop-in made real: the reference's own point_solver.cpp, patch_solver.cpp,
geometry.cpp, greens.cpp and quadrature.cpp, compiled unmodified against its
headers, with wos.cpp and field_eval.cpp replaced by the B200 binding
(integration/: wos_b200.cpp, field_eval_b200.cpp, bridge_b200.cpp), linked to
libbiewos_b200.so (integration/Makefile -> integration/_build/libbiewos_integrated.so).

Each case runs one reference entry point through both builds — the integrated
one (its estimate_u_batch / evaluate calls land on K1 / K3) and oracle/_ref
(the reference with its own wos.cpp / field_eval.cpp, on the host) — through the
same C shim (oracle/ref_capi.cpp), on the same seeded streams."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
from paper_1210_1491_b200.geometry import DomainSide, PointSource, Quadratic, Scene
from paper_1210_1491_b200.wos import WosConfig

pytestmark = pytest.mark.gpu
INTEG = Path(__file__).resolve().parents[1] / "integration" / "_build" / "libbiewos_integrated.so"
_P = C.c_void_p


def _bind(lib):
    lib.ref_estimate_u_batch.argtypes = [_P, _P, _P, C.c_int64, C.c_uint64, C.c_int, _P]
    lib.ref_evaluate.argtypes = [_P, C.c_int64, _P, C.c_int64, _P, _P]
    lib.ref_solve_point_wos.argtypes = [_P, _P, _P, C.c_double, _P, C.c_int, C.c_int, C.c_double,
                                        C.c_int, _P]
    lib.ref_solve_patch_wos.argtypes = [_P, _P, _P, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_int, C.c_int, _P, _P, _P, C.POINTER(C.c_int)]
    return lib


@pytest.fixture(scope="module")
def libs(reflib, gpu):
    if not INTEG.exists():
        pytest.fail(f"{INTEG} missing: build it with `make -C integration` (needs /root/reference)")
    return _bind(C.CDLL(str(INTEG))), _bind(reflib)


def test_estimate_u_batch_through_the_binding(libs):
    integ, ref = libs
    scene = Scene.sphere(1.0, DomainSide.Interior, Quadratic(g=(0, 0, 1.0), q=(1.0, -1.0, 0, 0, 0, 0)))
    cfg = WosConfig(eps_shell=1e-4, n_paths=2000, seed=11)
    pts = np.random.default_rng(2).uniform(-0.5, 0.5, (48, 3))
    a, b = (O.ref_estimate(l, scene.to_c(), cfg.to_c(), pts, base=5) for l in (integ, ref))
    assert a[0] == 0 and b[0] == 0
    ea, eb = a[1], b[1]
    assert (ea["n"] == eb["n"]).all()
    close = np.abs(ea["mean"] - eb["mean"]) <= 1e-10 * np.maximum(1, np.abs(eb["mean"]))
    assert close.mean() >= 0.95


def test_estimate_u_batch_through_the_binding_statistical_mode(libs, monkeypatch):
    """BW_RNG=philox4x32: the binding's estimate_u_batch on the library's
    statistical mode against the reference's own (independent streams): same
    walk counts, paired z-scores of a unit normal."""
    integ, ref = libs
    scene = Scene.sphere(1.0, DomainSide.Interior, Quadratic(g=(0, 0, 1.0), q=(1.0, -1.0, 0, 0, 0, 0)))
    cfg = WosConfig(eps_shell=1e-4, n_paths=2000, seed=11)
    pts = np.random.default_rng(4).uniform(-0.55, 0.55, (400, 3))
    monkeypatch.setenv("BW_RNG", "philox4x32")
    a = O.ref_estimate(integ, scene.to_c(), cfg.to_c(), pts, base=5)
    monkeypatch.delenv("BW_RNG")
    a64 = O.ref_estimate(integ, scene.to_c(), cfg.to_c(), pts, base=5)
    b = O.ref_estimate(ref, scene.to_c(), cfg.to_c(), pts, base=5)
    assert a[0] == 0 and b[0] == 0 and a64[0] == 0
    ea, eb = a[1], b[1]
    assert (ea["n"] == eb["n"]).all()
    assert not np.array_equal(ea["mean"], a64[1]["mean"])  # the switch took effect
    z = (ea["mean"] - eb["mean"]) / np.sqrt((ea["variance"] + eb["variance"]) / 2000)
    assert (np.abs(z) > 3).mean() <= 0.015 and abs(z.mean()) < 0.2 and 0.8 < z.var() < 1.2


def test_reference_solve_point_runs_on_the_device(libs):
    """point_solver.cpp's solve_point (sigma1_prime -> estimate_u_batch,
    point_solver.cpp:166) on the reference's half-space Test-1 scene
    (tests/test_point_solver.cpp:12-15, 146-157)."""
    integ, ref = libs
    scene = Scene.half_space(0.0, PointSource(q=1.0, s=(0.0, 0.0, -1.0)))
    cfg = WosConfig(n_paths=1000, seed=2024)
    c, ax = np.array([0.5, 0.0, 0.0]), np.array([0.0, 0.0, 1.0])
    out = []
    for lib in (integ, ref):
        r = np.zeros(4)
        st = lib.ref_solve_point_wos(C.byref(scene.to_c()), C.byref(cfg.to_c()), O.p(c), 0.5,
                                     O.p(ax), 20, 20, 0.5e-4, 8, O.p(r))
        assert st == 0
        out.append(r)
    di, dr = out
    assert di[1] == dr[1]                         # sigma2: deterministic, same CPU code
    assert abs(di[0] - dr[0]) <= 1e-9 * abs(dr[0]) + 0.25 * dr[3]  # same walks up to ulps
    analytic = 1.0 / 1.25 ** 1.5                   # test_point_solver.cpp:37
    assert abs(di[2] - analytic) < 4 * di[3] + 2e-4  # the reference's own gate (:154)


def test_reference_solve_patch_runs_on_the_device(libs):
    """patch_solver.cpp's solve_patch with a WOS-sampled Gamma grid
    (sample_gamma_grid -> estimate_u_batch, patch_solver.cpp:135) on the
    reference's exterior sphere case (tests/test_patch_solver.cpp:193-209)."""
    integ, ref = libs
    scene = Scene.sphere(3.0, DomainSide.Exterior, 1.0 / (12 * np.pi))
    cfg = WosConfig(n_paths=2000, seed=3)
    o = np.array([0.0, 0.0, 3.0])
    res = []
    for lib in (integ, ref):
        m = C.c_int()
        lib.ref_solve_patch_wos(C.byref(scene.to_c()), C.byref(cfg.to_c()), O.p(o), 1.0, 4, 8, 8,
                                16, 0, 8, None, None, None, C.byref(m))
        d, r, e = np.zeros(m.value), np.zeros(m.value), np.zeros(m.value)
        st = lib.ref_solve_patch_wos(C.byref(scene.to_c()), C.byref(cfg.to_c()), O.p(o), 1.0, 4,
                                     8, 8, 16, 0, 8, O.p(d), O.p(r), O.p(e), C.byref(m))
        assert st == 0
        res.append((d, r, e))
    (dg, rg, eg), (dr, rr, er) = res
    assert np.array_equal(rg, rr)
    # same streams: per-panel du/dn and the propagated error equal up to the
    # rounding of a few walks (the coarse 4 x 8 mesh and 8 x 16 grid of the
    # reference's grid test are not an accuracy case; test_patch_solver.cpp
    # gates them on the Gamma values only)
    assert (np.abs(dg - dr) <= 1e-9 * np.abs(dr).max() + 0.5 * er).all()
    assert np.allclose(eg, er, rtol=0.05)


def test_reference_evaluate_runs_on_the_device(libs):
    """field_eval.cpp's evaluate() replaced by K3: the reference's sphere case
    (tests/test_field_eval.cpp: R = 3 sphere, target at |x| = 4) and its
    NearFieldError."""
    integ, ref = libs
    rng = np.random.default_rng(5)
    n = 4000
    p = rng.normal(size=(n, 3))
    p = 3.0 * p / np.linalg.norm(p, axis=1, keepdims=True)
    nrm = p / 3.0
    area = np.full(n, 4 * np.pi * 9 / n)
    u = 1.0 / (4 * np.pi * 3.0) * np.ones(n)
    dudn = -1.0 / (4 * np.pi * 9) * np.ones(n)
    panels = np.concatenate([p, nrm, area[:, None], u[:, None], dudn[:, None]], axis=1)
    t = np.array([[0, 0, 4.0], [4.0, 0, 0], [0, 3.0, 0.001]])
    out = []
    for lib in (integ, ref):
        uu, near = np.zeros(3), np.zeros(3, np.uint8)
        lib.ref_evaluate(O.p(panels), n, O.p(t), 3, O.p(uu), O.p(near))
        out.append((uu, near))
    (ug, ng), (ur, nr) = out
    assert (ng == nr).all() and ng[2] == 1
    assert np.allclose(ug[:2], ur[:2], rtol=1e-12, atol=0)
