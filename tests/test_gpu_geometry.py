"""The reference's geometry tests (tests/test_geometry.cpp) on the device
geometry (bw_nearest_feature / bw_distance_to_boundary / bw_classify_exit),
plus: the device argmin equals the oracle's bit for bit, and the distance K1's
walk loop computes (cavity candidate grid with early exit) equals it."""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle_lib as O
import paper_1210_1491_b200 as bw
from paper_1210_1491_b200.geometry import DomainSide, PointSource, Scene, SinSin

pytestmark = pytest.mark.gpu


def _halfspace_test1():
    return Scene.half_space(0.0, PointSource(q=1.0, s=(0, 0, -1.0)))


def test_distance_half_space(gpu):  # test_geometry.cpp:20-27
    q = bw.distance_to_boundary(_halfspace_test1(), (3, -7, 2))
    assert abs(q.distance - 2.0) <= 1e-14 * 2 and q.feature == 0
    for p in ((0, 0, -0.1), (0, 0, 0.0)):
        with pytest.raises(bw.DomainError):
            bw.distance_to_boundary(_halfspace_test1(), p)


def test_distance_thin_disk(gpu):  # test_geometry.cpp:29-43
    s = Scene.thin_disk(1.0, 1.0)
    assert abs(bw.distance_to_boundary(s, (0, 0, 0.5)).distance - 0.5) < 1e-14
    assert abs(bw.distance_to_boundary(s, (2, 0, 0)).distance - 1.0) < 1e-12
    p = np.array([1.3, 0.4, 0.7])
    rho = np.arange(401) / 400.0
    th = 2 * math.pi * np.arange(1200) / 1200.0
    R, T = np.meshgrid(rho, th)
    y = np.stack([R * np.cos(T), R * np.sin(T), np.zeros_like(R)], -1)
    best = np.linalg.norm(y - p, axis=-1).min()
    d = bw.distance_to_boundary(s, p).distance
    assert abs(d - best) <= 2e-4 * (1 + best)


def test_distance_plates_argmin_low_index_ties(gpu):  # test_geometry.cpp:45-52
    s = Scene.four_plates([1, 0, 0, 0])
    q = bw.distance_to_boundary(s, (-0.5, 0.5, 0.25))
    assert abs(q.distance - 0.25) < 1e-12 and q.feature == 1
    assert bw.distance_to_boundary(s, (0.0, 0.5, 0.1)).feature == 0


def test_classify_exit_truncation_shell_plates(gpu):  # test_geometry.cpp:70-80
    hs = _halfspace_test1()
    assert bw.classify_exit(hs, (2e5, 0, 0), 1e-5, 1e5).feature == bw.kExitInfinity
    assert bw.classify_exit(hs, (0, 0, 1e-6), 1e-5, 1e5).feature == 0
    plates = Scene.four_plates([0, 0, 1, 0])
    r = bw.classify_exit(plates, (-0.5, -0.5, 1e-6), 1e-5, 1e5)
    assert r.feature == 2 and r.point[2] == 0.0
    with pytest.raises(bw.ClassificationError):
        bw.classify_exit(plates, (0, 0, 0.5), 1e-5, 1e5)


def test_classify_exit_idempotent(gpu):  # test_geometry.cpp:82-93
    s = Scene.four_plates([1, 0, 0, 0])
    rng = np.random.default_rng(5)
    p = np.stack([rng.uniform(-1, 1, 200), rng.uniform(-1, 1, 200), 1e-6 * rng.uniform(0, 1, 200)], 1)
    q1, f1 = bw.classify_exit_batch(s, p, 1e-5, 1e5)
    q2, f2 = bw.classify_exit_batch(s, q1, 1e-5, 1e5)
    assert (f1 == f2).all()
    assert np.abs(q1 - q2).max() <= 1e-15


def test_maximal_ball_empty_and_lipschitz(gpu):  # test_geometry.cpp:95-128
    rng = np.random.default_rng(17)
    for s in (Scene.thin_disk(1.0, 1.0), Scene.four_plates([1, 0, 0, 0])):
        p = np.stack([rng.uniform(-1.5, 1.5, 100), rng.uniform(-1.5, 1.5, 100),
                      rng.uniform(-1, 1, 100)], 1)
        p = p[np.abs(p[:, 2]) >= 1e-9]
        d, _ = bw.nearest_feature_batch(s, p)
        if s.kind == bw.SceneKind.ThinDisk:
            rho, th = rng.uniform(0, 1, 500), rng.uniform(0, 2 * math.pi, 500)
            y = np.stack([rho * np.cos(th), rho * np.sin(th), np.zeros(500)], 1)
        else:
            y = np.stack([rng.uniform(-1, 1, 500), rng.uniform(-1, 1, 500), np.zeros(500)], 1)
        dist = np.linalg.norm(p[:, None, :] - y[None], axis=-1)
        assert (dist >= d[:, None] * (1 - 1e-12)).all()
    s = Scene.thin_disk(1.0, 1.0)
    a = np.stack([rng.uniform(-2, 2, 500), rng.uniform(-2, 2, 500), 0.1 + rng.uniform(0, 1, 500)], 1)
    b = np.stack([rng.uniform(-2, 2, 500), rng.uniform(-2, 2, 500), 0.1 + rng.uniform(0, 1, 500)], 1)
    da, _ = bw.nearest_feature_batch(s, a)
    db, _ = bw.nearest_feature_batch(s, b)
    assert (np.abs(da - db) <= np.linalg.norm(a - b, axis=1) * (1 + 1e-12)).all()


def test_sphere_scenes_both_sides(gpu):  # test_geometry.cpp:136-144
    inn = Scene.sphere(2.0, DomainSide.Interior, 1.0)
    ext = Scene.sphere(2.0, DomainSide.Exterior, 1.0)
    assert abs(bw.distance_to_boundary(inn, (0, 0, 0)).distance - 2.0) < 1e-14
    assert abs(bw.distance_to_boundary(ext, (0, 0, 5)).distance - 3.0) < 1e-14
    with pytest.raises(bw.DomainError):
        bw.distance_to_boundary(inn, (0, 0, 3))
    with pytest.raises(bw.DomainError):
        bw.distance_to_boundary(ext, (0, 0, 1))
    q = bw.classify_exit(ext, (0, 0, 2.0 + 1e-7), 1e-5, 1e5)
    assert q.feature == 0 and abs(q.point[2] - 2.0) < 1e-15


@pytest.mark.parametrize("kind", ["plates_sine", "disk", "cube", "cavities", "cavities_fine"])
def test_device_geometry_matches_oracle(gpu, orc, kind, monkeypatch):
    """Argmin feature and distance equal the oracle's (the reference's
    geometry.cpp restated) bit for bit; K1's walk-loop distance equals them.
    "cavities_fine" asks for a 48^3 candidate grid, whose lists pass the 16-bit
    offset range: the upload coarsens it until they fit."""
    from paper_1210_1491_b200.workloads import make_cavities

    if kind == "cavities_fine":
        monkeypatch.setenv("BW_CAVITY_GRID", "48")

    rng = np.random.default_rng(3)
    if kind == "plates_sine":
        s = Scene.plate_set([[0, 1, 0, 1], [-1, 0, 0, 1], [-1, 0, -1, 0], [0, 1, -1, 0]],
                            SinSin(1.0, (1.0, 1.0)))
        p = rng.uniform(-1.5, 1.5, (3000, 3))
    elif kind == "disk":
        s = Scene.thin_disk(1.0, 1.0)
        p = rng.uniform(-1.5, 1.5, (3000, 3))
    elif kind == "cube":
        s = Scene.box((0, 0, 0), (1, 1, 1), [1.0] * 6)
        p = rng.uniform(0.0, 1.0, (3000, 3))
    else:  # cavities, cavities_fine
        cav = make_cavities(64, 3, clearance=0.04)
        s = Scene.box_with_cavities((-1, -1, -1), (1, 1, 1), cav, PointSource(1.0, tuple(cav[0, :3])))
        p = rng.uniform(-1.0, 1.0, (20000, 3))
    d, f, dw = bw.nearest_feature_batch(s, p, walk_distance=True)
    sc = s.to_c()
    ref_d = np.empty(len(p))
    ref_f = np.empty(len(p), np.int32)
    import ctypes as C
    for i, x in enumerate(p):
        ff = C.c_int()
        ref_d[i] = orc.or_nearest_feature(C.byref(sc), O.p(np.ascontiguousarray(x)), C.byref(ff))
        ref_f[i] = ff.value
    assert (f == ref_f).all()
    assert np.array_equal(d, ref_d) or np.abs(d - ref_d).max() <= 4e-16 * np.abs(ref_d).max()
    assert (np.abs(dw - d) <= 2.3e-16 * np.maximum(d, 1e-300) + 1e-300).all()
