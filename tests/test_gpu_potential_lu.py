"""GPU parity of K3 (potential sum) and K2 (batched LU) against the oracle:
<= 1e-10 relative in fp64 given identical inputs (BASELINE north star)."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
import paper_1210_1491_b200 as bw
from golden.make_golden import sphere_panels

pytestmark = pytest.mark.gpu
GOLD = np.load(Path(__file__).parent / "golden" / "ref_vectors.npz")


def test_potential_matches_reference_golden(gpu):
    u, near = bw.evaluate_batch(GOLD["pot_panels"], GOLD["pot_targets"])
    assert not near.any()
    assert np.allclose(u, GOLD["pot_u"], rtol=1e-10, atol=1e-13)


def test_potential_1e10_vs_long_double_oracle(gpu, orc):
    rng = np.random.default_rng(0)
    panels = sphere_panels(1.0, 1.0, 20000)
    panels[:, 7] = rng.uniform(-1, 1, len(panels))
    panels[:, 8] = rng.uniform(-1, 1, len(panels))
    t = rng.normal(size=(3000, 3))
    t *= (rng.uniform(0.05, 0.9, 3000) / np.linalg.norm(t, axis=1))[:, None]
    t = np.concatenate([t, rng.uniform(-3, 3, (1000, 3)) + [0, 0, 5]])
    u, near = bw.evaluate_batch(panels, t)
    u_ref, near_ref = O.or_potential(orc, panels, t, long_double=True)
    assert (near == near_ref).all()
    ok = ~near
    scale = np.abs(u_ref[ok]) + 1e-3 * np.abs(u_ref[ok]).max()
    assert (np.abs(u[ok] - u_ref[ok]) / scale).max() < 1e-10


def test_potential_point_charge_and_vanishing(gpu):  # test_field_eval.cpp:45-63
    d = sphere_panels(3.0, 1.0, 5000)
    u, _ = bw.evaluate_batch(d, [[4, 0, 0], [0, -4, 0], [0.2, 0.1, -0.3]])
    e = 1 / (16 * np.pi)
    assert abs(u[0] - e) < 0.01 * e and abs(u[1] - e) < 0.01 * e
    assert abs(u[2]) < 0.01 / (12 * np.pi)
    x, prev = [[0, 0, 4.5]], None
    for n in (500, 2000, 8000):
        err = abs(bw.evaluate_batch(sphere_panels(3.0, 1.0, n), x)[0][0] - 1 / (4 * np.pi * 4.5))
        if prev is not None:
            assert err < prev / 1.8
        prev = err


def test_potential_zero_linear_nearfield(gpu):  # test_field_eval.cpp:36-43, 65-87
    d = sphere_panels(3.0, 1.0, 500)
    z = d.copy()
    z[:, 7:] = 0
    assert bw.evaluate(z, [4, 0, 0]) == 0.0
    rng = np.random.default_rng(3)
    d1 = sphere_panels(2.0, 1.0, 800)
    d2 = d1.copy()
    d2[:, 7:] = rng.random((len(d2), 2)) - 0.5
    mix = d1.copy()
    mix[:, 7:] = 1.7 * d1[:, 7:] - 0.4 * d2[:, 7:]
    x = [3.5, -1, 0.5]
    assert np.isclose(bw.evaluate(mix, x), 1.7 * bw.evaluate(d1, x) - 0.4 * bw.evaluate(d2, x),
                      rtol=1e-13)
    with pytest.raises(bw.NearFieldError):
        bw.evaluate(d, d[7, :3] + [0.01, 0, 0])
    u, near = bw.evaluate_batch(d, [d[7, :3] + [0.01, 0, 0], [4, 0, 0]])
    assert near.tolist() == [True, False] and np.isnan(u[0])


@pytest.mark.parametrize("m", [1, 5, 33, 40, 64])
def test_lu_matches_oracle(gpu, orc, m):
    rng = np.random.default_rng(m)
    n = 300
    A = rng.normal(size=(n, m, m)) + 0.5 * np.eye(m) * m ** 0.5
    B = rng.normal(size=(n, 2, m))
    X, res, info = bw.lu_solve_batched(A, B)
    Xo, reso, infoo = np.empty_like(B), np.empty(n), np.empty(n, np.int32)
    orc.or_lu_solve_batched(m, n, O.p(A), O.p(B), 2, O.p(Xo), O.p(reso), O.p(infoo))
    assert (info == 0).all() and (infoo == 0).all()
    rel = np.abs(X - Xo).max(axis=(1, 2)) / np.abs(Xo).max(axis=(1, 2))
    cond = np.linalg.cond(A)
    assert (rel < 1e-13 * cond).all() and np.median(rel) < 1e-12
    assert (res < 1e-10).all()


def test_lu_pivot_ties_and_singular(gpu):
    A = np.array([[[0.0, 1.0], [0.0, 2.0]]])  # singular
    with pytest.raises(bw.SolverError):
        bw.lu_solve_batched(A, np.ones((1, 2)))
    X, res, info = bw.lu_solve_batched(A, np.ones((1, 2)), raise_on_fail=False)
    assert info[0] == 1
    # needs pivoting: zero leading entry
    A = np.array([[[0.0, 2.0], [3.0, 1.0]]])
    X, res, info = bw.lu_solve_batched(A, [[2.0, 4.0]])
    assert np.allclose(X[0], [1.0, 1.0]) and info[0] == 0
