"""GPU: the full pipeline (DtN -> all-gather -> potential) on a small sphere
problem: the potential equals the oracle's long-double sum over the same
panels to 1e-10, and approximates the analytic harmonic solution."""
from __future__ import annotations

import numpy as np
import pytest

import oracle_lib as O
from paper_1210_1491_b200 import pipeline, workloads

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rng_kind", [0, 1], ids=["philox4x64", "philox4x32"])
def test_pipeline_sphere(gpu, orc, rng_kind):
    w = workloads._ball("ball_small", 3000, 0.1, 8, 16, 1024, 1e-5, 7)
    rng = np.random.default_rng(1)
    t = rng.normal(size=(500, 3))
    t *= (rng.uniform(0.0, 0.6, 500) ** (1 / 3) / np.linalg.norm(t, axis=1))[:, None]
    u, near, res, panels = pipeline.run(w, t, device=0, rng=rng_kind)
    assert not near.any() and (res.status == 0).all()
    u_ref, near_ref = O.or_potential(orc, panels, t, long_double=True)
    assert (np.abs(u - u_ref) / (np.abs(u_ref) + 1e-3)).max() < 1e-10
    exact = w.exact_u(t)
    assert np.median(np.abs(u - exact)) < 0.02
