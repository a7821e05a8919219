"""GPU: last-passage estimator (K_lp) — the reference's LP test cases
(tests/test_last_passage.cpp of the reference)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1210_1491_b200 as bw
from paper_1210_1491_b200.last_passage import estimate_lp
from paper_1210_1491_b200.point_solver import HemisphereFrame
from paper_1210_1491_b200.geometry import PointSource, Scene

pytestmark = pytest.mark.gpu


def test_applicability(gpu):
    hs = Scene.half_space(0.0, PointSource(q=1.0, s=(0, 0, -1.0)))
    f = HemisphereFrame((0.5, 0, 0), 0.1)
    with pytest.raises(bw.ApplicabilityError):
        estimate_lp(hs, f, 100, bw.WosConfig())
    estimate_lp(hs, f, 100, bw.WosConfig(), allow_general_data=True)
    with pytest.raises(bw.ApplicabilityError):  # two-level but not {0,1}
        estimate_lp(Scene.four_plates([2, 0, 0, 0]), HemisphereFrame((0.5, 0.5, 0), 0.2), 100,
                    bw.WosConfig())
    with pytest.raises(bw.ApplicabilityError):  # base on a 0 V plate
        estimate_lp(Scene.four_plates([0, 1, 0, 0]), HemisphereFrame((0.5, 0.5, 0), 0.2), 100,
                    bw.WosConfig())


def test_thin_disk_density(gpu):
    s = Scene.thin_disk(1.0, 1.0)
    r = estimate_lp(s, HemisphereFrame((-0.5, 0, 0), 0.4), 100000, bw.WosConfig(seed=5))
    analytic = 0.735105
    assert abs(r.sigma_lp - analytic) < 4 * r.std_error + 0.01 * analytic
    assert r.n_paths == 100000
    assert r.n_infinity + r.n_failed + sum(r.feature_counts) == 100000


def test_four_plates_trend(gpu):
    s = Scene.four_plates([0, 1, 0, 0])
    A = (-0.2273, 0.2273, 0.0)
    cfg = bw.WosConfig(seed=9)
    ref = 2.607
    small = estimate_lp(s, HemisphereFrame(A, 0.2), 100000, cfg)
    assert abs(small.sigma_lp - ref) < 4 * small.std_error + 0.013 * ref
    errs = [abs(estimate_lp(s, HemisphereFrame(A, a), 40000, cfg).sigma_lp - ref) / ref
            for a in (0.3, 0.5, 0.7)]
    assert errs[1] > errs[0] and errs[2] > errs[1] and errs[2] > 0.2


def test_determinism(gpu):
    s = Scene.thin_disk(1.0, 1.0)
    f = HemisphereFrame((-0.5, 0, 0), 0.4)
    r1 = estimate_lp(s, f, 20000, bw.WosConfig(seed=31, workers=1))
    r2 = estimate_lp(s, f, 20000, bw.WosConfig(seed=31, workers=8))
    assert r1.sigma_lp == r2.sigma_lp and r1.n_infinity == r2.n_infinity
    assert r1.feature_counts == r2.feature_counts


def test_plate_and_disk_walks_match_oracle(gpu, orc):
    """WOS on the reference's flat scenes: device walks vs the oracle's."""
    import oracle_lib as O

    rng = np.random.default_rng(4)
    for scene in (Scene.four_plates([1, 0, 0, 0]), Scene.thin_disk(1.0, 1.0)):
        starts = np.column_stack([rng.uniform(-1.2, 1.2, 1000), rng.uniform(-1.2, 1.2, 1000),
                                  rng.uniform(0.05, 0.5, 1000)])
        cfg = bw.WosConfig(eps_shell=1e-5, seed=7)
        pids = np.arange(1000, dtype=np.uint64)
        ex, f, st = bw.walk_batch(scene, starts, cfg, pids, 3)
        s0, ex_o, f_o, st_o = O.or_walk(orc, scene.to_c(), cfg.to_c(), starts, pids, 3)
        assert s0 == 0
        same = (f == f_o) & (st == st_o)
        assert same.mean() >= 0.999
