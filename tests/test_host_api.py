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
