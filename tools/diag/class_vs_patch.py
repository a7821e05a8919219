"""Diagnostic: K7 (class tables) vs K4->K2->K5 vs the CPU oracle on a cfg3 mix."""
import sys
import numpy as np
sys.path.insert(0, "tests")
import oracle_lib as O
from paper_1210_1491_b200 import dtn
from test_gpu_dtn import _mixed_cfg3, _nodes, _oracle_dudn

orc = O.oracle()
w = _mixed_cfg3()
res = _nodes(w)
P = dtn.patches_for(w)
a = dtn.dtn_neumann(w.scene, P, w.dirs, w.weights, res.node_est, method=dtn.DTN_CLASSES)
b = dtn.dtn_neumann(w.scene, P, w.dirs, w.weights, res.node_est, method=dtn.DTN_PER_PATCH)
ref = _oracle_dudn(orc, w, res, range(w.n_bp))
np.set_printoptions(linewidth=200, precision=3)
for k in range(w.n_bp):
    print(k, w.cls[k], "%.4g" % w.radii[k], "%.6g" % ref[k, 0],
          "cls-ref %.2e" % ((a.dudn[k] - ref[k, 0]) / abs(ref[k, 0])),
          "patch-ref %.2e" % ((b.dudn[k] - ref[k, 0]) / abs(ref[k, 0])), a.status[k], b.status[k])
