"""K3 alone on config 5's panel set (200,000 panels with the analytic du/dn) at
N_TARGETS targets drawn like the benchmark's: one warm-up and one measured
launch, for `ncu --set full -k regex:potential_kernel -s 1 -c 1`. Not product code."""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1210_1491_b200 import field_eval, pipeline, workloads  # noqa: E402

n_t = int(os.environ.get("N_TARGETS", "100000"))
w = workloads.config5()
area = pipeline.panel_areas(w)
dudn_in = (w.exact_grad(w.points) * w.axes).sum(axis=1)
panels = np.concatenate([w.points, w.axes, area[:, None],
                         np.asarray(w.scene.phi(w.points))[:, None], dudn_in[:, None]], axis=1)
t = workloads.make_targets(w, n_t, seed=5)
for _ in range(2):
    t0 = time.perf_counter()
    u, near = field_eval.evaluate_batch(panels, t)
    print(f"{len(panels)} panels x {n_t} targets: {time.perf_counter() - t0:.3f} s "
          f"(host call), near {int(near.sum())}")
