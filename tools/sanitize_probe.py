"""Small invocations of every device kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): K1 on the sphere (both streams), K1 on the
cavity box with the candidate grid in shared memory, the DtN step (K7 class
tables and the K4 -> K2 -> K5 per-patch path), solve_patch through the large-
patch kernels, K3, the point formula, last passage, and the device group.
No torch (ctypes only). Not product code."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1210_1491_b200 as bw  # noqa: E402
from paper_1210_1491_b200 import dtn, field_eval, nodes, pipeline, workloads  # noqa: E402
from paper_1210_1491_b200.wos import RNG_PHILOX4X32  # noqa: E402

D = 0
w4 = workloads.config4(20000).subset(np.arange(0, 20000, 4000))
for rng in (0, RNG_PHILOX4X32):
    r = dtn.dtn_solve(w4.scene, w4.wos_config(64, rng), dtn.patches_for(w4), w4.dirs, w4.weights,
                      device=D)
    print("K1+K7 sphere rng", rng, r.dudn[:2])
w3 = workloads.config3()
idx = np.unique(np.linspace(0, w3.n_bp - 1, 12).astype(np.int64))
w3 = w3.subset(idx)
r3 = dtn.dtn_solve(w3.scene, w3.wos_config(64, RNG_PHILOX4X32), dtn.patches_for(w3), w3.dirs,
                   w3.weights, return_nodes=True, device=D)
print("K1+K7 cavities", r3.dudn[:2])
b = dtn.dtn_neumann(w3.scene, dtn.patches_for(w3), w3.dirs, w3.weights, r3.node_est,
                    method=dtn.DTN_PER_PATCH, device=D)
print("K4->K2->K5", b.dudn[:2])
f = dtn.solve_patch(w3.scene, dtn.patches_for(w3)[:2], w3.dirs, w3.weights, r3.node_est[:2],
                    dtn.DtnConfig(bands=8, azimuth=10), device=D)
print("large patch", f.dudn[0, :2])
area = pipeline.panel_areas(w3)
pan = np.concatenate([w3.points, w3.axes, area[:, None],
                      np.asarray(w3.scene.phi(w3.points))[:, None], -r3.dudn[:, None]], axis=1)
t = workloads.make_targets(workloads.config3(), 300, seed=5)
u, near = field_eval.evaluate_batch(pan, t, device=D)
print("K3", u[:2])
s = bw.Scene.half_space(0.0, bw.PointSource(q=1.0, s=(0, 0, -1.0)))
from paper_1210_1491_b200.last_passage import estimate_lp  # noqa: E402
from paper_1210_1491_b200.point_solver import HemisphereFrame, solve_point  # noqa: E402

lp = estimate_lp(s, HemisphereFrame((0.5, 0, 0), 0.1), 5000, bw.WosConfig(seed=3),
                 allow_general_data=True, device=D)
print("LP", lp.sigma_lp)
pr = solve_point(s, HemisphereFrame((0.5, 0, 0), 0.5), 8, 8, 0.5e-4,
                 bw.WosConfig(n_paths=64, seed=1), device=D)
print("point formula", pr.total)
g = bw.DeviceGroup([D, D])
res = g.pipeline(w3.scene, w3.wos_config(64), dtn.patches_for(w3), w3.dirs, w3.weights, area,
                 np.asarray(w3.scene.phi(w3.points)), t)
g.close()
print("group pipeline", res.u[:2])
