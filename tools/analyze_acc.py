"""Worst Neumann points of a config (accuracy diagnosis)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1210_1491_b200 import dtn  # noqa: E402
from paper_1210_1491_b200.workloads import CONFIGS  # noqa: E402

c = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
w = CONFIGS[c]()
w = w.subset(np.unique(np.linspace(0, w.n_bp - 1, n).astype(np.int64)))
r = dtn.dtn_solve_workload(w)
ex = w.exact_dudn_outward()
z = (r.dudn - ex) / r.err
o = np.argsort(-np.abs(z))[:12]
np.set_printoptions(precision=5, suppress=True, linewidth=200)
print("n", w.n_bp, "frac |z|>3:", np.mean(np.abs(z) > 3), "median |z|", np.median(np.abs(z)))
for i in o:
    print(i, "cls", w.cls[i], "a", round(w.radii[i], 5), "p", w.points[i], "ax", w.axes[i], "exact", ex[i],
          "got", r.dudn[i], "err", r.err[i], "z", z[i])
for cl in (0, 1):
    m = (w.cls == 0) if cl == 0 else (w.cls > 0)
    if m.any():
        print("class", "face" if cl == 0 else "cavity", "n", m.sum(), "frac|z|>3", np.mean(np.abs(z[m]) > 3),
              "median rel", np.median(np.abs(r.dudn[m] - ex[m]) / np.abs(ex[m])))
