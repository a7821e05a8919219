"""Time K4 (bw_dtn_assemble_d), K2 and K5 alone on config-4 patches (device data)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1210_1491_b200 import _native as N, dtn, nodes  # noqa: E402
from paper_1210_1491_b200.workloads import CONFIGS  # noqa: E402
from paper_1210_1491_b200.wos import WosConfig  # noqa: E402

cfgno = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nbp = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
w = CONFIGS[cfgno]()
w = w.subset(np.unique(np.linspace(0, w.n_bp - 1, nbp).astype(np.int64)))
ctx = N.context(0)
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
P = dtn.patches_for(w)
d_p = torch.from_numpy(P.view(np.uint8).copy()).to(dev)
d_dirs = torch.from_numpy(w.dirs).to(dev)
d_w = torch.from_numpy(np.ascontiguousarray(w.weights)).to(dev)
est, _ = nodes.wos_patch_nodes(w.scene, WosConfig(eps_shell=w.eps, n_paths=64, seed=1), w.points,
                               w.axes, w.radii, w.dirs, cls=w.cls)
d_est = torch.from_numpy(est.view(np.uint8).copy()).to(dev)
dc = dtn.DtnConfig()
m = dc.m
A = torch.empty(nbp * m * m, dtype=torch.float64, device=dev)
b = torch.empty(nbp * 2 * m, dtype=torch.float64, device=dev)
area = torch.empty(nbp * m, dtype=torch.float64, device=dev)
flags = torch.empty(nbp, dtype=torch.int32, device=dev)
sc, cc = w.scene.to_c(), dc.to_c()


def k4():
    ctx.check(ctx.lib.bw_dtn_assemble_d(ctx.handle, C.byref(sc), d_p.data_ptr(), nbp,
                                        d_dirs.data_ptr(), d_w.data_ptr(), w.dirs.shape[0],
                                        w.n_nodes, d_est.data_ptr(), C.byref(cc), A.data_ptr(),
                                        b.data_ptr(), area.data_ptr(), flags.data_ptr()))


k4()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(3):
    k4()
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"K4 cfg{cfgno} {nbp} patches: {ms:.2f} ms = {ms * 1e3 / nbp:.2f} us/patch "
      f"(-> {ms / nbp * 1e5:.0f} ms per 1e5)")
