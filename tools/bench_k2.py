"""K2 (batched LU + 2 right-hand sides + residual) timing on N systems of size
m (default: config 4's patch systems, m = 54, 1e5 systems, well-conditioned
random matrices), device-resident, CUDA events. Not product code.
usage: python tools/bench_k2.py [m] [n_sys] [nrhs] [dump.npz]
(the dump holds X, resid, info for a bitwise A/B of two library builds)"""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1210_1491_b200 import _native as N  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 54
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
nrhs = int(sys.argv[3]) if len(sys.argv) > 3 else 2
dump = sys.argv[4] if len(sys.argv) > 4 else None
rng = np.random.default_rng(1)
A = rng.standard_normal((n, m, m)) + m * np.eye(m)[None]
B = rng.standard_normal((n, nrhs, m))
dev = torch.device("cuda", 0)
dA, dB = torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev)
dX = torch.empty_like(dB)
dr = torch.empty(n, dtype=torch.float64, device=dev)
di = torch.empty(n, dtype=torch.int32, device=dev)
ctx = N.context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
f = ctx.lib.bw_lu_solve_batched_d


def run():
    ctx.check(f(ctx.handle, m, n, dA.data_ptr(), dB.data_ptr(), nrhs, 1e-10, dX.data_ptr(),
                dr.data_ptr(), di.data_ptr()))


run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
flops = n * (2.0 / 3.0 * m ** 3 + 2 * nrhs * m * m)
X = dX.cpu().numpy()
ok = np.allclose(np.einsum("nij,nrj->nri", A[:64], X[:64]), B[:64], rtol=1e-9, atol=1e-9)
if dump:
    np.savez(dump, X=X, resid=dr.cpu().numpy(), info=di.cpu().numpy())
print(json.dumps({"m": m, "nrhs": nrhs, "n_sys": n, "ms": ms, "systems_per_s": n / (ms * 1e-3),
                  "tflops": flops / (ms * 1e-3) / 1e12, "solutions_ok": bool(ok),
                  "max_resid": float(dr.max().item())}))
