"""Strong-scaling projection of the config-4 DtN step on ONE GPU (not product code).

Only 1-GPU boxes exist in this run, so N-GPU scaling is estimated from the one
thing that sets it: the device time of each rank's strided shard. For every
N in --worlds and every rank r < N, the rank's shard (distributed.shard_ids,
global stream ids, the same dtn_solve_device call bench.py times) runs alone
on the GPU: W warm-up steps, then K steps between CUDA events. The projected
whole-job value at N is total walk steps / max over ranks of the shard time,
i.e. bench.py's value with the ranks' kernels on separate GPUs. Not included:
NCCL (config 4's step has no data-path collective; bench.py's two all-reduces
of a scalar sit outside the timed region) and host/launch jitter across GPUs.

usage: python tools/shard_scaling.py [--config 4] [--worlds 1,2,4,8] [--steps 2] [--warmup 1]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--rng", type=int, default=32, choices=[32, 64])
    args = ap.parse_args()
    import torch

    import paper_1210_1491_b200 as bw
    from paper_1210_1491_b200 import _native as N
    from paper_1210_1491_b200 import dtn
    from paper_1210_1491_b200.distributed import shard_ids
    from paper_1210_1491_b200.workloads import CONFIGS

    w = CONFIGS[args.config]()
    dev = torch.device("cuda", 0)
    ctx = N.context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    cfg = w.wos_config(rng=bw.wos.RNG_PHILOX4X32 if args.rng == 32 else bw.wos.RNG_PHILOX4X64)
    dcfg = dtn.DtnConfig()
    all_patches = dtn.patches_for(w)
    d_dirs = torch.from_numpy(w.dirs).to(dev)
    d_wts = torch.from_numpy(np.ascontiguousarray(w.weights)).to(dev)
    n_cls = w.dirs.shape[0]

    def time_shard(rank, world):
        ids = shard_ids(w.n_bp, rank, world)
        n = len(ids)
        d_patches = torch.from_numpy(all_patches[ids].view(np.uint8).copy()).to(dev)
        d_ids = torch.from_numpy(ids).to(dev)
        d_dudn = torch.empty(n, dtype=torch.float64, device=dev)
        d_err = torch.empty(n, dtype=torch.float64, device=dev)
        d_status = torch.empty(n, dtype=torch.int32, device=dev)
        d_est = torch.empty(n * w.n_nodes * 40, dtype=torch.uint8, device=dev)
        d_steps = torch.empty(n * w.n_nodes, dtype=torch.int64, device=dev)

        def step():
            dtn.dtn_solve_device(w.scene, cfg, dcfg, d_patches.data_ptr(), d_ids.data_ptr(), n,
                                 d_dirs.data_ptr(), d_wts.data_ptr(), n_cls, w.n_nodes,
                                 d_dudn.data_ptr(), d_err.data_ptr(), d_status.data_ptr(),
                                 d_est.data_ptr(), d_steps.data_ptr(), device=0)

        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        bad = int((d_status != 0).sum().item())
        return ms, int(d_steps.sum().item()), d_dudn.cpu().numpy(), ids, bad

    out = {"config": args.config, "n_bp": w.n_bp, "steps": args.steps, "warmup": args.warmup,
           "worlds": {}}
    dudn_ref = None
    v1 = None
    for world in [int(x) for x in args.worlds.split(",")]:
        ms_r, steps_tot, bad = [], 0, 0
        dudn = np.empty(w.n_bp)
        for r in range(world):
            ms, st, du, ids, b = time_shard(r, world)
            ms_r.append(ms)
            steps_tot += st
            bad += b
            dudn[ids] = du
        if dudn_ref is None:
            dudn_ref = dudn
        value = steps_tot / (max(ms_r) * 1e-3)
        v1 = v1 or (value if world == 1 else None)
        rec = {"ms_per_rank": [round(x, 3) for x in ms_r], "ms_max": max(ms_r),
               "imbalance_max_over_mean": max(ms_r) / (sum(ms_r) / world),
               "walk_steps": steps_tot, "projected_value": value, "failed_points": bad,
               "dudn_bitwise_equal_to_first_world": bool(np.array_equal(dudn, dudn_ref))}
        if v1:
            rec["projected_efficiency"] = value / (world * v1)
        out["worlds"][str(world)] = rec
        print(json.dumps({str(world): rec}), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
