"""bench.py — walk-steps/s of the B200 WOS hot path on a BASELINE workload.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl b200|reference]

A step is one full pass of K1 over every Gamma node of the configuration's
boundary points (config 4 = the BASELINE scaling run: 100,000 Fibonacci
points on the unit ball x 128 nodes x 4,096 walks). Boundary points are
sharded strided across ranks (one process per GPU, torchrun); each point keeps
its global stream ids, so results do not depend on N. `value` = all ranks'
walk steps / max-over-ranks device time. `e2e` = the same metric through the
public host API (host arrays in pinned memory, H2D + kernel + D2H in the timed
region). `--impl reference` times the reference's own CPU code path
(oracle/_ref: the reference sources' estimate_u_batch) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# Algorithmic FP64 flops per WOS step: 18 geometry-independent
# + the distance (sphere 7, box 11, box + 64 cavities brute force 715).
F_STEP = {"sphere": 25, "box": 29, "cavities": 733}
# K1 warp-instructions per walk step (sphere scenes), from the ncu capture in
# executed warp-instructions / walk steps of one K1 launch (ncu --set full):
# profiles/r1/ncu_k1_summary.md 28,942,442,807 / 4,280,616,624 (sphere) and
# profiles/r1/ncu_k1_cavities_summary.md 28,570,923,739 / 2,646,657,884 (cavities)
K1_WARP_INSTR_PER_STEP = {"sphere": 6.473, "cavities": 10.650}
# dram__bytes_read.sum + dram__bytes_write.sum of one full config-4 K1 launch
# (1e5 points; profiles/r1/ncu_k1_dram_traffic_cfg4.csv): 374,476,800 + 1,206,835,200
K1_TRAFFIC_CFG4 = 374476800 + 1206835200
METRIC = "WOS walk-steps/s (fp64)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--n-bp", type=int, default=0, help="override boundary-point count")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--n-targets", type=int, default=0)
    ap.add_argument("--rng", type=int, default=64, choices=[64, 32],
                    help="K1 stream: 64 = the reference's Philox4x64-10 RngStream (bit-exact "
                         "parity mode), 32 = Philox4x32-10 (statistical parity)")
    return ap.parse_args()


def dist_setup():
    """One process per GPU (torchrun env). BW_BENCH_BACKEND=gloo (a check of
    the N > 1 bookkeeping on a one-GPU box: ranks share the device, their
    kernels never wait on each other) replaces NCCL; the driver's runs use NCCL."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        import torch

        backend = os.environ.get("BW_BENCH_BACKEND", "nccl")
        if backend != "nccl":
            local %= max(1, torch.cuda.device_count())
            torch.cuda.set_device(local)
            dist.init_process_group(backend)
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def scene_class(w) -> str:
    from paper_1210_1491_b200.geometry import SceneKind

    return {SceneKind.Sphere: "sphere", SceneKind.Box: "box"}.get(w.scene.kind, "cavities")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "power_w_max": max(float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit())
                if any(r[2].replace(".", "").isdigit() for r in self.rows) else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_reference_assembly_s(w, reps: int = 0):
    """Seconds per boundary point of the reference's own collocation step on
    one host thread: make_sphere_patch_setup + sample_gamma_grid (exact data) +
    assemble (patch_solver.cpp:197-309) through oracle/_ref, on a patch of the
    workload's mesh (5 bands x 6 azimuth = 54 panels, radius a of point 0). The
    reference's sphere patch is exterior-side; the cost is the same. None when
    the reference build is absent."""
    import ctypes as C

    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O
    from paper_1210_1491_b200.geometry import DomainSide, PointSource, Scene

    if not O.ref_available():
        return None
    lib = O.ref()
    f = lib.ref_sphere_patch_assemble_kind
    P = C.c_void_p
    f.argtypes = [P, P, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int] + [P] * 8
    sc = Scene.sphere(1.0, DomainSide.Exterior, PointSource(q=1 / (4 * np.pi), s=(0, 0, 0))).to_c()
    o = np.array([0.0, 0.0, 1.0])
    a = float(w.radii[0])
    m, ng = C.c_int(), C.c_int()
    f(C.byref(sc), O.p(o), a, 5, 6, 8, 16, 0, *([None] * 6), C.byref(m), C.byref(ng))
    A, b, bse = np.zeros((m.value, m.value)), np.zeros(m.value), np.zeros(m.value)
    gy, gw, gu = np.zeros((ng.value, 3)), np.zeros(ng.value), np.zeros(ng.value)

    def once():
        f(C.byref(sc), O.p(o), a, 5, 6, 8, 16, 0, O.p(A), O.p(b), O.p(bse), O.p(gy), O.p(gw),
          O.p(gu), C.byref(m), C.byref(ng))

    t0 = time.perf_counter()
    once()
    t1 = time.perf_counter() - t0
    reps = reps or max(3, min(200, int(2.0 / max(t1, 1e-4))))
    t0 = time.perf_counter()
    for _ in range(reps):
        once()
    return (time.perf_counter() - t0) / reps


def cpu_reference_rate(w, bp_idx, gpu_steps_of, seconds: float, workers: int):
    """The reference's own estimate_u_batch (oracle/_ref, compiled from the
    reference sources) over the Gamma nodes of the first boundary points, on
    `workers` host threads. Steps are counted from the identical device
    trajectories of the same nodes (same stream ids)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O
    from paper_1210_1491_b200 import nodes

    use_ref = O.ref_available()
    lib = O.ref() if use_ref else O.oracle()
    sc = w.scene.to_c()

    def run(k):
        b = bp_idx[:k]
        pos = nodes.patch_node_positions(w.points[b], w.axes[b], w.radii[b], w.cls[b], w.dirs)
        # one estimate_u_batch per boundary point (point ids b*n_nodes + j), with
        # that point's shell eps_b (Workload.eps_of), as the device walks it
        cfs = [w.wos_config(eps=w.eps_of(int(bi))).to_c() for bi in b]
        t0 = time.perf_counter()
        steps = 0
        for i, bi in enumerate(b):
            cf = cfs[i]
            if use_ref:
                st, _ = O.ref_estimate(lib, sc, cf, pos[i], base=int(bi) * w.n_nodes,
                                       workers=workers)
            else:
                st, _, s = O.or_estimate(lib, sc, cf, pos[i], base=int(bi) * w.n_nodes,
                                         workers=workers)
            steps += int(gpu_steps_of(bi))
        return time.perf_counter() - t0, steps

    k = 1
    dt, steps = run(k)
    # grow the sample until one run takes ~`seconds` of CPU time (10-30 s)
    while dt < 0.6 * seconds and k < len(bp_idx):
        k = min(len(bp_idx), max(k * 2, int(k * seconds / max(dt, 1e-3))))
        dt, steps = run(k)
    out = {"value": steps / dt, "unit": "walk-steps/s", "cores": workers,
           "kind": "reference" if use_ref else "port",
           "sample": f"{k} boundary points x {w.n_nodes} nodes x {w.n_paths} walks of "
                     f"{w.name} ({steps} steps, {dt:.1f} s), reference estimate_u_batch "
                     f"with workers={workers}"}
    t_a = cpu_reference_assembly_s(w)
    if t_a is not None:
        # WOS of a point on all threads, then its collocation (points in parallel)
        out["neumann_points_per_s"] = 1.0 / (dt / k + t_a / workers)
        out["assembly_s_per_point_1thread"] = t_a
    return out


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1210_1491_b200.workloads import CONFIGS

    w = CONFIGS[args.config]()
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O
    from paper_1210_1491_b200 import nodes

    use_ref = O.ref_available()
    lib = O.ref() if use_ref else O.oracle()
    orc = O.oracle()
    workers = os.cpu_count() or 1
    sc = w.scene.to_c()
    # bounded sample: Gamma nodes of `nb` boundary points spread over the
    # boundary; steps per sample counted once by the oracle (same streams); each
    # point walks with its shell eps_b (Workload.eps_of) as on the device
    budget = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    nb = 1
    while True:
        b = np.linspace(0, w.n_bp - 1, nb).astype(np.int64)
        pos = nodes.patch_node_positions(w.points[b], w.axes[b], w.radii[b], w.cls[b], w.dirs)
        cfs = [w.wos_config(eps=w.eps_of(int(bi))).to_c() for bi in b]
        t0 = time.perf_counter()
        for i, bi in enumerate(b):
            (O.ref_estimate if use_ref else O.or_estimate)(lib, sc, cfs[i], pos[i],
                                                           base=int(bi) * w.n_nodes,
                                                           workers=workers)
        dt = time.perf_counter() - t0
        if dt >= budget / 3 or nb >= w.n_bp:
            break
        nb = min(w.n_bp, max(nb * 2, int(nb * budget / max(dt, 1e-3) * 0.8)))
    steps_sample = 0
    for i, bi in enumerate(b):
        _, _, s = O.or_estimate(orc, sc, cfs[i], pos[i], base=int(bi) * w.n_nodes,
                                workers=workers)
        steps_sample += int(s.sum())

    def step():
        for i, bi in enumerate(b):
            (O.ref_estimate if use_ref else O.or_estimate)(lib, sc, cfs[i], pos[i],
                                                           base=int(bi) * w.n_nodes,
                                                           workers=workers)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    v = steps_sample / dt
    sample = (f"{nb} of {w.n_bp} boundary points (evenly spaced) x {w.n_nodes} Gamma nodes x "
              f"{w.n_paths} walks = {steps_sample} walk steps per step")
    cpu = {"value": v, "unit": "walk-steps/s", "cores": workers,
           "kind": "reference" if use_ref else "port", "sample": sample}
    t_a = cpu_reference_assembly_s(w)
    if t_a is not None:
        cpu["neumann_points_per_s"] = 1.0 / (dt / nb + t_a / workers)
        cpu["assembly_s_per_point_1thread"] = t_a
    print(json.dumps({
        "metric": METRIC, "value": v, "unit": "walk-steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config, seeded generators)", "impl": "reference",
        "config": {"workload": w.name, "n_bp": w.n_bp, "nodes_per_bp": w.n_nodes,
                   "walks_per_node": w.n_paths, "eps_shell": w.eps, "seed": w.seed},
        "cpu_baseline": cpu,
        "e2e": {"value": v, "unit": "walk-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }))


def run_pipeline_bench(args):
    """Config 5: WOS -> collocation -> LU -> all-gather -> potential at 1e6
    targets (pipeline.py); one step = the whole pipeline."""
    import torch

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    from paper_1210_1491_b200 import pipeline
    from paper_1210_1491_b200.workloads import config5, make_targets

    w = config5()
    if args.n_bp and args.n_bp < w.n_bp:
        w = w.subset(np.unique(np.linspace(0, w.n_bp - 1, args.n_bp).astype(np.int64)))
    n_t = args.n_targets or w.extra.get("n_targets", 1000000)
    targets = make_targets(w, n_t, seed=5)
    stream = torch.cuda.current_stream()
    marks = {}

    def timer(name):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        marks.setdefault(name, []).append(ev)

    for _ in range(args.warmup):
        pipeline.run(w, targets, device=local)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    from paper_1210_1491_b200 import _native as N5
    lctx = N5.context(local)
    launches0 = lctx.launch_count()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            u, near, res, panels = pipeline.run(w, targets, device=local, timer=timer)
        torch.cuda.synchronize()
    launches = lctx.launch_count() - launches0
    phases = ["start", "dtn", "allgather", "potential", "gather"]
    ph_ms = {}
    for a, b in zip(phases[:-1], phases[1:]):
        ph_ms[b] = float(np.mean([x.elapsed_time(y) for x, y in zip(marks[a], marks[b])]))
    ms = float(np.mean([x.elapsed_time(y) for x, y in zip(marks["start"], marks["gather"])]))
    t = torch.tensor([ms, float(res.steps)], dtype=torch.float64, device=torch.device("cuda", local))
    if world > 1:
        tmax = t.clone()
        torch.distributed.all_reduce(tmax, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(t)
        ms_max, steps = float(tmax[0]), float(t[1])
    else:
        ms_max, steps = ms, float(t[1])
    if rank != 0:
        return
    exact = w.exact_u(targets)
    ok = ~near
    dist_b = np.min(np.abs(np.abs(targets) - 1.0), axis=1)
    cav = w.extra["cavities"]
    for c in cav:
        dist_b = np.minimum(dist_b, np.linalg.norm(targets - c[:3], axis=1) - c[3])
    far = ok & (dist_b > 0.1)
    rel = np.abs(u - exact) / np.abs(exact)
    print(json.dumps({
        "metric": METRIC, "value": steps / (ms_max * 1e-3), "unit": "walk-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config 5, seeded generators)",
        "config": {"workload": w.name, "n_bp": w.n_bp, "n_targets": n_t,
                   "nodes_per_bp": w.n_nodes, "walks_per_node": w.n_paths},
        "phase_ms": ph_ms,
        "neumann_points_per_s": w.n_bp / (ph_ms["dtn"] * 1e-3),
        "potential_pairs_per_s": w.n_bp * n_t / (ph_ms["potential"] * 1e-3),
        "near_field_targets": int(near.sum()),
        "flagged_points": int((res.status != 0).sum()),
        "potential_rel_err_median_far": float(np.median(rel[far])),
        "potential_rel_err_p99_far": float(np.quantile(rel[far], 0.99)),
        "clocks": clk.summary(),
        "gpu_launches": launches,
    }))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.config == 5:
        run_pipeline_bench(args)
        return
    import torch

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    import paper_1210_1491_b200 as bw
    from paper_1210_1491_b200 import _native as N
    from paper_1210_1491_b200 import dtn, nodes
    from paper_1210_1491_b200.distributed import shard_ids
    from paper_1210_1491_b200.workloads import CONFIGS

    w = CONFIGS[args.config]()
    if args.n_bp and args.n_bp < w.n_bp:  # evenly spaced subset (faces and cavities alike)
        w = w.subset(np.unique(np.linspace(0, w.n_bp - 1, args.n_bp).astype(np.int64)))
    ctx = N.context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)

    # strided shard of boundary points; global ids keep the streams
    ids = shard_ids(w.n_bp, rank, world)
    n_loc = len(ids)
    dev = torch.device("cuda", local)
    patches = dtn.patches_for(w)[ids]
    d_patches = torch.from_numpy(patches.view(np.uint8).copy()).to(dev)
    d_ids = torch.from_numpy(ids).to(dev)
    d_dirs = torch.from_numpy(w.dirs).to(dev)
    d_wts = torch.from_numpy(np.ascontiguousarray(w.weights)).to(dev)
    d_dudn = torch.empty(n_loc, dtype=torch.float64, device=dev)
    d_err = torch.empty(n_loc, dtype=torch.float64, device=dev)
    d_status = torch.empty(n_loc, dtype=torch.int32, device=dev)
    d_est = torch.empty(n_loc * w.n_nodes * 40, dtype=torch.uint8, device=dev)
    d_steps = torch.empty(n_loc * w.n_nodes, dtype=torch.int64, device=dev)
    cfg = w.wos_config(rng=bw.wos.RNG_PHILOX4X32 if args.rng == 32 else bw.wos.RNG_PHILOX4X64)
    dcfg = dtn.DtnConfig()
    n_cls = w.dirs.shape[0]

    def step():
        """One pass of the hot path: K1 (all Gamma nodes) -> K7 (class-table DtN)."""
        dtn.dtn_solve_device(w.scene, cfg, dcfg, d_patches.data_ptr(), d_ids.data_ptr(), n_loc,
                             d_dirs.data_ptr(), d_wts.data_ptr(), n_cls, w.n_nodes,
                             d_dudn.data_ptr(), d_err.data_ptr(), d_status.data_ptr(),
                             d_est.data_ptr(), d_steps.data_ptr(), device=local)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lctx = N.context(local)
    launches0 = lctx.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = lctx.launch_count() - launches0
    if world > 1:
        torch.distributed.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    local_steps = int(d_steps.sum().item())
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    s = torch.tensor([local_steps], dtype=torch.int64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(s)
    ms_max = float(t.item())
    total_steps = int(s.item())
    value = total_steps / (ms_max * 1e-3)
    gpu_steps = d_steps.view(n_loc, w.n_nodes).sum(1).cpu().numpy()
    n_bad = int((d_status != 0).sum().item())

    # K1 alone (the dominant kernel) for the roofline line: same inputs
    d_c = torch.from_numpy(np.ascontiguousarray(w.points[ids])).to(dev)
    d_ax = torch.from_numpy(np.ascontiguousarray(w.axes[ids])).to(dev)
    d_r = torch.from_numpy(np.ascontiguousarray(w.radii[ids])).to(dev)
    d_cls = torch.from_numpy(w.cls[ids].astype(np.int32)).to(dev)
    k1_iters = 1
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k1_iters):
        nodes.wos_patch_nodes_device(w.scene, cfg, d_c.data_ptr(), d_ax.data_ptr(),
                                     d_r.data_ptr(), d_cls.data_ptr(), d_ids.data_ptr(), n_loc,
                                     d_dirs.data_ptr(), n_cls, w.n_nodes, 0, d_est.data_ptr(),
                                     d_steps.data_ptr(), device=local)
    e1.record(stream)
    torch.cuda.synchronize()
    k1_ms = e0.elapsed_time(e1) / k1_iters

    # ---- e2e: public host API (bw_dtn_solve), pinned host buffers, copies in the timed region
    e2e = None
    if not args.no_e2e:
        def pinned(a):
            t_ = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
            return t_.numpy()

        h_patches = pinned(patches.view(np.uint8)).view(dtn.PATCH_DTYPE)
        h_ids, h_dirs, h_wts = pinned(ids), pinned(w.dirs), pinned(w.weights)
        e2e_steps = max(1, min(args.steps, 2))
        dtn.dtn_solve(w.scene, cfg, h_patches, h_dirs, h_wts, dcfg, bp_ids=h_ids, device=local)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            r = dtn.dtn_solve(w.scene, cfg, h_patches, h_dirs, h_wts, dcfg, bp_ids=h_ids,
                              device=local)
        e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
        te = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        h2d = sum(a.nbytes for a in (h_patches, h_ids, h_dirs, h_wts))
        d2h = r.dudn.nbytes + r.err.nbytes + r.status.nbytes
        e2e = {"value": total_steps / (float(te.item()) * 1e-3), "unit": "walk-steps/s",
               "h2d_bytes_per_step": int(h2d) * world, "d2h_bytes_per_step": int(d2h) * world,
               "ms_per_step": float(te.item()),
               "neumann_points_per_s": w.n_bp / (float(te.item()) * 1e-3),
               "api": "dtn.dtn_solve -> bw_dtn_solve (host arrays in, Neumann data out)"}

    if rank != 0:
        return
    peak_tf, _ = ctx.fp64_peak()
    f_step = F_STEP[scene_class(w)]
    clock_summary = clk.summary()
    # K1's real bound is instruction issue (Philox integer work + fp64 chains):
    # achieved warp-instructions per SM-cycle against the 4 issue slots per SM
    issue = None
    ipc_k = K1_WARP_INSTR_PER_STEP.get(scene_class(w))
    if ipc_k is not None:
        n_sm, _ = ctx.device_info()
        mhz = clock_summary.get("sm_mhz") or 1965.0
        ipc = ipc_k * (local_steps / (k1_ms * 1e-3)) / (n_sm * mhz * 1e6)
        issue = {"bound": "issue", "kernel": "K1 wos_nodes_kernel",
                 "warp_instructions_per_step": ipc_k,
                 "source": "ncu executed instructions / walk steps (profiles/r1/ncu_k1_summary.md)",
                 "achieved_ipc_per_sm": ipc, "peak_ipc_per_sm": 4.0, "frac": ipc / 4.0}
        # the stream's own floor: 15 wide Philox products per block (= 64 lane-steps
        # of two jumps each over a warp), at the measured mulhilo64 rate of 0.205 per
        # SM-cycle (tools/diag/int_pipes.cu, profiles/r1/int_pipes_microbench.log)
        ceil = 0.205 / (15.0 / 64.0) * n_sm * mhz * 1e6
        issue["stream_product_bound"] = {
            "products_per_walk_step": 15.0 / 64.0, "mulhilo64_per_sm_cycle": 0.205,
            "ceiling_walk_steps_per_s": ceil,
            "frac": (local_steps / (k1_ms * 1e-3)) / ceil}
    achieved = f_step * local_steps / (k1_ms * 1e-3) / 1e12
    cpu = None
    if not args.no_cpu and world == 1:
        steps_of = dict(zip(ids.tolist(), gpu_steps.tolist()))
        cpu = cpu_reference_rate(w, ids, lambda b: steps_of[int(b)], args.cpu_seconds,
                                 os.cpu_count() or 1)
    exact = w.exact_dudn_outward()[ids] if w.exact_grad is not None else None
    out = {
        "metric": METRIC, "value": value, "unit": "walk-steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config, seeded generators; no dataset)",
        "config": {"workload": w.name, "n_bp": w.n_bp, "nodes_per_bp": w.n_nodes,
                   "walks_per_node": w.n_paths, "eps_shell": w.eps, "seed": w.seed,
                   "a": w.a, "patch_panels": dcfg.m, "parallelism": f"bp-sharded x{world}",
                   "l2": "compute-bound; per-step node/patch arrays (>2 GB) exceed L2"},
        "neumann_points_per_s": w.n_bp / (ms_max * 1e-3),
        "walk_steps_per_step": total_steps,
        "walks_per_s": w.n_bp * w.n_nodes * w.n_paths / (ms_max * 1e-3),
        "k1_share_of_step": k1_ms / ms,
        "neumann_check": None if exact is None else {
            "max_abs_dev_over_err": float(np.max(np.abs(d_dudn.cpu().numpy() - exact)
                                                 / np.maximum(d_err.cpu().numpy(), 1e-300))),
            "median_rel_err": float(np.median(np.abs(d_dudn.cpu().numpy() - exact)
                                              / np.maximum(np.abs(exact), 1e-12))),
            "flagged_points": n_bad,
            "scope": "all points" if world == 1 else f"rank 0's shard ({n_loc} of {w.n_bp} points)"},
        "roofline": {"bound": "fp64", "kernel": "K1 wos_nodes_kernel",
                     "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": achieved / peak_tf,
                     "peak_source": "measured on this device by bw_measure_fp64_peak (DFMA loop; "
                                    "MEASURED_PEAKS.json has no fp64 entry)",
                     "flops_per_walk_step": f_step,
                     "traffic": K1_TRAFFIC_CFG4 if (w.name == "cfg4_unit_ball_scaling"
                                                    and w.n_bp == 100000 and world == 1) else None,
                     "traffic_note": "bytes per K1 launch (ncu, DRAM read+write): 1.58 GB over "
                                     "~12.9 s, ~0.12 GB/s of the 6.5 TB/s HBM; the walk state "
                                     "stays on chip, only 40 B estimates + 8 B step counts "
                                     "per node leave it (0.61 GB algorithmic)"},
        "gpu_launches": launches,
        "clocks": clock_summary,
        "issue": issue,
        "cpu_baseline": cpu,
        "e2e": e2e,
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
