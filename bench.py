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
# + the distance (sphere 7, box 11). The cavity box counts the work K1 executes,
# not the reference's brute force over all 64 cavities (715 flops, culled here by
# the exact candidate grid): 11 for the faces + 11 per candidate a lane visits,
# 0.43 per step on config 3 (profiles/r1/cavity_loop_stats_cfg3.log).
F_STEP = {"sphere": 25, "box": 29, "cavities": 34}
F_STEP_REFERENCE = {"sphere": 25, "box": 29, "cavities": 733}
# ncu metrics of one K1 launch, measured by bench.py itself in a child process
# (k1_probe) on a bounded sample of the workload's nodes
NCU_METRICS = ["gpu__time_duration.sum", "smsp__inst_executed.sum",
               "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
               "sm__inst_issued.avg.pct_of_peak_sustained_active",
               "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
               "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second"]
# optional (a probe without it still counts): the fp64 share of the executed
# instructions, for the dispatch-port figure (K1)
NCU_OPTIONAL = ["smsp__inst_executed_pipe_fp64.sum"]
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
    ap.add_argument("--rng", type=int, default=32, choices=[64, 32],
                    help="K1 stream: 32 = Philox4x32-10 (statistical parity, the default "
                         "headline), 64 = the reference's Philox4x64-10 RngStream (bit-exact "
                         "parity mode, also timed in every run as `parity_mode`)")
    ap.add_argument("--no-parity-mode", action="store_true")
    ap.add_argument("--no-profile", action="store_true",
                    help="skip the ncu child process that measures K1's pipe utilisation")
    ap.add_argument("--k1-probe", type=int, default=0, help=argparse.SUPPRESS)
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


def shard_ids_all(n, rank, world):
    return np.arange(rank, n, world, dtype=np.int64)


def run_pipeline_bench(args):
    """Config 5: WOS -> collocation -> LU -> all-gather -> potential at 1e6
    targets (pipeline.py); one step = the whole pipeline."""
    import torch

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    from paper_1210_1491_b200 import pipeline
    from paper_1210_1491_b200.workloads import config5, make_targets

    from paper_1210_1491_b200 import wos as W

    w = config5()
    if args.n_bp and args.n_bp < w.n_bp:
        w = w.subset(np.unique(np.linspace(0, w.n_bp - 1, args.n_bp).astype(np.int64)))
    n_t = args.n_targets or w.extra.get("n_targets", 1000000)
    targets = make_targets(w, n_t, seed=5)
    rng = W.RNG_PHILOX4X32 if args.rng == 32 else W.RNG_PHILOX4X64
    stream = torch.cuda.current_stream()
    marks = {}

    def timer(name):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        marks.setdefault(name, []).append(ev)

    for _ in range(args.warmup):
        pipeline.run(w, targets, device=local, rng=rng)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    from paper_1210_1491_b200 import _native as N5
    lctx = N5.context(local)
    launches0 = lctx.launch_count()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            u, near, res, panels = pipeline.run(w, targets, device=local, timer=timer, rng=rng)
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
    # diagnosis of the potential error: the same panels with the analytic du/dn
    # (the quadrature error of the one-point panels alone), all targets, K3
    from paper_1210_1491_b200 import field_eval
    from paper_1210_1491_b200.pipeline import panel_areas

    pe = panels.copy()
    pe[:, 8] = (w.exact_grad(w.points) * w.axes).sum(axis=1)
    torch.cuda.synchronize()
    k0, k1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d_pe = torch.from_numpy(pe).to(torch.device("cuda", local))
    d_tg = torch.from_numpy(np.ascontiguousarray(targets)).to(torch.device("cuda", local))
    d_ue = torch.empty(n_t, dtype=torch.float64, device=d_tg.device)
    d_ne = torch.empty(n_t, dtype=torch.uint8, device=d_tg.device)
    field_eval.evaluate_device(d_pe.data_ptr(), w.n_bp, d_tg.data_ptr(), n_t, d_ue.data_ptr(),
                               d_ne.data_ptr(), device=local)  # warm-up
    k0.record(stream)
    field_eval.evaluate_device(d_pe.data_ptr(), w.n_bp, d_tg.data_ptr(), n_t, d_ue.data_ptr(),
                               d_ne.data_ptr(), device=local)
    k1e.record(stream)
    torch.cuda.synchronize()
    k3_ms = k0.elapsed_time(k1e)
    ue = d_ue.cpu().numpy()
    rel_e = np.abs(ue - exact) / np.abs(exact)
    # dudn error of the DtN on each stratum (the cavity-0 points carry the field)
    dd = res.dudn - w.exact_dudn_outward()[shard_ids_all(w.n_bp, rank, world)]
    cav0 = w.cls[shard_ids_all(w.n_bp, rank, world)] == 1
    ctx5 = N5.context(local)
    peak_tf, _ = ctx5.fp64_peak()
    pairs = float(w.n_bp) * n_t
    k3_pairs_s = pairs / (k3_ms * 1e-3)
    k3_bytes = 72.0 * w.n_bp + 32.0 * n_t   # panels + targets in, u + flag out
    print(json.dumps({
        "metric": METRIC, "value": steps / (ms_max * 1e-3), "unit": "walk-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config 5, seeded generators)",
        "config": {"workload": w.name, "n_bp": w.n_bp, "n_targets": n_t,
                   "nodes_per_bp": w.n_nodes, "walks_per_node": w.n_paths,
                   "rng": "philox4x32-10" if args.rng == 32 else "philox4x64-10"},
        "phase_ms": ph_ms,
        "neumann_points_per_s": w.n_bp / (ph_ms["dtn"] * 1e-3),
        "potential_pairs_per_s": w.n_bp * n_t / (ph_ms["potential"] * 1e-3),
        "near_field_targets": int(near.sum()),
        "flagged_points": int((res.status != 0).sum()),
        "potential_rel_err_median_far": float(np.median(rel[far])),
        "potential_rel_err_p99_far": float(np.quantile(rel[far], 0.99)),
        "potential_error_diagnosis": {
            "exact_dudn_rel_err_median_far": float(np.median(rel_e[far])),
            "exact_dudn_rel_err_p99_far": float(np.quantile(rel_e[far], 0.99)),
            "dtn_rel_err_median_cavity0": float(np.median(np.abs(dd[cav0]) /
                                                          np.abs(w.exact_dudn_outward()[
                                                              shard_ids_all(w.n_bp, rank, world)][cav0])))
            if cav0.any() else None,
            "dtn_signed_rel_err_mean_cavity0": float(np.mean(dd[cav0] / np.abs(w.exact_dudn_outward()[
                shard_ids_all(w.n_bp, rank, world)][cav0]))) if cav0.any() else None,
            "note": "the same 2e5 panels with the analytic du/dn give the quadrature error "
                    "alone; the rest is the DtN bias of the 54-panel sphere patch on cavity 0 "
                    "(whose single layer carries u = 1/|x - c0|): -0.44 % with exact Gamma data "
                    "(DESIGN.md section 3)"},
        "k3_roofline": {"bound": "fp64", "kernel": "K3 potential_kernel",
                        "achieved": 21.0 * k3_pairs_s / 1e12, "peak": peak_tf, "unit": "TFLOP/s",
                        "frac": 21.0 * k3_pairs_s / 1e12 / peak_tf, "pairs_per_s": k3_pairs_s,
                        "flops_per_pair": 21, "ms": k3_ms,
                        "hbm_gb_per_s_algorithmic": k3_bytes / (k3_ms * 1e-3) / 1e9,
                        "traffic_algorithmic_bytes": k3_bytes,
                        "note": "all 1e6 targets x all panels on one device, analytic du/dn "
                                "panels (same shapes as the pipeline's)"},
        "clocks": clk.summary(),
        "gpu_launches": launches,
    }))


def main():
    args = parse()
    if args.k1_probe:
        k1_probe(args)
        return
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
        """One pass of the hot path: K1 (all Gamma nodes) -> K7 (class-table DtN).
        A soft error on one rank's shard (reliability, solver) is flagged in
        d_status and reported in neumann_check; no rank raises alone."""
        dtn.dtn_solve_device(w.scene, cfg, dcfg, d_patches.data_ptr(), d_ids.data_ptr(), n_loc,
                             d_dirs.data_ptr(), d_wts.data_ptr(), n_cls, w.n_nodes,
                             d_dudn.data_ptr(), d_err.data_ptr(), d_status.data_ptr(),
                             d_est.data_ptr(), d_steps.data_ptr(), device=local, soft=True)

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
    main_dudn, main_err = d_dudn.clone(), d_err.clone()  # the timed steps' Neumann data

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

    # ---- the parity mode: the same step on the reference's Philox4x64 stream
    parity = None
    if not args.no_parity_mode and cfg.rng != bw.wos.RNG_PHILOX4X64:
        cfg64 = w.wos_config(rng=bw.wos.RNG_PHILOX4X64)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        dtn.dtn_solve_device(w.scene, cfg64, dcfg, d_patches.data_ptr(), d_ids.data_ptr(), n_loc,
                             d_dirs.data_ptr(), d_wts.data_ptr(), n_cls, w.n_nodes,
                             d_dudn.data_ptr(), d_err.data_ptr(), d_status.data_ptr(),
                             d_est.data_ptr(), d_steps.data_ptr(), device=local, soft=True)
        p1.record(stream)
        torch.cuda.synchronize()
        tp = torch.tensor([p0.elapsed_time(p1)], dtype=torch.float64, device=dev)
        sp = torch.tensor([int(d_steps.sum().item())], dtype=torch.int64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(tp, op=torch.distributed.ReduceOp.MAX)
            torch.distributed.all_reduce(sp)
        parity = {"rng": "philox4x64-10 (the reference's RngStream, rng.hpp:44-67; bit-exact "
                         "walks)", "value": int(sp.item()) / (float(tp.item()) * 1e-3),
                  "unit": "walk-steps/s", "ms_per_step": float(tp.item()), "steps_timed": 1,
                  "neumann_points_per_s": w.n_bp / (float(tp.item()) * 1e-3)}
        # the two stream modes on the same points (independent streams): the
        # z-scores of their Neumann values are those of a unit normal
        zz = (main_dudn - d_dudn) / torch.hypot(main_err, d_err)
        zz = zz[torch.isfinite(zz)]
        zs = torch.stack([zz.sum(), (zz * zz).sum(), (zz.abs() > 3).double().sum(),
                          torch.tensor(float(zz.numel()), dtype=torch.float64, device=dev)])
        if world > 1:
            torch.distributed.all_reduce(zs)
        s1_, s2_, n3_, nn_ = (float(v) for v in zs.tolist())
        if nn_ > 1:
            mz = s1_ / nn_
            parity["neumann_z_vs_headline_mode"] = {
                "n": int(nn_), "mean": mz, "std": max(s2_ / nn_ - mz * mz, 0.0) ** 0.5,
                "frac_abs_gt3": n3_ / nn_,
                "note": "z = (dudn_statistical - dudn_parity) / hypot(err, err) per boundary "
                        "point; independent streams, so N(0, 1) up to the error estimate's own noise"}

    # ---- e2e: public host API (bw_dtn_solve), pinned host buffers, copies in the
    # timed region; with N > 1 the Neumann data are gathered to rank 0 over NCCL
    e2e = None
    if not args.no_e2e:
        from paper_1210_1491_b200.distributed import allgather_strided

        def pinned(a):
            t_ = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
            return t_.numpy()

        h_patches = pinned(patches.view(np.uint8)).view(dtn.PATCH_DTYPE)
        h_ids, h_dirs, h_wts = pinned(ids), pinned(w.dirs), pinned(w.weights)
        e2e_steps = max(1, min(args.steps, 2))
        gathered = {}

        def e2e_step():
            r_ = dtn.dtn_solve(w.scene, cfg, h_patches, h_dirs, h_wts, dcfg, bp_ids=h_ids,
                               device=local)
            if world > 1:
                loc = torch.from_numpy(np.stack([r_.dudn, r_.err, r_.status.astype(np.float64)],
                                                axis=1)).to(dev)
                full = allgather_strided(loc, w.n_bp)
                if rank == 0:
                    gathered["all"] = full.cpu().numpy()
            return r_

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            r = e2e_step()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
        te = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        h2d = sum(a.nbytes for a in (h_patches, h_ids, h_dirs, h_wts)) * world
        d2h = (r.dudn.nbytes + r.err.nbytes + r.status.nbytes) * world
        if world > 1:  # the gathered copy of all Neumann data on rank 0
            h2d += 24 * w.n_bp
            d2h += 24 * w.n_bp
        e2e = {"value": total_steps / (float(te.item()) * 1e-3), "unit": "walk-steps/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": float(te.item()),
               "neumann_points_per_s": w.n_bp / (float(te.item()) * 1e-3),
               "api": "dtn.dtn_solve -> bw_dtn_solve (host arrays in, Neumann data out)" +
                      ("; all ranks' du/dn, err, status all-gathered over NCCL and copied to "
                       "rank 0's host" if world > 1 else "")}

    if rank != 0:
        return
    peak_tf, _ = ctx.fp64_peak()
    f_step = F_STEP[scene_class(w)]
    clock_summary = clk.summary()
    n_sm, _ = ctx.device_info()
    k1_rate = local_steps / (k1_ms * 1e-3)
    achieved = f_step * k1_rate / 1e12
    # ncu metrics of K1, measured now on a bounded sample of this workload
    prof = None if (args.no_profile or world > 1) else profile_k1(args, w)
    traffic, pipes = None, None
    if prof:
        per_node = (prof["dram__bytes_read.sum"] + prof["dram__bytes_write.sum"]) / prof["nodes"]
        traffic = per_node * n_loc * w.n_nodes
        mhz = clock_summary.get("sm_mhz") or 1965.0
        wi = prof["smsp__inst_executed.sum"] / prof["walk_steps"]
        pipes = {"source": f"ncu --metrics (child process, {prof['nodes']} Gamma nodes of this "
                           f"workload, one K1 launch after a warm-up)",
                 "fp64_pipe_pct": prof["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"],
                 "issue_slots_pct": prof["sm__inst_issued.avg.pct_of_peak_sustained_active"],
                 "fmaheavy_pipe_pct": prof["sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active"],
                 "warp_instructions_per_walk_step": wi,
                 "achieved_ipc_per_sm_full_launch": wi * k1_rate / (n_sm * mhz * 1e6),
                 "dram_bytes_per_node": per_node}
        n64 = prof.get("smsp__inst_executed_pipe_fp64.sum")
        if n64:
            # an fp64 warp-instruction holds the SMSP's dispatch port for two
            # cycles (tools/diag/dispatch_mix.cu): port use = issue (1 + share),
            # and the FP64 pipe cannot pass 2 share / (1 + share) for this mix
            share = n64 / prof["smsp__inst_executed.sum"]
            pipes["fp64_share_of_instructions"] = share
            pipes["dispatch_port_pct"] = pipes["issue_slots_pct"] * (1.0 + share)
            pipes["fp64_pipe_ceiling_pct_for_this_mix"] = 100.0 * 2.0 * share / (1.0 + share)
    cpu = None
    if not args.no_cpu and world == 1:
        steps_of = dict(zip(ids.tolist(), gpu_steps.tolist()))
        cpu = cpu_reference_rate(w, ids, lambda b: steps_of[int(b)], args.cpu_seconds,
                                 os.cpu_count() or 1)
    exact = w.exact_dudn_outward()[ids] if w.exact_grad is not None else None
    rng_name = "philox4x32-10" if cfg.rng == bw.wos.RNG_PHILOX4X32 else "philox4x64-10"
    out = {
        "metric": METRIC, "value": value, "unit": "walk-steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config, seeded generators; no dataset)",
        "config": {"workload": w.name, "n_bp": w.n_bp, "nodes_per_bp": w.n_nodes,
                   "walks_per_node": w.n_paths, "eps_shell": w.eps, "seed": w.seed,
                   "rng": rng_name, "a": w.a, "patch_panels": dcfg.m,
                   "parallelism": f"bp-sharded x{world}",
                   "l2": "compute-bound; per-step node/patch arrays (>2 GB) exceed L2"},
        "stream_mode": ("statistical: Philox4x32-10 keyed by (seed, point, path), one 32-bit word "
                        "per uniform (two walk steps per block), table sincos (<= 2e-13), "
                        "Newton-step roots (<= 3e-12), fp64 throughout; gated by z-score / "
                        "two-sample tests against the reference's estimate_u_batch; the reference's "
                        "own stream with correctly rounded arithmetic is timed in parity_mode"
                        if cfg.rng == bw.wos.RNG_PHILOX4X32 else
                        "parity: the reference's Philox4x64-10 RngStream, walk for walk"),
        "neumann_points_per_s": w.n_bp / (ms_max * 1e-3),
        "walk_steps_per_step": total_steps,
        "walks_per_s": w.n_bp * w.n_nodes * w.n_paths / (ms_max * 1e-3),
        "k1_share_of_step": k1_ms / ms,
        "neumann_check": None if exact is None else neumann_check(w, ids, main_dudn, main_err, exact,
                                                                   n_bad, world, n_loc),
        "roofline": {"bound": "fp64", "kernel": f"K1 wos_nodes_kernel ({rng_name})",
                     "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": achieved / peak_tf,
                     "peak_source": "measured on this device by bw_measure_fp64_peak (DFMA loop; "
                                    "MEASURED_PEAKS.json has no fp64 entry)",
                     "flops_per_walk_step": f_step,
                     "flops_per_walk_step_reference": F_STEP_REFERENCE[scene_class(w)],
                     "flops_note": "executed work (the cavity box: faces + the candidates a lane "
                                   "visits); the reference's brute-force count is reported "
                                   "beside it and is not used for frac",
                     "traffic": traffic,
                     "traffic_note": "DRAM read+write bytes of one K1 launch over this rank's "
                                     "nodes, scaled from the ncu child process's per-node bytes; "
                                     "the walk state stays on chip (40 B estimate + 8 B step "
                                     "count per node leave it)"},
        "k1_pipes": pipes,
        "parity_mode": parity,
        "gpu_launches": launches,
        "clocks": clock_summary,
        "cpu_baseline": cpu,
        "e2e": e2e,
    }
    print(json.dumps(out))


def neumann_check(w, ids, d_dudn, d_err, exact, n_bad, world, n_loc):
    """Accuracy of the step's Neumann data against the analytic du/dn, overall
    and per stratum (face interior / edge-shrunk face points / cavity points)."""
    dudn, err = d_dudn.cpu().numpy(), d_err.cpu().numpy()
    z = np.abs(dudn - exact) / np.maximum(err, 1e-300)
    rel = np.abs(dudn - exact) / np.maximum(np.abs(exact), 1e-12)
    cls, radii = w.cls[ids], w.radii[ids]
    from paper_1210_1491_b200.geometry import SceneKind

    if w.scene.kind == SceneKind.Sphere:
        strata = {"sphere": np.ones(len(ids), bool)}
    else:
        strata = {"face": (cls == 0) & (radii == w.a), "edge": (cls == 0) & (radii < w.a),
                  "cavity": cls > 0}
    out = {"max_abs_dev_over_err": float(z.max()), "frac_dev_over_err_gt3": float(np.mean(z > 3)),
           "median_rel_err": float(np.median(rel)), "flagged_points": n_bad,
           "scope": "all points" if world == 1 else f"rank 0's shard ({n_loc} of {w.n_bp} points)",
           "strata": {}}
    for k, m in strata.items():
        if m.any():
            out["strata"][k] = {"n": int(m.sum()), "max_abs_dev_over_err": float(z[m].max()),
                                "frac_dev_over_err_gt3": float(np.mean(z[m] > 3)),
                                "median_rel_err": float(np.median(rel[m]))}
    return out


def k1_probe(args):
    """Child of profile_k1 (run under ncu): one warm-up and one measured K1
    launch over the Gamma nodes of `args.k1_probe` evenly spaced boundary points
    of the workload; prints their walk-step count."""
    import torch

    from paper_1210_1491_b200 import nodes
    from paper_1210_1491_b200 import wos as W
    from paper_1210_1491_b200.workloads import CONFIGS

    w = CONFIGS[args.config]()
    w = w.subset(np.unique(np.linspace(0, w.n_bp - 1, args.k1_probe).astype(np.int64)))
    cfg = w.wos_config(rng=W.RNG_PHILOX4X32 if args.rng == 32 else W.RNG_PHILOX4X64)
    for _ in range(2):
        _, steps = nodes.wos_patch_nodes(w.scene, cfg, w.points, w.axes, w.radii, w.dirs,
                                         cls=w.cls, device=0)
    torch.cuda.synchronize()
    print(json.dumps({"walk_steps": int(steps.sum()), "nodes": int(w.n_bp * w.n_nodes)}))


def profile_k1(args, w, n_probe: int = 1000):
    """ncu --metrics of one K1 launch in a child process (never a timed value):
    fp64 / FMA-heavy pipe and issue utilisation, executed warp-instructions and
    DRAM bytes. None when ncu is unavailable or fails."""
    import shutil
    import tempfile

    ncu = shutil.which("ncu") or ("/usr/local/cuda/bin/ncu" if Path("/usr/local/cuda/bin/ncu").exists()
                                  else None)
    if ncu is None:
        return None
    n_probe = min(n_probe, w.n_bp)
    with tempfile.TemporaryDirectory() as td:
        log = Path(td) / "ncu.csv"
        cmd = [ncu, "--metrics", ",".join(NCU_METRICS + NCU_OPTIONAL), "--clock-control", "none",
               "-k", "regex:wos_nodes", "-s", "1", "-c", "1", "--csv", "--log-file", str(log),
               sys.executable, str(ROOT / "bench.py"), "--config", str(args.config),
               "--rng", str(args.rng), "--k1-probe", str(n_probe)]
        try:
            res = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
            meta = next(json.loads(l) for l in res.stdout.splitlines() if l.startswith("{"))
            import csv

            rows = list(csv.reader(log.read_text().splitlines()))
            hdr = next(i for i, r in enumerate(rows) if "Metric Name" in r)
            h = rows[hdr]
            im, iv, iu = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
            out = dict(meta)
            for r in rows[hdr + 1:]:
                if len(r) > iv and r[im] in NCU_METRICS + NCU_OPTIONAL:
                    try:
                        v = float(r[iv].replace(",", ""))
                    except ValueError:  # an optional metric ncu reports as n/a
                        continue
                    unit = r[iu].lower()
                    scale = {"kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "byte": 1.0}.get(unit, 1.0)
                    out[r[im]] = v * scale if "bytes" in r[im] else v
            return out if all(m in out for m in NCU_METRICS) else None
        except Exception:
            return None


if __name__ == "__main__":
    main()
