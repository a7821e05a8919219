"""K1 with the Philox4x32-10 stream (bw_wos_config.rng = BW_RNG_PHILOX4X32).

The stream is not the reference's RngStream, so parity is statistical against
the reference itself (oracle/_ref: its own estimate_u_batch on Philox4x64) and
walk-by-walk against the oracle's restatement of the same Philox4x32 stream.
Random123's known-answer vectors pin the block function on the device."""
from __future__ import annotations

import numpy as np
import pytest

import oracle_lib as O
import paper_1210_1491_b200 as bw
from paper_1210_1491_b200 import nodes, workloads
from paper_1210_1491_b200.geometry import DomainSide, ExpSinSin, Quadratic, Scene
from paper_1210_1491_b200.wos import RNG_PHILOX4X32, WosConfig
from test_gpu_strata import two_sample_gates
from test_gpu_wos import SQ2PI, _agree, _cavity_scene
from test_oracle import KATS32, p32

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ctr,key,expect", KATS32)
def test_philox4x32_kats_on_device(gpu, ctr, key, expect):
    assert p32(gpu.lib, ctr, key, "bw_philox4x32_blocks", gpu.handle) == expect


@pytest.mark.parametrize("seed,point,path", [(1, 0, 0), (4, 12799999, 4095),
                                             (2**63 + 5, 2**40 + 3, 9999)])
def test_factored_stream32_equals_oracle(gpu, orc, seed, point, path):
    """K1's factored Philox4x32 stream (per-node uint4 table for blocks < 64,
    per-walk round-1 product, the out-of-line entry past 63) equals the plain
    block function the oracle restates, for blocks 0..299."""
    n = 300
    got = np.zeros(2 * n, np.uint64)
    gpu.check(gpu.lib.bw_diag_wos_stream32(gpu.handle, seed, point, path, n, got.ctypes.data))
    ref = np.zeros(2 * n, np.uint64)
    orc.or_rng32_u64s(seed, point, path, 2 * n, O.p(ref))
    assert np.array_equal(got, ref)


def test_statistical_mode_math_accuracy(gpu):
    """The statistical mode's own arithmetic, as K1 evaluates it: the root
    (hardware estimate, ~2^-20, + one Newton step) to <= 3e-12 relative over
    the magnitudes a walk produces, and the table sincos of the azimuth
    2 pi (u + 1/2) 2^-32 to <= 2e-13 absolute with a unit norm to 4e-13 —
    more than six decades below the eps shell the walk resolves."""
    rng = np.random.default_rng(3)
    n = 400000
    a = np.concatenate([rng.uniform(2.0 ** -31, 1.0, n // 2),
                        10.0 ** rng.uniform(-12, 4, n - n // 2)])
    u = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    u[:8] = [0, 1, 2 ** 23 - 1, 2 ** 23, 2 ** 31 - 1, 2 ** 31, 2 ** 32 - 2, 2 ** 32 - 1]
    root, sn, cs = np.empty(n), np.empty(n), np.empty(n)
    gpu.check(gpu.lib.bw_diag_stat_math(gpu.handle, a.ctypes.data, u.ctypes.data, n,
                                        root.ctypes.data, sn.ctypes.data, cs.ctypes.data))
    assert (np.abs(root / np.sqrt(a) - 1.0)).max() <= 3e-12
    az = 2.0 * np.pi * ((u.astype(np.float64) + 0.5) / 2.0 ** 32)
    assert np.abs(sn - np.sin(az)).max() <= 2e-13
    assert np.abs(cs - np.cos(az)).max() <= 2e-13
    assert np.abs(sn * sn + cs * cs - 1.0).max() <= 4e-13


@pytest.mark.parametrize("kind", ["ball", "cube", "cavities"])
def test_walks32_match_oracle(gpu, orc, kind):
    rng = np.random.default_rng(12)
    if kind == "ball":
        scene = Scene.sphere(1.0, DomainSide.Interior,
                             Quadratic(g=(0, 0, 1.0), q=(1.0, -1.0, 0, 0, 0, 0)))
        starts = rng.uniform(-0.55, 0.55, (4000, 3))
    elif kind == "cube":
        scene = Scene.box((0, 0, 0), (1, 1, 1), ExpSinSin(1.0, (SQ2PI, np.pi, np.pi)))
        starts = rng.uniform(0.01, 0.99, (4000, 3))
    else:
        scene = _cavity_scene()[1]
        sc = scene.to_c()
        starts = []
        while len(starts) < 4000:
            p = rng.uniform(-0.99, 0.99, 3)
            if orc.or_in_domain(__import__("ctypes").byref(sc), O.p(p)):
                starts.append(p)
        starts = np.array(starts)
    cfg = WosConfig(eps_shell=1e-5, seed=5, rng=RNG_PHILOX4X32)
    pids = np.arange(len(starts), dtype=np.uint64) + (1 << 33)
    paths = np.arange(len(starts), dtype=np.uint64) % 97
    ex, f, s = bw.walk_batch(scene, starts, cfg, pids, paths)
    st, ex_o, f_o, s_o = O.or_walk(orc, scene.to_c(), cfg.to_c(), starts, pids, paths)
    assert st == 0
    # the statistical mode's roots and sincos carry ~1e-13 (see
    # test_statistical_mode_math_accuracy) against the oracle's libm, and a
    # trajectory amplifies a perturbation by its curved reflections: the same
    # steps and feature on >= 99.9 % of the walks, exit points to 1e-6 on 99 %
    same = (f == f_o) & (s == s_o)
    assert same.mean() >= 0.999, f"{(~same).sum()} of {len(same)} walks differ"
    d = np.abs(ex[same] - ex_o[same]).max(axis=1)
    assert (d > 1e-6).mean() <= 0.01 and np.median(d) < 1e-11


@pytest.mark.parametrize("n_paths", [1, 33, 65, 4096])
def test_estimates32_match_oracle_same_streams(gpu, orc, n_paths):
    """K1 (persistent warps, refill, tables) on the Philox4x32 stream runs the
    oracle's walks: same walk counts and step totals, means equal to rounding."""
    scene = Scene.sphere(1.0, DomainSide.Interior,
                         Quadratic(g=(0, 0, 1.0), q=(1.0, -1.0, 0, 0, 0, 0)))
    cfg = WosConfig(eps_shell=1e-4, n_paths=n_paths, seed=1, rng=RNG_PHILOX4X32)
    pts = np.random.default_rng(n_paths).uniform(-0.5, 0.5, (32, 3))
    est, steps = bw.estimate_u_batch_full(scene, pts, cfg, point_id_base=17)
    st, ref, steps_o = O.or_estimate(orc, scene.to_c(), cfg.to_c(), pts, base=17)
    assert st == 0
    assert (est["n"] == n_paths).all() and (ref["n"] == n_paths).all()
    assert (np.abs(steps - steps_o) <= 2).mean() >= 0.9
    # K1's statistical mode takes ~1e-13 roots and sincos, so a walk can end one
    # step apart from the oracle's now and then (walk-level agreement:
    # test_walks32_match_oracle); per node, most means agree to ~1e-9 and all
    # within a few SE
    close = np.abs(est["mean"] - ref["mean"]) <= 1e-9 * np.maximum(1, np.abs(ref["mean"]))
    assert close.mean() >= (0.9 if n_paths < 1000 else 0.5)
    se = np.sqrt(ref["variance"] / np.maximum(ref["n"], 1))
    assert (np.abs(est["mean"] - ref["mean"]) <= 5 * se + 1e-9).all()


@pytest.mark.parametrize("rng_kind", [RNG_PHILOX4X32, 0])
@pytest.mark.parametrize("kind", ["cube", "cavities"])
def test_estimates32_match_oracle_same_streams_boxes(gpu, orc, kind, rng_kind):
    """The same on the cube and on the cavity box (K1's LDS candidate loop and
    the statistical mode's own exit classification, classify_exit_fast): the
    oracle's walks on the same Philox4x32 stream, exits classified by the
    reference's rule; node means agree to rounding on most nodes and within a
    small fraction of a standard error on all."""
    rng = np.random.default_rng(21)
    if kind == "cube":
        scene = Scene.box((0, 0, 0), (1, 1, 1), ExpSinSin(1.0, (SQ2PI, np.pi, np.pi)))
        pts = rng.uniform(0.05, 0.95, (48, 3))
    else:
        scene = _cavity_scene()[1]
        sc = scene.to_c()
        pts = []
        while len(pts) < 48:
            q = rng.uniform(-0.95, 0.95, 3)
            if orc.or_in_domain(__import__("ctypes").byref(sc), O.p(q)):
                pts.append(q)
        pts = np.array(pts)
    cfg = WosConfig(eps_shell=1e-5, n_paths=1024, seed=9, rng=rng_kind)
    est, steps = bw.estimate_u_batch_full(scene, pts, cfg, point_id_base=5)
    st, ref, steps_o = O.or_estimate(orc, scene.to_c(), cfg.to_c(), pts, base=5)
    assert st == 0
    assert (est["n"] == 1024).all() and (ref["n"] == 1024).all()
    assert (est["n_failed"] == 0).all()
    assert (np.abs(steps - steps_o) <= 0.002 * steps_o + 4).mean() >= 0.9
    se = np.sqrt(ref["variance"] / ref["n"])
    close = np.abs(est["mean"] - ref["mean"]) <= 1e-9 * np.maximum(1, np.abs(ref["mean"]))
    # the parity mode (the reference's stream, correctly rounded roots, the
    # reference's classification rule) runs the oracle's walks almost surely
    assert close.mean() >= (0.5 if rng_kind == RNG_PHILOX4X32 else 0.9), close.mean()
    assert (np.abs(est["mean"] - ref["mean"]) <= 0.5 * se + 1e-12).all()


def _zgate(z):
    n = len(z)
    assert (np.abs(z) > 3).mean() <= 0.0027 + 3.1 * np.sqrt(0.0027 / n), (np.abs(z) > 3).mean()
    assert abs(z.mean()) < 4 / np.sqrt(n), z.mean()
    assert 0.85 < z.var() < 1.15, z.var()


@pytest.mark.parametrize("cfg_id,n_bp", [(1, 20), (4, 80)])
def test_rng32_zscores_vs_reference_estimate_u_batch(gpu, reflib, cfg_id, n_bp):
    """Philox4x32 node means on >= 1e4 real Gamma nodes of configs 1 and 4
    against the reference's own estimate_u_batch (Philox4x64 streams, i.e.
    independent): SURVEY.md 8(d) gates on the paired z-scores, and the same
    z-distribution against the analytic u as the reference's."""
    w = workloads.CONFIGS[cfg_id]().subset(np.arange(n_bp))
    pos = nodes.patch_node_positions(w.points, w.axes, w.radii, None, w.dirs[0]).reshape(-1, 3)
    assert len(pos) >= 10000
    cfg32 = WosConfig(eps_shell=w.eps, n_paths=w.n_paths, seed=w.seed, rng=RNG_PHILOX4X32)
    est, _ = nodes.wos_patch_nodes(w.scene, cfg32, w.points, w.axes, w.radii, w.dirs[0])
    e = est.reshape(-1)
    cfg_ref = WosConfig(eps_shell=w.eps, n_paths=w.n_paths, seed=w.seed)
    st, ref = O.ref_estimate(reflib, w.scene.to_c(), cfg_ref.to_c(), pos)
    assert st == 0
    se_g, se_r = bw.wos.std_error(e), bw.wos.std_error(ref)
    _zgate((e["mean"] - ref["mean"]) / np.sqrt(se_g ** 2 + se_r ** 2))
    # against the analytic u the node z-scores are skewed for BOTH streams
    # (nodes near the boundary: most walks exit next to the start, a few travel
    # far; see tests/test_gpu_strata.py), so the analytic comparison is the
    # two-sample one: the device's z-distribution equals the reference's
    two_sample_gates(e["mean"], se_g, ref["mean"], se_r, w.exact_u(pos), f"cfg{cfg_id}")


def test_rng32_dtn_matches_rng64_statistically(gpu):
    """The whole DtN step on config 4 points with either stream: Neumann data
    within 4 combined errors of each other and of the analytic du/dn."""
    from paper_1210_1491_b200 import dtn

    w = workloads.config4().subset(np.arange(0, 100000, 500))
    r64 = dtn.dtn_solve_workload(w)
    cfg = WosConfig(eps_shell=w.eps, n_paths=w.n_paths, seed=w.seed, rng=RNG_PHILOX4X32)
    r32 = dtn.dtn_solve(w.scene, cfg, dtn.patches_for(w), w.dirs, w.weights)
    ex = w.exact_dudn_outward()
    z = (r32.dudn - r64.dudn) / np.hypot(r32.err, r64.err)
    assert (np.abs(z) > 4).mean() <= 0.01
    assert (np.abs(r32.dudn - ex) <= 4 * r32.err + 1e-9).mean() >= 0.99
    assert not np.array_equal(r32.dudn, r64.dudn)


@pytest.mark.parametrize("max_steps", [6, 7, 1, 0])
def test_step_budget_in_blocks(gpu, orc, max_steps):
    """The statistical mode checks its step budget once per stream block: an odd
    max_steps acts as the even one below it. K1 and the oracle's restatement
    fail the same walks (reliability error aside: most walks fail here)."""
    scene = Scene.sphere(1.0, DomainSide.Interior,
                         Quadratic(g=(0, 0, 1.0), q=(1.0, -1.0, 0, 0, 0, 0)))
    cfg = WosConfig(eps_shell=1e-6, n_paths=512, seed=3, rng=RNG_PHILOX4X32, max_steps=max_steps)
    pts = np.random.default_rng(8).uniform(-0.5, 0.5, (16, 3))
    try:
        est, steps = bw.estimate_u_batch_full(scene, pts, cfg, point_id_base=2)
    except bw.errors.ReliabilityError as e:  # carries the estimates (wos.py)
        est, steps = e.estimates, e.steps
    st, ref, steps_o = O.or_estimate(orc, scene.to_c(), cfg.to_c(), pts, base=2)
    budget = max_steps & ~1
    assert (steps_o <= 512 * budget).all() and (ref["n_failed"] > 0).all()
    assert np.array_equal(est["n_failed"], ref["n_failed"])
    assert np.array_equal(steps, steps_o)


@pytest.mark.parametrize("kind", ["half_space", "four_plates", "thin_disk", "exterior_sphere"])
def test_estimates32_unbounded_scenes_match_oracle(gpu, orc, kind):
    """The statistical mode on the reference's unbounded scene kinds (their
    truncation-radius test is compiled into those instantiations): same
    streams as the oracle's restatement — equal absorbed / truncated walk
    counts on (almost) every point, step totals to a few per thousand, means
    within a small fraction of a standard error."""
    from paper_1210_1491_b200.geometry import PointSource

    rng = np.random.default_rng(31)
    if kind == "half_space":
        scene = Scene.half_space(0.0, PointSource(q=1.0, s=(0.0, 0.0, -1.0)))
        pts = np.c_[rng.uniform(-1, 1, (24, 2)), rng.uniform(0.05, 2.0, 24)]
    elif kind == "four_plates":
        scene = Scene.four_plates([1, 0, 0, 0])
        pts = np.c_[rng.uniform(-1, 1, (24, 2)), rng.uniform(0.05, 1.0, 24) * rng.choice([-1, 1], 24)]
    elif kind == "thin_disk":
        scene = Scene.thin_disk(1.0, 1.0)
        pts = np.c_[rng.uniform(-1.5, 1.5, (24, 2)), rng.uniform(0.05, 1.0, 24)]
    else:
        scene = Scene.sphere(3.0, DomainSide.Exterior, 0.25)
        d = rng.normal(size=(24, 3))
        pts = d / np.linalg.norm(d, axis=1)[:, None] * rng.uniform(3.2, 6.0, (24, 1))
    cfg = WosConfig(eps_shell=1e-4, n_paths=1024, seed=21, rng=RNG_PHILOX4X32, trunc_radius=50.0)
    est, steps = bw.estimate_u_batch_full(scene, pts, cfg, point_id_base=9)
    st, ref, steps_o = O.or_estimate(orc, scene.to_c(), cfg.to_c(), pts, base=9)
    assert st == 0
    assert (est["n"] == ref["n"]).all() and (est["n_failed"] == ref["n_failed"]).all()
    assert (ref["n_infinity"] > 0).any()
    assert (np.abs(est["n_infinity"] - ref["n_infinity"]) <= 1).all()
    assert (est["n_infinity"] == ref["n_infinity"]).mean() >= 0.9
    assert (np.abs(steps - steps_o) <= 0.005 * steps_o + 8).all()
    se = np.sqrt(ref["variance"] / np.maximum(ref["n"], 1))
    assert (np.abs(est["mean"] - ref["mean"]) <= 0.25 * se + 1e-9).all()
