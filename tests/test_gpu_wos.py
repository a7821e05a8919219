"""GPU parity of K1 (WOS) against the oracle and the reference's golden walks.

Every call goes through the C-ABI (libbiewos_b200.so). The oracle is only the
checker here."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
import paper_1210_1491_b200 as bw
from paper_1210_1491_b200 import nodes
from paper_1210_1491_b200.geometry import DomainSide, ExpSinSin, PointSource, Quadratic, Scene
from paper_1210_1491_b200.wos import WosConfig

pytestmark = pytest.mark.gpu
GOLD = np.load(Path(__file__).parent / "golden" / "ref_vectors.npz")
SQ2PI = np.sqrt(2.0) * np.pi


def test_philox_kats_on_device(gpu):
    import ctypes as C

    from test_oracle import KATS

    ctr = np.array([k[0] for k in KATS], np.uint64)
    key = np.array([k[1] for k in KATS], np.uint64)
    out = np.zeros((len(KATS), 4), np.uint64)
    gpu.check(gpu.lib.bw_philox_blocks(gpu.handle, ctr.ctypes.data, key.ctypes.data, len(KATS),
                                       out.ctypes.data))
    for row, k in zip(out, KATS):
        assert [int(v) for v in row] == k[2]


@pytest.mark.parametrize("seed,point,path", [(1, 0, 0), (4, 12799999, 4095), (2**63 + 5, 2**40 + 3, 9999)])
def test_factored_wos_stream_equals_philox(gpu, seed, point, path):
    """K1's factored stream (block table for rounds 0-1, per-walk round-1
    product, per-node round-2 table, direct rounds past block 63) equals the
    plain Philox4x64-10 block (rng.hpp:25-38) on ctr {blk, path, point, 0},
    key {seed, 0x1BD11BDAA9FC1A22}, for blocks 0..199."""
    n = 200
    got = np.zeros((n, 4), np.uint64)
    gpu.check(gpu.lib.bw_diag_wos_stream(gpu.handle, seed, point, path, n, got.ctypes.data))
    ctr = np.zeros((n, 4), np.uint64)
    ctr[:, 0] = np.arange(n, dtype=np.uint64)
    ctr[:, 1] = path
    ctr[:, 2] = point
    key = np.tile(np.array([seed, 0x1BD11BDAA9FC1A22], np.uint64), (n, 1))
    ref = np.zeros((n, 4), np.uint64)
    gpu.check(gpu.lib.bw_philox_blocks(gpu.handle, ctr.ctypes.data, key.ctypes.data, n,
                                       ref.ctypes.data))
    assert np.array_equal(got, ref)


def _agree(ex, f, s, ex_ref, f_ref, s_ref, frac=0.9999, dfrac=1e-3):
    same = (f == f_ref) & (s == s_ref)
    assert same.mean() >= frac, f"{(~same).sum()} of {len(same)} walks differ"
    # ulp-level differences (sincospi vs cos(2 pi u), FMA) can grow along a
    # trajectory; the exit point must still agree to 1e-9 on all but 0.1%
    d = np.abs(ex[same] - ex_ref[same]).max(axis=1)
    assert (d > 1e-9).mean() <= dfrac and d.max(initial=0.0) < 1e-6


def test_walks_match_reference_golden_ball(gpu):
    scene = Scene.sphere(1.0, DomainSide.Interior, Quadratic(g=(0.0, 0.0, 1.0)))
    ex, f, s = bw.walk_batch(scene, GOLD["ball_starts"], WosConfig(eps_shell=1e-4, seed=1),
                             GOLD["ball_pids"], GOLD["ball_paths"])
    _agree(ex, f, s, GOLD["ball_exit"], GOLD["ball_feat"], GOLD["ball_steps"], frac=1.0)


def test_walks_match_reference_golden_halfspace(gpu):
    scene = Scene.half_space(0.0, PointSource(q=1.0, s=(0.0, 0.0, -1.0)))
    ex, f, s = bw.walk_batch(scene, GOLD["hs_starts"], WosConfig(seed=0), GOLD["hs_pids"],
                             GOLD["hs_paths"])
    _agree(ex, f, s, GOLD["hs_exit"], GOLD["hs_feat"], GOLD["hs_steps"], frac=1.0)


def _cavity_scene(n=64, seed=3):
    from paper_1210_1491_b200.workloads import make_cavities

    cav = make_cavities(n, seed, clearance=0.04)
    return cav, Scene.box_with_cavities((-1, -1, -1), (1, 1, 1), cav,
                                        PointSource(q=1.0, s=tuple(cav[0, :3])))


def _lattice_scene(n_side):
    g = np.linspace(-0.75, 0.75, n_side)
    c = np.array([(x, y, z) for x in g for y in g for z in g])
    cav = np.concatenate([c, np.full((len(c), 1), 0.03)], axis=1)
    return Scene.box_with_cavities((-1, -1, -1), (1, 1, 1), cav,
                                   PointSource(q=1.0, s=tuple(cav[0, :3])))


@pytest.mark.parametrize("kind", ["ball", "cube", "cavities", "lattice343"])
def test_walks_match_oracle(gpu, orc, kind):
    rng = np.random.default_rng(11)
    if kind == "ball":
        scene = Scene.sphere(1.0, DomainSide.Interior,
                             Quadratic(g=(0, 0, 1.0), q=(1.0, -1.0, 0, 0, 0, 0)))
        starts = rng.uniform(-0.55, 0.55, (4000, 3))
    elif kind == "cube":
        scene = Scene.box((0, 0, 0), (1, 1, 1), ExpSinSin(1.0, (SQ2PI, np.pi, np.pi)))
        starts = rng.uniform(0.01, 0.99, (4000, 3))
    else:
        scene = _lattice_scene(7) if kind == "lattice343" else _cavity_scene()[1]
        sc = scene.to_c()
        starts = []
        while len(starts) < 4000:
            p = rng.uniform(-0.99, 0.99, 3)
            if orc.or_in_domain(__import__("ctypes").byref(sc), O.p(p)):
                starts.append(p)
        starts = np.array(starts)
    cfg = WosConfig(eps_shell=1e-5, seed=5)
    pids = np.arange(len(starts), dtype=np.uint64) + 1000
    paths = np.arange(len(starts), dtype=np.uint64) % 97
    ex, f, s = bw.walk_batch(scene, starts, cfg, pids, paths)
    st, ex_o, f_o, s_o = O.or_walk(orc, scene.to_c(), cfg.to_c(), starts, pids, paths)
    assert st == 0
    # 343 cavities: more curved reflections along a walk amplify ulp-level
    # differences of the exit point (steps and features still identical)
    _agree(ex, f, s, ex_o, f_o, s_o, dfrac=3e-3 if kind == "lattice343" else 1e-3)


def test_estimates_match_oracle_same_streams(gpu, orc):
    """Same seed -> the GPU runs the oracle's walks; means differ only by rounding."""
    scene = Scene.sphere(1.0, DomainSide.Interior,
                         Quadratic(g=(0, 0, 1.0), q=(1.0, -1.0, 0, 0, 0, 0)))
    cfg = WosConfig(eps_shell=1e-4, n_paths=2000, seed=1)
    pts = np.random.default_rng(3).uniform(-0.5, 0.5, (64, 3))
    est, steps = bw.estimate_u_batch_full(scene, pts, cfg, point_id_base=17)
    st, ref, steps_o = O.or_estimate(orc, scene.to_c(), cfg.to_c(), pts, base=17)
    assert st == 0
    assert (est["n"] == ref["n"]).all() and (est["n_failed"] == 0).all()
    close = np.abs(est["mean"] - ref["mean"]) <= 1e-10 * np.maximum(1, np.abs(ref["mean"]))
    assert close.mean() >= 0.97
    assert np.allclose(est["variance"], ref["variance"], rtol=1e-6)
    assert (np.abs(steps - steps_o) <= 2).mean() >= 0.97


def test_estimates_zscores_vs_analytic_and_independent_oracle(gpu, orc):
    """Independent seeds: z-score distribution gate (SURVEY.md 8(d) parity (ii))."""
    q = Quadratic(g=(0, 0, 1.0), q=(1.0, -1.0, 0, 0, 0, 0))
    scene = Scene.sphere(1.0, DomainSide.Interior, q)
    pts = np.random.default_rng(4).uniform(-0.5, 0.5, (400, 3))
    est = bw.estimate_u_batch(scene, pts, WosConfig(eps_shell=1e-5, n_paths=4096, seed=2))
    st, ref, _ = O.or_estimate(orc, scene.to_c(), WosConfig(eps_shell=1e-5, n_paths=4096,
                                                            seed=3).to_c(), pts)
    se_g = bw.wos.std_error(est)
    se_o = bw.wos.std_error(ref)
    for z in ((est["mean"] - q(pts)) / se_g,
              (est["mean"] - ref["mean"]) / np.sqrt(se_g ** 2 + se_o ** 2)):
        n = len(z)
        assert (np.abs(z) > 3).mean() <= 0.0027 + 3.1 * np.sqrt(0.0027 / n)
        assert abs(z.mean()) < 4 / np.sqrt(n)
        assert 0.75 < z.var() < 1.3


def test_constant_data_exact(gpu):  # test_wos.cpp:74-82
    e = bw.estimate_u(Scene.sphere(2.0, DomainSide.Interior, 1.0), [0.3, 0, 0.4],
                      WosConfig(n_paths=500))
    assert e.mean == 1.0 and e.variance == 0.0 and e.n == 500


def test_unit_ball_phi_z(gpu):  # test_wos.cpp:84-91
    e = bw.estimate_u(Scene.sphere(1.0, DomainSide.Interior, Quadratic(g=(0, 0, 1.0))),
                      [0, 0, 0.5], WosConfig(n_paths=20000))
    assert abs(e.mean - 0.5) < 4 * e.std_error()


def test_halfspace_half_and_leakage(gpu):  # test_wos.cpp:65-72, 93-99
    s = Scene.half_space(0.0, PointSource(q=1.0, s=(0, 0, -1.0)))
    e = bw.estimate_u(s, [0, 0, 1.0], WosConfig(n_paths=100000))
    assert abs(e.mean - 0.5) < 4 * e.std_error()
    assert e.n_infinity <= 10


def test_exit_uniform_from_center_ks(gpu):  # test_wos.cpp:50-63
    s = Scene.sphere(1.0, DomainSide.Interior, 1.0)
    n = 100000
    ex, f, _ = bw.walk_batch(s, np.zeros((n, 3)), WosConfig(), 0, np.arange(n))
    assert (f == 0).all()
    z = np.sort(ex[:, 2])
    cdf = (z + 1) / 2
    d = max(np.abs(cdf - np.arange(n) / n).max(), np.abs(cdf - np.arange(1, n + 1) / n).max())
    assert d < 1.628 / np.sqrt(n)


def test_mean_value_property_random_balls(gpu):  # test_wos.cpp:135-154
    rng = np.random.default_rng(7)
    for trial in range(20):
        R = 0.5 + 1.5 * rng.random()
        c0, c1, c2 = 2 * rng.random(3) - 1
        q = Quadratic(c=c0, g=(0, 0, c1), q=(c2, -c2, 0, 0, 0, 0))
        p = (rng.random(3) - 0.5) * R
        e = bw.estimate_u(Scene.sphere(R, DomainSide.Interior, q), p,
                          WosConfig(n_paths=4000, seed=trial))
        assert abs(e.mean - q(p)) < 4 * e.std_error() + 1e-12


def test_bookkeeping_empty_and_stream_separation(gpu):  # test_wos.cpp:101-116
    s = Scene.half_space(0.0, PointSource(q=1.0, s=(0, 0, -1.0)))
    cfg = WosConfig(n_paths=1000)
    assert len(bw.estimate_u_batch(s, np.zeros((0, 3)), cfg)) == 0
    est = bw.estimate_u_batch(s, np.tile([0.2, 0.1, 0.5], (3, 1)), cfg)
    assert est["mean"][0] != est["mean"][1]
    se = np.hypot(*bw.wos.std_error(est)[:2])
    assert abs(est["mean"][0] - est["mean"][1]) < 4 * se
    assert (est["n"] + est["n_failed"] == 1000).all()


def test_bit_identical_under_reordering(gpu):
    """Per-point results depend only on (seed, point id, start): any batch
    composition / launch shape gives the same bits (wos.hpp:43-44)."""
    s = Scene.half_space(0.0, PointSource(q=1.0, s=(0, 0, -1.0)))
    pts = np.array([[0.1 * i, -0.05 * i, 0.3 + 0.1 * i] for i in range(7)])
    cfg = WosConfig(n_paths=9000, seed=99)
    full = bw.estimate_u_batch(s, pts, cfg)
    for i in (0, 3, 6):
        one = bw.estimate_u_batch(s, pts[i:i + 1], cfg, point_id_base=i)
        assert one.tobytes() == full[i:i + 1].tobytes()
    again = bw.estimate_u_batch(s, pts, cfg)
    assert again.tobytes() == full.tobytes()


def test_reliability_gate(gpu):  # test_wos.cpp:184-190
    s = Scene.half_space(0.0, PointSource(q=1.0, s=(0, 0, -1.0)))
    with pytest.raises(bw.ReliabilityError):
        bw.estimate_u(s, [0, 0, 50], WosConfig(max_steps=1, n_paths=1000))


def test_applicability_without_closed_form(gpu):
    s = Scene.sphere(1.0, DomainSide.Interior, lambda y: y[2])
    with pytest.raises(bw.ApplicabilityError):
        bw.estimate_u(s, [0, 0, 0], WosConfig(n_paths=10))


def test_immediate_exit_and_determinism(gpu):  # test_wos.cpp:35-48
    s = Scene.half_space(0.0, PointSource(q=1.0, s=(0, 0, -1.0)))
    r = bw.walk(s, [0.3, -0.2, 5e-6], WosConfig(), 0, 0)
    assert r.steps == 0 and r.feature == 0 and r.point[2] == 0.0
    a = bw.walk(s, [0, 0, 1], WosConfig(), 3, 7)
    b = bw.walk(s, [0, 0, 1], WosConfig(), 3, 7)
    assert a.steps == b.steps and (a.point == b.point).all()


def test_patch_nodes_positions_and_estimates_match_oracle(gpu, orc):
    """K1 in patch mode generates node positions bit-identical to the oracle's
    and estimates them with the same streams."""
    R, a = 1.0, 0.2
    bp = nodes.fibonacci_sphere(12, R)
    axes = -bp
    dirs, _ = nodes.gamma_rule(4, 8, np.arccos(a / (2 * R)))
    scene = Scene.sphere(R, DomainSide.Interior,
                         Quadratic(g=(0, 0, 1.0), q=(1.0, -1.0, 0, 0, 0, 0)))
    cfg = WosConfig(eps_shell=1e-4, n_paths=512, seed=1)
    est, steps = nodes.wos_patch_nodes(scene, cfg, bp, axes, a, dirs, point_id_base=5)
    pos = O.or_patch_nodes(orc, bp, axes, a, None, dirs)
    st, ref, steps_o = O.or_estimate(orc, scene.to_c(), cfg.to_c(), pos.reshape(-1, 3), base=5)
    assert st == 0
    e = est.reshape(-1)
    close = np.abs(e["mean"] - ref["mean"]) <= 1e-10
    assert close.mean() >= 0.97
    assert (e["n"] == 512).all()


def test_patch_nodes_outside_domain_are_skipped(gpu):
    scene = Scene.box((0, 0, 0), (1, 1, 1), ExpSinSin(1.0, (SQ2PI, np.pi, np.pi)))
    dirs, _ = nodes.gamma_rule(4, 8, np.pi / 2)
    # a corner-adjacent face point: part of its hemisphere pokes out of the cube
    est, _ = nodes.wos_patch_nodes(scene, WosConfig(n_paths=64), [[0.5 / 32, 0.5 / 32, 0.0]],
                                   [[0, 0, 1.0]], 0.05, dirs)
    e = est.reshape(-1)
    assert (e["n"] == 0).any() and (e["n"] == 64).any()
    assert np.isnan(e["mean"][e["n"] == 0]).all()


@pytest.mark.parametrize("n_side", [4, 7])
def test_cavity_lattice_estimates_match_oracle(gpu, orc, n_side):
    """K1 with the cavity candidate grid: 64 cavities (packed lists with 8-bit
    lower bounds, early exit) and 343 cavities (> 256: unpacked lists) give the
    oracle's brute-force walks: same step counts and means on shared streams."""
    scene = _lattice_scene(n_side)
    rng = np.random.default_rng(5)
    sc = scene.to_c()
    pts = []
    while len(pts) < 48:
        p = rng.uniform(-0.95, 0.95, 3)
        if orc.or_in_domain(__import__("ctypes").byref(sc), O.p(p)):
            pts.append(p)
    pts = np.array(pts)
    cfg = WosConfig(eps_shell=1e-5, n_paths=512, seed=9)
    est, steps = bw.estimate_u_batch_full(scene, pts, cfg, point_id_base=3)
    st, ref, steps_o = O.or_estimate(orc, sc, cfg.to_c(), pts, base=3)
    assert st == 0
    assert (est["n"] == ref["n"]).all()
    assert (np.abs(steps - steps_o) <= 2).mean() >= 0.95
    # one walk that ends differently (ulp-level jumps near the eps shell) moves a
    # 512-walk mean far beyond 1e-9: most points agree to 1e-9, all within 5 SE
    close = np.abs(est["mean"] - ref["mean"]) <= 1e-9 * np.maximum(1, np.abs(ref["mean"]))
    assert close.mean() >= 0.85
    se = np.sqrt(ref["variance"] / ref["n"])
    assert (np.abs(est["mean"] - ref["mean"]) <= 5 * se + 1e-12).all()


def test_loop_sqrt_is_correctly_rounded(gpu):
    """The walk loop's branch-free sqrt (sqrt_fast) equals __dsqrt_rn bitwise
    over the range the walks feed it (1 - z^2, |p|^2, cavity d^2)."""
    import ctypes as C

    rng = np.random.default_rng(11)
    a = np.concatenate([
        rng.random(1 << 20),                                   # 1 - z^2 in [0, 1)
        np.ldexp(rng.random(1 << 20) + 0.5, rng.integers(-900, 900, 1 << 20)),
        1.0 - np.ldexp(np.arange(1, 4097, dtype=np.float64), -53),  # near 1
        np.ldexp(np.arange(1, 4097, dtype=np.float64), -60),        # tiny
        (np.arange(1, 1 << 16, dtype=np.float64) ** 2),        # exact squares
    ])
    fast, rn = np.empty_like(a), np.empty_like(a)
    gpu.check(gpu.lib.bw_diag_sqrt(gpu.handle, a.ctypes.data, len(a), fast.ctypes.data,
                                   rn.ctypes.data))
    assert np.array_equal(rn, np.sqrt(a))
    assert np.array_equal(fast.view(np.uint64), rn.view(np.uint64))
    z = np.zeros(1)
    f0, r0 = np.empty(1), np.empty(1)
    gpu.check(gpu.lib.bw_diag_sqrt(gpu.handle, z.ctypes.data, 1, f0.ctypes.data, r0.ctypes.data))
    assert r0[0] == 0.0 and 0.0 < f0[0] < 1e-150


@pytest.mark.parametrize("n_paths", [1, 31, 32, 33, 63, 65, 1000, 10000])
def test_walk_counts_around_the_warp_width(gpu, orc, n_paths):
    """Walk counts below, at and just past multiples of the warp width (the refill
    bookkeeping and the per-walk Philox product ring), and config 1's 10,000:
    every walk is run once, on the oracle's streams, with the same step total."""
    scene = Scene.sphere(1.0, DomainSide.Interior,
                         Quadratic(g=(0, 0, 1.0), q=(1.0, -1.0, 0, 0, 0, 0)))
    cfg = WosConfig(eps_shell=1e-4, n_paths=n_paths, seed=5)
    pts = np.random.default_rng(n_paths).uniform(-0.5, 0.5, (8, 3))
    est, steps = bw.estimate_u_batch_full(scene, pts, cfg, point_id_base=3)
    st, ref, steps_o = O.or_estimate(orc, scene.to_c(), cfg.to_c(), pts, base=3)
    assert st == 0
    assert (est["n"] == n_paths).all() and (ref["n"] == n_paths).all()
    assert (np.abs(steps - steps_o) <= 2).all()
    tol = 1e-10 * np.maximum(1, np.abs(ref["mean"]))
    assert (np.abs(est["mean"] - ref["mean"]) <= tol).mean() >= 0.87


def test_empty_inputs_every_batch_entry(gpu):
    """n = 0 is a no-op on every batch entry point (no launch, no error)."""
    from paper_1210_1491_b200 import field_eval, linalg

    s = Scene.sphere(1.0, DomainSide.Interior, Quadratic(g=(0, 0, 1.0)))
    z3 = np.zeros((0, 3))
    cfg = WosConfig(n_paths=64)
    est, steps = bw.estimate_u_batch_full(s, z3, cfg)
    assert len(est) == 0 and len(steps) == 0
    ex, f, st = bw.walk_batch(s, z3, cfg, np.zeros(0, np.uint64), np.zeros(0, np.uint64))
    assert len(ex) == len(f) == len(st) == 0
    assert len(bw.wos.nearest_feature_batch(s, z3)[0]) == 0
    u, near = field_eval.evaluate_batch(np.zeros((0, 9)), [[0, 0, 2.0]])
    assert u[0] == 0.0
    u, near = field_eval.evaluate_batch(np.zeros((3, 9)), z3)
    assert len(u) == 0
    X, res, info = linalg.lu_solve_batched(np.zeros((0, 4, 4)), np.zeros((0, 4)))
    assert len(X) == 0
    e, s_ = nodes.wos_patch_nodes(s, cfg, z3, z3, np.zeros(0), np.array([[0, 0, 1.0]]))
    assert e.size == 0
