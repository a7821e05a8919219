"""Pin the CPU oracle (oracle/biewos_oracle.c) before trusting it:
  * Philox KATs and stream tests of the reference (tests/test_rng.cpp:11-65),
  * walk-by-walk and estimate bit-identity with the reference's own sources
    (golden fixtures from oracle/_ref, tests/golden/make_golden.py),
  * the reference's WOS property tests (tests/test_wos.cpp) run on the oracle,
  * the new geometry (box, cavities) against brute-force definitions.
CPU only."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
from paper_1210_1491_b200.geometry import DomainSide, PointSource, Quadratic, Scene
from paper_1210_1491_b200.wos import WosConfig

GOLD = np.load(Path(__file__).parent / "golden" / "ref_vectors.npz")


def blk(lib, ctr, key):
    c = np.array(ctr, np.uint64)
    k = np.array(key, np.uint64)
    out = np.zeros(4, np.uint64)
    lib.or_philox_block(O.p(c), O.p(k), O.p(out))
    return [int(v) for v in out]


# tests/test_rng.cpp:11-34
KATS = [
    ([1, 0, 0, 0], [0, 0],
     [0x02F4BA6408E4D89B, 0x3DD62B0B9CA8C5B2, 0x1C8667A55D902E79, 0x907D7A052FD5B4DC]),
    ([2, 2, 3, 4], [0xDEADBEEF, 0xFACEB00C],
     [0x96D961AF5AD9FA36, 0xE83EE691304F0212, 0x9C4EEEAC1DBDA566, 0xE8977773828BC1B4]),
    ([0, 0, 0, 0], [2**64 - 1, 2**64 - 1],
     [0x44B7493D1ACFC229, 0x6636AF8E997921DD, 0x3F73E132B5B3780E, 0x605644DDE03B01B1]),
]


@pytest.mark.parametrize("ctr,key,expect", KATS)
def test_philox_known_answers(orc, ctr, key, expect):
    assert blk(orc, ctr, key) == expect


# Random123's published Philox4x32-10 known-answer vectors (kat_vectors:
# zero, all-ones and the pi-digits counter/key) pin the BW_RNG_PHILOX4X32 block
KATS32 = [
    ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
    ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
    ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
     [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
]


def p32(lib, ctr, key, fn="or_philox4x32_blocks", handle=None):
    c = np.array(ctr, np.uint32)
    k = np.array(key, np.uint32)
    o = np.zeros(4, np.uint32)
    if handle is None:
        getattr(lib, fn)(O.p(c), O.p(k), 1, O.p(o))
    else:
        getattr(lib, fn)(handle, c.ctypes.data, k.ctypes.data, 1, o.ctypes.data)
    return [int(v) for v in o]


@pytest.mark.parametrize("ctr,key,expect", KATS32)
def test_philox4x32_known_answers(orc, ctr, key, expect):
    assert p32(orc, ctr, key) == expect


def test_rng32_stream_layout(orc):
    """The PHILOX4X32 WOS stream: block b = Philox4x32-10 on ctr {b, path,
    lo(point), hi(point)}, key {lo(seed), hi(seed) ^ 0x1BD11BDA}; words
    (o0 << 32 | o1), (o2 << 32 | o3); distinct per point and path."""
    seed, point, path = 0x123456789ABCDEF0, 2**33 + 7, 5
    w = np.zeros(6, np.uint64)
    orc.or_rng32_u64s(seed, point, path, 6, O.p(w))
    for b in range(3):
        o = p32(orc, [b, path, point & 0xFFFFFFFF, point >> 32],
                [seed & 0xFFFFFFFF, (seed >> 32) ^ 0x1BD11BDA])
        assert int(w[2 * b]) == (o[0] << 32) | o[1] and int(w[2 * b + 1]) == (o[2] << 32) | o[3]
    w2 = np.zeros(6, np.uint64)
    orc.or_rng32_u64s(seed, point, path + 1, 6, O.p(w2))
    w3 = np.zeros(6, np.uint64)
    orc.or_rng32_u64s(seed, point + 1, path, 6, O.p(w3))
    assert (w != w2).all() and (w != w3).all()
    # the uniforms: one 32-bit word each, in the order o0..o3, centred on the
    # 2^-32 grid, so a block feeds two walk steps (z, azimuth, z, azimuth)
    u = np.zeros(12)
    orc.or_rng32_doubles(seed, point, path, 12, O.p(u))
    for b in range(3):
        o = p32(orc, [b, path, point & 0xFFFFFFFF, point >> 32],
                [seed & 0xFFFFFFFF, (seed >> 32) ^ 0x1BD11BDA])
        assert [float(v) for v in u[4 * b:4 * b + 4]] == [(x + 0.5) / 2.0**32 for x in o]
    assert (u > 0).all() and (u < 1).all()


def test_streams_deterministic_and_distinct(orc):  # test_rng.cpp:36-48
    def u64s(seed, pt, path):
        out = np.zeros(64, np.uint64)
        orc.or_rng_u64s(seed, pt, path, 0, 64, O.p(out))
        return out

    a, b, c, d = u64s(42, 7, 3), u64s(42, 7, 3), u64s(42, 7, 4), u64s(42, 8, 3)
    assert (a == b).all() and (a != c).any() and (a != d).any()


def test_uniform_doubles_chi2(orc):  # test_rng.cpp:50-65
    n = 100000
    u = np.empty(n)
    orc.or_rng_doubles(123, 0, 0, 0, n, O.p(u))
    assert (u >= 0).all() and (u < 1).all()
    assert abs(u.mean() - 0.5) < 4.0 * np.sqrt(1.0 / 12.0 / n)
    bins = np.bincount((u * 16).astype(int), minlength=16)
    chi2 = (((bins - n / 16) ** 2) / (n / 16)).sum()
    assert chi2 < 37.7


def test_rng_stream_matches_reference_golden(orc):
    d = np.empty(64)
    orc.or_rng_doubles(1, 0, 0, 0, 64, O.p(d))
    assert (d == GOLD["rng_1_0_0"]).all()
    # the first two draws quoted in SURVEY.md Appendix C
    assert d[0] == 0.30388614459531782 and d[1] == 0.63197269695242031


def test_oracle_walks_bit_identical_to_reference_ball(orc):
    ball = Scene.sphere(1.0, DomainSide.Interior, Quadratic(g=(0.0, 0.0, 1.0))).to_c()
    cfg = WosConfig(eps_shell=1e-4, seed=1).to_c()
    st, ex, f, s = O.or_walk(orc, ball, cfg, GOLD["ball_starts"], GOLD["ball_pids"],
                             GOLD["ball_paths"])
    assert st == 0
    assert (s == GOLD["ball_steps"]).all()
    assert (f == GOLD["ball_feat"]).all()
    assert (ex == GOLD["ball_exit"]).all()


def test_oracle_walks_bit_identical_to_reference_halfspace(orc):
    hs = Scene.half_space(0.0, PointSource(q=1.0, s=(0.0, 0.0, -1.0))).to_c()
    st, ex, f, s = O.or_walk(orc, hs, WosConfig(seed=0).to_c(), GOLD["hs_starts"],
                             GOLD["hs_pids"], GOLD["hs_paths"])
    assert st == 0
    assert (s == GOLD["hs_steps"]).all() and (f == GOLD["hs_feat"]).all()
    assert (ex == GOLD["hs_exit"]).all()


def test_oracle_estimates_bit_identical_to_reference(orc):
    quad = Scene.sphere(1.0, DomainSide.Interior,
                        Quadratic(g=(0.0, 0.0, 1.0), q=(1.0, -1.0, 0, 0, 0, 0))).to_c()
    cfg = WosConfig(eps_shell=1e-4, n_paths=5000, seed=1).to_c()
    for workers in (1, 3):
        st, est, steps = O.or_estimate(orc, quad, cfg, GOLD["est_points"], base=11,
                                       workers=workers)
        assert st == 0
        assert (est["mean"] == GOLD["est_mean"]).all()
        assert (est["variance"] == GOLD["est_var"]).all()
        assert (est["n"] == GOLD["est_n"]).all()
        assert (steps > 0).all()


def test_oracle_live_against_reference(orc, reflib):
    """Same as the golden checks, on fresh seeds, when oracle/_ref is built."""
    rng = np.random.default_rng(5)
    ball = Scene.sphere(1.3, DomainSide.Interior,
                        Quadratic(c=0.2, g=(0.1, 0.0, 1.0), q=(1.0, -1.0, 0, 0.3, 0, 0))).to_c()
    cfg = WosConfig(eps_shell=1e-5, seed=77).to_c()
    starts = rng.uniform(-0.7, 0.7, (500, 3))
    a = O.or_walk(orc, ball, cfg, starts, np.arange(500), np.arange(500) * 3)
    b = O.ref_walk(reflib, ball, cfg, starts, np.arange(500), np.arange(500) * 3)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    cfg2 = WosConfig(eps_shell=1e-4, n_paths=9000, seed=99).to_c()
    pts = rng.uniform(-0.5, 0.5, (5, 3))
    st1, e1, _ = O.or_estimate(orc, ball, cfg2, pts, workers=4)
    st2, e2 = O.ref_estimate(reflib, ball, cfg2, pts, workers=2)
    assert st1 == st2 == 0
    assert (e1 == e2).all()


# ---- the reference's WOS property tests (tests/test_wos.cpp) on the oracle ----

def test_constant_data_exact(orc):  # test_wos.cpp:74-82
    s = Scene.sphere(2.0, DomainSide.Interior, 1.0).to_c()
    st, e, _ = O.or_estimate(orc, s, WosConfig(n_paths=500).to_c(), [[0.3, 0, 0.4]])
    assert st == 0 and e["mean"][0] == 1.0 and e["variance"][0] == 0.0 and e["n"][0] == 500


def test_unit_ball_phi_z(orc):  # test_wos.cpp:84-91
    s = Scene.sphere(1.0, DomainSide.Interior, Quadratic(g=(0, 0, 1.0))).to_c()
    st, e, _ = O.or_estimate(orc, s, WosConfig(n_paths=20000).to_c(), [[0, 0, 0.5]])
    se = np.sqrt(e["variance"][0] / e["n"][0])
    assert abs(e["mean"][0] - 0.5) < 4 * se


def test_halfspace_test1(orc):  # test_wos.cpp:93-99 (+ leakage :65-72)
    hs = Scene.half_space(0.0, PointSource(q=1.0, s=(0, 0, -1.0))).to_c()
    st, e, _ = O.or_estimate(orc, hs, WosConfig(n_paths=20000).to_c(), [[0, 0, 1.0]])
    se = np.sqrt(e["variance"][0] / e["n"][0])
    assert abs(e["mean"][0] - 0.5) < 4 * se
    assert e["n_infinity"][0] <= 10


def test_reliability_gate(orc):  # test_wos.cpp:184-190
    hs = Scene.half_space(0.0, PointSource(q=1.0, s=(0, 0, -1.0))).to_c()
    st, e, _ = O.or_estimate(orc, hs, WosConfig(max_steps=1, n_paths=1000).to_c(), [[0, 0, 50]])
    assert st == 5  # BW_ERR_RELIABILITY
    assert e["n"][0] + e["n_failed"][0] == 1000


def test_immediate_exit(orc):  # test_wos.cpp:35-48
    hs = Scene.half_space(0.0, PointSource(q=1.0, s=(0, 0, -1.0))).to_c()
    st, ex, f, s = O.or_walk(orc, hs, WosConfig().to_c(), [[0.3, -0.2, 5e-6]], 0, 0)
    assert s[0] == 0 and f[0] == 0 and ex[0, 2] == 0.0


# ---- new geometry (BOX, BOX_CAVITIES) ----

def _cavity_scene():
    cav = np.array([[0.3, 0.2, -0.1, 0.1], [-0.4, 0.0, 0.2, 0.08], [0.0, -0.5, 0.5, 0.05]])
    return cav, Scene.box_with_cavities((-1, -1, -1), (1, 1, 1), cav, PointSource(s=(0.3, 0.2, -0.1)))


def test_box_cavity_distance_is_bruteforce_min(orc):
    cav, sc = _cavity_scene()
    s = sc.to_c()
    rng = np.random.default_rng(1)
    for _ in range(300):
        p = rng.uniform(-1, 1, 3)
        feat = C.c_int(0)
        d = orc.or_nearest_feature(C.byref(s), O.p(p), C.byref(feat))
        cands = [abs(p[0] + 1), abs(1 - p[0]), abs(p[1] + 1), abs(1 - p[1]), abs(p[2] + 1),
                 abs(1 - p[2])] + [abs(np.sqrt(((p - c[:3]) ** 2).sum()) - c[3]) for c in cav]
        assert d == min(cands)
        assert feat.value == int(np.argmin(cands))


def test_box_maximal_ball_is_empty(orc):  # test_geometry.cpp:95-128 style
    cav, sc = _cavity_scene()
    s = sc.to_c()
    rng = np.random.default_rng(2)
    for _ in range(100):
        p = rng.uniform(-1, 1, 3)
        if not orc.or_in_domain(C.byref(s), O.p(p)):
            continue
        d = orc.or_nearest_feature(C.byref(s), O.p(p), None)
        # random boundary samples never closer than d
        dirs = rng.normal(size=(200, 3))
        dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
        for c in cav:
            y = c[:3] + c[3] * dirs
            assert (np.linalg.norm(y - p, axis=1) >= d * (1 - 1e-12)).all()
        face = rng.uniform(-1, 1, (200, 3))
        face[:, 0] = 1.0
        assert (np.linalg.norm(face - p, axis=1) >= d * (1 - 1e-12)).all()


def test_box_walk_exits_on_boundary(orc):
    cav, sc = _cavity_scene()
    s = sc.to_c()
    cfg = WosConfig(eps_shell=1e-5, seed=3).to_c()
    st, ex, f, steps = O.or_walk(orc, s, cfg, np.tile([[0.0, 0.0, 0.0]], (200, 1)), 1,
                                 np.arange(200))
    assert st == 0
    assert ((f >= 0) & (f < 9)).all()
    for x, k in zip(ex, f):
        if k < 6:
            assert x[k // 2] == (1.0 if k & 1 else -1.0)
        else:
            c = cav[k - 6]
            assert abs(np.linalg.norm(x - c[:3]) - c[3]) < 1e-12


# ---- quadrature, nodes, potential, LU ----

@pytest.mark.parametrize("n", [8, 16, 30])
def test_gauss_legendre_matches_reference(orc, n):
    x, w = np.empty(n), np.empty(n)
    assert orc.or_gauss_legendre(n, O.p(x), O.p(w)) == 0
    assert (x == GOLD[f"gl{n}_x"]).all() and (w == GOLD[f"gl{n}_w"]).all()
    # exact for degree 2n-1 (test_quadrature.cpp:11-44)
    assert abs((w * x ** (2 * n - 2)).sum() - 2.0 / (2 * n - 1)) < 1e-13


def test_potential_matches_reference(orc):
    u, near = O.or_potential(orc, GOLD["pot_panels"], GOLD["pot_targets"])
    assert (u == GOLD["pot_u"]).all() and not near.any()
    uld, _ = O.or_potential(orc, GOLD["pot_panels"], GOLD["pot_targets"], long_double=True)
    assert np.allclose(uld, u, rtol=1e-12, atol=1e-15)
    # point-charge value 1/(16 pi) within 1% (test_field_eval.cpp:45-52)
    assert abs(u[0] - 1 / (16 * np.pi)) < 0.01 / (16 * np.pi)


def test_lu_oracle(orc):
    rng = np.random.default_rng(0)
    m, n = 20, 5
    A = rng.normal(size=(n, m, m)) + 4 * np.eye(m)
    B = rng.normal(size=(n, 2, m))
    X = np.empty_like(B)
    res = np.empty(n)
    info = np.empty(n, np.int32)
    assert orc.or_lu_solve_batched(m, n, O.p(A), O.p(B), 2, O.p(X), O.p(res), O.p(info)) == 0
    for s in range(n):
        assert np.allclose(X[s], np.linalg.solve(A[s], B[s].T).T, rtol=1e-12)
    assert (res < 1e-13).all()


def test_oracle_plates_sine_live_against_reference(orc, reflib):
    """four_plates_sine data (runner.cpp:318-324, bw_phi_kind SIN_SIN): the
    oracle's walks and estimates equal the reference's own code bit for bit."""
    from paper_1210_1491_b200.geometry import SinSin

    plates = [[0, 1, 0, 1], [-1, 0, 0, 1], [-1, 0, -1, 0], [0, 1, -1, 0]]
    sc = Scene.plate_set(plates, SinSin(1.0, (1.0, 2.0))).to_c()
    cfg = WosConfig(eps_shell=1e-5, trunc_radius=1e5, seed=6).to_c()
    rng = np.random.default_rng(8)
    starts = np.concatenate([rng.uniform(-0.9, 0.9, (200, 2)), rng.uniform(0.01, 0.3, (200, 1))], 1)
    a = O.or_walk(orc, sc, cfg, starts, np.arange(200), np.arange(200) * 5)
    b = O.ref_walk(reflib, sc, cfg, starts, np.arange(200), np.arange(200) * 5)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    cfg2 = WosConfig(eps_shell=1e-5, trunc_radius=1e5, n_paths=500, seed=6).to_c()
    st1, e1, _ = O.or_estimate(orc, sc, cfg2, starts[:4], workers=4)
    st2, e2 = O.ref_estimate(reflib, sc, cfg2, starts[:4], workers=2)
    assert st1 == st2 == 0
    assert (e1 == e2).all()
    y = np.array([0.3, -0.7, 0.0])
    assert O.or_eval_phi(orc, sc, y, 0) == np.sin(0.3) * np.sin(-1.4)
