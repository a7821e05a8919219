"""Generate tests/golden/ref_vectors.npz from the REFERENCE ITSELF.

Runs the reference's own, unmodified sources (compiled into
oracle/_ref/libbiewos_ref.so by `make -C oracle ref` from /root/reference) and
records their outputs on seeded inputs. The fixtures travel with the repo so
the parity tests can check the oracle and the B200 kernels where
/root/reference does not exist (the GPU box).

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import ctypes as C
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parents[1]))

import oracle_lib as O  # noqa: E402
from paper_1210_1491_b200.geometry import DomainSide, PointSource, Quadratic, Scene  # noqa: E402
from paper_1210_1491_b200.wos import WosConfig  # noqa: E402


def sphere_panels(R: float, q: float, n_panels: int) -> np.ndarray:
    """tests/test_field_eval.cpp:15-32 lat-long exterior point-charge data."""
    nlat = max(4, int(np.sqrt(n_panels / 2.0)))
    nlon = 2 * nlat
    out = []
    for i in range(nlat):
        th0, th1 = np.pi * i / nlat, np.pi * (i + 1) / nlat
        thc = 0.5 * (th0 + th1)
        area = (np.cos(th0) - np.cos(th1)) * 2.0 * np.pi / nlon * R * R
        for j in range(nlon):
            ph = 2.0 * np.pi * (j + 0.5) / nlon
            n = np.array([np.sin(thc) * np.cos(ph), np.sin(thc) * np.sin(ph), np.cos(thc)])
            out.append([*(R * n), *n, area, q / (4 * np.pi * R), -q / (4 * np.pi * R * R)])
    return np.array(out)


def main():
    if not O.ref_available():
        raise SystemExit("oracle/_ref not buildable (needs /root/reference)")
    ref = O.ref()
    rng = np.random.default_rng(20121004)
    g = {}

    # walks: interior unit ball, u = z (tests/test_wos.cpp:84-91 data), eps 1e-4
    ball = Scene.sphere(1.0, DomainSide.Interior, Quadratic(g=(0.0, 0.0, 1.0))).to_c()
    cfg = WosConfig(eps_shell=1e-4, seed=1).to_c()
    starts = rng.uniform(-0.5, 0.5, (256, 3))
    pids = np.arange(256, dtype=np.uint64) * 7 + 3
    paths = np.arange(256, dtype=np.uint64) % 17
    st, ex, f, s = O.ref_walk(ref, ball, cfg, starts, pids, paths)
    assert st == 0
    g.update(ball_starts=starts, ball_pids=pids, ball_paths=paths, ball_exit=ex, ball_feat=f,
             ball_steps=s)

    # walks: half-space Test-1 data (tests/test_wos.cpp:14-17), default config
    hs = Scene.half_space(0.0, PointSource(q=1.0, s=(0.0, 0.0, -1.0))).to_c()
    cfg_hs = WosConfig(seed=0).to_c()
    hs_starts = np.tile([[0.0, 0.0, 1.0]], (128, 1))
    hs_pids = np.full(128, 3, np.uint64)
    hs_paths = np.arange(128, dtype=np.uint64)
    st, ex, f, s = O.ref_walk(ref, hs, cfg_hs, hs_starts, hs_pids, hs_paths)
    assert st == 0
    g.update(hs_starts=hs_starts, hs_pids=hs_pids, hs_paths=hs_paths, hs_exit=ex, hs_feat=f,
             hs_steps=s)

    # estimates: interior unit ball, u = x^2 - y^2 + z (BASELINE cfg1 data)
    quad = Scene.sphere(1.0, DomainSide.Interior,
                        Quadratic(g=(0.0, 0.0, 1.0), q=(1.0, -1.0, 0.0, 0.0, 0.0, 0.0))).to_c()
    cfg_q = WosConfig(eps_shell=1e-4, n_paths=5000, seed=1).to_c()
    epts = rng.uniform(-0.45, 0.45, (8, 3))
    st, est = O.ref_estimate(ref, quad, cfg_q, epts, base=11, workers=4)
    assert st == 0
    g.update(est_points=epts, est_mean=est["mean"], est_var=est["variance"], est_n=est["n"])

    # potential sum (tests/test_field_eval.cpp:15-32 data) at far targets
    panels = sphere_panels(3.0, 1.0, 500)
    targets = np.array([[4.0, 0, 0], [0, -4.0, 0], [0, 0, 4.5], [0.2, 0.1, -0.3], [3.5, -1, 0.5]])
    u = np.empty(len(targets))
    near = np.zeros(len(targets), np.uint8)
    ref.ref_evaluate(O.p(panels), len(panels), O.p(targets), len(targets), O.p(u), O.p(near))
    g.update(pot_panels=panels, pot_targets=targets, pot_u=u)

    # Gauss-Legendre rules (quadrature.cpp:7-35)
    for n in (8, 16, 30):
        x, w = np.empty(n), np.empty(n)
        ref.ref_gauss_legendre(n, O.p(x), O.p(w))
        g[f"gl{n}_x"], g[f"gl{n}_w"] = x, w

    # RngStream doubles (rng.hpp:44-60)
    d = np.empty(64)
    ref.ref_rng_doubles(C.c_uint64(1), C.c_uint64(0), C.c_uint64(0), C.c_uint64(0), 64, O.p(d))
    g["rng_1_0_0"] = d

    np.savez_compressed(HERE / "ref_vectors.npz", **g)
    print("wrote", HERE / "ref_vectors.npz", sorted(g))


if __name__ == "__main__":
    main()
