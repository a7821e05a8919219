"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/biewos_b200.h declares, and its struct layouts match the
ctypes mirror; host-side setup code agrees with the oracle. No GPU calls."""
from __future__ import annotations

import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
from paper_1210_1491_b200 import _native as N
from paper_1210_1491_b200 import nodes, workloads
from paper_1210_1491_b200.build import LIB, build

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "biewos_b200.h"


def declared_symbols():
    txt = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:bw_status|const char\*|int32_t)\s+(bw_\w+)\s*\(", txt,
                                 re.M)))


def test_library_builds_and_loads():
    build()
    assert LIB.exists()
    lib = N.load_library()
    assert lib.bw_abi_version() == 3


def test_exports_every_declared_symbol():
    build()
    syms = declared_symbols()
    assert len(syms) >= 17
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (bw_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert set(N.EXPORTS) <= exported


def test_sm100a_cubin_embedded():
    build()
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_header():
    src = r"""
    #include <stdio.h>
    #include <stddef.h>
    #include "biewos_b200.h"
    int main(void){
      printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(bw_scene),
             offsetof(bw_scene, cavities), offsetof(bw_scene, phi), sizeof(bw_wos_config),
             offsetof(bw_wos_config, seed), sizeof(bw_estimate), sizeof(bw_dtn_config),
             offsetof(bw_dtn_config, kind), sizeof(bw_patch));
      return 0; }
    """
    tmp = Path("/tmp/bw_layout.c")
    tmp.write_text(src)
    subprocess.run(["gcc", "-I", str(ROOT / "include"), "-o", "/tmp/bw_layout", str(tmp)],
                   check=True)
    got = list(map(int, subprocess.run(["/tmp/bw_layout"], capture_output=True,
                                       text=True).stdout.split()))
    from paper_1210_1491_b200 import dtn

    assert got == [C.sizeof(N.BwScene), N.BwScene.cavities.offset, N.BwScene.phi.offset,
                   C.sizeof(N.BwWosConfig), N.BwWosConfig.seed.offset,
                   N.ESTIMATE_DTYPE.itemsize, C.sizeof(dtn.BwDtnConfig),
                   dtn.BwDtnConfig.kind.offset, dtn.PATCH_DTYPE.itemsize]


def test_no_device_means_loud_failure():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(Exception):
        N.Context(0)


def test_host_gauss_legendre_matches_oracle(orc):
    for n in (1, 2, 7, 8, 16, 30, 64):
        x, w = nodes.gauss_legendre(n)
        xo, wo = np.empty(n), np.empty(n)
        orc.or_gauss_legendre(n, O.p(xo), O.p(wo))
        assert np.array_equal(x, xo) and np.array_equal(w, wo)


def test_gamma_rule_matches_oracle(orc):
    tm = np.arccos(0.1)
    d, w = nodes.gamma_rule(16, 32, tm)
    do, wo = np.empty((512, 3)), np.empty(512)
    orc.or_gamma_rule(16, 32, tm, O.p(do), O.p(wo))
    assert np.allclose(d, do, rtol=0, atol=2e-16) and np.allclose(w, wo, rtol=1e-14)
    # integrates the cap area 2 pi (1 - cos theta_max) exactly-ish
    assert abs(w.sum() - 2 * np.pi * (1 - np.cos(tm))) < 1e-12


def test_fibonacci_and_node_positions(orc):
    pts = nodes.fibonacci_sphere(50)
    po = np.empty((50, 3))
    orc.or_fibonacci_sphere(50, 1.0, O.p(po))
    assert np.allclose(pts, po, atol=1e-15)
    dirs, _ = nodes.gamma_rule(4, 8, 1.3)
    host = nodes.patch_node_positions(pts, -pts, 0.2, None, dirs)
    orc_pos = O.or_patch_nodes(orc, pts, -pts, 0.2, None, dirs)
    assert np.allclose(host, orc_pos, atol=1e-15)
    # nodes sit on the hemisphere sphere and inside the unit ball
    assert np.allclose(np.linalg.norm(host - pts[:, None], axis=2), 0.2)
    assert (np.linalg.norm(host, axis=2) < 1).all()


def test_host_philox_matches_oracle(orc):
    d = workloads.stream_doubles(7, 3, 5, 2, 40)
    do = np.empty(40)
    orc.or_rng_doubles(7, 3, 5, 2, 40, O.p(do))
    assert np.array_equal(d, do)


def test_workloads_shapes():
    w = workloads.config1()
    assert (w.n_bp, w.n_nodes, w.n_paths, w.eps, w.seed) == (1000, 512, 10000, 1e-4, 1)
    w = workloads.config2()
    assert (w.n_bp, w.n_nodes, w.n_paths) == (6144, 128, 4096)
    w = workloads.config3()
    cav = w.extra["cavities"]
    assert w.n_bp == 20000 and len(cav) == 64
    d = np.linalg.norm(cav[:, None, :3] - cav[None, :, :3], axis=2)
    rr = cav[:, None, 3] + cav[None, :, 3]
    assert (d + np.eye(64) * 10 > rr + 0.04).all()
    assert ((cav[:, 3] >= 0.05) & (cav[:, 3] <= 0.1)).all()
    w = workloads.config4(1000)
    assert w.n_nodes == 128 and w.a == 0.05


def test_cpp_host_mirror_compiles_and_links():
    from paper_1210_1491_b200.build import CPP_TEST_BIN, build_cpp_tests

    build_cpp_tests()
    assert CPP_TEST_BIN.exists()
    out = subprocess.run(["ldd", str(CPP_TEST_BIN)], capture_output=True, text=True).stdout
    assert "libbiewos_b200.so" in out and "not found" not in out.split("libbiewos_b200.so")[1].split("\n")[0]


def test_library_loaded_before_torch_keeps_torch_importable():
    """NCCL is resolved at run time (bw_group.cu nccl_api), not linked: loading
    the library first must not bind the soname libnccl.so.2 to another NCCL
    than torch's (torch then fails on a missing symbol)."""
    import subprocess
    import sys

    code = ("import paper_1210_1491_b200._native as N; N.load_library(); import torch; "
            "print('ok')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       cwd=str(ROOT))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
