"""In-tree build of the native library (sm_100a) and of the test oracle.

`python -m paper_1210_1491_b200.build` compiles
  paper_1210_1491_b200/_lib/libbiewos_b200.so   (product: CUDA kernels + C-ABI)
The oracle (oracle/_build, oracle/_ref) is test infrastructure and is built by
__graft_entry__.build() through oracle/Makefile, never by the product.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB = LIB_DIR / "libbiewos_b200.so"
SOURCES = ["bw_capi.cu", "bw_wos.cu", "bw_potential.cu", "bw_lu.cu", "bw_diag.cu", "bw_patch.cu",
           "bw_point.cu", "bw_lp.cu", "bw_dtn_class.cu",
           "bw_patch_large.cu", "bw_group.cu"]
HEADERS = ["bw_device.cuh", "bw_internal.h", "bw_patch_common.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the B200 library cannot be built")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [PKG.parent / "include" / "biewos_b200.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every source to an object (in parallel; an object is reused
    while it is newer than its source and all headers) and link the library."""
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    LIB_DIR.mkdir(parents=True, exist_ok=True)
    obj_dir = LIB_DIR / "obj"
    obj_dir.mkdir(exist_ok=True)
    extra = os.environ.get("BW_NVCC_FLAGS", "").split()
    tag = obj_dir / "flags.txt"
    if extra != (tag.read_text().split() if tag.exists() else []):
        force = True
    hdr_t = max(d.stat().st_mtime for d in
                [CSRC / h for h in HEADERS] + [PKG.parent / "include" / "biewos_b200.h"])
    base = [nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
            *extra]

    def compile_one(src: str):
        obj = obj_dir / (src + ".o")
        if (not force and obj.exists() and obj.stat().st_mtime > hdr_t
                and obj.stat().st_mtime > (CSRC / src).stat().st_mtime):
            return src, 0, ""
        res = subprocess.run(base + ["-c", str(CSRC / src), "-o", str(obj)],
                             capture_output=True, text=True)
        return src, res.returncode, res.stdout + res.stderr

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    bad = [r for r in results if r[1] != 0]
    if bad:
        raise RuntimeError("nvcc failed:\n" + "\n".join(r[2] for r in bad))
    tag.write_text(" ".join(extra))
    if verbose:
        sys.stderr.write("".join(r[2] for r in results))
    tmp = LIB.with_suffix(".so.tmp")
    res = subprocess.run([nvcc(), *ARCH, "-shared", "-o", str(tmp)] +
                         [str(obj_dir / (s + ".o")) for s in SOURCES] + ["-ldl"],
                         capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("link failed:\n" + res.stdout + res.stderr)
    os.replace(tmp, LIB)
    return LIB


CPP_TEST_SRC = PKG.parent / "tests" / "cpp" / "test_reference_cases.cpp"
CPP_TEST_BIN = PKG.parent / "tests" / "cpp" / "_build" / "test_reference_cases"


def build_cpp_tests() -> Path:
    """The C++ host mirror's test program (links the library; runs on a GPU)."""
    build()
    CPP_TEST_BIN.parent.mkdir(parents=True, exist_ok=True)
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", str(PKG.parent / "include"), str(CPP_TEST_SRC),
           "-L", str(LIB_DIR), "-lbiewos_b200", "-Wl,-rpath," + str(LIB_DIR),
           "-Wl,-rpath,$ORIGIN/../../../paper_1210_1491_b200/_lib", "-o", str(CPP_TEST_BIN)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("g++ failed:\n" + res.stdout + res.stderr)
    return CPP_TEST_BIN


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
