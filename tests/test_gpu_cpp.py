"""GPU: the reference's WOS/potential test cases, restated in C++ against the
C++ host mirror (paper_1210_1491_b200/cpp/biewos_b200.hpp) and the C-ABI."""
import subprocess

import pytest

from paper_1210_1491_b200.build import CPP_TEST_BIN, CPP_TEST_SRC

pytestmark = pytest.mark.gpu


def test_cpp_reference_cases(gpu):
    from paper_1210_1491_b200.build import PKG

    hdr = PKG / "cpp" / "biewos_b200.hpp"
    newest = max(CPP_TEST_SRC.stat().st_mtime, hdr.stat().st_mtime)
    if not CPP_TEST_BIN.exists() or CPP_TEST_BIN.stat().st_mtime < newest:
        from paper_1210_1491_b200.build import build_cpp_tests

        build_cpp_tests()
    res = subprocess.run([str(CPP_TEST_BIN)], capture_output=True, text=True, timeout=600)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "0 failed" in res.stdout
