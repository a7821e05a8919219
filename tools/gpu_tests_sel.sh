#!/bin/bash
# selected GPU test files: TESTS="tests/a.py tests/b.py"
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest ${TESTS} -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_sel.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_sel.log
