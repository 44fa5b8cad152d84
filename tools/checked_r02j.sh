#!/bin/bash
# Bounds-checked runs (compute-sanitizer is closed on this pool): the library
# built with -DET_CHECKS (device-side traps on out-of-range shared-memory table
# offsets, record indices, candidate-buffer appends, table-build stores and
# finalize candidate reads), run on every kernel shape (tools/sanitize_cases.py,
# each result also checked against the oracle) and on the -m gpu parity suite.
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash tools/checked_r02.sh'
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "from paper_1509_05186_b200 import build; build.build(); build.build(out_dir='paper_1509_05186_b200/_build/checked', defines=['ET_CHECKS'])"
export ET_LIB_PATH=$PWD/paper_1509_05186_b200/_build/checked/libetree.so
timeout 1200 python tools/sanitize_cases.py > gpurun_out/r02j_checked_cases.log 2>&1; echo "checked cases: $?"
tail -3 gpurun_out/r02j_checked_cases.log
timeout 1800 python -m pytest tests -m gpu -q --ignore=tests/test_gpu_fullsize.py > gpurun_out/r02j_checked_pytest.log 2>&1; echo "checked pytest: $?"
tail -3 gpurun_out/r02j_checked_pytest.log
