#!/bin/bash
# Round-2 (last session) validation of HEAD: full -m gpu suite, smoke, default bench line.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02d_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02d_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02d_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02d_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02d_smoke.log
timeout 900 python bench.py > gpurun_out/r02d_bench_c2.json 2> gpurun_out/r02d_bench_c2.err; echo "bench c2 rc=$?"
python tools/summarize_bench.py gpurun_out/r02d_bench_c2.json 2>/dev/null | head -20
