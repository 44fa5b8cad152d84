#!/bin/bash
# tcgen05.cp TMEM levels: full -m gpu suite, smoke, bench lines of every config, c2 phases
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/cp_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/cp_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/cp_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/cp_smoke.log
timeout 900 python bench.py > gpurun_out/cp_bench_c2.json 2> gpurun_out/cp_bench_c2.err; echo "bench c2 rc=$?"
for c in c1 c3 c4 c5 u1m; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/cp_bench_$c.json 2> gpurun_out/cp_bench_$c.err; echo "bench $c rc=$?"
done
python tools/summarize_bench.py gpurun_out/cp_bench_*.json
timeout 600 python tools/phase_timing.py --config c2 > gpurun_out/cp_phases_c2.txt 2>&1; echo "phases c2: $?"; cat gpurun_out/cp_phases_c2.txt | head -12
