#!/bin/bash
# host-buffer top-k (et_etree_topk_host): GPU tests + c2 bench lines with the pipelined e2e per batch count
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
#timeout 900 python -m pytest tests/test_gpu_host.py -x -q > gpurun_out/host_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/host_pytest.log
for nb in 0 2 8; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-flat --host-batches $nb > gpurun_out/host_bench_c2_nb$nb.json 2> gpurun_out/host_bench_c2_nb$nb.err; echo "bench nb=$nb rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/host_bench_c2_nb$nb.json').read().strip().splitlines()[-1]); print("nb=$nb", d["ms_per_step"], d["e2e"]["ms_per_step"], d["e2e"]["serial_ms_per_step"])" || tail -20 gpurun_out/host_bench_c2_nb$nb.err
done
