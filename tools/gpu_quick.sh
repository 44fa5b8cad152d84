# quick GPU loop: parity tests (optionally a subset) + one bench line per config
#   bash tools/gpu_quick.sh "<pytest -k expr or empty>" "c2 u1m ..."
set -u
K="${1:-}"; CFGS="${2:-c2}"
mkdir -p gpurun_out
if [ -n "$K" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_gpu.log 2>&1; else timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; fi
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for c in $CFGS; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "bench $c rc=$?"; python -c "
import json,sys
d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1])
print('$c', 'ms/step %.4f'%d['ms_per_step'], 'value %.3e'%d['value'], 'frac %.3f'%d['roofline']['frac'], d['kernels_ms'])" 2>/dev/null || tail -5 gpurun_out/bench_$c.err
done
