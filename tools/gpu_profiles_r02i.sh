#!/bin/bash
# Round-2 final evidence (records through shared memory): bench lines of every config, the reference
# arm, the c2 launch list and one `ncu --set full` capture of each config's
# dominant kernel (every command runs once without ncu before its ncu run).
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash tools/gpu_profiles_r02i.sh'
# Outputs land in gpurun_out/ (r02i_*); tools/ncu_summary.py writes profiles/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "from paper_1509_05186_b200 import build; build.build()"
timeout 1300 python -m pytest tests -m gpu -x -q > gpurun_out/r02i_pytest_gpu.log 2>&1; echo "pytest: $?"; tail -n 2 gpurun_out/r02i_pytest_gpu.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02i_smoke.log 2>&1; echo "smoke: $?"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02i_smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02i_bench_c2.json 2> gpurun_out/r02i_bench_c2.err; echo "bench c2 (default): $?"
for c in c1 c3 c4 c5 u1m; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r02i_bench_$c.json 2> gpurun_out/r02i_bench_$c.err
  echo "bench $c: $?"
done
# the c2 launch list (the same step bench.py times)
python tools/prof_step.py --config c2 --steps 5 > gpurun_out/r02i_plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scan|narrow|finalize|gather|probe|ivf|fill|cb_chunks" -c 400 --csv \
    --log-file gpurun_out/r02i_launches_c2.csv python tools/prof_step.py --config c2 --steps 5 > gpurun_out/r02i_ncu_l_c2.log 2>&1
echo "launch list c2: $?"
for c in c2 u1m; do
  q=""
  if [ "$c" = "u1m" ]; then q="--Q 2048"; fi
  python tools/prof_step.py --config $c --steps 2 $q > gpurun_out/r02i_plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
  ncu --set full --clock-control none --import-source on -k regex:"scan_kernel|narrow_kernel" -s 1 -c 1 \
      -o gpurun_out/r02i_prof_$c python tools/prof_step.py --config $c --steps 2 $q > gpurun_out/r02i_ncu_$c.log 2>&1
  echo "ncu $c: $?"
done
