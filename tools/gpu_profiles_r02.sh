#!/bin/bash
# Round-2 profile captures (run under gpurun on one B200; every command runs
# once without ncu before its ncu run).  Outputs land in gpurun_out/ and are
# summarised into profiles/ by tools/ncu_summary.py on the host.
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash tools/gpu_profiles_r02.sh'
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "from paper_1509_05186_b200 import build; build.build()"
# the c2 launch list (the same command bench.py times, a few steps)
python tools/prof_step.py --config c2 --steps 5 > gpurun_out/r02_plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scan|finalize|gather|probe|ivf|fill" -c 400 --csv \
    --log-file gpurun_out/r02_launches_c2.csv python tools/prof_step.py --config c2 --steps 5 > gpurun_out/r02_ncu_l_c2.log 2>&1
echo "launch list c2: $?"
for c in c2 c1 c3 c4 c5 u1m; do
  q=""
  if [ "$c" = "u1m" ]; then q="--Q 2048"; fi
  python tools/prof_step.py --config $c --steps 2 $q > gpurun_out/r02_plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
  ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 1 -c 1 \
      -o gpurun_out/r02_prof_$c python tools/prof_step.py --config $c --steps 2 $q > gpurun_out/r02_ncu_$c.log 2>&1
  echo "ncu $c: $?"
done
ncu --set full --clock-control none --import-source on -k regex:finalize -s 1 -c 1 \
    -o gpurun_out/r02_prof_c2_finalize python tools/prof_step.py --config c2 --steps 2 > gpurun_out/r02_ncu_c2fin.log 2>&1
echo "ncu c2 finalize: $?"
