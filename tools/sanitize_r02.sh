#!/bin/bash
# compute-sanitizer runs of every hot-path shape (tools/sanitize_cases.py) on
# one B200; logs to gpurun_out/, copied to profiles/ by hand.
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash tools/sanitize_r02.sh'
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "from paper_1509_05186_b200 import build; build.build()"
python tools/sanitize_cases.py > gpurun_out/r02_san_plain.log 2>&1; echo "plain: $?"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_cases.py > gpurun_out/r02_sanitizer_$tool.log 2>&1
  echo "$tool: $?"
  tail -3 gpurun_out/r02_sanitizer_$tool.log
done
