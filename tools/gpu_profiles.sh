# Round-end evidence: default bench line, reference arm, launch list and one
# ncu --set full capture of the scan kernel per config (each command first
# runs without ncu and must exit 0).  Summaries are written on the box
# (gpurun_out/prof/*.md + traffic.json); only c2's report is kept (<64 MiB pull).
mkdir -p gpurun_out/prof
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench default rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "bench reference rc=$?"
timeout 300 python tools/prof_step.py --config c2 --steps 5 > gpurun_out/plain_c2.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scan|finalize|fill|gather" -c 400 --csv \
    --log-file gpurun_out/prof/launches_c2.csv python tools/prof_step.py --config c2 --steps 5 > gpurun_out/ncu_list_c2.log 2>&1
echo "launch list rc=$?"
for c in ${CFGS:-c2 c3 u1m c4 c5 c1}; do
  timeout 900 python tools/prof_step.py --config $c --steps 2 > gpurun_out/plain_$c.log 2>&1 && \
    timeout 1200 ncu --set full --import-source on --clock-control none -k regex:scan_kernel -s 1 -c 1 \
      -o gpurun_out/prof_full_$c python tools/prof_step.py --config $c --steps 2 > gpurun_out/ncu_full_$c.log 2>&1
  echo "ncu $c rc=$?"
  if [ -f gpurun_out/prof_full_$c.ncu-rep ]; then
    L=""; [ "$c" = c2 ] && L="--launches gpurun_out/prof/launches_c2.csv"
    python tools/ncu_summary.py gpurun_out/prof_full_$c.ncu-rep gpurun_out/prof/r01_${c}_scan.md --traffic-config $c \
      --title "round 1, config $c, scan_kernel (1 launch, --set full)" $L > /dev/null 2>&1
    [ "$c" = c2 ] || rm -f gpurun_out/prof_full_$c.ncu-rep
  fi
done
du -sh gpurun_out
