set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?"
cat gpurun_out/bench_c2.json
for c in c1 c3 c4 u1m; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; cat gpurun_out/bench_$c.json; done
timeout 300 python tools/prof_step.py --config c2 --steps 5 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c2.csv python tools/prof_step.py --config c2 --steps 5 > gpurun_out/ncu_l.log 2>&1; echo "ncu list rc=$?"
timeout 300 python tools/prof_step.py --config c2 --steps 5 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 2 -c 2 -o gpurun_out/prof_scan_c2 python tools/prof_step.py --config c2 --steps 5 > gpurun_out/ncu_f.log 2>&1; echo "ncu full rc=$?"
