# benchmark experiment builds side by side: bash tools/gpu_variants.sh "var1 var3" "c2 u1m"
VARS="$1"; CFGS="$2"
mkdir -p gpurun_out
for v in default $VARS; do
  if [ "$v" = default ]; then unset ET_LIB_PATH; else export ET_LIB_PATH=$PWD/paper_1509_05186_b200/_build/$v/libetree.so; fi
  for c in $CFGS; do
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/var_${v}_$c.json 2> gpurun_out/var_${v}_$c.err
    python -c "
import json
d=json.loads(open('gpurun_out/var_${v}_$c.json').read().strip().splitlines()[-1])
print('$v $c', 'ms/step %.4f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], d['kernels_ms'])" 2>/dev/null || { echo "$v $c FAILED"; tail -3 gpurun_out/var_${v}_$c.err; }
  done
done
