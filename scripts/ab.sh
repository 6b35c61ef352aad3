# A/B: alternate library builds in one process-sequence on one box.
# usage: bash scripts/ab.sh "--only cfg5" ab/lib_x.so ab/lib_y.so ...
ARGS=$1; shift
for rep in 1 2; do for lib in "$@"; do
  LH_LIBRARY=$lib python scripts/bench_configs.py $ARGS --steps 20 --warmup 3 > gpurun_out/ab.log 2>&1
  echo "$rep $lib: $(python -c "import json; [print(json.loads(l)['workload'][:14], json.loads(l)['ms'], end=' | ') for l in open('gpurun_out/ab.log') if l.startswith('{')]")"
done; done
