# A/B of library builds on the headline bench: bash scripts/ab_bench.sh REPS lib1 lib2 ...
REPS=$1; shift
for rep in $(seq 1 $REPS); do for lib in "$@"; do
  LH_LIBRARY=$lib python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 --e2e-msgs 65536 > gpurun_out/ab_bench.log 2>&1
  echo "$rep $lib $(python -c "import json; j=json.loads(open('gpurun_out/ab_bench.log').read().strip().splitlines()[-1]); print(j['value'], j['ms_per_step'], j['step_ms'], j['clocks']['reasons'])")"
done; done
