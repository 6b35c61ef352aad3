# Steady-state A/B: 150 steps per library, report first-20 and last-75 medians.
REPS=$1; shift
for rep in $(seq 1 $REPS); do for lib in "$@"; do
  LH_LIBRARY=$lib python bench.py --steps 150 --warmup 5 --no-cpu-baseline --e2e-steps 1 --e2e-msgs 65536 --dump-steps > gpurun_out/ab_steady.log 2>&1
  echo "$rep $lib $(python -c "
import json, numpy as np
j=json.loads(open('gpurun_out/ab_steady.log').read().strip().splitlines()[-1]); s=j['steps_ms']
print('first20', round(float(np.median(s[:20])),3), 'last75', round(float(np.median(s[-75:])),3), j['clocks'])")"
  sleep 5
done; done
