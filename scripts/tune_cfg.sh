# Parity first (unless SKIP_TESTS), then the bench under each TMA tile shape, REPS rounds alternating.
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_gpu.log
fi
for rep in $(seq 1 ${REPS:-1}); do
for cfg in ${CFGS:-512x3}; do for pf in ${PFS:-0}; do
  LH_TMA_CFG=$cfg LH_TMA_PF=$pf python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 --e2e-msgs 65536 > gpurun_out/bench_${cfg}_$pf.log 2>&1
  echo "$rep $cfg pf=$pf rc=$? $(python -c "import json,sys; j=json.loads(open('gpurun_out/bench_${cfg}_$pf.log').read().strip().splitlines()[-1]); print(j['value'], j['ms_per_step'], j['step_ms'], j['clocks']['reasons'])")"
done; done; done
