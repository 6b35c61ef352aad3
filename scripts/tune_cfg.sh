# Parity first, then the bench under each TMA tile shape / L2 prefetch distance.
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
for cfg in ${CFGS:-256x3 128x4 512x3}; do for pf in ${PFS:-0 2 4 8}; do
  LH_TMA_CFG=$cfg LH_TMA_PF=$pf python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 --e2e-msgs 65536 > gpurun_out/bench_${cfg}_$pf.log 2>&1
  echo "$cfg pf=$pf rc=$? $(python -c "import json,sys; j=json.loads(open('gpurun_out/bench_${cfg}_$pf.log').read().strip().splitlines()[-1]); print(j['value'], j['ms_per_step'], j['roofline']['frac'], j['clocks']['sm_mhz'], j['clocks']['reasons'])")"
done; done
