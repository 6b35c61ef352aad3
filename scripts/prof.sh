# usage: bash scripts/prof.sh TAG [extra bench args]
# quick bench (no CPU baseline) then one ncu --set full capture of the bench kernel.
TAG=$1; shift
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --e2e-msgs 65536 $*"
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 3 $* > gpurun_out/bench_$TAG.log 2>&1
echo bench rc=$?; tail -c 1500 gpurun_out/bench_$TAG.log
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tma_fixed -s 3 -c 1 \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo ncu rc=$?
