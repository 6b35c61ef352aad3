# Round evidence: full default bench line, ncu launch list, ncu --set full of the bench kernel.
TAG=${1:-r1}
python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/${TAG}_bench.log > gpurun_out/${TAG}_bench_line.json
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --e2e-msgs 65536"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
echo launches rc=$?
$CMD > gpurun_out/${TAG}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tma_fixed -s 3 -c 1 \
    -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo full rc=$?
