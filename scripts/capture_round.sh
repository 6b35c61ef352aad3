# Round evidence: full default bench line, reference arm, ncu launch list,
# ncu --set full of the bench kernel, per-class INT rates.
# usage: bash scripts/capture_round.sh TAG
TAG=${1:-r2}
python tools/intpeak.py > gpurun_out/${TAG}_intpeak.txt 2>&1; cp profiles/int_peak.json gpurun_out/${TAG}_int_peak.json
python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
tail -1 gpurun_out/${TAG}_bench.log > gpurun_out/${TAG}_bench_line.json
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_reference.log 2>&1; echo ref rc=$?
tail -1 gpurun_out/${TAG}_reference.log > gpurun_out/${TAG}_reference_line.json
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-sustained --e2e-steps 1 --e2e-msgs 65536"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_tma_fixed -s 3 -c 1 \
    -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo full rc=$?
