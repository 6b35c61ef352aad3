# ncu evidence for the bench kernel (1 GPU).  Plain run first, then ncu.
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --e2e-msgs 65536"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo launches rc=$?
$CMD > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tma_fixed -s 3 -c 1 \
    -o gpurun_out/prof_tma $CMD > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
tail -3 gpurun_out/ncu_full.log
