# usage: bash scripts/prof_kernel.sh TAG KERNEL_REGEX SKIP -- bench_configs args
TAG=$1; RE=$2; SKIP=$3; shift 4
CMD="python scripts/bench_configs.py --steps 1 --warmup 0 --cpu-seconds 0 $*"
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$RE -s $SKIP -c 1 \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo ncu rc=$?
