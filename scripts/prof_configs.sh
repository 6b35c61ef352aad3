# ncu --set full of the dominant kernel of each BASELINE config (one launch
# each), summarised on the box (reports are too large to bring back).
# usage: bash scripts/prof_configs.sh TAG
TAG=${1:-r1}
prof() {  # name kernel-regex skip bench_configs-args...
  local name=$1 re=$2 skip=$3; shift 3
  local CMD="python scripts/bench_configs.py --steps 1 --warmup 0 --cpu-seconds 0 $*"
  $CMD > gpurun_out/plain_$name.log 2>&1 && \
  ncu --set full --clock-control none -f -k regex:$re -s $skip -c 1 -o /tmp/prof_$name $CMD \
      > gpurun_out/ncu_$name.log 2>&1
  echo "$name ncu rc=$?"
  python scripts/ncu_summary.py /tmp/prof_$name.ncu-rep > gpurun_out/${TAG}_ncu_$name.json
}
prof cfg3_hh64 k_ragged_short 0 --only cfg3
prof cfg5_sip24 k_tma_fixed 1 --only cfg5
prof cfg5_tree24 k_tma_fixed 3 --only cfg5
prof cfg5_prf k_prf 0 --only prf
prof cfg2_ring k_ragged_ring 0 --only cfg2
prof cfg4_split k_tma_split 0 --only cfg4
