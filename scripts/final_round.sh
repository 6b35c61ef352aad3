# Final evidence of a round: GPU tests (with the full-size parity log), smoke,
# bench + reference arm, launch list, ncu summaries of every config's kernel,
# the ragged balance table.  usage: bash scripts/final_round.sh TAG
TAG=${1:-r2_final}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke rc=$?
python -m pytest tests -q -m gpu -s > gpurun_out/${TAG}_gputest.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/${TAG}_gputest.log
bash scripts/capture_round.sh ${TAG}
python scripts/ncu_summary.py gpurun_out/${TAG}_full.ncu-rep > gpurun_out/${TAG}_ncu_full_headline.json
rm -f gpurun_out/${TAG}_full.ncu-rep
bash scripts/prof_configs.sh ${TAG}
(cd scripts && python ragged_balance_bench.py) > gpurun_out/${TAG}_ragged_balance.jsonl 2>&1; echo balance rc=$?
tools/issuemix > gpurun_out/${TAG}_issuemix_raw.json 2>&1; echo issuemix rc=$?
