# A/B of the staged SipHash short-key path: ab/lib_base.so (round-1 form)
# against the in-tree library; then the Sip parity tests.
for lib in ab/lib_base.so paper_1612_06257_b200/libb200hash.so; do
  tag=$(basename $lib .so)
  LH_LIBRARY=$lib python scripts/bench_configs.py --only cfg3 --steps 20 --cpu-seconds 0 > gpurun_out/sipab_$tag.jsonl 2>&1
  LH_LIBRARY=$lib python -m paper_1612_06257_b200 bench --algo siphash24,siphash13 --sizes 12,24,31,48,63 --runs 3 > gpurun_out/sipab_sizes_$tag.txt 2>&1
done
python -m pytest tests/test_gpu_random_layouts.py tests/test_gpu_parity.py tests/test_gpu_sip_module.py tests/test_gpu_bounds.py -q -x -p no:cacheprovider 2>&1 | tail -2
