set -x
timeout 600 python bench.py --steps 20 --warmup 3 --cpu-seconds 5 > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -3 gpurun_out/bench.log
timeout 900 python -m pytest tests -x -q -m "gpu and slow" > gpurun_out/pytest_slow.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_slow.log
