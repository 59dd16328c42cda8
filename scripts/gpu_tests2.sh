# full GPU test suite (no -x: report every failure) + short bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q --durations=12 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -40 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1; echo "bench exit $?"
tail -1 gpurun_out/bench_quick.log | cut -c1-3000
