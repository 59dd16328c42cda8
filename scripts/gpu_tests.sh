# full GPU test suite + short bench
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1; echo "bench exit $?"
tail -1 gpurun_out/bench_quick.log | cut -c1-3000
