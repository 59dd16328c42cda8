# quick GPU check: SAD parity tests, then a short bench
timeout 300 python -m pytest tests/test_gpu_stages.py -x -q -k "match" > gpurun_out/pytest_match.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_match.log
timeout 300 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1; echo "bench exit $?"
tail -1 gpurun_out/bench_quick.log | cut -c1-3000
