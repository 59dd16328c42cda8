# quick GPU check: the given pytest selection (default: stage + pipeline tests)
sel=${1:-"tests/test_gpu_stages.py tests/test_gpu_pipeline.py"}
timeout 1200 python -m pytest $sel -m gpu -q -x --durations=5 > gpurun_out/pytest_quick.log 2>&1; echo "pytest exit $?"
tail -30 gpurun_out/pytest_quick.log
