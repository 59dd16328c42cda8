timeout 600 python -m pytest tests/test_gpu_stages.py tests/test_gpu_pipeline.py -x -q -k "peek or pipeline or reconstruct or frame or golden" > gpurun_out/pytest_peek.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/pytest_peek.log
for v in 0 1 0 1; do
STK_PEEK_V4=$v timeout 150 python bench.py --steps 250 --no-cpu-baseline > gpurun_out/bench_peek$v.log 2>&1
python - $v <<'P'
import json, sys
try:
    l = [x for x in open(f"gpurun_out/bench_peek{sys.argv[1]}.log") if x.startswith("{")][-1]
    d = json.loads(l)
    print("v4", sys.argv[1], "value", d["value"], "peek_ms", d["roofline_stages"]["peek"]["ms"])
except Exception as e:
    print("v4", sys.argv[1], "failed", e)
P
done
