timeout 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_stages.py -x -q > gpurun_out/pytest_lut.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/pytest_lut.log
for v in 1 0; do STK_LSTAR_LUT=$v timeout 300 python scripts/lut_probe.py 2>&1 | tail -2; done
for v in 1 0 1 0; do
STK_LSTAR_LUT=$v timeout 150 python bench.py --steps 250 --no-cpu-baseline > gpurun_out/bench_lut$v.log 2>&1
python - $v <<'P'
import json, sys
try:
    l = [x for x in open(f"gpurun_out/bench_lut{sys.argv[1]}.log") if x.startswith("{")][-1]
    d = json.loads(l)
    print("lut", sys.argv[1], "value", d["value"], "e2e", d["e2e"]["value"], "convert_ms", d["roofline_stages"]["convert"]["ms"])
except Exception as e:
    print("lut", sys.argv[1], "failed", e)
P
done
