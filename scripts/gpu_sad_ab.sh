# A/B of the SAD kernel variant (STK_SAD_SMR=1 vs 0): parity then bench (short timeouts: a hang must not eat the budget)
STK_SAD_SMR=1 timeout 240 python -m pytest tests/test_gpu_stages.py -k match -x -q > gpurun_out/pytest_sad.log 2>&1; echo "pytest exit $?"
tail -2 gpurun_out/pytest_sad.log
STK_SAD_SMR=1 timeout 300 python -m pytest tests/test_gpu_pipeline.py -x -q > gpurun_out/pytest_sad2.log 2>&1; echo "pytest2 exit $?"
tail -2 gpurun_out/pytest_sad2.log
for v in 1 0 1 0; do
STK_SAD_SMR=$v timeout 120 python bench.py --steps 150 --no-cpu-baseline > gpurun_out/bench_ab$v.log 2>&1
python - $v <<'P'
import json, sys
try:
    l = [x for x in open(f"gpurun_out/bench_ab{sys.argv[1]}.log") if x.startswith("{")][-1]
    d = json.loads(l)
    print("variant", sys.argv[1], "value", d["value"], "match_ms", d["roofline_stages"]["match"]["ms"])
except Exception as e:
    print("variant", sys.argv[1], "failed", e)
P
done
