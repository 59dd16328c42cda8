# SAD kernel change check: the SAD / frame parity tests, then a short bench
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_pipeline.py tests/test_gpu_eval.py -x -q > gpurun_out/pytest_sad.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_sad.log
timeout 300 python bench.py --steps 100 --no-cpu-baseline > gpurun_out/bench_sad.log 2>&1; echo "bench exit $?"
python - <<'P'
import json
l = [x for x in open("gpurun_out/bench_sad.log") if x.startswith("{")][-1]
d = json.loads(l)
print("value", d["value"], "e2e", d["e2e"]["value"], "match_ms", d["roofline_stages"]["match"]["ms"], {k: v["ms"] for k, v in d["roofline_stages"].items()})
P
