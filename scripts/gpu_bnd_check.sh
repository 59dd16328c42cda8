# boundary-chain change check: stage/pipeline/fuzz parity, a short bench, the B2-B8 launch times
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_pipeline.py tests/test_gpu_fuzz.py tests/test_gpu_parity_full.py -x -q > gpurun_out/pytest_bnd.log 2>&1; echo "pytest exit $?"
tail -2 gpurun_out/pytest_bnd.log
for i in 1 2; do
timeout 300 python bench.py --steps 200 --no-cpu-baseline > gpurun_out/bench_bnd.log 2>&1; echo "bench exit $?"
python - <<'P'
import json
l = [x for x in open("gpurun_out/bench_bnd.log") if x.startswith("{")][-1]
d = json.loads(l)
print("value", d["value"], "e2e", d["e2e"]["value"], {k: v["ms"] for k, v in d["roofline_stages"].items()})
P
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ccl|prune|apply|morph" --csv python scripts/prof_frame.py --config C --frames 4 2>/dev/null | grep '"' | awk -F, '{print $5, $NF}' | tail -14
