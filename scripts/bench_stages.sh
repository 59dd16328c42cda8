# quick bench: fps and per-stage ms (no CPU baseline)
mkdir -p gpurun_out
timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline ${@} > gpurun_out/bench_stages.log 2>&1
tail -1 gpurun_out/bench_stages.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], {k: v['ms'] for k, v in d['roofline_stages'].items()})"
