# configs B and E (one B200): device and e2e frames/s, per-stage ms
for c in B E; do
  n=100; [ $c = E ] && n=40
  timeout 600 python bench.py --config $c --steps $n --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "config $c exit $?"
  tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['e2e']['value'], {k: v['ms'] for k, v in d['roofline_stages'].items()})"
done
