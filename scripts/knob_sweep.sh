# fps / stage ms for each value of an env knob: scripts/knob_sweep.sh NAME v1 v2 ...
name=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  echo "== $name=$v"
  env $name=$v timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/knob.log 2>&1
  tail -1 gpurun_out/knob.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], {k: v['ms'] for k, v in d['roofline_stages'].items()})"
done
