# frames/s under alternating environment settings: scripts/ab_fps_env.sh "A=1" "A=2" ...
for i in 1 2 3; do for e in "$@"; do
 echo "$e $(env $e timeout 300 python bench.py --steps 300 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline_stages']['boundary']['ms'])")"
done; done
