# A/B of boundary-chain variants: main tree and each _ab/<variant> (parity subset, bench, B2-B8 launch times)
for d in . _ab/*/; do
 echo "=== $d"
 (cd $d && timeout 600 python -m pytest tests/test_gpu_stages.py -x -q -k "component or prune or boundar" 2>&1 | tail -1
  timeout 300 python bench.py --steps 200 --no-cpu-baseline > /tmp/b.log 2>&1; python -c "
import json
l=[x for x in open('/tmp/b.log') if x.startswith('{')][-1]; d=json.loads(l)
print('value', d['value'], 'e2e', d['e2e']['value'], {k: v['ms'] for k, v in d['roofline_stages'].items() if k in ('boundary','match')})"
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ccl|prune|apply" --csv python scripts/prof_frame.py --config C --frames 3 2>/dev/null | grep '"' | awk -F, '{print $5, $NF}' | tail -6)
done
