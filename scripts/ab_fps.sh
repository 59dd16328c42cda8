# frames/s of the main tree and each _ab/<variant>, alternating, 3 runs each
for i in 1 2 3; do for d in . _ab/*/; do
 (cd $d && echo "$d $(timeout 300 python bench.py --steps 300 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline_stages']['boundary']['ms'])")")
done; done
