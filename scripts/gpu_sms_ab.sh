# SAD SM cap (STK_SAD_SMS) vs full: lets other frames' kernels run beside the match kernel
for v in 0 128 112 0 128; do
if [ $v = 0 ]; then unset STK_SAD_SMS; else export STK_SAD_SMS=$v; fi
timeout 150 python bench.py --steps 250 --no-cpu-baseline > gpurun_out/bench_sms$v.log 2>&1
python - $v <<'P'
import json, sys
try:
    l = [x for x in open(f"gpurun_out/bench_sms{sys.argv[1]}.log") if x.startswith("{")][-1]
    d = json.loads(l)
    print("sms", sys.argv[1], "value", d["value"], "match_ms", d["roofline_stages"]["match"]["ms"])
except Exception as e:
    print("sms", sys.argv[1], "failed", e)
P
done
