# frames-in-flight sweep and a torchrun N=1 launch of both arms
for s in 3 4 6 8; do
  timeout 300 python bench.py --steps 150 --no-cpu-baseline --slots $s > gpurun_out/bench_s$s.log 2>&1
  python - $s <<'P'
import json, sys
l = [x for x in open(f"gpurun_out/bench_s{sys.argv[1]}.log") if x.startswith("{")][-1]
d = json.loads(l)
print("slots", sys.argv[1], "value", d["value"], "e2e", d["e2e"]["value"])
P
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_trun.log 2>&1; echo "torchrun exit $?"; tail -c 300 gpurun_out/bench_trun.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/bench_trun_ref.log 2>&1; echo "torchrun ref exit $?"; tail -c 400 gpurun_out/bench_trun_ref.log
