# bench.py under torchrun: world 1, and world 2 with both ranks on device 0
# (STK_BENCH_ONE_DEVICE=1: functional check of the gloo control plane + frame
# sharding on a one-GPU box; not a scaling measurement)
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/torchrun1.log 2>&1; echo "torchrun 1 exit $?"
tail -1 gpurun_out/torchrun1.log | cut -c1-300
STK_BENCH_ONE_DEVICE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 --steps 20 --warmup 3 --slots 4 --pool 4 > gpurun_out/torchrun2.log 2>&1; echo "torchrun 2 exit $?"
grep '^{' gpurun_out/torchrun2.log | cut -c1-300
