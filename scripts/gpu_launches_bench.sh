# per-launch device times over the bench's own frames (ncu, serialized; ~17 frames)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --pool 2 > gpurun_out/ncu_launch_bench.log 2>&1
echo "ncu exit $?"
python scripts/launches_summary.py gpurun_out/launches_bench.csv
