# full ncu capture of every kernel of the second 4K frame (device-resident path),
# plus the per-launch time list of the same command
set -x
python scripts/prof_frame.py --config C --frames 2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -s 12 -c 12 -f -o gpurun_out/prof_C \
  python scripts/prof_frame.py --config C --frames 2 > gpurun_out/ncu_full.log 2>&1
echo "ncu exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --pool 2 > gpurun_out/ncu_launch.log 2>&1
echo "ncu2 exit $?"
