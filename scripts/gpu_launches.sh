# per-launch device times of 2 device-resident 4K frames (ncu, serialized)
python scripts/prof_frame.py --config C --frames 3 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 20 -c 40 --csv --log-file gpurun_out/launches.csv python scripts/prof_frame.py --config C --frames 3 > gpurun_out/ncu_launch.log 2>&1
echo "ncu exit $?"
