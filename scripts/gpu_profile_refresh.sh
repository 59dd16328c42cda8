# Refresh profiles/: full ncu capture of the 12 kernels of the second 4K frame,
# the SASS source page of k_sad_ws, and the bench's own launch list.
set -x
python scripts/prof_frame.py --config C --frames 2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -s 12 -c 12 -f -o gpurun_out/prof_C \
  python scripts/prof_frame.py --config C --frames 2 > gpurun_out/ncu_full.log 2>&1
echo "ncu exit $?"
ncu -i gpurun_out/prof_C.ncu-rep --page source --csv --print-source sass -k regex:k_sad_ws > gpurun_out/sad_source.csv 2>/dev/null
echo "source exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --pool 2 > gpurun_out/ncu_launch.log 2>&1
echo "ncu2 exit $?"
