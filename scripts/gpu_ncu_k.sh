# ncu --set full of one kernel (regex $1) in the second 4K frame
K=${1:-sad_ws}
python scripts/prof_frame.py --config C --frames 2 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -f -o gpurun_out/prof_$K \
  python scripts/prof_frame.py --config C --frames 2 > gpurun_out/ncu_$K.log 2>&1
echo "ncu exit $?"
