# full ncu capture of every kernel of the second 4K frame (device-resident path)
set -x
python scripts/prof_frame.py --config C --frames 2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -s 15 -c 15 -f -o gpurun_out/prof_C \
  python scripts/prof_frame.py --config C --frames 2 > gpurun_out/ncu_full.log 2>&1
echo "ncu exit $?"
