# ncu --set full of every launch matching regex $1 in a 2-frame 4K run (both frames)
K=${1:-blur}
python scripts/prof_frame.py --config C --frames 2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -f -o gpurun_out/prof_k3 \
  python scripts/prof_frame.py --config C --frames 2 > gpurun_out/ncu_k3.log 2>&1
echo "ncu exit $?"
