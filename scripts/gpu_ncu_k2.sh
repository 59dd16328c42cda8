# ncu --set full of kernels matching regex $1 (one launch each) in the second 4K frame
K=${1:-ccl}
N=${2:-1}
python scripts/prof_frame.py --config C --frames 2 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $N -c $N -f -o gpurun_out/prof_k2 \
  python scripts/prof_frame.py --config C --frames 2 > gpurun_out/ncu_k2.log 2>&1
echo "ncu exit $?"
