# ncu --set full of kernels matching regex $1: skip $2 matching launches, capture $3
K=${1:-ccl}
python scripts/prof_frame.py --config C --frames 2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${2:-0} -c ${3:-1} -f -o gpurun_out/prof_k4 \
  python scripts/prof_frame.py --config C --frames 2 > gpurun_out/ncu_k4.log 2>&1
echo "ncu exit $?"
