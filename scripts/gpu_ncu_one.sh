# one full ncu capture of kernel $1 (second 4K frame) + its source page
K=$1
python scripts/prof_frame.py --config C --frames 2 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -f -o gpurun_out/prof_one \
  python scripts/prof_frame.py --config C --frames 2 > gpurun_out/ncu_one.log 2>&1
echo "ncu exit $?"
ncu -i gpurun_out/prof_one.ncu-rep --page source --csv --print-source sass > gpurun_out/one_source.csv 2>/dev/null
ncu -i gpurun_out/prof_one.ncu-rep --page details --csv > gpurun_out/one_details.csv 2>/dev/null
