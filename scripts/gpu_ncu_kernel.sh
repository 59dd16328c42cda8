# full ncu capture of one kernel (regex $1) of the second 4K frame + summaries
K=$1
python scripts/prof_frame.py --config C --frames 2 > gpurun_out/plain.log 2>&1 || { echo plain failed; tail gpurun_out/plain.log; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -f -o gpurun_out/prof_$K \
  python scripts/prof_frame.py --config C --frames 2 > gpurun_out/ncu_$K.log 2>&1
echo "ncu exit $?"
ncu -i gpurun_out/prof_$K.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$K.csv 2>/dev/null
ncu -i gpurun_out/prof_$K.ncu-rep --page details --csv > gpurun_out/det_$K.csv 2>/dev/null
python scripts/ncu_stalls.py gpurun_out/prof_$K.ncu-rep
