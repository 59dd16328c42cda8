# one full ncu capture of k_sad_ws (second 4K frame) + its SASS source page
python scripts/prof_frame.py --config C --frames 2 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sad_ws -s 1 -c 1 -f -o gpurun_out/prof_sad \
  python scripts/prof_frame.py --config C --frames 2 > gpurun_out/ncu_sad.log 2>&1
echo "ncu exit $?"
ncu -i gpurun_out/prof_sad.ncu-rep --page source --csv --print-source sass > gpurun_out/sad_source2.csv 2>/dev/null
