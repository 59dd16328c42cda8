# full ncu capture of kernels (regex list) on the second 4K frame, per CUDA-line csv for each
python scripts/prof_frame.py --config C --frames 2 > gpurun_out/plain.log 2>&1 || { echo plain failed; exit 1; }
for K in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 -f -o gpurun_out/prof_$K \
    python scripts/prof_frame.py --config C --frames 2 > gpurun_out/ncu_$K.log 2>&1
  echo "ncu $K exit $?"
  ncu -i gpurun_out/prof_$K.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/lines_$K.csv 2>/dev/null
  ncu -i gpurun_out/prof_$K.ncu-rep --page details --csv > gpurun_out/det_$K.csv 2>/dev/null
  python scripts/ncu_stalls.py gpurun_out/prof_$K.ncu-rep
done
