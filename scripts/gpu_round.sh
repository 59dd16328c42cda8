# Round checkpoint on one B200: GPU tests, default bench (+ CPU baseline), reference arm,
# ncu launch list of the bench, full ncu capture of one 4K frame (+ SAD source page),
# launch list of the stage-entry tests (which kernels the parity surface runs).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?"
tail -1 gpurun_out/bench.log | cut -c1-400
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?"
tail -1 gpurun_out/bench_ref.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --pool 2 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch exit $?"
python scripts/prof_frame.py --config C --frames 2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -s 13 -c 13 -f -o gpurun_out/prof_C \
  python scripts/prof_frame.py --config C --frames 2 > gpurun_out/ncu_full.log 2>&1
echo "ncu full exit $?"
ncu -i gpurun_out/prof_C.ncu-rep --page source --csv --print-source sass -k regex:k_sad_ws > gpurun_out/sad_source.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/stage_launches.csv \
  python -m pytest tests/test_gpu_stages.py -m gpu -q -k "detect or morph or components or prune" > gpurun_out/ncu_stage.log 2>&1
echo "ncu stage exit $?"
