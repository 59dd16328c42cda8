timeout 200 python bench.py --steps 250 --no-cpu-baseline > gpurun_out/b_img.log 2>&1
echo "img: $(grep -o '"e2e": {"value": [0-9.]*' gpurun_out/b_img.log) dev $(grep -o '"value": [0-9.]*' gpurun_out/b_img.log | head -1)"
timeout 200 python bench.py --steps 250 --no-cpu-baseline --e2e-dense > gpurun_out/b_dense.log 2>&1
echo "dense: $(grep -o '"e2e": {"value": [0-9.]*' gpurun_out/b_dense.log)"
timeout 200 python bench.py --steps 250 --no-cpu-baseline --slots 5 > gpurun_out/b_s5.log 2>&1
echo "slots5: $(grep -o '"e2e": {"value": [0-9.]*' gpurun_out/b_s5.log) dev $(grep -o '"value": [0-9.]*' gpurun_out/b_s5.log | head -1)"
