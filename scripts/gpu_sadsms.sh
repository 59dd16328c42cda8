for n in 0 128 112 96; do
  STK_SAD_SMS=$n timeout 200 python bench.py --steps 120 --no-cpu-baseline > gpurun_out/b_$n.log 2>&1
  echo "SMS=$n $(grep -o '"value": [0-9.]*' gpurun_out/b_$n.log | head -2 | tr '\n' ' ') $(grep -o '"match": {"ms": [0-9.]*' gpurun_out/b_$n.log)"
done
