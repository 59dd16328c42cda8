for n in 0 136 128 120; do
  for sl in 4 6; do
  STK_SAD_SMS=$n timeout 200 python bench.py --steps 250 --slots $sl --no-cpu-baseline > gpurun_out/b_$n.log 2>&1
  echo "SMS=$n slots=$sl $(grep -o '"value": [0-9.]*' gpurun_out/b_$n.log | head -2 | tr '\n' ' ') $(grep -o '"match": {"ms": [0-9.]*' gpurun_out/b_$n.log)"
  done
done
