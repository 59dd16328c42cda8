# frame period vs the SMs the SAD kernel may take (STK_SAD_SMS caps its bands)
for n in 0 128 112 96; do
  echo "STK_SAD_SMS=$n"; STK_SAD_SMS=$n bash scripts/bench_stages.sh
done
