for n in 2 1 3 4; do echo "STK_PRUNE_BPS=$n"; STK_PRUNE_BPS=$n bash scripts/bench_stages.sh; done
