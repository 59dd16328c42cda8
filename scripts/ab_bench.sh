# bench_stages in the main tree and each _ab/<variant>
bash scripts/bench_stages.sh; for d in _ab/*/; do echo "== $d"; (cd $d && bash ../../scripts/bench_stages.sh); done
