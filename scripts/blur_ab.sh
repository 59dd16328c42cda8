# blur kernel launch times (ncu, config C) in the main tree and each _ab/<variant>
export STK_BLUR_TC=${STK_BLUR_TC:-1}
t() { timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:blur --csv python scripts/prof_frame.py --config C --frames 4 2>/dev/null | grep -i blur | awk -F, '{print $5, $NF}' | tail -2; }
echo "== main"; t
for d in _ab/*/; do echo "== $d"; (cd $d && t); done
