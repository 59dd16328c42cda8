t() { timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:peek --csv python scripts/prof_frame.py --config C --frames 4 2>/dev/null | grep -i peek | awk -F, '{print $5, $NF}' | tail -2; }
echo "== main"; t
for d in _ab/*/; do echo "== $d"; (cd $d && t); done
