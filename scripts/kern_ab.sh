# one kernel's launch times (ncu, config C) in the main tree and each _ab/<variant>: scripts/kern_ab.sh REGEX
t() { timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$1 --csv python scripts/prof_frame.py --config C --frames 4 2>/dev/null | grep -v '^==' | grep '"' | awk -F, '{print $5, $NF}' | tail -2; }
echo "== main"; t $1
for d in _ab/*/; do echo "== $d"; (cd $d && t $1); done
