for m in 1 2 3; do echo "== mode $m"; timeout 300 python tools/diag_k24.py --mode $m 2>&1 | grep -E "^root|PULL|PUSHW/2 F=(3067|17797)"; done
python tools/prof_levels.py --pair 3 2 --pair 4 2
