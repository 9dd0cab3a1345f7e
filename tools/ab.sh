#!/bin/bash
# A/B the default library against alternative builds on the bench (value only).
# usage: tools/ab.sh "<bench args>" lib1 lib2 ...   (repeats twice, interleaved)
args="$1"; shift
for i in 1 2; do
  for L in "$@"; do
    v=$(ABFS_LIB=$L timeout 300 python bench.py $args 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('fixed_vs_switched',{}).get('switched_over_best_fixed'))")
    echo "$L $args -> $v"
  done
done
