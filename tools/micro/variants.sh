# usage: bash tools/micro/variants.sh tag1 tag2 ...  (tools/micro/libabfs_<tag>.so; "base" = in-tree build)
cp paper_1708_01159_b200/libabfs.so /tmp/lib_base.so
for v in "$@"; do
  if [ "$v" = base ]; then cp /tmp/lib_base.so paper_1708_01159_b200/libabfs.so; else cp tools/micro/libabfs_$v.so paper_1708_01159_b200/libabfs.so; fi
  echo "== $v"; timeout 300 python tools/diag_k24.py 2>&1 | grep -E "^root|PULL"; python tools/prof_levels.py --pair 3 2
  timeout 300 python bench.py --no-cpu-baseline --fixed-roots 1 2>&1 | tail -1 | cut -c1-160
done
cp /tmp/lib_base.so paper_1708_01159_b200/libabfs.so
