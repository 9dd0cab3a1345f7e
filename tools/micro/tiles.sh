cp paper_1708_01159_b200/libabfs.so /tmp/lib16.so
for t in 8 16 32; do
  if [ $t = 16 ]; then cp /tmp/lib16.so paper_1708_01159_b200/libabfs.so; else cp tools/micro/libabfs_t$t.so paper_1708_01159_b200/libabfs.so; fi
  echo "== tile $t"; timeout 300 python tools/diag_k24.py 2>&1 | grep -E "^root|PULL"; python tools/prof_levels.py --pair 3 2
done
cp /tmp/lib16.so paper_1708_01159_b200/libabfs.so
