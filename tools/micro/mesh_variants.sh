cp paper_1708_01159_b200/libabfs.so /tmp/lib_base.so
for v in "$@"; do
  if [ "$v" = base ]; then cp /tmp/lib_base.so paper_1708_01159_b200/libabfs.so; else cp tools/micro/libabfs_$v.so paper_1708_01159_b200/libabfs.so; fi
  echo "== $v"; python tools/diag_mesh.py 2>&1 | grep -E "^root|switched median|\(4, 2\)"
done
cp /tmp/lib_base.so paper_1708_01159_b200/libabfs.so
