cp paper_1708_01159_b200/libabfs.so /tmp/lib_base.so
for v in base c4 c2 off; do
  if [ "$v" = base ] || [ "$v" = off ]; then cp /tmp/lib_base.so paper_1708_01159_b200/libabfs.so; else cp tools/micro/libabfs_$v.so paper_1708_01159_b200/libabfs.so; fi
  S=1; [ "$v" = off ] && S=0
  echo "== $v"; ABFS_SOLO=$S ABFS_DEBUG_GRID=1 timeout 300 python bench.py --no-cpu-baseline --fixed-roots 1 2>&1 | grep -E "megakernel grid|metric" | cut -c1-120 | sed 's/{"metric.*"value"/value/'
  ABFS_SOLO=$S timeout 200 python tools/diag_mesh.py 2>&1 | grep -E "^root|switched median"
done
cp /tmp/lib_base.so paper_1708_01159_b200/libabfs.so
