cp paper_1708_01159_b200/libabfs.so /tmp/lib_base.so
for v in base prev; do
  if [ "$v" = base ]; then cp /tmp/lib_base.so paper_1708_01159_b200/libabfs.so; else cp tools/micro/libabfs_$v.so paper_1708_01159_b200/libabfs.so; fi
  for m in 1 2 3; do echo "== $v mode $m"; for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --fixed-roots 1 --mode $m 2>&1 | tail -1 | cut -c60-100; done; done
done
cp /tmp/lib_base.so paper_1708_01159_b200/libabfs.so
