# A/B of library variants on the stack kernel: config 2 (dense) and 3 (compacted)
for rep in 1 2; do
for lib in paper_2003_09446_b200/lib/libdetnet_b200.so build/r240_24/libdetnet_b200.so; do
  for c in 2 3; do
    echo "$lib c$c: $(DETNET_LIB=$lib PROF_TIME=1 timeout 120 python tools/prof_run.py 1048576 0 $c 2>&1 | tail -1)"
  done
done
done
