mkdir -p gpurun_out/s6
for v in "$@"; do for c in 2 3; do
  if [ "$v" = base ]; then unset DETNET_LIB; else export DETNET_LIB=build/$v/libdetnet_b200.so; fi
  timeout 200 python tools/kernel_ab.py 1048576 $c 10 2>&1 | tail -1
done; done
