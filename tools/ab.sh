#!/bin/bash
# A/B of stack-kernel variants: tools/ab.sh n lib1 lib2 ... (interleaved, 3 rounds)
n=$1; shift
for r in 1 2 3; do
  for lib in "$@"; do
    if [ "$lib" = default ]; then python tools/stack_time.py $n; else DETNET_LIB=$lib python tools/stack_time.py $n; fi
  done
done
