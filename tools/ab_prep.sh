#!/bin/bash
# A/B of K1 variants: tools/ab_prep.sh lib1 lib2 ... (interleaved, 2 rounds)
for r in 1 2; do
  for lib in "$@"; do
    echo "== $lib"
    if [ "$lib" = default ]; then python tools/prep_time.py; else DETNET_LIB=$lib python tools/prep_time.py; fi
  done
done
