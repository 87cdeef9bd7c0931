#!/bin/bash
# A/B of library variants on the single-grid kernel (dev tool):
#   scripts/ab_single.sh build/var/a.so build/var/b.so ...
# Each timed twice, interleaved, with scripts/sbench.py on configs 0 and 2.
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $(basename $lib)"
    PFGPU_LIB_PARTIAL=1 PFGPU_LIB=$lib timeout 300 python scripts/sbench.py ${SB_CFGS:-0 2} 2>&1 | tail -2
  done
done
