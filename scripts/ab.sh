#!/bin/bash
# A/B kernel timing of library variants on one box (dev tool):
#   scripts/ab.sh build/var/libA.so build/var/libB.so ...
# Each library is timed twice, interleaved, on config 3 (and config 4 when
# AB_C4=1).
for rep in 1 2; do
  for lib in "$@"; do
    PFGPU_LIB=$lib TAG="$(basename $lib) r$rep" python scripts/kbench.py
    if [ "${AB_C4:-0}" = 1 ]; then
      PFGPU_LIB=$lib WORKLOAD=config4 TAG="$(basename $lib) c4 r$rep" python scripts/kbench.py
    fi
  done
done
