#!/bin/bash
# A/B of library variants (dev tool): scripts/ab_libs.sh build/var/a.so build/var/b.so ...
# Each is timed twice, interleaved, on config 3 (and config 4 with AB_C4=1).
for rep in 1 2; do
  for lib in "$@"; do
    PFGPU_LIB=$lib TAG="$(basename $lib)" timeout 300 python scripts/kbench.py 2>&1 | tail -1
    if [ "${AB_C4:-0}" = 1 ]; then
      PFGPU_LIB=$lib WORKLOAD=config4 TAG="$(basename $lib)" timeout 300 python scripts/kbench.py 2>&1 | tail -1
    fi
  done
done
