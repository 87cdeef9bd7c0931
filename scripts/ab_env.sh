#!/bin/bash
# A/B of the batched kernels on one box (dev tool): gpu tests, then the staged
# kernel ("new") against the single-role kernel (PF_BATCHED_KERNEL=old),
# interleaved, on config 3 (and config 4 with AB_C4=1).
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in new old new old; do
  if [ $v = old ]; then export PF_BATCHED_KERNEL=old; else unset PF_BATCHED_KERNEL; fi
  TAG=$v timeout 300 python scripts/kbench.py 2>&1 | tail -1
  if [ "${AB_C4:-0}" = 1 ]; then WORKLOAD=config4 TAG=$v timeout 300 python scripts/kbench.py 2>&1 | tail -1; fi
done
