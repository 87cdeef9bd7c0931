#!/bin/bash
# A/B of the batched processing order (dev tool): PF_ORDER=bus against the
# default spanning-tree preorder, interleaved, configs 3 and 4.
for rep in 1 2; do
  for o in bus tree; do
    PF_ORDER=$o TAG="order=$o" timeout 300 python scripts/kbench.py 2>&1 | tail -1
    PF_ORDER=$o WORKLOAD=config4 TAG="order=$o" timeout 300 python scripts/kbench.py 2>&1 | tail -1
  done
done
