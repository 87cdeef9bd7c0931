#!/bin/bash
for L in "$@"; do echo "== $L"; for c in 0 2; do PFGPU_LIB=$L python scripts/dbg/graph_cost.py $c 2>&1 | grep -v "torch\|sincos"; done; done
