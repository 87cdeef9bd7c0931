"""Extended randomized parity campaign (dev tool): the body of
tests/test_gpu_parity.py::test_random_grids_fuzz over many more seeds.

Each seed builds a random grid (parallel and reversed branches, shifts, taps,
shunts, out-of-service rows, hubs, isolated buses), evaluates it single-grid
and scenario-batched on the GPU, and demands what the test demands: the
pattern bit-exact, every value within the north star's 1e-12 / 1e-14 bound
and bit-identical to the oracle's wf1.  There is no escape hatch: a seed
fails if any entry differs.  Prints one line per failing seed and a summary.

    python scripts/fuzz_campaign.py LO HI
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import test_gpu_parity as T  # noqa: E402

lo, hi = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (100, 300)))
bad = []
t0 = time.perf_counter()
for seed in range(lo, hi):
    try:
        T.test_random_grids_fuzz(seed)
    except AssertionError as e:
        bad.append(seed)
        print(f"seed {seed}: {str(e)[:400]}", flush=True)
print(f"fuzz seeds {lo}..{hi - 1}: {hi - lo - len(bad)} passed (bit-identical to wf1, "
      f"single grid and batched), {len(bad)} failed {bad}; "
      f"{time.perf_counter() - t0:.0f} s", flush=True)
