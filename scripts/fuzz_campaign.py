"""Extended randomized parity campaign (dev tool): the body of
tests/test_gpu_parity.py::test_random_grids_fuzz over many more seeds.
Prints one line per failing seed and a summary."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import test_gpu_parity as T  # noqa: E402

lo, hi = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (100, 300)))
bad = []
for seed in range(lo, hi):
    try:
        T.test_random_grids_fuzz(seed)
    except AssertionError as e:
        bad.append(seed)
        print(f"seed {seed}: {str(e)[:300]}", flush=True)
print(f"fuzz seeds {lo}..{hi - 1}: {hi - lo - len(bad)} passed, {len(bad)} failed {bad}")
