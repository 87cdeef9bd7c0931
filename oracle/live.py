"""Locate and import the live reference package ``pflow`` - TEST / BASELINE
INFRASTRUCTURE ONLY (same rules as the rest of ``oracle/``).

pflow is Python + Numba.  It is looked for, in order, at ``$PFLOW_SRC``,
``baseline/_ref`` (the offline ``pip install --target`` of /root/reference/pkg
that travels to the GPU box) and /root/reference/pkg/src (this
container only).  Numba's on-disk cache goes to a writable temp directory so
nothing is written into the reference tree.
"""

from __future__ import annotations

import importlib
import os
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
_CANDIDATES = [os.environ.get("PFLOW_SRC"), str(ROOT / "baseline" / "_ref"),
               "/root/reference/pkg/src"]
_STATE: dict = {}


def import_pflow():
    """(module, None) or (None, reason)."""
    if "mod" in _STATE:
        return _STATE["mod"], _STATE.get("why")
    os.environ.setdefault("NUMBA_CACHE_DIR", str(Path(tempfile.gettempdir()) / "pflow_numba"))
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    why = "pflow not found at $PFLOW_SRC, baseline/_ref or /root/reference/pkg/src"
    mod = None
    for c in _CANDIDATES:
        if c and (Path(c) / "pflow" / "__init__.py").exists():
            if c not in sys.path:
                sys.path.insert(0, c)
            try:
                mod = importlib.import_module("pflow")
                why = None
                _STATE["path"] = c
            except Exception as e:  # noqa: BLE001 (numba / scipy missing, ...)
                why = f"pflow at {c} failed to import: {e!r}"
            break
    _STATE["mod"], _STATE["why"] = mod, why
    return mod, why


def location() -> str | None:
    return _STATE.get("path")


def pflow_system(pflow, raw_case):
    """pflow's own PowerSystem for one of this package's RawCase objects: the
    case goes through MATPOWER text (case.write_case -> pflow.parse_case), so
    pflow builds it with its own parser and build_system."""
    from paper_2011_11880_b200 import case as C

    return pflow.build_system(pflow.parse_case(C.write_case(raw_case), name=raw_case.name))


def pflow_fixture(pflow, name: str):
    """pflow's bundled MATPOWER fixture (cases/<name>.m) through pflow."""
    path = Path(pflow.__file__).resolve().parent / "cases" / f"{name}.m"
    return pflow.build_system(pflow.parse_case_file(path))
