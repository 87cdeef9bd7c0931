"""Shared test helpers: golden fixtures and the parity criterion."""

from __future__ import annotations

from pathlib import Path

import numpy as np

from paper_2011_11880_b200 import case as C
from paper_2011_11880_b200 import system_model as SM

GOLDEN = Path(__file__).resolve().parent / "golden"
SINGLE = ["case2", "case5_shift", "case14", "tiny_edge", "slack_only", "edge300", "config0"]

# north star (BASELINE.json): per entry |d| <= max(1e-12 |ref|, 1e-14)
REL_TOL = 1e-12
ABS_TOL = 1e-14


def load(name: str):
    return np.load(GOLDEN / f"{name}.npz")


def case_of(d) -> C.RawCase:
    cols = {k[5:]: d[k] for k in d.files if k.startswith("case_")}
    return C.RawCase.from_arrays(cols, name=str(d["name"]))


def system_of(d):
    return SM.build_system(case_of(d))


def parity_failures(got, ref) -> int:
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    tol = np.maximum(REL_TOL * np.abs(ref), ABS_TOL)
    bad = ~(np.abs(got - ref) <= tol)
    return int(bad.sum())


def bit_mismatches(got, ref) -> int:
    """Entries whose fp64 bit patterns differ (signed zeros and NaN payloads
    included)."""
    got = np.ascontiguousarray(got, dtype=np.float64)
    ref = np.ascontiguousarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    return int((got.view(np.int64) != ref.view(np.int64)).sum())


def assert_parity(got, ref, what: str = "", bitwise: bool = True) -> None:
    """The north-star criterion (per entry within max(1e-12 |ref|, 1e-14)),
    then -- since the device sin/cos are glibc's own (csrc/pf_trig.h) and
    every other operation rounds where wf1 rounds -- bit-identity with the
    reference's wf1 (bitwise=False only where the reference value is not wf1
    itself)."""
    n = parity_failures(got, ref)
    if n:
        got = np.asarray(got)
        ref = np.asarray(ref)
        i = int(np.argmax(np.abs(got - ref) - np.maximum(REL_TOL * np.abs(ref), ABS_TOL)))
        raise AssertionError(f"{what}: {n} entries out of tolerance; worst at {i}: "
                             f"got {got.flat[i]!r} ref {ref.flat[i]!r}")
    if bitwise:
        nb = bit_mismatches(got, ref)
        if nb:
            g = np.ascontiguousarray(got, dtype=np.float64).ravel()
            r = np.ascontiguousarray(ref, dtype=np.float64).ravel()
            i = int(np.flatnonzero(g.view(np.int64) != r.view(np.int64))[0])
            raise AssertionError(f"{what}: {nb} of {g.size} entries within tolerance but not "
                                 f"bit-identical to wf1; first at {i}: got {g[i]!r} ref {r[i]!r}")


def csc_to_csr_perm(csc_indptr, csc_indices, csr_indptr, csr_indices):
    """perm such that csr_data = csc_data[perm] (pattern-only)."""
    n = csc_indptr.shape[0] - 1
    cols = np.repeat(np.arange(n), np.diff(csc_indptr))
    key_csc = csc_indices.astype(np.int64) * n + cols
    rows = np.repeat(np.arange(n), np.diff(csr_indptr))
    key_csr = rows.astype(np.int64) * n + csr_indices
    order = np.argsort(key_csc, kind="stable")
    pos = np.searchsorted(key_csc[order], key_csr)
    return order[pos]
