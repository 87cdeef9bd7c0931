"""SuperLU solves in worker processes: the batched Newton's host fallback
(batched_newton._host_solves).  scipy's ``splu`` holds the GIL, so threads do
not overlap it.  Only numpy and scipy are imported here, so spawned workers
start quickly."""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def solve(args):
    """(values, rhs, indptr, indices, n) of a CSR system -> solution, or None
    when SuperLU finds it exactly singular (pflow's solve raises there)."""
    vals, rhs, indptr, indices, n = args
    try:
        return spla.splu(sp.csr_matrix((vals, indices, indptr), shape=(n, n)).tocsc()).solve(rhs)
    except RuntimeError:
        return None


def solve_local(vals: np.ndarray, rhs: np.ndarray, indptr, indices, n: int):
    return solve((vals, rhs, indptr, indices, n))
