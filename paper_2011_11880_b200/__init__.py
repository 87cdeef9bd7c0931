"""B200-native power-flow residual and Jacobian evaluation (arXiv 2011.11880).

Host API mirrors the reference package ``pflow``'s evaluation path:

* ``build_system`` / ``PowerSystem`` / ``flat_start``  (pflow/system_model.py)
* ``ResidualWorkspace`` / ``evaluate_residual``          (pflow/residual.py)
* ``JacobianWorkspace`` / ``symbolic_pattern`` / ``evaluate_jacobian``
  (pflow/jacobian.py)
* ``Plan`` - the device plan; ``ScenarioBuffers`` - scenario-batched mode.

All evaluation runs in libpfgpu.so (hand-written sm_100a CUDA, C ABI in
include/pfgpu.h).  Modules that need the GPU import torch lazily, so the
host model layer works on CPU-only machines.
"""

from .case import (CaseFormatError, RawCase, Violation, from_rows, make_case, parse_case,
                   parse_case_file, validate_case, write_case)
from .system_model import (AddressMap, LineGroup, PowerSystem, PqGroup, PvGroup, ShuntGroup,
                           SlackGroup, build_system, count_variables, flat_start, random_state)

__version__ = "0.1.0"


def __getattr__(name):
    # GPU-facing modules load on first use (they import torch / the CUDA lib)
    if name in ("Plan", "to_blocked", "from_blocked", "n_blocks", "launch_count"):
        from . import plan

        return getattr(plan, name)
    if name in ("ResidualWorkspace", "evaluate_residual", "line_injections", "pq_injections",
                "pv_injections", "slack_injections", "shunt_injections"):
        from . import residual

        return getattr(residual, name)
    if name in ("JacobianWorkspace", "symbolic_pattern", "evaluate_jacobian",
                "finite_difference_jacobian", "export_matrix_market"):
        from . import jacobian

        return getattr(jacobian, name)
    if name in ("NewtonOptions", "SolveResult", "newton_solve", "SingularMatrixError",
                "SuperLUSolver", "QLimitResult", "newton_solve_q_limits"):
        from . import newton

        return getattr(newton, name)
    if name in ("BatchedLU", "BatchedResult", "batched_newton_solve"):
        from . import batched_newton

        return getattr(batched_newton, name)
    if name in ("ScenarioBuffers", "gather_norms", "shard"):
        from . import batched

        return getattr(batched, name)
    raise AttributeError(name)


__all__ = [
    "AddressMap", "BatchedLU", "BatchedResult", "CaseFormatError", "JacobianWorkspace", "LineGroup", "NewtonOptions", "Plan",
    "PowerSystem", "PqGroup", "PvGroup", "RawCase", "ResidualWorkspace", "ScenarioBuffers",
    "ShuntGroup", "SlackGroup", "SolveResult", "Violation", "build_system", "count_variables",
    "batched_newton_solve", "evaluate_jacobian", "evaluate_residual", "finite_difference_jacobian", "flat_start",
    "from_rows", "gather_norms", "make_case", "newton_solve", "newton_solve_q_limits",
    "QLimitResult", "parse_case", "parse_case_file",
    "random_state", "shard", "symbolic_pattern", "validate_case", "write_case",
    "SingularMatrixError", "SuperLUSolver",
]
