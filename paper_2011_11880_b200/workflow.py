"""Workflow selection, kept for API compatibility with pflow/workflow.py.

pflow runs its per-model kernels in one of six CPU workflows: inter-model
serial or threaded, times intra-model serial, threaded or SIMD
(workflow.py:1-30, 82-104). Its evaluate_* functions take the chosen
``WorkflowConfig``. The GPU path has a single execution strategy, the fused
kernels, so this module only reproduces the selection surface and its
validation. Code written against pflow (``workflow_config(5)``,
``set_worker_count(8)``, ``NewtonOptions(workflow=...)``) runs unchanged; the
configuration is accepted and then ignored. The thread pool itself is out of
scope.
"""

from __future__ import annotations

import os
from dataclasses import dataclass


class WorkflowConfigError(ValueError):
    """Invalid workflow selection: bad id, unknown strategy or worker count
    (pflow/workflow.py:44-46)."""


_KINDS = ("serial", "threaded", "simd")


@dataclass(frozen=True)
class IntraStrategy:
    kind: str
    n_threads: int = 1

    def __post_init__(self):
        if self.kind not in _KINDS:
            raise WorkflowConfigError(f"unknown intra-model strategy {self.kind!r}")
        if self.n_threads < 1:
            raise WorkflowConfigError("n_threads must be >= 1")

    @staticmethod
    def serial() -> "IntraStrategy":
        return IntraStrategy("serial")

    @staticmethod
    def threaded(n_threads: int) -> "IntraStrategy":
        return IntraStrategy("threaded", n_threads)

    @staticmethod
    def vectorized() -> "IntraStrategy":
        return IntraStrategy("simd")


@dataclass(frozen=True)
class WorkflowConfig:
    id: int
    inter: str
    intra: IntraStrategy


#: workflow id -> (inter-model, intra-model kind), pflow/workflow.py:82-89
WORKFLOW_TABLE = {1: ("serial", "serial"), 2: ("threaded", "serial"),
                  3: ("serial", "threaded"), 4: ("threaded", "threaded"),
                  5: ("serial", "simd"), 6: ("threaded", "simd")}

_workers: int | None = None


def _default_workers() -> int:
    env = os.environ.get("PFLOW_THREADS")
    if env:
        n = int(env)
        if n < 1:
            raise WorkflowConfigError(f"PFLOW_THREADS must be positive, got {env}")
        return n
    return os.cpu_count() or 1


def worker_count() -> int:
    return _workers if _workers is not None else _default_workers()


def set_worker_count(n: int) -> None:
    global _workers
    if n < 1:
        raise WorkflowConfigError("worker count must be >= 1")
    _workers = int(n)


def workflow_config(workflow_id: int, n_threads: int | None = None) -> WorkflowConfig:
    if workflow_id not in WORKFLOW_TABLE:
        raise WorkflowConfigError(f"workflow id must be 1..6, got {workflow_id}")
    inter, kind = WORKFLOW_TABLE[workflow_id]
    n = n_threads if n_threads is not None else worker_count()
    return WorkflowConfig(workflow_id, inter, IntraStrategy(kind, n if kind == "threaded" else 1))


def all_workflows(n_threads: int | None = None) -> list[WorkflowConfig]:
    return [workflow_config(i, n_threads) for i in sorted(WORKFLOW_TABLE)]
