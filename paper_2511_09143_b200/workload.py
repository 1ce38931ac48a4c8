"""Job record consumed by instance selection.

Only `Job` (reference `pkg/src/migsim/workload.py:50-57`) is on the path:
`fm_select` reads `job.size` (number of 1g leaves = ranks) and `job.job_id`.
Trace synthesis (workload.py:60-284) is a simulator input and out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Job:
    job_id: int
    kind: str  # "train" | "inference"
    size: int  # number of 1g leaves requested = data-parallel ranks
    base_duration_s: float
    arrival_s: float
    model_tag: str = ""


def _out_of_scope(name: str):
    def fn(*args, **kwargs):
        raise NotImplementedError(
            f"{name} belongs to trace synthesis, outside the one-to-many SHM data "
            "path this package implements (DESIGN.md §6)")
    fn.__name__ = name
    return fn


Trace = _out_of_scope("Trace")
TraceConfig = _out_of_scope("TraceConfig")
generate_trace = _out_of_scope("generate_trace")
