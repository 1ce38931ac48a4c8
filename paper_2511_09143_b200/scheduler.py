"""Flex-MIG (FM) instance selection: which leaves a job gets, and in which
rank order.

Semantics follow the reference `pkg/src/migsim/scheduler.py`:

* `make_cluster(mode, G)` (scheduler.py:64-74) - FM clusters are G copies of
  `flexmig_layout`;
* `fm_select` (scheduler.py:139-173) - size 1 takes the lowest
  (gpu, start, id) idle 1g.10gb, else 1g.5gb, transport "LOCAL"; size >= 2
  spreads over 1g.5gb leaves round-robin and tops up with 1g.10gb leaves,
  transport "SHM"; `None` while supply < size;
* `_round_robin_pick` (scheduler.py:117-136) - the RANK ORDER of the job:
  every round visits the GPUs with leaves left, most-remaining first (ties by
  lower gpu id), one leaf each (lowest start slice first);
* `schedule_step` FIFO / bounded backfill (scheduler.py:409-446).

The returned `AllocationDecision.instances` list is the communicator's rank
order: rank r is bound to `instances[r]` (see `launcher.py`).  The Dynamic-MIG
policy (scheduler.py:180-330) is outside the one-to-many path: `dm_select`
exists for import compatibility and raises NotImplementedError.  The small
Static-MIG `sm_select` (scheduler.py:336-366) is kept so the shared queue
discipline can be tested on SM clusters too.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Mapping, Union

from .errors import OversizedJobError, WrongModeError
from .mig import (
    DOUBLE_LEAF,
    LEAF,
    GpuLayout,
    MigInstance,
    MigProfile,
    Placement,
    ReconfigCosts,
    ReconfigPlan,
    flexmig_layout,
    profile_by_name,
    static_layout,
)
from .workload import Job

MODES = ("FM", "DM", "SM")


@dataclass
class Policy:
    kind: str = "fifo"  # "fifo" | "backfill"
    depth: int = 14

    def __post_init__(self) -> None:
        if self.kind not in ("fifo", "backfill"):
            raise ValueError(f"unknown policy {self.kind!r}")
        if self.depth < 1:
            raise ValueError("backfill depth must be >= 1")


@dataclass
class ClusterState:
    gpus: list[GpuLayout]
    mode: str
    wait_queue: list[int] = field(default_factory=list)
    clock_s: float = 0.0
    reconfiguring: dict[int, float] = field(default_factory=dict)

    def layout(self, gpu_id: int) -> GpuLayout:
        for g in self.gpus:
            if g.gpu_id == gpu_id:
                return g
        raise KeyError(gpu_id)

    def schedulable_gpus(self) -> list[GpuLayout]:
        return [g for g in self.gpus if g.gpu_id not in self.reconfiguring]


def make_cluster(mode: str, num_gpus: int = 2) -> ClusterState:
    if mode == "FM":
        build = flexmig_layout
    elif mode in ("SM", "DM"):
        build = static_layout
    else:
        raise ValueError(f"unknown mode {mode!r}")
    return ClusterState(gpus=[build(g) for g in range(num_gpus)], mode=mode)


@dataclass
class AllocationDecision:
    job_id: int
    instances: list[tuple[int, int]]  # (gpu_id, instance_id), index = rank
    transport_class: str              # "SHM" | "LOCAL"
    profiles: list[str] = field(default_factory=list)


@dataclass
class PlannedReconfig:
    """DM-only outcome (scheduler.py:85-97); never produced here."""

    job_id: int
    gpu_id: int
    plan: ReconfigPlan
    assignments: list[tuple[int | None, MigProfile, Placement]]


SelectOutcome = Union[AllocationDecision, PlannedReconfig, None]


def _idle_leaves(cluster: ClusterState, profile_name: str) -> dict[int, list[MigInstance]]:
    """gpu_id -> idle leaves of one profile by ascending start slice, for
    every schedulable GPU that has any (scheduler.py:107-114)."""
    pools: dict[int, list[MigInstance]] = {}
    for g in cluster.schedulable_gpus():
        mine = sorted((i for i in g.idle_instances() if i.profile.name == profile_name),
                      key=lambda i: i.placement.start_slice)
        if mine:
            pools[g.gpu_id] = mine
    return pools


def _round_robin_pick(per_gpu: dict[int, list[MigInstance]], count: int) -> list[tuple[int, int]]:
    """Rank order of a multi-leaf job (scheduler.py:117-136)."""
    left = {g: list(v) for g, v in per_gpu.items()}
    out: list[tuple[int, int]] = []
    while len(out) < count:
        visit = [g for g in left if left[g]]
        if not visit:
            break
        visit.sort(key=lambda g: (-len(left[g]), g))
        for g in visit:
            if len(out) == count:
                break
            out.append((g, left[g].pop(0).instance_id))
    return out


def fm_select(job: Job, cluster: ClusterState) -> AllocationDecision | None:
    if cluster.mode != "FM":
        raise WrongModeError(f"fm_select on a {cluster.mode} cluster")

    if job.size == 1:
        for name in (DOUBLE_LEAF, LEAF):
            best = None
            for g in cluster.schedulable_gpus():
                for i in g.idle_instances():
                    if i.profile.name == name:
                        key = (g.gpu_id, i.placement.start_slice, i.instance_id)
                        if best is None or key < best:
                            best = key
            if best is not None:
                return AllocationDecision(job.job_id, [(best[0], best[2])], "LOCAL", [name])
        return None

    small = _idle_leaves(cluster, LEAF)
    big = _idle_leaves(cluster, DOUBLE_LEAF)
    supply_small = sum(map(len, small.values()))
    supply_big = sum(map(len, big.values()))
    if supply_small + supply_big < job.size:
        return None
    n_small = min(job.size, supply_small)
    picks = _round_robin_pick(small, n_small)
    profiles = [LEAF] * n_small
    if n_small < job.size:
        extra = _round_robin_pick(big, job.size - n_small)
        picks.extend(extra)
        profiles.extend([DOUBLE_LEAF] * len(extra))
    return AllocationDecision(job.job_id, picks, "SHM", profiles)


def _out_of_scope(name: str):
    def fn(*args, **kwargs):
        raise NotImplementedError(
            f"{name} is a one-to-one (DM/SM) policy, outside the one-to-many "
            "SHM data path this package implements (DESIGN.md §6)")
    fn.__name__ = name
    return fn


dm_select = _out_of_scope("dm_select")

# Static MIG (one-to-one baseline, scheduler.py:336-366): small enough to keep,
# so queue-discipline tests that run on SM clusters stay runnable.
_SM_LADDER = ("1g.10gb", "2g.10gb", "4g.20gb")


def sm_rounded_profile(size: int) -> MigProfile:
    for name in _SM_LADDER:
        p = profile_by_name(name)
        if p.compute_slices >= size:
            return p
    raise OversizedJobError(f"size {size} exceeds the static partitioning")


def sm_select(job: Job, cluster: ClusterState) -> AllocationDecision | None:
    if cluster.mode != "SM":
        raise WrongModeError(f"sm_select on a {cluster.mode} cluster")
    if job.size > 4:
        raise OversizedJobError(f"job {job.job_id} has size {job.size} > 4")
    need = sm_rounded_profile(job.size)
    for name in _SM_LADDER:
        p = profile_by_name(name)
        if (p.compute_slices, p.memory_gb) < (need.compute_slices, need.memory_gb):
            continue
        for g in cluster.schedulable_gpus():
            for inst in g.idle_instances():
                if inst.profile.name == name:
                    return AllocationDecision(job.job_id, [(g.gpu_id, inst.instance_id)],
                                              "LOCAL", [name])
    return None


def select_for(job: Job, cluster: ClusterState, cost_params: ReconfigCosts,
               jobs_by_id: Mapping[int, Job]) -> SelectOutcome:
    if cluster.mode == "FM":
        return fm_select(job, cluster)
    if cluster.mode == "DM":
        return dm_select(job, cluster, cost_params, jobs_by_id)
    return sm_select(job, cluster)


@dataclass
class StepResult:
    dispatched: list
    examined: list[int]

    @property
    def started(self) -> list[AllocationDecision]:
        return [d for d in self.dispatched if isinstance(d, AllocationDecision)]

    @property
    def reconfigs(self) -> list[PlannedReconfig]:
        return [d for d in self.dispatched if isinstance(d, PlannedReconfig)]


def _apply(outcome, cluster: ClusterState):
    if not isinstance(outcome, AllocationDecision):
        raise NotImplementedError("reconfiguration plans (DM) are out of scope")
    for gpu_id, inst_id in outcome.instances:
        cluster.layout(gpu_id).assign(inst_id, outcome.job_id)
    return outcome


def schedule_step(cluster: ClusterState, jobs_by_id: Mapping[int, Job], policy: Policy,
                  cost_params: ReconfigCosts | None = None) -> StepResult:
    """One pass over the wait queue (scheduler.py:409-446): FIFO stops at the
    first job that must wait; backfill examines a snapshot of the first
    `policy.depth` entries and dispatches each that fits."""
    costs = cost_params or ReconfigCosts()
    res = StepResult([], [])

    def dispatch(job_id: int) -> bool:
        outcome = select_for(jobs_by_id[job_id], cluster, costs, jobs_by_id)
        if outcome is None:
            return False
        res.dispatched.append(_apply(outcome, cluster))
        return True

    if policy.kind == "fifo":
        while cluster.wait_queue:
            head = cluster.wait_queue[0]
            res.examined.append(head)
            if not dispatch(head):
                break
            cluster.wait_queue.pop(0)
    else:
        for job_id in cluster.wait_queue[: policy.depth]:
            res.examined.append(job_id)
            if dispatch(job_id):
                cluster.wait_queue.remove(job_id)
    return res
