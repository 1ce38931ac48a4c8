"""The leaf pool: MIG profile catalog, slice placements and per-GPU layouts.

Scope: `flexmig_layout` and the types it is built from.
Semantics follow the reference's `pkg/src/migsim/mig.py`:

* slice model - 7 compute slices, 8 memory slices of 5 GB (mig.py:28-30);
* catalog of six profiles, ascending by (slices, memory) (mig.py:45-52);
* fixed legal start slices per profile (mig.py:58-65);
* `GpuLayout` with instance ids handed out 1, 2, ... (mig.py:125-235);
* `flexmig_layout(g)` = 6 x 1g.5gb at slices 0-5 plus 1 x 1g.10gb at slice 6,
  instance ids 1..7 (mig.py:383-391).

The reconfiguration economics of Dynamic MIG (`mergeable`,
`plan_reconfiguration`, `pack_profiles`, `validate_target_config`;
mig.py:292-376, 403-439) are outside the one-to-many path: the names exist
so reference imports resolve, and calling them raises NotImplementedError.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

from .errors import (
    InstanceBusyError,
    InvalidTargetError,
    UnknownInstanceError,
    UnknownProfileError,
)

COMPUTE_SLICES_PER_GPU = 7
MEMORY_SLICES_PER_GPU = 8
MEMORY_GB_PER_SLICE = 5


@dataclass(frozen=True)
class MigProfile:
    name: str
    compute_slices: int
    memory_gb: int
    max_per_gpu: int

    @property
    def memory_slices(self) -> int:
        return self.memory_gb // MEMORY_GB_PER_SLICE


# (name, compute slices, memory GB, max per GPU, legal start slices)
_TABLE = (
    ("1g.5gb", 1, 5, 7, (0, 1, 2, 3, 4, 5, 6)),
    ("1g.10gb", 1, 10, 4, (0, 2, 4, 6)),
    ("2g.10gb", 2, 10, 2, (0, 2, 4)),
    ("3g.20gb", 3, 20, 2, (0, 4)),
    ("4g.20gb", 4, 20, 1, (0,)),
    ("7g.40gb", 7, 40, 1, (0,)),
)
_PROFILES = tuple(MigProfile(n, c, m, k) for n, c, m, k, _ in _TABLE)
_STARTS = {row[0]: row[4] for row in _TABLE}
_NAMED = {p.name: p for p in _PROFILES}

LEAF = "1g.5gb"          # the plain one-to-many leaf
DOUBLE_LEAF = "1g.10gb"  # the double-memory leaf at slice 6


def profile_catalog() -> list[MigProfile]:
    return list(_PROFILES)


def profile_by_name(name: str) -> MigProfile:
    if name not in _NAMED:
        raise UnknownProfileError(f"unknown profile {name!r}")
    return _NAMED[name]


@dataclass(frozen=True)
class Placement:
    start_slice: int
    span_slices: int
    memory_slices: int

    @property
    def compute_range(self) -> range:
        return range(self.start_slice, self.start_slice + self.span_slices)

    @property
    def memory_range(self) -> range:
        return range(self.start_slice, self.start_slice + self.memory_slices)

    def validate(self) -> None:
        if self.start_slice < 0 or self.start_slice >= COMPUTE_SLICES_PER_GPU:
            raise InvalidTargetError(f"start slice {self.start_slice} out of range")
        if self.start_slice + self.span_slices > COMPUTE_SLICES_PER_GPU:
            raise InvalidTargetError("placement exceeds the 7 compute slices")
        if self.start_slice + self.memory_slices > MEMORY_SLICES_PER_GPU:
            raise InvalidTargetError("placement exceeds the 8 memory slices")


def placement_for(profile: MigProfile, start: int) -> Placement:
    return Placement(start, profile.compute_slices, profile.memory_slices)


def legal_placements(profile: MigProfile) -> list[Placement]:
    starts = _STARTS.get(profile.name)
    if starts is None:
        raise UnknownProfileError(f"unknown profile {profile.name!r}")
    return [placement_for(profile, s) for s in starts]


@dataclass
class MigInstance:
    instance_id: int
    profile: MigProfile
    placement: Placement
    job_id: int | None = None

    @property
    def idle(self) -> bool:
        return self.job_id is None


@dataclass
class GpuLayout:
    """Instances carved out of one GPU (unpartitioned slices are free space)."""

    gpu_id: int
    instances: dict[int, MigInstance] = field(default_factory=dict)
    _next_id: int = field(default=1, compare=False, repr=False)

    def _get(self, instance_id: int) -> MigInstance:
        try:
            return self.instances[instance_id]
        except KeyError:
            raise UnknownInstanceError(
                f"instance {instance_id} not on gpu {self.gpu_id}") from None

    def occupied_compute(self) -> set[int]:
        return {s for i in self.instances.values() for s in i.placement.compute_range}

    def occupied_memory(self) -> set[int]:
        return {s for i in self.instances.values() for s in i.placement.memory_range}

    def busy_instances(self) -> list[MigInstance]:
        return [i for i in self.instances.values() if i.job_id is not None]

    def idle_instances(self) -> list[MigInstance]:
        return [i for i in self.instances.values() if i.job_id is None]

    def busy_compute_slices(self) -> int:
        return sum(i.profile.compute_slices for i in self.busy_instances())

    def free_compute_slices(self) -> int:
        return COMPUTE_SLICES_PER_GPU - self.busy_compute_slices()

    def profile_count(self, profile: MigProfile) -> int:
        return sum(i.profile.name == profile.name for i in self.instances.values())

    def add_instance(self, profile: MigProfile, placement: Placement,
                     job_id: int | None = None) -> MigInstance:
        inst = MigInstance(self._next_id, profile, placement, job_id)
        self.instances[inst.instance_id] = inst
        self._next_id += 1
        return inst

    def remove_instance(self, instance_id: int) -> MigInstance:
        inst = self._get(instance_id)
        del self.instances[instance_id]
        return inst

    def assign(self, instance_id: int, job_id: int) -> None:
        inst = self._get(instance_id)
        if inst.job_id is not None:
            raise InstanceBusyError(
                f"instance {instance_id} already runs job {inst.job_id}")
        inst.job_id = job_id

    def release(self, instance_id: int) -> None:
        self._get(instance_id).job_id = None

    def clone(self) -> "GpuLayout":
        twin = GpuLayout(self.gpu_id)
        for k, v in self.instances.items():
            twin.instances[k] = MigInstance(v.instance_id, v.profile, v.placement, v.job_id)
        twin._next_id = self._next_id
        return twin

    def to_json(self) -> str:
        recs = []
        for i in self.instances.values():
            pl = i.placement
            recs.append({
                "instance_id": i.instance_id,
                "profile": i.profile.name,
                "placement": {"start_slice": pl.start_slice,
                              "span_slices": pl.span_slices,
                              "memory_slices": pl.memory_slices},
                "job_id": i.job_id,
            })
        return json.dumps({"gpu_id": self.gpu_id, "instances": recs}, sort_keys=True)

    @classmethod
    def from_json(cls, text: str) -> "GpuLayout":
        doc = json.loads(text)
        layout = cls(doc["gpu_id"])
        for rec in doc["instances"]:
            pl = rec["placement"]
            inst = MigInstance(rec["instance_id"], profile_by_name(rec["profile"]),
                               Placement(pl["start_slice"], pl["span_slices"],
                                         pl["memory_slices"]),
                               rec["job_id"])
            layout.instances[inst.instance_id] = inst
        layout._next_id = max(layout.instances, default=0) + 1
        return layout


def try_allocate(layout: GpuLayout, profile: MigProfile) -> Placement | None:
    """Lowest legal start whose compute and memory slices are all free,
    respecting the per-profile cap (mig.py:272-289)."""
    if layout.profile_count(profile) >= profile.max_per_gpu:
        return None
    used_c, used_m = layout.occupied_compute(), layout.occupied_memory()
    for pl in legal_placements(profile):
        if used_c.isdisjoint(pl.compute_range) and used_m.isdisjoint(pl.memory_range):
            return pl
    return None


def flexmig_layout(gpu_id: int) -> GpuLayout:
    """Fixed one-to-many pool: 1g.5gb at slices 0..5, 1g.10gb at slice 6."""
    layout = GpuLayout(gpu_id)
    leaf, big = profile_by_name(LEAF), profile_by_name(DOUBLE_LEAF)
    for start in range(6):
        layout.add_instance(leaf, placement_for(leaf, start))
    layout.add_instance(big, placement_for(big, 6))
    return layout


def static_layout(gpu_id: int) -> GpuLayout:
    """One-to-one fixed layout (4g.20gb@0, 2g.10gb@4, 1g.10gb@6; mig.py:394-400).
    Kept for `make_cluster("SM"|"DM")`; those policies are out of scope."""
    layout = GpuLayout(gpu_id)
    for name, start in (("4g.20gb", 0), ("2g.10gb", 4), ("1g.10gb", 6)):
        p = profile_by_name(name)
        layout.add_instance(p, placement_for(p, start))
    return layout


# --------------------------------------------------------------------------
# Dynamic-MIG reconfiguration: out of scope for the one-to-many data path.


@dataclass
class ReconfigCosts:
    reconfigure_s: float = 110.0
    checkpoint_save_s: float = 5.0
    checkpoint_load_s: float = 5.0
    pod_cycle_s: float = 5.0

    def per_drained_job(self) -> float:
        return self.checkpoint_save_s + self.checkpoint_load_s + self.pod_cycle_s


@dataclass
class ReconfigPlan:
    gpu_id: int
    drained_jobs: list[int]
    destroy: list[int]
    create: list[tuple[MigProfile, Placement]]
    total_cost_s: float


def _out_of_scope(name: str):
    def fn(*args, **kwargs):
        raise NotImplementedError(
            f"{name} belongs to Dynamic-MIG reconfiguration, which is outside "
            "the one-to-many SHM data path this package implements (DESIGN.md §6)")
    fn.__name__ = name
    return fn


mergeable = _out_of_scope("mergeable")
validate_target_config = _out_of_scope("validate_target_config")
plan_reconfiguration = _out_of_scope("plan_reconfiguration")
pack_profiles = _out_of_scope("pack_profiles")
