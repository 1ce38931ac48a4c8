"""B200-native one-to-many data path of Flex-MIG (arxiv 2511.09143).

Drop-in for the reference `migsim` surface on the hot path (instance
selection / placement, process-group bootstrap) plus the data path the
reference leaves to NCCL: allreduce / broadcast over a flat gradient buffer
through host shared memory, with hand-written sm_100a kernels behind the C
ABI of `libflexshm.so` (include/flexshm.h).

Control half (pure Python, reference semantics):
    mig.flexmig_layout, scheduler.make_cluster / fm_select / schedule_step,
    commsim.PeerInfo / discover_peers / build_topology / restore_bus_id /
    select_transport / load_peers_jsonl, errors.*
Data half (native):
    comm.init_process_group -> ShmCommunicator.allreduce / broadcast,
    instance.bind, launcher.launch, ddp.flexshm_hook
"""

from . import commsim, errors, mig, scheduler, simcore, workload
from .mig import (
    GpuLayout,
    MigInstance,
    MigProfile,
    Placement,
    ReconfigCosts,
    flexmig_layout,
    legal_placements,
    profile_by_name,
    profile_catalog,
    try_allocate,
)
from .scheduler import (
    AllocationDecision,
    ClusterState,
    Policy,
    fm_select,
    make_cluster,
    schedule_step,
)
from .simcore import PerfModel, estimate_jct
from .workload import Job

__all__ = [name for name in dir() if not name.startswith("_")]
