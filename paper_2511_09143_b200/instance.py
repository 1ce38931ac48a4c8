"""Binding a rank process to its 1g instance, and the identity it publishes.

The paper's executor gives each rank `NVIDIA_VISIBLE_DEVICES` = one MIG UUID
and sets `CUDA_VISIBLE_DEVICES` + `NCCL_MIG_ID` per `LOCAL_RANK` (reference
PAPER.md:362-368, 377-384).  On a box whose GPUs expose MIG, `mode="mig"`
does exactly that.  Without MIG (the B200s this repo is measured on report
"MIG Mode: Disabled", profiles/r01_probe/system_summary.txt) a 1g instance is
stood in for by:

* `green` - a CUDA green context holding ~1/7 of the SMs (1g share of the 7
  compute slices, reference mig.py:28), its stream used for all of the
  rank's work, a 1g share of device memory via
  `torch.cuda.set_per_process_memory_fraction`, no peer access;
* `mps`   - an MPS client capped by `CUDA_MPS_ACTIVE_THREAD_PERCENTAGE`
  (set by the launcher before CUDA initialises); unlike green contexts in
  separate processes, which the driver time-slices, MPS clients run
  concurrently - the closest stand-in for a MIG slice (concurrent,
  SM-partitioned, separate address space).  A green context inside an MPS
  client is refused by this driver (CUDA "resources insufficient"), so the
  two are not combined;
* `full`  - the whole GPU (one rank per GPU, the NCCL-comparison layout).

In every mode the data path is the same host-SHM transport: P2P/NVLink are
never touched, matching what MIG permits (reference PAPER.md:262).

`peer_info()` builds the rank's `commsim.PeerInfo`: canonical PCIe bus id of
the physical GPU, and a per-instance identity token as `mig_id` (the MIG UUID,
or `<mode>-<gpu uuid>-<gpu id>.<instance id>`), which is what lets several ranks share
one bus id under MIG-aware discovery (reference commsim.py:67-88).
"""

from __future__ import annotations

import hashlib
import os
import socket
from dataclasses import dataclass, field

from .commsim import PeerInfo, canonical_bus_id

MODES = ("mig", "green", "mps", "full")
# Green contexts live as long as the process: tensors allocated under one are
# freed at interpreter exit, after any local Instance is gone.
_KEEP_ALIVE: list = []
ONE_G_FRACTION = 1.0 / 7.0   # compute share of a 1g slice (7 compute slices)
GREEN_SM_GRANULE = 8         # SM count granularity we request green contexts in


def _hash64(text: str) -> int:
    return int.from_bytes(hashlib.blake2b(text.encode(), digest_size=8).digest(), "little",
                          signed=True)


def host_hash() -> int:
    """Same value for every process on this host (NCCL's hostHash role)."""
    boot = ""
    try:
        with open("/proc/sys/kernel/random/boot_id") as f:
            boot = f.read().strip()
    except OSError:
        pass
    return _hash64(f"{socket.gethostname()}|{boot}")


def pid_hash() -> int:
    return _hash64(f"{socket.gethostname()}|{os.getpid()}")


def default_sm_count(total_sms: int) -> int:
    """SMs of a 1g stand-in: 1/7 of the GPU, floored to the request granule."""
    return max(GREEN_SM_GRANULE, int(total_sms * ONE_G_FRACTION) // GREEN_SM_GRANULE * GREEN_SM_GRANULE)


@dataclass
class Instance:
    gpu_id: int
    instance_id: int
    profile: str
    mode: str
    device: int = 0
    mig_uuid: str | None = None
    sm_count: int | None = None
    gpu_uuid: str = ""
    bus_id: str = ""
    stream: object = None
    green_ctx: object = field(default=None, repr=False)

    @property
    def mig_id(self) -> str:
        if self.mode == "mig" and self.mig_uuid:
            return self.mig_uuid
        return f"{self.mode}-{self.gpu_uuid}-{self.gpu_id}.{self.instance_id}"

    def cuda_stream(self) -> int:
        import torch
        s = self.stream if self.stream is not None else torch.cuda.current_stream(self.device)
        return int(s.cuda_stream)


def gpu_cpus(nvml_bus_id: str) -> set[int] | None:
    """CPUs of the GPU's NUMA node (NVML ideal affinity) for a PCI id in NVML's
    form (`00000000:9C:00.0`), or None if unknown."""
    try:
        import pynvml
        pynvml.nvmlInit()
        try:
            h = pynvml.nvmlDeviceGetHandleByPciBusId(nvml_bus_id)
            words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        finally:
            pynvml.nvmlShutdown()
    except Exception:  # noqa: BLE001 - no NVML / no such device: leave affinity alone
        return None
    cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
    allowed = os.sched_getaffinity(0)
    return (cpus & allowed) or None


def bind(gpu_id: int, instance_id: int, profile: str = "1g.5gb", mode: str = "green",
         device: int = 0, sm_count: int | None = None, memory_fraction: float | None = None,
         mig_uuid: str | None = None, pin_cpus: bool = True) -> Instance:
    """Bind this process to one instance.  `device` is the torch device index
    the instance's GPU has in this process (0 when the launcher narrowed
    CUDA_VISIBLE_DEVICES to it).  `pin_cpus` restricts the process to the
    CPUs of the GPU's NUMA node, so the SHM regions it first-touches in
    fmx_comm_init are allocated next to its GPU on multi-socket hosts."""
    import torch

    if mode not in MODES:
        raise ValueError(f"unknown instance mode {mode!r}")
    torch.cuda.set_device(device)
    props = torch.cuda.get_device_properties(device)
    inst = Instance(gpu_id, instance_id, profile, mode, device, mig_uuid=mig_uuid)
    inst.gpu_uuid = str(props.uuid)
    inst.bus_id = canonical_bus_id(
        f"{props.pci_domain_id:04x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0")
    if os.environ.get("FMX_FAKE_BUS"):
        # test only: several logical GPUs on one physical device get distinct bus
        # ids (F0:00.0, F1:00.0, ...), so communicators wider than the
        # reference's 10-ranks-per-bus rule (commsim.py:109-111) run on one B200
        inst.bus_id = f"{0xF0 + gpu_id:02X}:00:00.0"
    if pin_cpus:
        cpus = gpu_cpus(f"{props.pci_domain_id:08X}:{props.pci_bus_id:02X}:"
                        f"{props.pci_device_id:02X}.0")
        if cpus:
            os.sched_setaffinity(0, cpus)
    if mode == "green":
        inst.sm_count = sm_count or default_sm_count(props.multi_processor_count)
        gc = torch.cuda.GreenContext.create(inst.sm_count, device)
        gc.set_context()
        inst.green_ctx = gc
        _KEEP_ALIVE.append(gc)
        s = gc.Stream()
        inst.stream = s if isinstance(s, torch.cuda.Stream) else torch.cuda.ExternalStream(
            s.cuda_stream, device=device)
        torch.cuda.set_stream(inst.stream)
    else:
        inst.stream = torch.cuda.Stream(device)
        torch.cuda.set_stream(inst.stream)
    if memory_fraction is None and mode in ("green", "mps"):
        memory_fraction = ONE_G_FRACTION
    if memory_fraction:
        torch.cuda.set_per_process_memory_fraction(memory_fraction, device)
    return inst


def peer_info(inst: Instance, rank: int) -> PeerInfo:
    return PeerInfo(rank=rank, pcie_bus_id=inst.bus_id, mig_id=inst.mig_id,
                    host_hash=host_hash(), pid_hash=pid_hash())
