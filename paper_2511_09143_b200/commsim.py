"""Process-group bootstrap semantics for ranks that share a PCIe device.

Drop-in for the reference `pkg/src/migsim/commsim.py`:

* `PeerInfo` (commsim.py:27-42) - bus id upper-cased and required to be
  canonical `XX:XX:XX.0`, non-empty `mig_id`;
* `discover_peers(peers, mig_aware)` (commsim.py:67-88) - ranks must be
  exactly 0..n-1; duplicate key (host, bus, mig_id), or (host, bus) in
  legacy mode; first collision raises DuplicateDeviceError(earlier, later);
* `build_topology` (commsim.py:91-116) - k-th duplicate of a bus gets
  function digit k, k >= 10 is a MalformedLabelError, `mig_list` in
  first-seen order;
* `restore_bus_id` (commsim.py:119-123), `select_transport` (:126-132),
  `load_peers_jsonl` (:135-151).

These are the pure-Python rules; the native bootstrap in
`csrc/flexshm_host.cpp` (`fmx_validate_peers`, `fmx_topology_label`) applies
the same rules to the peer table the ranks exchange through POSIX SHM, and
`tests/test_bootstrap_native.py` holds both to the same golden vectors.

New helper: `canonical_bus_id` maps a CUDA/NVML bus id (`0000:4b:00.0`) to
the reference's canonical form (`00:4B:00.0`).
"""

from __future__ import annotations

import json
import re
from dataclasses import dataclass

from .errors import DuplicateDeviceError, MalformedLabelError

_HEX2 = "[0-9A-F]{2}"
_CANONICAL = re.compile(rf"^{_HEX2}:{_HEX2}:{_HEX2}\.0$")  # re.match semantics, as the reference
_LABEL = re.compile(rf"^{_HEX2}:{_HEX2}:{_HEX2}\.[0-9]$")
_CUDA_BUS = re.compile(r"^([0-9A-F]{4,8}):([0-9A-F]{2}):([0-9A-F]{2})\.([0-9A-F])$")

MAX_RANKS_PER_BUS = 10  # one decimal digit of synthetic ordinal


@dataclass(frozen=True)
class PeerInfo:
    rank: int
    pcie_bus_id: str
    mig_id: str
    host_hash: int
    pid_hash: int

    def __post_init__(self) -> None:
        bus = self.pcie_bus_id.upper()
        if _CANONICAL.match(bus) is None:
            raise MalformedLabelError(
                f"bus id {self.pcie_bus_id!r} is not a canonical device id")
        object.__setattr__(self, "pcie_bus_id", bus)
        if not self.mig_id:
            raise ValueError(f"rank {self.rank} has an empty mig_id")


@dataclass(frozen=True)
class Communicator:
    peers: tuple[PeerInfo, ...]

    @property
    def size(self) -> int:
        return len(self.peers)


@dataclass(frozen=True)
class TopoNode:
    label: str
    canonical: str
    rank: int


@dataclass
class TopologyGraph:
    nodes: list[TopoNode]
    mig_list: list[tuple[str, int]]


def device_key(peer: PeerInfo, mig_aware: bool) -> tuple:
    """Identity two ranks must not share (commsim.py:80-83)."""
    if mig_aware:
        return (peer.host_hash, peer.pcie_bus_id, peer.mig_id)
    return (peer.host_hash, peer.pcie_bus_id)


def discover_peers(peers: list[PeerInfo], mig_aware: bool = True) -> Communicator:
    n = len(peers)
    if sorted(p.rank for p in peers) != list(range(n)):
        raise ValueError(f"ranks must be 0..{n - 1} and distinct")
    by_rank = sorted(peers, key=lambda p: p.rank)
    owner: dict[tuple, int] = {}
    for p in by_rank:
        k = device_key(p, mig_aware)
        first = owner.setdefault(k, p.rank)
        if first != p.rank:
            raise DuplicateDeviceError(first, p.rank)
    return Communicator(tuple(by_rank))


def synthetic_label(canonical: str, ordinal: int) -> str:
    """Ordinal 0 keeps the canonical id; k >= 1 replaces the function digit."""
    if ordinal == 0:
        return canonical
    if ordinal >= MAX_RANKS_PER_BUS:
        raise MalformedLabelError(
            f"more than 10 ranks on bus {canonical}; ordinal does not fit one digit")
    return f"{canonical[:-1]}{ordinal}"


def build_topology(peers) -> TopologyGraph:
    ordered = list(peers.peers) if isinstance(peers, Communicator) \
        else sorted(peers, key=lambda p: p.rank)
    seen: dict[str, int] = {}
    nodes: list[TopoNode] = []
    for p in ordered:
        k = seen.get(p.pcie_bus_id, 0)
        nodes.append(TopoNode(synthetic_label(p.pcie_bus_id, k), p.pcie_bus_id, p.rank))
        seen[p.pcie_bus_id] = k + 1
    return TopologyGraph(nodes=nodes, mig_list=list(seen.items()))


def restore_bus_id(label: str) -> str:
    up = label.upper()
    if _LABEL.match(up) is None:
        raise MalformedLabelError(f"bad bus id label {label!r}")
    return up[:-1] + "0"


def select_transport(peer_a: PeerInfo, peer_b: PeerInfo) -> str:
    """"SHM" for a same-host pair, otherwise "NET"; never P2P/NVLink."""
    return "SHM" if peer_a.host_hash == peer_b.host_hash else "NET"


def load_peers_jsonl(data: bytes) -> list[PeerInfo]:
    out: list[PeerInfo] = []
    for line_no, line in enumerate(data.decode().splitlines(), start=1):
        if not line.strip():
            continue
        try:
            rec = json.loads(line)
            out.append(PeerInfo(rank=int(rec["rank"]),
                                pcie_bus_id=str(rec["pcie_bus_id"]),
                                mig_id=str(rec["mig_id"]),
                                host_hash=int(rec["host_hash"]),
                                pid_hash=int(rec["pid_hash"])))
        except (json.JSONDecodeError, KeyError, TypeError, ValueError) as exc:
            raise MalformedLabelError(f"peer file line {line_no}: {exc}") from None
    return out


def canonical_bus_id(cuda_bus_id: str) -> str:
    """`0000:4b:00.0` (cudaDeviceGetPCIBusId / NVML) -> `00:4B:00.0`.

    The reference's canonical form keeps two hex digits before the bus
    (commsim.py:23); we keep the low byte of the PCI domain there.  The
    function digit of a real GPU is 0; anything else is rejected.
    """
    m = _CUDA_BUS.fullmatch(cuda_bus_id.strip().upper())
    if m is None:
        if _CANONICAL.fullmatch(cuda_bus_id.strip().upper()):
            return cuda_bus_id.strip().upper()
        raise MalformedLabelError(f"bus id {cuda_bus_id!r} is not a PCI device id")
    domain, bus, dev, fn = m.groups()
    if fn != "0":
        raise MalformedLabelError(f"bus id {cuda_bus_id!r} is not function 0")
    return f"{domain[-2:]}:{bus}:{dev}.0"
