"""The native bootstrap rules of libflexshm (fmx_check_peer,
fmx_validate_peers, fmx_topology, fmx_restore_bus_id) against the golden
vectors produced by the REFERENCE (tests/golden/control_golden.json), and
the multi-process SHM bootstrap (host-only transport: no GPU needed) with
world sizes 2 and 7, including a MIG-aware duplicate across processes."""

from __future__ import annotations

import ctypes
import json
import multiprocessing as mp
import os
import uuid

import pytest

from paper_2511_09143_b200 import _lib
from paper_2511_09143_b200.errors import DuplicateDeviceError, MalformedLabelError

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "control_golden.json")))


def c_peers(recs):
    arr = (_lib.PeerInfoC * max(1, len(recs)))()
    for i, p in enumerate(recs):
        arr[i] = _lib.peer_to_c(p["rank"], p["pcie_bus_id"].upper(), p["mig_id"], p["host_hash"],
                                p["pid_hash"])
    return arr


def native_outcome(recs, mig_aware):
    L = _lib.lib()
    arr = c_peers(recs)
    a, b = ctypes.c_int(-1), ctypes.c_int(-1)
    rc = L.fmx_validate_peers(arr, len(recs), int(mig_aware), ctypes.byref(a), ctypes.byref(b))
    if rc == _lib.FMX_ERR_DUPLICATE_DEVICE:
        return {"error": "DuplicateDeviceError", "rank_a": a.value, "rank_b": b.value}, None
    if rc == _lib.FMX_ERR_BAD_RANKS:
        return {"error": "ValueError"}, None
    assert rc == 0, _lib.last_error()
    n = len(recs)
    labels = ctypes.create_string_buffer(_lib.BUS_ID_LEN * max(1, n))
    buses = ctypes.create_string_buffer(_lib.BUS_ID_LEN * max(1, n))
    counts = (ctypes.c_int * max(1, n))()
    nb = ctypes.c_int()
    rc = L.fmx_topology(arr, n, labels, buses, counts, ctypes.byref(nb))
    discover = {"ranks": list(range(n))}
    if rc == _lib.FMX_ERR_MALFORMED_LABEL:
        return discover, {"error": "MalformedLabelError"}
    assert rc == 0
    by_rank = sorted(recs, key=lambda p: p["rank"])

    def s(buf, i):
        return buf.raw[i * _lib.BUS_ID_LEN:(i + 1) * _lib.BUS_ID_LEN].split(b"\0")[0].decode()

    topo = {"labels": [[s(labels, i), by_rank[i]["pcie_bus_id"].upper(), by_rank[i]["rank"]]
                       for i in range(n)],
            "mig_list": [[s(buses, i), counts[i]] for i in range(nb.value)]}
    return discover, topo


def test_native_validation_and_topology_match_reference_golden():
    checked = 0
    for case in GOLDEN["discover_topology"]:
        disc, topo = native_outcome(case["peers"], case["mig_aware"])
        assert disc == case["discover"], case
        if topo is not None:
            assert topo == case["topology"], case
        checked += 1
    assert checked > 400


def test_native_check_peer_matches_reference_golden():
    L = _lib.lib()
    for case in GOLDEN["peerinfo"]:
        try:
            p = _lib.peer_to_c(0, case["bus"], case["mig"], 1, 1)
        except MalformedLabelError:
            assert case.get("error") == "MalformedLabelError"
            continue
        rc = L.fmx_check_peer(ctypes.byref(p))
        if "ok" in case:
            assert rc == 0, (case, _lib.last_error())
            assert p.pcie_bus_id.decode() == case["ok"]
        elif case["error"] == "MalformedLabelError":
            assert rc == _lib.FMX_ERR_MALFORMED_LABEL, case
        else:
            assert rc == _lib.FMX_ERR_EMPTY_MIG_ID, case


def test_native_restore_bus_id_matches_reference_golden():
    L = _lib.lib()
    for case in GOLDEN["restore_bus_id"]:
        out = ctypes.create_string_buffer(_lib.BUS_ID_LEN)
        rc = L.fmx_restore_bus_id(case["label"].encode(), out)
        if "ok" in case:
            assert rc == 0 and out.value.decode() == case["ok"], case
        else:
            assert rc == _lib.FMX_ERR_MALFORMED_LABEL, case


# ---------------------------------------------------------------- multi-process


def _host_rank(rank, n, key, mig_ids, q, hosts=None):
    from paper_2511_09143_b200.comm import init_process_group
    from paper_2511_09143_b200.commsim import PeerInfo
    from paper_2511_09143_b200.errors import TransportUnavailableError
    try:
        peer = PeerInfo(rank, "00:C0:00.0", mig_ids[rank], hosts[rank] if hosts else 7, 100 + rank)
        comm = init_process_group(None, rank, key, peer=peer, nranks=n, transport="host",
                                  timeout_s=30)
        for _ in range(3):
            comm.barrier(30)
        labels = [nd.label for nd in comm.topology.nodes]
        comm.destroy()
        q.put((rank, "ok", labels))
    except DuplicateDeviceError as exc:
        q.put((rank, "dup", (exc.rank_a, exc.rank_b)))
    except TransportUnavailableError as exc:
        q.put((rank, "net", str(exc)))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, "err", repr(exc)))


def run_host_world(n, mig_ids, hosts=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    key = f"cpu-{uuid.uuid4().hex[:10]}"
    ps = [ctx.Process(target=_host_rank, args=(r, n, key, mig_ids, q, hosts)) for r in range(n)]
    for p in ps:
        p.start()
    out = {}
    for _ in range(n):
        r, status, payload = q.get(timeout=120)
        out[r] = (status, payload)
    for p in ps:
        p.join(timeout=30)
    assert not os.path.exists(f"/dev/shm/fmx-{key}"), "segment name must be unlinked"
    return out


@pytest.mark.parametrize("n", [2, 7])
def test_multiprocess_bootstrap_labels(n):
    out = run_host_world(n, [f"GC-gpu0-{r + 1}" for r in range(n)])
    want = ["00:C0:00.0"] + [f"00:C0:00.{k}" for k in range(1, n)]
    for r in range(n):
        assert out[r] == ("ok", want)


def test_multiprocess_bootstrap_rejects_double_binding():
    out = run_host_world(3, ["MIG-a", "MIG-b", "MIG-a"])
    for r in range(3):
        assert out[r] == ("dup", (0, 2))


def test_multiprocess_bootstrap_refuses_cross_host_peers():
    """Peers on two hosts: select_transport answers NET for them (reference
    commsim.py:126-132), which the SHM transport cannot serve - every rank
    gets the same distinct error (FMX_ERR_UNSUPPORTED ->
    TransportUnavailableError), and the reference's own rule agrees."""
    from paper_2511_09143_b200.commsim import PeerInfo, select_transport
    hosts = [7, 7, 8]
    assert select_transport(PeerInfo(0, "00:C0:00.0", "a", 7, 1),
                            PeerInfo(2, "00:C0:00.0", "c", 8, 3)) == "NET"
    out = run_host_world(3, ["MIG-a", "MIG-b", "MIG-c"], hosts)
    for r in range(3):
        status, msg = out[r]
        assert status == "net", out[r]
        assert "rank 2" in msg and "NET" in msg


def test_graph_and_defer_api_argument_checks():
    """The fence / defer / graph entry points on a single-rank host-transport
    communicator (no CUDA): a host-only communicator has no device path, so
    capture, fence and flush are refused with a clear error; capture_end and
    launch_prepare validate their state and handles."""
    import ctypes

    from paper_2511_09143_b200 import _lib
    from paper_2511_09143_b200.comm import init_process_group
    from paper_2511_09143_b200.commsim import PeerInfo
    from paper_2511_09143_b200.errors import FlexShmError

    key = f"cpu-{uuid.uuid4().hex[:10]}"
    comm = init_process_group(None, 0, key, peer=PeerInfo(0, "00:C0:00.0", "MIG-x", 7, 100),
                              nranks=1, transport="host", timeout_s=30)
    L = _lib.lib()
    try:
        with pytest.raises(FlexShmError):          # host-only: no device path
            comm.capture_begin()
        with pytest.raises(FlexShmError):
            comm.fence(stream=0)
        with pytest.raises(ValueError):            # no capture is active
            comm.capture_end(0)
        with pytest.raises(FlexShmError):          # host-only, before the handle check
            _lib.check(L.fmx_graph_launch_prepare(comm._h, 3, ctypes.c_void_p(1), None))
        with pytest.raises(ValueError):            # bad handle
            _lib.check(L.fmx_graph_release(comm._h, 0))
        comm.set_defer(True)                       # no pending gather: toggles freely
        comm.set_defer(False)
        assert L.fmx_comm_flush(None, None) == _lib.FMX_ERR_INVALID_ARG
    finally:
        comm.destroy()
