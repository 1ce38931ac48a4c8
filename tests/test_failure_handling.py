"""Failure detection: a rank that never arrives, a rank with the
wrong world size, and abort releasing peers - on CPU over the host-only
transport, and on the GPU releasing a stream parked on a peer's flag."""

from __future__ import annotations

import multiprocessing as mp
import os
import time
import uuid

import pytest

from paper_2511_09143_b200.errors import CommAbortedError, ShmTimeoutError


def _peer(rank):
    from paper_2511_09143_b200.commsim import PeerInfo
    return PeerInfo(rank, "00:C1:00.0", f"MIG-{rank}", 7, 100 + rank)


def test_bootstrap_times_out_when_a_rank_never_arrives():
    from paper_2511_09143_b200.comm import init_process_group
    key = f"to-{uuid.uuid4().hex[:10]}"
    t0 = time.time()
    with pytest.raises(ShmTimeoutError):
        init_process_group(None, 0, key, peer=_peer(0), nranks=2, transport="host", timeout_s=1.5)
    assert time.time() - t0 < 10
    assert not os.path.exists(f"/dev/shm/fmx-{key}"), "a failed bootstrap must not leak the segment"


def _join(rank, n, key, q, action):
    from paper_2511_09143_b200.comm import init_process_group
    try:
        comm = init_process_group(None, rank, key, peer=_peer(rank), nranks=n, transport="host",
                                  timeout_s=20)
        if action == "abort":
            time.sleep(0.5)
            comm.abort()
            q.put((rank, "aborted", None))
            return
        t0 = time.time()
        comm.barrier(20)
        q.put((rank, "ok", time.time() - t0))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, type(exc).__name__, str(exc)[:200]))


def _run(specs):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    key = f"f-{uuid.uuid4().hex[:10]}"
    ps = [ctx.Process(target=_join, args=(r, n, key, q, a)) for r, n, a in specs]
    for p in ps:
        p.start()
        time.sleep(0.2)   # rank 0 creates the segment first
    out = {}
    for _ in specs:
        r, status, payload = q.get(timeout=60)
        out[r] = (status, payload)
    for p in ps:
        p.join(timeout=30)
    return out


def test_mismatched_world_size_is_rejected():
    out = _run([(0, 2, "barrier"), (1, 3, "barrier")])
    assert out[1][0] == "ValueError" and "2 ranks" in out[1][1], out
    assert out[0][0] in ("ShmTimeoutError", "ok") or "Timeout" in out[0][0], out


def test_abort_releases_a_peer_waiting_in_the_barrier():
    out = _run([(0, 2, "barrier"), (1, 2, "abort")])
    assert out[1] == ("aborted", None)
    assert out[0][0] == "CommAbortedError", out


# ---------------------------------------------------------------- GPU


def _stuck_worker(rank, job_key, n):
    """Rank 0 enqueues an allreduce that rank 1 never joins; rank 1 aborts the
    communicator.  Rank 0's stream must drain (no hang), and later calls fail."""
    import torch

    from paper_2511_09143_b200 import instance as inst_mod
    from paper_2511_09143_b200.comm import init_process_group

    inst = inst_mod.bind(0, rank + 1, mode="green")
    comm = init_process_group(None, rank, job_key, instance=inst, nranks=n, timeout_s=120)
    comm.barrier(60)
    if rank == 1:
        time.sleep(2.0)
        comm.abort()
        return {"rank": 1}
    x = torch.ones(1 << 20, device="cuda")
    t0 = time.time()
    comm.allreduce(x, stream=inst.stream)
    ev = torch.cuda.Event()
    ev.record(inst.stream)
    while not ev.query():
        if time.time() - t0 > 60:
            return {"rank": 0, "hung": True}
        time.sleep(0.01)
    released = time.time() - t0
    try:
        comm.allreduce(x, stream=inst.stream)
        after = "no error"
    except CommAbortedError:
        after = "aborted"
    return {"rank": 0, "hung": False, "released_s": released, "after": after}


@pytest.mark.gpu
def test_abort_releases_a_stream_parked_on_a_peer_flag():
    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job

    d = fm_select(Job(0, "train", 2, 0.0, 0.0), make_cluster("FM", 1))
    key = new_job_key("abort")
    res = launch(_stuck_worker, d, args=(key, 2), job_key=key, timeout_s=180)
    r0 = res[0]
    assert not r0["hung"], r0
    assert 1.0 < r0["released_s"] < 30, r0   # released by the abort, not before it
    assert r0["after"] == "aborted", r0
