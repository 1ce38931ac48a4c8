"""Randomised soak test: a seeded program of allreduce / reduce-scatter /
all-gather / broadcast calls (fp32 and bf16, all ops, ragged sizes, in and out
of place, some in join-stream mode) run by 7 MPS ranks and 3 green-context
ranks through one communicator each; every result is checked bit for bit
against the oracle (sha256)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as orc
from tests import _workers

pytestmark = pytest.mark.gpu

OPS = {"sum": orc.OP_SUM, "postscale": orc.OP_SUM_POSTSCALE, "prediv": orc.OP_PREDIV_SUM,
       "premul": orc.OP_PREMUL_SUM}


def expected_digest(o: dict, n: int, rank: int) -> str:
    xs = [_workers.stress_input(r, o, n) for r in range(n)]
    dt = orc.F32 if o["dtype"] == "f32" else orc.BF16
    if o["kind"] == "broadcast":
        return _workers.digest(xs[o["root"]])
    if o["kind"] == "allgather":
        return _workers.digest(np.concatenate(xs))
    op, factor = o["op"], (0.25 if o["op"] == "postscale" else 1.0)
    if op == "avg":
        op, factor = "premul", orc.ddp_mean(n)[1]
    full = orc.allreduce_c(xs, dt, OPS[op], factor)
    if o["kind"] == "reduce_scatter":
        c = o["size"]
        return _workers.digest(full[rank * c:(rank + 1) * c])
    return _workers.digest(full)


@pytest.mark.parametrize("n,mode,seed", [(7, "mps", 1), (3, "green", 2),
                                         (2, "mps", 4)])   # two ranks: the fetch-lane schedule
def test_random_collective_program_is_bit_exact(n, mode, seed):
    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job

    nops = 60
    d = fm_select(Job(0, "train", n, 0.0, 0.0), make_cluster("FM", 1))
    key = new_job_key("stress")
    res = launch(_workers.stress_worker, d, args=(key, n, seed, nops, mode), job_key=key,
                 timeout_s=600, mode=mode)
    ops = _workers.stress_ops(n, seed, nops)
    for i, o in enumerate(ops):
        for r in range(n):
            want = expected_digest(o, n, r)
            assert res[r]["digests"][i] == want, (i, o, r)


@pytest.mark.parametrize("n,gpus", [(14, 2), (28, 4)])
def test_wide_communicators_on_logical_gpus(monkeypatch, n, gpus):
    """The 2- and 4-GPU world sizes (14 and 28 ranks, fm_select round-robin
    order over the GPUs) run on one B200: every logical GPU's seven instances
    are MPS clients of the physical device, with distinct synthetic bus ids
    (FMX_FAKE_BUS).  The random program must stay bit-exact."""
    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job

    monkeypatch.setenv("FMX_FAKE_BUS", "1")
    nops, seed = 16, 3 + n
    d = fm_select(Job(0, "train", n, 0.0, 0.0), make_cluster("FM", gpus))
    assert len({g for g, _ in d.instances}) == gpus
    key = new_job_key("wide")
    res = launch(_workers.stress_worker, d, args=(key, n, seed, nops, "mps"), job_key=key,
                 timeout_s=900, mode="mps", gpu_map={g: "0" for g in range(gpus)})
    ops = _workers.stress_ops(n, seed, nops)
    for i, o in enumerate(ops):
        for r in range(n):
            assert res[r]["digests"][i] == expected_digest(o, n, r), (i, o, r)


@pytest.mark.parametrize("n,mode,seed,slice_bytes,sticky", [
    (3, "mps", 5, 0, False), (2, "mps", 6, 64 << 10, False), (7, "mps", 7, 0, False),
    # deferral switched on at the first join-stream call and left on for every
    # later call, whatever its kind (one-shots, broadcasts, ... flush it)
    (3, "mps", 5, 0, True)])
def test_random_program_as_a_captured_graph(n, mode, seed, slice_bytes, sticky):
    """The random program (every collective, dtype and op; join-stream allreduces
    with deferred gathers) captured once as a CUDA graph and replayed three times
    with fresh inputs: every replay's every result bit-exact against the oracle."""
    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job

    nops, replays = (16, 2) if n >= 7 else (24, 3)   # (the suite's runtime budget)
    d = fm_select(Job(0, "train", n, 0.0, 0.0), make_cluster("FM", 1))
    key = new_job_key("gstress")
    res = launch(_workers.graph_stress_worker, d,
                 args=(key, n, seed, nops, replays, mode, slice_bytes, sticky), job_key=key,
                 timeout_s=600, mode=mode)
    ops = _workers.stress_ops(n, seed, nops)
    for rep in range(replays):
        for i, o in enumerate(ops):
            o_r = dict(o, seed=o["seed"] + 100_000 * rep)
            for r in range(n):
                assert res[r]["digests"][rep][i] == expected_digest(o_r, n, r), (rep, i, o, r)
