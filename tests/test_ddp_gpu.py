"""DDP integration: parameters broadcast over SHM, and
every gradient bucket allreduced by ddp.flexshm_hook with DDP's default
arithmetic (bucket.div_(world) - on CUDA a multiply by fl32(1/world) - then
sum) fused into the fixed rank-order fp32 sum - bit-exact against the oracle
applied to the ranks' local gradients (tests/test_ddp_arith_gpu.py pins the
scaling against torch's own kernel)."""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import oracle as orc
from tests import _workers

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,overlap,mode,dtype", [
    (2, True, "green", "f32"), (3, True, "green", "f32"), (2, False, "green", "f32"),
    (3, True, "mps", "f32"), (3, True, "green", "bf16"), (2, True, "mps", "bf16")])
def test_ddp_hook_matches_oracle(n, overlap, mode, dtype):
    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job

    d = fm_select(Job(0, "train", n, 0.0, 0.0), make_cluster("FM", 1))
    key = new_job_key("ddp")
    port = 20000 + os.getpid() % 20000
    res = launch(_workers.ddp_worker, d, args=(key, n, port, mode, overlap, dtype), job_key=key,
                 timeout_s=300, mode=mode)
    for r in res[1:]:
        assert np.array_equal(r["params0"], res[0]["params0"]), "parameter broadcast"
    dt = orc.F32 if dtype == "f32" else orc.BF16
    want = orc.allreduce_c([r["local"] for r in res], dt, *orc.ddp_mean(n))
    bits = (lambda a: a.view(np.uint32)) if dtype == "f32" else (lambda a: a)
    for rank, r in enumerate(res):
        assert np.array_equal(bits(r["synced"]), bits(want)), rank


def test_ddp_bf16_compressed_exchange_matches_oracle():
    """flexshm_bf16_hook: fp32 buckets rounded to bf16, averaged over SHM with
    the bf16 contract, widened back - bit-exact against the oracle applied to
    the bf16-rounded local gradients."""
    import torch

    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job

    n = 3
    d = fm_select(Job(0, "train", n, 0.0, 0.0), make_cluster("FM", 1))
    key = new_job_key("ddpc")
    port = 21000 + os.getpid() % 20000
    res = launch(_workers.ddp_worker, d, args=(key, n, port, "green", True, "f32", "bf16"),
                 job_key=key, timeout_s=300)
    locals_bf16 = [torch.from_numpy(r["local"]).to(torch.bfloat16).view(torch.int16).numpy()
                   .view(np.uint16) for r in res]
    want = orc.allreduce_c(locals_bf16, orc.BF16, *orc.ddp_mean(n))
    want_f32 = orc.bf16_to_f32(want)
    for rank, r in enumerate(res):
        assert np.array_equal(r["synced"].view(np.uint32), want_f32.view(np.uint32)), rank


@pytest.mark.parametrize("n", [2, 5])
def test_zero_shard_sync_broadcast_and_allgather(n):
    """ZeRO parameter re-sync: after each rank writes only the
    shard it owns, both flavours leave every rank with every owner's values."""
    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job

    d = fm_select(Job(0, "train", n, 0.0, 0.0), make_cluster("FM", 1))
    key = new_job_key("zero")
    res = launch(_workers.zero_worker, d, args=(key, n), job_key=key, timeout_s=300)
    sizes = [300 * 7, 11, 64 * 64, 5 * 3 * 3, 1000]
    want_b = np.concatenate([np.full(k, o + 1.0, np.float32)
                             for k, o in zip(sizes, res[0]["owner"])])
    c = res[0]["block"]
    want_flat = np.concatenate([np.full(c, q + 1.0, np.float32) for q in range(n)])
    for r, out in enumerate(res):
        assert np.array_equal(out["bcast"], want_b), r
        assert np.array_equal(out["flat"], want_flat), r
        assert np.array_equal(out["params"], want_flat[:sum(sizes)]), r


@pytest.mark.parametrize("mode", ["green", "mps"])
def test_ddp_threaded_hook_matches_oracle(mode):
    """The enqueue-thread variant of the hook (collectives issued off the
    autograd thread) is bit-exact too."""
    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job

    n = 3
    d = fm_select(Job(0, "train", n, 0.0, 0.0), make_cluster("FM", 1))
    key = new_job_key("ddpt")
    port = 22000 + os.getpid() % 20000
    res = launch(_workers.ddp_worker, d, args=(key, n, port, mode, True, "f32", None, True),
                 job_key=key, timeout_s=300, mode=mode)
    want = orc.allreduce_c([r["local"] for r in res], orc.F32, *orc.ddp_mean(n))
    for rank, r in enumerate(res):
        assert np.array_equal(r["synced"].view(np.uint32), want.view(np.uint32)), rank
