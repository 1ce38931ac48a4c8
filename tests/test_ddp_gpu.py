"""DDP integration: parameters broadcast over SHM, and
every gradient bucket allreduced by ddp.flexshm_hook with DDP's default
arithmetic (divide by world size, then sum) fused into the fixed rank-order
fp32 sum - bit-exact against the oracle applied to the ranks' local
gradients."""

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
    want = orc.allreduce_c([r["local"] for r in res], dt, orc.OP_PREDIV_SUM, float(n))
    bits = (lambda a: a.view(np.uint32)) if dtype == "f32" else (lambda a: a)
    for rank, r in enumerate(res):
        assert np.array_equal(bits(r["synced"]), bits(want)), rank
