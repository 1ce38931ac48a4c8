"""The BASELINE configs at their own shapes and rank splits (BASELINE.json
configs[2], configs[3]), bit-exact against the oracle on the B200.

One box has one GPU, so the 2-GPU splits run as two *logical* GPUs of the one
B200: every rank is an MPS client of the physical device, and the ranks of
logical GPU g publish the synthetic bus id F<g>:00:00.0 (FMX_FAKE_BUS), so the
communicator, the rank order (fm_select round-robin over the GPUs, reference
scheduler.py:117-136) and the MIG-aware bootstrap are exactly those of a
2-GPU job.  All traffic crosses the one PCIe link.
"""

from __future__ import annotations

import pytest

from tests import _workers
from tests.test_allreduce_gpu import check_all

pytestmark = pytest.mark.gpu


def run_split(monkeypatch, n: int, gpus: int, want_split: list, scenarios: list):
    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job

    monkeypatch.setenv("FMX_FAKE_BUS", "1")
    d = fm_select(Job(0, "train", n, 0.0, 0.0), make_cluster("FM", gpus))
    split = [sum(1 for g, _ in d.instances if g == gg) for gg in range(gpus)]
    assert split == want_split, split
    key = new_job_key("cfg")
    return launch(_workers.suite_worker, d, args=(key, n, "auto", "mps", scenarios), job_key=key,
                  mode="mps", timeout_s=900, gpu_map={g: "0" for g in range(gpus)})


def test_c4_bert_base_bf16_14_ranks_on_2_gpus(monkeypatch):
    """configs[3]: the BERT-base gradient, 109,483,778 bf16, over 14 instances
    on 2 GPUs (7+7), DDP mean and plain sum, sha256-exact."""
    count = 109_483_778
    scen = [dict(kind="allreduce", count=count, dtype="bf16", op="avg", ret="sha"),
            dict(kind="allreduce", count=count, dtype="bf16", op="sum", ret="sha", seed=77)]
    res = run_split(monkeypatch, 14, 2, [7, 7], scen)
    check_all(14, scen, res)


def test_c3_mobilenet_v2_fp32_4_ranks_on_2_gpus(monkeypatch):
    """configs[2]: the MobileNetV2 gradient, 3,504,872 fp32, over 4 instances
    on 2 GPUs (2+2): DDP mean, sum, and the init broadcast."""
    count = 3_504_872
    scen = [dict(kind="allreduce", count=count, dtype="f32", op="avg"),
            dict(kind="allreduce", count=count, dtype="f32", op="sum", seed=5),
            dict(kind="broadcast", count=count, dtype="f32", root=3)]
    res = run_split(monkeypatch, 4, 2, [2, 2], scen)
    check_all(4, scen, res)
