"""ddp.ShmDataParallel and the captured-graph path (fmx_graph_*): a whole DP
training step with its bucket allreduces captured as one CUDA graph and
replayed, flag values re-based per replay by the library.

Checked: the first step's averaged gradient is the oracle's rank-order
DDP mean of the ranks' local gradients (bit-exact); the graph-replayed
training ends bit-identical to the same steps run eagerly, on every rank;
an eager allreduce between two replays (fence + counter continuity) is exact;
gradient accumulation under no_sync exchanges the DDP mean of the
accumulated local gradients; the SGD step fused into the collective
(fused_sgd / fmx_allreduce_sgd: owners step their chunk, the all-gather moves
parameters) ends bit-identical to torch.optim.SGD on every rank - momentum,
and weight decay + Nesterov - eager and replayed as a graph."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as orc
from tests import _workers

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,mode,defer,compress", [
    (2, "mps", True, None), (3, "mps", True, None), (3, "green", True, None),
    (3, "mps", False, None), (3, "mps", True, "bf16")])
def test_graphed_dp_matches_eager_and_oracle(n, mode, defer, compress):
    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job

    d = fm_select(Job(0, "train", n, 0.0, 0.0), make_cluster("FM", 1))
    key = new_job_key("gdp")
    res = launch(_workers.graph_dp_worker, d, args=(key, n, mode, defer, compress), job_key=key,
                 timeout_s=300,
                 mode=mode)
    assert res[0]["buckets"] >= 3
    if compress == "bf16":   # bf16 contract on the bf16-rounded local gradients, widened
        import torch
        loc = [torch.from_numpy(r["local"]).to(torch.bfloat16).view(torch.int16).numpy()
               .view(np.uint16) for r in res]
        want = orc.bf16_to_f32(orc.allreduce_c(loc, orc.BF16, *orc.ddp_mean(n)))
    else:
        want = orc.allreduce_c([r["local"] for r in res], orc.F32, *orc.ddp_mean(n))
    extra = [np.arange(1000, dtype=np.float32) * (r + 1) for r in range(n)]
    want_extra = orc.allreduce_c(extra, orc.F32, orc.OP_SUM)
    if compress == "bf16":
        loc = [torch.from_numpy(r["local_acc"]).to(torch.bfloat16).view(torch.int16).numpy()
               .view(np.uint16) for r in res]
        want_acc = orc.bf16_to_f32(orc.allreduce_c(loc, orc.BF16, *orc.ddp_mean(n)))
    else:
        want_acc = orc.allreduce_c([r["local_acc"] for r in res], orc.F32, *orc.ddp_mean(n))
    for rank, r in enumerate(res):
        assert np.array_equal(r["synced"].view(np.uint32), want.view(np.uint32)), rank
        assert np.array_equal(r["synced_acc"].view(np.uint32), want_acc.view(np.uint32)), rank
        if compress is None:   # the optimizer fused into the collective == torch SGD per rank
            assert np.array_equal(r["params_fused"].view(np.uint32),
                                  r["params_eager"].view(np.uint32)), rank
            assert np.array_equal(r["params_wd_fused"].view(np.uint32),
                                  r["params_wd_torch"].view(np.uint32)), rank
        assert np.array_equal(r["params_graph"].view(np.uint32),
                              r["params_eager"].view(np.uint32)), rank
        assert np.array_equal(r["params_graph"].view(np.uint32),
                              res[0]["params_graph"].view(np.uint32)), rank
        assert np.array_equal(r["extra"].view(np.uint32), want_extra.view(np.uint32)), rank


@pytest.mark.parametrize("n,mode,transport,slice_bytes", [
    (3, "mps", "auto", 0), (2, "green", "auto", 0),
    # copy engines in many small rounds: the two-rank fetch lane + copy-engine result
    # slot, and the three-rank pipeline, inside captured graphs
    (2, "mps", "ce", 64 << 10), (3, "mps", "ce", 64 << 10)])
def test_graph_api_and_deferred_gathers(n, mode, transport, slice_bytes):
    """The raw API: deferred gathers + flush (bit-exact, pending-gather guard);
    two captured graphs replayed on different streams with an eager collective
    on a third stream in between, fresh inputs each replay - every result
    bit-exact against the oracle."""
    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job

    d = fm_select(Job(0, "train", n, 0.0, 0.0), make_cluster("FM", 1))
    key = new_job_key("gapi")
    res = launch(_workers.graph_api_worker, d, args=(key, n, mode, transport, slice_bytes),
                 job_key=key, timeout_s=300, mode=mode)
    bits = lambda a: a.view(np.uint32)
    sizes = [300_001, 1000, 40_000]
    for i, c in enumerate(sizes):
        want = orc.allreduce_c([orc.synthetic_gradient(r, c, orc.F32, seed=50 + i)
                                for r in range(n)], orc.F32, orc.OP_SUM)
        for r in res:
            assert np.array_equal(bits(r["defer"][i]), bits(want)), (i, c)
    assert all(r["defer_raised"] for r in res)
    def gen(r, c, seed, key):
        return orc.synthetic_gradient(r, c, orc.F32, seed=seed + _workers.GRAPH_API_SEED[key])
    for step in range(len(res[0]["graphs"])):
        what, seed = res[0]["graphs"][step][:2]
        if what == "eager":
            want = orc.allreduce_c([orc.synthetic_gradient(r, 77_777, orc.F32, seed=seed)
                                    for r in range(n)], orc.F32, orc.OP_SUM)
            for r in res:
                assert np.array_equal(bits(r["graphs"][step][2]), bits(want)), step
        elif what == "G1":
            want = orc.allreduce_c([gen(r, 200_003, seed, "big") for r in range(n)], orc.F32,
                                   *orc.ddp_mean(n))
            want_bc = gen(n - 1, 3000, seed, "bc")
            for r in res:
                assert np.array_equal(bits(r["graphs"][step][2]), bits(want)), step
                assert np.array_equal(bits(r["graphs"][step][3]), bits(want_bc)), step
        else:
            want = orc.allreduce_c([gen(r, 5, seed, "small") for r in range(n)], orc.F32,
                                   orc.OP_SUM)
            full = orc.allreduce_c([gen(r, n * 999, seed, "rs") for r in range(n)], orc.F32,
                                   orc.OP_SUM)
            for rank, r in enumerate(res):
                assert np.array_equal(bits(r["graphs"][step][2]), bits(want)), step
                assert np.array_equal(bits(r["graphs"][step][3]),
                                      bits(full[rank * 999:(rank + 1) * 999])), step


@pytest.mark.parametrize("n,count,transport,slice_bytes", [
    (2, 3_000_001, "ce", 64 << 10),   # two ranks: fetch lane + copy-engine result (>= 8 rounds)
    (3, 1_000_003, "ce", 64 << 10),   # multi-round copy-engine pipeline
    (3, 100_003, "zc", 0),            # zero-copy: the reduction reads the slots itself
    (1, 10_007, "auto", 0)])          # one rank: the step alone
def test_fused_sgd_flat_buffer_matches_torch_sgd(n, count, transport, slice_bytes):
    """fmx_allreduce_sgd (weight decay, dampened momentum) over three steps on
    every transport / schedule: bit-identical to allreduce(avg) + torch SGD."""
    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job

    d = fm_select(Job(0, "train", n, 0.0, 0.0), make_cluster("FM", 1))
    key = new_job_key("fsgd")
    res = launch(_workers.fused_sgd_worker, d, args=(key, n, count, transport, slice_bytes),
                 job_key=key, timeout_s=300, mode="mps")
    for rank, r in enumerate(res):
        assert np.array_equal(r["fused"].view(np.uint32), r["torch"].view(np.uint32)), rank
        assert np.array_equal(r["fused"].view(np.uint32), res[0]["fused"].view(np.uint32)), rank
