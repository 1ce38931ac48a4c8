"""DDP's mean, pinned against torch itself on the B200.

DDP's default comm hook scales a bucket with `tensor.div_(world)` and then
SUM-allreduces it (torch/distributed/algorithms/ddp_comm_hooks/
default_hooks.py:26).  On CUDA, ATen computes a division by a CPU scalar as a
multiplication by its fp32 reciprocal (div_true_kernel_cuda,
aten/src/ATen/native/cuda/BinaryDivTrueKernel.cu), so op="avg" is
FMX_OP_PREMUL_SUM with factor fl32(1/n), not an IEEE division.  These tests
check that claim against torch's own CUDA kernel, and that the SHM DDP hook
equals "torch's div_ on every rank, then the fixed rank-order fp32 sum" bit for
bit.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import oracle as orc
from tests import _workers

pytestmark = pytest.mark.gpu


def _inputs(dtype: int, count: int) -> np.ndarray:
    x = np.concatenate([orc.synthetic_gradient(3, count, dtype),
                        orc.adversarial(1, 4099, dtype)])
    return x


@pytest.mark.parametrize("dtype", [orc.F32, orc.BF16])
@pytest.mark.parametrize("n", [2, 3, 5, 7, 14, 28, 56])
def test_torch_cuda_div_is_premul_by_fp32_reciprocal(dtype, n):
    import torch
    x = _inputs(dtype, 1_000_003)
    t = torch.from_numpy(x.view(np.float32) if dtype == orc.F32 else x.view(np.int16))
    t = t.cuda() if dtype == orc.F32 else t.cuda().view(torch.bfloat16)
    t.div_(n)                                      # what default_hooks.py:26 runs
    torch.cuda.synchronize()
    got = t.cpu()
    got = got.numpy() if dtype == orc.F32 else got.view(torch.int16).numpy().view(np.uint16)
    want = orc.allreduce_c([x], dtype, *orc.ddp_mean(n))   # one source: x * fl32(1/n)
    fa = got if dtype == orc.F32 else orc.bf16_to_f32(got)
    nan = np.isnan(fa)
    bits = (lambda a: a.view(np.uint32)) if dtype == orc.F32 else (lambda a: a)
    assert np.array_equal(nan, np.isnan(want if dtype == orc.F32 else orc.bf16_to_f32(want)))
    assert np.array_equal(bits(got)[~nan], bits(want)[~nan])
    if dtype == orc.F32 and n in (3, 7, 14, 28, 56):
        # the test has teeth: IEEE division rounds differently on many inputs
        div = orc.allreduce_c([x], dtype, orc.OP_PREDIV_SUM, float(n))
        assert np.count_nonzero(bits(div)[~nan] != bits(want)[~nan]) > 0


@pytest.mark.parametrize("n,mode,dtype", [(7, "mps", "f32"), (3, "green", "bf16")])
def test_ddp_hook_equals_torch_div_then_rank_order_sum(n, mode, dtype):
    """Every rank computes its local gradient and torch's own `div_(n)` of it
    on the GPU; the oracle SUMs those in rank order; the SHM hook's bucket
    (op="avg") must equal that bit for bit on every rank."""
    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job

    d = fm_select(Job(0, "train", n, 0.0, 0.0), make_cluster("FM", 1))
    key = new_job_key("ddpa")
    port = 23000 + os.getpid() % 20000
    res = launch(_workers.ddp_worker, d, args=(key, n, port, mode, True, dtype), job_key=key,
                 timeout_s=300, mode=mode)
    dt = orc.F32 if dtype == "f32" else orc.BF16
    want = orc.allreduce_c([r["local_div"] for r in res], dt, orc.OP_SUM)
    # the same thing restated by the oracle's DDP-mean op from the raw local gradients
    assert np.array_equal(orc.allreduce_c([r["local"] for r in res], dt, *orc.ddp_mean(n)), want)
    bits = (lambda a: a.view(np.uint32)) if dtype == "f32" else (lambda a: a)
    for rank, r in enumerate(res):
        assert np.array_equal(bits(r["synced"]), bits(want)), rank
