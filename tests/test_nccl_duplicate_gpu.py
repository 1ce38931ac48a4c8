"""The failure the paper starts from (reference PAPER.md:264-271): stock NCCL
refuses two ranks on one physical GPU ("Duplicate GPU detected"), which is
why the one-to-many path needs the MIG-aware bootstrap of fmx_comm_init
(tests/test_allreduce_gpu.py::test_mig_aware_rejects_double_binding shows the
legacy rule still firing on our side when mig_aware is off)."""

from __future__ import annotations

import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

CHILD = r"""
import os, sys, torch, torch.distributed as dist
rank = int(sys.argv[1])
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=rank, world_size=2, device_id=torch.device("cuda", 0))
x = torch.ones(4, device="cuda")
try:
    dist.all_reduce(x)
    torch.cuda.synchronize()
    print("ALLREDUCE_OK")
except Exception as exc:
    print("NCCL_ERROR", repr(exc)[:2000])
"""


def test_stock_nccl_rejects_two_ranks_on_one_gpu():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = {**os.environ, "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port),
           "NCCL_DEBUG": "WARN", "TORCH_NCCL_ASYNC_ERROR_HANDLING": "1"}
    procs = [subprocess.Popen([sys.executable, "-c", CHILD, str(r)], env=env, text=True,
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT) for r in range(2)]
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=180)[0])
        except subprocess.TimeoutExpired:
            p.kill()
            outs.append(p.communicate()[0])
    text = "\n".join(outs)
    assert "ALLREDUCE_OK" not in text, text[-3000:]
    assert "Duplicate GPU detected" in text, text[-3000:]
