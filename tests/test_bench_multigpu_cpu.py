"""The torchrun N>1 path of bench.py on CPU (gloo, world size 2): rank ->
GPU -> instance partition from fm_select, one job key for all ranks, MAX
over ranks of the step time, SUM of launches, a single JSON line from rank 0,
and the reference arm printing from rank 0 only.  --dry-run rank bodies make
no CUDA call: the 14 instance ranks of both torchrun processes join one
host-transport communicator (the real SHM bootstrap across processes) and
exchange data through their registered host regions; timings are stubs.  The
CUDA data path is covered by the -m gpu tests."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(args, nproc=2):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1",
           f"--master-port={_port()}", os.path.join(ROOT, "bench.py"), *args]
    env = {**os.environ, "OMP_NUM_THREADS": "1"}
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    return [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]


def test_two_gpu_launch_reduces_over_ranks():
    steps = 4
    lines = _torchrun(["--gpus", "2", "--steps", str(steps), "--warmup", "3", "--dry-run",
                       "--no-cpu-baseline", "--no-train"])
    assert len(lines) == 1, lines            # rank 0 alone prints
    ln = lines[0]
    assert ln["n_gpus"] == 2
    assert ln["config"]["ranks"] == 14 and ln["config"]["ranks_per_gpu"] == [7, 7]
    # stub rank r reports 10*(r+1) ms for the K steps: the line carries the max over all 14
    assert abs(ln["ms_per_step"] - 10.0 * 14 / steps) < 1e-9
    assert abs(ln["e2e"]["ms_per_step"] - 5.0 * 14 / steps) < 1e-9
    assert ln["gpu_launches"] == 14          # summed over both GPUs' instances
    # whole-job aggregate: all 14 ranks' gradients per second; algbw = one buffer's
    s_bytes = ln["config"]["bytes"]
    assert abs(ln["value"] - 14 * s_bytes / (ln["ms_per_step"] / 1e3) / 1e9) < 1e-6
    assert abs(ln["algbw_gbs"] * 14 - ln["value"]) < 1e-6
    assert ln["scaling"] == "weak"
    assert ln["step_roofline"]["link_bytes_per_gpu"]["d2h"] == 7 * ln["config"]["bytes"]
    # the cross-process exchange over the shared segment: 14 ranks, one answer
    assert ln["dry_exchange"]["ranks"] == 14 and ln["dry_exchange"]["agree"]


def test_reference_arm_prints_once_under_torchrun():
    lines = _torchrun(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1",
                       "--count", "70000"])
    assert len(lines) == 1
    assert lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
    ln = lines[0]
    assert abs(ln["value"] - 14 * 70000 * 4 / (ln["ms_per_step"] / 1e3) / 1e9) < 1e-6
    assert lines[0]["e2e"]["h2d_bytes_per_step"] == 0
