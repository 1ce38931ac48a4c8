"""Parity of the SHM allreduce / broadcast (CUDA, through the C ABI) with the
CPU oracle: bit-exact in fp32 and bf16 under the fixed ascending-rank fp32
summation (BASELINE.json north_star), NaN-aware where inputs hold NaN.

Each launch spawns one process per rank on cuda:0 (green-context instances,
the no-MIG stand-in for 1g slices) and runs a list of scenarios through one
communicator, so the round counters and double-buffered slots are exercised
across consecutive collectives of different sizes.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as orc
from tests import _workers

pytestmark = pytest.mark.gpu

OPS = {"sum": orc.OP_SUM, "postscale": orc.OP_SUM_POSTSCALE, "prediv": orc.OP_PREDIV_SUM,
       "premul": orc.OP_PREMUL_SUM}


def expected(sc: dict, n: int) -> np.ndarray:
    xs = [_workers.make_input(r, sc) for r in range(n)]
    dt = orc.F32 if sc["dtype"] == "f32" else orc.BF16
    if sc["kind"] == "broadcast":
        return xs[sc["root"]].copy()
    if sc["kind"] == "allgather":
        return np.concatenate(xs)
    # "allreduce" and "allreduce_host" share the contract
    op = sc.get("op", "sum")
    factor = sc.get("factor")
    if op == "avg":
        op, factor = "premul", orc.ddp_mean(n)[1]
    return orc.allreduce_c(xs, dt, OPS[op], 1.0 if factor is None else factor)


def assert_same(got: np.ndarray, want: np.ndarray, what: str):
    """Bit-exact, except every NaN position must be NaN (payloads may differ)."""
    if want.dtype == np.float32:
        gnan, wnan = np.isnan(got), np.isnan(want)
        bits_g, bits_w = got.view(np.uint32), want.view(np.uint32)
    else:
        fg, fw = orc.bf16_to_f32(got), orc.bf16_to_f32(want)
        gnan, wnan = np.isnan(fg), np.isnan(fw)
        bits_g, bits_w = got, want
    assert np.array_equal(gnan, wnan), f"{what}: NaN positions differ"
    ok = gnan | (bits_g == bits_w)
    bad = np.flatnonzero(~ok)
    assert bad.size == 0, (f"{what}: {bad.size} of {got.size} elements differ, first at "
                           f"{bad[:5]}: got {got[bad[:5]]} want {want[bad[:5]]}")


def run(n: int, scenarios: list, transport: str = "auto", mode: str = "green",
        slice_bytes: int = 0, peer_override=None, host_bytes: int = 0):
    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job

    decision = fm_select(Job(0, "train", n, 0.0, 0.0), make_cluster("FM", 1 if n <= 7 else 2))
    key = new_job_key("t")
    return launch(_workers.suite_worker, decision,
                  args=(key, n, transport, mode, scenarios, slice_bytes, peer_override, host_bytes),
                  job_key=key, mode=mode, timeout_s=300, gpu_map={0: "0", 1: "0"})


def check_all(n, scenarios, results):
    for r, res in enumerate(results):
        assert "stuck" not in res, f"rank {r} hung: {res}"
        assert "results" in res, f"rank {r}: {res}"
        assert res["launches"] > 0, "no CUDA kernel launched"
    for i, sc in enumerate(scenarios):
        want_all = expected(sc, n)
        for r, res in enumerate(results):
            want = want_all
            if sc["kind"] == "reduce_scatter":  # rank r's block of the allreduce result
                c = sc["count"] // n
                want = want_all[r * c:(r + 1) * c]
            got = res["results"][i]
            if isinstance(got, str):
                assert got == _workers.digest(want), f"scenario {i} {sc} rank {r}: sha mismatch"
            else:
                assert_same(got, want, f"scenario {i} {sc} rank {r}")


BASIC = [
    dict(kind="allreduce", count=1_000_003, dtype="f32"),
    dict(kind="allreduce", count=1_000_003, dtype="f32", op="avg"),
    dict(kind="allreduce", count=333_333, dtype="f32", op="postscale", factor=0.125, inplace=False),
    dict(kind="allreduce", count=1_000_005, dtype="bf16"),
    dict(kind="allreduce", count=1_000_005, dtype="bf16", op="avg"),
    dict(kind="allreduce", count=77_777, dtype="bf16", op="postscale", factor=1 / 3),
    dict(kind="allreduce", count=1, dtype="f32"),
    dict(kind="allreduce", count=5, dtype="bf16"),
    dict(kind="allreduce", count=17, dtype="f32", op="avg"),
    dict(kind="allreduce", count=50_001, dtype="f32", offset=1),   # unaligned -> scalar path
    dict(kind="allreduce", count=40_000, dtype="f32", inputs="adversarial"),
    dict(kind="allreduce", count=40_003, dtype="bf16", inputs="adversarial"),
    dict(kind="broadcast", count=2_000_001, dtype="f32", root=0),
    dict(kind="broadcast", count=999_999, dtype="bf16", root=1),
    dict(kind="allreduce", count=2_000_000, dtype="f32", seed=99),
]


@pytest.mark.parametrize("transport", ["ce", "zc"])
def test_two_ranks_one_gpu(transport):
    scen = BASIC
    check_all(2, scen, run(2, scen, transport=transport, slice_bytes=256 << 10))


@pytest.mark.parametrize("transport", ["ce", "zc"])
def test_seven_ranks_one_gpu(transport):
    scen = BASIC + [dict(kind="broadcast", count=300_000, dtype="f32", root=6)]
    check_all(7, scen, run(7, scen, transport=transport, slice_bytes=128 << 10))


def test_resnet50_gradient_seven_ranks_bit_exact():
    """BASELINE configs C1/C2 size: 25,557,032 fp32 (ResNet-50 gradient)."""
    scen = [dict(kind="allreduce", count=25_557_032, dtype="f32", ret="sha"),
            dict(kind="allreduce", count=25_557_032, dtype="f32", op="avg", ret="sha")]
    check_all(7, scen, run(7, scen))


HOST = [
    dict(kind="allreduce_host", count=1_000_003, dtype="f32"),
    dict(kind="allreduce_host", count=1_000_003, dtype="f32", op="avg"),
    dict(kind="allreduce_host", count=500_001, dtype="bf16", op="avg", host_offset=4096),
    dict(kind="allreduce_host", count=3, dtype="f32", op="postscale", factor=0.5),
    dict(kind="allreduce", count=200_000, dtype="f32"),            # mixed with device path
    dict(kind="allreduce_host", count=40_000, dtype="f32", inputs="adversarial"),
    dict(kind="allreduce_host", count=40_003, dtype="bf16", inputs="adversarial"),
]


@pytest.mark.parametrize("n", [2, 7])
def test_host_buffer_allreduce(n):
    """Registered host buffers (fmx_allreduce_host): inputs read and results
    written straight over the host link, same bit-exact contract."""
    check_all(n, HOST, run(n, HOST, slice_bytes=128 << 10, host_bytes=8 << 20))


def test_host_buffer_resnet50_gradient_bit_exact():
    scen = [dict(kind="allreduce_host", count=25_557_032, dtype="f32", op="avg", ret="sha")]
    check_all(7, scen, run(7, scen, host_bytes=25_557_032 * 4))


def test_mig_aware_rejects_double_binding():
    res = run(2, [], peer_override={0: "same-instance", 1: "same-instance"})
    for r in res:
        assert r["init_error"] == "DuplicateDeviceError"
        assert (r["args"], r["args_b"]) == (0, 1)


def rs_ag_scenarios(n: int) -> list:
    """Reduce-scatter / all-gather: NCCL layouts, fp32 and
    bf16, aligned and ragged block sizes, in place and out of place."""
    return [
        dict(kind="reduce_scatter", count=n * 250_000, dtype="f32"),
        dict(kind="reduce_scatter", count=n * 250_001, dtype="f32", op="avg", inplace=True),
        dict(kind="reduce_scatter", count=n * 77_777, dtype="bf16", op="postscale", factor=0.5),
        dict(kind="reduce_scatter", count=n * 3, dtype="bf16", op="avg"),
        dict(kind="reduce_scatter", count=n * 40_000, dtype="f32", inputs="adversarial"),
        dict(kind="allgather", count=300_001, dtype="f32"),
        dict(kind="allgather", count=300_000, dtype="bf16", inplace=True),
        dict(kind="allgather", count=5, dtype="f32", offset=1),
        dict(kind="allreduce", count=500_001, dtype="f32", op="avg"),   # shares the round counters
        dict(kind="allgather", count=1_000_000, dtype="f32", ret="sha"),
    ]


@pytest.mark.parametrize("transport", ["ce", "zc"])
@pytest.mark.parametrize("n", [2, 7])
def test_reduce_scatter_and_allgather(n, transport):
    sc = rs_ag_scenarios(n)
    check_all(n, sc, run(n, sc, transport=transport, slice_bytes=1 << 18))


@pytest.mark.parametrize("n,mode", [(2, "green"), (7, "green"), (7, "mps")])
def test_join_stream_mode_overlapping_allreduces(n, mode):
    """DDP-bucket pattern: back-to-back allreduces of distinct buffers in
    join-stream mode (fmx_comm_set_join_stream); every result is bit-exact."""
    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job

    counts = [2_000_003, 300_000, 1_000_000, 7, 2_500_000, 640_000, 1_048_576]
    d = fm_select(Job(0, "train", n, 0.0, 0.0), make_cluster("FM", 1))
    key = new_job_key("ovl")
    res = launch(_workers.overlap_worker, d, args=(key, n, counts, mode), job_key=key,
                 timeout_s=300, mode=mode)
    for i, c in enumerate(counts):
        xs = [orc.synthetic_gradient(r, c, orc.F32, seed=500 + i) for r in range(n)]
        want = orc.allreduce_c(xs, orc.F32, *orc.ddp_mean(n))
        for r, out in enumerate(res):
            assert np.array_equal(out["results"][i].view(np.uint32), want.view(np.uint32)), (i, r)


def test_schedule_settings_follow_rank0():
    """Ranks whose environments ask for different schedules (ramp, grain,
    lanes, transport cut) still run one protocol - rank 0's, published in the
    segment header - and stay bit-exact (per-rank knobs used to
    split pieces differently and could hang)."""
    from paper_2511_09143_b200.launcher import launch, new_job_key
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job

    n = 3
    envs = {1: {"FMX_RAMP": "1", "FMX_GRAIN": "fine", "FMX_ZC_MAX": "0"},
            2: {"FMX_LANES": "2", "FMX_MIN_ROUNDS": "4", "FMX_GATHER_GRAIN": "fine"}}
    scen = [dict(kind="allreduce", count=3_000_001, dtype="f32", op="avg"),
            dict(kind="allreduce", count=1_000_003, dtype="bf16", op="sum"),
            dict(kind="allreduce", count=700_001, dtype="f32", op="sum")]
    d = fm_select(Job(0, "train", n, 0.0, 0.0), make_cluster("FM", 1))
    key = new_job_key("env")
    res = launch(_workers.mixed_env_worker, d, args=(key, n, envs, scen, 262144), job_key=key,
                 timeout_s=300)
    check_all(n, scen, res)
