"""Parity of the one-shot small-message allreduce (plan_allreduce_oneshot,
taken by AUTO / ZC up to FMX_ONESHOT_MAX = 64 KiB) with the CPU oracle on the
B200: every rank reduces all n published buffers in ascending rank order, so
the result must be the same bits as the pipelined path's owner reduction.

Back-to-back calls cycle the two alternating slots many times, interleaved with
pipelined allreduces and broadcasts (separate slots and round counters)."""

from __future__ import annotations

import pytest

from tests.test_allreduce_gpu import check_all, run

pytestmark = pytest.mark.gpu

SMALL = [
    dict(kind="allreduce", count=1, dtype="f32"),
    dict(kind="allreduce", count=256, dtype="f32", op="avg"),
    dict(kind="allreduce", count=257, dtype="bf16", op="avg"),
    dict(kind="allreduce", count=3, dtype="bf16"),
    dict(kind="allreduce", count=1000, dtype="f32", op="postscale", factor=0.125, inplace=False),
    dict(kind="allreduce", count=999, dtype="f32", op="prediv", factor=7.0),
    dict(kind="allreduce", count=4_097, dtype="f32", offset=1),          # unaligned: scalar path
    dict(kind="allreduce", count=4_000, dtype="f32", inputs="adversarial"),
    dict(kind="allreduce", count=4_003, dtype="bf16", inputs="adversarial"),
    dict(kind="allreduce", count=16_384, dtype="f32", seed=3),            # exactly 64 KiB
    dict(kind="allreduce", count=32_768, dtype="bf16", op="avg", seed=4),  # exactly 64 KiB
    dict(kind="allreduce", count=16_385, dtype="f32", seed=5),            # one over: pipelined
    dict(kind="broadcast", count=1000, dtype="f32", root=1),
    dict(kind="allreduce", count=8, dtype="f32", seed=6),
    dict(kind="allreduce", count=300_000, dtype="f32", seed=7),           # pipelined, CE
    dict(kind="allreduce", count=12, dtype="bf16", op="avg", seed=8),
    dict(kind="allreduce", count=100, dtype="f32", op="premul", factor=0.5, seed=9),
]


@pytest.mark.parametrize("n,mode", [(2, "green"), (7, "mps"), (7, "green")])
def test_oneshot_allreduce_bit_exact(n, mode):
    check_all(n, SMALL, run(n, SMALL, transport="auto", mode=mode))


def test_oneshot_many_back_to_back():
    """40 one-shot calls in a row at 7 ranks: each slot is reused 20 times."""
    scen = [dict(kind="allreduce", count=64 + 37 * i, dtype="f32" if i % 3 else "bf16",
                 op="avg" if i % 2 else "sum", seed=100 + i) for i in range(40)]
    check_all(7, scen, run(7, scen, transport="auto", mode="mps"))
