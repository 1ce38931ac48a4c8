"""Model check of the SHM pipeline protocol, on a CPU, for any world size.

`fmx_trace_plan` (libflexshm) emits the exact schedule the CUDA path
enqueues for one rank - every SHM byte range it writes or reads (with the
writer/round it expects) and every flag it signals or waits on.  This test
runs all ranks' schedules under many random interleavings and checks:

* no deadlock - every rank finishes every collective;
* every read sees the bytes written by the rank and round it expects
  (no stale slot, no overwritten slot);
* no data race - every pair of conflicting SHM accesses by different ranks
  is ordered by happens-before through the flags (vector clocks: a signal
  publishes the signaller's clock, a satisfied wait joins it; stream order
  orders one rank's own operations).

This is the multi-GPU correctness argument: ranks on different GPUs run the
same schedule against the same segment; only the timing differs, and the
random scheduler explores timings.
"""

from __future__ import annotations

import random

import pytest

from paper_2511_09143_b200 import _lib


def parse(text: str):
    ops = []
    for line in text.splitlines():
        if not line or line == "#":
            continue
        f = line.split()
        if f[0] == "W":
            ops.append(("W", int(f[1]), int(f[2]), int(f[3])))
        elif f[0] == "R":
            ops.append(("R", int(f[1]), int(f[2]), int(f[3]), int(f[4])))
        elif f[0] == "S":
            ops.append(("S", int(f[1]), int(f[2])))
        elif f[0] == "A":
            ops.append(("A", int(f[1]), int(f[2]), int(f[3])))
        else:
            raise AssertionError(line)
    return ops


def geq(a: int, b: int) -> bool:
    """Cyclic 32-bit >= (CU_STREAM_WAIT_VALUE_GEQ)."""
    d = (a - b) & 0xFFFFFFFF
    return d < 0x80000000


def simulate(progs, seed: int, burst: int = 3):
    n = len(progs)
    rng = random.Random(seed)
    pc = [0] * n
    clock = [[0] * n for _ in range(n)]
    flags = {}
    last_write = {}   # off -> (rank, time, bytes, round)
    reads = {}        # off -> [(rank, time)] since last write
    starts = []
    while True:
        runnable = []
        for r in range(n):
            if pc[r] >= len(progs[r]):
                continue
            op = progs[r][pc[r]]
            if op[0] == "A":
                v, _ = flags.get((op[1], op[2]), (0, None))
                if not geq(v, op[3]):
                    continue
            runnable.append(r)
        if not runnable:
            stuck = [(r, progs[r][pc[r]]) for r in range(n) if pc[r] < len(progs[r])]
            assert not stuck, f"deadlock: {stuck[:4]}"
            return
        r = rng.choice(runnable)
        for _ in range(rng.randint(1, burst)):
            if pc[r] >= len(progs[r]):
                break
            op = progs[r][pc[r]]
            me = clock[r]
            if op[0] == "A":
                v, c = flags.get((op[1], op[2]), (0, None))
                if not geq(v, op[3]):
                    break
                if c is not None:
                    for k in range(n):
                        me[k] = max(me[k], c[k])
            elif op[0] == "S":
                me[r] += 1
                prev = flags.get((r, op[1]), (0, None))[0]
                assert geq(op[2], prev), f"rank {r} flag {op[1]} went backwards"
                flags[(r, op[1])] = (op[2], list(me))
            elif op[0] == "W":
                me[r] += 1
                _, off, nbytes, rnd = op
                lw = last_write.get(off)
                if lw is not None and lw[0] != r:
                    assert lw[1] <= me[lw[0]], f"write-write race at {off} ({lw[0]} vs {r})"
                for rr, t in reads.get(off, []):
                    if rr != r:
                        assert t <= me[rr], f"read-write race at {off}: rank {rr} read, {r} wrote"
                last_write[off] = (r, me[r], nbytes, rnd)
                reads[off] = []
                starts.append(off)
            else:  # R
                me[r] += 1
                _, off, nbytes, writer, rnd = op
                lw = last_write.get(off)
                assert lw is not None, f"rank {r} reads {off} before anyone wrote it"
                assert (lw[0], lw[3]) == (writer, rnd), (
                    f"rank {r} expected round {rnd} of rank {writer} at {off}, "
                    f"found round {lw[3]} of rank {lw[0]}")
                assert nbytes <= lw[2], f"rank {r} reads {nbytes} B, only {lw[2]} written"
                assert lw[1] <= me[lw[0]], f"read of {off} not ordered after its write"
                reads.setdefault(off, []).append((r, me[r]))
            pc[r] += 1


def programs(n, ops, slice_bytes, transport):
    ops = [o if o[0] == "allreduce" else (o[0], o[1], o[2], o[3] % n) for o in ops]
    return [parse(_lib.trace_plan(n, r, ops, slice_bytes, transport)) for r in range(n)]


SEQUENCES = {
    "allreduce-multi-round": [("allreduce", 200_003, 0), ("allreduce", 200_003, 1)],
    "mixed": [("allreduce", 50_000, 0), ("broadcast", 70_001, 0, 1), ("allreduce", 7, 1),
              ("broadcast", 5, 1, 0), ("allreduce", 123_457, 0), ("broadcast", 90_000, 0, 2),
              ("allreduce", 1, 0)],
    "broadcast-roots": [("broadcast", 40_000, 0, r % 3) for r in range(6)],
}


@pytest.mark.parametrize("transport", ["ce", "zc"])
@pytest.mark.parametrize("n", [2, 3, 7])
@pytest.mark.parametrize("seq", sorted(SEQUENCES))
def test_protocol_is_race_and_deadlock_free(n, seq, transport):
    progs = programs(n, SEQUENCES[seq], 4096, transport)
    for seed in range(12):
        simulate(progs, seed)


@pytest.mark.parametrize("n", [14, 28])
def test_protocol_multi_gpu_world_sizes(n):
    """World sizes of the 2/4-GPU configs (C4: 14 ranks; 28 = 7 x 4)."""
    ops = [("allreduce", 3 * n * 1024 + 5, 0), ("broadcast", 5000, 0, n - 1),
           ("allreduce", 999, 1)]
    progs = programs(n, ops, 4096, "ce")
    for seed in range(3):
        simulate(progs, seed, burst=8)


def test_model_catches_a_broken_schedule():
    """Sanity: drop one rank's STAGED wait and the checker must object."""
    progs = programs(3, [("allreduce", 30_000, 0)], 4096, "ce")
    victim = progs[1]
    i = next(k for k, op in enumerate(victim) if op[0] == "A" and op[2] == 0)
    broken = [victim[:i] + victim[i + 1:] if r == 1 else p for r, p in enumerate(progs)]
    failures = 0
    for seed in range(40):
        try:
            simulate(broken, seed)
        except AssertionError:
            failures += 1
    assert failures > 0
