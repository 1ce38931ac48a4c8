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


LANES = 3  # 0 stage (D2H), 1 fetch + reduce (the caller's stream), 2 gather (H2D)


def parse(text: str, merged: bool = False):
    """-> [lane0 ops, lane1 ops, lane2 ops]; a 'J' line is a join point in
    every lane.  merged=True reads the trace as ONE sequential program in
    enqueue order - what the hardware runs if the driver puts all lane streams
    on one FIFO."""
    lanes = [[] for _ in range(LANES)]
    joins = 0
    for line in text.splitlines():
        if not line:
            continue
        if merged:
            if line != "J":
                f = line.split()
                lanes[0].append((f[1], *[int(x) for x in f[2:]]))
            continue
        if line == "J":
            for ops in lanes:
                ops.append(("J", joins))
            joins += 1
            continue
        f = line.split()
        lane, kind, rest = int(f[0]), f[1], [int(x) for x in f[2:]]
        lanes[lane].append((kind, *rest))
    return lanes


def geq(a: int, b: int) -> bool:
    """Cyclic 32-bit >= (CU_STREAM_WAIT_VALUE_GEQ)."""
    d = (a - b) & 0xFFFFFFFF
    return d < 0x80000000


def simulate(progs, seed: int, burst: int = 3):
    """progs[rank] = [lane0, lane1, lane2].  Actors are (rank, lane) pairs,
    each a sequential program (one CUDA stream); lanes of a rank meet at joins."""
    n = len(progs)
    actors = [(r, l) for r in range(n) for l in range(LANES)]
    idx = {a: i for i, a in enumerate(actors)}
    m = len(actors)
    rng = random.Random(seed)
    pc = {a: 0 for a in actors}
    clock = {a: [0] * m for a in actors}
    flags = {}
    events = {}       # (rank, event id, seq) -> clock at record
    last_write = {}   # key -> (actor, time, bytes, round)
    reads = {}        # key -> [(actor, time)] since last write

    def op_of(a):
        prog = progs[a[0]][a[1]]
        return prog[pc[a]] if pc[a] < len(prog) else None

    def ready(a):
        op = op_of(a)
        if op is None:
            return False
        if op[0] == "A":
            return geq(flags.get((op[1], op[2]), (0, None))[0], op[3])
        if op[0] == "J":
            return all(op_of((a[0], l)) == op for l in range(LANES))
        if op[0] == "X":
            return (a[0], op[1], op[2]) in events
        return True

    def hb(prev_actor, prev_time, me):
        return prev_time <= clock[me][idx[prev_actor]]

    def access(a, key, nbytes, write, expect=None):
        me = clock[a]
        me[idx[a]] += 1
        lw = last_write.get(key)
        if write:
            if lw is not None and lw[0] != a:
                assert hb(lw[0], lw[1], a), f"write-write race on {key}: {lw[0]} vs {a}"
            for ra, t in reads.get(key, []):
                if ra != a:
                    assert hb(ra, t, a), f"read-write race on {key}: {ra} read, {a} wrote"
            last_write[key] = (a, me[idx[a]], nbytes, expect)
            reads[key] = []
        else:
            if expect is not None:
                assert lw is not None, f"{a} reads {key} before anyone wrote it"
                assert (lw[0][0], lw[3]) == expect, (
                    f"{a} expected {expect} at {key}, found round {lw[3]} of rank {lw[0][0]}")
                assert nbytes <= lw[2], f"{a} reads {nbytes} B of {key}, only {lw[2]} written"
            if lw is not None and lw[0] != a:
                assert hb(lw[0], lw[1], a), f"read of {key} not ordered after its write"
            reads.setdefault(key, []).append((a, me[idx[a]]))

    while True:
        runnable = [a for a in actors if ready(a)]
        if not runnable:
            stuck = [(a, op_of(a)) for a in actors if op_of(a) is not None]
            assert not stuck, f"deadlock: {stuck[:4]}"
            return
        a = rng.choice(runnable)
        for _ in range(rng.randint(1, burst)):
            if not ready(a):
                break
            op = op_of(a)
            me = clock[a]
            r = a[0]
            if op[0] == "A":
                c = flags.get((op[1], op[2]), (0, None))[1]
                if c is not None:
                    for k in range(m):
                        me[k] = max(me[k], c[k])
            elif op[0] == "J":
                others = [(r, l) for l in range(LANES) if l != a[1]]
                joined = [max(xs) for xs in zip(me, *(clock[o] for o in others))]
                clock[a][:] = joined
                for o in others:
                    clock[o][:] = joined
                    pc[o] += 1
            elif op[0] == "E":
                me[idx[a]] += 1
                events[(r, op[1], op[2])] = list(me)
            elif op[0] == "X":
                c = events[(r, op[1], op[2])]
                for k in range(m):
                    me[k] = max(me[k], c[k])
            elif op[0] == "S":
                me[idx[a]] += 1
                prev = flags.get((r, op[1]), (0, None))[0]
                assert geq(op[2], prev), f"rank {r} flag {op[1]} went backwards"
                flags[(r, op[1])] = (op[2], list(me))
            elif op[0] == "W":
                access(a, ("shm", op[1]), op[2], True, op[3])
            elif op[0] == "R":
                access(a, ("shm", op[1]), op[2], False, (op[3], op[4]))
            elif op[0] == "UW":
                access(a, ("user", r, op[1]), op[2], True)
            elif op[0] == "UR":
                access(a, ("user", r, op[1]), op[2], False)
            elif op[0] == "SW":   # the rank's HBM scratch (host path slots, CE fetch slots)
                access(a, ("scratch", r, op[1]), op[2], True)
            elif op[0] == "SR":
                access(a, ("scratch", r, op[1]), op[2], False)
            else:
                raise AssertionError(op)
            pc[a] += 1


def programs(n, ops, slice_bytes, transport, merged=False):
    ops = [o if o[0] != "broadcast" else (o[0], o[1], o[2], o[3] % n) for o in ops]
    return [parse(_lib.trace_plan(n, r, ops, slice_bytes, transport), merged) for r in range(n)]


SEQUENCES = {
    "host-buffer": [("allreduce_host", 90_001, 0), ("allreduce_host", 5, 1),
                    ("allreduce", 30_000, 0), ("allreduce_host", 40_000, 1),
                    ("broadcast", 9_000, 0, 1), ("allreduce_host", 123_456, 0)],
    "allreduce-multi-round": [("allreduce", 200_003, 0), ("allreduce", 200_003, 1)],
    "mixed": [("allreduce", 50_000, 0), ("broadcast", 70_001, 0, 1), ("allreduce", 7, 1),
              ("broadcast", 5, 1, 0), ("allreduce", 123_457, 0), ("broadcast", 90_000, 0, 2),
              ("allreduce", 1, 0)],
    "broadcast-roots": [("broadcast", 40_000, 0, r % 3) for r in range(6)],
    "rs-ag": [("reduce_scatter", 30_001, 0), ("allgather", 20_000, 1), ("allreduce", 50_000, 0),
              ("allgather", 3, 0), ("reduce_scatter", 70_000, 1), ("broadcast", 9_000, 0, 1),
              ("reduce_scatter", 1, 0), ("allgather", 45_000, 0)],
}


@pytest.mark.parametrize("transport", ["ce", "zc"])
@pytest.mark.parametrize("n", [2, 3, 7])
@pytest.mark.parametrize("seq", sorted(SEQUENCES))
def test_protocol_is_race_and_deadlock_free(n, seq, transport):
    progs = programs(n, SEQUENCES[seq], 4096, transport)
    for seed in range(12):
        simulate(progs, seed)


@pytest.mark.parametrize("n", [2, 3, 7])
@pytest.mark.parametrize("seq", sorted(SEQUENCES))
def test_enqueue_order_is_a_valid_single_stream_schedule(n, seq):
    """If the driver serialises a rank's two lane streams onto one hardware
    FIFO, the rank executes its trace in enqueue order: that must not deadlock
    either (the bug a first two-lane version hit on the B200)."""
    progs = programs(n, SEQUENCES[seq], 4096, "ce", merged=True)
    for seed in range(8):
        simulate(progs, seed)


@pytest.mark.parametrize("n", [14, 28])
def test_protocol_multi_gpu_world_sizes(n):
    """World sizes of the 2/4-GPU configs (C4: 14 ranks; 28 = 7 x 4)."""
    ops = [("allreduce", 3 * n * 1024 + 5, 0), ("broadcast", 5000, 0, n - 1),
           ("allreduce", 999, 1)]
    progs = programs(n, ops, 4096, "ce")
    for seed in range(3):
        simulate(progs, seed, burst=8)


def default_slice(n: int, slots: int = 2) -> int:
    """fmx_comm_init's default slice (flexshm_comm.cu default_slice_cap /
    segment_budget): min(cap, budget / (K (n^2 + 2n))), floored to 4 KiB."""
    cap = (16 << 20) if n <= 2 else (4 << 20)
    budget = (2 << 30) if n > 14 else (1 << 30)
    sb = min(cap, budget // (slots * (n * n + 2 * n)))
    return max(4096, sb // 4096 * 4096)


@pytest.mark.parametrize("n,ops", [
    # C4 at its own shape: BERT-base bf16 gradient over 14 ranks (2 GPUs, 7+7)
    (14, [("allreduce", 109_483_778, 1), ("allreduce", 25_557_032, 0)]),
    # C3: MobileNetV2 fp32 gradient over 4 ranks (2+2)
    (4, [("allreduce", 3_504_872, 0), ("broadcast", 3_504_872, 0, 3)]),
    # 8 GPUs x 7 instances: the north_star's top configuration, ResNet-50 and
    # BERT-base gradients with the 56-rank default slice (320 KiB)
    (56, [("allreduce", 25_557_032, 0), ("allreduce", 109_483_778, 1)]),
])
def test_protocol_at_baseline_config_shapes(n, ops):
    """The BASELINE configs' own message sizes, world sizes and default slice
    geometry (not a shrunken slice): race-, stale-read- and deadlock-free."""
    sb = default_slice(n)
    if n == 56:
        assert sb == 320 << 10
    progs = programs(n, ops, sb, "auto")
    for seed in range(1 if n == 56 else 2):
        simulate(progs, seed, burst=8)


def test_model_catches_a_broken_host_schedule():
    """Drop the REDUCED wait at the end of a host-buffer allreduce: the next
    call's host write of the input races with a slow owner's result write."""
    progs = programs(3, [("allreduce_host", 60_000, 0), ("allreduce_host", 60_000, 0)], 4096, "ce")
    lanes = progs[1]
    broken_lanes = [[op for op in lane if not (op[0] == "A" and op[2] == 1)] for lane in lanes]
    broken = [broken_lanes if r == 1 else p for r, p in enumerate(progs)]
    failures = 0
    for seed in range(60):
        try:
            simulate(broken, seed)
        except AssertionError:
            failures += 1
    assert failures > 0


STAGED_TO = 8   # kStagedTo: per-(contributor, owner) flags start here
REDUCED = 1


@pytest.mark.parametrize("flag", ["staged_to", "reduced"])
def test_model_catches_a_broken_schedule(flag):
    """Sanity: drop every wait of one rank on one kind of flag (STAGED_TO or
    REDUCED) and the checker must object.  (A GATHERED flag was dropped from
    the protocol after this checker showed its waits were implied.)"""
    progs = programs(3, [("allreduce", 60_000, 0), ("allreduce", 60_000, 0)], 4096, "ce")
    lanes = progs[1]
    hit = (lambda f: f == 0 or f >= STAGED_TO) if flag == "staged_to" else (lambda f: f == REDUCED)
    broken_lanes = [[op for op in lane if not (op[0] == "A" and hit(op[2]))] for lane in lanes]
    assert broken_lanes != lanes
    broken = [broken_lanes if r == 1 else p for r, p in enumerate(progs)]
    failures = 0
    for seed in range(60):
        try:
            simulate(broken, seed)
        except AssertionError:
            failures += 1
    assert failures > 0


@pytest.mark.parametrize("n", [2, 7])
@pytest.mark.parametrize("grain,gather,ramp,lanes,slots", [
    ("fine", "fine", "1", "3", "2"), ("coarse", "coarse", "0", "3", "2"),
    ("fine", "fine", "0", "2", "2"), ("coarse", "fine", "1", "3", "2"),
    ("coarse", "coarse", "1", "2", "2"), ("coarse", "fine", "1", "1", "2"),
    ("coarse", "coarse", "1", "3", "3"), ("fine", "fine", "1", "3", "4"),
    ("coarse", "coarse", "2", "3", "2"), ("coarse", "fine", "2", "2", "3"),
    ("coarse", "coarse", "3", "3", "2"), ("first", "coarse", "0", "3", "2"),
    ("first", "fine", "0", "2", "3"), ("first", "coarse", "1", "1", "2"),
    ("coarse", "coarse", "0", "2", "3"), ("coarse", "fine", "1", "3", "4"),
    ("coarse", "coarse", "4", "3", "2"), ("fine", "fine", "4", "2", "3")])
def test_schedule_variants(monkeypatch, n, grain, gather, ramp, lanes, slots):
    monkeypatch.setenv("FMX_GRAIN", grain)
    monkeypatch.setenv("FMX_GATHER_GRAIN", gather)
    monkeypatch.setenv("FMX_RAMP", ramp)
    monkeypatch.setenv("FMX_LANES", lanes)
    monkeypatch.setenv("FMX_SLOTS", slots)
    progs = programs(n, SEQUENCES["mixed"], 4096, "ce")
    for seed in range(6):
        simulate(progs, seed)
    merged = programs(n, SEQUENCES["mixed"], 4096, "ce", merged=True)
    for seed in range(6):
        simulate(merged, seed)


def test_result_via_copy_engine_variant(monkeypatch):
    monkeypatch.setenv("FMX_RESULT_VIA_CE", "1")
    progs = programs(4, SEQUENCES["mixed"], 4096, "ce")
    for seed in range(8):
        simulate(progs, seed)


@pytest.mark.parametrize("event", [0, 4])
def test_model_catches_a_missing_gather_lane_event(event):
    """Three-lane schedule: drop lane 1's waits on W (event ids 0..3: "every peer
    reduced the previous round") or on G (4..7: "my previous gather is done").
    Either lets an owner overwrite its result slot while a peer's gather still
    reads it, and the checker must object."""
    progs = programs(3, [("allreduce", 60_000, 0), ("allreduce", 60_000, 0)], 4096, "ce")
    lanes = progs[1]
    broken_lanes = [lanes[0], [op for op in lanes[1] if not (op[0] == "X" and event <= op[1] < event + 4)],
                    lanes[2]]
    assert broken_lanes[1] != lanes[1]
    broken = [broken_lanes if r == 1 else p for r, p in enumerate(progs)]
    failures = 0
    for seed in range(80):
        try:
            simulate(broken, seed)
        except AssertionError:
            failures += 1
    assert failures > 0


def test_model_catches_a_broken_host_scratch_reuse():
    """Host-buffer path: drop lane 0's waits on "fetch slot consumed" (event
    ids 10/11) and a fetch overwrites a scratch slot the reduce still reads."""
    progs = programs(2, [("allreduce_host", 200_000, 0)], 4096, "ce")
    lanes = progs[0]
    broken_lanes = [[op for op in lanes[0] if not (op[0] == "X" and op[1] in (10, 11))],
                    lanes[1], lanes[2]]
    assert broken_lanes[0] != lanes[0]
    broken = [broken_lanes if r == 0 else p for r, p in enumerate(progs)]
    failures = 0
    for seed in range(80):
        try:
            simulate(broken, seed)
        except AssertionError:
            failures += 1
    assert failures > 0


def test_model_catches_a_broken_host_push_lane():
    """Host-buffer path, three lanes: drop lane 1's waits on "result slot
    pushed" (event ids 13/14) and a reduce overwrites a result slot the push
    lane still reads."""
    progs = programs(2, [("allreduce_host", 200_000, 0)], 4096, "ce")
    lanes = progs[0]
    broken_lanes = [lanes[0], [op for op in lanes[1] if not (op[0] == "X" and op[1] in (13, 14))],
                    lanes[2]]
    assert broken_lanes[1] != lanes[1]
    broken = [broken_lanes if r == 0 else p for r, p in enumerate(progs)]
    failures = 0
    for seed in range(80):
        try:
            simulate(broken, seed)
        except AssertionError:
            failures += 1
    assert failures > 0


@pytest.mark.parametrize("ramp", ["0", "1", "2", "3", "4"])
@pytest.mark.parametrize("min_rounds", ["1", "3", "4", "7"])
@pytest.mark.parametrize("slice_bytes", [4096, 1 << 20, 4 << 20, 12288])
@pytest.mark.parametrize("dtype", [0, 1])
def test_piece_starts_are_16_byte_aligned(monkeypatch, ramp, min_rounds, slice_bytes, dtype):
    """The vector reduction needs every pipeline piece to start on 16 bytes:
    ramp pieces and the min-rounds slice are whole vectors for any slice size
    (a misaligned ramp piece once crashed the B200 with FMX_MIN_ROUNDS=4)."""
    import re
    monkeypatch.setenv("FMX_MIN_ROUNDS", min_rounds)
    monkeypatch.setenv("FMX_RAMP", ramp)
    for count in (1_000_003, 2_000_000, 333_333, 64_001, 17):
        for rank in (0, 3, 6):
            t = _lib.trace_plan(7, rank, [("allreduce", count, dtype)], slice_bytes)
            offs = [int(m.group(1)) for m in re.finditer(r"^\d UW (\d+) ", t, re.M)]
            assert offs and all(o % 16 == 0 for o in offs), (count, rank, offs[:8])


@pytest.mark.parametrize("n", [2, 7])
def test_auto_transport_mixes_zc_and_ce_calls(monkeypatch, n):
    """AUTO picks ZC or CE per collective by size; consecutive calls of either
    kind share slots and round counters, so mixed sequences must stay race- and
    deadlock-free."""
    monkeypatch.setenv("FMX_ZC_MAX", "100000")
    for seq in ("mixed", "rs-ag", "host-buffer"):
        progs = programs(n, SEQUENCES[seq], 4096, "auto")
        for seed in range(6):
            simulate(progs, seed)
        merged = programs(n, SEQUENCES[seq], 4096, "auto", merged=True)
        for seed in range(3):
            simulate(merged, seed)


OVERLAP_SEQUENCES = {
    "allreduces": [("allreduce", 30_001, 0), ("allreduce", 4_000, 1), ("allreduce", 50_000, 0),
                   ("allreduce", 1, 0), ("allreduce", 77_777, 1), ("allreduce", 20_000, 0)],
    "buckets+rs-ag": [("allreduce", 20_000, 0), ("reduce_scatter", 9_001, 0),
                      ("allgather", 12_000, 1), ("allreduce", 60_000, 0),
                      ("broadcast", 5_000, 0, 1), ("allreduce", 10_000, 0),
                      ("allreduce_host", 30_000, 0), ("allreduce", 40_000, 1)],
}


@pytest.mark.parametrize("n", [2, 3, 7])
@pytest.mark.parametrize("seq", sorted(OVERLAP_SEQUENCES))
@pytest.mark.parametrize("slots,lanes,transport", [("2", "3", "ce"), ("3", "3", "ce"),
                                                   ("2", "2", "ce"), ("2", "3", "zc"),
                                                   ("2", "3", "auto")])
def test_overlapping_collectives_join_stream_mode(monkeypatch, n, seq, slots, lanes, transport):
    """Join-stream mode (DDP buckets): consecutive device collectives on
    distinct buffers run on the lanes without a join in between, so call k+1
    stages while call k still fetches and gathers.  Slot reuse across calls
    rests on the global-round W / G events alone."""
    monkeypatch.setenv("FMX_TRACE_OVERLAP", "1")
    monkeypatch.setenv("FMX_SLOTS", slots)
    monkeypatch.setenv("FMX_LANES", lanes)
    monkeypatch.setenv("FMX_ZC_MAX", "100000")
    progs = programs(n, OVERLAP_SEQUENCES[seq], 4096, transport)
    for seed in range(10):
        simulate(progs, seed, burst=4)
    merged = programs(n, OVERLAP_SEQUENCES[seq], 4096, transport, merged=True)
    for seed in range(3):
        simulate(merged, seed)


def test_overlap_mode_needs_the_cross_call_waits(monkeypatch):
    """Drop the stage lane's W waits of the first K rounds of each later
    collective (what the pre-overlap plan omitted, relying on the join) and
    the checker must object in join-stream mode."""
    monkeypatch.setenv("FMX_TRACE_OVERLAP", "1")
    ops = [("allreduce", 3000, 0), ("allreduce", 3000, 0), ("allreduce", 3000, 0)]
    progs = programs(3, ops, 4096, "ce")
    lanes = progs[1]
    broken0 = [op for op in lanes[0] if not (op[0] == "X" and op[1] < 4)]
    assert broken0 != lanes[0]
    broken = [[broken0, lanes[1], lanes[2]] if r == 1 else p for r, p in enumerate(progs)]
    failures = 0
    for seed in range(80):
        try:
            simulate(broken, seed, burst=4)
        except AssertionError:
            failures += 1
    assert failures > 0


# ---- one-shot small-message allreduce (plan_allreduce_oneshot) ----------------

OS_READY = 4  # kOsReady
ONESHOT_SEQ = ([("allreduce", 1 + 37 * i, i % 2) for i in range(9)]
               + [("allreduce", 60_000, 0), ("allreduce", 5, 1), ("broadcast", 300, 0, 1),
                  ("allreduce", 16_384, 0), ("reduce_scatter", 11, 0), ("allreduce", 3, 0),
                  ("allreduce_host", 700, 0), ("allreduce", 32_768, 1)])


def test_oneshot_is_selected_by_size():
    """AUTO takes the one-shot path up to FMX_ONESHOT_MAX bytes (64 KiB): one
    publish + OS_READY, one wait, one reduce - no pipeline flags."""
    small = _lib.trace_plan(7, 3, [("allreduce", 16_384, 0)], 4096, "auto")
    assert f" S {OS_READY} 1" in small and small.count(" S ") == 1
    assert " S 0 " not in small and " S 1 " not in small  # no STAGED / REDUCED
    big = _lib.trace_plan(7, 3, [("allreduce", 16_385, 0)], 4096, "auto")
    assert f" S {OS_READY} " not in big
    ce = _lib.trace_plan(7, 3, [("allreduce", 5, 0)], 4096, "ce")
    assert f" S {OS_READY} " not in ce


@pytest.mark.parametrize("n", [2, 3, 7])
def test_oneshot_mixed_with_pipelined_collectives(n):
    """More one-shot calls than slots (slot reuse), interleaved with pipelined
    allreduces, broadcasts, reduce-scatters and host-path calls."""
    progs = programs(n, ONESHOT_SEQ, 4096, "auto")
    for seed in range(10):
        simulate(progs, seed)
    merged = programs(n, ONESHOT_SEQ, 4096, "auto", merged=True)
    for seed in range(4):
        simulate(merged, seed)


def test_oneshot_at_56_ranks():
    ops = [("allreduce", 256, 0)] * 6 + [("allreduce", 32_768, 1)]
    progs = programs(56, ops, 320 << 10, "auto")
    simulate(progs, 0, burst=8)


def test_model_catches_a_broken_oneshot():
    """Drop one rank's OS_READY waits: it reduces peer slots before they were
    published (and overwrites its own slot while a slow peer still reads it)."""
    ops = [("allreduce", 1000, 0)] * 5
    progs = programs(3, ops, 4096, "auto")
    lanes = progs[1]
    broken_lanes = [[op for op in lane if not (op[0] == "A" and op[2] == OS_READY)] for lane in lanes]
    assert broken_lanes != lanes
    broken = [broken_lanes if r == 1 else p for r, p in enumerate(progs)]
    failures = 0
    for seed in range(100):
        try:
            simulate(broken, seed)
        except AssertionError:
            failures += 1
    assert failures > 0


def test_oneshot_slot_reuse_needs_no_credit_flag():
    """Twelve back-to-back one-shot calls reuse the two slots six times each:
    race-free without a credit flag, because a peer publishes call J+1 only
    after its reduce of call J read my slot."""
    ops = [("allreduce", 64, 0)] * 12
    progs = programs(4, ops, 4096, "auto")
    for seed in range(20):
        simulate(progs, seed, burst=1)


# ---- deferred gather (fmx_comm_set_defer, the DP bucket order) ----------------

DEFER_SEQUENCES = {
    "buckets": [("allreduce", 30_001, 0), ("allreduce", 50_000, 0), ("allreduce", 200_003, 0),
                ("allreduce", 7, 0), ("allreduce", 77_777, 1), ("allreduce", 20_000, 0),
                ("flush", 0, 0)],
    "mixed": [("allreduce", 20_000, 0), ("allreduce", 60_000, 1), ("reduce_scatter", 9_001, 0),
              ("allreduce", 40_000, 0), ("broadcast", 5_000, 0, 1), ("allreduce", 10_000, 0),
              ("allreduce_host", 30_000, 0), ("allreduce", 300, 0), ("allreduce", 40_000, 1),
              ("allgather", 12_000, 1), ("allreduce", 90_000, 0), ("flush", 0, 0)],
}


@pytest.mark.parametrize("n", [2, 3, 7])
@pytest.mark.parametrize("seq", sorted(DEFER_SEQUENCES))
@pytest.mark.parametrize("slots,lanes,transport", [("2", "3", "ce"), ("3", "3", "ce"),
                                                   ("2", "1", "ce"), ("2", "3", "zc"),
                                                   ("2", "3", "auto")])
def test_deferred_gather(monkeypatch, n, seq, slots, lanes, transport):
    """An allreduce's last gather enqueued after the next collective's first
    stage (or by the flush / any other collective first): race-, stale-read-
    and deadlock-free in join-stream mode, on the lanes and as one FIFO."""
    monkeypatch.setenv("FMX_TRACE_OVERLAP", "1")
    monkeypatch.setenv("FMX_TRACE_DEFER", "1")
    monkeypatch.setenv("FMX_SLOTS", slots)
    monkeypatch.setenv("FMX_LANES", lanes)
    monkeypatch.setenv("FMX_ZC_MAX", "100000")
    progs = programs(n, DEFER_SEQUENCES[seq], 4096, transport)
    for seed in range(10):
        simulate(progs, seed, burst=4)
    merged = programs(n, DEFER_SEQUENCES[seq], 4096, transport, merged=True)
    for seed in range(6):
        simulate(merged, seed)


def test_deferred_gather_order(monkeypatch):
    """The deferred gather of call k sits after call k+1's first stage and
    before call k+1's REDUCED signal (merged enqueue order of one rank)."""
    monkeypatch.setenv("FMX_TRACE_DEFER", "1")
    text = _lib.trace_plan(3, 0, [("allreduce", 30_000, 0), ("allreduce", 30_000, 0),
                                  ("flush", 0, 0)], 1 << 20, "ce")
    ops = [ln.split()[1:] for ln in text.splitlines() if ln and ln != "J"]
    reduced_waits = [i for i, o in enumerate(ops) if o[0] == "A" and o[2] == str(REDUCED)]
    staged = [i for i, o in enumerate(ops) if o[0] == "S" and o[1] == "0"]
    reduced = [i for i, o in enumerate(ops) if o[0] == "S" and o[1] == str(REDUCED)]
    # call 0's gather waits come after call 1's STAGED signal, before its REDUCED
    assert staged[1] < reduced_waits[0] < reduced[1]


def test_deferred_gather_must_be_flushed(monkeypatch):
    monkeypatch.setenv("FMX_TRACE_DEFER", "1")
    with pytest.raises(ValueError):
        _lib.trace_plan(2, 0, [("allreduce", 30_000, 0)], 4096, "ce")


# ---- captured CUDA graphs (fmx_graph_*): replays of one captured schedule ------

REPLAY_SEQUENCES = {
    "dp-step": [("allreduce", 30_001, 0), ("allreduce", 200_003, 0), ("allreduce", 77_777, 0),
                ("allreduce", 5, 0), ("allreduce", 20_000, 0), ("flush", 0, 0)],
    "mixed": [("allreduce", 20_000, 0), ("reduce_scatter", 9_001, 0), ("broadcast", 5_000, 0, 1),
              ("allreduce", 123_457, 1), ("allgather", 3, 0), ("allreduce", 300, 0),
              ("flush", 0, 0)],
}


@pytest.mark.parametrize("n", [2, 3, 7])
@pytest.mark.parametrize("seq", sorted(REPLAY_SEQUENCES))
@pytest.mark.parametrize("lanes,transport,defer", [("1", "ce", "1"), ("3", "ce", "1"),
                                                   ("3", "zc", "0"), ("3", "auto", "1"),
                                                   ("1", "auto", "0")])
def test_graph_replays(monkeypatch, n, seq, lanes, transport, defer):
    """A captured step replayed 3 times: every replay runs the captured slots
    and rounds with flag values re-based by the counters' advance, drops waits
    on events of other replays, and ends with the appended fence - race-,
    stale-read- and deadlock-free on the lanes and as one FIFO."""
    monkeypatch.setenv("FMX_TRACE_REPLAYS", "3")
    monkeypatch.setenv("FMX_TRACE_OVERLAP", "1")
    monkeypatch.setenv("FMX_TRACE_DEFER", defer)
    monkeypatch.setenv("FMX_LANES", lanes)
    monkeypatch.setenv("FMX_ZC_MAX", "100000")
    progs = programs(n, REPLAY_SEQUENCES[seq], 4096, transport)
    for seed in range(8):
        simulate(progs, seed, burst=4)
    merged = programs(n, REPLAY_SEQUENCES[seq], 4096, transport, merged=True)
    for seed in range(4):
        simulate(merged, seed)


def test_graph_replays_need_the_fence(monkeypatch):
    """Without the end-of-replay fence, a replay's baked slots are reused while
    a slow peer still reads the previous replay's: the checker must object.
    (Pipelined allreduces alone would be safe - every rank's first stage of
    replay r+1 follows its complete replay r, whose gathers waited for every
    owner's REDUCED - but a one-shot publish or a broadcast root does not wait
    for its readers: their slot alternation / reuse wait is decided on the
    captured round, so a replay writes the slot a slow peer still reads.)"""
    monkeypatch.setenv("FMX_TRACE_REPLAYS", "3")
    monkeypatch.setenv("FMX_TRACE_OVERLAP", "1")
    for ops in ([("allreduce", 5, 0)], [("broadcast", 3000, 0, 0)]):
        monkeypatch.setenv("FMX_TRACE_REPLAY_FENCE", "0")
        progs = programs(3, ops, 4096, "auto")
        failures = 0
        for seed in range(80):
            try:
                simulate(progs, seed, burst=4)
            except AssertionError:
                failures += 1
        assert failures > 0, ops
        monkeypatch.setenv("FMX_TRACE_REPLAY_FENCE", "1")
        progs = programs(3, ops, 4096, "auto")
        for seed in range(80):
            simulate(progs, seed, burst=4)


@pytest.mark.parametrize("n", [2, 3, 7])
@pytest.mark.parametrize("lanes,slots,transport", [("3", "2", "ce"), ("3", "3", "ce"),
                                                   ("2", "2", "ce"), ("1", "2", "ce"),
                                                   ("3", "2", "zc")])
def test_stage_after_reduce(monkeypatch, n, lanes, slots, transport):
    """FMX_STAGE_AFTER_REDUCE: stage(R+K-1) enqueued after reduce(R) and
    waiting for it - still race- and deadlock-free, on the lanes, as one FIFO,
    and in join-stream / deferred-gather mode."""
    monkeypatch.setenv("FMX_STAGE_AFTER_REDUCE", "1")
    monkeypatch.setenv("FMX_LANES", lanes)
    monkeypatch.setenv("FMX_SLOTS", slots)
    seq = SEQUENCES["mixed"] + [("allreduce", 200_003, 0), ("reduce_scatter", 40_000, 1)]
    progs = programs(n, seq, 4096, transport)
    for seed in range(6):
        simulate(progs, seed)
    merged = programs(n, seq, 4096, transport, merged=True)
    for seed in range(4):
        simulate(merged, seed)
    monkeypatch.setenv("FMX_TRACE_OVERLAP", "1")
    monkeypatch.setenv("FMX_TRACE_DEFER", "1")
    progs = programs(n, DEFER_SEQUENCES["buckets"], 4096, transport)
    for seed in range(4):
        simulate(progs, seed, burst=4)


@pytest.mark.parametrize("n", [2, 3, 7])
@pytest.mark.parametrize("slots,transport,grain", [("2", "ce", "coarse"), ("3", "ce", "coarse"),
                                                   ("2", "ce", "fine"), ("4", "auto", "coarse"),
                                                   ("2", "zc", "coarse")])
def test_fetch_lane(monkeypatch, n, slots, transport, grain):
    """FMX_FETCH_LANE: the fetch of round R+1 on the gather lane into a
    double-buffered HBM scratch while lane 1 reduces round R - race-free on
    the scratch (S(R-2) before fetch(R)), deadlock-free on the lanes and as
    one FIFO, across calls in join-stream / deferred-gather mode."""
    monkeypatch.setenv("FMX_FETCH_LANE", "1")
    monkeypatch.setenv("FMX_RCE_ROUNDS", "3")      # result slot by copy engine on long pipelines
    monkeypatch.setenv("FMX_SLOTS", slots)
    monkeypatch.setenv("FMX_GRAIN", grain)
    monkeypatch.setenv("FMX_ZC_MAX", "100000")
    seq = SEQUENCES["mixed"] + [("allreduce", 200_003, 0), ("reduce_scatter", 40_000, 1),
                                ("allreduce", 77_777, 1)]
    progs = programs(n, seq, 4096, transport)
    for seed in range(6):
        simulate(progs, seed)
    merged = programs(n, seq, 4096, transport, merged=True)
    for seed in range(4):
        simulate(merged, seed)
    monkeypatch.setenv("FMX_TRACE_OVERLAP", "1")
    monkeypatch.setenv("FMX_TRACE_DEFER", "1")
    progs = programs(n, DEFER_SEQUENCES["mixed"], 4096, transport)
    for seed in range(4):
        simulate(progs, seed, burst=4)


def test_fetch_lane_needs_the_scratch_wait(monkeypatch):
    """Drop lane 2's waits on S (reduce(R-2) done reading scratch slot R%2)
    and the checker must see fetch(R) overwrite scratch a reduction still
    reads.  (With K = 2 slots the wait is implied - peers stage R only after
    seeing my REDUCED(R-2) - so the check runs at K = 3.)"""
    monkeypatch.setenv("FMX_FETCH_LANE", "1")
    monkeypatch.setenv("FMX_SLOTS", "3")
    ops = [("allreduce", 3 * 8 * 1024, 0)]        # 8 rounds of 1 KiB pieces at n=3
    progs = programs(3, ops, 4096, "ce")
    lanes = progs[1]
    s_events = {2 * 4 + 10, 2 * 4 + 11}            # kEvScratchFree + 0/1 (FMX_MAX_SLOTS = 4)
    broken2 = [op for op in lanes[2] if not (op[0] == "X" and op[1] in s_events)]
    assert broken2 != lanes[2]
    broken = [[lanes[0], lanes[1], broken2] if r == 1 else p for r, p in enumerate(progs)]
    failures = 0
    for seed in range(80):
        try:
            simulate(broken, seed, burst=4)
        except AssertionError:
            failures += 1
    assert failures > 0


@pytest.mark.parametrize("n,ops,slots", [
    # C1: the ResNet-50 gradient over two ranks of one GPU (16 MiB slices, K = 4)
    (2, [("allreduce", 25_557_032, 0), ("allreduce", 268_435_456, 0)], "4"),
    # C3: MobileNetV2 over 4 ranks, two per GPU
    (4, [("allreduce", 3_504_872, 0), ("broadcast", 3_504_872, 0, 3)], "2"),
])
def test_two_ranks_per_gpu_defaults_at_config_shapes(monkeypatch, n, ops, slots):
    """The <= 2-ranks-per-GPU defaults (fetch lane, copy-engine result from 8
    rounds) at the BASELINE configs' own shapes and default slice geometry."""
    monkeypatch.setenv("FMX_FETCH_LANE", "1")
    monkeypatch.setenv("FMX_RCE_ROUNDS", "8")
    monkeypatch.setenv("FMX_SLOTS", slots)
    sb = (16 << 20) if n <= 2 else default_slice(n)
    progs = programs(n, ops, sb, "auto")
    for seed in range(2):
        simulate(progs, seed, burst=8)
    merged = programs(n, ops, sb, "auto", merged=True)
    simulate(merged, 0)
