"""Analyse a GPU-clock pipeline timeline (bench.py --stamps FILE).

Every stamp marks the completion of one operation on one lane of one rank,
on the GPU's global timer (one clock for all processes on the GPU).  An
operation starts when the previous stamp of its lane completed.  Copies are
attributed to a link direction by lane (device path: lane 0 stages D2H,
lanes 1 and 2 fetch / gather H2D, the reduction on lane 1 stores its result
slot D2H; host path: lane 0 fetches H2D, lane 1 pushes D2H).

Prints, per path: span, bytes per direction, the fraction of the span in
which at least one transfer of that direction was in flight ("busy"), the
achieved GB/s over busy time and over the span, and per-rank waits.

usage: python tools/analyze_stamps.py FILE [--ops RANK]
"""
from __future__ import annotations

import json
import sys
from collections import defaultdict

KIND = {1: "wait_peers", 2: "wait_rank", 3: "wait_event", 4: "copy", 5: "reduce", 6: "signal"}


def intervals(stamps):
    """[(lane, kind, info, start, end)] in enqueue order for one rank."""
    last = {}
    t0 = min(s[0] for s in stamps)
    out = []
    for t, lane, kind, info in stamps:
        start = last.get(lane, t0)
        out.append((lane, kind, info, start, t))
        last[lane] = t
    return out


def direction(path, lane, kind):
    if path == "device":
        if kind == 4:
            return "d2h" if lane == 0 else "h2d"
        if kind == 5:
            return "d2h"   # zero-copy store of the result slot
    else:
        if kind == 4:
            return "h2d" if lane == 0 else "d2h"
    return None


def union_len(iv):
    iv = sorted(iv)
    tot, cur_s, cur_e = 0, None, None
    for s, e in iv:
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        tot += cur_e - cur_s
    return tot


def analyse(path, per_rank, esz=4, show_ops=None):
    if not any(per_rank.values()):
        print(f"{path}: no stamps")
        return
    t0 = min(s[0] for v in per_rank.values() for s in v if v)
    t1 = max(s[0] for v in per_rank.values() for s in v if v)
    span = (t1 - t0) / 1e6
    busy = defaultdict(list)
    nbytes = defaultdict(int)
    waits = {}
    for r, st in sorted(per_rank.items(), key=lambda kv: int(kv[0])):
        ivs = intervals(st)
        w = 0.0
        for lane, kind, info, s, e in ivs:
            d = direction(path, lane, kind)
            if d:
                b = info * esz if kind == 5 else info
                nbytes[d] += b
                busy[d].append((s, e))
            if kind in (1, 2, 3):
                w += (e - s) / 1e6
        waits[r] = w
        if show_ops is not None and int(r) == show_ops:
            for lane, kind, info, s, e in ivs:
                print(f"  r{r} L{lane} {KIND.get(kind, kind):10s} info={info:>10d} "
                      f"{(s - t0) / 1e6:8.3f} -> {(e - t0) / 1e6:8.3f} ms ({(e - s) / 1e3:8.1f} us)")
    print(f"{path}: span {span:.2f} ms over {len(per_rank)} ranks")
    for d in ("h2d", "d2h"):
        b = union_len(busy[d]) / 1e6
        print(f"  {d}: {nbytes[d] / 1e6:8.1f} MB, busy {b:6.2f} ms ({b / span:5.1%} of span), "
              f"{nbytes[d] / max(b, 1e-9) / 1e6:6.1f} GB/s while busy, "
              f"{nbytes[d] / span / 1e6:6.1f} GB/s over span")
    # idle gaps of the H2D direction (the binding one on the device path)
    iv = sorted(busy["h2d"])
    gaps, cur = [], None
    for s_, e_ in iv:
        if cur is not None and s_ > cur:
            gaps.append((cur, s_))
        cur = e_ if cur is None else max(cur, e_)
    big = [(a, b) for a, b in gaps if b - a > 50_000]
    print(f"  h2d idle gaps > 50 us: {len(big)}, total {sum(b - a for a, b in big) / 1e6:.2f} ms: " +
          ", ".join(f"{(a - t0) / 1e6:.2f}+{(b - a) / 1e3:.0f}us" for a, b in big[:30]))
    # the link around the dominant kernel: all ranks' D2H traffic (stage copies +
    # result stores, each spread evenly over its interval) that overlaps each
    # reduce launch, over the launch's duration - is the D2H direction saturated
    # while the reduce kernel stores its result slot?
    if path == "device":
        d2h_ops = []
        for r, st in per_rank.items():
            for lane, kind, info, s, e in intervals(st):
                if direction(path, lane, kind) == "d2h" and e > s:
                    d2h_ops.append((s, e, info * esz if kind == 5 else info))
        tot_t = tot_b = 0.0
        for r, st in per_rank.items():
            for lane, kind, info, s, e in intervals(st):
                if kind != 5 or e <= s:
                    continue
                ov = sum(b * max(0, min(e, e2) - max(s, s2)) / (e2 - s2) for s2, e2, b in d2h_ops)
                tot_t += e - s
                tot_b += ov
        if tot_t:
            print(f"  d2h link while a reduce kernel runs: {tot_b / tot_t:.1f} GB/s of all ranks' "
                  f"traffic (time-weighted over {tot_t / 1e6:.2f} ms of reduce launches)")
    print("  lane-time in waits per rank (ms): " +
          " ".join(f"{r}:{w:.2f}" for r, w in sorted(waits.items(), key=lambda kv: int(kv[0]))))


def main():
    path = sys.argv[1]
    show = int(sys.argv[sys.argv.index("--ops") + 1]) if "--ops" in sys.argv else None
    d = json.load(open(path))
    for p in ("device", "host"):
        analyse(p, d.get(p, {}), show_ops=show)


if __name__ == "__main__":
    main()
