"""Summarise a host-polled flag timeline (bench.py --timeline): for every
round, when each rank finished staging (last STAGED / STAGED_TO flag) and
reducing (REDUCED), in ms from the first event."""
import json
import sys
from collections import defaultdict


def main(path):
    d = json.load(open(path))
    n = d["n"]
    ev = d["events"]
    if not ev:
        print("no events")
        return
    t0 = ev[0][0]
    staged = defaultdict(dict)   # (rank, value) -> last time any stage flag hit value
    reduced = defaultdict(dict)
    for t, r, f, v in ev:
        ms = (t - t0) / 1e6
        if f == 0 or f >= 8:
            staged[v][r] = max(staged[v].get(r, 0), ms)
        elif f == 1:
            reduced[v][r] = ms
    rounds = sorted(set(staged) | set(reduced))
    print(f"{path}: n={n} slice={d['slice_bytes']} events={len(ev)} span={(ev[-1][0]-t0)/1e6:.2f} ms")
    for v in rounds:
        s = staged.get(v, {})
        rr = reduced.get(v, {})
        fmt = lambda m: " ".join(f"{m.get(r, float('nan')):6.2f}" for r in range(n))
        print(f"round {v-1:3d} staged  {fmt(s)}")
        print(f"          reduced {fmt(rr)}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
