"""One DP training step on the GPU clock (bench.py --train-only --stamps F):
per rank, the step window (markers 1 and 2 on the compute stream) and every
collective of the DDP hook (a collective = the ops between two joins; its
span = first op start .. last op completion), in ms from the step start."""
import json
import sys


def main(path):
    d = json.load(open(path))
    for r, st in sorted(d["train"].items(), key=lambda kv: int(kv[0])):
        if not st:
            continue
        t_begin = next(t for t, lane, kind, info in st if kind == 7 and info == 1)
        t_end = next(t for t, lane, kind, info in st if kind == 7 and info == 2)
        ops = [(t, lane, kind, info) for t, lane, kind, info in st if kind != 7]
        # collectives: REDUCED signals (lane 1, kind 6) close one round; group by
        # gaps: a new collective starts when lane-0/1 ops resume after a gather
        spans, cur = [], None
        last = {}
        for t, lane, kind, info in ops:
            start = last.get(lane, t)
            last[lane] = t
            if cur is None or start > cur[1] + 200_000:   # > 0.2 ms idle: next collective
                cur = [start, t, 0]
                spans.append(cur)
            cur[1] = max(cur[1], t)
            if kind == 4:
                cur[2] += info
        ms = lambda x: (x - t_begin) / 1e6
        busy = sum(b - a for a, b, _ in spans) / 1e6
        print(f"rank {r}: step {ms(t_end):7.2f} ms; {len(spans)} comm spans, busy {busy:6.2f} ms; "
              f"last comm ends {ms(spans[-1][1]) if spans else 0:7.2f}")
        if r == "0":
            for a, b, byt in spans:
                print(f"    {ms(a):7.2f} -> {ms(b):7.2f} ms  ({(b - a) / 1e6:6.2f} ms, {byt / 1e6:7.1f} MB copied)")


if __name__ == "__main__":
    main(sys.argv[1])
