"""Host-link capacity under the rank layout of the bench: P processes on one
GPU (MPS clients or plain time-sliced contexts), each moving data between
pinned host memory and HBM with the copy engines, H2D only / D2H only / both
directions on two streams.  Prints one JSON line per case: aggregate GB/s.

Tells apart "the link (or CE arbitration across processes) caps at X" from
"the pipeline's synchronisation leaves the link idle"."""
from __future__ import annotations

import json
import multiprocessing as mp
import os
import sys
import time


def worker(rank, P, mb, reps, direction, barrier, q, pieces):
    import torch
    torch.cuda.set_device(0)
    n = mb * (1 << 20) // 4
    host_in = torch.empty(n, dtype=torch.float32).pin_memory()
    host_out = torch.empty(n, dtype=torch.float32).pin_memory()
    dev_in = torch.empty(n, dtype=torch.float32, device="cuda")
    dev_out = torch.randn(n, device="cuda")
    s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
    step = n // pieces

    if direction.startswith("zc") or direction.startswith("ce+zc"):
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_2511_09143_b200.comm import reduce_local
    scratch = torch.empty(n, dtype=torch.float32, device="cuda")

    def go():
        for _ in range(reps):
            for k in range(pieces):
                sl = slice(k * step, (k + 1) * step)
                if direction in ("h2d", "bidir", "ce+zc_d2h"):
                    with torch.cuda.stream(s_h2d):
                        dev_in[sl].copy_(host_in[sl], non_blocking=True)
                if direction in ("d2h", "bidir"):
                    with torch.cuda.stream(s_d2h):
                        host_out[sl].copy_(dev_out[sl], non_blocking=True)
                if direction in ("zc_d2h", "ce+zc_d2h"):  # SM stores into pinned host memory
                    reduce_local([dev_out[sl]], scratch[sl], out_host=host_out[sl], stream=s_d2h)
                if direction == "zc_h2d":  # SM loads from pinned host memory
                    reduce_local([host_in[sl]], scratch[sl], host_sources=[0], stream=s_h2d)
                if direction == "zc_bidir":  # one kernel: host loads + host stores
                    reduce_local([host_in[sl]], scratch[sl], host_sources=[0],
                                 out_host=host_out[sl], stream=s_h2d)
        torch.cuda.synchronize()

    go()  # warm-up
    barrier.wait()
    t0 = time.perf_counter()
    go()
    t1 = time.perf_counter()
    barrier.wait()
    q.put((rank, t0, t1))


def case(P, mb, reps, direction, pieces=1):
    ctx = mp.get_context("spawn")
    barrier = ctx.Barrier(P)
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, P, mb, reps, direction, barrier, q, pieces))
          for r in range(P)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(P)]
    for p in ps:
        p.join()
    t = max(r[2] for r in res) - min(r[1] for r in res)
    per_dir = P * mb * (1 << 20) * reps
    total = per_dir * (2 if "bidir" in direction or "+" in direction else 1)
    return {"P": P, "mb_per_proc": mb, "reps": reps, "pieces": pieces, "direction": direction,
            "mps": "CUDA_MPS_PIPE_DIRECTORY" in os.environ, "s": t, "gbs_total": total / t / 1e9}


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    lines = []
    dirs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["h2d", "d2h", "bidir"]
    for P, mb, reps in [(1, 512, 4), (7, 96, 4)]:
        for direction in dirs:
            for pieces in (1, 24):
                r = case(P, mb, reps, direction, pieces)
                print(json.dumps(r), flush=True)
                lines.append(r)
    if out:
        with open(out, "a") as f:
            f.writelines(json.dumps(r) + "\n" for r in lines)


if __name__ == "__main__":
    main()
