"""Probe: the reduce kernel's zero-copy traffic - its result store (SM stores
to mapped host memory), or in the ZC flavour its n-1 source reads (SM loads
from mapped host memory) - alone and while copy engines stream host->device (H2D) and/or
device->host (D2H) on other streams - the live conditions of the pipeline,
where every rank's fetch / gather (H2D) and stage (D2H) copies run while an
owner reduces.  One process, one full 4 MiB piece of 7 sources, CUDA events
on the kernel's stream.  Prints JSON lines."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_09143_b200.comm import reduce_local  # noqa: E402

n, piece = 7, (4 << 20) // 4
srcs = [torch.randn(piece, device="cuda") for _ in range(n)]
out = torch.empty(piece, device="cuda")
out_host = torch.empty(piece).pin_memory()
big = 256 << 20
h_src = torch.empty(big, dtype=torch.uint8).pin_memory()
h_dst = torch.empty(big, dtype=torch.uint8).pin_memory()
d_buf = torch.empty(big, dtype=torch.uint8, device="cuda")
d_buf2 = torch.empty(big, dtype=torch.uint8, device="cuda")
ks = torch.cuda.Stream()
s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()


# the ZC-transport flavour: n-1 contributions read zero-copy from mapped host
# memory (the fetch fused into the reduction), result to HBM only
host_srcs = [srcs[0]] + [torch.randn(piece).pin_memory() for _ in range(n - 1)]


def run_once(kind):
    if kind == "store":
        reduce_local(srcs, out, op="avg", out_host=out_host, stream=ks)
    else:
        reduce_local(host_srcs, out, op="avg", host_sources=range(1, n), stream=ks)


def time_kernel(kind, iters=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(ks):
        for _ in range(3):
            run_once(kind)
        e0.record(ks)
        for _ in range(iters):
            run_once(kind)
        e1.record(ks)
    e1.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3  # us


for kind, load in [(k, ld) for k in ("store", "load") for ld in ("none", "h2d", "d2h", "both")]:
    torch.cuda.synchronize()
    if load in ("h2d", "both"):
        with torch.cuda.stream(s_h2d):
            for _ in range(8):
                d_buf.copy_(h_src, non_blocking=True)
    if load in ("d2h", "both"):
        with torch.cuda.stream(s_d2h):
            for _ in range(8):
                h_dst.copy_(d_buf2, non_blocking=True)
    us = time_kernel(kind)
    torch.cuda.synchronize()
    moved = piece * 4 * (1 if kind == "store" else n - 1)
    print(json.dumps({"probe": f"reduce_zc_{kind}_under_load", "load": load,
                      "kernel_us": round(us, 1), "link_gbs": round(moved / us / 1e3, 2)}),
          flush=True)
