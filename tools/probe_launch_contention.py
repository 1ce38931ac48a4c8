"""Probe: does host-link traffic slow the GPU's own compute?

In DP training the exchange's copy-engine traffic alone (bench FMX_HOOK_NOOP=3)
costs ~12 ms of a 54.7 ms ResNet-50 step, the reduce kernels alone nothing
(profiles/r02/r2n).  Hypothesis: every eager kernel launch makes the GPU read
its launch descriptor / pushbuffer from host memory, and those reads queue
behind bulk H2D traffic on the same PCIe direction; a CUDA graph's launch
descriptors live in device memory.  This measures, in one process (optionally
an MPS client), a ResNet-50 fwd+bwd step eager and as a CUDA graph, and a chain
of tiny spin kernels, each alone and while copy engines stream H2D / D2H /
both on other streams.  Prints JSON lines."""
import json
import os
import sys

import torch
import torch.nn.functional as F
import torchvision

batch = int(os.environ.get("PROBE_BATCH", "32"))
big = 256 << 20
h_src = torch.empty(big, dtype=torch.uint8).pin_memory()
h_dst = torch.empty(big, dtype=torch.uint8).pin_memory()
d_buf = torch.empty(big, dtype=torch.uint8, device="cuda")
d_buf2 = torch.empty(big, dtype=torch.uint8, device="cuda")
s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
ks = torch.cuda.Stream()

model = torchvision.models.resnet50().cuda().to(memory_format=torch.channels_last)
x = torch.randn(batch, 3, 224, 224, device="cuda").to(memory_format=torch.channels_last)
y = torch.randint(0, 1000, (batch,), device="cuda")


def fwd_bwd():
    with torch.autocast("cuda", dtype=torch.bfloat16):
        loss = F.cross_entropy(model(x), y)
    loss.backward()


with torch.cuda.stream(ks):
    for _ in range(3):
        fwd_bwd()
torch.cuda.synchronize()
# the same step as one CUDA graph (grads accumulate into static .grad tensors)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=ks):
    fwd_bwd()
torch.cuda.synchronize()


def traffic(load, copies):
    if load in ("h2d", "both"):
        with torch.cuda.stream(s_h2d):
            for _ in range(copies):
                d_buf.copy_(h_src, non_blocking=True)
    if load in ("d2h", "both"):
        with torch.cuda.stream(s_d2h):
            for _ in range(copies):
                h_dst.copy_(d_buf2, non_blocking=True)


def timed(fn, iters):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(ks):
        fn()
        e0.record(ks)
        for _ in range(iters):
            fn()
        e1.record(ks)
    e1.synchronize()
    return e0.elapsed_time(e1) / iters


def spin_chain():
    for _ in range(500):
        torch.cuda._sleep(2000)   # ~1 us of spinning per launch


cases = {"resnet50_eager": (fwd_bwd, 5), "resnet50_graph": (g.replay, 5),
         "spin500_eager": (spin_chain, 5)}
for name, (fn, iters) in cases.items():
    for load in ("none", "h2d", "d2h", "both"):
        torch.cuda.synchronize()
        # enough traffic to outlast the timed region (then drained, untimed)
        traffic(load, int(os.environ.get("PROBE_COPIES", "24")))
        ms = timed(fn, iters)
        torch.cuda.synchronize()
        print(json.dumps({"probe": "compute_under_link_traffic", "case": name, "load": load,
                          "batch": batch, "ms_per_iter": round(ms, 3),
                          "mps_pct": os.environ.get("CUDA_MPS_ACTIVE_THREAD_PERCENTAGE")}),
              flush=True)
