"""Probe: one training step of a model, eager vs captured as a CUDA graph, in
one process (optionally an MPS client): where does a graph replay lose to
eager (BERT-base, bf16 weights, AdamW)?  Prints JSON lines."""
import json
import os
import sys

import torch
import torch.nn.functional as F

name = sys.argv[1] if len(sys.argv) > 1 else "bert"
batch = int(os.environ.get("PROBE_BATCH", "32"))
torch.manual_seed(0)
if name == "bert":
    from transformers import BertConfig, BertForSequenceClassification
    model = BertForSequenceClassification(BertConfig(num_labels=2)).cuda().to(torch.bfloat16)
    x = torch.randint(0, 30522, (batch, 128), device="cuda")
    y = torch.randint(0, 2, (batch,), device="cuda")
    fwd = lambda: F.cross_entropy(model(input_ids=x).logits.float(), y)
else:
    import torchvision
    model = torchvision.models.resnet50().cuda().to(memory_format=torch.channels_last)
    x = torch.randn(batch, 3, 224, 224, device="cuda").to(memory_format=torch.channels_last)
    y = torch.randint(0, 1000, (batch,), device="cuda")

    def fwd():
        with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):
            return F.cross_entropy(model(x), y)


def timed(fn, iters=10):
    s = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(iters):
        fn()
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / iters


s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for opt_kind in ("foreach", "capturable", "none"):
        if opt_kind == "none":
            opt = None
        elif name == "bert":
            opt = torch.optim.AdamW(model.parameters(), lr=2e-5, capturable=opt_kind == "capturable")
        else:
            opt = torch.optim.SGD(model.parameters(), lr=0.01, momentum=0.9)

        def step():
            model.zero_grad(set_to_none=False)
            loss = fwd()
            loss.backward()
            if opt is not None:
                opt.step()
            return loss

        eager = timed(step)
        res = {"probe": "graph_step", "model": name, "opt": opt_kind, "eager_ms": round(eager, 3)}
        if opt_kind != "foreach":
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                step()
            res["graph_ms"] = round(timed(g.replay), 3)
            res["graph_nodes"] = None
        res["mps_pct"] = os.environ.get("CUDA_MPS_ACTIVE_THREAD_PERCENTAGE")
        print(json.dumps(res), flush=True)
