"""Probe: why is a CUDA-graph replay of a BERT-base training step slower than
eager inside a 14 % MPS client (r02/r2s), while ResNet-50's is faster?  Times,
eager vs graph, in one process: BERT fwd+bwd with SDPA / eager attention, and
bare bf16 GEMMs of BERT's shapes.  Prints JSON lines."""
import json
import os

import torch
import torch.nn.functional as F


def timed(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = torch.cuda.current_stream()
    e0.record(s)
    for _ in range(iters):
        fn()
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / iters


def both(name, fn, **kw):
    eager = timed(fn)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    graph = timed(g.replay)
    print(json.dumps({"probe": "mps_graph", "case": name, "eager_ms": round(eager, 3),
                      "graph_ms": round(graph, 3),
                      "mps_pct": os.environ.get("CUDA_MPS_ACTIVE_THREAD_PERCENTAGE"), **kw}),
          flush=True)


s = torch.cuda.Stream()
with torch.cuda.stream(s):
    # bare GEMMs of BERT-base's shapes (tokens = 32 x 128), bf16
    a = torch.randn(4096, 768, device="cuda", dtype=torch.bfloat16)
    w1 = torch.randn(3072, 768, device="cuda", dtype=torch.bfloat16)
    w2 = torch.randn(768, 768, device="cuda", dtype=torch.bfloat16)

    def gemms():
        for _ in range(20):
            h = F.linear(a, w1)
            F.linear(a, w2)
            F.linear(h, w1.t())
    both("gemm_ffn_qkv_x20", gemms)

    from torch.nn.attention import SDPBackend, sdpa_kernel
    from transformers import BertConfig, BertForSequenceClassification
    torch.manual_seed(0)
    model = BertForSequenceClassification(BertConfig(num_labels=2)).cuda().to(torch.bfloat16).eval()
    x = torch.randint(0, 30522, (32, 128), device="cuda")
    for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION,
               SDPBackend.EFFICIENT_ATTENTION, SDPBackend.MATH):
        try:
            with sdpa_kernel([be]):
                both(f"bert_fwd_eval_{be.name}", lambda: model(input_ids=x))
        except Exception as exc:  # noqa: BLE001
            print(json.dumps({"probe": "mps_graph", "case": f"bert_fwd_eval_{be.name}",
                              "error": repr(exc)[:200]}), flush=True)
    # single layers of the encoder
    h = torch.randn(32, 128, 768, device="cuda", dtype=torch.bfloat16)
    ln = torch.nn.LayerNorm(768).cuda().to(torch.bfloat16)
    both("layernorm_x20", lambda: [ln(h) for _ in range(20)])
    both("gelu_x20", lambda: [F.gelu(h) for _ in range(20)])
    q = torch.randn(32, 12, 128, 64, device="cuda", dtype=torch.bfloat16)
    for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION,
               SDPBackend.EFFICIENT_ATTENTION, SDPBackend.MATH):
        try:
            with sdpa_kernel([be]):
                both(f"sdpa_x20_{be.name}",
                     lambda: [F.scaled_dot_product_attention(q, q, q) for _ in range(20)])
        except Exception as exc:  # noqa: BLE001
            print(json.dumps({"probe": "mps_graph", "case": f"sdpa_x20_{be.name}",
                              "error": repr(exc)[:200]}), flush=True)
    for attn in ("sdpa",):
        torch.manual_seed(0)
        model = BertForSequenceClassification(BertConfig(num_labels=2, attn_implementation=attn)) \
            .cuda().to(torch.bfloat16)
        x = torch.randint(0, 30522, (32, 128), device="cuda")
        y = torch.randint(0, 2, (32,), device="cuda")

        def fwd():
            return F.cross_entropy(model(input_ids=x).logits.float(), y)

        def fwd_bwd():
            model.zero_grad(set_to_none=False)
            fwd().backward()
        both(f"bert_fwd_{attn}", fwd)
        both(f"bert_fwd_bwd_{attn}", fwd_bwd)
        model.eval()
        both(f"bert_fwd_nodropout_{attn}", fwd)
