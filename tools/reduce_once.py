"""One full pipeline piece of the CE transport's reduction, for ncu: 7 HBM
sources of one slice each (4 MiB), rank-order fp32 sum with DDP's pre-divide,
result to HBM and (zero-copy) to a pinned host slot - exactly what
fmx_reduce_kernel does per round of the default configuration.

FMX_NO_HOST=1: no zero-copy result (the result slot written by a copy engine,
FMX_RESULT_VIA_CE / the fetch lane's CE result): the HBM-only launch.
FMX_GREEN=1: run inside a 1g-sized green-context partition (instance.bind),
as a rank does, instead of on the whole GPU."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_09143_b200.comm import reduce_local  # noqa: E402

stream = None
if os.environ.get("FMX_GREEN", "0") != "0":
    from paper_2511_09143_b200 import instance  # noqa: E402
    inst = instance.bind(0, 1, mode="green")
    stream = inst.stream
    torch.cuda.set_stream(stream)
n = int(os.environ.get("FMX_N", "7"))
piece = int(os.environ.get("FMX_PIECE_BYTES", str(4 << 20))) // 4
srcs = [torch.randn(piece, device="cuda") for _ in range(n)]
out = torch.empty(piece, device="cuda")
out_host = None if os.environ.get("FMX_NO_HOST", "0") != "0" else torch.empty(piece).pin_memory()
for _ in range(int(os.environ.get("FMX_ITERS", "5"))):
    reduce_local(srcs, out, op="avg", out_host=out_host, stream=stream)
torch.cuda.synchronize()
if os.environ.get("FMX_TIME", "0") != "0":   # not under a profiler: CUDA events on the stream
    s = stream if stream is not None else torch.cuda.current_stream()
    k = 50
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(s)
    for _ in range(k):
        reduce_local(srcs, out, op="avg", out_host=out_host, stream=stream)
    t1.record(s)
    t1.synchronize()
    us = t0.elapsed_time(t1) * 1e3 / k
    hbm = (n + 1) * piece * 4
    print(f"time n={n} piece={piece * 4} host={out_host is not None} "
          f"green={stream is not None} us={us:.1f} hbm_gbs={hbm / us / 1e3:.0f}")
print("ok", n, piece * 4)
