"""One full pipeline piece of the CE transport's reduction, for ncu: 7 HBM
sources of one slice each (4 MiB), rank-order fp32 sum with DDP's pre-divide,
result to HBM and (zero-copy) to a pinned host slot - exactly what
fmx_reduce_kernel does per round of the default configuration."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_09143_b200.comm import reduce_local  # noqa: E402

n = int(os.environ.get("FMX_N", "7"))
piece = int(os.environ.get("FMX_PIECE_BYTES", str(4 << 20))) // 4
srcs = [torch.randn(piece, device="cuda") for _ in range(n)]
out = torch.empty(piece, device="cuda")
out_host = torch.empty(piece).pin_memory()
for _ in range(int(os.environ.get("FMX_ITERS", "5"))):
    reduce_local(srcs, out, op="avg", out_host=out_host)
torch.cuda.synchronize()
print("ok", n, piece * 4)
