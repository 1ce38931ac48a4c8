"""fmx_reduce_kernel alone (fmx_reduce_local) against the oracle, in one
process: every dtype/op, source counts 1..64, lengths around the vector
width, unaligned pointers (scalar path), mapped-host sources (cache-volatile
loads) and the zero-copy store of the result to pinned host memory."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu

OPS = {"sum": orc.OP_SUM, "postscale": orc.OP_SUM_POSTSCALE, "prediv": orc.OP_PREDIV_SUM,
       "premul": orc.OP_PREMUL_SUM}


def to_torch(x, dtype, device):
    import torch
    t = torch.from_numpy(x.view(np.int16)).view(torch.bfloat16) if dtype == orc.BF16 \
        else torch.from_numpy(x)
    return t.to(device) if device == "cuda" else t.pin_memory()


def to_np(t, dtype):
    import torch
    t = t.cpu()
    return t.view(torch.int16).numpy().view(np.uint16) if dtype == orc.BF16 else t.numpy()


def bits_equal_nan_aware(a, b, dtype):
    fa = orc.bf16_to_f32(a) if dtype == orc.BF16 else a
    fb = orc.bf16_to_f32(b) if dtype == orc.BF16 else b
    na, nb = np.isnan(fa), np.isnan(fb)
    va = a.view(np.uint32) if dtype == orc.F32 else a
    vb = b.view(np.uint32) if dtype == orc.F32 else b
    return np.array_equal(na, nb) and np.array_equal(va[~na], vb[~nb])


@pytest.mark.parametrize("dtype", [orc.F32, orc.BF16])
@pytest.mark.parametrize("op,factor", [("sum", 1.0), ("postscale", 0.25), ("prediv", 7.0),
                                       ("premul", 1.0 / 7.0), ("premul", 0.1)])
@pytest.mark.parametrize("n", [1, 2, 7, 9, 64])
@pytest.mark.parametrize("count", [1, 7, 8, 9, 4099, 300_001])
def test_reduce_kernel_matches_oracle(dtype, op, factor, n, count):
    import torch
    from paper_2511_09143_b200.comm import reduce_local
    xs = [orc.synthetic_gradient(r, count, dtype) for r in range(n)]
    if n >= 2:
        xs[1] = orc.adversarial(1, count, dtype)
    host_idx = [q for q in range(n) if q % 3 == 2]      # some sources in mapped host memory
    srcs = [to_torch(x, dtype, "cpu" if q in host_idx else "cuda") for q, x in enumerate(xs)]
    out = torch.empty_like(to_torch(xs[0], dtype, "cuda"))
    out_host = torch.empty(out.shape, dtype=out.dtype).pin_memory()
    reduce_local(srcs, out, op=op, factor=factor, out_host=out_host, host_sources=host_idx)
    torch.cuda.synchronize()
    want = orc.allreduce_c(xs, dtype, OPS[op], factor)
    assert bits_equal_nan_aware(to_np(out, dtype), want, dtype)
    assert bits_equal_nan_aware(to_np(out_host, dtype), want, dtype)


def test_reduce_kernel_unaligned_scalar_path():
    import torch
    from paper_2511_09143_b200.comm import reduce_local
    n, count = 5, 10_001
    xs = [orc.synthetic_gradient(r, count + 1, orc.F32) for r in range(n)]
    srcs = [torch.from_numpy(x).cuda()[1:] for x in xs]      # 4-byte offset
    out = torch.empty(count + 1, device="cuda")[1:]
    reduce_local(srcs, out, op="avg")
    torch.cuda.synchronize()
    want = orc.allreduce_c([x[1:] for x in xs], orc.F32, *orc.ddp_mean(n))
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32))
