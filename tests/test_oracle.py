"""The CPU oracle itself: the C and numpy restatements agree bit for bit on
normal, adversarial and bf16 inputs under all three scale conventions; the
multi-threaded CPU SHM path (the timed baseline) equals the single-threaded
checker; bf16 rounding is pinned to torch's RNE conversion; and the fixed
rank order really is observable (a different association changes bits)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as orc


def bits(a):
    return a.view(np.uint32) if a.dtype == np.float32 else a


def same(a, b):
    fa = a if a.dtype == np.float32 else orc.bf16_to_f32(a)
    fb = b if b.dtype == np.float32 else orc.bf16_to_f32(b)
    na, nb = np.isnan(fa), np.isnan(fb)
    return np.array_equal(na, nb) and np.array_equal(bits(a)[~na], bits(b)[~nb])


@pytest.mark.parametrize("dtype", [orc.F32, orc.BF16])
@pytest.mark.parametrize("op,factor", [(orc.OP_SUM, 1.0), (orc.OP_SUM_POSTSCALE, 0.125),
                                       (orc.OP_PREDIV_SUM, 7.0), (orc.OP_PREDIV_SUM, 3.0),
                                       (orc.OP_PREMUL_SUM, 1 / 7), (orc.OP_PREMUL_SUM, 0.1)])
@pytest.mark.parametrize("n", [1, 2, 7, 14])
def test_c_and_numpy_restatements_agree(dtype, op, factor, n):
    count = 10_007
    xs = [orc.synthetic_gradient(r, count, dtype) for r in range(n)]
    xs += [orc.adversarial(r, count, dtype) for r in range(2)]
    assert same(orc.allreduce_np(xs, dtype, op, factor), orc.allreduce_c(xs, dtype, op, factor))


@pytest.mark.parametrize("dtype", [orc.F32, orc.BF16])
@pytest.mark.parametrize("n,count,threads", [(2, 1, 3), (7, 5, 2), (7, 100_003, 4), (3, 64, 8)])
def test_cpu_shm_path_equals_checker(dtype, n, count, threads):
    xs = [orc.synthetic_gradient(r, count, dtype) for r in range(n)]
    want = orc.allreduce_c(xs, dtype, *orc.ddp_mean(n))
    bufs = [x.copy() for x in xs]
    orc.ShmAllreduce(n, count, dtype, threads)(bufs, *orc.ddp_mean(n))
    for b in bufs:
        assert same(b, want)


def test_bf16_rounding_matches_torch_rne():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(5)
    x = rng.standard_normal(200_000).astype(np.float32) * np.float32(100)
    # exact ties and specials
    ties = (np.arange(1, 1000, dtype=np.uint32) << 16 | np.uint32(0x8000)).view(np.float32)
    special = np.array([0.0, -0.0, np.inf, -np.inf, 1e-40, -1e-40, 3.4e38, 1.0000001],
                       dtype=np.float32)
    x = np.concatenate([x, ties, special])
    want = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(orc.f32_to_bf16(x), want)
    nan = orc.f32_to_bf16(np.array([np.nan], dtype=np.float32))
    assert np.isnan(orc.bf16_to_f32(nan))[0]


def test_summation_order_is_observable():
    """The contract is a fixed left-to-right rank order: another association
    of the same values gives different bits on ordinary gradients."""
    n, count = 7, 200_000
    xs = [orc.synthetic_gradient(r, count) for r in range(n)]
    left = orc.allreduce_np(xs)
    pairwise = ((xs[0] + xs[1]) + (xs[2] + xs[3])) + ((xs[4] + xs[5]) + xs[6])
    assert not np.array_equal(left.view(np.uint32), pairwise.view(np.uint32))


def test_golden_allreduce_vectors():
    """Small committed vectors (tests/golden/make_golden_data.py, torch fp32
    elementwise adds in rank order + torch bf16 RNE)."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "allreduce_golden.npz")
    g = np.load(path)
    for key in sorted(k for k in g.files if k.endswith("_out")):
        stem = key[:-4]
        meta = g[stem + "_meta"]
        n, dtype, op, factor = int(meta[0]), int(meta[1]), int(meta[2]), float(meta[3])
        xs = [g[f"{stem}_in{r}"] for r in range(n)]
        assert same(orc.allreduce_c(xs, dtype, op, factor), g[key]), stem
        assert same(orc.allreduce_np(xs, dtype, op, factor), g[key]), stem


@pytest.mark.parametrize("dtype", [orc.F32, orc.BF16])
@pytest.mark.parametrize("n,count,cores", [(2, 1, None), (7, 100_003, None), (4, 3_504_872 // 64, [0]),
                                           (14, 4099, [0, 1])])
def test_multiprocess_shm_cpu_path_equals_checker(dtype, n, count, cores):
    """BASELINE.md §3's CPU reference path - one process per rank over a POSIX
    SHM segment (oracle/shm_cpu_allreduce.c) - is bit-identical to the
    checker, also when ranks outnumber the cores it is given."""
    xs = [orc.synthetic_gradient(r, count, dtype) for r in range(n)]
    xs[0] = orc.adversarial(0, count, dtype)
    for op, factor in (orc.ddp_mean(n), (orc.OP_SUM, 1.0)):
        want = orc.allreduce_c(xs, dtype, op, factor)
        stats, outs = orc.mp_shm_allreduce(n, count, dtype, op, factor, xs=xs, want_out=True,
                                           cores=cores)
        assert stats["processes"] == n
        assert stats["oversubscribed"] == (cores is not None and len(cores) < n)
        for r in range(n):
            assert same(outs[r], want), r


@pytest.mark.parametrize("dtype", [orc.F32, orc.BF16])
def test_inplace_host_reduction_equals_checker(dtype):
    n, count = 7, 50_001
    xs = [orc.synthetic_gradient(r, count, dtype) for r in range(n)]
    want = orc.allreduce_c(xs, dtype, *orc.ddp_mean(n))
    bufs = [x.copy() for x in xs]
    orc.inplace_allreduce(bufs, dtype, *orc.ddp_mean(n), nthreads=3)
    for b in bufs:
        assert same(b, want)
