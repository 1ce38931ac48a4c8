"""TEST INFRASTRUCTURE ONLY - the CPU oracle of the SHM allreduce/broadcast.

Two independent restatements of one contract (see flexshm_oracle.c header for
the full statement and its provenance):

* `allreduce_np` - numpy, vectorised over elements, loop over ranks in
  ascending order: out = (((x0 + x1) + x2) + ...), fp32, then the scale
  convention; bf16 is widened exactly, summed in fp32, rounded once (RNE).
* `allreduce_c` / `shm_allreduce_c` - the C restatement (oracle/_build/
  liboracle.so), single-threaded checker and the multi-threaded CPU SHM
  path timed as the CPU baseline.

The reference has no arithmetic for this path (its allreduce is NCCL 2.21.5
plus an unpublished MIG patch, reference PAPER.md:353-354, 386-388, 830), so
the allreduce values are "parity unpinned" against the reference; the two
restatements are checked against each other and against torch's bf16 RNE
(tests/golden/make_golden_data.py).

Scale conventions (int codes shared with include/flexshm.h):
  OP_SUM = 0, OP_SUM_POSTSCALE = 1 (sum * factor), OP_PREDIV_SUM = 2
  (each contribution / factor, IEEE division), OP_PREMUL_SUM = 3 (each
  contribution * factor).  DDP's mean (`ddp_mean`) is OP_PREMUL_SUM with
  factor = fl32(1/world): the default hook's bucket.div_(world)
  (torch/distributed/algorithms/ddp_comm_hooks/default_hooks.py:26) multiplies
  by the fp32 reciprocal on CUDA (ATen BinaryDivTrueKernel.cu, CPU-scalar
  branch); tests/test_ddp_arith_gpu.py pins this against torch on the B200.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

F32, BF16 = 0, 1
OP_SUM, OP_SUM_POSTSCALE, OP_PREDIV_SUM, OP_PREMUL_SUM = 0, 1, 2, 3


def ddp_mean(n: int) -> tuple[int, float]:
    """(op, factor) of DDP's gradient mean over n ranks: x * fl32(1/n)."""
    return OP_PREMUL_SUM, float(np.float32(1.0) / np.float32(n))

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")


# ---------------------------------------------------------------- bf16 bits


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32)


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit patterns (NaN stays quiet NaN)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    nan = (u & np.uint32(0x7F800000)) == np.uint32(0x7F800000)
    nan &= (u & np.uint32(0x007FFFFF)) != 0
    rounded = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    quiet = (u >> np.uint32(16)) | np.uint32(0x40)
    return np.where(nan, quiet, rounded).astype(np.uint16)


# ---------------------------------------------------------------- numpy


def _contrib(x: np.ndarray, dtype: int, op: int, factor: float) -> np.ndarray:
    f = np.float32(factor)
    if dtype == F32:
        v = x.astype(np.float32, copy=False)
        return v / f if op == OP_PREDIV_SUM else v * f if op == OP_PREMUL_SUM else v
    v = bf16_to_f32(x)
    if op == OP_PREDIV_SUM:
        v = bf16_to_f32(f32_to_bf16(v / f))
    elif op == OP_PREMUL_SUM:
        v = bf16_to_f32(f32_to_bf16(v * f))
    return v


def allreduce_np(xs: list[np.ndarray], dtype: int = F32, op: int = OP_SUM,
                 factor: float = 1.0) -> np.ndarray:
    """xs[q] = rank q's buffer (float32, or uint16 bf16 bits)."""
    with np.errstate(all="ignore"):
        acc = _contrib(xs[0], dtype, op, factor).copy()
        for x in xs[1:]:
            acc = acc + _contrib(x, dtype, op, factor)
        if op == OP_SUM_POSTSCALE:
            acc = acc * np.float32(factor)
    return acc if dtype == F32 else f32_to_bf16(acc)


def broadcast_np(xs: list[np.ndarray], root: int) -> np.ndarray:
    return xs[root].copy()


# ---------------------------------------------------------------- C oracle


_MP_PATH = os.path.join(_HERE, "_build", "shm_cpu_allreduce")


def build() -> str:
    """Compile oracle/flexshm_oracle.c -> _build/liboracle.so and
    oracle/shm_cpu_allreduce.c -> _build/shm_cpu_allreduce (TEST / BASELINE
    INFRASTRUCTURE)."""
    stale = False
    for out, src in ((_LIB_PATH, "flexshm_oracle.c"), (_MP_PATH, "shm_cpu_allreduce.c")):
        src = os.path.join(_HERE, src)
        stale |= not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src)
    if stale:
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.oracle_allreduce.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                                          ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_float]
        _lib.oracle_shm_allreduce.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                                              ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_float, ctypes.c_int, ctypes.c_void_p]
        _lib.oracle_shm_allreduce.restype = ctypes.c_int
        _lib.oracle_shm_scratch_bytes.argtypes = [ctypes.c_int, ctypes.c_size_t, ctypes.c_int]
        _lib.oracle_shm_scratch_bytes.restype = ctypes.c_size_t
        _lib.oracle_inplace_allreduce.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                                                  ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                                                  ctypes.c_float, ctypes.c_int]
        _lib.oracle_inplace_allreduce.restype = ctypes.c_int
    return _lib


def _np_dtype(dtype: int):
    return np.float32 if dtype == F32 else np.uint16


def allreduce_c(xs: list[np.ndarray], dtype: int = F32, op: int = OP_SUM,
                factor: float = 1.0) -> np.ndarray:
    xs = [np.ascontiguousarray(x, dtype=_np_dtype(dtype)) for x in xs]
    out = np.empty_like(xs[0])
    ptrs = (ctypes.c_void_p * len(xs))(*[x.ctypes.data for x in xs])
    lib().oracle_allreduce(len(xs), ptrs, out.ctypes.data, out.size, dtype, op, factor)
    return out


class ShmAllreduce:
    """Multi-threaded CPU SHM allreduce over `n` rank buffers (in place)."""

    def __init__(self, n: int, count: int, dtype: int = F32, nthreads: int | None = None):
        self.n, self.count, self.dtype = n, count, dtype
        self.nthreads = nthreads or os.cpu_count() or 1
        self.scratch = np.empty(lib().oracle_shm_scratch_bytes(n, count, dtype), np.uint8)

    def __call__(self, bufs: list[np.ndarray], op: int = OP_SUM, factor: float = 1.0) -> None:
        ptrs = (ctypes.c_void_p * self.n)(*[b.ctypes.data for b in bufs])
        rc = lib().oracle_shm_allreduce(self.n, ptrs, self.count, self.dtype, op, factor,
                                        self.nthreads, self.scratch.ctypes.data)
        if rc != 0:
            raise RuntimeError(f"oracle_shm_allreduce rc={rc}")


def inplace_allreduce(bufs: list[np.ndarray], dtype: int = F32, op: int = OP_SUM,
                      factor: float = 1.0, nthreads: int | None = None) -> None:
    """In-place threaded rank-order reduction over n host buffers (one
    address space, no staging): the host-memory bound next to the GPU e2e."""
    ptrs = (ctypes.c_void_p * len(bufs))(*[b.ctypes.data for b in bufs])
    rc = lib().oracle_inplace_allreduce(len(bufs), ptrs, bufs[0].size, dtype, op, factor,
                                        nthreads or os.cpu_count() or 1)
    if rc != 0:
        raise RuntimeError(f"oracle_inplace_allreduce rc={rc}")


def host_cores() -> list[int]:
    """The host cores this process may run on."""
    return sorted(os.sched_getaffinity(0))


def mp_shm_allreduce(n: int, count: int, dtype: int = F32, op: int = OP_SUM,
                     factor: float = 1.0, iters: int = 1, warmup: int = 0,
                     cores: list[int] | None = None, xs: list[np.ndarray] | None = None,
                     want_out: bool = False, timeout: float = 600.0):
    """Run the multi-process POSIX-SHM CPU allreduce (oracle/shm_cpu_allreduce.c:
    one process per rank pinned to its own core).  xs: the
    ranks' inputs (default: the program's synthetic data).  Returns (stats
    dict, outputs [n][count] or None)."""
    import json
    import tempfile
    build()
    cores = host_cores() if cores is None else cores
    esz = 4 if dtype == F32 else 2
    tmp = tempfile.mkdtemp(prefix="fmx-cpuref-", dir="/dev/shm" if os.path.isdir("/dev/shm")
                           else None)
    inp, outp = "-", "-"
    try:
        if xs is not None:
            inp = os.path.join(tmp, "in")
            np.concatenate([np.ascontiguousarray(x, _np_dtype(dtype)) for x in xs]).tofile(inp)
        if want_out:
            outp = os.path.join(tmp, "out")
        r = subprocess.run([_MP_PATH, str(n), str(count), str(dtype), str(op), repr(float(factor)),
                            str(iters), str(warmup), ",".join(map(str, cores)), inp, outp],
                           capture_output=True, text=True, timeout=timeout)
        if r.returncode != 0:
            raise RuntimeError(f"shm_cpu_allreduce rc={r.returncode}: {r.stderr[-500:]}")
        stats = json.loads(r.stdout.strip().splitlines()[-1])
        outs = None
        if want_out:
            flat = np.fromfile(outp, dtype=_np_dtype(dtype))
            outs = [flat[i * count:(i + 1) * count].copy() for i in range(n)]
        return stats, outs
    finally:
        for f in ("in", "out"):
            try:
                os.unlink(os.path.join(tmp, f))
            except OSError:
                pass
        os.rmdir(tmp)


# ---------------------------------------------------------------- inputs


def synthetic_gradient(rank: int, count: int, dtype: int = F32, seed: int = 1234) -> np.ndarray:
    """SURVEY §8d inputs: rank r draws N(0,1) with seed 1234+r, x1e-3 (fp32)
    or x1e-2 rounded to bf16 bits."""
    rng = np.random.default_rng(seed + rank)
    g = rng.standard_normal(count, dtype=np.float32)
    if dtype == F32:
        return g * np.float32(1e-3)
    return f32_to_bf16(g * np.float32(1e-2))


def adversarial(rank: int, count: int, dtype: int = F32) -> np.ndarray:
    """Order-sensitive values: +-1e8 alternating with 1.0, signed zeros,
    subnormals, +-inf and NaN at fixed positions."""
    i = np.arange(count)
    x = np.where(i % 2 == 0, np.float32(1e8) * (1 if rank % 2 == 0 else -1), np.float32(1.0))
    x = x.astype(np.float32)
    x[i % 7 == 3] = np.float32(-0.0) if rank % 2 else np.float32(0.0)
    x[i % 11 == 5] = np.float32(1e-40) * (rank + 1)   # subnormal
    x[i % 97 == 13] = np.float32(np.inf) if rank == 0 else np.float32(1.0)
    x[i % 101 == 17] = np.float32(np.nan) if rank == 1 else np.float32(2.0)
    x[i % 103 == 19] = np.float32(3.4e38)              # overflow to inf when summed
    return x if dtype == F32 else f32_to_bf16(x)
