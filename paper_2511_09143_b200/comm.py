"""Process-group init over a set of instances, and the collectives.

New Python surface (the reference has none; shaped like torch / NCCL):

    comm = init_process_group(decision, rank, job_key, instance=inst)
    comm.allreduce(flat_grad)                 # fixed rank-order fp32 sum
    comm.allreduce(flat_grad, op="avg")       # DDP's mean: sum of x * fl32(1/n)
    comm.reduce_scatter(full, block)          # NCCL layouts
    comm.allgather(block, full)
    comm.broadcast(flat_params, root=0)
    comm.allreduce_host(comm.host_buffer()[:nbytes].view(torch.float32))  # host-resident data
    comm.set_join_stream(side)                # complete on `side`, not the calling stream
    comm.destroy()

`decision` is the `AllocationDecision` from `fm_select`; its `instances`
order is the rank order (reference scheduler.py:117-136), which is also the
summation order of every allreduce.  Bootstrap runs natively inside
`fmx_comm_init` (MIG-aware duplicate check and topology labels, reference
commsim.py:67-116 / PAPER.md:386-399); the Python side then rebuilds the
reference's `Communicator` and `TopologyGraph` from the exchanged peer table
so callers see the same objects `discover_peers` / `build_topology` return.
"""

from __future__ import annotations

import ctypes
import math

from . import _lib
from .commsim import Communicator, PeerInfo, TopologyGraph, build_topology, discover_peers
from .scheduler import AllocationDecision

OPS = {
    "sum": _lib.OP_SUM,
    "postscale": _lib.OP_SUM_POSTSCALE,
    "prediv": _lib.OP_PREDIV_SUM,
    "premul": _lib.OP_PREMUL_SUM,
}


def mean_factor(n: int) -> float:
    """fl32(1/n), the multiplier of DDP's mean.  The default comm hook does
    `bucket.div_(world)` (torch/distributed/algorithms/ddp_comm_hooks/
    default_hooks.py:26); for a CPU-scalar divisor ATen's CUDA kernel
    multiplies by the fp32 reciprocal (BinaryDivTrueKernel.cu), and the
    hook-less reducer multiplies by 1/div_factor - so "avg" is PREMUL_SUM
    with this factor, bit-exact with DDP on the B200
    (tests/test_ddp_arith_gpu.py)."""
    import numpy as np
    return float(np.float32(1.0) / np.float32(n))


def resolve_op(op: str, factor: float | None, n: int) -> tuple[str, float]:
    """Map the user-facing op name (+ optional factor) to (native op, factor)."""
    if op == "avg":
        return "premul", mean_factor(n)
    if op not in OPS:
        raise ValueError(f"unknown op {op!r}")
    factor = 1.0 if factor is None else float(factor)
    if op != "sum" and not math.isfinite(factor):
        raise ValueError("factor must be finite")
    return op, factor


def _dtype_code(tensor) -> int:
    import torch
    if tensor.dtype == torch.float32:
        return _lib.FLOAT32
    if tensor.dtype == torch.bfloat16:
        return _lib.BFLOAT16
    raise TypeError(f"unsupported dtype {tensor.dtype} (float32 or bfloat16)")


def _check_tensor(t, what: str):
    if not t.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous (flat gradient buffer)")


def reduce_local(sources, out, op: str = "sum", factor: float | None = None, out_host=None,
                 host_sources=(), stream=None):
    """The owner-side reduction kernel alone: out = rank-order fp32 sum of
    `sources` (same-size CUDA tensors, or host tensors listed by index in
    `host_sources` that live in mapped pinned memory), op/factor as in
    allreduce; `out_host` (pinned host tensor) also receives the result."""
    import torch
    op, factor = resolve_op(op, factor, len(sources))
    ptrs = (ctypes.c_void_p * len(sources))(*[t.data_ptr() for t in sources])
    mask = 0
    for q in host_sources:
        mask |= 1 << q
    s = stream if stream is not None else torch.cuda.current_stream()
    rc = _lib.lib().fmx_reduce_local(ptrs, len(sources), mask, out.data_ptr(),
                                     out_host.data_ptr() if out_host is not None else None,
                                     out.numel(), _dtype_code(out), OPS[op], ctypes.c_float(factor),
                                     int(s.cuda_stream))
    _lib.check(rc, "fmx_reduce_local")
    return out


class ShmCommunicator:
    """Handle of one rank's membership in a host-SHM communicator."""

    def __init__(self, handle: int, rank: int, peers: list[PeerInfo], instance=None):
        self._h = ctypes.c_void_p(handle)
        self.rank = rank
        self.size = len(peers)
        self.comm: Communicator = Communicator(tuple(peers))
        self.topology: TopologyGraph = build_topology(self.comm)
        self.instance = instance
        sb, tr, shm = ctypes.c_size_t(), ctypes.c_int(), ctypes.c_size_t()
        _lib.check(_lib.lib().fmx_comm_config(self._h, ctypes.byref(sb), ctypes.byref(tr),
                                              ctypes.byref(shm)))
        self.slice_bytes, self.transport, self.shm_bytes = sb.value, tr.value, shm.value

    # -- helpers -------------------------------------------------------------
    def _stream(self, stream) -> int:
        import torch
        if stream is None:
            stream = torch.cuda.current_stream()
        return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)

    def _alive(self):
        if self._h is None or not self._h.value:
            raise RuntimeError("communicator was destroyed")

    # -- collectives -----------------------------------------------------------
    def allreduce(self, tensor, op: str = "sum", factor: float | None = None, out=None,
                  stream=None):
        """In-place (or into `out`) allreduce of a flat float32/bf16 buffer.

        op: "sum"; "avg" (DDP's mean: each contribution * fl32(1/size),
        = "premul" with mean_factor(size)); "premul" (each contribution *
        factor); "prediv" (each contribution / factor, IEEE division);
        "postscale" (sum * factor).
        """
        self._alive()
        _check_tensor(tensor, "tensor")
        op, factor = resolve_op(op, factor, self.size)
        dst = tensor if out is None else out
        if dst is not tensor:
            _check_tensor(dst, "out")
            if dst.dtype != tensor.dtype or dst.numel() != tensor.numel():
                raise ValueError("out must match tensor dtype and size")
        rc = _lib.lib().fmx_allreduce(self._h, tensor.data_ptr(), dst.data_ptr(),
                                      tensor.numel(), _dtype_code(tensor), OPS[op],
                                      ctypes.c_float(factor), self._stream(stream))
        _lib.check(rc, "fmx_allreduce")
        return dst

    def shard(self, count: int, dtype=None) -> tuple[int, int]:
        """(offset, len) of this rank's owner chunk of an allreduce of `count`
        elements (fmx_allreduce_shard)."""
        import torch
        code = _dtype_code(torch.empty(0, dtype=dtype or torch.float32))
        off, ln = ctypes.c_size_t(), ctypes.c_size_t()
        _lib.check(_lib.lib().fmx_allreduce_shard(self._h, int(count), code, ctypes.byref(off),
                                                  ctypes.byref(ln)), "fmx_allreduce_shard")
        return off.value, ln.value

    def allreduce_sgd(self, grad, param, momentum, lr: float, momentum_coef: float = 0.0,
                      dampening: float = 0.0, weight_decay: float = 0.0, nesterov: bool = False,
                      first_step: bool = False, op: str = "avg", stream=None):
        """Fused optimizer step (fmx_allreduce_sgd): `param` <- torch's SGD step
        with the `op`-reduced `grad`, computed once by each chunk's owner and
        all-gathered.  `momentum`: this rank's shard (self.shard(numel)), fp32."""
        self._alive()
        _check_tensor(grad, "grad")
        _check_tensor(param, "param")
        if grad.dtype != param.dtype or grad.numel() != param.numel():
            raise ValueError("grad and param must match in dtype and size")
        op, factor = resolve_op(op, None, self.size)
        sgd = _lib.SgdC(lr, momentum_coef, dampening, weight_decay, int(bool(nesterov)),
                        int(bool(first_step)))
        mom = momentum.data_ptr() if momentum is not None else None
        rc = _lib.lib().fmx_allreduce_sgd(self._h, grad.data_ptr(), param.data_ptr(), mom,
                                          grad.numel(), OPS[op], ctypes.c_float(factor),
                                          ctypes.byref(sgd), self._stream(stream))
        _lib.check(rc, "fmx_allreduce_sgd")
        return param

    def broadcast(self, tensor, root: int = 0, stream=None):
        self._alive()
        _check_tensor(tensor, "tensor")
        rc = _lib.lib().fmx_broadcast(self._h, tensor.data_ptr(), tensor.data_ptr(),
                                      tensor.numel(), _dtype_code(tensor), int(root),
                                      self._stream(stream))
        _lib.check(rc, "fmx_broadcast")
        return tensor

    def reduce_scatter(self, tensor, out, op: str = "sum", factor: float | None = None,
                       stream=None):
        """NCCL layout: `tensor` holds size * out.numel() elements; this rank
        receives the rank-order reduction of its block (op/factor as in
        allreduce) in `out`."""
        self._alive()
        _check_tensor(tensor, "tensor")
        _check_tensor(out, "out")
        if out.dtype != tensor.dtype or tensor.numel() != out.numel() * self.size:
            raise ValueError("tensor must hold size * out.numel() elements of out's dtype")
        op, factor = resolve_op(op, factor, self.size)
        rc = _lib.lib().fmx_reduce_scatter(self._h, tensor.data_ptr(), out.data_ptr(), out.numel(),
                                           _dtype_code(tensor), OPS[op], ctypes.c_float(factor),
                                           self._stream(stream))
        _lib.check(rc, "fmx_reduce_scatter")
        return out

    def allgather(self, tensor, out, stream=None):
        """NCCL layout: every rank's `tensor` lands at out[r * tensor.numel()]."""
        self._alive()
        _check_tensor(tensor, "tensor")
        _check_tensor(out, "out")
        if out.dtype != tensor.dtype or out.numel() != tensor.numel() * self.size:
            raise ValueError("out must hold size * tensor.numel() elements of tensor's dtype")
        rc = _lib.lib().fmx_allgather(self._h, tensor.data_ptr(), out.data_ptr(), tensor.numel(),
                                      _dtype_code(tensor), self._stream(stream))
        _lib.check(rc, "fmx_allgather")
        return out

    def host_buffer(self, rank: int | None = None):
        """This rank's (or `rank`'s) registered host buffer as a uint8 CPU
        tensor over the pinned, device-mapped SHM region (no copy)."""
        import numpy as np
        import torch
        ptr, nbytes = ctypes.c_void_p(), ctypes.c_size_t()
        _lib.check(_lib.lib().fmx_host_buffer(self._h, self.rank if rank is None else rank,
                                              ctypes.byref(ptr), ctypes.byref(nbytes)))
        if nbytes.value == 0:
            raise ValueError("communicator was created with host_bytes=0")
        arr = np.ctypeslib.as_array((ctypes.c_uint8 * nbytes.value).from_address(ptr.value))
        return torch.from_numpy(arr)

    def allreduce_host(self, tensor, op: str = "sum", factor: float | None = None, stream=None):
        """In-place allreduce of `tensor`, a view into this rank's host_buffer()
        (float32 / bfloat16): inputs are read and results written over the host
        link directly, no device copy of the buffer is made."""
        self._alive()
        base = self.host_buffer()
        offset = tensor.data_ptr() - base.data_ptr()
        if tensor.is_cuda or not tensor.is_contiguous() or offset < 0 or \
                offset + tensor.numel() * tensor.element_size() > base.numel():
            raise ValueError("tensor must be a contiguous view into host_buffer()")
        op, factor = resolve_op(op, factor, self.size)
        rc = _lib.lib().fmx_allreduce_host(self._h, offset, tensor.numel(), _dtype_code(tensor),
                                           OPS[op], ctypes.c_float(factor), self._stream(stream))
        _lib.check(rc, "fmx_allreduce_host")
        return tensor

    def barrier(self, timeout_s: float = 120.0) -> None:
        self._alive()
        _lib.check(_lib.lib().fmx_barrier(self._h, timeout_s), "fmx_barrier")

    def kernel_launches(self) -> int:
        v = ctypes.c_uint64()
        _lib.check(_lib.lib().fmx_comm_kernel_launches(self._h, ctypes.byref(v)))
        return v.value

    def set_kernel_timing(self, on: bool) -> None:
        """Bracket every reduction kernel with CUDA events (on its own stream)."""
        _lib.check(_lib.lib().fmx_comm_set_timing(self._h, 1 if on else 0))

    def kernel_time(self) -> tuple[float, int]:
        """(summed device ms, launches) of the reduction kernels timed so far."""
        ms, n = ctypes.c_double(), ctypes.c_uint64()
        _lib.check(_lib.lib().fmx_comm_kernel_time(self._h, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def monitor(self, seconds: float, cap: int = 1 << 20) -> list[tuple[int, int, int, int]]:
        """Poll every rank's flags from the host for `seconds` (call it from a
        helper thread while collectives run): [(ns, rank, flag, value)]."""
        buf = (ctypes.c_uint64 * (2 * cap))()
        n = ctypes.c_size_t()
        _lib.check(_lib.lib().fmx_comm_monitor(self._h, seconds, buf, 2 * cap, ctypes.byref(n)))
        return [(buf[2 * i], buf[2 * i + 1] >> 48, (buf[2 * i + 1] >> 32) & 0xFFFF,
                 buf[2 * i + 1] & 0xFFFFFFFF) for i in range(n.value)]

    def set_stamps(self, capacity: int) -> None:
        """Timeline probe on (capacity entries) or off (0); see fmx_comm_set_stamps."""
        _lib.check(_lib.lib().fmx_comm_set_stamps(self._h, int(capacity)), "fmx_comm_set_stamps")

    def set_join_stream(self, stream) -> None:
        """Collectives join into `stream` instead of the calling stream (None:
        back to the default); see fmx_comm_set_join_stream."""
        h = 0 if stream is None else self._stream(stream)
        _lib.check(_lib.lib().fmx_comm_set_join_stream(self._h, h or None),
                   "fmx_comm_set_join_stream")

    def completion_stream(self) -> int:
        """cudaStream_t (as int) the last collective completed on."""
        s = ctypes.c_void_p()
        _lib.check(_lib.lib().fmx_comm_completion_stream(self._h, ctypes.byref(s)),
                   "fmx_comm_completion_stream")
        return s.value or 0

    def stamp(self, info: int, stream=None) -> None:
        """Caller's marker (op kind 7) on the timeline, enqueued on `stream`."""
        _lib.check(_lib.lib().fmx_comm_stamp(self._h, self._stream(stream), int(info)),
                   "fmx_comm_stamp")

    def stamps(self, cap: int = 1 << 16) -> list[tuple[int, int, int, int]]:
        """[(t_ns, lane, op kind, info)] of the stamps recorded so far."""
        buf = (ctypes.c_uint64 * (2 * cap))()
        n = ctypes.c_size_t()
        _lib.check(_lib.lib().fmx_comm_stamps(self._h, buf, 2 * cap, ctypes.byref(n)),
                   "fmx_comm_stamps")
        out = []
        for i in range(n.value):
            t, w = buf[2 * i], buf[2 * i + 1]
            tag, info = w >> 32, w & 0xFFFFFFFF
            out.append((t, tag >> 8, tag & 0xFF, info))
        return out

    def set_defer(self, on: bool) -> None:
        """Deferred gather (fmx_comm_set_defer): an allreduce's last gather is
        enqueued by the next collective / flush()."""
        self._alive()
        _lib.check(_lib.lib().fmx_comm_set_defer(self._h, int(bool(on))), "fmx_comm_set_defer")

    def flush(self, stream=None) -> None:
        """Enqueue a deferred gather, if any, on `stream` (or the join stream)."""
        self._alive()
        _lib.check(_lib.lib().fmx_comm_flush(self._h, self._stream(stream)), "fmx_comm_flush")

    # -- fences and CUDA graphs (fmx_comm_fence, fmx_graph_*) ------------------
    def fence(self, stream=None) -> None:
        """Every rank reached this point of its stream (after its earlier
        collectives); see fmx_comm_fence."""
        self._alive()
        _lib.check(_lib.lib().fmx_comm_fence(self._h, self._stream(stream)), "fmx_comm_fence")

    def capture_begin(self) -> None:
        """Announce a stream capture of collectives (before cudaStreamBeginCapture
        / torch.cuda.graph)."""
        self._alive()
        _lib.check(_lib.lib().fmx_graph_capture_begin(self._h), "fmx_graph_capture_begin")

    def capture_end(self, graph) -> int:
        """After the capture ended, before instantiation: `graph` is the captured
        cudaGraph_t (int, e.g. torch CUDAGraph(keep_graph=True).raw_cuda_graph()).
        Appends the end-of-replay fence; returns the graph handle."""
        self._alive()
        h = ctypes.c_int()
        _lib.check(_lib.lib().fmx_graph_capture_end(self._h, ctypes.c_void_p(int(graph) or None),
                                                    ctypes.byref(h)), "fmx_graph_capture_end")
        return h.value

    def launch_prepare(self, handle: int, graph_exec, stream=None) -> None:
        """Before every launch of an instance (cudaGraphExec_t as int) of
        captured graph `handle` on `stream`."""
        self._alive()
        _lib.check(_lib.lib().fmx_graph_launch_prepare(self._h, int(handle),
                                                       ctypes.c_void_p(int(graph_exec)),
                                                       self._stream(stream)),
                   "fmx_graph_launch_prepare")

    def graph_release(self, handle: int) -> None:
        self._alive()
        _lib.check(_lib.lib().fmx_graph_release(self._h, int(handle)), "fmx_graph_release")

    def flags(self) -> list[list[int]]:
        """Every rank's [STAGED, REDUCED, BC_STAGED, BC_DONE] counters."""
        buf = (ctypes.c_uint32 * (4 * self.size))()
        _lib.check(_lib.lib().fmx_comm_flags(self._h, buf, 4 * self.size))
        return [list(buf[4 * r:4 * r + 4]) for r in range(self.size)]

    def abort(self) -> None:
        if self._h is not None and self._h.value:
            _lib.lib().fmx_comm_abort(self._h)

    def destroy(self) -> None:
        if self._h is not None and self._h.value:
            h, self._h = self._h, None
            _lib.check(_lib.lib().fmx_comm_destroy(h), "fmx_comm_destroy")

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.destroy()


def init_process_group(decision: AllocationDecision | None, rank: int, job_key: str, *,
                       instance=None, peer: PeerInfo | None = None, nranks: int | None = None,
                       mig_aware: bool = True, slice_bytes: int = 0, transport: str = "auto",
                       host_bytes: int = 0, timeout_s: float = 120.0) -> ShmCommunicator:
    """Join the communicator of `decision` as `rank` (collective, blocking).

    The published identity is `peer` if given, else `instance.peer_info`.
    Raises DuplicateDeviceError / MalformedLabelError / ValueError exactly
    where the reference's discover_peers / build_topology would.
    """
    from .instance import peer_info as _peer_info

    if decision is None and nranks is None:
        raise ValueError("need a decision or nranks")
    n = nranks if nranks is not None else len(decision.instances)
    if decision is not None and nranks is not None and nranks != len(decision.instances):
        raise ValueError("nranks disagrees with the decision")
    if peer is None:
        if instance is None:
            raise ValueError("need an instance binding or an explicit PeerInfo")
        peer = _peer_info(instance, rank)
    if peer.rank != rank:
        raise ValueError(f"peer rank {peer.rank} != rank {rank}")
    if transport not in _lib.TRANSPORTS:
        raise ValueError(f"unknown transport {transport!r}")
    me = _lib.peer_to_c(peer.rank, peer.pcie_bus_id, peer.mig_id, peer.host_hash, peer.pid_hash)
    h = ctypes.c_void_p()
    rc = _lib.lib().fmx_comm_init(ctypes.byref(h), job_key.encode(), n, rank, ctypes.byref(me),
                                  1 if mig_aware else 0, slice_bytes, 0, host_bytes,
                                  _lib.TRANSPORTS[transport], timeout_s)
    _lib.check(rc, "fmx_comm_init")
    peers = []
    for r in range(n):
        pc = _lib.PeerInfoC()
        _lib.check(_lib.lib().fmx_comm_peer(h, r, ctypes.byref(pc)))
        peers.append(PeerInfo(pc.rank, pc.pcie_bus_id.decode(), pc.mig_id.decode(),
                              pc.host_hash, pc.pid_hash))
    # Same checks, reference semantics, on the exchanged table (cannot fail
    # where the native check passed; kept as the drop-in object model).
    comm = discover_peers(peers, mig_aware=mig_aware)
    return ShmCommunicator(h.value, rank, list(comm.peers), instance)
