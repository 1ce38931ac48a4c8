"""PyTorch DDP / ZeRO integration of the SHM communicator.

In the paper the SHM allreduce is reached from DDP's gradient buckets and
ZeRO's shard broadcasts (reference PAPER.md:353-354, 485).  Stock NCCL cannot
even initialise with several ranks on one GPU ("Duplicate GPU detected",
PAPER.md:264-271), so here:

* the DDP control plane (parameter-shape verification) runs on a gloo
  process group over the same ranks - small metadata only;
* the init-time parameter broadcast (DDP `_sync_module_states`) goes through
  `ShmCommunicator.broadcast` of the flattened parameters;
* every gradient bucket is allreduced by `flexshm_hook` on a side stream
  (overlapping the rest of the backward pass), keeping DDP's
  default-hook arithmetic bit for bit - `bucket.div_(world)`, then SUM
  (torch/distributed/algorithms/ddp_comm_hooks/default_hooks.py:18-33),
  where the CUDA div_ by a CPU scalar is a multiply by fl32(1/world) -
  fused into one pass (op="avg" = FMX_OP_PREMUL_SUM, comm.mean_factor) with
  the fixed ascending-rank fp32 summation (tests/test_ddp_arith_gpu.py);
* `ZeroShardBroadcast` re-broadcasts each owner's updated parameter shard
  after a sharded optimizer step (the ZeroRedundancyOptimizer pattern,
  torch/distributed/optim/zero_redundancy_optimizer.py:785-801);
  `ZeroShardAllgather` keeps the parameters in one flat buffer of equal
  blocks and re-assembles it with a single in-place all-gather.
"""

import contextlib
import os
import time

import torch

from .comm import ShmCommunicator

# host seconds spent inside flexshm_hook's collective enqueue, and calls (a
# measurement aid: is the autograd thread held up by the driver calls?)
HOOK_HOST = [0.0, 0]
# FMX_HOOK_STAMP=1: stamp each bucket's readiness on the GPU timeline;
# FMX_HOOK_NOOP=1: skip the exchange (measurement of the bare backward pass);
# FMX_HOOK_NOOP=2: skip it but keep the side-stream future plumbing
_SCRATCH = {}
_MEASURE = {"stamp": os.environ.get("FMX_HOOK_STAMP") == "1",
            "noop": os.environ.get("FMX_HOOK_NOOP", "0")}


class HookState:
    """What flexshm_hook needs: the communicator and a side stream for the
    collectives, created in the same context as the rank's work (a green
    context's stream in green mode), so bucket allreduces overlap the rest of
    the backward pass instead of queueing on the autograd stream."""

    def __init__(self, comm: ShmCommunicator, stream=None, threaded: bool = False):
        self.comm = comm
        if stream is None:
            inst = getattr(comm, "instance", None)
            gc = getattr(inst, "green_ctx", None) if inst is not None else None
            if gc is not None:
                s = gc.Stream()
                stream = s if isinstance(s, torch.cuda.Stream) else torch.cuda.ExternalStream(
                    s.cuda_stream, device=inst.device)
            else:
                # high priority: every peer's pipeline waits on this rank's reductions,
                # so they must not queue behind the backward pass's kernels
                # (FMX_HOOK_PRIORITY overrides, for measurements)
                stream = torch.cuda.Stream(priority=int(os.environ.get("FMX_HOOK_PRIORITY", "-1")))
        self.stream = stream
        self.threaded = threaded
        self._queue = None
        if threaded:
            import queue
            import threading
            self._queue = queue.SimpleQueue()
            self._device = torch.cuda.current_device()
            self._thread = threading.Thread(target=self._run, name="flexshm-hook", daemon=True)
            self._thread.start()

    def _run(self):
        """Enqueue thread: issues every bucket's collective (the ~30 driver calls
        of a round) off the autograd thread, in hook order - the same order on
        every rank.  ctypes releases the GIL inside the library."""
        torch.cuda.set_device(self._device)
        while True:
            item = self._queue.get()
            if item is None:
                return
            buf, ready, fut, op = item
            try:
                with torch.cuda.stream(self.stream):
                    self.stream.wait_event(ready)          # the bucket's producers
                    self.comm.set_join_stream(self.stream)
                    try:
                        self.comm.allreduce(buf, op=op, stream=self.stream)
                    finally:
                        self.comm.set_join_stream(None)
                    fut.set_result(buf)                     # event on the side stream
            except BaseException as exc:  # noqa: BLE001 - surface in DDP's wait
                fut.set_exception(exc)

    def close(self):
        if self._queue is not None:
            self._queue.put(None)
            self._queue = None


def flexshm_hook(state, bucket) -> torch.futures.Future[torch.Tensor]:
    """DDP communication hook: bucket.buffer() <- mean over ranks.

    The collective forks from the current (autograd) stream, where the
    bucket's producers ran, and runs in order on the side stream (join-stream
    mode), where it completes; the CUDA-aware future records its completion
    there.  DDP's wait on the future makes the consumer stream wait for that
    event, so later backward kernels are not queued behind the collective's
    flag waits.  Consecutive buckets are serialised on the side stream.
    `state` may also be a bare ShmCommunicator (collective on the current
    stream, no overlap).
    """
    buf = bucket.buffer()
    if isinstance(state, ShmCommunicator):
        state.allreduce(buf, op="avg")
        fut = torch.futures.Future()
        fut.set_result(buf)
        return fut
    cur = torch.cuda.current_stream(buf.device)
    if _MEASURE["stamp"]:
        # timeline probe: when this bucket's gradient is ready on the GPU
        state.comm.stamp(100 + bucket.index(), stream=cur)
    if _MEASURE["noop"] == "1":
        # measurement only: no exchange at all (replicas diverge) - the backward
        # pass's own progress, for comparison with the exchanging step
        fut = torch.futures.Future(devices=[buf.device])
        fut.set_result(buf)
        return fut
    if _MEASURE["noop"] in ("3", "4"):
        # measurement only, no exchange: "3" the exchange's copy-engine traffic
        # alone (bucket D2H to pinned host memory, twice H2D back into scratch);
        # "4" its reduction kernel alone (7 HBM sources, result to HBM)
        from .comm import reduce_local
        state.stream.wait_stream(cur)
        buf.record_stream(state.stream)
        with torch.cuda.stream(state.stream):
            key = (buf.numel(), buf.dtype)
            if key not in _SCRATCH:
                _SCRATCH[key] = (torch.empty(buf.numel(), dtype=buf.dtype).pin_memory(),
                                 torch.empty_like(buf))
            host, dev = _SCRATCH[key]
            if _MEASURE["noop"] == "3":
                host.copy_(buf, non_blocking=True)
                dev.copy_(host, non_blocking=True)
                dev.copy_(host, non_blocking=True)
            else:
                reduce_local([buf] * 7, dev, op="avg", stream=state.stream)
            fut = torch.futures.Future(devices=[buf.device])
            fut.set_result(buf)
        return fut
    if _MEASURE["noop"] == "2":
        # measurement only: the hook's stream / future plumbing without the exchange
        state.stream.wait_stream(cur)
        buf.record_stream(state.stream)
        with torch.cuda.stream(state.stream):
            fut = torch.futures.Future(devices=[buf.device])
            fut.set_result(buf)
        return fut
    if state.threaded:
        # hand the bucket to the enqueue thread: the autograd thread only records
        # an event and returns
        ready = torch.cuda.Event()
        ready.record(cur)
        buf.record_stream(state.stream)
        fut = torch.futures.Future(devices=[buf.device])
        state._queue.put((buf, ready, fut, "avg"))
        return fut
    # fork from the autograd stream (the bucket's producers), run and complete
    # on the side stream (join-stream mode): the autograd stream never waits
    # for a collective
    t0 = time.perf_counter()
    state.comm.set_join_stream(state.stream)
    try:
        state.comm.allreduce(buf, op="avg", stream=cur)
        done = state.comm.completion_stream()
    finally:
        state.comm.set_join_stream(None)
    HOOK_HOST[0] += time.perf_counter() - t0
    HOOK_HOST[1] += 1
    # the collective ran on the side stream (tell the allocator) and completed
    # on the stream completion_stream() names - the future's event is recorded
    # there (the side stream in join-stream mode).
    buf.record_stream(state.stream)
    done_stream = state.stream if done in (0, state.stream.cuda_stream) else \
        torch.cuda.ExternalStream(done, device=buf.device)
    with torch.cuda.stream(done_stream):
        fut = torch.futures.Future(devices=[buf.device])
        fut.set_result(buf)
    return fut


def flexshm_bf16_hook(state, bucket) -> torch.futures.Future[torch.Tensor]:
    """Like flexshm_hook, with the gradient exchanged in bf16 (the idea of
    torch's bf16_compress_hook): the fp32 bucket is rounded to bf16, averaged
    over SHM (bf16 in, fp32 rank-order accumulation, one RNE rounding), and
    widened back.  Half the host-link bytes; within the north_star's bf16
    tolerance, not bit-exact to the fp32 sum.  `state` is a HookState."""
    buf = bucket.buffer()
    cur = torch.cuda.current_stream(buf.device)
    comp = buf.to(torch.bfloat16)            # on the autograd stream, after the producers
    state.comm.set_join_stream(state.stream)
    try:
        state.comm.allreduce(comp, op="avg", stream=cur)
        done = state.comm.completion_stream()
    finally:
        state.comm.set_join_stream(None)
    done_stream = state.stream if done in (0, state.stream.cuda_stream) else \
        torch.cuda.ExternalStream(done, device=buf.device)
    comp.record_stream(state.stream)
    buf.record_stream(state.stream)
    with torch.cuda.stream(done_stream):
        buf.copy_(comp)                      # widen on the completion stream
        fut = torch.futures.Future(devices=[buf.device])
        fut.set_result(buf)
    return fut


def broadcast_parameters(module: torch.nn.Module, comm: ShmCommunicator, root: int = 0) -> None:
    """Make every rank's parameters (and floating buffers) equal to root's."""
    tensors = [p.data for p in module.parameters()] + \
              [b for b in module.buffers() if b.is_floating_point()]
    by_dtype = {}
    for t in tensors:
        by_dtype.setdefault(t.dtype, []).append(t)
    for dtype, group in by_dtype.items():
        if dtype not in (torch.float32, torch.bfloat16):
            raise TypeError(f"cannot broadcast {dtype} parameters over SHM")
        flat = torch.cat([t.reshape(-1) for t in group])
        comm.broadcast(flat, root=root)
        off = 0
        with torch.no_grad():
            for t in group:
                k = t.numel()
                t.copy_(flat[off:off + k].view_as(t))
                off += k


def wrap(module: torch.nn.Module, comm: ShmCommunicator, control_group=None,
         bucket_cap_mb: float = 8.0, overlap: bool = True, compress: str | None = None,
         threaded: bool = False, **ddp_kwargs):
    """DistributedDataParallel over `control_group` (gloo) with gradients on
    the SHM path.  Parameters are synchronised from rank 0 first.  With
    `overlap` the bucket allreduces run on a side stream (HookState);
    compress="bf16" exchanges fp32 buckets in bf16 (flexshm_bf16_hook).
    bucket_cap_mb defaults to 8 (not DDP's 25): the last bucket's allreduce is
    exposed after the backward pass, and 5-10 MB measured best for ResNet-50 on
    7 instances (profiles/r01/r1y: 3357 img/s at 8 MB, 3218 at 25, 2905 at 50)."""
    from torch.nn.parallel import DistributedDataParallel as DDP

    broadcast_parameters(module, comm, root=0)
    # gradients live in the bucket buffers the hook reduces in place: no copy
    # into the buckets per step (+1 % ResNet-50 img/s, profiles/r01/r3t)
    ddp_kwargs.setdefault("gradient_as_bucket_view", True)
    ddp = DDP(module, process_group=control_group, bucket_cap_mb=bucket_cap_mb,
              broadcast_buffers=False, init_sync=False, **ddp_kwargs)
    if compress == "bf16":
        ddp.register_comm_hook(HookState(comm), flexshm_bf16_hook)
    elif compress is None:
        ddp.register_comm_hook(HookState(comm, threaded=threaded) if overlap else comm,
                               flexshm_hook)
    else:
        raise ValueError(f"unknown gradient compression {compress!r}")
    return ddp


def _dense(t: torch.Tensor) -> bool:
    """Strides that cover exactly numel() elements with no overlap."""
    dims = sorted((st, sz) for st, sz in zip(t.stride(), t.size()) if sz > 1)
    expect = 1
    for st, sz in dims:
        if st != expect:
            return False
        expect *= sz
    return True


class ShmDataParallel(torch.nn.Module):
    """Data parallelism over the SHM communicator whose whole training step
    can be captured into ONE CUDA graph (`graphed_step`).

    Same contract as DDP + flexshm_hook - parameters broadcast from rank 0,
    gradients averaged bucket by bucket while the backward pass runs, DDP's
    default-hook arithmetic (x * fl32(1/n), rank-order fp32 sum) - re-expressed
    without torch's C++ Reducer, whose futures and host callbacks cannot live
    in a graph:

    * buckets follow DDP's rebuilt assignment: the order gradients became
      ready in the first backward pass (reducer.cpp rebuild_buckets), a
      first bucket of `first_bucket_mb` (dist._DEFAULT_FIRST_BUCKET_BYTES),
      the rest up to `bucket_cap_mb`; one flat buffer per bucket, each
      parameter's .grad a view of it (gradient_as_bucket_view);
    * a post-accumulate-grad hook counts each bucket's gradients; a complete
      bucket - and every complete one after it, in index order, the same on
      every rank - is allreduced (op="avg") forking from the autograd stream
      onto a side stream (join-stream mode); an autograd final callback
      launches any bucket left and joins the side stream back.

    Why a graph: eager kernel launches make the GPU fetch each launch's work
    from host memory, and those reads queue behind the exchange's own PCIe
    traffic - ResNet-50 fwd+bwd 10.7 -> 18.2 ms under D2H copy traffic eager,
    8.5 -> 8.7 ms replayed as a graph (profiles/r02/r2o).  The collectives
    inside are re-based per replay by the library (fmx_graph_*).

    Call `zero_grad()` (in-place zeroing of the buckets) instead of the
    optimizer's set_to_none; gradients that arrive detached from their bucket
    view are copied into it.  compress="bf16": each fp32 bucket is rounded to a
    bf16 shadow, averaged over SHM with the bf16 contract (fp32 rank-order
    accumulation, one RNE rounding) and widened back after the backward pass -
    half the host-link bytes, torch's bf16_compress_hook idea; within the
    north_star's bf16 tolerance, not the fp32 bit-exact path.

    fused_sgd=dict(lr=..., momentum=0., dampening=0., weight_decay=0.,
    nesterov=False): the optimizer runs inside the collective
    (fmx_allreduce_sgd) - each bucket's owner applies torch's SGD step to its
    chunk of the parameters with the averaged gradient, and the all-gather
    distributes parameters instead of gradients; the momentum lives only for
    the owner's shard (ZeRO-1).  Bit-identical to torch.optim.SGD (foreach) on
    every rank; no optimizer.step() then, and .grad keeps the LOCAL gradient.
    fp32 parameters; a fixed lr (it is baked into a captured graph).
    """

    def __init__(self, module: torch.nn.Module, comm: ShmCommunicator, bucket_cap_mb: float = 8.0,
                 first_bucket_mb: float = 1.0, stream=None, defer_gather: bool | None = None,
                 compress: str | None = None, fused_sgd: dict | None = None):
        super().__init__()
        self.module = module
        self.comm = comm
        broadcast_parameters(module, comm, root=0)
        self.params = [p for p in module.parameters() if p.requires_grad]
        self.cap = int(bucket_cap_mb * (1 << 20))
        self.first_cap = int(first_bucket_mb * (1 << 20))
        # each bucket's last gather is enqueued after the next bucket's stage
        # (fmx_comm_set_defer) while the backward pass runs; flushed at its end
        self.defer = os.environ.get("FMX_DEFER", "1") != "0" if defer_gather is None else defer_gather
        if compress not in (None, "bf16"):
            raise ValueError(f"unknown gradient compression {compress!r}")
        self.compress = compress
        self._shadow = []
        if fused_sgd is not None:
            if compress is not None:
                raise ValueError("fused_sgd exchanges fp32 gradients: no compression")
            unknown = set(fused_sgd) - {"lr", "momentum", "dampening", "weight_decay", "nesterov"}
            if unknown or "lr" not in fused_sgd:
                raise ValueError(f"fused_sgd needs lr (and optionally momentum, dampening, "
                                 f"weight_decay, nesterov); got {sorted(fused_sgd)}")
        self.fused_sgd = fused_sgd
        self._pflat, self._mom, self._first = [], [], []
        self.hook_state = HookState(comm, stream)
        self.stream = self.hook_state.stream
        self.buckets = None          # [(flat tensor, [param index])]
        self.bucket_of = None        # param index -> bucket index
        self._order = []             # first backward: gradient-ready order
        self._pending = []
        self._next = 0
        self._armed = False
        self._sync = True            # no_sync(): gradients accumulate locally
        index = {id(p): i for i, p in enumerate(self.params)}
        self._hooks = [p.register_post_accumulate_grad_hook(
            lambda p, i=index[id(p)]: self._on_grad(i)) for p in self.params]

    def forward(self, *args, **kwargs):
        return self.module(*args, **kwargs)

    @contextlib.contextmanager
    def no_sync(self):
        """DDP.no_sync: backward passes inside accumulate gradients in the
        buckets without exchanging them; the next backward outside exchanges
        the accumulated sum."""
        prev, self._sync = self._sync, False
        try:
            yield
        finally:
            self._sync = prev

    # -- buckets -------------------------------------------------------------
    def _build(self):
        seen = set(self._order)
        order = self._order + [i for i in range(len(self.params)) if i not in seen]
        groups, cur, cur_bytes, cur_dtype = [], [], 0, None
        for i in order:
            p = self.params[i]
            nb = p.numel() * p.element_size()
            cap = self.first_cap if not groups else self.cap
            if cur and (p.dtype != cur_dtype or cur_bytes + nb > cap):
                groups.append(cur)
                cur, cur_bytes = [], 0
            cur.append(i)
            cur_bytes += nb
            cur_dtype = p.dtype
        if cur:
            groups.append(cur)
        self.buckets, self.bucket_of, self._views = [], {}, {}
        for b, idx in enumerate(groups):
            p0 = self.params[idx[0]]
            flat = torch.zeros(sum(self.params[i].numel() for i in idx), dtype=p0.dtype,
                               device=p0.device)
            off = 0
            for i in idx:
                p = self.params[i]
                # the view takes the parameter's strides (channels_last convs): the
                # gradient layout contract of AccumulateGrad, as DDP's bucket views do
                view = flat.as_strided(p.size(), p.stride(), off) if _dense(p) else \
                    flat[off:off + p.numel()].view_as(p)
                if p.grad is not None:
                    view.copy_(p.grad)
                p.grad = view
                off += p.numel()
                self.bucket_of[i] = b
                self._views[i] = view
            self.buckets.append((flat, idx))
            if self.fused_sgd is not None:
                # parameters move into a flat buffer laid out like the gradient bucket
                if flat.dtype != torch.float32:
                    raise TypeError("fused_sgd needs fp32 parameters")
                pflat = torch.empty_like(flat)
                off = 0
                for i in idx:
                    p = self.params[i]
                    pv = pflat.as_strided(p.size(), p.stride(), off) if _dense(p) else \
                        pflat[off:off + p.numel()].view_as(p)
                    with torch.no_grad():
                        pv.copy_(p.data)
                    p.data = pv
                    off += p.numel()
                _, ln = self.comm.shard(flat.numel(), flat.dtype)
                self._pflat.append(pflat)
                self._mom.append(torch.zeros(max(1, ln), dtype=torch.float32, device=flat.device)
                                 if self.fused_sgd.get("momentum", 0.0) else None)
                self._first.append(True)
            if self.compress == "bf16" and flat.dtype == torch.float32:
                self._shadow.append(torch.empty(flat.numel(), dtype=torch.bfloat16,
                                                device=flat.device))
            else:
                self._shadow.append(None)

    def zero_grad(self, set_to_none: bool = False):  # noqa: ARG002 - buckets are persistent
        if self.buckets is None:
            for p in self.params:
                p.grad = None
            return
        for flat, _ in self.buckets:
            flat.zero_()

    # -- hooks ---------------------------------------------------------------
    def _arm(self):
        if not self._armed:
            self._armed = True
            if self.buckets is not None:
                self._pending = [len(idx) for _, idx in self.buckets]
                self._next = 0
            torch.autograd.Variable._execution_engine.queue_callback(self._finish)

    def _on_grad(self, i):
        self._arm()
        if self.buckets is None:
            self._order.append(i)
            return
        p, view = self.params[i], self._views[i]
        if p.grad is None or p.grad.data_ptr() != view.data_ptr():
            # the gradient left its bucket view (set_to_none): move it back
            if p.grad is None:
                view.zero_()
            else:
                view.copy_(p.grad)
            p.grad = view
        if not self._sync:
            return
        b = self.bucket_of[i]
        self._pending[b] -= 1
        while self._next < len(self.buckets) and self._pending[self._next] == 0:
            self._launch(self._next)
            self._next += 1

    def _launch(self, b):
        flat, _ = self.buckets[b]
        cur = torch.cuda.current_stream(flat.device)
        if _MEASURE["stamp"]:     # timeline probe: when this bucket is ready on the GPU
            self.comm.stamp(100 + b, stream=cur)
        buf = flat
        if self._shadow[b] is not None:   # round to bf16 after the bucket's producers
            buf = self._shadow[b]
            buf.copy_(flat)
        if _MEASURE["noop"] == "3":
            # measurement only, no exchange: the exchange's copy-engine traffic alone
            # (bucket D2H to pinned host memory, twice H2D back) on the side stream
            self.stream.wait_stream(cur)
            with torch.cuda.stream(self.stream):
                key = (buf.numel(), buf.dtype)
                if key not in _SCRATCH:
                    _SCRATCH[key] = (torch.empty(buf.numel(), dtype=buf.dtype).pin_memory(),
                                     torch.empty_like(buf))
                host, dev = _SCRATCH[key]
                host.copy_(buf, non_blocking=True)
                dev.copy_(host, non_blocking=True)
                dev.copy_(host, non_blocking=True)
            return
        self.comm.set_join_stream(self.stream)
        try:
            if self.defer:
                self.comm.set_defer(True)
            if self.fused_sgd is not None:
                f = self.fused_sgd
                self.comm.allreduce_sgd(buf, self._pflat[b], self._mom[b], lr=f["lr"],
                                        momentum_coef=f.get("momentum", 0.0),
                                        dampening=f.get("dampening", 0.0),
                                        weight_decay=f.get("weight_decay", 0.0),
                                        nesterov=f.get("nesterov", False),
                                        first_step=self._first[b], op="avg", stream=cur)
                self._first[b] = False
            else:
                self.comm.allreduce(buf, op="avg", stream=cur)
        finally:
            self.comm.set_join_stream(None)

    def _finish(self):
        self._armed = False
        if self.buckets is None:
            self._build()          # first backward: buckets in gradient-ready order
            self._pending = [0] * len(self.buckets)
            self._next = 0
        if not self._sync:
            return
        while self._next < len(self.buckets):
            self._launch(self._next)
            self._next += 1
        cur = torch.cuda.current_stream(self.params[0].device)
        if self.defer:   # the last bucket's gather, then back to immediate completion
            self.comm.set_join_stream(self.stream)
            try:
                self.comm.flush(stream=cur)
            finally:
                self.comm.set_join_stream(None)
                self.comm.set_defer(False)
        if any(sh is not None for sh in self._shadow):
            with torch.cuda.stream(self.stream):    # widen the averaged bf16 buckets
                for (flat, _), sh in zip(self.buckets, self._shadow):
                    if sh is not None:
                        flat.copy_(sh)
        cur.wait_stream(self.stream)

    # -- CUDA graph ----------------------------------------------------------
    def graphed_step(self, step_fn, warmup: int = 3, before_capture=None):
        """Capture `step_fn` - forward, backward and optimizer step on static
        input tensors, returning its outputs - into one CUDA graph; returns
        `replay()`, which runs one training step and returns the same (static)
        outputs.  Runs `warmup` eager steps first (bucket assignment,
        optimizer state, cuDNN plans).  Every rank must capture the same step."""
        dev = self.params[0].device
        # capture on the caller's stream (an instance's stream lives in its
        # green / MPS context) unless that is the legacy default stream
        cur = torch.cuda.current_stream(dev)
        s = cur if cur.cuda_stream != 0 else torch.cuda.Stream(device=dev)
        s.wait_stream(cur)
        with torch.cuda.stream(s):
            for _ in range(max(1, warmup)):
                step_fn()
        cur.wait_stream(s)
        torch.cuda.synchronize(dev)
        if before_capture is not None:
            before_capture()
        g = torch.cuda.CUDAGraph(keep_graph=True)
        self.comm.capture_begin()
        try:
            with torch.cuda.graph(g, stream=s):
                out = step_fn()
        except BaseException:
            self.comm.capture_end(0)       # abandon the capture (counters roll back)
            self.comm.set_join_stream(None)
            self.comm.set_defer(False)
            self._armed = False
            raise
        handle = self.comm.capture_end(g.raw_cuda_graph())
        g.instantiate()
        exec_ = g.raw_cuda_graph_exec()
        comm = self.comm

        def replay():
            comm.launch_prepare(handle, exec_, torch.cuda.current_stream(dev))
            g.replay()
            return out

        replay.graph = g
        replay.handle = handle
        return replay


class ZeroShardBroadcast:
    """After a sharded optimizer step, rank r owns parameter shard r; every
    shard is broadcast from its owner so all replicas agree again."""

    def __init__(self, params: list[torch.nn.Parameter], comm: ShmCommunicator):
        self.comm = comm
        self.params = list(params)
        sizes = [p.numel() for p in self.params]
        total = sum(sizes)
        per = (total + comm.size - 1) // comm.size
        # greedy contiguous partition of the parameter list into size-balanced shards
        self.owner, acc, r = [], 0, 0
        for s in sizes:
            if acc >= per * (r + 1) and r < comm.size - 1:
                r += 1
            self.owner.append(r)
            acc += s

    def owned(self, rank: int) -> list[torch.nn.Parameter]:
        return [p for p, o in zip(self.params, self.owner) if o == rank]

    @torch.no_grad()
    def sync(self) -> None:
        for r in range(self.comm.size):
            group = [p for p, o in zip(self.params, self.owner) if o == r]
            if not group:
                continue
            flat = torch.cat([p.data.reshape(-1) for p in group])
            self.comm.broadcast(flat, root=r)
            off = 0
            for p in group:
                k = p.numel()
                p.data.copy_(flat[off:off + k].view_as(p))
                off += k


class ZeroShardAllgather:
    """ZeRO-style flat parameter shards re-assembled with ONE all-gather.

    The parameters (one dtype) are moved into a flat buffer padded to
    size * c elements and become views of it; rank r owns elements
    [r*c, (r+1)*c) - its optimizer updates only `shard()` - and `sync()`
    all-gathers every owner's block in place (NCCL in-place layout:
    send = recv + rank*c).  One collective per step instead of one broadcast
    per owner, and every byte crosses the host link once per reader."""

    def __init__(self, params: list[torch.nn.Parameter], comm: ShmCommunicator):
        self.comm = comm
        self.params = list(params)
        dtypes = {p.dtype for p in self.params}
        if len(dtypes) != 1:
            raise TypeError("ZeroShardAllgather needs parameters of one dtype")
        total = sum(p.numel() for p in self.params)
        n = comm.size
        self.block = (total + n - 1) // n
        dev = self.params[0].device
        self.flat = torch.zeros(n * self.block, dtype=self.params[0].dtype, device=dev)
        off = 0
        with torch.no_grad():
            for p in self.params:
                k = p.numel()
                self.flat[off:off + k].copy_(p.data.reshape(-1))
                p.data = self.flat[off:off + k].view_as(p)
                off += k

    def shard(self, rank: int | None = None) -> torch.Tensor:
        r = self.comm.rank if rank is None else rank
        return self.flat[r * self.block:(r + 1) * self.block]

    @torch.no_grad()
    def sync(self, stream=None) -> None:
        self.comm.allgather(self.shard(), self.flat, stream=stream)
