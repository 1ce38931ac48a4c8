"""Rank-process bodies for the multi-process GPU tests (spawned by
paper_2511_09143_b200.launcher.launch).  Inputs are drawn with the oracle's
seeded generators so the parent can recompute the expected result."""

from __future__ import annotations

import hashlib
import os
import time

import numpy as np


def make_input(rank: int, sc: dict) -> np.ndarray:
    from oracle import oracle as orc
    dt = orc.F32 if sc["dtype"] == "f32" else orc.BF16
    if sc.get("inputs", "normal") == "adversarial":
        return orc.adversarial(rank, sc["count"], dt)
    return orc.synthetic_gradient(rank, sc["count"], dt, seed=sc.get("seed", 1234))


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8)).hexdigest()


def suite_worker(rank: int, job_key: str, n: int, transport: str, mode: str, scenarios: list,
                 slice_bytes: int = 0, peer_override: dict | None = None,
                 host_bytes: int = 0):
    import torch

    from paper_2511_09143_b200 import instance as inst_mod
    from paper_2511_09143_b200.comm import init_process_group
    from paper_2511_09143_b200.commsim import PeerInfo

    # the launcher names this rank's instance (fm_select order over the GPUs)
    inst = inst_mod.bind(int(os.environ.get("FMX_GPU_ID", "0")),
                         int(os.environ.get("FMX_INSTANCE_ID", str(rank + 1))), mode=mode)
    peer = inst_mod.peer_info(inst, rank)
    if peer_override and rank in peer_override:
        peer = PeerInfo(rank, peer.pcie_bus_id, peer_override[rank], peer.host_hash, peer.pid_hash)
    try:
        comm = init_process_group(None, rank, job_key, instance=inst, peer=peer, nranks=n,
                                  slice_bytes=slice_bytes, transport=transport, timeout_s=120,
                                  host_bytes=host_bytes)
    except Exception as exc:  # bootstrap failures are part of what we test
        return {"init_error": type(exc).__name__, "args": getattr(exc, "rank_a", None),
                "args_b": getattr(exc, "rank_b", None)}
    out = []
    stream = inst.stream
    for sc in scenarios:
        x = make_input(rank, sc)
        tdtype = torch.float32 if sc["dtype"] == "f32" else torch.bfloat16
        if sc["kind"] == "allreduce_host":
            region = comm.host_buffer()
            off = sc.get("host_offset", 0)
            view = region[off:off + x.nbytes].view(tdtype)
            view.view(torch.uint8).copy_(torch.from_numpy(x.view(np.uint8)))
            comm.allreduce_host(view, op=sc.get("op", "sum"), factor=sc.get("factor"),
                                stream=stream)
            ev = torch.cuda.Event()
            ev.record(stream)
            t0 = time.time()
            while not ev.query():
                if time.time() - t0 > 60:
                    return {"stuck": sc, "index": len(out), "flags": comm.flags(), "rank": rank}
                time.sleep(0.002)
            comm.barrier(60)  # every rank done reading before anyone rewrites its region
            got = view.view(torch.uint8).numpy().view(x.dtype).copy()
            out.append(digest(got) if sc.get("ret") == "sha" else got)
            continue
        host = torch.from_numpy(x.view(np.float32) if sc["dtype"] == "f32" else x.view(np.int16))
        off = sc.get("offset", 0)
        buf = torch.empty(sc["count"] + off, dtype=tdtype, device="cuda")
        t = buf[off:]
        t.copy_(host.view(tdtype) if sc["dtype"] != "f32" else host, non_blocking=False)
        if sc["kind"] == "allreduce":
            if sc.get("inplace", True):
                comm.allreduce(t, op=sc.get("op", "sum"), factor=sc.get("factor"), stream=stream)
                res = t
            else:
                res = torch.empty_like(t)
                comm.allreduce(t, op=sc.get("op", "sum"), factor=sc.get("factor"), out=res,
                               stream=stream)
        elif sc["kind"] == "reduce_scatter":   # t holds n blocks; mine comes back reduced
            c = sc["count"] // n
            res = t[rank * c:(rank + 1) * c] if sc.get("inplace") else torch.empty(
                c, dtype=tdtype, device="cuda")
            comm.reduce_scatter(t, res, op=sc.get("op", "sum"), factor=sc.get("factor"),
                                stream=stream)
        elif sc["kind"] == "allgather":        # t is my block of the n-block result
            c = sc["count"]
            res = torch.empty(n * c + off, dtype=tdtype, device="cuda")[off:]
            if sc.get("inplace"):
                res[rank * c:(rank + 1) * c].copy_(t)
                comm.allgather(res[rank * c:(rank + 1) * c], res, stream=stream)
            else:
                comm.allgather(t, res, stream=stream)
        else:
            comm.broadcast(t, root=sc["root"], stream=stream)
            res = t
        ev = torch.cuda.Event()
        ev.record(stream)
        t0 = time.time()
        while not ev.query():
            if time.time() - t0 > 60:
                return {"stuck": sc, "index": len(out), "flags": comm.flags(), "rank": rank}
            time.sleep(0.002)
        r = res.cpu()
        arr = r.numpy() if sc["dtype"] == "f32" else r.view(torch.int16).numpy().view(np.uint16)
        out.append(digest(arr) if sc.get("ret") == "sha" else arr.copy())
    launches = comm.kernel_launches()
    comm.barrier()
    comm.destroy()
    return {"results": out, "launches": launches, "pid": os.getpid()}


def mixed_env_worker(rank: int, job_key: str, n: int, envs: dict, scenarios: list,
                     slice_bytes: int = 0):
    """suite_worker with per-rank schedule settings in the environment: every
    rank must still run rank 0's (published in the segment header)."""
    os.environ.update(envs.get(rank, {}))
    return suite_worker(rank, job_key, n, "auto", "green", scenarios, slice_bytes)


def ddp_worker(rank: int, job_key: str, n: int, port: int, mode: str = "green",
               overlap: bool = True, dtype: str = "f32", compress: str | None = None,
               threaded: bool = False):
    """Tiny model: local gradients without DDP, then the same step under DDP
    with the flexshm comm hook; returns both (flattened fp32)."""
    import torch
    import torch.distributed as dist

    from paper_2511_09143_b200 import ddp as fddp
    from paper_2511_09143_b200 import instance as inst_mod
    from paper_2511_09143_b200.comm import init_process_group

    inst = inst_mod.bind(0, rank + 1, mode=mode)
    comm = init_process_group(None, rank, job_key, instance=inst, nranks=n, timeout_s=120)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=n)
    stream = inst.stream
    with torch.cuda.stream(stream):
        torch.manual_seed(1000 + rank)     # different init per rank: broadcast must fix it
        model = torch.nn.Sequential(torch.nn.Linear(64, 300), torch.nn.GELU(),
                                    torch.nn.Linear(300, 10)).cuda()
        if dtype == "bf16":   # bf16 parameters -> bf16 gradient buckets (BERT leg's path)
            model = model.to(torch.bfloat16)
        g = torch.Generator(device="cpu").manual_seed(7 + rank)
        x = torch.randn(32, 64, generator=g).cuda().to(next(model.parameters()).dtype)
        y = torch.randint(0, 10, (32,), generator=g).cuda()
        net = fddp.wrap(model, comm, control_group=dist.group.WORLD, bucket_cap_mb=0.05,
                        overlap=overlap, compress=compress, threaded=threaded)
        params0 = torch.cat([p.detach().reshape(-1) for p in model.parameters()]).cpu()
        # local gradient (no communication): no_sync skips the reducer
        with net.no_sync():
            torch.nn.functional.cross_entropy(net(x), y).backward()
        local = torch.cat([p.grad.reshape(-1) for p in model.parameters()]).clone()
        # what DDP's default hook does to a bucket before its SUM allreduce
        # (default_hooks.py:26): an in-place CUDA div_ by the world size
        local_div = local.clone().div_(n)
        for p in model.parameters():
            p.grad = None
        torch.nn.functional.cross_entropy(net(x), y).backward()
        synced = torch.cat([p.grad.reshape(-1) for p in model.parameters()]).clone()
    stream.synchronize()
    dist.destroy_process_group()
    comm.destroy()
    as_np = (lambda t: t.float().numpy()) if dtype == "f32" else \
        (lambda t: t.cpu().view(torch.int16).numpy().view(np.uint16))
    return {"params0": as_np(params0.cpu()), "local": as_np(local.cpu()),
            "local_div": as_np(local_div.cpu()), "synced": as_np(synced.cpu())}


def overlap_worker(rank: int, job_key: str, n: int, counts: list, mode: str = "green"):
    """Join-stream mode: several allreduces on distinct buffers issued back to
    back on one stream, completing on a side stream (the DDP-bucket pattern);
    returns every result."""
    import torch

    from oracle import oracle as orc
    from paper_2511_09143_b200 import instance as inst_mod
    from paper_2511_09143_b200.comm import init_process_group

    inst = inst_mod.bind(0, rank + 1, mode=mode)
    comm = init_process_group(None, rank, job_key, instance=inst, nranks=n, timeout_s=120)
    main = inst.stream
    side = torch.cuda.Stream() if inst.green_ctx is None else torch.cuda.ExternalStream(
        inst.green_ctx.Stream().cuda_stream)
    bufs = []
    with torch.cuda.stream(main):
        for i, c in enumerate(counts):
            x = orc.synthetic_gradient(rank, c, orc.F32, seed=500 + i)
            bufs.append(torch.from_numpy(x).to("cuda"))
    main.synchronize()
    comm.set_join_stream(side)
    for b in bufs:
        comm.allreduce(b, op="avg", stream=main)
    done = comm.completion_stream()
    comm.set_join_stream(None)
    torch.cuda.ExternalStream(done).synchronize()   # the last call completes there ...
    side.synchronize()                              # ... and every call's lane 1 ran here
    out = [b.cpu().numpy() for b in bufs]
    comm.barrier(60)
    comm.destroy()
    return {"results": out}


def stress_ops(n: int, seed: int, nops: int) -> list:
    """A seeded random program of collectives every rank runs in the same order."""
    import random
    rng = random.Random(seed)
    ops = []
    for i in range(nops):
        kind = rng.choice(["allreduce"] * 4 + ["reduce_scatter", "allgather", "broadcast"])
        dtype = rng.choice(["f32", "f32", "bf16"])
        size = rng.choice([1, 7, 64, 4096, 100_003, 524_288, 1_000_001, 2_500_000])
        op = rng.choice(["sum", "avg", "postscale"]) if kind in ("allreduce", "reduce_scatter") \
            else "sum"
        ops.append({"kind": kind, "dtype": dtype, "size": size, "op": op,
                    "root": rng.randrange(n), "inplace": rng.random() < 0.5,
                    "join": rng.random() < 0.3, "seed": 10_000 + i})
    return ops


def stress_input(rank: int, o: dict, n: int) -> np.ndarray:
    from oracle import oracle as orc
    dt = orc.F32 if o["dtype"] == "f32" else orc.BF16
    count = o["size"] * (n if o["kind"] == "reduce_scatter" else 1)
    return orc.synthetic_gradient(rank, count, dt, seed=o["seed"])


def stress_worker(rank: int, job_key: str, n: int, seed: int, nops: int, mode: str = "mps"):
    """Run the random program; return a sha256 per op of this rank's result."""
    import torch

    from paper_2511_09143_b200 import instance as inst_mod
    from paper_2511_09143_b200.comm import init_process_group

    # the launcher names this rank's instance (fm_select order over the GPUs)
    inst = inst_mod.bind(int(os.environ.get("FMX_GPU_ID", "0")),
                         int(os.environ.get("FMX_INSTANCE_ID", str(rank + 1))), mode=mode)
    comm = init_process_group(None, rank, job_key, instance=inst, nranks=n, timeout_s=300)
    s = inst.stream
    side = torch.cuda.Stream()
    digests = []
    for o in stress_ops(n, seed, nops):
        x = stress_input(rank, o, n)
        tdt = torch.float32 if o["dtype"] == "f32" else torch.bfloat16
        host = torch.from_numpy(x.view(np.float32) if o["dtype"] == "f32" else x.view(np.int16))
        with torch.cuda.stream(s):
            t = host.to("cuda", non_blocking=False).view(tdt) if o["dtype"] != "f32" else \
                host.to("cuda", non_blocking=False)
        s.synchronize()
        factor = 0.25 if o["op"] == "postscale" else None
        if o["join"]:
            comm.set_join_stream(side)
        k = o["kind"]
        if k == "allreduce":
            res = t if o["inplace"] else torch.empty_like(t)
            comm.allreduce(t, op=o["op"], factor=factor, out=None if o["inplace"] else res,
                           stream=s)
        elif k == "reduce_scatter":
            c = o["size"]
            res = t[rank * c:(rank + 1) * c] if o["inplace"] else torch.empty(c, dtype=tdt,
                                                                              device="cuda")
            comm.reduce_scatter(t, res, op=o["op"], factor=factor, stream=s)
        elif k == "allgather":
            c = o["size"]
            res = torch.empty(n * c, dtype=tdt, device="cuda")
            if o["inplace"]:
                res[rank * c:(rank + 1) * c].copy_(t)
                comm.allgather(res[rank * c:(rank + 1) * c], res, stream=s)
            else:
                comm.allgather(t, res, stream=s)
        else:
            comm.broadcast(t, root=o["root"], stream=s)
            res = t
        done = comm.completion_stream()
        comm.set_join_stream(None)
        torch.cuda.ExternalStream(done).synchronize()
        s.synchronize()
        r = res.cpu()
        arr = r.numpy() if o["dtype"] == "f32" else r.view(torch.int16).numpy().view(np.uint16)
        digests.append(digest(arr))
    comm.barrier(120)
    comm.destroy()
    return {"digests": digests}


def zero_worker(rank: int, job_key: str, n: int, mode: str = "green"):
    """Both ZeRO shard-sync flavours: every rank writes only what it owns, then
    syncs; returns the parameters every rank ends up with."""
    import torch

    from paper_2511_09143_b200 import ddp as fddp
    from paper_2511_09143_b200 import instance as inst_mod
    from paper_2511_09143_b200.comm import init_process_group

    inst = inst_mod.bind(0, rank + 1, mode=mode)
    comm = init_process_group(None, rank, job_key, instance=inst, nranks=n, timeout_s=120)
    s = inst.stream
    out = {}
    with torch.cuda.stream(s):
        torch.manual_seed(0)
        shapes = [(300, 7), (11,), (64, 64), (5, 3, 3), (1000,)]
        # broadcast flavour: parameter-granular owners
        ps = [torch.nn.Parameter(torch.zeros(sh, device="cuda")) for sh in shapes]
        zb = fddp.ZeroShardBroadcast(ps, comm)
        for p, o in zip(ps, zb.owner):
            if o == rank:
                p.data.fill_(o + 1.0)
        zb.sync()
        out["bcast"] = torch.cat([p.detach().reshape(-1) for p in ps]).cpu().numpy()
        out["owner"] = list(zb.owner)
        # all-gather flavour: flat element blocks
        qs = [torch.nn.Parameter(torch.zeros(sh, device="cuda")) for sh in shapes]
        za = fddp.ZeroShardAllgather(qs, comm)
        za.shard().fill_(rank + 1.0)
        za.sync(stream=s)
        out["flat"] = za.flat.cpu().numpy()
        out["params"] = torch.cat([q.detach().reshape(-1) for q in qs]).cpu().numpy()
        out["block"] = za.block
    s.synchronize()
    comm.barrier(60)
    comm.destroy()
    return out


def graph_dp_worker(rank: int, job_key: str, n: int, mode: str = "mps", defer: bool = True,
                    compress: str | None = None, steps: int = 5, warmup: int = 2):
    """ddp.ShmDataParallel on a small MLP: (1) the first step's averaged
    gradient next to this rank's local gradient (oracle check in the test);
    (2) `steps` eager training steps; (3) the same from the same start as a
    captured CUDA graph (warmup eager steps, then replays), with an eager
    allreduce between two replays.  Returns flattened fp32 arrays."""
    import torch
    import torch.nn.functional as F

    from paper_2511_09143_b200 import ddp as fddp
    from paper_2511_09143_b200 import instance as inst_mod
    from paper_2511_09143_b200.comm import init_process_group

    inst = inst_mod.bind(0, rank + 1, mode=mode)
    comm = init_process_group(None, rank, job_key, instance=inst, nranks=n, timeout_s=120)
    stream = inst.stream
    out = {}

    def build():
        torch.manual_seed(1000 + rank)   # different init per rank: the broadcast must fix it
        return torch.nn.Sequential(torch.nn.Linear(64, 300), torch.nn.GELU(),
                                   torch.nn.Linear(300, 10)).cuda()

    flat = lambda ts: torch.cat([t.detach().reshape(-1) for t in ts]).float().cpu().numpy()
    with torch.cuda.stream(stream):
        g = torch.Generator(device="cpu").manual_seed(7 + rank)
        x = torch.randn(32, 64, generator=g).cuda()
        y = torch.randint(0, 10, (32,), generator=g).cuda()
        # local gradient from the broadcast start (no exchange)
        ref = build()
        fddp.broadcast_parameters(ref, comm)
        F.cross_entropy(ref(x), y).backward()
        out["local"] = flat([p.grad for p in ref.parameters()])

        runs = {}
        for kind in ("eager", "graph"):
            model = build()
            net = fddp.ShmDataParallel(model, comm, bucket_cap_mb=0.05, first_bucket_mb=0.01,
                                       defer_gather=defer, compress=compress)
            opt = torch.optim.SGD(net.parameters(), lr=0.05, momentum=0.9)

            def step():
                net.zero_grad()
                loss = F.cross_entropy(net(x), y)
                loss.backward()
                opt.step()
                return loss

            if kind == "eager":
                for k in range(steps):
                    step()
                    if k == 0:
                        out["synced"] = flat([p.grad for p in model.parameters()])
                out["buckets"] = len(net.buckets)
            else:
                replay = net.graphed_step(step, warmup=warmup)
                extra = torch.arange(1000, dtype=torch.float32, device="cuda") * (rank + 1)
                for k in range(steps - warmup):
                    replay()
                    if k == 0:       # an eager collective between two replays
                        comm.allreduce(extra, op="sum")
                out["extra"] = extra.cpu().numpy()
                out["launches_per_replay"] = comm.kernel_launches()
            runs[kind] = flat(model.parameters())
        # the optimizer fused into the collective (fmx_allreduce_sgd): eager steps then
        # graph replays, against torch.optim.SGD on every rank (the eager run above)
        model4 = build()
        net4 = fddp.ShmDataParallel(model4, comm, bucket_cap_mb=0.05, first_bucket_mb=0.01,
                                    defer_gather=defer, fused_sgd=dict(lr=0.05, momentum=0.9))

        def step4():
            net4.zero_grad()
            loss = F.cross_entropy(net4(x), y)
            loss.backward()
            return loss

        replay4 = net4.graphed_step(step4, warmup=warmup)
        for _ in range(steps - warmup):
            replay4()
        out["params_fused"] = flat(model4.parameters())
        # weight decay + Nesterov, eager, against torch's SGD with the same settings
        cfg = dict(lr=0.03, momentum=0.8, weight_decay=1e-3, nesterov=True)
        for kind in ("torch", "fused"):
            m = build()
            if kind == "torch":
                nt = fddp.ShmDataParallel(m, comm, bucket_cap_mb=0.05, first_bucket_mb=0.01)
                o = torch.optim.SGD(nt.parameters(), **cfg)
            else:
                nt = fddp.ShmDataParallel(m, comm, bucket_cap_mb=0.05, first_bucket_mb=0.01,
                                          fused_sgd=cfg)
            for _ in range(4):
                nt.zero_grad()
                F.cross_entropy(nt(x), y).backward()
                if kind == "torch":
                    o.step()
            out[f"params_wd_{kind}"] = flat(m.parameters())
        # gradient accumulation: one backward under no_sync, one outside - the
        # exchanged gradient is the DDP mean of the ranks' accumulated gradients
        x2 = torch.randn(32, 64, generator=g).cuda()
        y2 = torch.randint(0, 10, (32,), generator=g).cuda()
        ref2 = build()
        fddp.broadcast_parameters(ref2, comm)
        F.cross_entropy(ref2(x), y).backward()
        F.cross_entropy(ref2(x2), y2).backward()
        out["local_acc"] = flat([p.grad for p in ref2.parameters()])
        model3 = build()
        net3 = fddp.ShmDataParallel(model3, comm, bucket_cap_mb=0.05, first_bucket_mb=0.01,
                                    defer_gather=defer, compress=compress)
        with net3.no_sync():
            F.cross_entropy(net3(x), y).backward()
        F.cross_entropy(net3(x2), y2).backward()
        out["synced_acc"] = flat([p.grad for p in model3.parameters()])
    stream.synchronize()
    out.update(params_eager=runs["eager"], params_graph=runs["graph"])
    comm.destroy()
    return out


GRAPH_API_SEED = {"big": 1000, "small": 2000, "rs": 3000, "bc": 4000}


def graph_api_worker(rank: int, job_key: str, n: int, mode: str = "mps", transport: str = "auto",
                     slice_bytes: int = 0):
    """The raw fmx_graph_* / deferred-gather API on one rank.

    (1) Deferred gathers in join-stream mode: three allreduces (multi-round,
        one-shot size, one-round) forked from the compute stream, then a flush;
        set_defer(False) with a gather pending must raise.
    (2) Two captured graphs - G1: copy inputs in, allreduce (avg) of a
        multi-round buffer, broadcast from the last rank; G2: allreduce of a
        one-shot-sized buffer, reduce-scatter - replayed G1, G2, G1 (on another
        stream), eager allreduce (third stream), G2, G1 with fresh inputs
        before every replay.  Returns every result (flattened fp32)."""
    import torch

    from oracle import oracle as orc
    from paper_2511_09143_b200 import instance as inst_mod
    from paper_2511_09143_b200.comm import init_process_group

    inst = inst_mod.bind(0, rank + 1, mode=mode)
    comm = init_process_group(None, rank, job_key, instance=inst, nranks=n, timeout_s=120,
                              transport=transport, slice_bytes=slice_bytes)
    out = {}
    s0 = inst.stream
    dev = torch.device("cuda")
    t = lambda a: torch.from_numpy(a).to(dev)
    with torch.cuda.stream(s0):
        # (1) deferred gathers
        sizes = [300_001, 1000, 40_000]
        bufs = [t(orc.synthetic_gradient(rank, c, orc.F32, seed=50 + i)) for i, c in enumerate(sizes)]
        side = torch.cuda.Stream()
        comm.set_join_stream(side)
        comm.set_defer(True)
        for b in bufs:
            comm.allreduce(b, op="sum", stream=s0)
        raised = False
        try:
            comm.set_defer(False)
        except ValueError:
            raised = True
        comm.flush(stream=s0)
        comm.set_join_stream(None)
        comm.set_defer(False)
        s0.wait_stream(side)
        out["defer_raised"] = raised
        out["defer"] = [b.cpu().numpy() for b in bufs]

        # (2) two captured graphs
        c_big, c_small, c_rs, c_bc = 200_003, 5, 999, 3000
        inp = {k: torch.empty(c, device=dev) for k, c in
               (("big", c_big), ("small", c_small), ("rs", n * c_rs), ("bc", c_bc))}
        work = {k: torch.empty_like(v) for k, v in inp.items()}
        rs_out = torch.empty(c_rs, device=dev)
        torch.cuda.synchronize()

        def capture(body):
            g = torch.cuda.CUDAGraph(keep_graph=True)
            comm.capture_begin()
            with torch.cuda.graph(g, stream=s0):
                body()
            h = comm.capture_end(g.raw_cuda_graph())
            g.instantiate()
            return g, h, g.raw_cuda_graph_exec()

        def g1_body():
            cur = torch.cuda.current_stream()
            work["big"].copy_(inp["big"])
            work["bc"].copy_(inp["bc"])
            comm.allreduce(work["big"], op="avg", stream=cur)
            comm.broadcast(work["bc"], root=n - 1, stream=cur)

        def g2_body():
            cur = torch.cuda.current_stream()
            work["small"].copy_(inp["small"])
            work["rs"].copy_(inp["rs"])
            comm.allreduce(work["small"], op="sum", stream=cur)
            comm.reduce_scatter(work["rs"], rs_out, op="sum", stream=cur)

        G1, G2 = capture(g1_body), capture(g2_body)
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        plan = [("G1", s0), ("G2", s0), ("G1", s1), ("eager", s2), ("G2", s1), ("G1", s0)]
        results = []
        for k, (what, st) in enumerate(plan):
            seed = 100 + k
            with torch.cuda.stream(st):
                st.wait_stream(s0)   # the fresh inputs are written on s0 below
            if what == "eager":
                x = t(orc.synthetic_gradient(rank, 77_777, orc.F32, seed=seed))
                torch.cuda.synchronize()
                with torch.cuda.stream(st):
                    comm.allreduce(x, op="sum", stream=st)
                st.synchronize()
                results.append(("eager", seed, x.cpu().numpy()))
                continue
            torch.cuda.synchronize()
            for key in inp:
                inp[key].copy_(t(orc.synthetic_gradient(rank, inp[key].numel(), orc.F32,
                                                        seed=seed + GRAPH_API_SEED[key])))
            torch.cuda.synchronize()
            g, h, ex = G1 if what == "G1" else G2
            with torch.cuda.stream(st):
                comm.launch_prepare(h, ex, st)
                g.replay()
            st.synchronize()
            if what == "G1":
                results.append(("G1", seed, work["big"].cpu().numpy(), work["bc"].cpu().numpy()))
            else:
                results.append(("G2", seed, work["small"].cpu().numpy(), rs_out.cpu().numpy()))
        out["graphs"] = results
    torch.cuda.synchronize()
    comm.destroy()
    return out


def fused_sgd_worker(rank: int, job_key: str, n: int, count: int, transport: str,
                     slice_bytes: int, mode: str = "mps", steps: int = 3):
    """fmx_allreduce_sgd on a flat buffer against the same steps done the
    unfused way on this rank: comm.allreduce(op="avg") of the gradient, then
    torch.optim.SGD (foreach) on a Parameter.  Returns both parameter vectors."""
    import torch

    from oracle import oracle as orc
    from paper_2511_09143_b200 import instance as inst_mod
    from paper_2511_09143_b200.comm import init_process_group

    inst = inst_mod.bind(0, rank + 1, mode=mode)
    comm = init_process_group(None, rank, job_key, instance=inst, nranks=n, transport=transport,
                              slice_bytes=slice_bytes, timeout_s=120)
    s = inst.stream
    cfg = dict(lr=0.02, momentum=0.9, weight_decay=1e-3, nesterov=False, dampening=0.1)
    with torch.cuda.stream(s):
        p0 = torch.from_numpy(orc.synthetic_gradient(0, count, orc.F32, seed=77)).cuda() * 100
        ref = torch.nn.Parameter(p0.clone())
        opt = torch.optim.SGD([ref], lr=cfg["lr"], momentum=cfg["momentum"],
                              weight_decay=cfg["weight_decay"], dampening=cfg["dampening"],
                              foreach=True)
        fused = p0.clone()
        _, ln = comm.shard(count)
        mom = torch.zeros(max(1, ln), device="cuda")
        for k in range(steps):
            g = torch.from_numpy(orc.synthetic_gradient(rank, count, orc.F32, seed=500 + k)).cuda()
            comm.allreduce_sgd(g, fused, mom, lr=cfg["lr"], momentum_coef=cfg["momentum"],
                               dampening=cfg["dampening"], weight_decay=cfg["weight_decay"],
                               first_step=k == 0, op="avg", stream=s)
            gr = g.clone()
            comm.allreduce(gr, op="avg", stream=s)
            ref.grad = gr
            opt.step()
    s.synchronize()
    out = {"fused": fused.cpu().numpy(), "torch": ref.detach().cpu().numpy()}
    comm.destroy()
    return out


def graph_stress_worker(rank: int, job_key: str, n: int, seed: int, nops: int, replays: int = 3,
                        mode: str = "mps", slice_bytes: int = 0, sticky_defer: bool = False,
                        check_every: int = 1):
    """The random program of stress_ops captured ONCE as a CUDA graph (join-stream
    ops with deferred gathers included) and replayed `replays` times with fresh
    inputs written before each replay (seed + 100000 * replay); returns a
    sha256 per replay per op."""
    import torch

    from paper_2511_09143_b200 import instance as inst_mod
    from paper_2511_09143_b200.comm import init_process_group

    inst = inst_mod.bind(0, rank + 1, mode=mode)
    comm = init_process_group(None, rank, job_key, instance=inst, nranks=n, timeout_s=300,
                              slice_bytes=slice_bytes)
    s = inst.stream
    side = torch.cuda.Stream()
    ops = stress_ops(n, seed, nops)
    dev = torch.device("cuda")

    def as_tensor(x, dtype):
        host = torch.from_numpy(x.view(np.float32) if dtype == "f32" else x.view(np.int16))
        t = host.to(dev)
        return t if dtype == "f32" else t.view(torch.bfloat16)

    inp, work, res = [], [], []
    for o in ops:
        t = as_tensor(stress_input(rank, o, n), o["dtype"])
        inp.append(t)
        work.append(torch.empty_like(t))
        c = o["size"]
        k = o["kind"]
        if k == "reduce_scatter" and not o["inplace"]:
            res.append(torch.empty(c, dtype=t.dtype, device=dev))
        elif k == "allgather":
            res.append(torch.empty(n * c, dtype=t.dtype, device=dev))
        elif k == "allreduce" and not o["inplace"]:
            res.append(torch.empty_like(t))
        else:
            res.append(None)
    torch.cuda.synchronize()

    def is_join(o):
        return o["join"] and o["kind"] == "allreduce"

    def program():
        used_side = False
        for i, o in enumerate(ops):
            k, c = o["kind"], o["size"]
            factor = 0.25 if o["op"] == "postscale" else None
            join = is_join(o)
            if join:   # a run of join-stream allreduces with deferred gathers
                comm.set_join_stream(side)
                comm.set_defer(True)
                used_side = True
            if k == "allreduce":
                if o["inplace"]:
                    work[i].copy_(inp[i])
                    comm.allreduce(work[i], op=o["op"], factor=factor, stream=s)
                else:
                    comm.allreduce(inp[i], op=o["op"], factor=factor, out=res[i], stream=s)
            elif k == "reduce_scatter":
                work[i].copy_(inp[i])
                out = work[i][rank * c:(rank + 1) * c] if o["inplace"] else res[i]
                comm.reduce_scatter(work[i], out, op=o["op"], factor=factor, stream=s)
            elif k == "allgather":
                if o["inplace"]:
                    res[i][rank * c:(rank + 1) * c].copy_(inp[i])
                    comm.allgather(res[i][rank * c:(rank + 1) * c], res[i], stream=s)
                else:
                    comm.allgather(inp[i], res[i], stream=s)
            else:
                work[i].copy_(inp[i])
                comm.broadcast(work[i], root=o["root"], stream=s)
            if join and not sticky_defer and (i + 1 == len(ops) or not is_join(ops[i + 1])):
                comm.flush(stream=s)          # the run's last gather, on the join stream
                comm.set_defer(False)
            if join:
                comm.set_join_stream(None)
        if sticky_defer:   # deferral stayed on across every later call: flush at the end
            comm.flush(stream=s)
            comm.set_defer(False)
        if used_side:   # the join stream rejoins the capture
            s.wait_stream(side)

    g = torch.cuda.CUDAGraph(keep_graph=True)
    comm.capture_begin()
    with torch.cuda.graph(g, stream=s):
        program()
    h = comm.capture_end(g.raw_cuda_graph())
    g.instantiate()
    ex = g.raw_cuda_graph_exec()
    digests = []
    for rep in range(replays):
        check = rep % check_every == 0   # (soaks: fresh inputs and digests every k-th replay)
        if check:
            for i, o in enumerate(ops):
                x = stress_input(rank, dict(o, seed=o["seed"] + 100_000 * rep), n)
                inp[i].copy_(as_tensor(x, o["dtype"]))
            torch.cuda.synchronize()
        with torch.cuda.stream(s):
            comm.launch_prepare(h, ex, s)
            g.replay()
        if not check:
            digests.append(None)
            continue
        s.synchronize()
        row = []
        for i, o in enumerate(ops):
            k, c = o["kind"], o["size"]
            if k == "allreduce":
                t = work[i] if o["inplace"] else res[i]
            elif k == "reduce_scatter":
                t = work[i][rank * c:(rank + 1) * c] if o["inplace"] else res[i]
            elif k == "allgather":
                t = res[i]
            else:
                t = work[i]
            r = t.cpu()
            arr = r.numpy() if o["dtype"] == "f32" else r.view(torch.int16).numpy().view(np.uint16)
            row.append(digest(arr))
        digests.append(row)
    comm.barrier(120)
    comm.destroy()
    return {"digests": digests}
