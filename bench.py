"""Benchmark of the one-to-many SHM allreduce (BASELINE.json metric:
"SHM allreduce GB/s vs host-link peak; ResNet-50 img/s on 1g slices").

Workload (N=1): BASELINE configs[1]'s communication step - the ResNet-50
gradient (25,557,032 fp32 = 102,228,128 B, the size torchvision's resnet50
has) allreduced across the 7 1g instances of one B200 (rank order from
fm_select, one process per instance).  N>1 (torchrun, one process per GPU):
7 instances per GPU, 7N ranks in one communicator, rank order from fm_select
over N GPUs (weak scaling: the per-rank gradient is fixed).

A step = one allreduce of every rank's gradient.  `value` = the whole job's
aggregate: n_ranks x gradient bytes / step time (device time, CUDA events on
each rank's stream, max over ranks); `algbw_gbs` = gradient bytes / step
time, the usual per-buffer allreduce figure.  Inputs are device-resident and
7 x 102 MB per GPU of gradients plus the SHM slots exceed the 126 MB L2.
`e2e` = the same metric through the public API with host-resident data: every
rank's gradient sits in its registered pinned host buffer, the GPUs read it
and write the result back inside the timed region (fmx_allreduce_host).

`--impl reference` times the CPU restatement of the same algorithm
(oracle/flexshm_oracle.c: multi-threaded SHM reduce-scatter/all-gather,
bit-identical results) on the box's host cores - the reference itself has no
runnable allreduce (its data path is NCCL).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

RESNET50_PARAMS = 25_557_032
RANKS_PER_GPU = 7
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
# Host-link peaks measured on this pool's B200 box (profiles/r01_probe/bw.jsonl):
# copy-engine pinned H2D / D2H / bidirectional, PCIe Gen5 x16.
LINK_PEAK_FALLBACK = {"h2d": 55.61, "d2h": 56.77, "bidir": 100.21}
UNIT = "GB/s (aggregate: all ranks' gradient bytes allreduced per second; algbw_gbs = per-buffer)"


def parse_args(argv=None):
    p = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--ranks-per-gpu", type=int, default=RANKS_PER_GPU)
    p.add_argument("--count", type=int, default=RESNET50_PARAMS)
    p.add_argument("--dtype", choices=["f32", "bf16"], default="f32")
    p.add_argument("--transport", choices=["auto", "ce", "zc"], default="auto")
    p.add_argument("--mode", choices=["green", "mps", "full"], default="mps",
                   help="instance stand-in on a GPU without MIG (instance.py)")
    p.add_argument("--slice-bytes", type=int, default=0)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--out", default=None, help="also write the JSON line here")
    p.add_argument("--no-train", action="store_true", help="skip the ResNet-50 DP img/s leg")
    p.add_argument("--timeline", default=None, help="write a host-polled flag timeline here")
    p.add_argument("--stamps", default=None,
                   help="write a GPU-clock timeline of one allreduce (every op of every rank)")
    p.add_argument("--train-only", action="store_true")
    p.add_argument("--train-mode", choices=["green", "mps", "full"], default="mps")
    p.add_argument("--nccl", action="store_true",
                   help="N>1: also time stock NCCL over NVLink, one rank per GPU (comparison "
                        "point; opt-in because NCCL inside MPS clients is untested here)")
    p.add_argument("--nccl-shm", action="store_true",
                   help="N>1: the NCCL comparison point over NCCL's own SHM transport "
                        "(NCCL_P2P_DISABLE=1, NCCL_NVLS_ENABLE=0: the paper's SHM-vs-NET "
                        "setting, PAPER.md:750-770); a separate run from --nccl, because NCCL "
                        "reads these variables once per process")
    p.add_argument("--buckets", type=int, default=0,
                   help="probe: allreduce the gradient as K back-to-back buckets (join-stream mode)")
    p.add_argument("--bucket-serial", action="store_true",
                   help="with --buckets: default completion (each bucket joins the caller's stream)")
    p.add_argument("--load", type=int, default=0,
                   help="interference probe: N bf16 GEMMs per instance during the timed loop")
    p.add_argument("--dry-run", action="store_true",
                   help="orchestration only (no CUDA): stub rank bodies; for the CPU tests of "
                        "the torchrun N>1 path")
    p.add_argument("--sweep", action="store_true", help="message-size sweep (configs[4]) instead")
    p.add_argument("--sweep-max", type=int, default=1 << 30)
    p.add_argument("--sweep-op", choices=["allreduce", "reduce_scatter", "allgather", "broadcast"],
                   default="allreduce", help="collective of the --sweep (bytes = full buffer)")
    p.add_argument("--train-model", choices=["resnet50", "mobilenet_v2", "bert"],
                   default="resnet50", help="model of the --train-only leg")
    p.add_argument("--train-engine", choices=["auto", "graph", "ddp"], default="auto",
                   help="graph: ddp.ShmDataParallel, whole step captured as one CUDA graph; "
                        "ddp: torch DDP + flexshm_hook, eager; auto (default): graph")
    p.add_argument("--fused-sgd", action="store_true",
                   help="graph engine, conv nets: the SGD step fused into the collective "
                        "(ShmDataParallel fused_sgd / fmx_allreduce_sgd) instead of torch's "
                        "optimizer after it")
    p.add_argument("--train-no-sync", action="store_true",
                   help="--train-only: also time the step without gradient sync (compute bound)")
    p.add_argument("--bucket-mb", type=float, default=None,
                   help="bucket cap (MiB) of the DP legs; default 14 for ResNet-50 (graph "
                        "engine 4027-4037 img/s vs 3947-3949 at 8, r02/r3n), 25 for BERT-base "
                        "(2917-2958 seq/s vs 2284 at 8, r02/r3c-r3d), 8 otherwise")
    p.add_argument("--first-bucket-mb", type=float, default=1.0,
                   help="first bucket cap of the graph engine (DDP's first_bucket_bytes)")
    p.add_argument("--compress", choices=["bf16"], default=None,
                   help="DP legs: exchange fp32 gradients in bf16 (flexshm_bf16_hook)")
    p.add_argument("--batch", type=int, default=32)
    p.add_argument("--train-steps", type=int, default=10)
    p.add_argument("--train-warmup", type=int, default=5)
    return p.parse_args(argv)


# ----------------------------------------------------------------------------- helpers


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return int(os.environ.get("RANK", "0")), ws, int(os.environ.get("LOCAL_RANK", "0"))


def decision_for(gpus: int, ranks_per_gpu: int):
    from paper_2511_09143_b200.scheduler import fm_select, make_cluster
    from paper_2511_09143_b200.workload import Job
    d = fm_select(Job(0, "train", gpus * ranks_per_gpu, 0.0, 0.0), make_cluster("FM", gpus))
    assert d is not None and len(d.instances) == gpus * ranks_per_gpu
    return d


def link_bytes(n: int, per_gpu: list[int], s_bytes: int):
    """Algorithmic host-link bytes per allreduce for each GPU:
    D2H_g = k_g * S, H2D_g = 2 k_g (n-1)/n * S."""
    return [(k * s_bytes, 2 * k * (n - 1) * s_bytes / n) for k in per_gpu]


# Host memory bandwidth (read + write bytes, all host threads), measured on the
# GPU box (profiles/r01_probe/bw.jsonl "host_memcpy"); bench.py re-measures it
# in the run (host_dram_gbs) and uses that when it can.
HOST_DRAM_FALLBACK = 184.78


def host_dram_gbs(nbytes: int = 1 << 30) -> float:
    """Best-of-3 multithreaded host copy, read+write bytes per second (GB/s):
    the B_dram of the roofline's host-memory term."""
    import torch
    torch.set_num_threads(os.cpu_count() or 1)
    a = torch.ones(nbytes // 4)
    b = torch.empty_like(a)
    best = float("inf")
    for _ in range(3):
        t0 = time.perf_counter()
        b.copy_(a)
        best = min(best, time.perf_counter() - t0)
    return 2 * nbytes / best / 1e9


def step_roofline(n, per_gpu, s_bytes, t_s, peaks):
    """T* = max_g max(D2H_g/B_d2h, H2D_g/B_h2d, (D2H_g+H2D_g)/B_bidir),
    per_gpu = ranks on each PHYSICAL GPU (logical GPUs sharing one device share
    its link).  The host-DRAM term sum_g (D2H_g+H2D_g) / B_dram is reported
    beside it (t_dram_ms) but does not enter T* / frac: the only B_dram this box
    can measure is a CPU copy on its 16 vCPUs (host_dram_gbs), a LOWER bound of
    the DRAM bandwidth - GPU DMA alone has been measured above it (bidir 100.2
    vs ~93 GB/s) - so it would overstate T* and inflate frac.  It is the term to
    watch when 8 GPUs share one host (N>1 runs)."""
    tstar = 0.0
    lb = link_bytes(n, per_gpu, s_bytes)
    for d2h, h2d in lb:
        tstar = max(tstar, d2h / (peaks["d2h"] * 1e9), h2d / (peaks["h2d"] * 1e9),
                    (d2h + h2d) / (peaks["bidir"] * 1e9))
    dram_bytes = sum(d + h for d, h in lb)
    b_dram = peaks.get("dram", HOST_DRAM_FALLBACK)
    t_dram = dram_bytes / (b_dram * 1e9)
    d2h0, h2d0 = lb[0]
    return {"bound": "host_link", "t_star_ms": tstar * 1e3, "frac": tstar / t_s,
            "achieved": (d2h0 + h2d0) / t_s / 1e9, "unit": "GB/s",
            "peak_bidir": peaks["bidir"], "peak_h2d": peaks["h2d"], "peak_d2h": peaks["d2h"],
            "link_bytes_per_gpu": {"d2h": d2h0, "h2d": h2d0}, "ranks_per_physical_gpu": per_gpu,
            "host_dram": {"bytes": dram_bytes, "b_dram_cpu_copy_gbs": b_dram,
                          "t_dram_ms": t_dram * 1e3,
                          "note": "B_dram = multithreaded CPU copy (read+write bytes), a lower "
                                  "bound of host DRAM bandwidth: t_dram is an upper estimate, "
                                  "reported, not used for frac"},
            "peak_source": "host link: profiles/r01_probe/bw.jsonl (cudaMemcpyAsync pinned, "
                           "best of 5); host DRAM: " + peaks.get("dram_source", "r01 probe")}


def physical_split(d, gpus: int) -> list[int]:
    """Ranks per physical GPU: the decision's per-GPU counts, merged where
    FMX_DEVICE_MAP puts several logical GPUs on one device."""
    per = [sum(1 for g, _ in d.instances if g == gg) for gg in range(gpus)]
    dm = os.environ.get("FMX_DEVICE_MAP")
    if not dm:
        return per
    phys: dict[str, int] = {}
    for gg, dev in enumerate(dm.split(",")[:gpus]):
        phys[dev] = phys.get(dev, 0) + per[gg]
    return list(phys.values())


def workload_name(count: int, dtype: str) -> str:
    return {RESNET50_PARAMS: "ResNet-50", 3_504_872: "MobileNetV2",
            109_483_778: "BERT-base"}.get(count, "synthetic") + f"-sized gradient ({count} {dtype})"


# SM zero-copy store peak to mapped host memory (profiles/r01_probe/bw.jsonl, "zc"
# write_gbs, any grid >= 8 CTAs) - the bound of the reduce kernel's result store.
ZC_WRITE_PEAK = 52.7
# ... and the same store while copy engines stream H2D and D2H concurrently
# (profiles/r02/r2k/probe_zc_*.jsonl, load=both, mean of full-GPU and 14 % MPS)
ZC_WRITE_UNDER_LOAD = 21.1
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def kernel_roofline(args, n, s_bytes, kernel_ms, kernel_count, iso_us=None, iso_piece=None):
    """Roofline of the dominant kernel, fmx_reduce_kernel, from its live
    CUDA-event durations (lane stream) over the timed region.

    Algorithmic bytes of all reduce launches of one allreduce (all ranks):
    HBM reads n*S (CE: n-1 contributions from scratch + own piece), HBM
    write S, and - unless the result slot is written by the copy engine
    (FMX_RESULT_VIA_CE=1) - a zero-copy store of S over PCIe, which is then
    the binding resource.  ZC transport: (n-1)*S cross PCIe as loads."""
    if kernel_count == 0:
        return None
    steps = args.steps
    t_launch = kernel_ms / kernel_count / 1e3          # mean launch duration, s
    per_launch = lambda total: total * steps / kernel_count
    via_ce = os.environ.get("FMX_RESULT_VIA_CE", "0") not in ("", "0")
    zc = args.transport == "zc"
    traffic = None
    try:
        # ncu --set full capture of one full piece (profiles/ncu_traffic.json), DRAM bytes
        # per piece byte, scaled to the mean piece of the live launches like `achieved`
        t = json.load(open(TRAFFIC_PATH))
        traffic = (t["dram_read_bytes"] + t["dram_write_bytes"]) / t["piece_bytes"] * \
            per_launch(s_bytes)
    except (OSError, ValueError, KeyError):
        pass
    if zc:
        link = per_launch((n - 1) * s_bytes + s_bytes)
        return {"kernel": "fmx_reduce_kernel", "bound": "host_link", "achieved": link / t_launch / 1e9,
                "peak": LINK_PEAK_FALLBACK["bidir"], "unit": "GB/s",
                "frac": link / t_launch / 1e9 / LINK_PEAK_FALLBACK["bidir"], "traffic": None,
                "launch_us": t_launch * 1e6, "launches": kernel_count,
                "peak_source": "measured CE bidirectional (profiles/r01_probe/bw.jsonl)"}
    if via_ce:
        hbm = per_launch((n + 1) * s_bytes)
        peak = json.load(open(PEAKS_PATH))["hbm_gbs"] if os.path.exists(PEAKS_PATH) else 6552.3
        return {"kernel": "fmx_reduce_kernel", "bound": "hbm", "achieved": hbm / t_launch / 1e9,
                "peak": peak, "unit": "GB/s", "frac": hbm / t_launch / 1e9 / peak,
                "traffic": traffic, "launch_us": t_launch * 1e6, "launches": kernel_count,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    link = per_launch(s_bytes)
    line = {"kernel": "fmx_reduce_kernel", "bound": "host_link",
            "achieved": link / t_launch / 1e9, "peak": ZC_WRITE_PEAK, "unit": "GB/s",
            "frac": link / t_launch / 1e9 / ZC_WRITE_PEAK, "traffic": traffic,
            "bytes_per_launch": {"pcie_store": link, "hbm_read": per_launch(n * s_bytes),
                                 "hbm_write": link},
            "launch_us": t_launch * 1e6, "launches": kernel_count,
            "timing": "CUDA events around every reduce launch on its lane stream, inside the "
                      "timed region",
            "peak_source": "measured SM zero-copy store peak (profiles/r01_probe/bw.jsonl)",
            # the same store while copy engines stream both directions, as they do
            # throughout the pipeline (other ranks' stages / fetches / gathers):
            # the contended ceiling the live launches run against
            "under_link_load": {"peak": ZC_WRITE_UNDER_LOAD,
                                "frac": link / t_launch / 1e9 / ZC_WRITE_UNDER_LOAD,
                                "peak_source": "tools/probe_zc_contention.py, load=both: the "
                                               "same kernel and piece alone 48 GB/s, with "
                                               "concurrent CE H2D + D2H 20.4-21.7 GB/s "
                                               "(profiles/r02/r2k)"}}
    if iso_us:
        line["isolated"] = {"launch_us": iso_us, "piece_bytes": iso_piece,
                            "achieved": iso_piece / (iso_us * 1e-6) / 1e9,
                            "frac": iso_piece / (iso_us * 1e-6) / 1e9 / ZC_WRITE_PEAK,
                            "hbm_gbs": (n + 1) * iso_piece / (iso_us * 1e-6) / 1e9,
                            "timing": "same kernel, same piece, rank 0 alone (peers parked)"}
    return line


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- rank body


def graphed(comm, stream, step):
    """`step` (collectives enqueued on `stream`) captured once as a CUDA graph;
    returns the replay function (fmx_graph_* re-bases its flags per launch)."""
    import torch
    g = torch.cuda.CUDAGraph(keep_graph=True)
    comm.capture_begin()
    try:
        with torch.cuda.graph(g, stream=stream):
            step()
    except BaseException:
        comm.capture_end(0)
        raise
    h = comm.capture_end(g.raw_cuda_graph())
    g.instantiate()
    ex = g.raw_cuda_graph_exec()

    def replay():
        comm.launch_prepare(h, ex, stream)
        with torch.cuda.stream(stream):
            g.replay()
    replay.graph = g
    return replay


def rank_body(rank: int, job_key: str, n: int, cfg: dict, inst_mode: str, gpu_local: int):
    """One instance rank: bind, join, warm up, then time K allreduces three
    ways - (1) device-resident gradient (`value`), (2) host-resident
    gradient in the rank's registered host buffer, read and written over the
    host link by fmx_allreduce_host (`e2e`), (3) host gradient copied H2D,
    allreduced on the device, copied D2H (`e2e_device_buffers`).  Every
    allreduce uses DDP's convention (divide by world size, then sum)."""
    import torch

    from paper_2511_09143_b200 import instance as inst_mod
    from paper_2511_09143_b200.comm import init_process_group

    gpu_id, inst_id = cfg["instances"][rank]
    inst = inst_mod.bind(gpu_id, inst_id, cfg["profiles"][rank], mode=inst_mode, device=gpu_local)
    count = cfg["count"]
    tdt = torch.float32 if cfg["dtype"] == "f32" else torch.bfloat16
    esz = 4 if cfg["dtype"] == "f32" else 2
    comm = init_process_group(None, rank, job_key, instance=inst, nranks=n,
                              transport=cfg["transport"], slice_bytes=cfg["slice_bytes"],
                              host_bytes=count * esz if cfg["e2e"] else 0, timeout_s=300)
    stream = inst.stream
    gen = torch.Generator(device="cpu").manual_seed(1234 + rank)
    host = (torch.randn(count, generator=gen) * (1e-3 if cfg["dtype"] == "f32" else 1e-2)).to(tdt)
    with torch.cuda.stream(stream):
        buf = host.to(f"cuda:{gpu_local}")
    out = {"rank": rank}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(k: int, step, kernel_timing: bool = False):
        comm.barrier(300)
        torch.cuda.synchronize()
        comm.barrier(300)
        l0 = comm.kernel_launches()
        comm.set_kernel_timing(kernel_timing)
        ev0.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(k):
                step()
        ev1.record(stream)
        ev1.synchronize()
        comm.barrier(300)
        if kernel_timing:
            out["kernel_ms"], out["kernel_count"] = comm.kernel_time()
            comm.set_kernel_timing(False)
        return ev0.elapsed_time(ev1), comm.kernel_launches() - l0

    if cfg.get("buckets", 0) > 1:
        # DDP-bucket pattern: the gradient as K back-to-back allreduces of distinct
        # views, forked from `stream`, overlapping in join-stream mode; the step
        # ends when the last completes (waited for on `stream`)
        views = list(buf.chunk(cfg["buckets"]))
        side = torch.cuda.Stream(device=gpu_local) if inst.green_ctx is None else \
            torch.cuda.ExternalStream(inst.green_ctx.Stream().cuda_stream)
        done_ev = torch.cuda.Event()

        def device_step():
            if cfg.get("bucket_join", True):
                comm.set_join_stream(side)
            for v in views:
                comm.allreduce(v, op="avg", stream=stream)
            done = comm.completion_stream()
            comm.set_join_stream(None)
            done_ev.record(torch.cuda.ExternalStream(done))
            stream.wait_event(done_ev)
    else:
        def device_step():
            comm.allreduce(buf, op="avg", stream=stream)

    for _ in range(cfg["warmup"]):
        device_step()
    torch.cuda.synchronize()
    if os.environ.get("FMX_BENCH_GRAPH") == "1":
        # experiment: the allreduce captured once, replayed per step (fmx_graph_*)
        device_step = graphed(comm, stream, device_step)
        for _ in range(cfg["warmup"]):
            device_step()
        torch.cuda.synchronize()
    if cfg.get("load"):
        # interference probe: keep this instance's SMs busy with bf16 GEMMs on
        # another stream while the allreduces run (what DP training does)
        load_stream = torch.cuda.Stream()
        a = torch.randn(4096, 4096, device=f"cuda:{gpu_local}", dtype=torch.bfloat16)
        with torch.cuda.stream(load_stream):
            for _ in range(cfg["load"]):
                a = (a @ a).clamp_(-1, 1)
    out["ms_total"], out["launches"] = timed(cfg["steps"], device_step, kernel_timing=True)
    if cfg.get("timeline"):
        # host-side flag timeline of 2 allreduces (rank 0 polls the segment)
        import threading as _th
        rec = {}
        comm.barrier(300)
        torch.cuda.synchronize()
        if rank == 0:
            mon = _th.Thread(target=lambda: rec.setdefault("ev", comm.monitor(0.4)))
            mon.start()
            time.sleep(0.01)
        comm.barrier(300)
        t_host = time.perf_counter()
        for _ in range(2):
            device_step()
        torch.cuda.synchronize()
        out["timeline_host_s"] = time.perf_counter() - t_host
        if rank == 0:
            mon.join()
            with open(cfg["timeline"], "w") as f:
                json.dump({"n": n, "slice_bytes": comm.slice_bytes, "count": count,
                           "events": rec.get("ev", [])}, f)
        comm.barrier(300)
    if cfg.get("stamps"):
        # pipeline timeline probe: one device-buffer allreduce with a GPU-clock
        # stamp after every operation of every lane (bench --stamps)
        comm.barrier(300)
        torch.cuda.synchronize()
        comm.set_stamps(1 << 14)
        comm.barrier(300)
        for _ in range(int(os.environ.get("FMX_STAMP_STEPS", "1"))):
            device_step()
        torch.cuda.synchronize()
        out["stamps_device"] = comm.stamps(1 << 14)
        comm.set_stamps(0)
        comm.barrier(300)
    # isolated kernel timing (rank 0 only, every other rank parked at the
    # barrier, so no time-slicing with peers): fmx_reduce_kernel on one
    # pipeline piece, n HBM sources, zero-copy result store to pinned host
    # memory - exactly what each round of the CE transport launches
    if rank == 0:
        from paper_2511_09143_b200.comm import reduce_local
        piece = min(comm.slice_bytes // esz, (count + n - 1) // n)
        srcs = [torch.randn(piece, device=f"cuda:{gpu_local}").to(tdt) for _ in range(n)]
        kout = torch.empty(piece, dtype=tdt, device=f"cuda:{gpu_local}")
        kout_host = torch.empty(piece, dtype=tdt).pin_memory()
        with torch.cuda.stream(stream):
            for _ in range(3):
                reduce_local(srcs, kout, op="avg", out_host=kout_host, stream=stream)
            ev0.record(stream)
            for _ in range(20):
                reduce_local(srcs, kout, op="avg", out_host=kout_host, stream=stream)
            ev1.record(stream)
        ev1.synchronize()
        out["iso_kernel_us"] = ev0.elapsed_time(ev1) * 1e3 / 20
        out["iso_piece_bytes"] = piece * esz
        del srcs, kout, kout_host
    comm.barrier(300)
    if cfg["e2e"]:
        # (2) registered host buffer: the gradient lives in pinned host memory
        region = comm.host_buffer()[:count * esz].view(tdt)
        region.copy_(host)

        def host_step():
            comm.allreduce_host(region, op="avg", stream=stream)

        for _ in range(cfg["warmup"]):
            host_step()
        torch.cuda.synchronize()
        if os.environ.get("FMX_BENCH_GRAPH") == "1":
            host_step = graphed(comm, stream, host_step)
            for _ in range(cfg["warmup"]):
                host_step()
            torch.cuda.synchronize()
        out["ms_total_e2e"], out["launches_e2e"] = timed(cfg["steps"], host_step)
        out["e2e_digest"] = int(region.view(torch.int32 if esz == 4 else torch.int16)
                                .to(torch.int64).sum().item())
        if cfg.get("stamps"):
            comm.barrier(300)
            torch.cuda.synchronize()
            comm.set_stamps(1 << 14)
            comm.barrier(300)
            host_step()
            torch.cuda.synchronize()
            out["stamps_host"] = comm.stamps(1 << 14)
            comm.set_stamps(0)
            comm.barrier(300)
        # (3) device buffers with explicit H2D / D2H copies of the gradient
        pin_in = host.pin_memory()
        pin_out = torch.empty_like(pin_in).pin_memory()

        def copy_step():
            buf.copy_(pin_in, non_blocking=True)
            comm.allreduce(buf, op="avg", stream=stream)
            pin_out.copy_(buf, non_blocking=True)

        with torch.cuda.stream(stream):
            copy_step()
        torch.cuda.synchronize()
        out["ms_total_e2e_dev"], _ = timed(cfg["steps"], copy_step)
    comm.destroy()
    return out


def _spawned_rank(rank, job_key, n, cfg, inst_mode, gpu_local):
    return rank_body(rank, job_key, n, cfg, inst_mode, gpu_local)


SWEEP_SIZES = [1 << k for k in range(10, 31, 2)]  # 1 KiB ... 1 GiB (BASELINE configs[4])


def sweep_body(rank: int, job_key: str, n: int, cfg: dict, inst_mode: str, gpu_local: int):
    """Size sweep (BASELINE configs[4]): device-buffer allreduce latency /
    algbw from 1 KiB to 1 GiB.  Per size: warm-up, then enough back-to-back
    calls for ~0.2 s of work, CUDA events on the rank's stream."""
    import torch

    from paper_2511_09143_b200 import instance as inst_mod
    from paper_2511_09143_b200.comm import init_process_group

    gpu_id, inst_id = cfg["instances"][rank]
    inst = inst_mod.bind(gpu_id, inst_id, cfg["profiles"][rank], mode=inst_mode, device=gpu_local)
    comm = init_process_group(None, rank, job_key, instance=inst, nranks=n,
                              transport=cfg["transport"], slice_bytes=cfg["slice_bytes"],
                              timeout_s=300)
    stream = inst.stream
    esz = 4 if cfg["dtype"] == "f32" else 2
    tdt = torch.float32 if esz == 4 else torch.bfloat16
    sizes = [b for b in cfg["sizes"]]
    with torch.cuda.stream(stream):
        buf = torch.randn(max(sizes) // esz, device=f"cuda:{gpu_local}").to(tdt)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = {"rank": rank, "ms": {}}
    op = cfg.get("sweep_op", "allreduce")
    with torch.cuda.stream(stream):
        obuf = torch.empty(max(sizes) // esz, dtype=tdt, device=f"cuda:{gpu_local}")
    torch.cuda.synchronize()

    def call(x, b):
        # b = bytes of the full (n-block) buffer for reduce_scatter / allgather
        if op == "allreduce":
            comm.allreduce(x, op="avg", stream=stream)
        elif op == "broadcast":
            comm.broadcast(x, root=0, stream=stream)
        elif op == "reduce_scatter":
            blk = x.numel() // n
            comm.reduce_scatter(x[:blk * n], obuf[:blk], op="avg", stream=stream)
        else:
            blk = x.numel() // n
            comm.allgather(x[:blk], obuf[:blk * n], stream=stream)

    for b in sizes:
        x = buf[: b // esz]
        k = max(3, min(200, int(0.2 / max(b * 2 / 50e9 * n, 40e-6))))
        for _ in range(3):
            call(x, b)
        comm.barrier(300)
        torch.cuda.synchronize()
        comm.barrier(300)
        ev0.record(stream)
        for _ in range(k):
            call(x, b)
        ev1.record(stream)
        ev1.synchronize()
        out["ms"][b] = (ev0.elapsed_time(ev1) / k, k)
    comm.barrier(300)
    comm.destroy()
    return out


def _spawned_sweep(rank, job_key, n, cfg, inst_mode, gpu_local):
    return sweep_body(rank, job_key, n, cfg, inst_mode, gpu_local)


def run_sweep(args) -> list[dict]:
    """One JSON line per message size, ranks of one GPU (1-GPU layout)."""
    d = decision_for(args.gpus, args.ranks_per_gpu)
    n = len(d.instances)
    cfg = {"instances": d.instances, "profiles": d.profiles, "transport": args.transport,
           "slice_bytes": args.slice_bytes, "dtype": args.dtype,
           "sizes": [b for b in SWEEP_SIZES if b <= args.sweep_max], "sweep_op": args.sweep_op}
    res = run_ranks(sweep_body, _spawned_sweep, list(range(n)), f"sweep-{os.getpid()}", n, cfg,
                    args.mode, 0)
    lines = []
    # every sweep rank runs on device 0 of this node (gpus > 1: logical GPUs of
    # one device), so all n ranks share one physical link
    per_gpu = [n]
    peaks = dict(LINK_PEAK_FALLBACK, dram=host_dram_gbs(), dram_source="measured in this run")
    for b in cfg["sizes"]:
        ms = max(r["ms"][b][0] for r in res.values())
        lines.append({"sweep": f"{args.sweep_op} size sweep (BASELINE configs[4])", "bytes": b,
                      "op": args.sweep_op,
                      "ranks": n, "instance_mode": args.mode, "dtype": args.dtype,
                      "ms": ms, "algbw_gbs": b / ms / 1e6,
                      "busbw_gbs": b / ms / 1e6 * 2 * (n - 1) / n,
                      "iters": res[0]["ms"][b][1],
                      "step_roofline_frac": step_roofline(n, per_gpu, b, ms / 1e3,
                                                          peaks)["frac"]
                      if args.sweep_op == "allreduce" else None})
    return lines


def train_body(rank: int, job_key: str, n: int, cfg: dict, inst_mode: str, gpu_local: int):
    """One instance rank of ResNet-50 data-parallel training (BASELINE
    configs[1]): batch 32 per instance, synthetic ImageNet-shaped inputs,
    random init, bf16 autocast with fp32 weights and gradients, SGD; DDP
    gradient buckets allreduced over SHM by ddp.flexshm_hook."""
    import torch
    import torch.distributed as dist
    import torch.nn.functional as F
    import torchvision

    from paper_2511_09143_b200 import ddp as fddp
    from paper_2511_09143_b200 import instance as inst_mod
    from paper_2511_09143_b200.comm import init_process_group

    gpu_id, inst_id = cfg["instances"][rank]
    inst = inst_mod.bind(gpu_id, inst_id, cfg["profiles"][rank], mode=inst_mode, device=gpu_local)
    comm = init_process_group(None, rank, job_key, instance=inst, nranks=n,
                              transport=cfg["transport"], timeout_s=300)
    pg, own_pg = None, False
    if cfg.get("engine", "graph") != "graph":
        # torch DDP's control plane (parameter-shape checks) on gloo over the same ranks
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(cfg["port"])
        pg = dist.new_group(backend="gloo") if dist.is_initialized() else None
        if pg is None:
            dist.init_process_group("gloo", rank=rank, world_size=n)
            pg, own_pg = dist.group.WORLD, True
    stream = inst.stream
    torch.manual_seed(0)
    name = cfg.get("model", "resnet50")
    graph = cfg.get("engine", "graph") == "graph"
    g = torch.Generator(device="cpu").manual_seed(100 + rank)
    with torch.cuda.stream(stream):
        if name == "bert":
            # BASELINE configs[3]: BERT-base fine-tune shape, bf16 weights and gradients
            # (bf16 SHM allreduce), seq 128, 2 labels
            from transformers import BertConfig, BertForSequenceClassification
            if graph:
                _sdpa_mask_skip_in_capture()
            model = BertForSequenceClassification(BertConfig(num_labels=2)).cuda(gpu_local)
            model = model.to(torch.bfloat16)
            x = torch.randint(0, 30522, (cfg["batch"], 128), generator=g).cuda(gpu_local)
            y = torch.randint(0, 2, (cfg["batch"],), generator=g).cuda(gpu_local)
        else:
            ctor = {"resnet50": torchvision.models.resnet50,
                    "mobilenet_v2": torchvision.models.mobilenet_v2}[name]
            model = ctor().cuda(gpu_local).to(memory_format=torch.channels_last)
            x = torch.randn(cfg["batch"], 3, 224, 224, generator=g).cuda(gpu_local)
            x = x.to(memory_format=torch.channels_last)
            y = torch.randint(0, 1000, (cfg["batch"],), generator=g).cuda(gpu_local)
        if not graph:
            net = fddp.wrap(model, comm, control_group=pg, bucket_cap_mb=cfg.get("bucket_mb", 25.0),
                            compress=cfg.get("compress"),
                            threaded=bool(os.environ.get("FMX_HOOK_THREAD")))
        elif cfg.get("no_sync"):
            fddp.broadcast_parameters(model, comm)   # same start, no exchange in the step
            net = model
        else:
            fused = dict(lr=0.01, momentum=0.9) if cfg.get("fused_sgd") else None
            net = fddp.ShmDataParallel(model, comm, bucket_cap_mb=cfg.get("bucket_mb", 8.0),
                                       first_bucket_mb=cfg.get("first_bucket_mb", 1.0),
                                       compress=cfg.get("compress"), fused_sgd=fused)
        if name == "bert":
            # in a graph: the fused multi-tensor AdamW (capturable), one kernel per step
            opt = torch.optim.AdamW(net.parameters(), lr=2e-5, capturable=graph,
                                    fused=True if graph else None)
        elif cfg.get("fused_sgd") and graph and not cfg.get("no_sync"):
            opt = None   # the same SGD step runs inside the collective (fmx_allreduce_sgd)
        else:
            opt = torch.optim.SGD(net.parameters(), lr=0.01, momentum=0.9)

    from contextlib import nullcontext

    def step():
        with (net.no_sync() if cfg.get("no_sync") and not graph else nullcontext()):
            return _step()

    host_phase = {"fwd": 0.0, "bwd": 0.0, "opt": 0.0}  # host enqueue seconds per phase

    def _step():
        t0 = time.perf_counter()
        if graph:   # the buckets (or .grad) stay in place: zero them, do not drop them
            net.zero_grad(set_to_none=False)
        if name == "bert":
            loss = F.cross_entropy(net(input_ids=x).logits.float(), y)
        else:
            # (no autocast weight cache: a graph replays the casts every step)
            with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=not graph):
                loss = F.cross_entropy(net(x), y)
        if not graph:
            opt.zero_grad(set_to_none=True)
        t1 = time.perf_counter()
        loss.backward()
        t2 = time.perf_counter()
        if opt is not None:
            opt.step()
        t3 = time.perf_counter()
        host_phase["fwd"] += t1 - t0
        host_phase["bwd"] += t2 - t1
        host_phase["opt"] += t3 - t2
        return loss

    replay = None
    with torch.cuda.stream(stream):
        if graph and not cfg.get("no_sync"):
            # warmup eager steps, then the whole step as one CUDA graph (with
            # --stamps: stamp slots baked into it, rewritten by every replay)
            replay = net.graphed_step(step, warmup=cfg["train_warmup"], before_capture=(
                (lambda: comm.set_stamps(1 << 15)) if cfg.get("stamps") else None))
        elif graph:
            replay = graphed_plain(step, cfg["train_warmup"])
        else:
            for _ in range(cfg["train_warmup"]):
                step()
    torch.cuda.synchronize()
    stamps = None
    if cfg.get("stamps") and (not graph or replay is not None and not cfg.get("no_sync")):
        # one step on the GPU clock: markers 1/2 around it on the compute stream,
        # every collective op of the hook's side stream in between
        comm.barrier(300)
        if not graph:
            comm.set_stamps(1 << 15)
        comm.barrier(300)
        with torch.cuda.stream(stream):
            comm.stamp(1, stream)
            replay() if replay is not None else step()
            comm.stamp(2, stream)
        torch.cuda.synchronize()
        stamps = comm.stamps(1 << 15)
        if replay is None:   # a captured graph keeps writing its baked stamp slots
            comm.set_stamps(0)
    comm.barrier(300)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = comm.kernel_launches()
    h0 = list(fddp.HOOK_HOST)
    for k in host_phase:
        host_phase[k] = 0.0
    t_host = time.perf_counter()
    ev0.record(stream)
    with torch.cuda.stream(stream):
        for _ in range(cfg["train_steps"]):
            loss = replay() if replay is not None else step()
    ev1.record(stream)
    t_host = time.perf_counter() - t_host  # enqueue time of the timed steps (no sync inside)
    ev1.synchronize()
    comm.barrier(300)
    out = {"rank": rank, "ms_total": ev0.elapsed_time(ev1), "loss": float(loss.item()),
           "host_enqueue_ms": t_host * 1e3,
           "hook_host_ms": (fddp.HOOK_HOST[0] - h0[0]) * 1e3, "hook_calls": fddp.HOOK_HOST[1] - h0[1],
           "host_phase_ms": {k: v * 1e3 for k, v in host_phase.items()},
           "stamps": stamps,
           "launches": comm.kernel_launches() - l0,
           "param_digest": float(sum(p.detach().double().sum().item() for p in model.parameters()))}
    if own_pg:
        dist.destroy_process_group()
    comm.destroy()
    return out


def _sdpa_mask_skip_in_capture():
    """HF BERT skips its all-ones attention mask in eager mode (no padding:
    SDPA dispatches to the flash / cuDNN kernels) but cannot check the mask
    while a CUDA graph is captured, so the captured step would carry a dense
    mask down SDPA's math path: 3x slower inside a 14 % MPS client
    (profiles/r02/r2u).  The synthetic sequences have no padding and pass no
    mask, so skip it under capture too - the same computation as eager."""
    import transformers.masking_utils as mu
    if getattr(mu, "_fmx_patched", False):
        return
    orig = mu._ignore_bidirectional_mask_sdpa

    def skip(padding_mask, kv_length, local_attention_size=None):
        if padding_mask is None and local_attention_size is None:
            return True
        return orig(padding_mask, kv_length, local_attention_size)
    mu._ignore_bidirectional_mask_sdpa = skip
    mu._fmx_patched = True


def graphed_plain(step, warmup: int):
    """A step without collectives as one CUDA graph (the no-sync bound of the
    graph engine): `warmup` eager steps on the current stream, then capture."""
    import torch
    s = torch.cuda.current_stream()
    for _ in range(max(1, warmup)):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        out = step()

    def replay():
        g.replay()
        return out
    return replay


def _spawned_train(rank, job_key, n, cfg, inst_mode, gpu_local):
    return train_body(rank, job_key, n, cfg, inst_mode, gpu_local)


# ----------------------------------------------------------------------------- arms


def run_ranks(body, spawned, mine, job_key, n, cfg, inst_mode, gpu_local, sampler=None):
    """Rank mine[0] runs in this process, the rest in spawned processes."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    results, errors = {}, []
    if inst_mode == "mps" and "CUDA_MPS_PIPE_DIRECTORY" not in os.environ:
        raise RuntimeError("MPS instance mode needs the daemon started by main()")
    try:
        with ctx.Pool(max(1, len(mine) - 1)) as pool:
            pending = [pool.apply_async(spawned, (r, job_key, n, cfg, inst_mode, gpu_local))
                       for r in mine[1:]]
            if sampler is not None:
                sampler.start()
            try:
                results[mine[0]] = body(mine[0], job_key, n, cfg, inst_mode, gpu_local)
            except BaseException as exc:  # noqa: BLE001
                errors.append((mine[0], exc))
            for r, a in zip(mine[1:], pending):
                try:
                    results[r] = a.get(timeout=900)
                except BaseException as exc:  # noqa: BLE001
                    errors.append((r, exc))
    finally:
        pass
    if errors:
        raise RuntimeError(f"rank {errors[0][0]} failed: {errors[0][1]!r}") from errors[0][1]
    return results


TRAIN_MODELS = {
    "resnet50": ("torchvision resnet50, random init, synthetic 224x224 inputs",
                 "bf16 autocast, fp32 weights/grads (fp32 SHM allreduce)", "img_s"),
    "mobilenet_v2": ("torchvision mobilenet_v2, random init, synthetic 224x224 inputs "
                     "(BASELINE configs[2] model)",
                     "bf16 autocast, fp32 weights/grads (fp32 SHM allreduce)", "img_s"),
    "bert": ("HF BertForSequenceClassification (bert-base config), random init, synthetic "
             "seq-128 token ids (BASELINE configs[3] model)",
             "bf16 weights and gradients (bf16 SHM allreduce, fp32 accumulate)", "seq_s"),
}


def run_train(args, d, job_key, model: str = "resnet50", no_sync: bool = False) -> dict | None:
    """Data-parallel training throughput on the instances of `d`: one
    communicator over all of them; under torchrun (N > 1) each process runs its
    GPU's instance ranks, the time is the max over every rank of every process
    and rank 0 returns the line (the others None).  Graph engine:
    ddp.ShmDataParallel, the step as one CUDA graph; ddp engine: torch DDP +
    ddp.flexshm_hook (gloo control group, single-process layouts only)."""
    import torch

    grank, world, local = dist_env()
    n = len(d.instances)
    engine = args.train_engine if args.train_engine != "auto" else "graph"
    if world > 1 and engine == "ddp":
        raise ValueError("the eager DDP engine's gloo control group is single-process: "
                         "use --train-engine graph under torchrun")
    cfg = {"instances": d.instances, "profiles": d.profiles, "transport": args.transport,
           "batch": args.batch, "train_steps": args.train_steps, "train_warmup": args.train_warmup,
           "port": 29000 + os.getpid() % 1000, "model": model, "no_sync": no_sync,
           "bucket_mb": args.bucket_mb if args.bucket_mb is not None else
           {"bert": 25.0, "resnet50": 14.0}.get(model, 8.0),
           "first_bucket_mb": args.first_bucket_mb,
           # (the default run's --stamps is for the allreduce; a training timeline
           # is asked for with --train-only --stamps: stamp kernels slow the step)
           "stamps": bool(args.stamps) and args.train_only and not no_sync, "engine": engine,
           "compress": args.compress, "fused_sgd": args.fused_sgd}
    mine, gpu_local = list(range(n)), 0
    if world > 1:
        import torch.distributed as dist
        obj = [job_key if grank == 0 else None]
        dist.broadcast_object_list(obj, src=0)     # one job key for every process
        job_key = obj[0]
        mine = [r for r, (g, _) in enumerate(d.instances) if g == grank]
        gpu_local = local if not os.environ.get("FMX_ONE_GPU_VISIBLE") else 0
        if os.environ.get("FMX_DEVICE_MAP"):
            gpu_local = int(os.environ["FMX_DEVICE_MAP"].split(",")[local])
    res, err = {}, None
    try:
        res = run_ranks(train_body, _spawned_train, mine, job_key + "-t", n, cfg,
                        args.train_mode, gpu_local)
    except Exception as exc:  # noqa: BLE001 - every process must reach the reductions below
        err = exc
    t_local = max((r["ms_total"] for r in res.values()), default=-1.0) if err is None else -1.0
    launches = sum(r["launches"] for r in res.values())
    digests = {r: round(r_["param_digest"], 3) for r, r_ in res.items()}
    if world > 1:
        import torch.distributed as dist
        v = torch.tensor([t_local, -t_local, float(launches)], dtype=torch.float64)
        mx = v.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        every = [None] * world
        dist.all_gather_object(every, digests)
        digests = {k: x for part in every for k, x in part.items()}
        sm = torch.tensor([float(launches)], dtype=torch.float64)
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        launches = int(sm.item())
        if err is None and -mx[1].item() < 0:
            err = RuntimeError("a training rank of another process failed")
        t_local = mx[0].item()
    if err is not None:
        raise err
    if grank != 0:
        return None
    t = t_local / 1e3
    desc, precision, unit = TRAIN_MODELS[model]
    if cfg["stamps"]:
        path = args.stamps if args.train_only else os.path.splitext(args.stamps)[0] + "_train.json"
        with open(path, "w") as f:
            json.dump({"n": n, "model": model, "train": {r: v["stamps"] for r, v in res.items()}}, f)
    r0 = res[min(res)]
    out = {unit: n * args.batch * args.train_steps / t, "instances": n, "batch_per_instance":
           args.batch, "ms_per_step": t * 1e3 / args.train_steps, "steps": args.train_steps,
           "warmup": args.train_warmup, "instance_mode": args.train_mode,
           "precision": (precision.replace("(fp32 SHM allreduce)",
                                           "(bf16 SHM allreduce of the fp32 buckets)")
                         if args.compress else precision),
           "replicas_agree": len(set(digests.values())) == 1, "loss": r0["loss"],
           "host": {"enqueue_ms_per_step": max(r["host_enqueue_ms"] for r in res.values())
                    / args.train_steps,
                    "hook_ms_per_step": max(r["hook_host_ms"] for r in res.values())
                    / args.train_steps,
                    "hooks_per_step": r0["hook_calls"] / args.train_steps,
                    "phase_ms_per_step_rank0": {k: v / args.train_steps for k, v in
                                                r0["host_phase_ms"].items()},
                    "what": "host time to enqueue the timed steps (max over this process's "
                            "ranks; loss.item() syncs once per step only in the last one) and "
                            "the part spent inside flexshm_hook's collective calls"},
           "gpu_launches": launches, "model": desc, "bucket_mb": cfg["bucket_mb"],
           "optimizer": ("AdamW" if model == "bert" else
                         "SGD(momentum 0.9) fused into the allreduce (fmx_allreduce_sgd)"
                         if args.fused_sgd and engine == "graph" and not no_sync else
                         "torch.optim.SGD(momentum 0.9) after the exchange"),
           "engine": ("ddp.ShmDataParallel: whole step (fwd, bwd with bucket allreduces, "
                      "optimizer) replayed as one CUDA graph" if engine == "graph" else
                      "torch DDP + ddp.flexshm_hook, eager")}
    if world > 1:
        out["n_gpus"] = world
        out["scaling"] = "weak"
        if os.environ.get("FMX_DEVICE_MAP"):
            out["logical_gpus"] = (f"{world} LOGICAL GPUs (FMX_DEVICE_MAP="
                                   f"{os.environ['FMX_DEVICE_MAP']}): all instances share the "
                                   "physical devices listed - not a scaling number")
    return out


def dry_exchange(d, mine: list[int], job_key: str, m: int = 4099) -> dict[int, int]:
    """--dry-run data path without CUDA: this process's instance ranks, one
    thread each, join the job's FMX_TRANSPORT_HOST communicator (the real SHM
    bootstrap, peer table and MIG-aware checks, across every torchrun process),
    each writes m seeded fp32 values into its registered host region, and after
    a barrier reads every rank's region and sums them in rank order.  Returns
    rank -> crc32 of that sum; all ranks of all processes must agree."""
    import threading
    import zlib

    import numpy as np

    from paper_2511_09143_b200.comm import init_process_group
    from paper_2511_09143_b200.commsim import PeerInfo

    n = len(d.instances)
    host = zlib.crc32(os.uname().nodename.encode())
    out, errs = {}, []

    def one(r):
        try:
            g, i = d.instances[r]
            peer = PeerInfo(r, f"{0x1B + g:02X}:00:00.0", f"MIG-dry-{g}-{i}", host, os.getpid())
            comm = init_process_group(None, r, job_key + "-dry", peer=peer, nranks=n,
                                      transport="host", host_bytes=4 * m, timeout_s=120)
            x = np.random.default_rng(1000 + r).standard_normal(m).astype(np.float32)
            comm.host_buffer()[:4 * m].numpy()[:] = x.view(np.uint8)
            comm.barrier(120)
            acc = np.zeros(m, np.float32)
            for q in range(n):
                acc = acc + comm.host_buffer(q)[:4 * m].numpy().view(np.float32)
            comm.barrier(120)  # nobody leaves while a peer still reads its region
            out[r] = zlib.crc32(acc.tobytes())
            comm.destroy()
        except BaseException as exc:  # noqa: BLE001
            errs.append((r, exc))

    ths = [threading.Thread(target=one, args=(r,)) for r in mine]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if errs:
        raise RuntimeError(f"dry-run rank {errs[0][0]} failed: {errs[0][1]!r}") from errs[0][1]
    return out


def run_ours(args) -> dict | None:
    import torch

    grank, world, local = dist_env()
    gpus = args.gpus if world == 1 else world
    if world > 1:
        import torch.distributed as dist
        if not dist.is_initialized():
            dist.init_process_group("gloo")
    d = decision_for(gpus, args.ranks_per_gpu)
    n = len(d.instances)
    cfg = {"instances": d.instances, "profiles": d.profiles, "transport": args.transport,
           "slice_bytes": args.slice_bytes, "dtype": args.dtype, "count": args.count,
           "warmup": args.warmup, "steps": args.steps, "e2e": not args.no_e2e,
           "timeline": args.timeline, "stamps": bool(args.stamps), "load": args.load,
           "buckets": args.buckets, "bucket_join": not args.bucket_serial}
    # one job key for all processes of all GPUs
    job_key = os.environ.get("FMX_BENCH_KEY") or f"bench-{os.environ.get('MASTER_PORT', '0')}-" \
        f"{os.environ.get('TORCHELASTIC_RUN_ID', str(os.getppid()))}"
    if world > 1:
        import torch.distributed as dist
        obj = [job_key if grank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        job_key = obj[0]
    my_gpu = grank if world > 1 else 0
    mine = [r for r, (g, _) in enumerate(d.instances) if g == my_gpu] if world > 1 else list(range(n))
    gpu_local = local if world > 1 and not os.environ.get("FMX_ONE_GPU_VISIBLE") else 0
    if os.environ.get("FMX_DEVICE_MAP"):
        # e.g. "0,0": run the N>1 orchestration with several logical GPUs on one device
        gpu_local = int(os.environ["FMX_DEVICE_MAP"].split(",")[local])
    inst_mode = args.mode
    sampler = ClockSampler() if not args.dry_run else None
    results = {}
    errors = []

    if args.dry_run:
        # no CUDA: every instance rank joins ONE host-transport communicator across
        # all torchrun processes and exchanges data through the registered host
        # regions of the shared segment (dry_exchange); stub timings, distinct and
        # known, so the MAX-over-ranks reduction is checkable
        digests_dry = dry_exchange(d, mine, job_key)
        results = {r: {"rank": r, "ms_total": 10.0 * (r + 1), "launches": 1, "kernel_ms": 0.0,
                       "kernel_count": 0, "ms_total_e2e": 5.0 * (r + 1),
                       "ms_total_e2e_dev": 6.0 * (r + 1), "e2e_digest": digests_dry[r],
                       "job_key": job_key}
                   for r in mine}
    else:
        try:
            results = run_ranks(rank_body, _spawned_rank, mine, job_key, n, cfg, inst_mode,
                                gpu_local, sampler)
        except BaseException as exc:  # noqa: BLE001
            errors.append((mine[0], exc))
    clocks = sampler.stop() if sampler is not None else {"sm_mhz": None, "sm_max_mhz": None,
                                                          "reasons": ["dry run"]}
    if errors:
        raise RuntimeError(f"rank {errors[0][0]} failed: {errors[0][1]!r}") from errors[0][1]
    if args.stamps and results:
        with open(args.stamps, "w") as f:
            json.dump({"n": n, "slots": int(os.environ.get("FMX_SLOTS", "2")),
                       "lanes": int(os.environ.get("FMX_LANES", "3")),
                       "device": {r: v.get("stamps_device", []) for r, v in results.items()},
                       "host": {r: v.get("stamps_host", []) for r, v in results.items()}}, f)
    local_max = max(r["ms_total"] for r in results.values())
    local_max_e2e = max(r.get("ms_total_e2e", 0.0) for r in results.values())
    local_max_e2e_dev = max(r.get("ms_total_e2e_dev", 0.0) for r in results.values())
    launches = sum(r["launches"] for r in results.values())
    kernel_ms = sum(r.get("kernel_ms", 0.0) for r in results.values())
    kernel_count = sum(r.get("kernel_count", 0) for r in results.values())
    digests = {r.get("e2e_digest") for r in results.values()}
    if world > 1:
        import torch.distributed as dist
        every = [None] * world
        dist.all_gather_object(every, {r: v.get("e2e_digest") for r, v in results.items()})
        all_digests = {k: v for part in every for k, v in part.items()}
        digests = set(all_digests.values())
        t = torch.tensor([local_max, local_max_e2e, float(launches), kernel_ms, float(kernel_count),
                          local_max_e2e_dev], dtype=torch.float64)
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        local_max, local_max_e2e, local_max_e2e_dev = mx[0].item(), mx[1].item(), mx[5].item()
        launches, kernel_ms, kernel_count = int(sm[2].item()), sm[3].item(), int(sm[4].item())
        if grank != 0:
            return None
    esz = 4 if args.dtype == "f32" else 2
    s_bytes = args.count * esz
    t_step = local_max / 1e3 / args.steps
    per_gpu = [sum(1 for g, _ in d.instances if g == gg) for gg in range(gpus)]
    per_phys = physical_split(d, gpus)
    peaks = dict(LINK_PEAK_FALLBACK)
    if not args.dry_run:
        peaks.update(dram=host_dram_gbs(), dram_source="host copy measured in this run, all "
                                                       "threads, read+write bytes")
    line = {
        "metric": "SHM allreduce GB/s vs host-link peak; ResNet-50 img/s on 1g slices",
        # whole-job aggregate: every rank's S-byte gradient is one unit of work
        # (weak scaling: S per rank is fixed as ranks / GPUs grow); algbw = S / T
        "value": n * s_bytes / t_step / 1e9,
        "unit": UNIT,
        "algbw_gbs": s_bytes / t_step / 1e9,
        "n_gpus": gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "float32" if args.dtype == "f32" else "bfloat16",
        "data": "synthetic (seeded N(0,1)*1e-3 gradient per rank); op = DDP mean: each "
                "contribution x fl32(1/n) (what the default hook's bucket.div_(n) computes "
                "on CUDA), then the rank-order fp32 sum",
        "config": {"workload": f"{workload_name(args.count, args.dtype)} allreduce across "
                               f"{args.ranks_per_gpu} 1g instances per B200 x {gpus}"
                               + (" (BASELINE configs[1] comm step)"
                                  if args.count == RESNET50_PARAMS and gpus == 1 else ""),
                   "ranks": n, "ranks_per_gpu": per_gpu, "bytes": s_bytes,
                   "instance_mode": inst_mode,
                   "transport": args.transport,
                   "l2": (f"inputs {max(per_phys)} x {s_bytes / 1e6:.1f} MB per GPU "
                          + ("> L2 (126 MB): no flush needed"
                             if max(per_phys) * s_bytes > 126e6 else
                             "< L2 (126 MB), not flushed: every byte crosses the host link, "
                             "which bounds the path")),
                   "slots": int(os.environ.get("FMX_SLOTS", "2")),
                   "lanes": int(os.environ.get("FMX_LANES", "3")),
                   "rank_order": "fm_select round-robin"},
        "busbw_gbs": s_bytes / t_step / 1e9 * 2 * (n - 1) / n,
        "roofline": kernel_roofline(args, n, s_bytes, kernel_ms, kernel_count,
                                    results.get(0, {}).get("iso_kernel_us"),
                                    results.get(0, {}).get("iso_piece_bytes")),
        "step_roofline": step_roofline(n, per_phys, s_bytes, t_step, peaks),
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if args.dry_run:
        line["dry_exchange"] = {
            "ranks": len(all_digests) if world > 1 else len(results), "agree": len(digests) == 1,
            "what": "no CUDA: every instance rank (threads of its GPU's torchrun process) joined "
                    "one FMX_TRANSPORT_HOST communicator, wrote seeded fp32 values into its "
                    "registered host region of the shared segment and rank-order summed every "
                    "rank's region after a barrier; crc32 of the sums agree across processes"}
    if getattr(args, "mps_fallback", None):
        line["config"]["mps_fallback"] = args.mps_fallback
    if os.environ.get("FMX_DEVICE_MAP"):
        line["config"]["logical_gpus"] = (
            f"{gpus} LOGICAL GPUs on {len(per_phys)} physical B200 (FMX_DEVICE_MAP="
            f"{os.environ['FMX_DEVICE_MAP']}, synthetic bus ids FMX_FAKE_BUS): the communicator, "
            "rank order and bootstrap are the multi-GPU ones, but all host-link traffic shares "
            "one PCIe link - not a multi-GPU scaling number")
    if not args.no_e2e:
        t_e2e = local_max_e2e / 1e3 / args.steps
        t_dev = local_max_e2e_dev / 1e3 / args.steps
        line["e2e"] = {"value": n * s_bytes / t_e2e / 1e9, "unit": line["unit"],
                       "algbw_gbs": s_bytes / t_e2e / 1e9,
                       "ms_per_step": t_e2e * 1e3,
                       "api": "ShmCommunicator.allreduce_host -> fmx_allreduce_host (C ABI): "
                              "every rank's gradient in its registered pinned host buffer; the "
                              "GPUs read the inputs (H2D) and write the results (D2H) in the "
                              "timed region",
                       "h2d_bytes_per_step": n * s_bytes, "d2h_bytes_per_step": n * s_bytes,
                       "ranks_agree": len(digests) == 1}
        # host path roofline: k*S each way per GPU, T* = max(one-way, bidirectional);
        # the host-DRAM estimate is reported beside it (see step_roofline)
        k_max = max(per_phys)
        t_link = max(k_max * s_bytes / (peaks["h2d"] * 1e9), k_max * s_bytes / (peaks["d2h"] * 1e9),
                     2 * k_max * s_bytes / (peaks["bidir"] * 1e9))
        t_dram = 2 * n * s_bytes / (peaks.get("dram", HOST_DRAM_FALLBACK) * 1e9)
        line["e2e"]["step_roofline"] = {"bound": "host_link", "t_star_ms": t_link * 1e3,
                                        "frac": t_link / t_e2e,
                                        "host_dram_t_ms_cpu_copy_estimate": t_dram * 1e3}
        line["e2e_device_buffers"] = {
            "value": n * s_bytes / t_dev / 1e9, "unit": line["unit"], "ms_per_step": t_dev * 1e3,
            "api": "pinned host -> device copy, ShmCommunicator.allreduce, device -> pinned host",
            "h2d_bytes_per_step": n * s_bytes, "d2h_bytes_per_step": n * s_bytes}
    return line


def run_nccl_point(args, transport: str = "nvlink") -> dict:
    """Comparison point (north_star): stock NCCL allreduce of the same gradient
    bytes, one rank per GPU (the torchrun ranks), CUDA events, max over ranks;
    transport "nvlink" (NCCL's default P2P / NVLS over NVSwitch) or "shm"
    (P2P and NVLS off: NCCL's host shared-memory transport, the stock
    equivalent of this repo's path).  Not the product path; never raises into
    the bench line."""
    import torch
    import torch.distributed as dist
    if transport == "shm":
        os.environ.update(NCCL_P2P_DISABLE="1", NCCL_NVLS_ENABLE="0", NCCL_SHM_DISABLE="0",
                          NCCL_IB_DISABLE="1")
    try:
        local = int(os.environ.get("LOCAL_RANK", "0"))
        dev = torch.device("cuda", local)
        torch.cuda.set_device(dev)
        pg = dist.new_group(backend="nccl")
        x = torch.randn(args.count, device=dev)
        for _ in range(3):
            dist.all_reduce(x, group=pg)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            dist.all_reduce(x, group=pg)
        e1.record()
        e1.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        n = dist.get_world_size()
        s_bytes = args.count * 4
        dist.destroy_process_group(pg)
        return {"ms_per_step": ms, "algbw_gbs": s_bytes / ms / 1e6,
                "busbw_gbs": s_bytes / ms / 1e6 * 2 * (n - 1) / n, "ranks": n,
                "transport": transport,
                "note": f"stock NCCL ({'NVLink/NVSwitch' if transport == 'nvlink' else 'SHM: '
                                      'NCCL_P2P_DISABLE=1 NCCL_NVLS_ENABLE=0'}), one rank per "
                        "GPU (this process is also an instance's MPS client, so NCCL runs on "
                        "its SM share)"}
    except Exception as exc:  # noqa: BLE001
        return {"error": repr(exc)[:300]}


def run_cpu_reference(count: int, n: int, dtype: str, steps: int, warmup: int,
                      seconds: float | None = None, extras: bool = True) -> dict:
    """The CPU reference path of BASELINE.md §3, timed on this box's cores:
    oracle/shm_cpu_allreduce.c - one process per rank, each pinned to its own
    host core, a real /dev/shm segment, the same reduce-scatter / all-gather
    and rank-order fp32 sum (DDP mean), bit-identical to the GPU path.  At
    least `steps` timed allreduces, more up to ~`seconds` of work.  With
    `extras`, two more CPU figures on the same workload: the single-process
    threaded port of the same algorithm (oracle ShmAllreduce, all threads)
    and the in-place host-reduction bound (all buffers in one address space,
    rank-order sum written back, no staging: n*S read + n*S written)."""
    from oracle import oracle as orc
    dt = orc.F32 if dtype == "f32" else orc.BF16
    esz = 4 if dtype == "f32" else 2
    cores = orc.host_cores()
    op, factor = orc.ddp_mean(n)
    probe, _ = orc.mp_shm_allreduce(n, count, dt, op, factor, iters=1, warmup=max(warmup, 1),
                                    cores=cores)
    k = max(steps, min(500, int((seconds or 0) * 1e3 / max(probe["ms_per_step"], 1e-3))))
    st, _ = orc.mp_shm_allreduce(n, count, dt, op, factor, iters=k, warmup=max(warmup, 1),
                                 cores=cores)
    t = st["ms_per_step"] / 1e3
    out = {"value": n * count * esz / t / 1e9, "algbw_gbs": count * esz / t / 1e9,
           "ms_per_step": t * 1e3, "iters": k, "cores": st["cores"], "processes": n,
           "oversubscribed": st["oversubscribed"], "host_cpus": len(cores),
           "kind": "port",
           "sample": f"full workload: {n} rank processes x {count} {dtype}, one per host core "
                     f"({st['cores']} of {len(cores)} cores"
                     f"{', OVERSUBSCRIBED' if st['oversubscribed'] else ''}), POSIX SHM "
                     f"reduce-scatter/all-gather, {k} timed allreduces "
                     "(oracle/shm_cpu_allreduce.c)"}
    if extras:
        nthreads = len(cores)
        bufs = [orc.synthetic_gradient(r, count, dt) for r in range(n)]
        shm = orc.ShmAllreduce(n, count, dt, nthreads)
        shm(bufs, op, factor)
        reps = max(3, min(20, k // 4))
        t0 = time.perf_counter()
        for _ in range(reps):
            shm(bufs, op, factor)
        tp = (time.perf_counter() - t0) / reps
        out["threaded_port"] = {"ms_per_step": tp * 1e3, "value": n * count * esz / tp / 1e9,
                                "threads": nthreads,
                                "what": "one process, n rank buffers, same staging RS/AG "
                                        "(oracle ShmAllreduce)"}
        orc.inplace_allreduce(bufs, dt, op, factor, nthreads)
        t0 = time.perf_counter()
        for _ in range(reps):
            orc.inplace_allreduce(bufs, dt, op, factor, nthreads)
        ti = (time.perf_counter() - t0) / reps
        out["inplace_bound"] = {"ms_per_step": ti * 1e3, "value": n * count * esz / ti / 1e9,
                                "threads": nthreads,
                                "what": "in-place rank-order reduction of the n host buffers in "
                                        "one address space (no staging; 2 n S bytes of host "
                                        "memory traffic): the host's own floor for host-resident "
                                        "gradients, to read the GPU e2e against"}
    return out


def main(argv=None):
    args = parse_args(argv)
    grank, world, _ = dist_env()
    n = (args.gpus if world == 1 else world) * args.ranks_per_gpu
    unit = UNIT
    if args.impl == "reference":
        if grank != 0:
            return 0
        # bounded sample: at least --steps allreduces, at most ~20 s of work
        r = run_cpu_reference(args.count, n, args.dtype, args.steps, args.warmup, seconds=20.0)
        sample = r["sample"]
        line = {"impl": "reference", "metric": "SHM allreduce GB/s vs host-link peak; ResNet-50 "
                "img/s on 1g slices", "value": r["value"], "unit": unit,
                "n_gpus": args.gpus if world == 1 else world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None,
                "dtype": "float32" if args.dtype == "f32" else "bfloat16", "data": "synthetic",
                "config": {"workload": f"{workload_name(args.count, args.dtype)} allreduce "
                                       f"across {n} ranks", "ranks": n},
                "cpu_baseline": {"value": r["value"], "unit": unit, "cores": r["cores"],
                                 "kind": "port", "sample": sample,
                                 "threaded_port": r.get("threaded_port"),
                                 "inplace_bound": r.get("inplace_bound")},
                "e2e": {"value": r["value"], "unit": unit, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0},
                "note": "the reference has no runnable allreduce (its data path is NCCL, "
                        "PAPER.md:353-354, 830); this arm is BASELINE.md §3's CPU reference "
                        "path: one process per rank pinned to its own core, POSIX SHM "
                        "reduce-scatter/all-gather, rank-order fp32 sum "
                        "(oracle/shm_cpu_allreduce.c), bit-identical to the GPU path"}
        print(json.dumps(line))
        return 0
    mps = start_mps(args, world)
    if args.nccl and args.nccl_shm:
        raise SystemExit("--nccl and --nccl-shm are separate runs (NCCL caches its env per process)")
    if world > 1 and not args.dry_run and not (args.nccl or args.nccl_shm) and \
            not os.environ.get("FMX_DEVICE_MAP"):
        # one GPU per torchrun process and its instance processes (they inherit
        # the variable): no peer device is even visible, so P2P / NVLink cannot
        # be used - the transport is what MIG allows.  After the
        # MPS daemon started (it must see every GPU); --nccl keeps every GPU
        # visible for the NVLink comparison point.
        os.environ["CUDA_VISIBLE_DEVICES"] = os.environ.get("LOCAL_RANK", "0")
        os.environ["FMX_ONE_GPU_VISIBLE"] = "1"
    try:
        return _main(args, world, n, unit)
    finally:
        stop_mps(mps, world)
        if world > 1:
            import torch.distributed as dist
            if dist.is_initialized():
                dist.destroy_process_group()


def _local_rank0() -> bool:
    return int(os.environ.get("LOCAL_RANK", "0")) == 0


def start_mps(args, world):
    """Instances are MPS clients by default (concurrent, 1g SM share each:
    the closest stand-in for MIG slices on a box without MIG).  One private
    MPS control daemon per node, started by local rank 0 (all torchrun ranks
    of the node share it).  If it cannot start, every rank falls back to
    green-context instances and says so in the JSON line."""
    # --train-only runs only the training leg: its instance mode alone decides
    # (a `full` one-to-one run must not become a capped MPS client)
    wants = args.train_mode == "mps" if args.train_only else \
        args.mode == "mps" or (not args.no_train and args.train_mode == "mps")
    if not wants:
        return None
    from paper_2511_09143_b200.launcher import MPS_PERCENT, MpsDaemon
    tag = f"bench-{os.environ.get('MASTER_PORT', os.getpid())}"
    mps = MpsDaemon(tag)
    ok = mps.start() if _local_rank0() else True
    if world > 1:
        import torch
        import torch.distributed as dist
        if not dist.is_initialized():
            dist.init_process_group("gloo")
        flag = torch.tensor([1 if ok else 0])
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        ok = bool(flag.item())
    if not ok:
        args.mps_fallback = "MPS daemon failed to start: green-context instances instead"
        if args.mode == "mps":
            args.mode = "green"
        if args.train_mode == "mps":
            args.train_mode = "green"
        return mps if _local_rank0() else None
    os.environ.update(mps.env)
    os.environ["CUDA_MPS_ACTIVE_THREAD_PERCENTAGE"] = str(MPS_PERCENT)
    return mps


def stop_mps(mps, world):
    """Every rank meets here (N>1) before local rank 0 asks the daemon to quit."""
    if world > 1:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.barrier()
    if mps is not None and _local_rank0():
        mps.stop()


def _main(args, world, n, unit):
    if args.sweep:
        lines = run_sweep(args)
        for ln in lines:
            print(json.dumps(ln))
        if args.out:
            with open(args.out, "w") as f:
                f.writelines(json.dumps(ln) + "\n" for ln in lines)
        return 0
    if args.train_only:
        d = decision_for(args.gpus if world == 1 else world, args.ranks_per_gpu)
        tr = run_train(args, d, f"train-{os.getpid()}", args.train_model)
        ns = None
        if args.train_no_sync:
            # same instances, same step, gradients NOT synchronised: the compute-only bound
            ns = run_train(args, d, f"train-ns-{os.getpid()}", args.train_model, no_sync=True)
        if tr is None:       # torchrun rank != 0
            return 0
        line = {args.train_model: tr}
        if ns is not None:
            line[args.train_model]["no_sync"] = ns
        print(json.dumps(line))
        if args.out:
            with open(args.out, "w") as f:
                f.write(json.dumps(line) + "\n")
        return 0
    line = run_ours(args)
    if world > 1 and not args.dry_run and (args.nccl or args.nccl_shm):
        tr = "shm" if args.nccl_shm else "nvlink"
        nccl = run_nccl_point(args, tr)      # collective: every torchrun rank takes part
        if line is not None:
            line[f"nccl_{tr}"] = nccl
    train = None
    if not args.no_train and not args.dry_run and (world > 1 or args.gpus == 1):
        # every torchrun process takes part (its GPU's instance ranks); rank 0 reports
        d = decision_for(world if world > 1 else 1, args.ranks_per_gpu)
        try:
            train = run_train(args, d, f"train-{os.getpid()}")
        except Exception as exc:  # noqa: BLE001 - report, keep the allreduce line
            train = {"error": repr(exc)[:300]}
    if line is None:
        return 0
    if train is not None:
        line["resnet50"] = train
    if not args.no_cpu_baseline:
        r = run_cpu_reference(args.count, n, args.dtype, 3, 1, seconds=args.cpu_seconds)
        line["cpu_baseline"] = {"value": r["value"], "unit": line["unit"], "cores": r["cores"],
                                "kind": "port", "sample": r["sample"],
                                "ms_per_step": r["ms_per_step"],
                                "threaded_port": r.get("threaded_port"),
                                "inplace_bound": r.get("inplace_bound")}
    print(json.dumps(line))
    if args.out:
        with open(args.out, "w") as f:
            f.write(json.dumps(line) + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
