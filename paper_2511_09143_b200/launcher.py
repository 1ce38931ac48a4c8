"""Local launcher: one process per instance of an AllocationDecision.

Stands in for the paper's Kubernetes Job Executor (reference PAPER.md:362-368,
out of scope as such).  It keeps the paper's per-rank environment contract
(PAPER.md:377-384): rank r gets `LOCAL_RANK`/`RANK` = r, `WORLD_SIZE` = n,
`CUDA_VISIBLE_DEVICES` narrowed to its GPU (or its MIG UUID), plus
`FMX_*` variables naming its instance, so `init_from_env()` in the child binds
the instance and joins the communicator.  Rank r is `decision.instances[r]`,
the fm_select round-robin order (reference scheduler.py:117-136).

`mode="mps"` starts a private MPS control daemon for the job (pipe directory
under /tmp) and caps every client at a 1g share of the SMs
(`CUDA_MPS_ACTIVE_THREAD_PERCENTAGE`), then shuts it down.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import shutil
import subprocess
import time
import traceback
import uuid

from .scheduler import AllocationDecision

MPS_PERCENT = 14  # ~1/7 of the SMs per client


def new_job_key(prefix: str = "job") -> str:
    return f"{prefix}-{os.getpid()}-{uuid.uuid4().hex[:12]}"


def rank_env(decision: AllocationDecision, rank: int, job_key: str, mode: str,
             gpu_map: dict[int, str] | None = None, mig_uuids: dict | None = None) -> dict:
    gpu_id, inst_id = decision.instances[rank]
    profile = decision.profiles[rank] if decision.profiles else "1g.5gb"
    env = {
        "RANK": str(rank), "LOCAL_RANK": str(rank), "WORLD_SIZE": str(len(decision.instances)),
        "FMX_JOB_KEY": job_key, "FMX_GPU_ID": str(gpu_id), "FMX_INSTANCE_ID": str(inst_id),
        "FMX_PROFILE": profile, "FMX_INSTANCE_MODE": mode,
    }
    if mode == "mig" and mig_uuids and (gpu_id, inst_id) in mig_uuids:
        env["CUDA_VISIBLE_DEVICES"] = mig_uuids[(gpu_id, inst_id)]
        env["FMX_MIG_UUID"] = mig_uuids[(gpu_id, inst_id)]
    else:
        env["CUDA_VISIBLE_DEVICES"] = (gpu_map or {}).get(gpu_id, str(gpu_id))
    return env


def init_from_env(**kw):
    """In a launched rank: bind the instance named by FMX_* and join the
    communicator.  Returns (instance, communicator)."""
    from .comm import init_process_group
    from .instance import bind

    rank, n = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    inst = bind(int(os.environ["FMX_GPU_ID"]), int(os.environ["FMX_INSTANCE_ID"]),
                os.environ.get("FMX_PROFILE", "1g.5gb"),
                mode=os.environ.get("FMX_INSTANCE_MODE", "green"),
                sm_count=kw.pop("sm_count", None),
                mig_uuid=os.environ.get("FMX_MIG_UUID"))
    comm = init_process_group(None, rank, os.environ["FMX_JOB_KEY"], instance=inst, nranks=n, **kw)
    return inst, comm


def _child(fn, rank, env, args, q):
    os.environ.update(env)
    try:
        q.put((rank, "ok", fn(rank, *args)))
    except BaseException:  # noqa: BLE001 - report everything to the parent
        q.put((rank, "err", traceback.format_exc()))
        raise SystemExit(1)


class MpsDaemon:
    """Private MPS control daemon for one job (no-op if unavailable)."""

    def __init__(self, tag: str):
        self.dir = f"/tmp/fmx-mps-{tag}"
        self.env = {"CUDA_MPS_PIPE_DIRECTORY": f"{self.dir}/pipe",
                    "CUDA_MPS_LOG_DIRECTORY": f"{self.dir}/log"}
        self.started = False

    def start(self) -> bool:
        exe = shutil.which("nvidia-cuda-mps-control")
        if exe is None:
            return False
        for d in self.env.values():
            os.makedirs(d, exist_ok=True)
        r = subprocess.run([exe, "-d"], env={**os.environ, **self.env}, timeout=30,
                           capture_output=True)
        self.started = r.returncode == 0
        time.sleep(0.5)
        return self.started

    def stop(self) -> None:
        """Ask the daemon to quit.  It exits once its last client does (the
        calling process may itself be a client), so do not wait for it."""
        if self.started:
            p = subprocess.Popen(["nvidia-cuda-mps-control"], stdin=subprocess.PIPE,
                                 stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL,
                                 env={**os.environ, **self.env})
            try:
                p.stdin.write(b"quit\n")
                p.stdin.close()
            except OSError:
                pass
            self.started = False


def launch(fn, decision: AllocationDecision, args: tuple = (), *, job_key: str | None = None,
           mode: str = "green", timeout_s: float = 900.0, gpu_map=None, mig_uuids=None,
           env_extra: dict | None = None, inline_rank0: bool = False) -> list:
    """Run fn(rank, *args) in one spawned process per rank; return the
    results in rank order.  Raises RuntimeError with the first failing
    rank's traceback.  inline_rank0 runs rank 0 in the calling process (its
    GPU must then be the caller's current device; CUDA_VISIBLE_DEVICES of
    the caller is left alone)."""
    job_key = job_key or new_job_key()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mps = None
    extra = dict(env_extra or {})
    if mode == "mps":
        mps = MpsDaemon(job_key)
        if not mps.start():
            raise RuntimeError("mode='mps' requested but the MPS daemon could not start")
        extra.update(mps.env)
        extra["CUDA_MPS_ACTIVE_THREAD_PERCENTAGE"] = str(MPS_PERCENT)
    procs = []
    try:
        first = 1 if inline_rank0 else 0
        for r in range(first, len(decision.instances)):
            env = rank_env(decision, r, job_key, mode, gpu_map, mig_uuids)
            env.update(extra)
            p = ctx.Process(target=_child, args=(fn, r, env, args, q), daemon=False)
            p.start()
            procs.append(p)
        results, errors = {}, []
        if inline_rank0:
            env = rank_env(decision, 0, job_key, mode, gpu_map, mig_uuids)
            env.pop("CUDA_VISIBLE_DEVICES", None)
            env.update({k: v for k, v in extra.items() if k != "CUDA_VISIBLE_DEVICES"})
            os.environ.update(env)
            try:
                results[0] = fn(0, *args)
            except BaseException:  # noqa: BLE001
                errors.append((0, traceback.format_exc()))
        deadline = time.time() + timeout_s
        while not errors and len(results) < len(decision.instances):
            left = deadline - time.time()
            if left <= 0:
                raise RuntimeError(f"launch timed out after {timeout_s}s "
                                   f"({len(results)} of {len(procs)} ranks done)")
            try:
                rank, status, payload = q.get(timeout=min(left, 1.0))
            except Exception:  # queue.Empty
                if any(p.exitcode not in (None, 0) for p in procs) and q.empty():
                    time.sleep(0.5)
                    if q.empty():
                        bad = [i for i, p in enumerate(procs) if p.exitcode not in (None, 0)]
                        raise RuntimeError(f"rank(s) {bad} died without a result") from None
                continue
            if status == "ok":
                results[rank] = payload
            else:
                errors.append((rank, payload))
                break
        if errors:
            rank, tb = errors[0]
            raise RuntimeError(f"rank {rank} failed:\n{tb}")
        for p in procs:
            p.join(timeout=60)
        return [results[r] for r in range(len(decision.instances))]
    finally:
        for p in procs:
            if p.is_alive():
                p.kill()
                p.join(timeout=10)
        if mps is not None:
            mps.stop()
