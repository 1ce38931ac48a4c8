"""Generate tests/golden/control_golden.json by running the REFERENCE
implementation (/root/reference/pkg/src/migsim, imported read-only in the
build container) on seeded random cases of the control half of the path:
fm_select / schedule_step (rank order), PeerInfo validation, discover_peers,
build_topology, restore_bus_id, estimate_jct and the bootstrap-check CLI.

Run:  python tests/golden/make_golden_control.py
The fixture is committed; tests read it on any box (the reference tree is not
needed at test time).
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import random
import sys
import tempfile

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from migsim import cli as ref_cli  # noqa: E402
from migsim import commsim as ref_comm  # noqa: E402
from migsim.scheduler import Policy, fm_select, make_cluster, schedule_step  # noqa: E402
from migsim.simcore import PerfModel, estimate_jct  # noqa: E402
from migsim.scheduler import AllocationDecision  # noqa: E402
from migsim.workload import Job  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "control_golden.json")


def err_record(exc):
    rec = {"error": type(exc).__name__}
    if hasattr(exc, "rank_a"):
        rec["rank_a"], rec["rank_b"] = exc.rank_a, exc.rank_b
    return rec


def fm_cases(rng):
    cases = []
    for g in range(1, 9):
        for _ in range(40):
            cluster = make_cluster("FM", g)
            p = rng.choice([0.0, 0.0, 0.2, 0.5, 0.8])
            busy = []
            for lay in cluster.gpus:
                for inst in lay.instances.values():
                    if rng.random() < p:
                        inst.job_id = 900
                        busy.append([lay.gpu_id, inst.instance_id])
            reconf = []
            if g > 1 and rng.random() < 0.15:
                gid = rng.randrange(g)
                cluster.reconfiguring[gid] = 1.0
                reconf.append(gid)
            size = rng.randint(1, 7 * g + 2)
            d = fm_select(Job(7, "train", size, 1.0, 0.0), cluster)
            cases.append({"gpus": g, "busy": busy, "reconfiguring": reconf, "size": size,
                          "decision": None if d is None else {
                              "job_id": d.job_id, "instances": d.instances,
                              "transport": d.transport_class, "profiles": d.profiles}})
    # the BASELINE configs' rank orders
    for g, size in ((1, 2), (1, 7), (2, 4), (2, 14), (4, 14), (8, 14), (4, 28), (8, 56)):
        d = fm_select(Job(0, "train", size, 1.0, 0.0), make_cluster("FM", g))
        cases.append({"gpus": g, "busy": [], "reconfiguring": [], "size": size,
                      "decision": {"job_id": 0, "instances": d.instances,
                                   "transport": d.transport_class, "profiles": d.profiles}})
    return cases


def queue_cases(rng):
    cases = []
    for _ in range(60):
        g = rng.randint(1, 4)
        cluster = make_cluster("FM", g)
        njobs = rng.randint(1, 20)
        jobs = {i: Job(i, "train", rng.randint(1, 7 * g), 1.0, 0.0) for i in range(njobs)}
        cluster.wait_queue = list(range(njobs))
        kind = rng.choice(["fifo", "backfill"])
        depth = rng.randint(1, 16)
        res = schedule_step(cluster, jobs, Policy(kind, depth))
        cases.append({"gpus": g, "sizes": [jobs[i].size for i in range(njobs)], "policy": kind,
                      "depth": depth,
                      "dispatched": [{"job_id": d.job_id, "instances": d.instances,
                                      "profiles": d.profiles} for d in res.started],
                      "examined": res.examined, "queue_after": cluster.wait_queue})
    return cases


BUSES = ["00:4B:00.0", "00:65:00.0", "00:C0:00.0", "1a:00:00.0"]


def peer_cases(rng):
    cases = []
    for _ in range(400):
        n = rng.randint(1, 16)
        ranks = list(range(n))
        corrupt = rng.random()
        if corrupt < 0.05 and n > 1:
            ranks[rng.randrange(n)] = ranks[rng.randrange(n)]       # duplicate rank
        elif corrupt < 0.1:
            ranks[rng.randrange(n)] = n + rng.randint(0, 3)          # gap
        rng.shuffle(ranks)
        nbus = rng.randint(1, 3)
        peers = []
        for r in ranks:
            bus = rng.choice(BUSES[:nbus])
            mig = f"MIG-{rng.randint(0, 3 * n)}" if rng.random() < 0.3 else f"MIG-u-{r}-{rng.random()}"
            peers.append({"rank": r, "pcie_bus_id": bus, "mig_id": mig,
                          "host_hash": rng.choice([1, 1, 1, 2]), "pid_hash": 1000 + r})
        mig_aware = rng.random() < 0.6
        objs = [ref_comm.PeerInfo(**p) for p in peers]
        rec = {"peers": peers, "mig_aware": mig_aware}
        try:
            comm = ref_comm.discover_peers(objs, mig_aware=mig_aware)
            rec["discover"] = {"ranks": [p.rank for p in comm.peers]}
            try:
                topo = ref_comm.build_topology(comm)
                rec["topology"] = {"labels": [[nd.label, nd.canonical, nd.rank] for nd in topo.nodes],
                                   "mig_list": topo.mig_list}
            except Exception as exc:  # noqa: BLE001
                rec["topology"] = err_record(exc)
        except Exception as exc:  # noqa: BLE001
            rec["discover"] = err_record(exc)
        cases.append(rec)
    # > 10 ranks on one bus: topology must fail, discovery must not
    peers = [{"rank": r, "pcie_bus_id": "00:4B:00.0", "mig_id": f"m{r}", "host_hash": 1,
              "pid_hash": r} for r in range(12)]
    objs = [ref_comm.PeerInfo(**p) for p in peers]
    rec = {"peers": peers, "mig_aware": True,
           "discover": {"ranks": [p.rank for p in ref_comm.discover_peers(objs).peers]}}
    try:
        ref_comm.build_topology(objs)
    except Exception as exc:  # noqa: BLE001
        rec["topology"] = err_record(exc)
    cases.append(rec)
    return cases


def peerinfo_cases():
    out = []
    for bus in ["00:4B:00.0", "00:4b:00.0", "00:4B:00.3", "0000:4B:00.0", "4B:00.0", "00:4G:00.0",
                "00:4B:00.0\n", "00:4b:00.0 ", "", "zz:zz:zz.0", "AB:CD:EF.0", "ab:cd:ef.0"]:
        for mig in ["MIG-x", ""]:
            try:
                p = ref_comm.PeerInfo(0, bus, mig, 1, 1)
                out.append({"bus": bus, "mig": mig, "ok": p.pcie_bus_id})
            except Exception as exc:  # noqa: BLE001
                out.append({"bus": bus, "mig": mig, **err_record(exc)})
    return out


def restore_cases(rng):
    labels = ["00:4B:00.2", "00:4B:00.0", "00:4b:00.9", "garbage", "00:4B:00", "00:4B:00.A",
              "0:4B:00.0", "", "00:4B:00.2\n", "00:4B:00.22"]
    for _ in range(100):
        labels.append(f"{rng.randrange(256):02X}:{rng.randrange(256):02x}:{rng.randrange(256):02X}"
                      f".{rng.randrange(10)}")
    out = []
    for lab in labels:
        try:
            out.append({"label": lab, "ok": ref_comm.restore_bus_id(lab)})
        except Exception as exc:  # noqa: BLE001
            out.append({"label": lab, **err_record(exc)})
    return out


def transport_cases(rng):
    out = []
    for _ in range(50):
        a = {"rank": 0, "pcie_bus_id": rng.choice(BUSES), "mig_id": "a",
             "host_hash": rng.randint(1, 3), "pid_hash": 1}
        b = {"rank": 1, "pcie_bus_id": rng.choice(BUSES), "mig_id": "b",
             "host_hash": rng.randint(1, 3), "pid_hash": 2}
        out.append({"a": a, "b": b, "transport": ref_comm.select_transport(
            ref_comm.PeerInfo(**a), ref_comm.PeerInfo(**b))})
    return out


def jct_cases(rng):
    out = []
    for _ in range(80):
        g = rng.randint(1, 4)
        n = rng.randint(1, 6)
        inst = [[rng.randrange(g + (1 if rng.random() < 0.05 else 0)), rng.randint(1, 7)]
                for _ in range(n)]
        profiles = [rng.choice(["1g.5gb", "1g.10gb"]) for _ in range(n)]
        if rng.random() < 0.05:
            profiles = profiles[:-1]
        size = rng.randint(1, 6)
        model = {"speedup_1g10": rng.choice([0.8, 0.9]), "multi_overhead": rng.choice([1.0, 1.07, 1.2]),
                 "placement_penalty_slope": 0.03, "placement_penalty_cap": 1.15,
                 "contention_factor": 1.06, "net_transport_factor": rng.choice([1.0, 1.5])}
        job = Job(3, "train", size, 1000.0, 0.0)
        d = AllocationDecision(3, [tuple(x) for x in inst], "SHM", profiles)
        rec = {"gpus": g, "size": size, "instances": inst, "profiles": profiles, "model": model}
        try:
            rec["jct"] = estimate_jct(job, d, PerfModel(**model), num_gpus=g)
        except Exception as exc:  # noqa: BLE001
            rec.update(err_record(exc))
        out.append(rec)
    return out


def cli_cases():
    files = {
        "seven_on_one_bus": [{"rank": r, "pcie_bus_id": "00:4B:00.0", "mig_id": f"MIG-{r}",
                              "host_hash": 1, "pid_hash": 100 + r} for r in range(7)],
        "two_buses": [{"rank": r, "pcie_bus_id": "00:4B:00.0" if r % 2 else "00:65:00.0",
                       "mig_id": f"MIG-{r}", "host_hash": 1, "pid_hash": r} for r in range(6)],
        "double_binding": [{"rank": r, "pcie_bus_id": "00:4B:00.0", "mig_id": "MIG-same",
                            "host_hash": 1, "pid_hash": r} for r in range(2)],
        "bad_bus": [{"rank": 0, "pcie_bus_id": "0000:4B:00.0", "mig_id": "m", "host_hash": 1,
                     "pid_hash": 1}],
        "empty_mig": [{"rank": 0, "pcie_bus_id": "00:4B:00.0", "mig_id": "", "host_hash": 1,
                       "pid_hash": 1}],
        "eleven": [{"rank": r, "pcie_bus_id": "00:4B:00.0", "mig_id": f"m{r}", "host_hash": 1,
                    "pid_hash": r} for r in range(11)],
    }
    out = []
    with tempfile.TemporaryDirectory() as d:
        for name, recs in files.items():
            path = os.path.join(d, name + ".jsonl")
            with open(path, "w") as f:
                f.write("\n".join(json.dumps(r) for r in recs) + "\n")
            for legacy in (False, True):
                argv = ["bootstrap-check", "--peers", path] + (["--legacy"] if legacy else [])
                so, se = io.StringIO(), io.StringIO()
                with contextlib.redirect_stdout(so), contextlib.redirect_stderr(se):
                    rc = ref_cli.main(argv)
                out.append({"name": name, "records": recs, "legacy": legacy, "rc": rc,
                            "stdout": so.getvalue(), "stderr": se.getvalue()})
    return out


def main():
    rng = random.Random(20251109)
    doc = {
        "source": "reference migsim (pkg/src/migsim) run by tests/golden/make_golden_control.py",
        "fm_select": fm_cases(rng),
        "schedule_step": queue_cases(rng),
        "discover_topology": peer_cases(rng),
        "peerinfo": peerinfo_cases(),
        "restore_bus_id": restore_cases(rng),
        "select_transport": transport_cases(rng),
        "estimate_jct": jct_cases(rng),
        "bootstrap_check": cli_cases(),
    }
    with open(OUT, "w") as f:
        json.dump(doc, f, separators=(",", ":"), sort_keys=True)
    print(f"wrote {OUT}: " + ", ".join(f"{k}={len(v)}" for k, v in doc.items() if isinstance(v, list)))


if __name__ == "__main__":
    main()
