"""The control half of the path against golden vectors produced by the
REFERENCE itself (tests/golden/make_golden_control.py runs
/root/reference/pkg/src/migsim): rank order from fm_select / schedule_step,
PeerInfo validation, discover_peers, build_topology, restore_bus_id,
select_transport, estimate_jct and the bootstrap-check CLI.  Zero tolerance.
"""

from __future__ import annotations

import contextlib
import io
import json
import os

import pytest

from paper_2511_09143_b200 import cli, commsim
from paper_2511_09143_b200.scheduler import AllocationDecision, Policy, fm_select, make_cluster, schedule_step
from paper_2511_09143_b200.simcore import PerfModel, estimate_jct
from paper_2511_09143_b200.workload import Job

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "control_golden.json")))


def err_record(exc):
    rec = {"error": type(exc).__name__}
    if hasattr(exc, "rank_a"):
        rec["rank_a"], rec["rank_b"] = exc.rank_a, exc.rank_b
    return rec


def as_lists(x):
    return json.loads(json.dumps(x))


def test_fm_select_rank_order_matches_reference():
    assert len(GOLDEN["fm_select"]) > 300
    for case in GOLDEN["fm_select"]:
        cluster = make_cluster("FM", case["gpus"])
        for g, i in case["busy"]:
            cluster.layout(g).instances[i].job_id = 900
        for g in case["reconfiguring"]:
            cluster.reconfiguring[g] = 1.0
        jid = case["decision"]["job_id"] if case["decision"] else 7
        d = fm_select(Job(jid, "train", case["size"], 1.0, 0.0), cluster)
        got = None if d is None else {"job_id": d.job_id, "instances": d.instances,
                                      "transport": d.transport_class, "profiles": d.profiles}
        assert as_lists(got) == case["decision"], case


def test_schedule_step_matches_reference():
    for case in GOLDEN["schedule_step"]:
        cluster = make_cluster("FM", case["gpus"])
        jobs = {i: Job(i, "train", s, 1.0, 0.0) for i, s in enumerate(case["sizes"])}
        cluster.wait_queue = list(range(len(jobs)))
        res = schedule_step(cluster, jobs, Policy(case["policy"], case["depth"]))
        got = [{"job_id": d.job_id, "instances": d.instances, "profiles": d.profiles}
               for d in res.started]
        assert as_lists(got) == case["dispatched"]
        assert res.examined == case["examined"]
        assert cluster.wait_queue == case["queue_after"]


def test_discover_and_topology_match_reference():
    for case in GOLDEN["discover_topology"]:
        peers = [commsim.PeerInfo(**p) for p in case["peers"]]
        try:
            comm = commsim.discover_peers(peers, mig_aware=case["mig_aware"])
            got = {"ranks": [p.rank for p in comm.peers]}
        except Exception as exc:  # noqa: BLE001
            got = err_record(exc)
            comm = None
        assert got == case["discover"], case
        if comm is not None or "topology" in case and "discover" not in case:
            src = comm if comm is not None else peers
            try:
                topo = commsim.build_topology(src)
                tgot = {"labels": [[n.label, n.canonical, n.rank] for n in topo.nodes],
                        "mig_list": as_lists(topo.mig_list)}
            except Exception as exc:  # noqa: BLE001
                tgot = err_record(exc)
            assert tgot == case["topology"], case


def test_more_than_ten_ranks_per_bus_is_malformed():
    case = GOLDEN["discover_topology"][-1]
    peers = [commsim.PeerInfo(**p) for p in case["peers"]]
    with pytest.raises(commsim.MalformedLabelError):
        commsim.build_topology(peers)
    assert case["topology"]["error"] == "MalformedLabelError"


def test_peerinfo_validation_matches_reference():
    for case in GOLDEN["peerinfo"]:
        try:
            got = {"ok": commsim.PeerInfo(0, case["bus"], case["mig"], 1, 1).pcie_bus_id}
        except Exception as exc:  # noqa: BLE001
            got = err_record(exc)
        want = {k: v for k, v in case.items() if k not in ("bus", "mig")}
        assert got == want, case


def test_restore_bus_id_matches_reference():
    for case in GOLDEN["restore_bus_id"]:
        try:
            got = {"ok": commsim.restore_bus_id(case["label"])}
        except Exception as exc:  # noqa: BLE001
            got = err_record(exc)
        assert got == {k: v for k, v in case.items() if k != "label"}, case


def test_select_transport_matches_reference():
    for case in GOLDEN["select_transport"]:
        a, b = commsim.PeerInfo(**case["a"]), commsim.PeerInfo(**case["b"])
        assert commsim.select_transport(a, b) == case["transport"]


def test_estimate_jct_matches_reference():
    for case in GOLDEN["estimate_jct"]:
        d = AllocationDecision(3, [tuple(x) for x in case["instances"]], "SHM", case["profiles"])
        try:
            got = {"jct": estimate_jct(Job(3, "train", case["size"], 1000.0, 0.0), d,
                                       PerfModel(**case["model"]), num_gpus=case["gpus"])}
        except Exception as exc:  # noqa: BLE001
            got = err_record(exc)
        want = {k: v for k, v in case.items() if k in ("jct", "error")}
        assert got == want, case


def test_bootstrap_check_cli_matches_reference(tmp_path):
    for case in GOLDEN["bootstrap_check"]:
        path = tmp_path / f"{case['name']}.jsonl"
        path.write_text("\n".join(json.dumps(r) for r in case["records"]) + "\n")
        argv = ["bootstrap-check", "--peers", str(path)] + (["--legacy"] if case["legacy"] else [])
        so, se = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(so), contextlib.redirect_stderr(se):
            rc = cli.main(argv)
        assert rc == case["rc"], case["name"]
        assert so.getvalue() == case["stdout"], case["name"]
        # error text names the same ranks / label; paths differ
        if case["stderr"]:
            assert se.getvalue().split(":")[0] == case["stderr"].split(":")[0]
            if "resolve to the same device" in case["stderr"]:
                assert se.getvalue() == case["stderr"]
