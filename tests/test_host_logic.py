"""Host-side logic that runs without a GPU: the launcher's per-rank
environment contract (reference PAPER.md:377-384), instance identity,
ZeRO shard ownership, the cost-model calibration hook, the CLI `select`
command, and the canonical bus-id mapping."""

from __future__ import annotations

import json
import subprocess
import sys

import pytest

from paper_2511_09143_b200 import instance
from paper_2511_09143_b200.commsim import PeerInfo, canonical_bus_id
from paper_2511_09143_b200.errors import MalformedLabelError
from paper_2511_09143_b200.launcher import new_job_key, rank_env
from paper_2511_09143_b200.scheduler import fm_select, make_cluster
from paper_2511_09143_b200.simcore import PerfModel
from paper_2511_09143_b200.workload import Job


def test_rank_env_follows_fm_rank_order():
    d = fm_select(Job(0, "train", 14, 0, 0), make_cluster("FM", 2))
    envs = [rank_env(d, r, "k", "green") for r in range(14)]
    assert [e["RANK"] for e in envs] == [str(r) for r in range(14)]
    assert all(e["WORLD_SIZE"] == "14" for e in envs)
    # round-robin over GPUs: rank r on GPU r % 2 for the 1g.5gb leaves
    assert [e["CUDA_VISIBLE_DEVICES"] for e in envs[:12]] == ["0", "1"] * 6
    assert [(e["FMX_GPU_ID"], e["FMX_INSTANCE_ID"]) for e in envs[:4]] == [
        ("0", "1"), ("1", "1"), ("0", "2"), ("1", "2")]
    assert envs[12]["FMX_PROFILE"] == "1g.10gb"


def test_rank_env_mig_uuid():
    d = fm_select(Job(0, "train", 2, 0, 0), make_cluster("FM", 1))
    uuids = {(0, 1): "MIG-aaaa", (0, 2): "MIG-bbbb"}
    e = rank_env(d, 1, "k", "mig", mig_uuids=uuids)
    assert e["CUDA_VISIBLE_DEVICES"] == "MIG-bbbb" and e["FMX_MIG_UUID"] == "MIG-bbbb"


def test_job_keys_are_unique():
    assert len({new_job_key() for _ in range(100)}) == 100


def test_instance_identity_token():
    a = instance.Instance(0, 3, "1g.5gb", "green", gpu_uuid="u", bus_id="00:C0:00.0")
    b = instance.Instance(0, 4, "1g.5gb", "green", gpu_uuid="u", bus_id="00:C0:00.0")
    assert a.mig_id != b.mig_id and a.mig_id.startswith("green-u-")
    m = instance.Instance(0, 3, "1g.5gb", "mig", mig_uuid="MIG-x")
    assert m.mig_id == "MIG-x"
    assert instance.host_hash() == instance.host_hash()
    assert instance.default_sm_count(148) == 16


@pytest.mark.parametrize("raw,want", [("0000:c0:00.0", "00:C0:00.0"), ("00000000:4B:00.0", "00:4B:00.0"),
                                      ("00:4b:00.0", "00:4B:00.0")])
def test_canonical_bus_id(raw, want):
    assert canonical_bus_id(raw) == want
    PeerInfo(0, canonical_bus_id(raw), "x", 1, 1)   # accepted by the reference rules


def test_canonical_bus_id_rejects_non_function_zero():
    with pytest.raises(MalformedLabelError):
        canonical_bus_id("0000:4b:00.1")


def test_zero_shard_ownership_is_contiguous_and_balanced():
    torch = pytest.importorskip("torch")
    from paper_2511_09143_b200.ddp import ZeroShardBroadcast

    class FakeComm:
        size = 4

    params = [torch.nn.Parameter(torch.zeros(n)) for n in (100, 5, 300, 7, 50, 50, 200, 1)]
    z = ZeroShardBroadcast(params, FakeComm())
    assert z.owner == sorted(z.owner) and z.owner[0] == 0 and max(z.owner) <= 3
    assert sum(len(z.owned(r)) for r in range(4)) == len(params)


def test_perf_model_calibration():
    m = PerfModel.from_measurement(1.07, 1.0)
    assert m.multi_overhead == pytest.approx(1.07)
    with pytest.raises(ValueError):
        PerfModel.from_measurement(0.0, 1.0)


def test_perf_model_one_to_one_calibration():
    """tools/calibrate_perfmodel.py: multi_overhead = T(k x 1g, batch b each) /
    T(1 instance of the combined size, batch k*b) - the reference's
    one-to-many over one-to-one (simcore.py:46-51)."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "calib", os.path.join(os.path.dirname(__file__), "..", "tools", "calibrate_perfmodel.py"))
    calib = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(calib)
    many = {"resnet50": {"instances": 7, "batch_per_instance": 32, "ms_per_step": 70.0,
                         "no_sync": {"ms_per_step": 56.0}}}
    one = {"resnet50": {"instances": 1, "batch_per_instance": 224, "ms_per_step": 50.0}}
    res = calib.calibrate(many, one)["resnet50"]
    assert res["perf_model"]["multi_overhead"] == pytest.approx(1.4)
    assert res["sync_overhead"] == pytest.approx(1.25)
    with pytest.raises(ValueError):
        calib.calibrate(many, {"resnet50": {"instances": 1, "batch_per_instance": 32,
                                            "ms_per_step": 9.0}})


def test_cli_select_prints_rank_order():
    out = subprocess.run([sys.executable, "-m", "paper_2511_09143_b200.cli", "select", "--gpus", "2",
                          "--size", "4"], capture_output=True, text=True, check=True).stdout
    doc = json.loads(out)
    assert doc["instances"] == [[0, 1], [1, 1], [0, 2], [1, 2]] and doc["transport"] == "SHM"
