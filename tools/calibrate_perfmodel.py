"""Recalibrate the simulator's PerfModel.multi_overhead (reference
simcore.py:46-51, 91-100) from measured
B200 step times.

The reference defines multi_overhead as one-to-many over one-to-one
execution of the SAME job: one-to-many = the DP step over k 1g instances
(batch b each, SHM gradient allreduce), one-to-one = the job on ONE instance
of the combined size (here the whole GPU, `mode=full`, batch k*b).  Each
one-to-many step processes k*b samples, so the ratio of step times is the
ratio of job completion times.

usage: calibrate_perfmodel.py OUT MANY.json ONE.json
  MANY.json: `bench.py --train-only --train-model M [--train-no-sync]` (k ranks)
  ONE.json:  `bench.py --train-only --train-model M --ranks-per-gpu 1
              --train-mode full --batch k*b`
The sync-only overhead (DP step / the same step without gradient sync, when
MANY.json carries `no_sync`) is reported beside it."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_09143_b200.simcore import PerfModel  # noqa: E402


def calibrate(many: dict, one: dict) -> dict:
    out = {}
    for model, d in many.items():
        o = one.get(model)
        if not o or "ms_per_step" not in d or "ms_per_step" not in o:
            continue
        k, b = d["instances"], d["batch_per_instance"]
        if o.get("instances") != 1 or o.get("batch_per_instance") != k * b:
            raise ValueError(f"{model}: one-to-one run must be 1 instance x batch {k * b}, got "
                             f"{o.get('instances')} x {o.get('batch_per_instance')}")
        pm = PerfModel.from_measurement(d["ms_per_step"] / 1e3, o["ms_per_step"] / 1e3)
        rec = {"one_to_many": {"instances": k, "batch_per_instance": b,
                               "ms_per_step": d["ms_per_step"],
                               "instance_mode": d.get("instance_mode")},
               "one_to_one": {"instances": 1, "batch": k * b, "ms_per_step": o["ms_per_step"],
                              "instance_mode": o.get("instance_mode")},
               "perf_model": pm.to_dict()}
        if "no_sync" in d:
            rec["sync_overhead"] = d["ms_per_step"] / d["no_sync"]["ms_per_step"]
            rec["one_to_many"]["no_sync_ms_per_step"] = d["no_sync"]["ms_per_step"]
        out[model] = rec
    return out


def main(argv):
    if len(argv) != 4:
        sys.exit(__doc__)
    res = calibrate(json.load(open(argv[2])), json.load(open(argv[3])))
    for v in res.values():
        v["source"] = {"one_to_many": argv[2], "one_to_one": argv[3]}
    json.dump(res, open(argv[1], "w"), indent=1)
    print(json.dumps({k: round(v["perf_model"]["multi_overhead"], 3) for k, v in res.items()}))


if __name__ == "__main__":
    main(sys.argv)
