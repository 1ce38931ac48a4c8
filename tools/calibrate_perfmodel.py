"""Recalibrate the simulator's PerfModel.multi_overhead (reference
simcore.py:46-51, 91-100) from measured B200 step times:
one-to-many = the DP step over n instances with the SHM allreduce, one-to-one
= the same step on the same instances without gradient sync (bench.py
--train-only --train-no-sync).  usage: calibrate_perfmodel.py OUT train_*.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_09143_b200.simcore import PerfModel  # noqa: E402

out = {}
for path in sys.argv[2:]:
    doc = json.load(open(path))
    for model, d in doc.items():
        if "no_sync" not in d:
            continue
        pm = PerfModel.from_measurement(d["ms_per_step"] / 1e3, d["no_sync"]["ms_per_step"] / 1e3)
        out[model] = {"instances": d["instances"], "dp_step_ms": d["ms_per_step"],
                      "no_sync_step_ms": d["no_sync"]["ms_per_step"],
                      "perf_model": pm.to_dict(), "source": path}
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps({k: round(v["perf_model"]["multi_overhead"], 3) for k, v in out.items()}))
