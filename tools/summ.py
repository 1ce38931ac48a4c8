"""One line per bench JSON: ms/step, mode, step-roofline frac, e2e ms, img/s."""
import json
import sys

for p in sys.argv[1:]:
    try:
        d = json.load(open(p))
    except Exception as e:  # noqa: BLE001
        print(p, "unreadable", e)
        continue
    r = d.get("resnet50") or {}
    e = d.get("e2e") or {}
    print(f"{p:50s} {d.get('ms_per_step', 0):7.2f} ms  {d['config'].get('instance_mode'):6s} "
          f"frac={d.get('step_roofline', {}).get('frac', 0):.3f} e2e={e.get('ms_per_step')} "
          f"img/s={r.get('img_s')}")
