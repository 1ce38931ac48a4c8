"""Summarise ncu artefacts for profiles/: launch list (per-kernel counts and
mean device time) and the key counters of a --set full capture."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "pcie__read_bytes.sum.per_second", "pcie__write_bytes.sum.per_second",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "syslts__t_sectors_srcunit_tex_aperture_sysmem_op_write_lookup_miss.sum",
        "syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard"]


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    agg = defaultdict(list)
    for r in rows[start + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(d["Metric Unit"], 1.0)
            agg[d["Kernel Name"]].append(float(d["Metric Value"]) * scale)
    total = sum(sum(v) for v in agg.values())
    return {k: {"launches": len(v), "mean_us": sum(v) / len(v), "total_us": sum(v),
                "share": sum(v) / total} for k, v in agg.items()}


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{vals[i]} {units[i]}".strip()
        res.append(d)
    return res


if __name__ == "__main__":
    doc = {}
    for a in sys.argv[1:]:
        doc[a] = launches(a) if a.endswith(".csv") else full(a)
    print(json.dumps(doc, indent=1))
