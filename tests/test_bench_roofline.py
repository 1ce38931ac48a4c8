"""bench.py's roofline arithmetic against BASELINE.md §3's exact per-GPU link
bytes and the T* DESIGN.md §4.4 quotes; rank placement from
fm_select (reference scheduler.py:117-136).  CPU only."""

from __future__ import annotations

import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


R50 = 25_557_032 * 4
MBV2 = 3_504_872 * 4
BERT = 109_483_778 * 2


@pytest.mark.parametrize("n,gpus,s,d2h,h2d", [
    (2, 1, R50, 204_456_256, 204_456_256),            # C1
    (7, 1, R50, 715_596_896, 1_226_737_536),          # C2
    (4, 2, MBV2, 28_038_976, 42_058_464),             # C3, per GPU (2+2)
    (14, 2, BERT, 1_532_772_892, 2_846_578_228),      # C4 at 2 GPUs (7+7)
])
def test_link_bytes_match_baseline_table(n, gpus, s, d2h, h2d):
    b = _bench()
    d = b.decision_for(gpus, n // gpus)
    per_gpu = [sum(1 for g, _ in d.instances if g == gg) for gg in range(gpus)]
    got = b.link_bytes(n, per_gpu, s)
    assert int(got[0][0]) == d2h
    assert int(round(got[0][1])) == h2d


def test_step_roofline_c2_t_star():
    b = _bench()
    peaks = dict(b.LINK_PEAK_FALLBACK, dram=100.0)
    r = b.step_roofline(7, [7], R50, 27.0e-3, peaks)
    assert r["t_star_ms"] == pytest.approx(22.06, abs=0.01)     # H2D-bound, DESIGN §4.4
    assert r["frac"] == pytest.approx(22.06 / 27.0, abs=1e-3)
    assert r["host_dram"]["bytes"] == 715_596_896 + 1_226_737_536


def test_kernel_roofline_uses_the_live_launch_and_the_store_peak():
    b = _bench()

    class A:
        steps, transport = 10, "auto"
    # 40 launches over 10 steps, 6 ms of kernel time: 150 us per launch
    r = b.kernel_roofline(A(), 7, R50, 6.0, 40)
    per_launch = 10 * R50 / 40
    assert r["bound"] == "host_link" and r["peak"] == b.ZC_WRITE_PEAK
    assert r["launch_us"] == pytest.approx(150.0)
    assert r["achieved"] == pytest.approx(per_launch / 150e-6 / 1e9)
    assert r["frac"] == pytest.approx(r["achieved"] / b.ZC_WRITE_PEAK)
