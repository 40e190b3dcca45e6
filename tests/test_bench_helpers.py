"""bench.py's accounting on CPU: SURVEY.md 8(d)'s algorithmic bytes per pixel
(the figures DESIGN.md section 4 states), the per-step launch list the live
per-kernel timing maps events onto, and the step-DRAM supplement."""
import json
import os

import pytest

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("h,w,L,k,s,fwd,bwd,dom", [
    (1080, 1920, 3, 5, 4, 187.25, 374.5, 304.0),        # c4a: fp32 logits and gradients
    (2160, 3840, 4, 7, 2, 176.66, 353.31, 284.0),       # c3: bf16 logits and gradients
])
def test_algorithmic_bytes_per_pixel(h, w, L, k, s, fwd, bwd, dom):
    f, b, d = bench.algorithmic_bytes(h, w, L, k, s, s)
    n = h * w
    assert abs(f / n - fwd) < 0.01 and abs(b / n - bwd) < 0.01 and abs(d / n - dom) < 0.01


def test_launch_list_matches_the_library_order(monkeypatch):
    monkeypatch.delenv("SSB_NO_CHAIN", raising=False)
    names = bench.launches_per_step(3)
    assert names == ["pool0->1", "pool1->2", "fwd_l2", "fwd_l1", "fwd_l0",
                     "bwd_up", "bwd_l1", "bwd_l2", "bwd_chain", "bwd_l0"]
    assert bench.launches_per_step(2)[-3:] == ["bwd_up", "bwd_l1", "bwd_l0"]  # no pool chain below L = 3
    assert bench.launches_per_step(4, fwd_only=True) == ["pool0->1", "pool1->2", "pool2->3",
                                                         "fwd_l3", "fwd_l2", "fwd_l1", "fwd_l0"]
    monkeypatch.setenv("SSB_NO_CHAIN", "1")
    assert bench.launches_per_step(3)[-4:] == ["bwd_l0", "bwd_l1", "bwd_l2", "bwd_final"]


def test_step_dram_from_committed_traffic():
    tr = json.load(open(os.path.join(ROOT, "profiles", "step_traffic.json")))
    for wl in ("c4a", "c3"):
        d = bench.step_dram(wl, 5000.0, 6551.4)
        assert d["dram_bytes_per_px"] == tr[wl]["dram_bytes_per_px"]
        assert abs(d["achieved"] - tr[wl]["dram_bytes_per_px"] * 5.0) < 0.2
        assert abs(d["frac"] - d["achieved"] / 6551.4) < 1e-4
    assert bench.step_dram("c2", 1.0, 1.0) is None
