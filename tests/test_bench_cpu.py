"""bench.py host logic (CPU): the ncu counter parser, the roofline levels arithmetic, the
binding-level choice and the staleness rule of the committed-counter fallback."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

CSV = '''==PROF== Connected to process 123
"ID","Process ID","Process Name","Host Name","Kernel Name","Context","Stream","Block Size","Grid Size","Device","CC","Section Name","Metric Name","Metric Unit","Metric Value"
"0","123","python3.12","127.0.0.1","void vsr::trace_kernel<1, vsr::alpha_bits_intersector, 0, 0>(vsr::TraceParams)","1","7","(128, 1, 1)","(16200, 1, 1)","0","10.0","Command line profiler metrics","dram__bytes_read.sum","byte","68660736"
"0","123","python3.12","127.0.0.1","void vsr::trace_kernel<1, vsr::alpha_bits_intersector, 0, 0>(vsr::TraceParams)","1","7","(128, 1, 1)","(16200, 1, 1)","0","10.0","Command line profiler metrics","dram__bytes_write.sum","byte","6023936"
"0","123","python3.12","127.0.0.1","void vsr::trace_kernel<1, vsr::alpha_bits_intersector, 0, 0>(vsr::TraceParams)","1","7","(128, 1, 1)","(16200, 1, 1)","0","10.0","Command line profiler metrics","smsp__inst_executed.sum","inst","73,580,318"
"0","123","python3.12","127.0.0.1","void vsr::trace_kernel<1, vsr::alpha_bits_intersector, 0, 0>(vsr::TraceParams)","1","7","(128, 1, 1)","(16200, 1, 1)","0","10.0","Command line profiler metrics","l1tex__t_bytes.sum","byte","391133920"
"0","123","python3.12","127.0.0.1","void vsr::trace_kernel<1, vsr::alpha_bits_intersector, 0, 0>(vsr::TraceParams)","1","7","(128, 1, 1)","(16200, 1, 1)","0","10.0","Command line profiler metrics","lts__t_bytes.sum","byte","217018400"
==PROF== Disconnected from process 123
'''


def test_parse_ncu_csv():
    r = bench.parse_ncu_csv(CSV)
    assert r["kernel"].startswith("void vsr::trace_kernel<1")
    m = r["metrics"]
    assert m["smsp__inst_executed.sum"] == 73580318.0      # thousands separators stripped
    assert m["dram__bytes_read.sum"] == 68660736.0 and m["lts__t_bytes.sum"] == 217018400.0
    assert bench.parse_ncu_csv("no csv here") is None


def test_roofline_levels_and_bound():
    r = bench.parse_ncu_csv(CSV)
    lv = bench.roofline_levels(r, ms_kernel=0.1036, sm_mhz=1965.0, sms=148, hbm_peak=6535.1)
    t = 0.1036e-3
    assert lv["issue"]["peak"] == pytest.approx(148 * 4 * 1965e6 / 1e9, rel=1e-3)
    assert lv["issue"]["frac"] == pytest.approx(73580318 / t / (148 * 4 * 1965e6), rel=1e-3)
    assert lv["l1"]["frac"] == pytest.approx(391133920 / t / (148 * 128 * 1965e6), rel=1e-3)
    assert lv["l2"]["frac"] == pytest.approx(217018400 / t / (6300 * 1965e6), rel=1e-3)
    assert lv["dram"]["frac"] == pytest.approx((68660736 + 6023936) / t / 1e9 / 6535.1, rel=1e-3)
    key = max(lv, key=lambda k: lv[k]["frac"])
    assert key == "issue" and bench.BOUND_NAME[key] == "alu"


def test_committed_counters_only_for_the_current_source(tmp_path, monkeypatch):
    class A:
        config, query, isect = "C2", "any", "alpha_texture"
    prof = tmp_path / "profiles"
    prof.mkdir()
    entry = {"dram_bytes_per_launch": 1, "warp_instructions_per_launch": 2, "source": "x"}
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    (prof / "ncu_traffic.json").write_text(json.dumps({"C2:any:alpha_texture": {**entry, "source_sha": "stale"}}))
    monkeypatch.setattr(bench, "source_hash", lambda: "current")
    got, why = bench.committed_counters(A)
    assert got is None and "stale" in why
    (prof / "ncu_traffic.json").write_text(json.dumps({"C2:any:alpha_texture": {**entry, "source_sha": "current"}}))
    got, why = bench.committed_counters(A)
    assert got["metrics"]["smsp__inst_executed.sum"] == 2


def test_source_hash_tracks_the_kernel_sources():
    h = bench.source_hash()
    assert len(h) == 16 and h == bench.source_hash()
