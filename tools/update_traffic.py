"""Record ncu DRAM traffic, L1/L2 bytes and instruction counts of a trace kernel capture in
profiles/ncu_traffic.json, keyed "<config>:<query>:<isect>" — bench.py's roofline fallback
when its live ncu probe cannot run; used only while `source_sha` equals the current
kernel sources' hash (bench.source_hash), so a kernel change never reuses stale counters.

    python tools/update_traffic.py <report.ncu-rep> <key> <profile summary path>"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import raw  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import source_hash  # noqa: E402

rep, key, src = sys.argv[1], sys.argv[2], sys.argv[3]
d = raw(rep)[0]
mb = lambda k: float(d[k][0]) * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}[d[k][1]]  # noqa: E731
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                    "ncu_traffic.json")
db = json.load(open(path)) if os.path.exists(path) else {}
dur = float(d["gpu__time_duration.sum"][0]) * (1e-3 if d["gpu__time_duration.sum"][1] == "us" else 1.0)
db[key] = {
    "dram_bytes_per_launch": int(mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")),
    "warp_instructions_per_launch": int(float(d["smsp__inst_executed.sum"][0])),
    "ncu_duration_ms": dur,
    "issue_active_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
    "simt_threads_per_inst": float(d["smsp__thread_inst_executed_per_inst_executed.ratio"][0]),
    "kernel": d["kernel"],
    "source": src,
    "source_sha": source_hash(),
}
for k in ("l1tex__t_bytes.sum", "lts__t_bytes.sum"):
    if k in d:
        db[key][k] = int(mb(k))
json.dump(db, open(path, "w"), indent=2)
print(key, db[key])
