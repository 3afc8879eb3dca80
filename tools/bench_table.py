"""Print DESIGN.md §14 table rows from bench.py JSON lines.
    python tools/bench_table.py label=path.json ..."""
import json
import sys


def last(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


for arg in sys.argv[1:]:
    label, path = arg.split("=", 1)
    d = last(path)
    r = d["roofline"]
    lv = r.get("levels", {})
    fr = lambda k: f"{lv[k]['frac']:.2f}" if k in lv else "?"  # noqa: E731
    simt = lv.get("issue", {}).get("simt_threads_per_inst")
    alg = r.get("algorithmic", {})
    print(f"| {label} | {d['config'].get('query')} / {d['config'].get('intersector')} | {d['value']:,.0f} | "
          f"{d['ms_per_step']:.4f} | {r.get('kernel_ms')} | {r['bound']}, {r['frac']:.2f} | "
          f"{fr('l1')} / {fr('l2')} / {fr('dram')} | {simt} | "
          f"{alg.get('bytes_per_ray', 0):,.0f} ({alg.get('cache_reuse_ratio', 0):.2f}) |")
