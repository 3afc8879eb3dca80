"""Summarise an ncu report: key raw metrics + hottest SASS regions (run on the dev box)."""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'l1tex__t_sector_hit_rate.pct', 'lts__t_sector_hit_rate.pct', 'sm__inst_executed.sum',
        'smsp__inst_executed.sum', 'smsp__thread_inst_executed_per_inst_executed.ratio',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'sm__cycles_active.avg', 'gpc__cycles_elapsed.max',
        'smsp__sass_average_branch_targets_threads_uniform.pct', 'sass__inst_executed_local_loads',
        'sass__inst_executed_local_stores', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__t_bytes.sum',
        'lts__t_bytes.sum', 'smsp__thread_inst_executed.sum']


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = (r[i], units[i])
        res.append(d)
    return res


def sass_hot(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    isrc, iex, ist = hdr.index("Source"), hdr.index("Instructions Executed"), \
        hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            break
        try:
            data.append((r[0], r[isrc], int(r[iex] or 0), int(r[ist] or 0)))
        except ValueError:
            break
    return data


if __name__ == "__main__":
    rep = sys.argv[1]
    for d in raw(rep):
        print("kernel:", d.pop("kernel"))
        for k, (v, u) in d.items():
            print(f"  {k:60s} {v} {u}")
    data = sass_hot(rep)
    tot = sum(x[2] for x in data)
    print("total warp instructions (source page):", tot)
    # stall reasons: the source page's per-instruction pc-sampling columns, summed
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    sums = {hdr[i][6:]: 0 for i in cols}
    for r in rows[2:]:
        if len(r) < len(hdr):
            break
        for i in cols:
            try:
                sums[hdr[i][6:]] += int(r[i] or 0)
            except ValueError:
                pass
    allv = sum(sums.values())
    if allv:
        print("stall reasons (pc sampling, share of samples):")
        for k, v in sorted(sums.items(), key=lambda kv: -kv[1])[:8]:
            print(f"  {k:24s} {100.0 * v / allv:5.1f}%")
