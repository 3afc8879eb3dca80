#!/usr/bin/env python
"""bench.py — Mrays/s of the custom-intersector trace path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl own|reference]
                    [--config C2] [--query closest|any] [--isect alpha_texture|...]

A step is one pass of the whole hot path (ray fetch,
root test, inner-node loop, leaf loop with the intersector, hit write) over one
1920×1080 frame of the C2 billboard forest (BASELINE.json configs[1]): ONE
`vsr_trace` launch.  Inputs are resident in HBM when the timed region starts;
L2 is flushed (256 MiB read) before every timed step, outside the events.

N > 1: `--gpus N` without torchrun re-launches itself under torch.distributed.run
(one process per GPU, 127.0.0.1 rendezvous).  The headline is weak scaling —
every rank traces its own 1080p frame (camera shifted per rank) against a scene
built once on rank 0 and broadcast with NCCL; the timed path has no collective
(rays are independent).  The `strong` object is SURVEY §8(e)'s
C5 frame dealt round-robin in 8×8 tiles over the ranks, each trace kernel storing
its hits straight into rank 0's double-buffered frame over CUDA IPC (NVLink peer
stores), F frames in flight with a barrier per frame pair.
Timing: CUDA events on the launching stream, max over ranks.

Roofline: the trace kernel's counters (warp instructions, L1/L2/DRAM bytes) are
measured by an `ncu` pass over a short probe run of the same launch (--probe),
so they track the kernel that was timed; `bound` is whichever level is nearest
its peak.

--impl reference: the CPU oracle (oracle S, brute force, as it stands) on the
host cores, each step a bounded ray sample of the same workload.
"""
from __future__ import annotations

import argparse
import csv
import hashlib
import io
import json
import math
import os
import shutil
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "Mrays/s per B200 (alpha-mask any-hit, 1080p) at 1/2/4/8 GPUs; % HBM roofline"
UNIT = "Mrays/s"
ISECTS = ("none", "default", "alpha_texture", "alpha_procedural", "count", "count_alpha_texture",
          "alpha_texture_bilinear", "alpha_procedural_uv",
          "runtime_switch_default", "runtime_fnptr_default", "runtime_switch_alpha_texture",
          "runtime_fnptr_alpha_texture")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="own", choices=["own", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--query", default="any", choices=["closest", "any"])
    ap.add_argument("--isect", default="alpha_texture")
    ap.add_argument("--no-variants", action="store_true", help="skip the C3 intersector sweep")
    ap.add_argument("--graph", type=int, default=0,
                    help="1: replay the headline trace call from a CUDA graph each step")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--bvh", default="binary", choices=["binary", "wide"],
                    help="binary: 64-B pair-node SAH BVH (default); wide: the same tree collapsed "
                         "into the 8-wide compressed BVH (vsr_bvh8_build / vsr_trace_bvh8)")
    ap.add_argument("--max-leaf", type=int, default=2, help="BVH build: max triangles per leaf")
    ap.add_argument("--sah-bins", type=int, default=16, help="BVH build: SAH bins per axis")
    ap.add_argument("--mode", default="weak", choices=["weak", "tiles", "tiles-nccl"],
                    help="weak: a frame per rank; tiles: one frame's tiles over the ranks, each "
                         "trace kernel storing its hits into rank 0's frame over CUDA IPC/NVLink "
                         "(vsr_trace_tiles); tiles-nccl: the same with an NCCL all-gather")
    ap.add_argument("--strong-config", default="C5",
                    help="config of the strong-scaling tile line (SURVEY §8(e)); 'none' skips it")
    ap.add_argument("--strong-frames", type=int, default=20)
    ap.add_argument("--no-counters", action="store_true",
                    help="skip the ncu counter probe (roofline falls back to profiles/)")
    ap.add_argument("--probe", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--plumbing", action="store_true", help=argparse.SUPPRESS)
    return ap.parse_args()


def config_desc(name):
    import workloads as W
    return {"workload": f"{name}: {W.CONFIGS[name]}"}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML in a background thread)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device_index=0, period=0.0):   # back-to-back NVML reads (~0.1 ms each)
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self.period = period
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "samples": len(self.samples), "reasons": names}


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------
def make_workload(name, rank=0):
    """Scene + this rank's frame (camera shifted 2 m sideways per rank)."""
    import workloads as W
    return W.scene(name), W.rays_for(name, shift_x=2.0 * rank)


def algorithmic_bytes(counts_np, isect_has_alpha, counts_out=False):
    """B(r) = 32 + 16 [+ counts] + 64*I + 48*T + 36*A, I = (boxes-1)/2; the
    counting intersectors write a 16-B counts record per ray (the layout's, vsr.h vsr_counts)."""
    boxes = counts_np["boxes"].astype(np.int64)
    tris = counts_np["tris"].astype(np.int64)
    alpha = counts_np["alpha"].astype(np.int64) if isect_has_alpha else 0
    inner = (boxes - 1) // 2
    per_ray = 48 + (16 if counts_out else 0) + 64 * inner + 48 * tris + 36 * alpha
    return int(per_ray.sum()), {"inner_per_ray": float(inner.mean()), "tris_per_ray": float(tris.mean()),
                                "alpha_per_ray": float(np.mean(alpha)) if isect_has_alpha else 0.0}


# ---------------------------------------------------------------------------
# roofline counters (ncu over a probe run of the same launch) and levels
# ---------------------------------------------------------------------------
COUNTER_METRICS = ("smsp__inst_executed.sum", "smsp__thread_inst_executed.sum",
                   "l1tex__t_bytes.sum", "lts__t_bytes.sum", "dram__bytes_read.sum",
                   "dram__bytes_write.sum", "gpu__time_duration.sum")
L1_BYTES_PER_CLK_SM = 128.0    # L1TEX data path per SM per clock (nominal, Volta+)
L2_BYTES_PER_CLK = 6300.0      # full-chip LTS throughput cap, B300_MICROARCH.md "L2 cache"
ISSUE_PER_CLK_SM = 4.0         # 4 SMSPs, one warp-instruction issued per clock each


def source_hash():
    """Hash of everything that shapes the trace kernel (sources + build flags): a committed
    counter capture is only reused when it was taken from this exact source."""
    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_1912_12786_b200", "csrc")
    for f in sorted(os.listdir(csrc)):
        with open(os.path.join(csrc, f), "rb") as fh:
            h.update(f.encode() + fh.read())
    for extra in (os.path.join(ROOT, "include", "vsr.h"),
                  os.path.join(ROOT, "paper_1912_12786_b200", "_build.py")):
        with open(extra, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def parse_ncu_csv(text):
    """{metric: float} of the (single) profiled launch in `ncu --csv --print-units base`
    output, plus its kernel name; None if no row was found."""
    rows = [ln for ln in text.splitlines() if ln.startswith('"')]
    if not rows:
        return None
    rd = list(csv.reader(io.StringIO("\n".join(rows))))
    hdr = rd[0]
    try:
        im, iv, ik = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Kernel Name")
    except ValueError:
        return None
    out, kernel = {}, None
    for r in rd[1:]:
        if len(r) <= max(im, iv, ik):
            continue
        try:
            out[r[im]] = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        kernel = r[ik]
    return {"metrics": out, "kernel": kernel} if out else None


def probe_counters(args, timeout=420):
    """Run `ncu` on a short probe of the headline launch (same config, query, intersector,
    build) and return its counters, or (None, reason).  Counts, not times, are taken from
    ncu; --clock-control none leaves the GPU clocks alone."""
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, "ncu not found"
    cmd = [ncu, "--metrics", ",".join(COUNTER_METRICS), "--print-units", "base", "--csv",
           "--clock-control", "none", "-k", "regex:trace_(wide_)?kernel", "-s", "2", "-c", "1",
           sys.executable, os.path.abspath(__file__), "--probe", "--config", args.config,
           "--query", args.query, "--isect", args.isect, "--max-leaf", str(args.max_leaf),
           "--sah-bins", str(args.sah_bins), "--bvh", args.bvh]
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env)
    except Exception as e:   # timeout, no permission
        return None, f"ncu probe failed: {type(e).__name__}"
    res = parse_ncu_csv(r.stdout)
    if res is None or "smsp__inst_executed.sum" not in res["metrics"]:
        tail = (r.stdout + r.stderr).strip().splitlines()[-1:] or ["no output"]
        return None, f"ncu probe rc={r.returncode}: {tail[0][:200]}"
    return res, "ncu live probe (same config/query/intersector/build, 3rd trace launch)"


def committed_counters(args):
    """Fallback: profiles/ncu_traffic.json, only if captured from this exact source."""
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        tr = json.load(open(prof)).get(f"{args.config}:{args.query}:{args.isect}")
    except Exception:
        tr = None
    if not tr:
        return None, "no committed capture for this config"
    if tr.get("source_sha") != source_hash():
        return None, f"committed capture {tr.get('source')} is stale (source hash differs)"
    m = {"smsp__inst_executed.sum": tr["warp_instructions_per_launch"],
         "dram__bytes_read.sum": tr["dram_bytes_per_launch"], "dram__bytes_write.sum": 0.0}
    for k in ("l1tex__t_bytes.sum", "lts__t_bytes.sum", "smsp__thread_inst_executed.sum"):
        if k in tr:
            m[k] = tr[k]
    return {"metrics": m, "kernel": tr.get("kernel")}, tr.get("source")


def roofline_levels(ctr, ms_kernel, sm_mhz, sms, hbm_peak):
    """Per-level achieved/peak of the trace kernel: issue (warp-instructions), L1, L2, DRAM,
    each measured quantity per launch over the event-timed kernel duration."""
    t = ms_kernel * 1e-3
    f = sm_mhz * 1e6
    m = ctr["metrics"]
    lv = {}
    inst = m.get("smsp__inst_executed.sum")
    if inst:
        pk = sms * ISSUE_PER_CLK_SM * f
        lv["issue"] = {"per_launch": inst, "achieved": round(inst / t / 1e9, 1),
                       "peak": round(pk / 1e9, 1), "unit": "G warp-inst/s",
                       "frac": round(inst / t / pk, 4),
                       "peak_source": f"derived: {sms} SMs x 4 SMSP x 1 warp-inst/clk x {sm_mhz:.0f} MHz"}
        th = m.get("smsp__thread_inst_executed.sum")
        if th:
            lv["issue"]["simt_threads_per_inst"] = round(th / inst, 2)
    for key, metric, pk, src in (
            ("l1", "l1tex__t_bytes.sum", sms * L1_BYTES_PER_CLK_SM * f,
             f"nominal: {sms} SMs x 128 B/clk x {sm_mhz:.0f} MHz"),
            ("l2", "lts__t_bytes.sum", L2_BYTES_PER_CLK * f,
             f"B300_MICROARCH.md LTS cap 6300 B/clk x {sm_mhz:.0f} MHz")):
        b = m.get(metric)
        if b:
            lv[key] = {"per_launch": b, "achieved": round(b / t / 1e9, 1), "peak": round(pk / 1e9, 1),
                       "unit": "GB/s", "frac": round(b / t / pk, 4), "peak_source": src}
    if "dram__bytes_read.sum" in m:
        b = m["dram__bytes_read.sum"] + m.get("dram__bytes_write.sum", 0.0)
        lv["dram"] = {"per_launch": b, "achieved": round(b / t / 1e9, 1), "peak": hbm_peak,
                      "unit": "GB/s", "frac": round(b / t / 1e9 / hbm_peak, 4),
                      "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)"}
    return lv


BOUND_NAME = {"issue": "alu", "dram": "hbm", "l1": "l1", "l2": "l2"}


# ---------------------------------------------------------------------------
# own arm
# ---------------------------------------------------------------------------
def run_own(args):
    import torch
    import torch.distributed as dist

    from paper_1912_12786_b200 import _build, shard, vsr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    # VSR_DIST_BACKEND=gloo: plumbing test of the N-rank path on fewer GPUs
    # (ranks share devices; no kernel waits on another rank's kernel).
    backend = os.environ.get("VSR_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    cdev = "cuda" if backend == "nccl" else "cpu"   # device of collective tensors
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    if rank == 0:
        _build.build()
    if world > 1:
        dist.barrier()

    q = vsr.CLOSEST if args.query == "closest" else vsr.ANY
    isect = getattr(vsr, args.isect.upper())
    sc, rays = make_workload(args.config, rank)
    t0 = time.time()
    if world > 1:
        base = vsr.Scene.from_workload(sc, device=local).build(max_leaf_size=args.max_leaf, sah_bins=args.sah_bins) if rank == 0 else None
        scene, _ = shard.broadcast_scene(base, local, dist,
                                         tensor_device=None if backend == "nccl" else "cpu")
    else:
        scene = vsr.Scene.from_workload(sc, device=local).build(max_leaf_size=args.max_leaf, sah_bins=args.sah_bins)
    setup_s = time.time() - t0
    stats = scene.stats()
    wide_info = None
    if args.bvh == "wide":
        scene.build_wide()
        we = scene.export_wide()
        wide_info = {"nodes": int(we["nodes"].shape[0]), "max_depth": we["max_depth"],
                     "build_ms": round(we["build_ms"], 1), "node_bytes": 80}
        del we
    tiles = args.mode in ("tiles", "tiles-nccl")
    fused = args.mode == "tiles"
    tile_rays = 64 * rays.spp
    if tiles:   # strong scaling: this rank's round-robin 8x8-tile shard of ONE frame
        local_rays = rays.data[shard.rank_ray_indices(rays.n, tile_rays, rank, world)]
    else:       # weak scaling: this rank's own frame
        local_rays = rays.data
    n = local_rays.shape[0]
    d_rays = torch.from_numpy(np.ascontiguousarray(local_rays)).cuda()
    hits = torch.empty((n, 4), dtype=torch.float32, device="cuda")
    gathered = None
    peer = None
    if fused:   # rank 0's frame, mapped into every rank (IPC); each kernel stores its tiles there
        peer = shard.PeerFrame(rays.n, local, dist) if world > 1 else None
        frame_local = None if peer is not None else torch.empty((rays.n, 4), dtype=torch.float32,
                                                                 device="cuda")
        frame_ptr = peer.ptr if peer is not None else frame_local.data_ptr()
    elif tiles and world > 1:
        gathered = torch.empty((world * n, 4), dtype=torch.float32, device="cuda" if backend == "nccl" else "cpu")
    counts = torch.empty((n, 4), dtype=torch.int32, device="cuda")
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    # L2 flush by READING a buffer > 2x L2: it evicts the scene, rays and hits
    # and leaves only clean lines behind, so no write-back of flush data lands
    # inside the next timed launch (a write-based flush would).
    flush = torch.zeros(max(2 * l2, 256 << 20) // 4, dtype=torch.float32, device="cuda")
    flush_acc = torch.zeros((), dtype=torch.float32, device="cuda")

    def flush_l2():
        torch.sum(flush, 0, out=flush_acc)

    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream

    multi_k = 4
    multi_hits = None

    def trace(kind, query=q):
        sh = torch.cuda.current_stream().cuda_stream   # the capture stream under a CUDA graph
        if query == "multi":   # multi-hit query, k = 4
            scene.trace_multi(d_rays, multi_k, kind, hits=multi_hits, num_hits=multi_n,
                              counts=counts, stream=sh)
            return
        if fused and kind not in (vsr.COUNT, vsr.COUNT_ALPHA_TEXTURE):
            scene.trace_tiles(d_rays, tile_rays, rank, world, frame_ptr, query, kind, stream=sh)
            return
        if args.bvh == "wide":
            scene.trace_wide(d_rays, query, kind, hits=hits, counts=counts, stream=sh)
            return
        scene.trace_raw(d_rays.data_ptr(), n, query, kind, hits.data_ptr(),
                        counts.data_ptr(), sh)
        if gathered is not None:   # tile mode: assemble the frame's hits on every rank
            src = hits if backend == "nccl" else hits.cpu()
            shard.gather_hits(src, rays.n, tile_rays, dist, out=gathered, reorder=False)

    def timed(kind, steps, warmup, query=q, sampler=None, kernel_ms=None, graph=False):
        for _ in range(warmup):
            flush_l2()
            trace(kind, query)
        torch.cuda.synchronize()
        g = None
        per_call = 0
        if graph:   # one trace call (order pass + trace kernel) captured once, replayed per step
            g = torch.cuda.CUDAGraph()
            c0 = vsr.launch_count()
            with torch.cuda.graph(g):
                trace(kind, query)
            per_call = vsr.launch_count() - c0
            torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)] if kernel_ms is not None else None
        for pair in kev or []:   # create the CUDA events (torch creates them on first record)
            for e in pair:
                e.record(stream)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = vsr.launch_count()
        ctx = sampler if sampler is not None else _Null()
        with ctx:
            for i, (a, b) in enumerate(evs):
                flush_l2()
                if kev:   # events around the trace kernel alone (after the order pass)
                    vsr.set_kernel_events(*kev[i])
                a.record(stream)
                if g is not None:
                    g.replay()
                else:
                    trace(kind, query)
                b.record(stream)
            torch.cuda.synchronize()
        vsr.set_kernel_events(None, None)
        launches = vsr.launch_count() - l0 + per_call * (steps if g is not None else 0)
        if world > 1:
            dist.barrier()
        ms = [a.elapsed_time(b) for a, b in evs]
        if kev:
            kernel_ms.extend(a.elapsed_time(b) for a, b in kev)
        return ms, launches

    if args.probe:   # the ncu counter probe (probe_counters): 3 headline launches, no output
        for _ in range(3):
            flush_l2()
            trace(isect, q)
        torch.cuda.synchronize()
        return

    # ---- headline ----
    sampler = ClockSampler(local)
    use_graph = args.graph and not tiles
    ms, launches = timed(isect, args.steps, args.warmup, sampler=sampler, graph=use_graph)
    torch.cuda.synchronize()
    head_hits = vsr.hits_to_numpy(hits).copy() if not tiles else None   # for the parity summary
    # the trace kernel alone (roofline denominator), in a second pass: events
    # between the order pass and the trace kernel would break their PDL overlap
    kms = []
    timed(isect, args.steps, 1, kernel_ms=kms)
    ms_step = float(np.mean(ms))
    ms_kernel = float(np.mean(kms))   # the trace kernel alone (roofline denominator)
    if world > 1:
        t = torch.tensor([ms_step], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step_max = float(t.item())
    else:
        ms_step_max = ms_step
    value = world * n / (ms_step_max * 1e-3) / 1e6

    # ---- algorithmic bytes from the counting intersector (untimed) ----
    has_alpha = args.isect in ("alpha_texture", "count_alpha_texture",
                               "runtime_switch_alpha_texture", "runtime_fnptr_alpha_texture")
    cnt_kind = vsr.COUNT_ALPHA_TEXTURE if has_alpha else vsr.COUNT
    trace(cnt_kind)
    torch.cuda.synchronize()
    cnp = vsr.counts_to_numpy(counts)
    bytes_launch, work = algorithmic_bytes(cnp, has_alpha,
                                           counts_out=args.isect in ("count", "count_alpha_texture"))
    if args.bvh == "wide":   # SURVEY 8(d)'s bytes per ray are defined on the binary tree's visits
        bytes_launch, work = None, None
    peak, peak_src = load_peaks()
    touched = bytes_launch / (ms_kernel * 1e-3) / 1e9 if bytes_launch else None
    mhz = sampler.summary().get("sm_mhz") or 1965.0
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    ctr, ctr_src = (None, "skipped (--no-counters)")
    if rank == 0 and not args.no_counters:
        ctr, ctr_src = probe_counters(args)
        if ctr is None:
            fb, fb_src = committed_counters(args)
            ctr, ctr_src = (fb, fb_src) if fb else (None, f"{ctr_src}; {fb_src}")
    levels = roofline_levels(ctr, ms_kernel, mhz, sms, peak) if ctr else {}
    roofline = {"bound": None, "achieved": None, "peak": None, "unit": None, "frac": None,
                "traffic": levels.get("dram", {}).get("per_launch"),
                "kernel": (ctr or {}).get("kernel") or f"trace_kernel<{args.query}, {args.isect}>",
                "kernel_ms": round(ms_kernel, 4), "levels": levels, "counters_source": ctr_src,
                "algorithmic": None if bytes_launch is None else {
                    "bytes_per_launch": bytes_launch, "bytes_per_ray": round(bytes_launch / n, 1),
                    "work_per_ray": work, "touched_gbs": round(touched, 1),
                    "cache_reuse_ratio": round(touched / peak, 4),
                    "note": "SURVEY.md 8(d) bytes per ray (32 + 16 + 64 I + 48 T + 36 A) over the "
                            "kernel time, divided by the HBM peak: a touched-bytes / cache-reuse "
                            "ratio (the scene is re-read per ray from L1/L2), NOT a roofline "
                            "fraction; DRAM carries `traffic`."}}
    if levels:   # the binding level: the one nearest its peak
        key = max(levels, key=lambda k: levels[k]["frac"])
        b = levels[key]
        roofline.update({"bound": BOUND_NAME[key], "achieved": b["achieved"], "peak": b["peak"],
                         "unit": b["unit"], "frac": b["frac"], "peak_source": b["peak_source"]})

    # ---- variants: any-hit + the C3 zero-cost sweep (rank 0 only reports) ----
    extra = {}
    if not args.no_variants:
        ms_any, _ = timed(isect, max(5, args.steps // 2), 3, query=vsr.ANY if q == vsr.CLOSEST else vsr.CLOSEST)
        extra["other_query"] = {"query": "any" if q == vsr.CLOSEST else "closest",
                                "value": round(n / (np.mean(ms_any) * 1e-3) / 1e6, 1),
                                "ms": round(float(np.mean(ms_any)), 4)}
        var = {}
        for name in ISECTS:
            kind = getattr(vsr, name.upper())
            m, _ = timed(kind, max(5, args.steps // 2), 3)
            var[name] = round(n / (np.mean(m) * 1e-3) / 1e6, 1)
        # the listing's storage (A8 texel plane, VSR_ALPHA_BITS=0) beside the default 1-bit
        # decision plane (storage variants reported apart; same results)
        os.environ["VSR_ALPHA_BITS"] = "0"
        try:
            m, _ = timed(vsr.ALPHA_TEXTURE, max(5, args.steps // 2), 3)
        finally:
            del os.environ["VSR_ALPHA_BITS"]
        var["alpha_texture_a8"] = round(n / (np.mean(m) * 1e-3) / 1e6, 1)
        var["storage"] = {"alpha_texture": "1-bit decision plane (default)",
                          "alpha_texture_a8": "A8 texel plane (VSR_ALPHA_BITS=0)"}
        # interleaved A/B for the zero-cost claim
        a_ms, b_ms = [], []
        for _ in range(max(5, args.steps // 2)):
            a_ms += timed(vsr.NONE, 1, 1)[0]
            b_ms += timed(vsr.DEFAULT, 1, 1)[0]
        extra["variants_mrays"] = var
        # multi-hit query (4 nearest accepted hits per ray), same intersector
        multi_hits = torch.empty((n, multi_k, 4), dtype=torch.float32, device="cuda")
        multi_n = torch.empty((n,), dtype=torch.int32, device="cuda")
        m, _ = timed(isect, max(5, args.steps // 2), 3, query="multi")
        extra["multi_hit"] = {"k": multi_k, "value": round(n / (np.mean(m) * 1e-3) / 1e6, 1),
                              "ms": round(float(np.mean(m)), 4)}
        del multi_hits, multi_n
    if not args.no_variants and args.config in ("C2", "C3"):
        # NEXT-2: two-level instancing — instanced tree models over the
        # same ground square, this rank's frame, same query and intersector
        import workloads as W
        models, ibvh, imat = W.instanced_forest()
        iscenes = [vsr.Scene.from_workload(s, device=local).build() for s in models]
        inst = vsr.Instances(iscenes, ibvh, imat)
        inst_ids = torch.empty((n,), dtype=torch.int32, device="cuda")

        def trace_inst():
            inst.trace(d_rays, q, isect, hits=hits, inst=inst_ids, stream=stream)

        for _ in range(3):
            flush_l2()
            trace_inst()
        torch.cuda.synchronize()
        ievs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(max(5, args.steps // 2))]
        for a, b in ievs:
            flush_l2()
            a.record(stream)
            trace_inst()
            b.record(stream)
        torch.cuda.synchronize()
        im = float(np.mean([a.elapsed_time(b) for a, b in ievs]))
        extra["instanced"] = {"workload": f"{len(ibvh)} instances of {len(models)} tree models "
                                          f"({models[0].num_tris} tris each), C2 camera",
                              "value": round(n / (im * 1e-3) / 1e6, 1), "ms": round(im, 4),
                              "hit_fraction": round(float((inst_ids != -1).float().mean()), 3)}
        del inst, iscenes, inst_ids
    import workloads as W
    if not args.no_variants and args.config in W.CAMERAS and not tiles:
        # NEXT-4: the same frame with its primary rays generated inside the trace kernel
        # (vsr_trace_pinhole: no ray buffer); e2e = that + the hits' copy to pinned host memory
        eye, look, up, fov, cw, chh, cspp = W.CAMERAS[args.config]
        sh_x = 2.0 * rank
        cam = vsr.pinhole_camera((eye[0] + sh_x, eye[1], eye[2]), (look[0] + sh_x, look[1], look[2]),
                                 up, fov, cw, chh, cspp)
        h_out = torch.empty((n, 4), dtype=torch.float32).pin_memory()
        gen_ms, gen_e2e = [], []
        for it in range(3 + 2 * max(5, args.steps // 2)):
            flush_l2()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            c = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            scene.trace_pinhole(cam, q, isect, hits=hits, stream=stream)
            b.record(stream)
            h_out.copy_(hits, non_blocking=True)
            c.record(stream)
            c.synchronize()
            if it >= 3:
                gen_ms.append(a.elapsed_time(b))
                gen_e2e.append(a.elapsed_time(c))
        gm, ge = float(np.mean(gen_ms)), float(np.mean(gen_e2e))
        extra["raygen"] = {"api": "vsr_trace_pinhole (rays generated in the trace kernel)",
                           "value": round(n / (gm * 1e-3) / 1e6, 1), "ms": round(gm, 4),
                           "e2e": {"value": round(n / (ge * 1e-3) / 1e6, 1), "ms": round(ge, 4),
                                   "h2d_bytes_per_step": 0, "d2h_bytes_per_step": n * 16}}
        del h_out
    if not args.no_variants:
        # NEXT-3: the same scene built by the GPU linear-BVH builder (build time, trace speed)
        gb = {"host_sah_build_ms": round(stats["build_ms"], 2)}
        for name, how in (("lbvh", lambda s: s.build_gpu(args.max_leaf)),
                          ("ploc", lambda s: s.build_ploc(args.max_leaf, 16))):
            gscene = vsr.Scene.from_workload(sc, device=local)
            how(gscene)   # first call: CUDA module / CUB setup
            how(gscene)
            gst = gscene.stats()
            saved = scene
            scene = gscene
            mg, _ = timed(isect, max(5, args.steps // 2), 3)
            scene = saved
            gb[name] = {"build_ms": round(gst["build_ms"], 2), "nodes": gst["num_nodes"],
                        "max_depth": gst["max_depth"],
                        "value": round(n / (np.mean(mg) * 1e-3) / 1e6, 1),
                        "ms": round(float(np.mean(mg)), 4)}
            del gscene
        # NEXT-3: the same SAH tree collapsed into the 8-wide compressed BVH (vsr_trace_bvh8)
        if args.bvh == "binary" and not tiles:
            scene.build_wide()
            we = scene.export_wide()
            args.bvh = "wide"
            try:
                mw, _ = timed(isect, max(5, args.steps // 2), 3)
                mwo, _ = timed(isect, max(5, args.steps // 2), 3,
                               query=vsr.ANY if q == vsr.CLOSEST else vsr.CLOSEST)
            finally:
                args.bvh = "binary"
            extra["wide_bvh"] = {
                "api": "vsr_bvh8_build + vsr_trace_bvh8 (80-B nodes, 8 children, 8-bit planes)",
                "nodes": int(we["nodes"].shape[0]), "max_depth": we["max_depth"],
                "build_ms": round(we["build_ms"], 1),
                "value": round(n / (np.mean(mw) * 1e-3) / 1e6, 1), "ms": round(float(np.mean(mw)), 4),
                "other_query": {"query": "any" if q == vsr.CLOSEST else "closest",
                                "value": round(n / (np.mean(mwo) * 1e-3) / 1e6, 1)}}
            del we
        extra["gpu_build"] = {"builders": "vsr_bvh_build_gpu (LBVH, Karras 2012), "
                                          "vsr_bvh_build_ploc (PLOC, radius 16)", **gb}
        extra["zero_cost"] = {"none_ms": round(float(np.median(a_ms)), 4),
                              "default_ms": round(float(np.median(b_ms)), 4),
                              "overhead_pct": round(100 * (np.median(b_ms) / np.median(a_ms) - 1), 2)}

    # ---- strong scaling: one frame's tiles over the ranks ----
    strong = None
    if args.strong_config != "none" and not tiles and not args.probe:
        try:
            strong = run_strong(args, rank, world, local, dist, backend, cdev, q, isect)
        except Exception as e:   # reported, never silently dropped
            strong = {"error": f"{type(e).__name__}: {e}"}
        torch.cuda.synchronize()

    # ---- end to end through vsr_trace_host (pinned host buffers) ----
    h_rays = torch.from_numpy(np.ascontiguousarray(local_rays)).pin_memory()
    h_hits = torch.empty((n, 4), dtype=torch.float32).pin_memory()
    for _ in range(2):
        scene.trace_host(h_rays, q, isect, hits=h_hits, stream=stream)
    torch.cuda.synchronize()
    e2e_ms = []
    for _ in range(max(3, args.steps // 2)):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        scene.trace_host(h_rays, q, isect, hits=h_hits, stream=stream)
        b.record(stream)
        b.synchronize()
        e2e_ms.append(a.elapsed_time(b))
    e2e_step = float(np.mean(e2e_ms))
    if world > 1:
        t = torch.tensor([e2e_step], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_step = float(t.item())
    e2e = {"value": round(world * n / (e2e_step * 1e-3) / 1e6, 2), "unit": UNIT,
           "h2d_bytes_per_step": n * 32, "d2h_bytes_per_step": n * 16,
           "ms_per_step": round(e2e_step, 4), "api": "vsr_trace_host (pinned host buffers)"}

    # ---- cpu baseline (rank 0, N = 1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(sc, rays, args, target_s=args.cpu_seconds, scene=scene,
                           gpu_hits=head_hits)

    if rank == 0:
        clocks = sampler.summary()
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step_max, 4),
            "higher_is_better": True, "scaling": "strong" if tiles else "weak", "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (seeded generators, workloads/)",
            "config": {**config_desc(args.config), "query": args.query, "intersector": args.isect,
                       "rays_per_gpu": n, "resolution": f"{rays.width}x{rays.height}x{rays.spp}spp",
                       "triangles": int(stats["num_tris"]), "bvh_nodes": int(stats["num_nodes"]),
                       "bvh": f"binned SAH, {args.sah_bins} bins, max_leaf {args.max_leaf}"
                              + (", collapsed to the 8-wide compressed BVH" if args.bvh == "wide"
                                 else ""),
                       "wide_bvh": wide_info,
                       "textures": f"{len(sc.textures)}x{sc.textures[0].shape[1]}x{sc.textures[0].shape[0]} RGBA8",
                       "l2": "flushed before every timed step (read of a 256 MiB buffer, outside the events)",
                       "launch": ("one CUDA-graph replay of the trace call per step" if use_graph
                                  else "eager vsr_trace call per step"),
                       "parallelism": (f"one frame's 8x8 tiles dealt round-robin over {world} rank(s), "
                                       + ("each trace kernel stores its hits into rank 0's frame "
                                          "(CUDA IPC, NVLink peer stores; vsr_trace_tiles)" if fused
                                          else "hits all-gathered (NCCL) inside each step") if tiles else
                                       f"rays sharded by frame, {world} rank(s), no data-path collective"),
                       "setup_s": round(setup_s, 2)},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "strong": strong,
            "clocks": clocks, "ms_per_step_each": [round(x, 4) for x in ms],
            "ms_median": round(float(np.median(ms)), 4), "ms_min": round(float(np.min(ms)), 4),
            **extra,
        }
        print(json.dumps(line))
    if peer is not None:
        peer.release(dist)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_strong(args, rank, world, local, dist, backend, cdev, q, isect):
    """the `--strong-config` frame (C5: 3840x2160x4 spp, 10.2 M triangles)
    dealt round-robin in 8x8-pixel tiles (x spp) over the ranks; every rank's trace kernel
    stores its hits at their frame positions in rank 0's frame (vsr_trace_tiles; CUDA IPC
    mapping, NVLink peer stores from inside the kernel — the hit assembly is fused into the
    trace, no collective).  Two frame buffers: frame f+2 reuses frame f's buffer only after
    every rank has finished frame f (event + barrier), so the barrier of frame f overlaps the
    trace of frame f+1.  Time = max over ranks of F frames; value = frame rays / frame time.
    Inputs (1.06 GB rays, 1.1 GB scene) exceed L2, so no flush between frames."""
    import torch

    import workloads as W
    from paper_1912_12786_b200 import shard, vsr

    name = args.strong_config
    t0 = time.time()
    rays = W.rays_for(name)
    tile_rays = 64 * rays.spp
    if world > 1:
        base = (vsr.Scene.from_workload(W.scene(name), device=local).build(
            max_leaf_size=args.max_leaf, sah_bins=args.sah_bins) if rank == 0 else None)
        scene, _ = shard.broadcast_scene(base, local, dist,
                                         tensor_device=None if backend == "nccl" else "cpu")
    else:
        scene = vsr.Scene.from_workload(W.scene(name), device=local).build(
            max_leaf_size=args.max_leaf, sah_bins=args.sah_bins)
    n_frame = rays.n
    idx = shard.rank_ray_indices(n_frame, tile_rays, rank, world)
    d_rays = torch.from_numpy(np.ascontiguousarray(rays.data[idx])).cuda()
    rays = idx = None
    if world > 1:
        frames = [shard.PeerFrame(n_frame, local, dist) for _ in range(2)]
        ptrs = [f.ptr for f in frames]
    else:
        frames = [torch.empty((n_frame, 4), dtype=torch.float32, device="cuda") for _ in range(2)]
        ptrs = [f.data_ptr() for f in frames]
    setup_s = time.time() - t0
    stream = torch.cuda.current_stream()

    def frame(f):
        scene.trace_tiles(d_rays, tile_rays, rank, world, ptrs[f % 2], q, isect, stream=stream)

    def barrier():
        if world > 1:
            dist.barrier()

    for f in range(2):   # warm-up
        frame(f)
    torch.cuda.synchronize()
    barrier()
    F = max(4, args.strong_frames)
    done = [torch.cuda.Event() for _ in range(F)]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = vsr.launch_count()
    a.record(stream)
    for f in range(F):
        if f >= 2:
            done[f - 2].synchronize()   # this rank's frame f-2 is written ...
            barrier()                   # ... and every rank's: its buffer may be reused
        frame(f)
        done[f].record(stream)
    b.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = a.elapsed_time(b) / F
    launches = vsr.launch_count() - l0
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    out = {"workload": f"{name}: {W.CONFIGS[name]}", "rays_per_frame": n_frame,
           "tiles": n_frame // tile_rays, "tile_rays": tile_rays, "frames": F,
           "value": round(n_frame / (ms * 1e-3) / 1e6, 2), "unit": UNIT, "ms_per_frame": round(ms, 4),
           "scaling": "strong", "gpu_launches": int(launches), "setup_s": round(setup_s, 1),
           "assembly": ("fused: each trace kernel stores its hits into rank 0's frame (CUDA IPC, "
                        "NVLink peer stores), 2 frame buffers, event + barrier per frame")
           if world > 1 else "single rank: the frame traced in place (vsr_trace_tiles, world 1)",
           "l2": "not flushed (rays 1.06 GB + scene > L2)"}
    if rank == 0:   # the assembled frame equals one plain launch over the whole frame
        ref_rays = W.rays_for(name)
        dr = torch.from_numpy(ref_rays.data).cuda()
        del ref_rays
        ref, _ = scene.trace(dr, query=q, isect=isect)
        fr = frames[(F - 1) % 2].tensor() if world > 1 else frames[(F - 1) % 2]
        torch.cuda.synchronize()
        out["frame_bit_identical_to_single_launch"] = bool(torch.equal(
            ref.view(torch.int32), fr.view(torch.int32)))
        del dr, ref
    if world > 1:
        for fb in frames:
            fb.release(dist)
    scene.close()
    return out


def run_plumbing(args):
    """CPU launcher check (tests/test_bench_launcher.py): the N-rank path's host plumbing —
    rendezvous, the round-robin tile deal, frame assembly by all-gather, max-over-ranks —
    with NO tracing (the payload is each ray's frame index).  Prints one JSON line with
    n_gpus = world and whether the assembled frame equals the P = 1 frame; never a value."""
    import torch
    import torch.distributed as dist

    from paper_1912_12786_b200 import shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    n, tile = 64 * 8 * 3 * max(1, world), 64
    t0 = time.perf_counter()
    idx = shard.rank_ray_indices(n, tile, rank, world)
    local = torch.from_numpy(np.stack([idx.astype(np.float32)] * 4, axis=1))
    frame = shard.gather_hits(local, n, tile, dist) if world > 1 else local
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    same = bool(np.array_equal(frame[:, 0].numpy(), np.arange(n, dtype=np.float32)))
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world,
                          "plumbing": True, "rays": n, "frame_identical_to_p1": same,
                          "max_rank_s": round(float(dt.item()), 4)}))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def spawn_ranks(args):
    """`--gpus N` outside torchrun: re-launch this command as N ranks (one per GPU) with
    torch.distributed.run on 127.0.0.1; rank 0's JSON line is the output."""
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


# ---------------------------------------------------------------------------
# CPU oracle (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------
def _oracle_kind(name):
    import oracle
    base = name.replace("runtime_switch_", "").replace("runtime_fnptr_", "").replace("count_", "")
    return {"none": oracle.NONE, "default": oracle.DEFAULT, "alpha_texture": oracle.ALPHA_TEX,
            "alpha_procedural": oracle.ALPHA_PROC, "count": oracle.DEFAULT}[base]


def cpu_baseline(sc, rays, args, target_s=12.0, scene=None, gpu_hits=None):
    """Oracle S as it stands (brute force, all host cores) on a bounded seeded sample; with
    the headline frame's GPU hits it also reports a parity summary against the oracle on that
    sample and against walker C on the whole frame."""
    import oracle
    oq = oracle.CLOSEST if args.query == "closest" else oracle.ANY
    ok = _oracle_kind(args.isect)
    osc = oracle.OracleScene(sc)
    cores = host_cores()
    rng = np.random.default_rng(12345)
    probe = rays.data[rng.choice(rays.n, min(rays.n, 1024 * cores), replace=False)]  # oracle hands out 1024-ray chunks
    t0 = time.perf_counter()
    oracle.trace(osc, probe, oq, ok, nthreads=cores)
    per_ray = (time.perf_counter() - t0) / probe.shape[0]
    m = int(min(rays.n, max(256, target_s / max(per_ray, 1e-9))))
    for _ in range(4):   # re-calibrate until the sample takes about target_s
        idx = np.sort(rng.choice(rays.n, m, replace=False))
        sample = rays.data[idx]
        t0 = time.perf_counter()
        ref = oracle.trace(osc, sample, oq, ok, nthreads=cores)
        dt = time.perf_counter() - t0
        if dt >= 0.5 * target_s or m >= rays.n:
            break
        m = int(min(rays.n, m * target_s / max(dt, 1e-3)))
    out = {"value": round(m / dt / 1e6, 6), "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": f"{m} seeded rays of the {rays.n}-ray frame, brute force vs all "
                     f"{sc.num_tris} triangles, {dt:.1f} s", "cpu": cpu_model()}
    if scene is not None:
        # second, fairer CPU baseline: walker C, the contract BVH
        # traversal, over the product's exported BVH, the full frame on all cores
        from tests import bvh_check
        b = bvh_check.to_oracle(scene.export())
        oracle.walk(b, rays.data[: min(rays.n, 65536)], oq, ok, nthreads=cores)   # warm
        t0 = time.perf_counter()
        oracle.walk(b, rays.data, oq, ok, nthreads=cores)
        wdt = time.perf_counter() - t0
        out["walker"] = {"value": round(rays.n / wdt / 1e6, 3), "unit": UNIT, "cores": cores,
                         "kind": "oracle walker C (BVH traversal, CPU)",
                         "sample": f"full {rays.n}-ray frame, {wdt:.2f} s"}
    if gpu_hits is not None:
        # parity of the timed headline frame (the GPU hits of the last timed step)
        g = gpu_hits[idx]
        ghit, rhit = g["prim"] != 0xFFFFFFFF, ref["prim"] != 0xFFFFFFFF
        par = {"oracle_sample_rays": int(m), "hit_miss_mismatches": int((ghit != rhit).sum())}
        if oq == oracle.CLOSEST:
            same = (g.view(np.uint32).reshape(-1, 4) == ref.view(np.uint32).reshape(-1, 4)).all(axis=1)
            par["bit_exact_rays"] = int(same.sum())
            par["differing_rays"] = int((~same).sum())   # allowed only on exact t ties
        else:   # every returned any-hit: prim in the accepted set, its (t, u, v) bit-equal
            hi = np.nonzero(ghit)[0]
            acc, e = oracle.eval_pairs(osc, sample[hi], g["prim"][hi], ok)
            gi = g[hi]
            good = acc & (e["t"] == gi["t"]) & (e["u"] == gi["u"]) & (e["v"] == gi["v"])
            par["any_hit_checked"] = int(hi.size)
            par["any_hit_invalid"] = int((~good).sum())
        if scene is not None:
            wh, _ = oracle.walk(b, rays.data, oq, ok, nthreads=cores)
            par["walker_full_frame_bit_exact"] = bool(np.array_equal(wh.view(np.uint32),
                                                                     gpu_hits.view(np.uint32)))
        out["parity"] = par
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    oracle.build()
    sc, rays = make_workload(args.config, 0)
    oq = oracle.CLOSEST if args.query == "closest" else oracle.ANY
    ok = _oracle_kind(args.isect)
    osc = oracle.OracleScene(sc)
    cores = host_cores()
    rng = np.random.default_rng(777)
    probe = rays.data[rng.choice(rays.n, min(rays.n, 1024 * cores), replace=False)]  # oracle hands out 1024-ray chunks
    t0 = time.perf_counter()
    oracle.trace(osc, probe, oq, ok, nthreads=cores)
    per_ray = (time.perf_counter() - t0) / probe.shape[0]
    budget = 150.0 / max(1, args.steps + args.warmup)       # whole run ~2.5 min
    m = int(min(rays.n, max(128, budget / max(per_ray, 1e-9))))
    times = []
    for step in range(args.warmup + args.steps):
        idx = np.sort(rng.choice(rays.n, m, replace=False))
        sample = rays.data[idx]
        t0 = time.perf_counter()
        oracle.trace(osc, sample, oq, ok, nthreads=cores)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
    ms = float(np.mean(times)) * 1e3
    value = m / (ms * 1e-3) / 1e6
    line = {"metric": METRIC, "value": round(value, 6), "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded generators, workloads/)", "impl": "reference",
            "config": {**config_desc(args.config), "query": args.query, "intersector": args.isect,
                       "rays_per_step": m, "triangles": sc.num_tris},
            "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{m} seeded rays per step of the {rays.n}-ray frame, brute "
                                       f"force vs {sc.num_tris} triangles", "cpu": cpu_model()},
            "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.plumbing:
        run_plumbing(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_own(args)


if __name__ == "__main__":
    main()
