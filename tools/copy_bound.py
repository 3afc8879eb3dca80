"""Host<->device copy bounds for the end-to-end path (vsr_trace_host): pinned H2D of a frame's
rays, D2H of its hits, and both at once on two streams, CUDA events, median of 20.

    python tools/copy_bound.py [rays]        (default 2073600 = C2 1080p)
"""
import statistics
import sys

import torch


def timed(fn, reps=20):
    ts = []
    for _ in range(reps + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts[3:])


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2073600
    hin = torch.empty(n * 32, dtype=torch.uint8).pin_memory()
    hout = torch.empty(n * 16, dtype=torch.uint8).pin_memory()
    din = torch.empty(n * 32, dtype=torch.uint8, device="cuda")
    dout = torch.empty(n * 16, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            din.copy_(hin, non_blocking=True)
        with torch.cuda.stream(s2):
            hout.copy_(dout, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    h2d = timed(lambda: din.copy_(hin, non_blocking=True))
    d2h = timed(lambda: hout.copy_(dout, non_blocking=True))
    bi = timed(both)
    print(f"rays {n}: H2D {n*32/1e6:.1f} MB {h2d:.4f} ms ({n*32/h2d/1e6:.1f} GB/s); "
          f"D2H {n*16/1e6:.1f} MB {d2h:.4f} ms ({n*16/d2h/1e6:.1f} GB/s); "
          f"both concurrently {bi:.4f} ms -> e2e bound {n/bi/1e3:.1f} Mrays/s")


if __name__ == "__main__":
    main()
