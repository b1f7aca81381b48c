"""H2D DMA rate of pinned X (1024 x 1000 fp64) by copy shape: linear, row ranges, 2D column
blocks of a row range.  Device-timed with events on the copy stream (tuning aid for the host
evaluation path)."""
import numpy as np
import torch
import cuda.bindings.runtime as rt

P, D = 1024, 1000
Xh = torch.empty((P, D), dtype=torch.float64).pin_memory()
Xd = torch.empty((P, D), dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
h = s.cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
H2D = rt.cudaMemcpyKind.cudaMemcpyHostToDevice


def timed(fn, reps=60):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0.record(s)
        fn()
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts[10:]))


def lin(r0, r1):
    rt.cudaMemcpyAsync(Xd.data_ptr() + r0 * D * 8, Xh.data_ptr() + r0 * D * 8, (r1 - r0) * D * 8, H2D, h)


def blk(r0, r1, c0, c1):
    rt.cudaMemcpy2DAsync(Xd.data_ptr() + (r0 * D + c0) * 8, D * 8, Xh.data_ptr() + (r0 * D + c0) * 8, D * 8,
                         (c1 - c0) * 8, r1 - r0, H2D, h)


def report(name, us, nbytes):
    print(f"{name:48s} {us:8.1f} us  {nbytes / us / 1e3:6.1f} GB/s", flush=True)


report("linear all", timed(lambda: lin(0, P)), P * D * 8)
report("linear 576 rows", timed(lambda: lin(0, 576)), 576 * D * 8)
report("linear 64 rows", timed(lambda: lin(0, 64)), 64 * D * 8)
for rows in (1024, 576, 448):
    for w in (1000, 512, 256, 128, 64, 32):
        def f(rows=rows, w=w):
            c = 0
            while c < D:
                blk(0, rows, c, min(D, c + w))
                c += w
        report(f"2D {rows} rows in {w}-col blocks", timed(f), rows * D * 8)
for rows in (1024, 576):
    report(f"2D one block {rows} x 256", timed(lambda rows=rows: blk(0, rows, 0, 256)), rows * 256 * 8)

# two copy streams (two DMA engines) sharing each block: rows split in halves
s2 = torch.cuda.Stream()
h2 = s2.cuda_stream
ev_a, ev_b = torch.cuda.Event(), torch.cuda.Event()


def blk_on(hh, r0, r1, c0, c1):
    rt.cudaMemcpy2DAsync(Xd.data_ptr() + (r0 * D + c0) * 8, D * 8, Xh.data_ptr() + (r0 * D + c0) * 8, D * 8,
                         (c1 - c0) * 8, r1 - r0, H2D, hh)


def two_streams(rows, w, split):
    ev_a.record(s)
    s2.wait_event(ev_a)
    c = 0
    while c < D:
        c1 = min(D, c + w)
        if split == "rows":
            blk_on(h, 0, rows // 2, c, c1)
            blk_on(h2, rows // 2, rows, c, c1)
        else:  # alternate whole blocks between the engines
            blk_on(h if (c // w) % 2 == 0 else h2, 0, rows, c, c1)
        c = c1
    ev_b.record(s2)
    s.wait_event(ev_b)


for rows in (1024, 576):
    for w in (512, 256, 128):
        for split in ("rows", "alt"):
            report(f"2 streams {split}: {rows} rows in {w}-col blocks",
                   timed(lambda rows=rows, w=w, split=split: two_streams(rows, w, split)), rows * D * 8)


def lin2():
    ev_a.record(s)
    s2.wait_event(ev_a)
    rt.cudaMemcpyAsync(Xd.data_ptr(), Xh.data_ptr(), 512 * D * 8, H2D, h)
    rt.cudaMemcpyAsync(Xd.data_ptr() + 512 * D * 8, Xh.data_ptr() + 512 * D * 8, 512 * D * 8, H2D, h2)
    ev_b.record(s2)
    s.wait_event(ev_b)


report("2 streams linear halves", timed(lin2), P * D * 8)
report("linear all, 2 copies of 512 rows one stream", timed(lambda: (lin(0, 512), lin(512, P))), P * D * 8)
