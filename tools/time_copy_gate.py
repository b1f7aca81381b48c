"""Copy-stream timing for the gated host path: 4 column-chunk 2D copies of X (1024 x 1000 fp64,
pinned) alone, with stream value writes between them, and next to a busy fp64 kernel."""
import time
import numpy as np, torch
import cuda.bindings.runtime as rt
import cuda.bindings.driver as drv
Xh = torch.empty((1024, 1000), dtype=torch.float64).pin_memory()
Xd = torch.empty((1024, 1000), dtype=torch.float64, device="cuda")
gate = torch.zeros(8, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream(); h = s.cuda_stream
busy_s = torch.cuda.Stream()
A = torch.randn(2048, 2048, dtype=torch.float64, device="cuda")
ep = torch.arange(1, 9, dtype=torch.int32).pin_memory()
g2 = torch.cuda.Stream(); h2 = g2.cuda_stream
evs = [rt.cudaEventCreateWithFlags(rt.cudaEventDisableTiming)[1] for _ in range(8)]
def run(n, writes, busy, linear=False):
    ts = []
    for it in range(80):
        torch.cuda.synchronize()
        if busy:
            with torch.cuda.stream(busy_s):
                for _ in range(2): A @ A
        t = time.perf_counter()
        cols = -(-(-(-1000 // n)) // 16) * 16
        c0, c = 0, 0
        while c0 < 1000:
            w = min(cols, 1000 - c0)
            if linear:
                rt.cudaMemcpyAsync(Xd.data_ptr() + c0 * 8 * 1024, Xh.data_ptr() + c0 * 8 * 1024, w * 8 * 1024,
                                   rt.cudaMemcpyKind.cudaMemcpyHostToDevice, h)
            else:
                rt.cudaMemcpy2DAsync(Xd.data_ptr() + c0 * 8, 8000, Xh.data_ptr() + c0 * 8, 8000, w * 8, 1024,
                                     rt.cudaMemcpyKind.cudaMemcpyHostToDevice, h)
            if writes == 2:  # the copy engine writes the gate: 4-byte H2D after the chunk
                rt.cudaMemcpyAsync(gate.data_ptr() + 4 * c, ep.data_ptr() + 4 * c, 4, rt.cudaMemcpyKind.cudaMemcpyHostToDevice, h)
            elif writes == 3:  # event after the chunk, the write on a side stream
                rt.cudaEventRecord(evs[c], h)
                rt.cudaStreamWaitEvent(h2, evs[c], 0)
                drv.cuStreamWriteValue32(drv.CUstream(h2), drv.CUdeviceptr(gate.data_ptr() + 4 * c), it + 1, 0)
            elif writes:
                drv.cuStreamWriteValue32(drv.CUstream(h), drv.CUdeviceptr(gate.data_ptr() + 4 * c), it + 1, 0)
            c0 += w; c += 1
        s.synchronize(); g2.synchronize(); ts.append(time.perf_counter() - t)
    return np.median(ts[10:]) * 1e6
for n in (1, 2, 4, 8):
    print(f"{n} chunks: 2D {run(n,0,0):.0f}  2D+writes {run(n,1,0):.0f}  2D+4B-copy {run(n,2,0):.0f}  2D+event/side-write {run(n,3,0):.0f} us")
