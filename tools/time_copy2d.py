"""H2D time of X (1024 x 1000 fp64, pinned) copied whole vs in n column chunks (2D copies)."""
import time
import numpy as np, torch
import cuda.bindings.runtime as rt
Xh = torch.empty((1024, 1000), dtype=torch.float64).pin_memory()
Xd = torch.empty((1024, 1000), dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
h = s.cuda_stream
for n in (1, 2, 4, 8, 16):
    cols = -(-1000 // n); cols = -(-cols // 16) * 16
    ts = []
    for it in range(120):
        torch.cuda.synchronize(); t = time.perf_counter()
        c0 = 0
        while c0 < 1000:
            w = min(cols, 1000 - c0)
            rt.cudaMemcpy2DAsync(Xd.data_ptr() + c0 * 8, 8000, Xh.data_ptr() + c0 * 8, 8000, w * 8, 1024,
                                 rt.cudaMemcpyKind.cudaMemcpyHostToDevice, h)
            c0 += w
        s.synchronize(); ts.append(time.perf_counter() - t)
    print(n, "chunks: med us", round(np.median(ts[20:]) * 1e6, 1))
