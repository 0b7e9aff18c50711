"""Fixed cost of the bench's timing scheme (events around a graph replay after an L2 flush)
for graphs of 1..3 empty kernels (development tool)."""
import torch
import numpy as np

dev = torch.device("cuda:0")
x = torch.zeros(1, device=dev)
flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)
for nk in (1, 2, 3):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(nk):
            x.add_(1)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(nk):
            x.add_(1)
    for flushed in (False, True):
        ts = []
        for i in range(60):
            if flushed:
                flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            e1.synchronize()
            if i >= 10:
                ts.append(e0.elapsed_time(e1) * 1e3)
        print(f"{nk} kernel(s), flush={flushed}: median {np.median(ts):.2f} us")
