"""Back-to-back dyq_select_route calls in a CUDA graph (E episodes): per-call
time of the selection kernel alone, and one bench-style step with and without it."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_07904_b200 import dyq  # noqa: E402

dev = "cuda:0"
for E in (1, 8, 64):
    cal = dyq.default_calib()
    st = torch.zeros(dyq.state_size(E, cal), dtype=torch.uint8, device=dev)
    dyq.state_init(E, cal, st)
    a = torch.rand(300, E, 7, device=dev) * 0.1
    bits = torch.zeros(E, dtype=torch.int32, device=dev)
    rb = torch.zeros(E * 8, dtype=torch.int32, device=dev)
    for t in range(300):  # fill the histories (p95 over H = 256)
        dyq.select_route(st, E, a[t], bits, 8, rb)
    torch.cuda.synchronize()
    R = 200
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        for i in range(R):
            dyq.select_route(st, E, a[i % 300], bits, 8, rb, stream=s)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / R * 1e3)
    print(f"E={E}: select_route {statistics.median(ts):.2f} us/call")
