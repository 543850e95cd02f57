"""Time the fused TP decode epilogue on one GPU (simulated ranks): a Llama-2
gate|up shard (N/P x 4096, M = 8, W4A4) through dyq_qlinear, dyq_qlinear_tp
(P output copies + flags) + dyq_tp_wait, and dyq_qlinear + NCCL world-1
all-gather.  CUDA graphs of R calls, events on the capture stream."""
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2603_07904_b200 import dyq  # noqa: E402

dev = "cuda:0"
N, K, M, R = 22016, 4096, 8, 32


def graph_ms(fn):
    fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        for i in range(R):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    out = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / R * 1e3)
    return statistics.median(out)


res = {}
x = torch.from_numpy(synth.activations_bf16(M, K, seed=3).view(np.int16)).to(dev)
for P in (1, 2, 8):
    Ns = N // P
    # 4 distinct shard copies so consecutive calls do not hit L2
    lins = [dyq.PackedLinear.from_bf16(torch.from_numpy(synth.weights_bf16(Ns, K, seed=10 + c).view(np.int16)).to(dev))
            for c in range(4)]
    ws = lins[0].workspace(M)
    y = torch.empty(M, Ns, dtype=torch.bfloat16, device=dev)
    t_plain = graph_ms(lambda i: dyq.qlinear(lins[i % 4].wd, lins[i % 4].codes, lins[i % 4].meta, x, M, None, 4, y, 1,
                                             ws))
    ys = [[torch.empty(M, N, dtype=torch.int16, device=dev) for _ in range(P)] for _ in range(2)]
    flags = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(P)]
    cnt = [0]

    def fused(i):
        s = i % 2
        peers = dyq.tp_peers(P, 0, [t.data_ptr() for t in ys[s]], [f.data_ptr() for f in flags])
        dyq.qlinear_tp(lins[i % 4], x, M, None, 4, peers, ws)
    t_fused = graph_ms(fused)
    res[P] = {"Ns": Ns, "qlinear_us": round(t_plain, 2), "qlinear_tp_us (P stores + flags)": round(t_fused, 2)}
comm = dyq.Comm(dyq.comm_unique_id(), 0, 1)
lin = dyq.PackedLinear.from_bf16(torch.from_numpy(synth.weights_bf16(N, K, seed=9).view(np.int16)).to(dev))
ws = lin.workspace(M)
ysh = torch.empty(M, N, dtype=torch.int16, device=dev)
yf = torch.empty_like(ysh)
gb = torch.empty_like(ysh)


def nccl(i):
    dyq.qlinear(lin.wd, lin.codes, lin.meta, x, M, None, 4, ysh, 1, ws)
    comm.allgather(ysh, M, N, gb, yf)


try:
    res["nccl_world1_us"] = round(graph_ms(nccl), 2)
except Exception as e:  # NCCL graph capture may be unavailable
    res["nccl_world1_us"] = f"n/a ({e})"
print(res)
