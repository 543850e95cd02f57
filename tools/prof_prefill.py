"""Prefill qlinear timing (tcgen05 path): one Llama linear at M tokens.

usage: python tools/prof_prefill.py [gate_up|qkv|o|down|block] [M] [wbits] [bits] [G]
Prints us/launch, int TOPS and the fraction of nominal dense int8 (4.5 POPS).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_07904_b200 import dyq  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "gate_up"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 288
WB = int(sys.argv[3]) if len(sys.argv) > 3 else 4
bits = int(sys.argv[4]) if len(sys.argv) > 4 else 4
G = int(sys.argv[5]) if len(sys.argv) > 5 else 64
dev = "cuda:0"
shapes = {n: (N, K) for n, N, K in synth.LLAMA_BLOCK_LINEARS}
names = list(shapes) if name == "block" else [name]
lins, xs, ys, wss = [], [], [], []
for i, n in enumerate(names):
    N, K = shapes[n]
    w = synth.weights_bf16_torch(N, K, seed=1 + i, device=dev)
    lin = dyq.PackedLinear.from_bf16(w, group=G, wbits=WB)
    del w
    lins.append(lin)
    xs.append(synth.activations_bf16_torch(M, K, seed=1000 + i, device=dev))
    ys.append(torch.empty(M, N, dtype=torch.bfloat16, device=dev))
    wss.append(lin.workspace(M))
for _ in range(3):
    for lin, x, y, ws in zip(lins, xs, ys, wss):
        dyq.qlinear(lin.wd, lin.codes, lin.meta, x, M, None, bits, y, 1, ws)
torch.cuda.synchronize()
R = int(os.environ.get("PROF_R", "10"))
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.graph(g, stream=s):
    for _ in range(R):
        for lin, x, y, ws in zip(lins, xs, ys, wss):
            dyq.qlinear(lin.wd, lin.codes, lin.meta, x, M, None, bits, y, 1, ws)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / R
ops = sum(2 * M * shapes[n][0] * shapes[n][1] for n in names)
tops = ops / (ms * 1e-3) / 1e12
print(f"prefill {name} M={M} W{WB} A{bits} G{G}: {ms * 1e3:.1f} us/pass  {tops:.1f} int TOPS  "
      f"{tops / 4500 * 100:.1f}% of 4.5 POPS nominal")
