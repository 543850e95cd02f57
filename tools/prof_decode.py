"""Minimal driver for ncu: one Llama linear at decode, a few launches.

usage: python tools/prof_decode.py [gate_up|qkv|o|down] [M] [wbits] [bits] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_07904_b200 import dyq  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "gate_up"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 8
WB = int(sys.argv[3]) if len(sys.argv) > 3 else 4
bits = int(sys.argv[4]) if len(sys.argv) > 4 else 4
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 6
N, K = dict({n: (N, K) for n, N, K in synth.LLAMA_BLOCK_LINEARS}, tiny=(128, 128), small=(4096, 512))[name]
dev = "cuda:0"
copies = 4
lins = []
for c in range(copies):
    w = synth.weights_bf16_torch(N, K, seed=1 + c, device=dev)
    lins.append(dyq.PackedLinear.from_bf16(w, group=64, wbits=WB))
    del w
x = synth.activations_bf16_torch(M, K, seed=1000, device=dev)
y = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
ws = lins[0].workspace(M)
p = lins[0]
for r in range(reps):
    p = lins[r % copies]
    dyq.qlinear(p.wd, p.codes, p.meta, x, M, None, bits, y, 1, ws)
torch.cuda.synchronize()
# timing without the profiler: one CUDA graph of R launches (rotating copies)
R = int(os.environ.get('PROF_R', '40'))
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.graph(g, stream=s):
    for r in range(R):
        p = lins[r % copies]
        dyq.qlinear(p.wd, p.codes, p.meta, x, M, None, bits, y, 1, ws)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / R
b = N * K * WB // 8 + N * (K // 64) * 5 + M * K * 2 + M * N * 2
print(f"{name} M={M} W{WB} A{bits}: {ms * 1e3:.2f} us/launch  {b / ms / 1e6:.1f} GB/s (graph of 40 back-to-back launches)")
