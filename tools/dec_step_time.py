"""Block decode step timing (the bench's configs[1] step without the selector):
4 Llama-2-7B block linears at M tokens and fixed activation bits, rotating C
packed block copies (> L2), CUDA graph of R steps, median of 5 replays.
usage: python tools/dec_step_time.py [M] [bits] [wbits] [G] [C] [R]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_07904_b200 import dyq  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 8
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 4
WB = int(sys.argv[3]) if len(sys.argv) > 3 else 4
G = int(sys.argv[4]) if len(sys.argv) > 4 else 64
C = int(sys.argv[5]) if len(sys.argv) > 5 else 8
R = int(sys.argv[6]) if len(sys.argv) > 6 else 64
dev = "cuda:0"
lins = synth.LLAMA_BLOCK_LINEARS
blk = [[dyq.PackedLinear.from_bf16(synth.weights_bf16_torch(N, K, seed=1 + 4 * c + i, device=dev), group=G, wbits=WB)
        for i, (_, N, K) in enumerate(lins)] for c in range(C)]
xs = [synth.activations_bf16_torch(M, K, seed=100 + i, device=dev) for i, (_, N, K) in enumerate(lins)]
ys = [torch.empty(M, N, dtype=torch.bfloat16, device=dev) for _, N, K in lins]
wss = [blk[0][i].workspace(M) for i in range(len(lins))]


def step(t):
    for i in range(len(lins)):
        p = blk[t % C][i]
        dyq.qlinear(p.wd, p.codes, p.meta, xs[i], M, None, bits, ys[i], 1, wss[i])


for t in range(2 * C):
    step(t)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.graph(g, stream=s):
    for t in range(R):
        step(t)
g.replay()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / R)
ms = statistics.median(ts)
nbytes = sum(N * K * WB // 8 + (N * K // G) * 5 + M * K * 2 + M * N * 2 for _, N, K in lins)
print(f"decode block M={M} A{bits} W{WB} G{G}: {ms * 1e3:.2f} us/step  {nbytes / ms / 1e6:.1f} GB/s")
