"""Split one decode qlinear into its parts: act-quant alone, decode kernel alone
(pre-quantized activations, dyq_qlinear_q), the full call, and an empty-kernel
graph for the launch floor.  usage: python tools/prof_parts.py [linear] [M]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_07904_b200 import dyq  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "o"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 8
N, K = {n: (N, K) for n, N, K in synth.LLAMA_BLOCK_LINEARS}[name]
dev = "cuda:0"
lins = [dyq.PackedLinear.from_bf16(synth.weights_bf16_torch(N, K, seed=1 + c, device=dev), group=64, wbits=4)
        for c in range(4)]
x = synth.activations_bf16_torch(M, K, seed=1000, device=dev)
y = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
ws = lins[0].workspace(M)
R = 40


def timed(fn):
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        for r in range(R):
            fn(r)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / R * 1e3


p0 = lins[0]
full = timed(lambda r: dyq.qlinear(lins[r % 4].wd, lins[r % 4].codes, lins[r % 4].meta, x, M, None, 4, y, 1, ws))
aq = timed(lambda r: dyq.act_quant(p0.wd, x, M, None, 4, ws))
dq = timed(lambda r: dyq.qlinear_q(lins[r % 4].wd, lins[r % 4].codes, lins[r % 4].meta, x, M, None, 4, y, 1, ws))
z = torch.zeros(1, device=dev)
empty = timed(lambda r: z.add_(1))
b = N * K // 2 + N * (K // 64) * 5
print(f"{name} M={M}: full {full:.2f} us | act_quant {aq:.2f} | decode-only {dq:.2f} ({b / dq / 1e3:.0f} GB/s) | "
      f"empty kernel {empty:.2f} us | weights {b / 1e6:.1f} MB -> {b / 6.45e6:.2f} us at 6.45 TB/s")
