"""Per-CTA timeline of the persistent prefill kernel from the %globaltimer
trace (dyq_trace_enable, kernel id 4).  Runs R back-to-back qlinear calls of
one Llama linear (act-quant + prefill, as in the block step) inside a CUDA
graph with tracing on, then prints per prefill launch (relative to the first
CTA entry of that launch, us): CTA entry spread, promotion past
griddepcontrol.wait, first accumulator ready, first / last segment end,
epilogue + reducer wait, CTA exit.
usage: python tools/trace_prefill.py [linear] [M] [bits] [R]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_07904_b200 import dyq  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "gate_up"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 288
bits = int(sys.argv[3]) if len(sys.argv) > 3 else 4
R = int(sys.argv[4]) if len(sys.argv) > 4 else 3
N, K = {n: (N, K) for n, N, K in synth.LLAMA_BLOCK_LINEARS}[name]
dev = "cuda:0"
ps = [dyq.PackedLinear.from_bf16(synth.weights_bf16_torch(N, K, seed=1 + c, device=dev), group=64, wbits=4)
      for c in range(2)]
x = synth.activations_bf16_torch(M, K, seed=1000, device=dev)
y = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
ws = ps[0].workspace(M)
for _ in range(3):
    dyq.qlinear(ps[0].wd, ps[0].codes, ps[0].meta, x, M, None, bits, y, 1, ws)
torch.cuda.synchronize()
tr = torch.zeros(1 << 20, dtype=torch.int64, device=dev)
dyq.trace_enable(tr)
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.graph(g, stream=s):
    for r in range(R):
        p = ps[r % 2]
        dyq.qlinear(p.wd, p.codes, p.meta, x, M, None, bits, y, 1, ws)
dyq.trace_enable(None)
torch.cuda.synchronize()
tr.zero_()
tr[1] = (tr.numel() * 8 - 16) // 16
g.replay()
torch.cuda.synchronize()
t = tr.cpu().numpy().view(np.uint64)
n = int(t[0])
rec = t[2:2 + 2 * n].reshape(-1, 2)
tag, ns = rec[:, 0], rec[:, 1].astype(np.int64)
serial = (tag >> 32).astype(np.int64)
kern = ((tag >> 24) & 0xff).astype(np.int64)
ev = ((tag >> 16) & 0xff).astype(np.int64)
cta = (tag & 0xffff).astype(np.int64)
sel = kern == 4
t0g = ns[sel].min() if sel.any() else 0
prev_end = None
for sr in sorted(set(serial[sel].tolist())):
    m = sel & (serial == sr)
    base = ns[m & (ev == 0)].min()

    def q(e, f=np.median):
        v = ns[m & (ev == e)]
        return f(v - base) / 1e3 if len(v) else float("nan")
    e4 = ns[m & (ev == 4)]
    e3 = ns[m & (ev == 3)]
    line = (f"launch {sr}: start {(base - t0g) / 1e3:8.1f}  gap {(base - prev_end) / 1e3 if prev_end else 0:6.1f} | "
            f"entry spread {q(0, np.max):6.1f}  pdl-wait done {q(1):6.1f}  first acc {q(2):6.1f} / max {q(2, np.max):6.1f} | "
            f"seg end med {q(3):6.1f}  epi done med {q(4):6.1f}  max {q(4, np.max):6.1f} | exit max {q(5, np.max):6.1f}")
    print(line)
    # epilogue cost per segment (ev4 - ev3 pairs, per CTA in order)
    d = []
    for c in set(cta[m].tolist()):
        a3 = np.sort(ns[m & (ev == 3) & (cta == c)])
        a4 = np.sort(ns[m & (ev == 4) & (cta == c)])
        d += list((a4 - a3)[: min(len(a3), len(a4))])
    if d:
        d = np.array(d) / 1e3
        print(f"           epilogue (ev4 - ev3) per segment: median {np.median(d):.2f} us, max {d.max():.2f} us, "
              f"n {len(d)}")
    prev_end = ns[m & (ev == 5)].max()
