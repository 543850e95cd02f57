import os, sys, statistics, torch
sys.path.insert(0, "/root/repo")
import synth
from paper_2603_07904_b200 import dyq
dev = "cuda:0"; M = 8; C = 8
lins = synth.LLAMA_BLOCK_LINEARS
packed = [[dyq.PackedLinear.from_bf16(synth.weights_bf16_torch(N, K, seed=1 + 4 * c + i, device=dev), group=64, wbits=4)
           for i, (_, N, K) in enumerate(lins)] for c in range(C)]
xs = [synth.activations_bf16_torch(M, K, seed=1000 + i, device=dev) for i, (_, _, K) in enumerate(lins)]
ys = [torch.empty(M, N, dtype=torch.bfloat16, device=dev) for (_, N, _) in lins]
wss = [packed[0][i].workspace(M) for i in range(len(lins))]
def step(c, bits=4):
    for i in range(len(lins)):
        p = packed[c][i]
        dyq.qlinear(p.wd, p.codes, p.meta, xs[i], M, None, bits, ys[i], 1, wss[i])
for c in range(C): step(c)
torch.cuda.synchronize()
ref = [y.clone() for y in ys]  # copy C-1 results
# (1) big graph: R steps rotating copies
def graph_of(steps):
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        for r in steps: step(r % C)
    g.replay(); torch.cuda.synchronize(); return g
def tgraph(g, n=5):
    out = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize(); out.append(e0.elapsed_time(e1))
    return statistics.median(out)
for R in (8, 64, 400):
    g = graph_of(range(R)); print(f"graph of {R} steps: {tgraph(g) / R * 1e3:.2f} us/step"); del g
# (2) per-copy single-step graphs replayed back to back (no sync) and with sync
gs = [graph_of([c]) for c in range(C)]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for t in range(400): gs[t % C].replay()
e1.record(); torch.cuda.synchronize(); print(f"400 single-step graph replays, no sync: {e0.elapsed_time(e1) / 400 * 1e3:.2f} us/step")
import time
tc = time.perf_counter()
for t in range(200):
    gs[t % C].replay(); torch.cuda.current_stream().synchronize()
print(f"200 single-step replays with sync (wall): {(time.perf_counter() - tc) / 200 * 1e6:.2f} us/step")
print("results equal to eager:", all(torch.equal(a, b) for a, b in zip(ref, ys)))
