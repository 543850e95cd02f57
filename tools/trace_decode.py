"""Timeline of the decode path from the %globaltimer trace (dyq_trace_enable).

Runs a CUDA graph of R block steps (QKV, o, gate|up, down at M=8, fixed bits)
on rotating weight copies, replays it once with tracing on and prints per
kernel launch: start of first CTA, consumers' first data, end of last CTA
(relative us), so launch gaps and per-call fixed costs are visible.
usage: python tools/trace_decode.py [bits] [R]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_07904_b200 import dyq  # noqa: E402

bits = int(sys.argv[1]) if len(sys.argv) > 1 else 4
R = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = "cuda:0"
lins = synth.LLAMA_BLOCK_LINEARS
C = 3
packed = [[dyq.PackedLinear.from_bf16(synth.weights_bf16_torch(N, K, seed=1 + 4 * c + i, device=dev), group=64, wbits=4)
           for i, (_, N, K) in enumerate(lins)] for c in range(C)]
xs = [synth.activations_bf16_torch(8, K, seed=1000 + i, device=dev) for i, (_, _, K) in enumerate(lins)]
ys = [torch.empty(8, N, dtype=torch.bfloat16, device=dev) for (_, N, _) in lins]
wss = [packed[0][i].workspace(8) for i in range(len(lins))]


PF = int(os.environ.get("PF", "0"))


side = torch.cuda.Stream()


def step(r):
    cur = torch.cuda.current_stream()
    for i in range(len(lins)):
        p = packed[r % C][i]
        nxt = packed[(r + (i + 1) // len(lins)) % C][(i + 1) % len(lins)]
        if PF == 1:  # prefetch the next linear's weights into L2 (same stream)
            nxt.prefetch_l2()
        elif PF == 2:  # ... on a side stream forked here (off the dependency chain)
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                nxt.prefetch_l2()
        dyq.qlinear(p.wd, p.codes, p.meta, xs[i], 8, None, bits, ys[i], 1, wss[i])
    if PF == 2:
        cur.wait_stream(side)


for r in range(3):
    step(r)
torch.cuda.synchronize()
tr = torch.zeros(1 << 22, dtype=torch.int64, device=dev)
dyq.trace_enable(tr)
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.graph(g, stream=s):
    for r in range(R):
        step(r)
torch.cuda.synchronize()
dyq.trace_enable(None)
for rep in range(2):
    tr[0] = 0
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
ev = dyq.trace_read(tr)
t0 = min(e[4] for e in ev)
by = {}
for ser, k, e, b, t in ev:
    by.setdefault((ser, k), {}).setdefault(e, []).append((t - t0) / 1e3)
names = {1: "decode", 2: "actq", 3: "pf"}
lin_names = [n for n, _, _ in lins]
prev_end = None
print(f"{'launch':>16} {'start0':>8} {'startN':>8} {'pdl_ok':>8} {'data0':>8} {'issued':>8} {'end0':>8} {'endN':>8}")
for idx, key in enumerate(sorted(by, key=lambda k: min(min(v) for v in by[k].values()))):
    d = by[key]
    f = lambda e, fn: fn(d[e]) if e in d else float('nan')  # noqa: E731
    nm = names.get(key[1], key[1])
    if key[1] == 1:
        print(f"{nm:>8}#{key[0]:<7} {f(0, min):8.2f} {f(0, max):8.2f} {f(1, max):8.2f} {f(3, max):8.2f} "
              f"{f(2, max):8.2f} {f(4, min):8.2f} {f(4, max):8.2f}")
    else:
        print(f"{nm:>8}#{key[0]:<7} {f(0, min):8.2f} {f(0, max):8.2f} {f(1, max):8.2f} {'':>8} {'':>8} "
              f"{f(2, min):8.2f} {f(2, max):8.2f}")
tot = max(e[4] for e in ev) - t0
print(f"total {tot / 1e3:.2f} us for {R} block steps -> {tot / 1e3 / R:.2f} us/step")
if os.environ.get("PERCTA"):
    ser = int(os.environ["PERCTA"])
    rows = {}
    for s_, k, e, b, t in ev:
        if s_ == ser and k == 1:
            rows.setdefault(b, {})[e] = (t - t0) / 1e3
    ends = sorted(rows.items(), key=lambda kv: kv[1].get(4, 0))
    print("per-CTA (block: start, pdl, data0, issued, spin0, spin1, end) for serial", ser)
    for b, d in ends[:5] + ends[-12:]:
        print(b, [round(d.get(e, -1), 2) for e in (0, 1, 3, 2, 5, 6, 4)])
