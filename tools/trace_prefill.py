"""Per-group pipeline timeline of the prefill kernel, CTA (0,0), from the
non-blocking trace (dyq_trace_enable; buffer slots 16 + 512 ev + g).
usage: python tools/build_variant.py trace -DDYQ_PREFILL_TRACE=1
       DYQ_LIB=tools/variants/libdyq_trace.so python tools/trace_prefill.py [linear] [M] [bits]
(the product build compiles the per-group hooks out; DYQ_PRE_E4M3=1 for the e4m3 path)"""
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
N, K = {n: (N, K) for n, N, K in synth.LLAMA_BLOCK_LINEARS}[name]
dev = "cuda:0"
p = dyq.PackedLinear.from_bf16(synth.weights_bf16_torch(N, K, seed=1, device=dev), group=64, wbits=4)
x = synth.activations_bf16_torch(M, K, seed=1000, device=dev)
y = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
ws = p.workspace(M)
for _ in range(3):
    dyq.qlinear(p.wd, p.codes, p.meta, x, M, None, bits, y, 1, ws)
torch.cuda.synchronize()
tr = torch.zeros(1 << 14, dtype=torch.int64, device=dev)
dyq.trace_enable(tr)
dyq.qlinear(p.wd, p.codes, p.meta, x, M, None, bits, y, 1, ws)
torch.cuda.synchronize()
dyq.trace_enable(None)
raw = tr.cpu().numpy().astype(np.int64)
NG = K // 64
ev = {e: raw[16 + 512 * e: 16 + 512 * e + NG] for e in range(1, 8)}
t0 = ev[1].min()
names = {1: "issued", 2: "B_landed", 3: "A_ready", 4: "acc_free", 5: "xf_done", 6: "pr_start", 7: "pr_done"}
print("group " + " ".join(f"{names[e]:>9}" for e in range(1, 8)) + "   (us, CTA (0,0))")
for g in list(range(8)) + list(range(NG - 4, NG)):
    print(f"{g:5d} " + " ".join(f"{(ev[e][g] - t0) / 1e3:9.2f}" for e in range(1, 8)))
d = lambda a, b: np.median((ev[b][8:] - ev[a][8:]) / 1e3)  # noqa: E731
print(f"median per group: cadence {np.median(np.diff(ev[6][8:])) / 1e3:.3f} us; acc_free->pr_start (MMA+commit) "
      f"{d(4, 6):.3f}; pr_start->pr_done {d(6, 7):.3f}; B_landed-issued {d(1, 2):.3f}")
