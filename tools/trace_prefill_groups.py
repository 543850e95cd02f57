"""Per-group pipeline stamps of CTA 0 of the persistent prefill kernel
(build with tools/build_variant.py gtrace -DDYQ_PRE_GTRACE=1, run with
DYQ_LIB=tools/variants/libdyq_gtrace.so).  Events per group i: 0 MMA saw
full, 1 MMA saw afull, 2 MMA saw tempty (issues next), 3 promotion saw
tfull, 4 promotion done, 5 transform done, 6 activation copy issued, 7 transform warp 4 done.
Prints the median interval of each stage over the steady state.
usage: python tools/trace_prefill_groups.py [linear] [M] [bits]"""
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
tr = torch.zeros(16 + 512 * 8, dtype=torch.int64, device=dev)
dyq.trace_enable(tr)
tr[1] = 0  # no per-CTA trace_ev records: the buffer holds only the per-group stamps
dyq.qlinear(p.wd, p.codes, p.meta, x, M, None, bits, y, 1, ws)
torch.cuda.synchronize()
dyq.trace_enable(None)
t = tr.cpu().numpy()[16:].reshape(8, 512).astype(np.int64)
n = int((t[4] > 0).sum())
t = t[:, :n]
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, -1) / 1e3
lo, hi = min(10, n // 4), n - 5
d = lambda a, b: np.median(t[a, lo:hi] - t[b, lo:hi])  # noqa: E731
print(f"groups {n}; cadence (promotion done) {np.median(np.diff(t[4, lo:hi])):.3f} us/group")
print(f"act copy issued -> MMA full  {d(0, 6):.3f}")
print(f"MMA full -> afull            {d(1, 0):.3f}")
print(f"MMA afull -> tempty          {d(2, 1):.3f}")
print(f"MMA tempty -> promo tfull    {d(3, 2):.3f}  (MMA issue + commit + wake)")
print(f"promo tfull -> promo done    {d(4, 3):.3f}")
print(f"transform done -> MMA afull  {d(1, 5):.3f} (warp 3), {d(1, 7):.3f} (warp 4)")
print(f"cadence of each stamp: " + ", ".join(f"ev{e} {np.median(np.diff(t[e, lo:hi])):.3f}" for e in range(8)))
