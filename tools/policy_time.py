"""Policy-step timing (graph of R steps, median of N) for A/B of library builds:
DYQ_LIB=... python tools/policy_time.py [E] [R] [N]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_07904_b200 import dyq  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 1
R = int(sys.argv[2]) if len(sys.argv) > 2 else 3
NT = int(sys.argv[3]) if len(sys.argv) > 3 else 5
dev, C, d_m, NL = "cuda:0", 8, 4096, 32
lins = synth.LLAMA_BLOCK_LINEARS
packed = [[dyq.PackedLinear.from_bf16(synth.weights_bf16_torch(N, K, seed=1 + 4 * c + i, device=dev), group=64, wbits=4)
           for i, (_, N, K) in enumerate(lins)] for c in range(C)]
layers = [packed[l % C] for l in range(NL)]
one = torch.full((d_m,), 0x3F80, dtype=torch.int16, device=dev)
norms = one.repeat(NL)
embed = synth.activations_bf16_torch(32000, d_m, seed=7000, device=dev)
head = synth.weights_bf16_torch(256, d_m, seed=7001, device=dev)
model = dyq.Model(layers, norms, norms, one, embed, head, E=E, n_heads=32)
cal = dyq.default_calib()
pst = torch.zeros(dyq.state_size(E, cal), dtype=torch.uint8, device=dev)
dyq.state_init(E, cal, pst)
vis = synth.activations_bf16_torch(E * 256, d_m, seed=7100, device=dev)
text = torch.randint(0, 32000, (E, 32), dtype=torch.int32, device=dev, generator=torch.Generator(device=dev).manual_seed(7))
act_o = torch.zeros(E, 7, dtype=torch.float32, device=dev)
bits_o = torch.zeros(E, dtype=torch.int32, device=dev)
for _ in range(2):
    model.step(pst, E, vis, text, act_o, bits_o)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.graph(g, stream=s):
    for _ in range(R):
        model.step(pst, E, vis, text, act_o, bits_o, stream=s)
g.replay()
torch.cuda.synchronize()
ts = []
for _ in range(NT):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / R)
print(f"E={E}: {statistics.median(ts):.3f} ms/step (min {min(ts):.3f})")
