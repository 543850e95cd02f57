"""One dyq_policy_step (OpenVLA-7B shapes, 8 rotating packed block copies) for ncu
launch-list profiling: python tools/prof_policy.py [E] [copies]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_07904_b200 import dyq  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 1
C = int(sys.argv[2]) if len(sys.argv) > 2 else 4
dev = "cuda:0"
lins = synth.LLAMA_BLOCK_LINEARS
packed = [[dyq.PackedLinear.from_bf16(synth.weights_bf16_torch(N, K, seed=1 + 4 * c + i, device=dev), group=64, wbits=4)
           for i, (_, N, K) in enumerate(lins)] for c in range(C)]
d_m, NL = 4096, 32
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
text = torch.randint(0, 32000, (E, 32), dtype=torch.int32, device=dev)
act_o = torch.zeros(E, 7, dtype=torch.float32, device=dev)
bits_o = torch.zeros(E, dtype=torch.int32, device=dev)
for _ in range(int(os.environ.get("STEPS", "2"))):
    model.step(pst, E, vis, text, act_o, bits_o)
torch.cuda.synchronize()
print("ok", bits_o.cpu().numpy().tolist())
