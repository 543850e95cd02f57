import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2603_07904_b200 import dyq
name = sys.argv[1] if len(sys.argv) > 1 else "gate_up"
N, K = {n: (N, K) for n, N, K in synth.LLAMA_BLOCK_LINEARS}[name]
lin = dyq.PackedLinear.from_bf16(synth.weights_bf16_torch(N, K, seed=1, device="cuda"), group=64, wbits=4)
x = synth.activations_bf16_torch(8, K, seed=1000, device="cuda")
y = torch.empty(8, N, dtype=torch.bfloat16, device="cuda")
ws = lin.workspace(8)
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    dyq.qlinear(lin.wd, lin.codes, lin.meta, x, 8, None, 4, y, 1, ws)
    torch.cuda.synchronize()
    print("launch", i, "ok", flush=True)
