# tiny prefill run with a watchdog-friendly exit code (used before the full tests)
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, oracle
from paper_2603_07904_b200 import dyq
M, N, K, G = 130, 256, 128, 64
w = synth.weights_bf16(N, K, seed=1); x = synth.activations_bf16(M, K, seed=2)
wt = torch.from_numpy(w.view(np.int16)).cuda(); xt = torch.from_numpy(x.view(np.int16)).cuda()
lin = dyq.PackedLinear.from_bf16(wt, 64, 4)
ws = lin.workspace(M)
I = torch.zeros(M, N, K // G, dtype=torch.int32, device="cuda")
dyq.qlinear_i32_partials(lin.wd, lin.codes, lin.meta, xt, M, None, 8, I, ws)
torch.cuda.synchronize()
_, Iref = oracle.qlinear(x, oracle.pack_weights(w, G, 4), G, 8, want_I=True)
got = I.cpu().numpy()
print("prefill partials mismatches:", int((got != Iref).sum()), "of", got.size)
y = torch.zeros(M, N, dtype=torch.float32, device="cuda")
dyq.qlinear(lin.wd, lin.codes, lin.meta, xt, M, None, 8, y, 0, ws)
torch.cuda.synchronize()
yref, _ = oracle.qlinear(x, oracle.pack_weights(w, G, 4), G, 8)
print("max rel err", float(np.abs(y.cpu().numpy() - yref).max() / np.abs(yref).max()))
