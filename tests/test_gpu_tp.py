"""GPU checks of the TP join on one device: the interleave
kernel, a world-1 NCCL communicator through dyq_tp_allgather, and a 2-shard
column split composed on one GPU against the unsharded qlinear."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2603_07904_b200 import dyq  # noqa: E402
from test_gpu_parity import check_close  # noqa: E402

DEV = "cuda:0"


@pytest.mark.parametrize("P,M,Ns", [(4, 1, 64), (2, 5, 128), (8, 8, 512)])
def test_interleave(P, M, Ns):
    buf = torch.randint(-30000, 30000, (P, M, Ns), dtype=torch.int16, device=DEV)
    y = torch.empty(M, P * Ns, dtype=torch.int16, device=DEV)
    dyq.tp_interleave(buf, P, M, Ns, y)
    ref = buf.permute(1, 0, 2).reshape(M, P * Ns)
    assert torch.equal(y, ref)


@pytest.mark.parametrize("M", [1, 6])
def test_world1_allgather(M):
    comm = dyq.Comm(dyq.comm_unique_id(), 0, 1)
    ys = torch.randint(-30000, 30000, (M, 256), dtype=torch.int16, device=DEV)
    y = torch.empty_like(ys)
    buf = torch.empty_like(ys)
    comm.allgather(ys, M, 256, buf, y)
    torch.cuda.synchronize()
    assert torch.equal(y, ys)
    comm.close()


@pytest.mark.parametrize("M", [1, 8, 40])
def test_two_shard_composition(M):
    N, K, P = 1024, 512, 2
    W = torch.from_numpy(synth.weights_bf16(N, K, seed=21).view(np.int16)).to(DEV)
    x = torch.from_numpy(synth.activations_bf16(M, K, seed=22).view(np.int16)).to(DEV)
    full = dyq.PackedLinear.from_bf16(W, group=64, wbits=4)
    y_full = full(x, bits=4, out_dtype=torch.float32)
    parts = []
    for r in range(P):
        a, b = dyq.tp_shard(N, P, r)
        parts.append(dyq.PackedLinear.from_bf16(W[a:b].contiguous(), group=64, wbits=4)(x, bits=4,
                                                                                    out_dtype=torch.float32))
    y_tp = torch.cat(parts, dim=1)
    # same codes and integer sums; fp32 split-K order may differ per tile assignment
    torch.testing.assert_close(y_tp, y_full, rtol=1e-5, atol=1e-5 * float(y_full.abs().max()))
    # and the joined shards are the oracle qlinear of the UNSHARDED weight
    w_h, x_h = W.cpu().numpy().view(np.uint16), x.cpu().numpy().view(np.uint16)
    yref, _ = oracle.qlinear(x_h, oracle.pack_weights(w_h, 64, 4), 64, 4)
    check_close(y_tp.cpu().numpy(), yref, 1e-3)
