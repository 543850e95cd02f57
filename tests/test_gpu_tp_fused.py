"""Fused tensor-parallel decode epilogue (dyq_qlinear_tp):
each rank's decode kernel stores its column shard into every rank's full y and
announces it on every rank's flag.  On one GPU: P simulated ranks in one
process (peer buffers = plain device buffers), and two real processes sharing
cuda:0 with their buffers mapped through CUDA IPC.  Outputs must equal the
per-shard dyq_qlinear results bit-for-bit (same kernel, same plan)."""
import socket

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


@pytest.mark.parametrize("P,M,N", [(1, 1, 512), (2, 8, 1024), (4, 16, 2048), (8, 3, 1024), (2, 5, 22016),
                                   (2, 17, 1024), (4, 288, 2048), (8, 40, 1024)])
def test_fused_simulated_ranks(P, M, N):
    K = 512
    W = torch.from_numpy(synth.weights_bf16(N, K, seed=N + P).view(np.int16)).to(DEV)
    x = torch.from_numpy(synth.activations_bf16(M, K, seed=M + 7).view(np.int16)).to(DEV)
    lins, wss = [], []
    for r in range(P):
        a, b = dyq.tp_shard(N, P, r)
        lins.append(dyq.PackedLinear.from_bf16(W[a:b].contiguous(), group=64, wbits=4))
        wss.append(lins[-1].workspace(M))
    ys = [[torch.full((M, N), -1, dtype=torch.int16, device=DEV) for _ in range(P)] for _ in range(2)]
    flags = [torch.zeros(1, dtype=torch.int64, device=DEV) for _ in range(P)]
    to = torch.zeros(1, dtype=torch.int32, device=DEV)
    rb = torch.tensor([[2, 4, 8, 16][m % 4] for m in range(M)], dtype=torch.int32, device=DEV)
    delta = dyq.tp_flag_delta(N, M)
    assert delta == N // 16 * (1 if M <= 16 else -(-M // 144))
    # oracle reference: the UNSHARDED weight's qlinear (a K-group never spans
    # ranks, so the gathered column shards must be exactly its columns)
    w_h, x_h = W.cpu().numpy().view(np.uint16), x.cpu().numpy().view(np.uint16)
    pk_full = oracle.pack_weights(w_h, 64, 4)
    for c, (bits, row_bits) in enumerate([(4, None), (2, None), (0, rb), (16, None)], start=1):
        s = (c - 1) % 2
        for r in range(P):
            peers = dyq.tp_peers(P, r, [t.data_ptr() for t in ys[s]], [f.data_ptr() for f in flags])
            dyq.qlinear_tp(lins[r], x, M, row_bits, bits, peers, wss[r])
        for r in range(P):
            dyq.tp_wait(flags[r], c * delta, to)
        torch.cuda.synchronize()
        assert int(to.item()) == 0
        assert [int(f.item()) for f in flags] == [c * delta] * P
        ref = torch.cat([lin(x, row_bits=row_bits, bits=bits, out_dtype=torch.bfloat16) for lin in lins],
                        dim=1).view(torch.int16)
        for r in range(P):
            assert torch.equal(ys[s][r], ref), (c, r)
        yref, _ = oracle.qlinear(x_h, pk_full, 64, bits if row_bits is None else row_bits.cpu().numpy())
        check_close(ys[s][0].view(torch.bfloat16).float().cpu().numpy(), yref, 2e-2)


def test_fused_rejects_bad_peers_and_forced_decode_over_16():
    N, K, M = 256, 256, 20
    W = torch.from_numpy(synth.weights_bf16(N, K, seed=1).view(np.int16)).to(DEV)
    lin = dyq.PackedLinear.from_bf16(W, group=64, wbits=4)
    x = torch.from_numpy(synth.activations_bf16(M, K, seed=2).view(np.int16)).to(DEV)
    ws = lin.workspace(M)
    y = torch.zeros(M, N, dtype=torch.int16, device=DEV)
    f = torch.zeros(1, dtype=torch.int64, device=DEV)
    peers = dyq.tp_peers(1, 0, [y.data_ptr()], [f.data_ptr()])
    dyq.set_path(1)  # force the decode kernel: one fused launch covers at most 16 rows
    try:
        with pytest.raises(dyq.DyqError) as e:
            dyq.qlinear_tp(lin, x, M, None, 4, peers, ws)
        assert e.value.code == 3  # DYQ_EUNSUPPORTED
    finally:
        dyq.set_path(0)
    bad = dyq.tp_peers(2, 1, [y.data_ptr(), 0], [f.data_ptr(), f.data_ptr()])
    with pytest.raises(dyq.DyqError):
        dyq.qlinear_tp(lin, x, 4, None, 4, bad, ws)


def test_tp_wait_returns_once_reached():
    f = torch.full((1,), 5, dtype=torch.int64, device=DEV)
    to = torch.zeros(1, dtype=torch.int32, device=DEV)
    dyq.tp_wait(f, 5, to)
    torch.cuda.synchronize()
    assert int(to.item()) == 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(300)
def test_fused_two_processes_ipc():
    import torch.multiprocessing as mp
    import _tp_fused_worker
    mp.spawn(_tp_fused_worker.worker, args=(2, _free_port()), nprocs=2, join=True)
