"""Column-sharded TP on CPU: world_size-2 gloo process group.

Each rank packs rows dyq_tp_shard(N, P, r) of the weight (the C shard rule of
libdyq.so, which needs no GPU), runs the oracle qlinear on its shard, and the
shards are joined with an all-gather + column interleave.  The result must equal
the unsharded oracle exactly: a K-group never spans ranks, so every output
element depends only on its own row's codes and scales."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth
from paper_2603_07904_b200 import dyq

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


@pytest.mark.parametrize("N,P", [(4096, 2), (12288, 8), (22016, 8), (256, 4)])
def test_shards_partition_rows_in_multiples_of_16(N, P):
    rows = []
    for r in range(P):
        a, b = dyq.tp_shard(N, P, r)
        assert a % 16 == 0 and b % 16 == 0 and b - a == N // P
        rows.extend(range(a, b))
    assert rows == list(range(N))
    with pytest.raises(dyq.DyqError):
        dyq.tp_shard(N + 8, P, 0)


def test_shard_pack_is_row_slice_of_full_pack():
    W = synth.weights_bf16(64, 256, seed=3)
    full = oracle.pack_weights(W, 64, 4)
    a, b = dyq.tp_shard(64, 2, 1)
    part = oracle.pack_weights(W[a:b], 64, 4)
    assert np.array_equal(part.q, full.q[a:b]) and np.array_equal(part.s, full.s[a:b])
    assert np.array_equal(part.z, full.z[a:b])


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir, M, N, K, bits):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W = synth.weights_bf16(N, K, seed=11)
        x = synth.activations_bf16(M, K, seed=12)
        a, b = dyq.tp_shard(N, world, rank)
        ys, Is = oracle.qlinear(x, oracle.pack_weights(W[a:b], 64, 4), 64, bits, want_I=True)
        got = [torch.zeros(M, N // world, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(got, torch.from_numpy(np.ascontiguousarray(ys)))
        gotI = [torch.zeros(M, N // world, K // 64, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(gotI, torch.from_numpy(np.ascontiguousarray(Is)))
        if rank == 0:
            # the interleave: y[m, r Ns + j] = shard_r[m, j]
            np.save(os.path.join(outdir, "y.npy"), torch.cat(got, dim=1).numpy())
            np.save(os.path.join(outdir, "I.npy"), torch.cat(gotI, dim=1).numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("bits", [4, 16])
def test_two_rank_column_sharded_qlinear_is_exact(tmp_path, bits):
    M, N, K = 3, 256, 256
    mp.spawn(_worker, args=(2, _port(), str(tmp_path), M, N, K, bits), nprocs=2, join=True)
    W = synth.weights_bf16(N, K, seed=11)
    x = synth.activations_bf16(M, K, seed=12)
    y, I = oracle.qlinear(x, oracle.pack_weights(W, 64, 4), 64, bits, want_I=True)
    assert np.array_equal(np.load(tmp_path / "y.npy"), y)
    assert np.array_equal(np.load(tmp_path / "I.npy"), I)


def test_fused_tp_peers_struct_and_validation():
    """dyq_tp_peers_t layout (include/dyq.h) and dyq_qlinear_tp's host-side
    argument checks, which run before any CUDA call."""
    import ctypes as C
    from paper_2603_07904_b200 import dyq
    assert C.sizeof(dyq.TpPeers) == 8 + 8 * 8 + 8 * 8
    assert dyq.TpPeers.y.offset == 8 and dyq.TpPeers.flag.offset == 72
    t = dyq.tp_peers(2, 1, [0x1000, 0x2000], [0x3000, 0x4000])
    assert (t.world, t.rank, t.y[1], t.flag[0]) == (2, 1, 0x2000, 0x3000)
    L = dyq.lib()
    wd = dyq.WDesc(256, 256, 64, 4, 0)
    assert L.dyq_qlinear_tp(C.byref(wd), None, None, None, 1, None, 4, None, None, 0, None, None) == 1
    bad = dyq.tp_peers(1, 0, [0x1000], [0x2000])
    bad.world = 9  # > DYQ_TP_MAX
    assert L.dyq_qlinear_tp(C.byref(wd), None, None, None, 1, None, 4, C.byref(bad), None, 0, None, None) == 1
    bad = dyq.tp_peers(2, 0, [0x1000, 0], [0x2000, 0x3000])  # null y of rank 1
    assert L.dyq_qlinear_tp(C.byref(wd), None, None, None, 1, None, 4, C.byref(bad), None, 0, None, None) == 1
    assert b"rank 1" in L.dyq_last_error()
