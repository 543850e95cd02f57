"""Episode data parallelism on CPU: world_size-2 gloo process groups (127.0.0.1).

The N > 1 path of bench.py shards independent episodes across ranks with no
collective on the data path; these tests check that the sharding is a
partition, that the per-episode bit sequences of a 2-rank run equal those of a
single-rank run (episodes are independent control streams), and that
the end-of-run reductions (max time over ranks, summed counters) are right.
The kinematic selector here is the oracle's (tests may use it; the product
path never does).
"""
import os
import socket

import numpy as np
import pytest

from paper_2603_07904_b200 import episodes

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


@pytest.mark.parametrize("E,world", [(64, 1), (64, 2), (64, 8), (7, 2), (3, 4), (0, 2), (1, 3)])
def test_shard_is_a_balanced_partition(E, world):
    seen = []
    sizes = []
    for r in range(world):
        rg = episodes.shard(E, world, r)
        assert rg.step == 1
        seen.extend(rg)
        sizes.append(len(rg))
    assert seen == list(range(E))
    assert max(sizes) - min(sizes) <= 1


def test_shard_rejects_bad_ranks():
    with pytest.raises(ValueError):
        episodes.shard(4, 2, 2)
    with pytest.raises(ValueError):
        episodes.shard(4, 0, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bits_for(eps, T):
    import oracle
    import synth
    out = []
    for e in eps:
        acts = synth.trajectory(T, episodes.episode_seed(e))[0]
        st = oracle.SelectState(1)
        seq = []
        for t in range(T):
            r = st.step(None if t == 0 else acts[t - 1][None, :])
            seq.append(int(r["bits"][0]))
        out.append(seq)
    return out


def _worker(rank, world, port, E, T, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = episodes.shard(E, world, rank)
        rows = _bits_for(mine, T)
        allrows = episodes.gather_per_episode(rows, E)
        hist = {}
        for seq in rows:
            for b in seq:
                hist[b] = hist.get(b, 0) + 1
        merged = episodes.merge_histograms(hist)
        tmax = episodes.max_over_ranks(1.0 + rank)
        tput = episodes.throughput(10.0 * len(mine), tmax)
        if rank == 0:
            np.save(os.path.join(outdir, "bits.npy"), np.array(allrows, np.int32))
            np.save(os.path.join(outdir, "hist.npy"), np.array([merged[k] for k in (2, 4, 8, 16)]))
            np.save(os.path.join(outdir, "scalars.npy"), np.array([tmax, tput]))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_matches_single_rank(tmp_path):
    E, T, world = 6, 60, 2
    mp.spawn(_worker, args=(world, _free_port(), E, T, str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / "bits.npy")
    ref = np.array(_bits_for(range(E), T), np.int32)
    assert got.shape == (E, T)
    assert np.array_equal(got, ref)
    hist = np.load(tmp_path / "hist.npy")
    assert hist.sum() == E * T
    assert list(hist) == [int((ref == b).sum()) for b in (2, 4, 8, 16)]
    tmax, tput = np.load(tmp_path / "scalars.npy")
    assert tmax == 2.0                      # max over ranks of (1 + rank)
    assert tput == pytest.approx(10.0 * E / 2.0)  # all ranks' units / slowest rank's time
