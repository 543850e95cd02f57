"""Worker of tests/test_gpu_tp_fused.py::test_fused_two_processes_ipc (one
process per rank, all on cuda:0; peer buffers mapped with CUDA IPC, handles
exchanged over a gloo process group)."""
import numpy as np
import torch
import torch.distributed as dist

import synth
from paper_2603_07904_b200 import dyq

N, K, M, MP = 1024, 512, 8, 160  # MP > 16: the tcgen05 prefill path (two token tiles)
HDR = 256  # flag lives in the first bytes of the rank's buffer


def shard_refs(W, x, world, bits):
    out = []
    for r in range(world):
        a, b = dyq.tp_shard(N, world, r)
        lin = dyq.PackedLinear.from_bf16(W[a:b].contiguous(), group=64, wbits=4)
        out.append(lin(x, bits=bits, out_dtype=torch.bfloat16))
    return torch.cat(out, dim=1).view(torch.int16)


def worker(rank, world, port):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dev = "cuda:0"
    W = torch.from_numpy(synth.weights_bf16(N, K, seed=41).view(np.int16)).to(dev)
    x = torch.from_numpy(synth.activations_bf16(M, K, seed=42).view(np.int16)).to(dev)
    xp = torch.from_numpy(synth.activations_bf16(MP, K, seed=43).view(np.int16)).to(dev)
    a, b = dyq.tp_shard(N, world, rank)
    lin = dyq.PackedLinear.from_bf16(W[a:b].contiguous(), group=64, wbits=4)
    ws = lin.workspace(MP)
    ybytes = MP * N * 2
    buf = torch.zeros(HDR + 2 * ybytes, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    h, off = dyq.ipc_handle(buf)
    allh = [None] * world
    dist.all_gather_object(allh, (h, off))
    base, opened = [], []
    for p in range(world):
        if p == rank:
            base.append(buf.data_ptr())
        else:
            ptr = dyq.ipc_open(*allh[p])
            base.append(ptr)
            opened.append((ptr, allh[p][1]))
    flag = buf[:8].view(torch.int64)
    timed_out = torch.zeros(1, dtype=torch.int32, device=dev)
    dist.barrier()
    target = 0
    for c, (bits, m) in enumerate([(2, M), (4, M), (16, MP), (8, M), (4, MP)], start=1):
        s = (c - 1) % 2
        xm = x if m == M else xp
        peers = dyq.tp_peers(world, rank, [q + HDR + s * ybytes for q in base], base)
        dyq.qlinear_tp(lin, xm, m, None, bits, peers, ws)
        target += dyq.tp_flag_delta(N, m)
        dyq.tp_wait(flag, target, timed_out)
        torch.cuda.synchronize()
        assert int(timed_out.item()) == 0, f"rank {rank}: wait timed out at call {c}"
        assert int(flag.item()) == target, (rank, c, int(flag.item()))
        y = buf[HDR + s * ybytes:HDR + s * ybytes + m * N * 2].view(torch.int16).view(m, N)
        ref = shard_refs(W, xm, world, bits)
        assert torch.equal(y, ref), f"rank {rank} call {c}: fused TP output differs"
    dist.barrier()
    for ptr, o in opened:
        dyq.ipc_close(ptr, o)
    dist.destroy_process_group()
