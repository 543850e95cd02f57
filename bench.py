#!/usr/bin/env python
"""bench.py -- DyQ-VLA runtime-switchable qlinear hot path on B200.

Workload (BASELINE.json configs[1], the config the metric's "qlinear HBM GB/s"
is quoted on): one Llama-2-7B-shaped block (d=4096, ffn=11008) at decode,
M action tokens (default 8), W4 (the paper's INT4-pinned weights).
One STEP = one pass of the whole hot path for one control step:
    dyq_select_route (kinematic proxies -> S_t -> Alg. 1 on a[t-1], then
    b* -> per-token activation bits through the W4-pinned table, one kernel)
    -> for QKV, o, gate|up, down: dyq_qlinear (act-quant + decode kernels)
with b* chosen each step by the kinematic dispatcher from a synthetic
LIBERO-shaped trajectory (120 untimed history steps first).
L2 is defeated by rotating 8 packed copies of the block (8 x 117 MB > 126 MB).

value = algorithmic bytes per step (packed weight codes + metadata + bf16
activations in + bf16 outputs) / device time per step, summed
over ranks / max-over-ranks time (weak scaling: every rank runs its own
episode with replicated weights, no collective on the data path).

Extra objects on the same line: the roofline of the dominant kernel, the
fixed-width variants (W4 and the optional W8 copy, G=64 and G=128), the
M sweep, configs[0] (256x256 int4/int8 switch trajectory), the configs[2]
prefill slice, the configs[3] policy slice (E=1, 8 per GPU and the 64-episode
strong-scaling slice sharded over ranks), the Table IV selector overhead,
e2e through the public API, and the oracle on the host cores.

--gpus N without torchrun self-launches N ranks (torch.distributed.run on
127.0.0.1); ranks map to cuda:(local_rank % device_count), the control plane
(barriers, max-over-ranks timing) runs on gloo, so a 1-GPU box can execute
the N>1 path.  --impl reference times the CPU oracle (oracle/, plain C).
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HISTORY_STEPS = 120
METRIC = "qlinear decode HBM GB/s (Llama-2-7B block, M action tokens, kinematic bit switching)"


def make_config(args, copies, world, bytes_step=None):
    M, G, WB = args.M, args.group, args.wbits
    cfg = {"workload": f"configs[1]: llama2-7b block decode (QKV 12288x4096, o 4096x4096, "
                       f"gate|up 22016x4096, down 4096x11008), M={M} tokens, W{WB} G={G}",
           "bits": "per-step b* from dyq_select_bits (W4-pinned table)",
           "parallelism": f"dp{world} (episode-parallel, replicated weights)"}
    if bytes_step:
        cfg["l2"] = f"rotating {copies} packed block copies ({copies * bytes_step / 1e6:.0f} MB) > 126 MB L2"
    return cfg


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=400)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", default="dyq", choices=["dyq", "reference"])
    p.add_argument("--M", type=int, default=8, help="action tokens per decode step")
    p.add_argument("--wbits", type=int, default=4)
    p.add_argument("--group", type=int, default=64)
    p.add_argument("--copies", type=int, default=8, help="rotated block copies (L2 defeat)")
    p.add_argument("--trials", type=int, default=5, help="timed repetitions of the K-step region")
    p.add_argument("--no-variants", action="store_true")
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    p.add_argument("--no-prefill", action="store_true", help="skip the configs[2] prefill slice")
    p.add_argument("--no-policy", action="store_true", help="skip the configs[3] policy-step slice")
    p.add_argument("--no-ncu", action="store_true", help="skip the live ncu DRAM-traffic capture")
    p.add_argument("--policy-E", default="1,8", help="episodes per GPU for the policy slice")
    p.add_argument("--policy-E-total", type=int, default=64, help="configs[3] episodes sharded over ranks")
    p.add_argument("--profile", action="store_true", help="short run for ncu (no clocks / cpu)")
    return p.parse_args()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


def hbm_peak():
    pk = peaks()
    if pk and pk.get("hbm_gbs"):
        return float(pk["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def i8_peak():
    """(measured dense int8 TOPS, source) -- tools/umma_bench.cu kind::i8
    issue-rate measurement committed under profiles/, else None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "i8_peak.json")))
        return float(d["tops"]), d.get("how", "profiles/i8_peak.json")
    except Exception:
        return None, None


def algo_bytes(N, K, M, G, wbits):
    """N*K*wbits/8 + N*(K/G)*5 + M*K*2 + M*N*2."""
    return N * K * wbits // 8 + N * (K // G) * 5 + M * K * 2 + M * N * 2


def host_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


# --------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons through NVML while running."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index=0, period=0.002):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self._t = None
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------ oracle legs
def _oracle_block_pass(lins, packs, xs, G, b, threads):
    """One act_quant + qlinear of every sampled block linear through the C
    oracle, the rows of each linear split over `threads` host threads (ctypes
    releases the GIL, so the threads run the oracle on separate cores)."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor

    def one(job):
        name, part = job
        aq = oracle.act_quant(xs[name], G, b)
        oracle.qlinear(xs[name], part, G, b, actq=aq)

    jobs = [(name, part) for name in packs for part in packs[name]]
    if threads <= 1:
        for j in jobs:
            one(j)
    else:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(one, jobs))


def _oracle_packs(w_rows, G, wb, threads):
    import oracle
    import numpy as np
    packs = {}
    for name, w in w_rows.items():
        parts = np.array_split(w, max(1, threads))
        packs[name] = [oracle.pack_weights(np.ascontiguousarray(p), G, wb) for p in parts if len(p)]
    return packs


def run_reference(args, rank):
    """The oracle as it stands, on the host cores (one thread per core over
    row slices), on a bounded sample of the same workload and metric (GB/s of
    algorithmic qlinear bytes)."""
    if rank != 0:
        return
    import oracle
    import synth
    M, G, wb = args.M, args.group, args.wbits
    threads = os.cpu_count() or 1
    rows = 16 * threads  # bounded sample: the first rows of every block linear (same K)
    lins = synth.LLAMA_BLOCK_LINEARS
    w_rows = {n: synth.weights_bf16(rows, K, seed=1 + i) for i, (n, N, K) in enumerate(lins)}
    packs = _oracle_packs(w_rows, G, wb, threads)
    xs = {n: synth.activations_bf16(M, K, seed=1000 + i) for i, (n, N, K) in enumerate(lins)}
    acts = synth.trajectories(1, HISTORY_STEPS + args.warmup + args.steps + 2)
    st = oracle.SelectState(1)
    for t in range(HISTORY_STEPS):
        st.step(None if t == 0 else acts[t - 1])

    def one(t):
        b = int(st.step(acts[t - 1])["bits"][0])
        _oracle_block_pass(lins, packs, xs, G, b, threads)

    t0 = HISTORY_STEPS
    tc = time.perf_counter()
    one(t0)
    per = time.perf_counter() - tc
    budget = 120.0
    scale = max(1, int(per * (args.warmup + args.steps) / budget + 0.999))
    steps = max(1, args.steps // scale)
    warm = args.warmup
    for i in range(warm):
        one(t0 + 1 + i)
    tc = time.perf_counter()
    for i in range(steps):
        one(t0 + 1 + warm + i)
    dt = (time.perf_counter() - tc) / steps
    bytes_step = sum(algo_bytes(rows, K, M, G, wb) for _, _, K in lins)
    val = bytes_step / dt / 1e9
    sample = (f"first {rows} rows of each of the 4 block linears (K=4096/11008), M={M}, W{wb} G={G}, "
              f"select_bits+act_quant+qlinear per step, rows split over {threads} host threads; "
              f"{steps} timed steps (of {args.steps} requested)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC,
        "value": round(val, 4), "unit": "GB/s", "higher_is_better": True, "n_gpus": 1,
        "steps": steps, "warmup": warm, "ms_per_step": dt * 1e3,
        "dtype": "int64/f64 (oracle)", "data": "synthetic",
        "config": make_config(args, args.copies, 1),
        "cpu_baseline": dict({"value": round(val, 4), "unit": "GB/s", "cores": threads, "kind": "oracle",
                              "sample": sample}, **host_info()),
        "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "vs_baseline": None,
    }), flush=True)


def cpu_baseline(args, w_host, budget_s=15.0):
    """Oracle on this box's host cores (one thread per core over row slices):
    the first rows of every block linear (full K), as many block passes as fit
    ~budget_s (>= 1)."""
    import synth
    M, G, wb = args.M, args.group, args.wbits
    threads = os.cpu_count() or 1
    rows = 64 * threads
    w_rows = {name: w_host[name][:rows] for name, _, _ in synth.LLAMA_BLOCK_LINEARS}
    packs = _oracle_packs(w_rows, G, wb, threads)
    xs = {name: synth.activations_bf16(M, K, seed=1000 + i)
          for i, (name, N, K) in enumerate(synth.LLAMA_BLOCK_LINEARS)}
    tot_bytes, tot_t, n_done = 0, 0.0, 0
    t_start = time.perf_counter()
    while n_done < 1 or (time.perf_counter() - t_start) < budget_s:
        tc = time.perf_counter()
        _oracle_block_pass(synth.LLAMA_BLOCK_LINEARS, packs, xs, G, 8, threads)
        tot_t += time.perf_counter() - tc
        tot_bytes += sum(algo_bytes(len(w_rows[n]), K, M, G, wb) for n, _, K in synth.LLAMA_BLOCK_LINEARS)
        n_done += 1
    return dict({"value": round(tot_bytes / tot_t / 1e9, 4), "unit": "GB/s", "cores": threads, "kind": "oracle",
                 "sample": f"first {rows} rows of each block linear (full K), M={M}, A8 W{wb} G={G}, "
                           f"act_quant+qlinear, rows split over {threads} host threads, {n_done} block passes "
                           f"({tot_t:.1f} s)"}, **host_info())


# ------------------------------------------------------------ launching
def self_launch(args):
    """--gpus N outside torchrun: run this script under torch.distributed.run
    with N local ranks on 127.0.0.1 and return its exit code."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


class Ctl:
    """Control plane: barriers and max-over-ranks timing on a gloo group (the
    data path has no collective), so N ranks may share one GPU."""

    def __init__(self, world, rank):
        self.world, self.rank = world, rank
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
            self.dist = dist

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def reduce(self, v, op="max"):
        if self.world == 1:
            return float(v)
        import torch
        t = torch.tensor([float(v)], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.barrier()
            self.dist.destroy_process_group()


# ------------------------------------------------------------------- main
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import numpy as np
    import torch

    import synth
    from paper_2603_07904_b200 import dyq, episodes
    from paper_2603_07904_b200 import build as _b
    if rank == 0:
        _b.build()
    ctl = Ctl(world, rank)
    ctl.barrier()

    ndev = torch.cuda.device_count()
    dev_i = local % ndev
    torch.cuda.set_device(dev_i)
    dev = torch.device("cuda", dev_i)
    M, G, WB, C = args.M, args.group, args.wbits, args.copies
    if args.profile:
        C = min(C, 2)
    lins = synth.LLAMA_BLOCK_LINEARS
    extras = not args.profile and world == 1  # single-GPU-only legs

    def timed(g, reps=1):
        """Device time of `reps` replays of graph g: barrier + synchronize on
        both sides, CUDA events on the current stream, max over ranks."""
        ctl.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return ctl.reduce(e0.elapsed_time(e1))

    def graph_of(fn):
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(g, stream=s):
            fn()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        return g

    def pack_block(c, wbits, group, keep_host=False):
        out = []
        for li, (name, N, K) in enumerate(lins):
            w = synth.weights_bf16_torch(N, K, seed=1 + 4 * c + li, device=dev)
            if keep_host:
                w_host[name] = w[:64 * (os.cpu_count() or 1)].cpu().numpy().view(np.uint16).copy()
            out.append(dyq.PackedLinear.from_bf16(w, group=group, wbits=wbits))
            del w
        return out

    # ---- packed block copies (weights replicated on every rank)
    w_host = {}
    packed = [pack_block(c, WB, G, keep_host=(c == 0 and rank == 0)) for c in range(C)]
    torch.cuda.synchronize()

    # ---- activations (8 rotating sets), outputs, workspaces
    xs = [[synth.activations_bf16_torch(M, K, seed=1000 + 4 * s + li + 100 * rank, device=dev)
           for li, (_, _, K) in enumerate(lins)] for s in range(8)]
    ys = [torch.empty(M, N, dtype=torch.bfloat16, device=dev) for (_, N, _) in lins]
    wss = [packed[0][li].workspace(M) for li in range(len(lins))]

    # ---- kinematic state and trajectory (episode seed per rank)
    T = HISTORY_STEPS + args.warmup + args.steps * (args.trials + 2) + 2
    my_eps = episodes.shard(world, world, rank)  # one episode (control stream) per rank
    acts_np = synth.trajectories(1, T, seed0=episodes.episode_seed(my_eps[0]))
    acts = torch.from_numpy(acts_np).to(dev)
    cal = dyq.default_calib()
    state = torch.zeros(dyq.state_size(1, cal), dtype=torch.uint8, device=dev)
    dyq.state_init(1, cal, state)
    bits = torch.zeros(1, dtype=torch.int32, device=dev)
    bits_all = torch.zeros(args.steps, dtype=torch.int32, device=dev)  # b* of every timed step
    row_bits = torch.zeros(M, dtype=torch.int32, device=dev)
    for t in range(HISTORY_STEPS):
        dyq.select_bits(state, 1, None if t == 0 else acts[t - 1], bits)
    t_cur = HISTORY_STEPS

    bytes_step = sum(algo_bytes(N, K, M, G, WB) for _, N, K in lins)
    gate_li = [n for n, _, _ in lins].index("gate_up")
    n_launch_step = 1 + 2 * len(lins)  # select_route, then act-quant + qlinear kernel per linear

    def step(t, bslot=None, fixed_bits=None, blk=None, xset=None, yset=None, wsset=None, MM=M, rbt=None):
        blk = blk if blk is not None else packed
        c = t % len(blk)
        rbt = rbt if rbt is not None else row_bits
        if fixed_bits is None:
            dyq.select_route(state, 1, acts[t - 1], bits if bslot is None else bits_all[bslot:bslot + 1], MM, rbt)
            rb, b = rbt, 0
        else:
            rb, b = None, fixed_bits
        xset = xset if xset is not None else xs[t % 8]
        for li in range(len(lins)):
            p = blk[c][li]
            dyq.qlinear(p.wd, p.codes, p.meta, xset[li], MM, rb, b, (yset or ys)[li], 1, (wsset or wss)[li])

    # ---- warm-up (eager), then capture the K-step region as one CUDA graph;
    # every replay advances the selector state (the graph replays the same
    # a_{t-1} inputs), b* of each timed step lands in bits_all[i]
    for i in range(args.warmup):
        step(t_cur)
        t_cur += 1
    torch.cuda.synchronize()

    def run_steps():
        for i in range(args.steps):
            step(t_cur + i, bslot=i)

    graph = graph_of(run_steps)  # includes one untimed replay
    hist = {}
    trial_ms = []
    with ClockSampler(dev_i) as clk:
        for _ in range(args.trials):
            trial_ms.append(timed(graph))
            for k in bits_all.tolist():
                hist[k] = hist.get(k, 0) + 1
    ms_total = statistics.median(trial_ms)
    ms_step = ms_total / args.steps
    value = ctl.reduce(bytes_step, "sum") / (ms_step * 1e-3) / 1e9  # all ranks' bytes / slowest rank
    hist = {k: int(ctl.reduce(v, "sum")) for k, v in sorted(hist.items())} if world == 1 else \
        {k: int(ctl.reduce(hist.get(k, 0), "sum")) for k in (2, 4, 8, 16)}

    # ---- roofline of the dominant kernel (decode qlinear on gate|up): graphs
    # of R back-to-back launches per activation width, weighted by the timed
    # b* histogram (W4-pinned table: b* = activation bits)
    N_g, K_g = lins[gate_li][1], lins[gate_li][2]
    gate_bytes = algo_bytes(N_g, K_g, M, G, WB)
    peak, peak_kind = hbm_peak()
    R = 64
    k_by_bits, q_by_bits = {}, {}
    widths = sorted(b for b in hist if hist[b] > 0) or [4]
    for b in widths:
        def calls(b=b):
            for r in range(R):
                p = packed[r % C][gate_li]
                dyq.qlinear(p.wd, p.codes, p.meta, xs[0][gate_li], M, None, b, ys[gate_li], 1, wss[gate_li])
        g3 = graph_of(calls)
        k_by_bits[b] = statistics.median(timed(g3) for _ in range(5)) / R
        del g3
        p0 = packed[0][gate_li]
        dyq.act_quant(p0.wd, xs[0][gate_li], M, None, b, wss[gate_li])

        def kern(b=b):
            for r in range(R):
                p = packed[r % C][gate_li]
                dyq.qlinear_q(p.wd, p.codes, p.meta, xs[0][gate_li], M, None, b, ys[gate_li], 1, wss[gate_li])
        g4 = graph_of(kern)
        q_by_bits[b] = statistics.median(timed(g4) for _ in range(5)) / R
        del g4
    n_h = sum(hist.get(b, 0) for b in widths) or 1
    call_ms = sum(k_by_bits[b] * hist.get(b, 0) / n_h for b in widths) or k_by_bits[widths[0]]
    k_ms = sum(q_by_bits[b] * hist.get(b, 0) / n_h for b in widths) or q_by_bits[widths[0]]
    traffic, traffic_src = None, None
    if extras and not args.no_ncu:
        traffic, traffic_src = ncu_traffic(M, WB, G, widths, hist)
    roofline = {"bound": "hbm", "kernel": "qlinear_decode_kernel (gate|up 22016x4096)",
                "achieved": round(gate_bytes / (k_ms * 1e-3) / 1e9, 1),
                "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": round(gate_bytes / (k_ms * 1e-3) / 1e9 / peak, 4),
                "traffic": traffic, "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": gate_bytes, "kernel_ms": round(k_ms, 5),
                "timing": (f"cuda events around graphs of {R} back-to-back qlinear_decode_kernel launches "
                           f"(dyq_qlinear_q, rotating copies) per width "
                           f"{ {b: round(v * 1e3, 2) for b, v in q_by_bits.items()} } us, weighted by the timed b* "
                           f"histogram; per dyq_qlinear call incl. the act-quant kernel: "
                           f"{ {b: round(v * 1e3, 2) for b, v in k_by_bits.items()} } us"),
                "call_ms": round(call_ms, 5),
                "call_frac": round(gate_bytes / (call_ms * 1e-3) / 1e9 / peak, 4)}

    # ---- fixed-width variants: W4 (this block), the optional W8 copy and
    # G=128, each a graph of 64 block steps over rotating copies
    variants = {}
    if extras and not args.no_variants:
        def variant_line(blk, wbits, group, b):
            g2 = graph_of(lambda: [step(t_cur + i, fixed_bits=b, blk=blk, wsset=wv) for i in range(64)])
            ms = statistics.median(timed(g2) for _ in range(3)) / 64
            del g2
            bs = sum(algo_bytes(N, K, M, group, wbits) for _, N, K in lins)
            return {"GB/s": round(bs / (ms * 1e-3) / 1e9, 1),
                    "int_TOPS" if b != 16 else "TFLOPS": round(
                        sum(2 * M * N * K for _, N, K in lins) / (ms * 1e-3) / 1e12, 3),
                    "us_per_block": round(ms * 1e3, 2)}
        wv = wss
        for b in (2, 4, 8, 16):
            variants[f"W{WB}A{b}"] = variant_line(packed, WB, G, b)
        alt = [(8, G), (WB, 128)] if (WB, G) == (4, 64) else []
        for wbits, group in alt:
            blk = [pack_block(c, wbits, group) for c in range(C)]
            wv = [blk[0][li].workspace(M) for li in range(len(lins))]
            for b in (2, 4, 8, 16):
                variants[f"W{wbits}A{b}" + ("" if group == G else f"_G{group}")] = variant_line(blk, wbits, group, b)
            del blk, wv
            torch.cuda.empty_cache()

    # ---- M sweep (decode, the step's b* routing): M = 1, 2, 4, 8, 16
    m_sweep = {}
    if extras and not args.no_variants:
        for MM in (1, 2, 4, 8, 16):
            xm = [[synth.activations_bf16_torch(MM, K, seed=3000 + 4 * s + li, device=dev)
                   for li, (_, _, K) in enumerate(lins)] for s in range(2)]
            ym = [torch.empty(MM, N, dtype=torch.bfloat16, device=dev) for (_, N, _) in lins]
            wm = [packed[0][li].workspace(MM) for li in range(len(lins))]
            rbm = torch.zeros(MM, dtype=torch.int32, device=dev)
            st0 = state.clone()
            g5 = graph_of(lambda: [step(t_cur + i, xset=xm[i % 2], yset=ym, wsset=wm, MM=MM, rbt=rbm)
                                   for i in range(64)])
            ms = statistics.median(timed(g5) for _ in range(3)) / 64
            state.copy_(st0)
            bs = sum(algo_bytes(N, K, MM, G, WB) for _, N, K in lins)
            m_sweep[f"M{MM}"] = {"us_per_step": round(ms * 1e3, 2), "GB/s": round(bs / (ms * 1e-3) / 1e9, 1),
                                 "frac_hbm": round(bs / (ms * 1e-3) / 1e9 / peak, 4)}
            del g5, xm, ym, wm

    # ---- Table IV: selector latency and state bytes
    selector = None
    if extras:
        st1 = state.clone()
        g6 = graph_of(lambda: [dyq.select_route(st1, 1, acts[t_cur + i], bits, M, row_bits) for i in range(64)])
        us = statistics.median(timed(g6) for _ in range(5)) / 64 * 1e3
        del g6
        selector = {"select_route_us": round(us, 2), "state_bytes_per_stream": dyq.state_size(1, cal),
                    "paper_bound": "Table IV: < 0.5 ms dispatcher latency, < 64 KB state (P:594-598)",
                    "timing": "graph of 64 back-to-back dyq_select_route launches (one stream)"}

    # ---- configs[0]: one 256x256 linear, G=64, over a 20-step synthetic
    # trajectory: per step select_route + qlinear at the step's b*; the switch
    # cost is the trajectory time minus the same steps at a fixed width
    cfg0 = None
    if extras:
        cfg0 = config0(dyq, synth, torch, dev, graph_of, timed)

    # ---- configs[2] slice: prefill of one block at M = 288 tokens (256 vision +
    # 32 text) with the step's b*, on the tcgen05 path (tensor-bound)
    prefill = None
    if extras and not args.no_prefill:
        prefill = prefill_slice(args, dyq, synth, torch, dev, lins, packed, pack_block, bits, graph_of, timed, C)

    # ---- configs[3] slice: whole VLA policy steps/s
    policy = None
    if not args.profile and not args.no_policy:
        policy = policy_slice(args, dyq, synth, torch, dev, packed, C, rank, world, graph_of, timed, ctl)

    # ---- e2e through the public API
    e2e = None
    if not args.profile:
        e2e = e2e_leg(args, dyq, torch, dev, lins, packed, xs, ys, wss, state, row_bits, acts, t_cur, C, ctl,
                      bytes_step, world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        cpu = cpu_baseline(args, w_host)

    if rank == 0:
        out = {
            "metric": METRIC,
            "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 6), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8/s32 (int MMA) + f32 epilogue",
            "data": "synthetic (seeded weights/activations/trajectories, random-init)",
            "config": dict(make_config(args, C, world, bytes_step),
                           timed=f"median of {args.trials} replays of one CUDA graph of {args.steps} steps",
                           devices=f"{world} rank(s) on {ndev} visible GPU(s)"),
            "gpu_launches": n_launch_step * args.steps,
            "bytes_per_step": bytes_step,
            "bits_hist_timed": {str(k): v for k, v in sorted(hist.items())},
            "roofline": roofline,
            "variants": variants,
            "m_sweep": m_sweep,
            "selector": selector,
            "config0": cfg0,
            "prefill": prefill,
            "policy": policy,
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "trial_ms": [round(x, 4) for x in trial_ms],
        }
        print(json.dumps(out), flush=True)
    ctl.close()


def ncu_traffic(M, WB, G, widths, hist):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel, captured live by ncu on tools/prof_decode.py (same shape, each
    timed width), weighted by the b* histogram."""
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, None
    per = {}
    for b in widths:
        try:
            r = subprocess.run([ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--csv",
                                "--clock-control", "none", "-k", "regex:qlinear_decode_kernel", "-s", "4", "-c", "1",
                                sys.executable, os.path.join(ROOT, "tools", "prof_decode.py"), "gate_up", str(M),
                                str(WB), str(b)], capture_output=True, text=True, timeout=180)
            tot = 0.0
            for line in r.stdout.splitlines():
                if "dram__bytes_" in line:
                    f = [x.strip('"') for x in line.split('","')]
                    unit, val = f[-2], float(f[-1].replace(",", ""))
                    tot += val * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            if tot > 0:
                per[b] = tot
        except Exception:
            pass
    if not per:
        return None, None
    n = sum(hist.get(b, 0) for b in per) or 1
    tr = sum(per[b] * hist.get(b, 0) / n for b in per) if n > 1 else list(per.values())[0]
    return round(tr), f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (live, this run) per width {per}"


def config0(dyq, synth, torch, dev, graph_of, timed):
    """BASELINE configs[0]: 256x256, G=64, 20-step trajectory, int4/int8
    weight copies; per step select_route + qlinear (M = 8 tokens)."""
    import numpy as np
    N = K = 256
    G, M, T = 64, 8, 20
    w = synth.weights_bf16_torch(N, K, seed=1, device=dev)
    lin4 = dyq.PackedLinear.from_bf16(w, group=G, wbits=4)
    lin8 = dyq.PackedLinear.from_bf16(w, group=G, wbits=8)
    x = synth.activations_bf16_torch(M, K, seed=1000, device=dev)
    y = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
    cal = dyq.default_calib()
    acts = torch.from_numpy(synth.trajectories(1, HISTORY_STEPS + T + 1)).to(dev)
    st = torch.zeros(dyq.state_size(1, cal), dtype=torch.uint8, device=dev)
    bits = torch.zeros(1, dtype=torch.int32, device=dev)
    rb = torch.zeros(M, dtype=torch.int32, device=dev)
    res = {}
    for wb, lin in ((4, lin4), (8, lin8)):
        ws = lin.workspace(M)

        def traj(fixed=None):
            for t in range(HISTORY_STEPS, HISTORY_STEPS + T):
                dyq.select_route(st, 1, acts[t - 1], bits, M, rb)
                dyq.qlinear(lin.wd, lin.codes, lin.meta, x, M, None if fixed else rb, fixed or 0, y, 1, ws)

        def reset():
            dyq.state_init(1, cal, st)
            for t in range(HISTORY_STEPS):
                dyq.select_bits(st, 1, None if t == 0 else acts[t - 1], bits)
        reset()
        g = graph_of(traj)
        times = []
        for _ in range(5):
            reset()
            times.append(timed(g))
        seq = []
        reset()
        for t in range(HISTORY_STEPS, HISTORY_STEPS + T):
            dyq.select_bits(st, 1, acts[t - 1], bits)
            seq.append(int(bits.item()))
        switches = sum(1 for a, b in zip(seq, seq[1:]) if a != b)
        fixed = {}
        for b in (4, 8):
            reset()
            gf = graph_of(lambda b=b: traj(fixed=b))
            fixed[b] = statistics.median(timed(gf) for _ in range(5))
        t_traj = statistics.median(times)
        t_fix = sum(fixed[b] * seq.count(b) for b in (4, 8)) / max(1, sum(seq.count(b) for b in (4, 8))) \
            if any(b in (4, 8) for b in seq) else fixed[4]
        res[f"W{wb}"] = {"us_per_step": round(t_traj / T * 1e3, 2), "bits_seq": seq, "switches": switches,
                         "us_per_step_fixed_A4": round(fixed[4] / T * 1e3, 2),
                         "us_per_step_fixed_A8": round(fixed[8] / T * 1e3, 2)}
    del lin4, lin8
    return {"workload": "configs[0]: 256x256 linear, G=64, M=8, 20-step synthetic trajectory; per step "
                        "select_route + qlinear at b* (W4 and W8 weight copies)",
            "results": res, "timing": "cuda events around one graph of the 20 steps (median of 5, state reset)",
            "note": "a precision switch is data (per-row bits read by the kernel): the switching trajectory "
                    "costs the same per step as fixed widths"}


def prefill_slice(args, dyq, synth, torch, dev, lins, packed, pack_block, bits, graph_of, timed, C):
    MP = 288
    xps = [synth.activations_bf16_torch(MP, K, seed=5000 + li, device=dev) for li, (_, _, K) in enumerate(lins)]
    yps = [torch.empty(MP, N, dtype=torch.bfloat16, device=dev) for (_, N, _) in lins]
    rbp = torch.zeros(MP, dtype=torch.int32, device=dev)
    ops_block = sum(2 * MP * N * K for _, N, K in lins)
    i8_nom = 4500.0  # TOPS, nominal dense int8 (north_star: integer tensor-pipe peak)
    i8_meas, i8_src = i8_peak()
    bf16_peak = float((peaks() or {}).get("bf16_tflops", 2250.0))

    def run(blk, wps, fb, tag):
        def pstep(t):
            if fb is None:
                dyq.route_bits(bits, 1, MP, rbp)
                rb, b = rbp, 0
            else:
                rb, b = None, fb
            for li in range(len(lins)):
                p = blk[t % len(blk)][li]
                dyq.qlinear(p.wd, p.codes, p.meta, xps[li], MP, rb, b, yps[li], 1, wps[li])
        for i in range(2):
            pstep(i)
        RP = 10
        gp = graph_of(lambda: [pstep(i) for i in range(RP)])
        ms = statistics.median(timed(gp) for _ in range(3)) / RP
        del gp
        tops = ops_block / (ms * 1e-3) / 1e12
        r = {"us_per_block": round(ms * 1e3, 1), "int_TOPS": round(tops, 1),
             "frac_i8_nominal": round(tops / i8_nom, 4), "frac_bf16_pipe": round(tops / bf16_peak, 4)}
        if i8_meas:
            r["frac_i8_measured"] = round(tops / i8_meas, 4)
        return r

    pres = {}
    wps = [packed[0][li].workspace(MP) for li in range(len(lins))]
    for fb in (None, 2, 4, 8, 16):
        pres["step_bits" if fb is None else f"W{args.wbits}A{fb}"] = run(packed, wps, fb, "")
    # gate|up alone (the verdict's per-linear figure), W4A4
    gi = [n for n, _, _ in lins].index("gate_up")
    p = packed[0][gi]
    gq = graph_of(lambda: [dyq.qlinear(packed[i % C][gi].wd, packed[i % C][gi].codes, packed[i % C][gi].meta,
                                       xps[gi], MP, None, 4, yps[gi], 1, wps[gi]) for i in range(20)])
    gu_ms = statistics.median(timed(gq) for _ in range(3)) / 20
    del gq
    if (args.wbits, args.group) == (4, 64):
        for wbits, group in ((4, 128), (8, 64)):
            blk = [pack_block(c, wbits, group) for c in range(2)]
            wq = [blk[0][li].workspace(MP) for li in range(len(lins))]
            for fb in (None, 4, 8, 16):
                pres[("step_bits" if fb is None else f"W{wbits}A{fb}") + f"_W{wbits}G{group}"] = run(blk, wq, fb, "")
            del blk, wq
            torch.cuda.empty_cache()
    return {"workload": "configs[2] slice: one Llama-2-7B block prefill, M=288 (256 vision + 32 text), "
                        f"W{args.wbits} G={args.group}, b* of the current step; whole backbone = 32 x this",
            "kernel": "qlinear_prefill_kernel (persistent stream-K tcgen05 kind::f16, exact integer operands, "
                      "A in TMEM) + prefill_fixup_kernel",
            "peak_i8_TOPS_nominal": i8_nom, "peak_i8_TOPS_measured": i8_meas, "peak_i8_source": i8_src,
            "peak_bf16_TFLOPS": bf16_peak, "results": pres,
            "gate_up_W4A4_us": round(gu_ms * 1e3, 1),
            "timing": "cuda events around a graph of 10 blocks (median of 3)"}


def policy_slice(args, dyq, synth, torch, dev, packed, C, rank, world, graph_of, timed, ctl):
    """configs[3]: dyq_policy_step (select_bits, 288-token prefill and 6 decode
    passes through 32 Llama-2-7B blocks, action head + detok).  E per GPU
    (weak), and args.policy_E_total episodes sharded over the ranks (strong)."""
    from paper_2603_07904_b200 import episodes
    d_m, NL = 4096, 32
    layers = [packed[l % C] for l in range(NL)]
    one = torch.full((d_m,), 0x3F80, dtype=torch.int16, device=dev)  # bf16 1.0
    norms = one.repeat(NL)
    embed = synth.activations_bf16_torch(32000, d_m, seed=7000, device=dev)
    head = synth.weights_bf16_torch(256, d_m, seed=7001, device=dev)

    def run(E, eps_seed, **mkw):
        model = dyq.Model(layers, norms, norms, one, embed, head, E=E, n_heads=32, **mkw)
        cal = dyq.default_calib()
        pst = torch.zeros(dyq.state_size(E, cal), dtype=torch.uint8, device=dev)
        dyq.state_init(E, cal, pst)
        vis = synth.activations_bf16_torch(E * 256, d_m, seed=eps_seed, device=dev)
        gen = torch.Generator(device=dev).manual_seed(eps_seed + 100)
        text = torch.randint(0, 32000, (E, 32), dtype=torch.int32, device=dev, generator=gen)
        act_o = torch.zeros(E, 7, dtype=torch.float32, device=dev)
        bits_o = torch.zeros(E, dtype=torch.int32, device=dev)
        for _ in range(2):
            model.step(pst, E, vis, text, act_o, bits_o)
        torch.cuda.synchronize()
        R = 3
        sp = torch.cuda.Stream()
        gp = torch.cuda.CUDAGraph()
        sp.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(gp, stream=sp):
            for _ in range(R):
                model.step(pst, E, vis, text, act_o, bits_o, stream=sp)
        gp.replay()
        torch.cuda.synchronize()
        ms = statistics.median(timed(gp) for _ in range(3)) / R
        del gp, model
        torch.cuda.empty_cache()
        return ms

    pres = {}
    if world == 1:
        for E in [int(e) for e in args.policy_E.split(",")]:
            ms = run(E, 7100 + rank)
            pres[f"E{E}"] = {"episodes_per_gpu": E, "ms_per_step": round(ms, 3),
                            "policy_steps_per_s": round(E / (ms * 1e-3), 2)}
        # paper mode: selector on a side stream overlapping the
        # prefill, prefill at BF16, decode at b*_t
        ms = run(1, 7100 + rank, paper_mode=1, prefill_bits=16)
        pres["E1_paper_mode"] = {"episodes_per_gpu": 1, "ms_per_step": round(ms, 3),
                                 "policy_steps_per_s": round(1 / (ms * 1e-3), 2),
                                 "what": "dyq_policy_step paper_mode=1: prefill at BF16 (fixed), select_bits on a "
                                         "forked stream joined before the decode passes"}
    Et = args.policy_E_total
    mine = episodes.shard(Et, world, rank)
    ms = run(len(mine), 7100 + mine.start) if len(mine) else 0.0
    ms = ctl.reduce(ms)
    pres[f"E{Et}_total"] = {"episodes_total": Et, "episodes_per_rank": len(mine), "n_ranks": world,
                            "ms_per_step": round(ms, 3), "policy_steps_per_s": round(Et / (ms * 1e-3), 2),
                            "scaling": "strong (episodes sharded over ranks, episodes.shard)"}
    return {"workload": "configs[3] slice: dyq_policy_step, OpenVLA-7B shapes (32 blocks, d=4096, "
                        "ffn=11008, 32 heads), 256 vision + 32 text tokens, 7 action tokens, W4 G64, "
                        "per-episode b* from the kinematic dispatcher",
            "value_unit": "policy steps/s (whole job: episodes x steps / max-over-ranks time)",
            "results": pres, "timing": "cuda events around a graph of 3 steps (median of 3)"}


def e2e_leg(args, dyq, torch, dev, lins, packed, xs, ys, wss, state, row_bits, acts, t_cur, C, ctl, bytes_step,
            world):
    """The step through the public API with host buffers: per step one pinned
    H2D copy of [a_{t-1} | x_qkv | x_o | x_gate_up | x_down], select_route,
    4 x dyq_qlinear, one D2H copy of [y_down | b*]; captured per step index in
    a CUDA graph (eager figure alongside)."""
    M = args.M
    HP = 32  # int16 elements of the action header (64 B)
    sizes = [xs[0][li].numel() for li in range(len(lins))]
    offs = [HP + sum(sizes[:li]) for li in range(len(lins))]
    tot = HP + sum(sizes)
    in_host = []
    for k in range(8):
        hb = torch.zeros(tot, dtype=torch.int16).pin_memory()
        for li in range(len(lins)):
            hb[offs[li]:offs[li] + sizes[li]] = xs[k][li].reshape(-1).view(torch.int16).cpu()
        in_host.append(hb)
    in_dev = torch.empty(tot, dtype=torch.int16, device=dev)
    a_dev = in_dev[:14].view(torch.float32).view(1, 7)
    x_dev = [in_dev[offs[li]:offs[li] + sizes[li]].view(torch.bfloat16).view(xs[0][li].shape)
             for li in range(len(lins))]
    n_last = lins[-1][1]
    out_dev = torch.empty(M * n_last + 2, dtype=torch.int16, device=dev)
    y_dev = out_dev[:M * n_last].view(torch.bfloat16).view(M, n_last)
    b_dev = out_dev[M * n_last:].view(torch.int32)
    out_host = torch.empty_like(out_dev, device="cpu").pin_memory()
    a_host = acts.cpu().numpy().reshape(-1, 7)
    # the host's per-step write of a_{t-1}: numpy views of the pinned staging
    # buffers (a plain 28-byte store, no tensor-op dispatch)
    a_stage = [hb.numpy()[:14].view("float32") for hb in in_host]
    h2d = tot * 2
    d2h = out_host.numel() * 2
    n_e2e = min(args.steps, 200)

    side = torch.cuda.Stream()

    def e2e_step(k, stream=None, split=False):
        # graph form (split): H2D in two parts, [a_{t-1} | x_qkv] ahead of the
        # selector on the step's stream, the other linears' inputs on a side
        # stream overlapping the selector and QKV, joined before the o
        # projection (graph e2e 1203 -> 1233 GB/s same session); eager: one copy
        # (the host-side fork / join costs more than it hides there)
        cur = stream if stream is not None else torch.cuda.current_stream()
        hb = in_host[k]
        if split:
            in_dev[:offs[1]].copy_(hb[:offs[1]], non_blocking=True)
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                in_dev[offs[1]:].copy_(hb[offs[1]:], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
        else:
            in_dev.copy_(hb, non_blocking=True)
        dyq.select_route(state, 1, a_dev, b_dev, M, row_bits, stream=stream)
        for li in range(len(lins)):
            if li == 1 and split:
                cur.wait_event(ev)
            p = packed[k % C][li]
            yo = y_dev if li == len(lins) - 1 else ys[li]
            dyq.qlinear(p.wd, p.codes, p.meta, x_dev[li], M, row_bits, 0, yo, 1, wss[li], stream=stream)
        out_host.copy_(out_dev, non_blocking=True)

    t0 = t_cur + args.steps * (args.trials + 2)
    cs = torch.cuda.current_stream()  # the step's stream (one object, not one per step)
    ctl.barrier()
    torch.cuda.synchronize()
    tc = time.perf_counter()
    for i in range(n_e2e):
        t = t0 + i
        a_stage[t % 8][:] = a_host[min(t - 1, len(a_host) - 1)]
        e2e_step(t % 8)
        cs.synchronize()
    dt_eager = ctl.reduce((time.perf_counter() - tc) / n_e2e)
    se = torch.cuda.Stream()
    graphs = []
    for k in range(8):
        ge = torch.cuda.CUDAGraph()
        se.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(ge, stream=se):
            e2e_step(k, stream=se, split=True)
        graphs.append(ge)
    torch.cuda.synchronize()
    ctl.barrier()
    torch.cuda.synchronize()
    tc = time.perf_counter()
    for i in range(n_e2e):
        t = t0 + i
        a_stage[t % 8][:] = a_host[min(t - 1, len(a_host) - 1)]
        graphs[t % 8].replay()  # enqueued on the current stream
        cs.synchronize()
    dt = ctl.reduce((time.perf_counter() - tc) / n_e2e)
    del graphs
    return {"value": round(bytes_step * world / dt / 1e9, 2), "unit": "GB/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": round(dt * 1e3, 4), "steps": n_e2e,
            "path": "public API (select_route + 4 x dyq_qlinear) captured per step index in a CUDA graph with "
                    "the pinned H2D copy of the step's inputs [a_{t-1} | x x 4] in two parts ([a_{t-1} | x_qkv] "
                    "first, the rest on a side stream joined before the o projection) and one D2H copy of [y | b*]; "
                    "per step: host writes a_{t-1} into the pinned staging buffer, graph replay, stream sync",
            "eager": {"value": round(bytes_step * world / dt_eager / 1e9, 2),
                      "ms_per_step": round(dt_eager * 1e3, 4),
                      "path": "eager dyq_* calls via the Python binding, same staging buffers, sync per step"}}


if __name__ == "__main__":
    main()
