#!/usr/bin/env python
"""bench.py -- DyQ-VLA runtime-switchable qlinear hot path on B200.

Workload (BASELINE.json configs[1], the config the metric's "qlinear HBM GB/s"
is quoted on): one Llama-2-7B-shaped block (d=4096, ffn=11008) at decode,
M action tokens (default 8), W4 (the paper's INT4-pinned weights).
One STEP = one pass of the whole hot path for one control step:
    dyq_select_route (kinematic proxies -> S_t -> Alg. 1 on a[t-1], then
    b* -> per-token activation bits through the W4-pinned table, one kernel)
    -> for QKV, o, gate|up, down: dyq_act_quant + dyq_qlinear_q
with b* chosen each step by the kinematic dispatcher from a synthetic
LIBERO-shaped trajectory (120 untimed history steps first).
L2 is defeated by rotating 8 packed copies of the block (8 x 117 MB > 126 MB).

value = algorithmic bytes per step (packed weight codes + metadata + bf16
activations in + bf16 outputs) / device time per step, summed
over ranks / max-over-ranks time (weak scaling: every rank runs its own
episodes with replicated weights, no collective on the data path).

--impl reference times the CPU oracle (oracle/, plain C) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
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
    p.add_argument("--policy-E", default="1,8", help="episodes per GPU for the policy slice")
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


def algo_bytes(N, K, M, G, wbits):
    """N*K*wbits/8 + N*(K/G)*5 + M*K*2 + M*N*2."""
    return N * K * wbits // 8 + N * (K // G) * 5 + M * K * 2 + M * N * 2


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


# ------------------------------------------------------------ reference
def run_reference(args, rank):
    """The oracle as it stands, on host cores, on a bounded sample of the same
    workload and metric (GB/s of algorithmic qlinear bytes)."""
    if rank != 0:
        return
    import numpy as np

    import oracle
    import synth
    M, G, wb = args.M, args.group, args.wbits
    # bounded sample: the first R rows of every linear of the block (same K),
    # sized so that (warmup + steps) reference steps fit in ~2 minutes
    rows = 16
    lins = synth.LLAMA_BLOCK_LINEARS
    Ws = {n: synth.weights_bf16(rows, K, seed=1 + i) for i, (n, N, K) in enumerate(lins)}
    Ps = {n: oracle.pack_weights(Ws[n], G, wb) for n, _, _ in lins}
    Xs = {n: synth.activations_bf16(M, K, seed=1000 + i) for i, (n, N, K) in enumerate(lins)}
    acts = synth.trajectories(1, HISTORY_STEPS + args.warmup + args.steps + 2)
    st = oracle.SelectState(1)
    for t in range(HISTORY_STEPS):
        st.step(None if t == 0 else acts[t - 1])

    def one(t):
        b = int(st.step(acts[t - 1])["bits"][0])
        for n, N, K in lins:
            aq = oracle.act_quant(Xs[n], G, b)
            oracle.qlinear(Xs[n], Ps[n], G, b, actq=aq)

    t0 = HISTORY_STEPS
    tc = time.perf_counter()
    one(t0)
    per = time.perf_counter() - tc
    budget = 120.0
    scale = max(1, int(per * (args.warmup + args.steps) / budget + 0.999))
    steps = max(1, args.steps // scale)
    for i in range(min(args.warmup, 3)):
        one(t0 + 1 + i)
    tc = time.perf_counter()
    for i in range(steps):
        one(t0 + 4 + i)
    dt = (time.perf_counter() - tc) / steps
    bytes_step = sum(algo_bytes(rows, K, M, G, wb) for _, _, K in lins)
    val = bytes_step / dt / 1e9
    sample = (f"first {rows} rows of each of the 4 block linears (K=4096/11008), M={M}, W{wb} G={G}, "
              f"select_bits+act_quant+qlinear per step; {steps} timed steps (of {args.steps} requested)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC,
        "value": round(val, 4), "unit": "GB/s", "higher_is_better": True, "n_gpus": args.gpus,
        "steps": steps, "warmup": min(args.warmup, 3), "ms_per_step": dt * 1e3,
        "dtype": "int64/f64 (oracle)", "data": "synthetic",
        "config": make_config(args, args.copies, args.gpus),
        "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "vs_baseline": None,
    }), flush=True)


def cpu_baseline(args, w_host, budget_s=15.0):
    """Oracle on this box's host cores: full-size o-proj + down (rows sampled)
    step of the block, as many steps as fit ~budget_s (>= 1)."""
    import numpy as np

    import oracle
    import synth
    M, G, wb = args.M, args.group, args.wbits
    rows = 256
    tot_bytes, tot_t, n_done = 0, 0.0, 0
    t_start = time.perf_counter()
    packs = {}
    for name, N, K in synth.LLAMA_BLOCK_LINEARS:
        packs[name] = oracle.pack_weights(w_host[name][:rows], G, wb)
    xs = {name: synth.activations_bf16(M, K, seed=1000 + i)
          for i, (name, N, K) in enumerate(synth.LLAMA_BLOCK_LINEARS)}
    while n_done < 1 or (time.perf_counter() - t_start) < budget_s:
        for name, N, K in synth.LLAMA_BLOCK_LINEARS:
            tc = time.perf_counter()
            aq = oracle.act_quant(xs[name], G, 8)
            oracle.qlinear(xs[name], packs[name], G, 8, actq=aq)
            tot_t += time.perf_counter() - tc
            tot_bytes += algo_bytes(rows, K, M, G, wb)
        n_done += 1
    return {"value": round(tot_bytes / tot_t / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"first {rows} rows of each block linear (full K), M={M}, A8 W{wb} G={G}, "
                      f"act_quant+qlinear, {n_done} block passes ({tot_t:.1f} s)"}


# ------------------------------------------------------------------- main
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_2603_07904_b200 import dyq, episodes
    from paper_2603_07904_b200 import build as _b
    _b.build()

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    M, G, WB, C = args.M, args.group, args.wbits, args.copies
    if args.profile:
        C = min(C, 2)
    lins = synth.LLAMA_BLOCK_LINEARS

    # ---- packed block copies (weights replicated on every rank)
    packed = [[None] * len(lins) for _ in range(C)]
    w_host = {}
    for c in range(C):
        for li, (name, N, K) in enumerate(lins):
            w = synth.weights_bf16_torch(N, K, seed=1 + 4 * c + li, device=dev)
            if c == 0 and rank == 0:
                w_host[name] = w[:256].cpu().numpy().view(np.uint16).copy()
            packed[c][li] = dyq.PackedLinear.from_bf16(w, group=G, wbits=WB)
            del w
    torch.cuda.synchronize()

    # ---- activations (8 rotating sets), outputs, workspaces
    xs = [[synth.activations_bf16_torch(M, K, seed=1000 + 4 * s + li + 100 * rank, device=dev)
           for li, (_, _, K) in enumerate(lins)] for s in range(8)]
    ys = [torch.empty(M, N, dtype=torch.bfloat16, device=dev) for (_, N, _) in lins]
    wss = [packed[0][li].workspace(M) for li in range(len(lins))]

    # ---- kinematic state and trajectory (episode seed per rank)
    T = HISTORY_STEPS + args.warmup + args.steps * (args.trials + 1) + 2
    my_eps = episodes.shard(world, world, rank)  # one episode (control stream) per rank
    acts_np = synth.trajectories(1, T, seed0=episodes.episode_seed(my_eps[0]))
    acts = torch.from_numpy(acts_np).to(dev)
    cal = dyq.default_calib()
    state = torch.zeros(dyq.state_size(1, cal), dtype=torch.uint8, device=dev)
    dyq.state_init(1, cal, state)
    bits = torch.zeros(1, dtype=torch.int32, device=dev)
    row_bits = torch.zeros(M, dtype=torch.int32, device=dev)
    for t in range(HISTORY_STEPS):
        dyq.select_bits(state, 1, None if t == 0 else acts[t - 1], bits)
    t_cur = HISTORY_STEPS

    bytes_step = sum(algo_bytes(N, K, M, G, WB) for _, N, K in lins)
    gate_li = [n for n, _, _ in lins].index("gate_up")
    n_launch_step = 1 + 2 * len(lins)  # select_route, then act-quant + qlinear kernel per linear

    def step(t, fixed_bits=None, ev=None):
        c = t % C
        if fixed_bits is None:
            dyq.select_route(state, 1, acts[t - 1], bits, M, row_bits)
            rb, b = row_bits, 0
        else:
            rb, b = None, fixed_bits
        for li, (name, N, K) in enumerate(lins):
            p = packed[c][li]
            x = xs[t % 8][li]
            if ev is not None and li == gate_li:
                ev[0].record()
            dyq.qlinear(p.wd, p.codes, p.meta, x, M, rb, b, ys[li], 1, wss[li])
            if ev is not None and li == gate_li:
                ev[1].record()

    # ---- warm-up (eager), then capture the K-step region as one CUDA graph
    for i in range(args.warmup):
        step(t_cur)
        t_cur += 1
    torch.cuda.synchronize()

    def capture(n_steps, t0, fixed_bits=None, with_events=True):
        g = torch.cuda.CUDAGraph()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(n_steps)] if with_events else None
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(g, stream=s):
            for i in range(n_steps):
                step(t0 + i, fixed_bits, evs[i] if evs else None)
        torch.cuda.synchronize()
        return g, evs

    events_ok = True
    try:
        graph, evs = capture(args.steps, t_cur)
    except Exception as e:  # events inside capture unsupported -> time without them
        events_ok = False
        sys.stderr.write(f"[bench] graph capture with events failed ({e}); retrying without\n")
        graph, evs = capture(args.steps, t_cur, with_events=False)

    def timed(g):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        return episodes.max_over_ranks(e0.elapsed_time(e1), device=dev)

    graph.replay()  # one untimed replay (warm graph)
    torch.cuda.synchronize()
    trial_ms, kern_ms = [], []
    with ClockSampler(local) as clk:
        for _ in range(args.trials):
            ms = timed(graph)
            trial_ms.append(ms)
            if events_ok and evs:
                try:
                    kern_ms.append(sum(a.elapsed_time(b) for a, b in evs) / len(evs))
                except Exception as e:
                    sys.stderr.write(f"[bench] in-graph event timing unavailable: {e}\n")
                    events_ok = False
    ms_total = statistics.median(trial_ms)
    ms_step = ms_total / args.steps
    value = episodes.throughput(bytes_step, ms_step * 1e-3) / 1e9  # all ranks' bytes / slowest rank

    # ---- bits histogram over the timed steps (read back once, outside timing)
    hist = {}
    st2 = torch.zeros_like(state)
    dyq.state_init(1, cal, st2)
    bb = torch.zeros(1, dtype=torch.int32, device=dev)
    for t in range(t_cur + args.steps):
        dyq.select_bits(st2, 1, None if t == 0 else acts[t - 1], bb)
        if t >= t_cur:
            k = int(bb.item())
            hist[k] = hist.get(k, 0) + 1

    # ---- roofline of the dominant kernel (decode qlinear on gate|up)
    N_g, K_g = lins[gate_li][1], lins[gate_li][2]
    gate_bytes = algo_bytes(N_g, K_g, M, G, WB)
    peak, peak_kind = hbm_peak()
    call_ms = None
    if kern_ms:
        k_ms = statistics.median(kern_ms)
        k_src = "cuda events around the gate|up qlinear inside the timed graph"
    else:
        # events recorded inside a captured graph cannot be timed: time the
        # gate|up qlinear (act-quant + decode kernels) per activation width in a
        # graph of R back-to-back launches (rotating copies), and weight the
        # widths by the timed region's b* histogram (W4-pinned table: b* = abits)
        R = 64
        k_by_bits = {}
        for b in sorted(hist):
            g3 = torch.cuda.CUDAGraph()
            s3 = torch.cuda.Stream()
            s3.wait_stream(torch.cuda.current_stream())
            with torch.cuda.graph(g3, stream=s3):
                for r in range(R):
                    p = packed[r % C][gate_li]
                    dyq.qlinear(p.wd, p.codes, p.meta, xs[0][gate_li], M, None, b, ys[gate_li], 1, wss[gate_li])
            g3.replay()
            torch.cuda.synchronize()
            k_by_bits[b] = statistics.median(timed(g3) for _ in range(5)) / R
            del g3
        n_h = sum(hist.values())
        call_ms = sum(k_by_bits[b] * hist[b] / n_h for b in hist)
        # the decode kernel alone: R back-to-back dyq_qlinear_q launches (the same
        # kernel) on activations quantized once by dyq_act_quant -- the dominant
        # kernel's launch duration, without the act-quant kernel between launches
        q_by_bits = {}
        for b in sorted(hist):
            p0 = packed[0][gate_li]
            dyq.act_quant(p0.wd, xs[0][gate_li], M, None, b, wss[gate_li])
            g4 = torch.cuda.CUDAGraph()
            s4 = torch.cuda.Stream()
            s4.wait_stream(torch.cuda.current_stream())
            with torch.cuda.graph(g4, stream=s4):
                for r in range(R):
                    p = packed[r % C][gate_li]
                    dyq.qlinear_q(p.wd, p.codes, p.meta, xs[0][gate_li], M, None, b, ys[gate_li], 1, wss[gate_li])
            g4.replay()
            torch.cuda.synchronize()
            q_by_bits[b] = statistics.median(timed(g4) for _ in range(5)) / R
            del g4
        k_ms = sum(q_by_bits[b] * hist[b] / n_h for b in hist)
        k_src = (f"cuda events around graphs of {R} back-to-back qlinear_decode_kernel launches (dyq_qlinear_q, "
                 f"rotating copies) per width { {b: round(v * 1e3, 2) for b, v in q_by_bits.items()} } us, weighted "
                 f"by the timed b* histogram; per dyq_qlinear call incl. the act-quant kernel: "
                 f"{ {b: round(v * 1e3, 2) for b, v in k_by_bits.items()} } us")
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_decode_summary.json")))
        traffic = prof.get("dram_bytes_per_launch", {}).get(f"gate_up_M{M}_W{WB}")
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": "qlinear_decode_kernel (gate|up 22016x4096)",
                "achieved": round(gate_bytes / (k_ms * 1e-3) / 1e9, 1) if k_ms else None,
                "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": round(gate_bytes / (k_ms * 1e-3) / 1e9 / peak, 4) if k_ms else None,
                "traffic": traffic, "algorithmic_bytes_per_launch": gate_bytes,
                "kernel_ms": round(k_ms, 5) if k_ms else None, "timing": k_src}
    if not kern_ms:
        roofline["call_ms"] = round(call_ms, 5)
        roofline["call_frac"] = round(gate_bytes / (call_ms * 1e-3) / 1e9 / peak, 4)

    # ---- per-variant table (fixed widths), W4 and the optional W8 copy
    variants = {}
    if not args.no_variants and not args.profile:
        for b in (2, 4, 8, 16):
            g2, _ = capture(64, t_cur, fixed_bits=b, with_events=False)
            g2.replay()
            ms = statistics.median(timed(g2) for _ in range(3)) / 64
            variants[f"W{WB}A{b}"] = {
                "GB/s": round(bytes_step / (ms * 1e-3) / 1e9, 1),
                "int_TOPS" if b != 16 else "TFLOPS": round(
                    sum(2 * M * N * K for _, N, K in lins) / (ms * 1e-3) / 1e12, 3),
                "us_per_block": round(ms * 1e3, 2)}
            del g2

    # ---- configs[2] slice: prefill of one block at M = 288 tokens (256 vision +
    # 32 text) with the step's b*, on the tcgen05 path (tensor-bound)
    prefill = None
    if not args.profile and not args.no_prefill:
        MP = 288
        xps = [synth.activations_bf16_torch(MP, K, seed=5000 + li, device=dev) for li, (_, _, K) in enumerate(lins)]
        yps = [torch.empty(MP, N, dtype=torch.bfloat16, device=dev) for (_, N, _) in lins]
        wps = [packed[0][li].workspace(MP) for li in range(len(lins))]
        rbp = torch.zeros(MP, dtype=torch.int32, device=dev)

        def pstep(t, fixed_bits=None):
            if fixed_bits is None:
                dyq.route_bits(bits, 1, MP, rbp)
                rb, b = rbp, 0
            else:
                rb, b = None, fixed_bits
            for li in range(len(lins)):
                p = packed[t % C][li]
                dyq.qlinear(p.wd, p.codes, p.meta, xps[li], MP, rb, b, yps[li], 1, wps[li])

        ops_block = sum(2 * MP * N * K for _, N, K in lins)
        i8_peak = 4500.0  # TOPS, nominal dense int8 (north_star: integer tensor-pipe peak)
        bf16_peak = float((peaks() or {}).get("bf16_tflops", 2250.0))
        pres = {}
        for fb in (None, 2, 4, 8, 16):
            for i in range(2):
                pstep(i, fb)
            torch.cuda.synchronize()
            gp = torch.cuda.CUDAGraph()
            sp = torch.cuda.Stream()
            sp.wait_stream(torch.cuda.current_stream())
            RP = 10
            with torch.cuda.graph(gp, stream=sp):
                for i in range(RP):
                    pstep(i, fb)
            gp.replay()
            torch.cuda.synchronize()
            ms = statistics.median(timed(gp) for _ in range(3)) / RP
            tops = ops_block / (ms * 1e-3) / 1e12
            pres["step_bits" if fb is None else f"W{WB}A{fb}"] = {
                "us_per_block": round(ms * 1e3, 1), "int_TOPS": round(tops, 1),
                "frac_i8_nominal": round(tops / i8_peak, 4), "frac_bf16_pipe": round(tops / bf16_peak, 4)}
            del gp
        prefill = {"workload": "configs[2] slice: one Llama-2-7B block prefill, M=288 (256 vision + 32 text), "
                               f"W{WB} G={G}, b* of the current step; whole backbone = 32 x this",
                   "kernel": "qlinear_prefill_kernel (tcgen05 kind::f16, exact integer operands, A in TMEM)",
                   "peak_i8_TOPS": i8_peak, "peak_bf16_TFLOPS": bf16_peak, "results": pres,
                   "timing": "cuda events around a graph of 10 blocks (median of 3)"}

    # ---- configs[3] slice: whole VLA policy steps/s (dyq_policy_step: select_bits,
    # 288-token prefill and 6 decode passes through 32 Llama-2-7B blocks, action
    # head + detok) for E episodes on this rank; layers cycle through the C
    # packed block copies (all distinct from L2's point of view)
    policy = None
    if not args.profile and not args.no_policy:
        d_m, NL = 4096, 32
        layers = [packed[l % C] for l in range(NL)]
        one = torch.full((d_m,), 0x3F80, dtype=torch.int16, device=dev)        # bf16 1.0
        norms = one.repeat(NL)
        embed = synth.activations_bf16_torch(32000, d_m, seed=7000, device=dev)
        head = synth.weights_bf16_torch(256, d_m, seed=7001, device=dev)
        pres = {}
        for E in [int(e) for e in args.policy_E.split(",")]:
            model = dyq.Model(layers, norms, norms, one, embed, head, E=E, n_heads=32)
            cal = dyq.default_calib()
            pst = torch.zeros(dyq.state_size(E, cal), dtype=torch.uint8, device=dev)
            dyq.state_init(E, cal, pst)
            vis = synth.activations_bf16_torch(E * 256, d_m, seed=7100 + rank, device=dev)
            gen = torch.Generator(device=dev).manual_seed(7200 + rank)
            text = torch.randint(0, 32000, (E, 32), dtype=torch.int32, device=dev, generator=gen)
            act_o = torch.zeros(E, 7, dtype=torch.float32, device=dev)
            bits_o = torch.zeros(E, dtype=torch.int32, device=dev)
            for _ in range(2):
                model.step(pst, E, vis, text, act_o, bits_o)
            torch.cuda.synchronize()
            R = 3
            gp = torch.cuda.CUDAGraph()
            sp = torch.cuda.Stream()
            sp.wait_stream(torch.cuda.current_stream())
            with torch.cuda.graph(gp, stream=sp):
                for _ in range(R):
                    model.step(pst, E, vis, text, act_o, bits_o, stream=sp)
            gp.replay()
            torch.cuda.synchronize()
            ms = statistics.median(timed(gp) for _ in range(3)) / R
            sps = episodes.throughput(E, ms * 1e-3)
            pres[f"E{E}"] = {"episodes_per_gpu": E, "ms_per_step": round(ms, 3),
                            "policy_steps_per_s": round(sps, 2)}
            del gp, model
            torch.cuda.empty_cache()
        # offline calibration collection (NEXT-3): Ec streams, one batched step of
        # 4 Ec replicas at b = 16 | 2 | 4 | 8 per calibration step
        Ec = 2
        model = dyq.Model(layers, norms, norms, one, embed, head, E=4 * Ec, n_heads=32)
        cal = dyq.default_calib()
        pst = torch.zeros(dyq.state_size(Ec, cal), dtype=torch.uint8, device=dev)
        dyq.state_init(Ec, cal, pst)
        vis = synth.activations_bf16_torch(Ec * 256, d_m, seed=7300 + rank, device=dev)
        gen = torch.Generator(device=dev).manual_seed(7400 + rank)
        text = torch.randint(0, 32000, (Ec, 32), dtype=torch.int32, device=dev, generator=gen)
        acts_c = torch.zeros(4 * Ec, 7, dtype=torch.float32, device=dev)
        S_c = torch.zeros(Ec, dtype=torch.float64, device=dev)
        e_c = torch.zeros(Ec, 3, dtype=torch.float64, device=dev)
        for _ in range(2):
            model.calib_collect(pst, Ec, vis, text, acts_c, S_c, e_c)
        torch.cuda.synchronize()
        R = 3
        gp = torch.cuda.CUDAGraph()
        sp = torch.cuda.Stream()
        sp.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(gp, stream=sp):
            for _ in range(R):
                model.calib_collect(pst, Ec, vis, text, acts_c, S_c, e_c, stream=sp)
        gp.replay()
        torch.cuda.synchronize()
        ms = statistics.median(timed(gp) for _ in range(3)) / R
        pres[f"calib_Ec{Ec}"] = {"streams_per_gpu": Ec, "replicas": 4 * Ec, "ms_per_step": round(ms, 3),
                                 "calib_steps_per_s": round(episodes.throughput(Ec, ms * 1e-3), 2),
                                 "what": "dyq_calib_collect: S_t + a* + a^(2,4,8) + e^(b) per stream-step"}
        del gp, model
        torch.cuda.empty_cache()
        policy = {"workload": "configs[3] slice: dyq_policy_step, OpenVLA-7B shapes (32 blocks, d=4096, "
                              "ffn=11008, 32 heads), 256 vision + 32 text tokens, 7 action tokens, W4 G64, "
                              "per-episode b* from the kinematic dispatcher",
                  "value_unit": "policy steps/s (whole job: episodes x steps / max-over-ranks time)",
                  "results": pres, "timing": "cuda events around a graph of 3 steps (median of 3)"}

    # ---- e2e through the public API: pinned H2D of the step's inputs, eager
    # launches, D2H of the step's result (block output y and b*), per step
    e2e = None
    if not args.profile:
        # one pinned staging buffer per step index k = t % 8: [a_{t-1} (7 f32,
        # padded to 64 B) | x_qkv | x_o | x_gate_up | x_down] (bf16 bits), one H2D
        # copy per step into the same layout on the device; the step's result
        # [y_down | b*] comes back in one D2H copy
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
        a_host = acts.cpu()
        h2d = tot * 2
        d2h = out_host.numel() * 2
        n_e2e = min(args.steps, 200)

        def e2e_step(k, stream=None):
            in_dev.copy_(in_host[k], non_blocking=True)
            dyq.select_route(state, 1, a_dev, b_dev, M, row_bits, stream=stream)
            for li, (name, N, K) in enumerate(lins):
                p = packed[k % C][li]
                yo = y_dev if li == len(lins) - 1 else ys[li]
                dyq.qlinear(p.wd, p.codes, p.meta, x_dev[li], M, row_bits, 0, yo, 1, wss[li], stream=stream)
            out_host.copy_(out_dev, non_blocking=True)

        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        tc = time.perf_counter()
        for i in range(n_e2e):
            t = t_cur + args.steps + i
            in_host[t % 8][:14].view(torch.float32).copy_(a_host[t - 1].reshape(-1))
            e2e_step(t % 8)
            torch.cuda.current_stream().synchronize()
        dt_eager = episodes.max_over_ranks((time.perf_counter() - tc) / n_e2e, device=dev)
        # the same public-API step captured as a CUDA graph, one per step index k
        # (input set k, weight copy k % C): H2D of the staging buffer,
        # select_route, 4 x dyq_qlinear, D2H of [y | b*].  Per step the host
        # writes a_{t-1} into staging buffer t % 8, replays graph t % 8 and waits.
        assert 8 % C == 0 or C % 8 == 0
        se = torch.cuda.Stream()
        graphs = []
        for k in range(8):
            ge = torch.cuda.CUDAGraph()
            se.wait_stream(torch.cuda.current_stream())
            with torch.cuda.graph(ge, stream=se):
                e2e_step(k, stream=se)
            graphs.append(ge)
        torch.cuda.synchronize()
        t_e = t_cur + args.steps + n_e2e
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        tc = time.perf_counter()
        for i in range(n_e2e):
            t = t_e + i
            in_host[t % 8][:14].view(torch.float32).copy_(a_host[t - 1].reshape(-1))
            graphs[t % 8].replay()  # enqueued on the current stream
            torch.cuda.current_stream().synchronize()
        dt = episodes.max_over_ranks((time.perf_counter() - tc) / n_e2e, device=dev)
        del graphs
        e2e = {"value": round(bytes_step * world / dt / 1e9, 2), "unit": "GB/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": round(dt * 1e3, 4), "steps": n_e2e,
               "path": "public API (select_route + 4 x dyq_qlinear) captured per step index in a CUDA graph with "
                       "one pinned H2D copy of the step's inputs [a_{t-1} | x x 4] and one D2H copy of [y | b*]; "
                       "per step: host writes a_{t-1} into the pinned staging buffer, graph replay, stream sync",
               "eager": {"value": round(bytes_step * world / dt_eager / 1e9, 2),
                         "ms_per_step": round(dt_eager * 1e3, 4),
                         "path": "eager dyq_* calls via the Python binding, same staging buffers, sync per step"}}

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
                           timed=f"median of {args.trials} replays of one CUDA graph of {args.steps} steps"),
            "gpu_launches": n_launch_step * args.steps,
            "bytes_per_step": bytes_step,
            "bits_hist_timed": {str(k): v for k, v in sorted(hist.items())},
            "roofline": roofline,
            "variants": variants,
            "prefill": prefill,
            "policy": policy,
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "trial_ms": [round(x, 4) for x in trial_ms],
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
