"""SPEC toy environment, step-wise sensitivity profiler and closed-loop
harness -- a desk-scale closed loop
around the B200 hot path.

The environment (`envpolicy`) is a deterministic point-mass
manipulator: an end effector moves to an object (Transit: large saturated
translations), closes in on it slowly with an oscillating wrist (Align: small
translations planned from the offset seen on arrival, high rotational jerk
-- the kinematic regimes of §III), closes the gripper (Grasp; the object attaches RIGIDLY at its current offset from
the effector), carries it to the goal (Place) and releases it (Done).  The
place controller steers the EFFECTOR to the goal, so an offset baked in while
aligning or grasping survives to the terminal deviation D_T, while a Transit
error is corrected on the way -- Eq. (3)'s error propagation by construction.

The policy (pi_theta of Eq. (1)) is a scripted controller whose feature
vector (64 values: the commanded action terms, gains, phase one-hot and
derived terms -- one K-group) runs through the hot path itself: the action is
`dyq_qlinear` of that feature row against a W4-packed read-out matrix, at the
step's activation bits (b = 16: the BF16 bypass, the full-precision
baseline; the weights stay INT4-pinned as in P:221).  The dispatcher is
`dyq_select_bits` on the episodes' previous actions.  Episodes are batched
(one row per episode), so one control step of E episodes is one decode
qlinear call and one selector call on the GPU; the environment dynamics and
the bookkeeping run on the host (they are the robot, not the method).

`head` and `dispatcher` are injectable (anything with the same call
signature), which is how the CPU tests drive this module with the oracle.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np

TRANSIT, ALIGN, GRASP, PLACE, DONE = 0, 1, 2, 3, 4
PHASES = ("Transit", "Align", "Grasp", "Place", "Done")
FEAT = 64  # feature vector = one K-group of the read-out linear
COST_MODEL = {16: 1.00, 8: 0.70, 4: 0.55, 2: 0.45}  # S:531 artifact defaults (not paper numbers)


@dataclasses.dataclass(frozen=True)
class EnvConfig:
    """workspace, per-step clip, grasp radius, success tolerance,
    max steps (artifact choices, not paper values)."""
    bound: float = 1.0
    clip: float = 0.05
    grasp_radius: float = 0.03
    success_tol: float = 0.02
    max_steps: int = 300
    align_radius: float = 0.1    # Transit -> Align
    transit_gain: float = 0.4    # Transit: per-axis saturated, proportional on the final approach
    align_gain: float = 0.3      # fine approach gain
    align_steps: int = 15        # Align -> Grasp after this many steps (or when converged)
    align_done: float = 0.004
    grasp_steps: int = 3
    place_gain: float = 0.3
    place_steps: int = 15        # fine placement length
    wrist_amp: float = 0.02      # Align / Grasp wrist oscillation amplitude (rad per step)
    wrist_period: int = 4
    ctx: float = 0.03            # context-feature magnitude (sets the activation group's range)


class State:
    """EnvState for E episodes as arrays."""

    def __init__(self, E: int):
        self.ee = np.zeros((E, 3))
        self.rot = np.zeros((E, 3))
        self.grip = np.zeros(E)
        self.obj = np.zeros((E, 3))
        self.goal = np.zeros((E, 3))
        self.phase = np.zeros(E, np.int64)
        self.step = np.zeros(E, np.int64)
        self.attached = np.zeros(E, bool)
        self.offset = np.zeros((E, 3))     # object - effector at attachment
        self.phase_t = np.zeros(E, np.int64)  # steps spent in the current phase
        self.d0 = np.zeros((E, 3))             # object - effector when Align began (the fine plan)
        self.near = np.zeros(E, bool)          # Place: within align_radius of the goal (fine placement)
        self.near_t = np.zeros(E, np.int64)
        self.d0p = np.zeros((E, 3))            # goal - effector when the fine placement began
        self.seed = np.zeros(E, np.int64)

    def copy(self) -> "State":
        s = State(0)
        for k, v in self.__dict__.items():
            setattr(s, k, v.copy())
        return s

    def take(self, idx) -> "State":
        s = State(0)
        for k, v in self.__dict__.items():
            setattr(s, k, v[idx].copy())
        return s


def reset(seeds: Sequence[int], cfg: EnvConfig = EnvConfig()) -> State:
    """deterministic initial state per seed; object, goal and
    effector uniformly inside the workspace, object and goal apart."""
    E = len(seeds)
    s = State(E)
    b = cfg.bound * 0.8
    for i, sd in enumerate(seeds):
        rng = np.random.default_rng(int(sd))
        s.ee[i] = rng.uniform(-b, b, 3)
        s.obj[i] = rng.uniform(-b, b, 3)
        g = rng.uniform(-b, b, 3)
        while np.linalg.norm(g - s.obj[i]) < 0.5:
            g = rng.uniform(-b, b, 3)
        s.goal[i] = g
        s.seed[i] = sd
    return s


def _clip_norm(v: np.ndarray, c: float) -> np.ndarray:
    n = np.linalg.norm(v, axis=-1, keepdims=True)
    return v * np.minimum(1.0, c / np.maximum(n, 1e-12))


def features(s: State, cfg: EnvConfig = EnvConfig()) -> np.ndarray:
    """The controller's intermediate feature vector [E, 64]:
    0:3 commanded translation, 3:6 wrist increment, 6 gripper command, then
    context: phase code, squashed geometry, gains and an oscillator bank."""
    E = s.ee.shape[0]
    f = np.zeros((E, FEAT))
    d_obj = s.obj - s.ee
    d_goal = s.goal - s.ee
    cmd = np.zeros((E, 3))
    wrist = np.zeros((E, 3))
    grip = np.zeros(E)
    tr = s.phase == TRANSIT
    al = s.phase == ALIGN
    gr = s.phase == GRASP
    pl = s.phase == PLACE
    # coarse motion: per-axis saturated steps toward the target (Transit, and
    # Place while far from the goal); fine motion: proportional (Align, Place
    # near the goal)
    cs = cfg.clip / math.sqrt(3.0)
    far_pl = pl & ~s.near
    cmd[tr] = np.clip(cfg.transit_gain * d_obj[tr], -cs, cs)
    # Align follows the fine approach planned from the offset seen when it
    # began (a geometric schedule, no re-observation): an error made while
    # aligning is never corrected and becomes the grasp offset
    cmd[al] = cfg.align_gain * (1.0 - cfg.align_gain) ** s.phase_t[al][:, None] * s.d0[al]
    cmd[far_pl] = np.clip(d_goal[far_pl], -cs, cs)
    near_pl = pl & s.near  # fine placement: planned like Align (no re-observation)
    cmd[near_pl] = cfg.place_gain * (1.0 - cfg.place_gain) ** s.near_t[near_pl][:, None] * s.d0p[near_pl]
    osc = np.sin(2 * math.pi * s.phase_t / cfg.wrist_period)[:, None] * np.array([1.0, -0.7, 0.5])
    wrist[al | gr] = cfg.wrist_amp * osc[al | gr]
    grip[gr] = 1.0
    grip[pl] = 1.0
    f[:, 0:3] = cmd
    f[:, 3:6] = wrist
    f[:, 6] = cfg.ctx * grip  # read out with weight 1 / ctx
    # context features (phase code, gains, geometry, an oscillator bank),
    # all scaled into [-ctx, ctx]: they set the dynamic range of the
    # activation group, so the fine-phase commands (a few mm) sit far below
    # its quantization step at low bits while the saturated Transit commands
    # (clip-sized) do not -- the sensitivity structure of §III
    c = cfg.ctx
    f[np.arange(E), 8 + s.phase] = c
    f[:, 13:16] = c * np.tanh(d_obj / cfg.bound)
    f[:, 16:19] = c * np.tanh(d_goal / cfg.bound)
    f[:, 19] = c * cfg.align_gain
    f[:, 20] = c * cfg.place_gain
    k = np.arange(21, FEAT)
    f[:, 21:] = c * np.sin(0.37 * k[None, :] * (1 + s.step[:, None] % 7) + 0.11 * s.seed[:, None])
    return f


def readout_weights(cfg: EnvConfig = EnvConfig()) -> np.ndarray:
    """[16, 64] fp32 read-out of the controller: action dim i <- feature i
    (7 rows; the gripper feature is stored scaled by ctx), padding rows
    7..15 zero.  Packed W4 by the hot path."""
    w = np.zeros((16, FEAT), np.float32)
    for i in range(6):
        w[i, i] = 1.0
    w[6, 6] = 1.0 / cfg.ctx
    return w


def env_step(s: State, a: np.ndarray, cfg: EnvConfig = EnvConfig()) -> State:
    """translation clipped, wrist integrates, gripper follows,
    rigid attachment, monotone phase advance.  Done episodes stay put."""
    s = s.copy()
    live = s.phase != DONE
    a = np.where(live[:, None], a, 0.0)
    s.ee = s.ee + _clip_norm(a[:, 0:3], cfg.clip)
    s.ee = np.clip(s.ee, -cfg.bound, cfg.bound)
    s.rot = s.rot + a[:, 3:6]
    s.grip = np.where(live, np.clip(a[:, 6], 0.0, 1.0), s.grip)
    s.obj = np.where(s.attached[:, None], s.ee + s.offset, s.obj)
    s.step = s.step + live
    s.phase_t = s.phase_t + live
    d_obj = np.linalg.norm(s.obj - s.ee, axis=1)
    nxt = s.phase.copy()
    nxt[(s.phase == TRANSIT) & (d_obj < cfg.align_radius)] = ALIGN
    nxt[(s.phase == ALIGN) & ((s.phase_t >= cfg.align_steps) | (d_obj < cfg.align_done))] = GRASP
    g_done = (s.phase == GRASP) & (s.phase_t >= cfg.grasp_steps)
    att = g_done & (d_obj <= cfg.grasp_radius) & (s.grip >= 0.5)
    s.offset = np.where(att[:, None], s.obj - s.ee, s.offset)
    s.attached = s.attached | att
    nxt[g_done] = PLACE
    # Place: coarse (closed loop) until the effector is within align_radius of
    # the goal, then the planned fine placement for place_steps steps; it
    # steers the EFFECTOR (the controller does not see the object offset).  A
    # missed grasp (nothing attached) ends the episode.
    d_goal_ee = np.linalg.norm(s.goal - s.ee, axis=1)
    in_pl = s.phase == PLACE
    s.near_t = np.where(in_pl & s.near, s.near_t + 1, s.near_t)
    start = in_pl & ~s.near & (d_goal_ee < cfg.align_radius)
    s.d0p = np.where(start[:, None], s.goal - s.ee, s.d0p)
    s.near = s.near | start
    nxt[in_pl & ((s.near & (s.near_t >= cfg.place_steps)) | ~s.attached)] = DONE
    s.attached = s.attached & (nxt != DONE)
    s.d0 = np.where(((nxt == ALIGN) & (s.phase != ALIGN))[:, None], s.obj - s.ee, s.d0)
    s.phase_t = np.where(nxt != s.phase, 0, s.phase_t)
    s.phase = nxt
    return s


def episode_status(s: State, cfg: EnvConfig = EnvConfig()):
    """(done, success, terminal deviation D_T)."""
    dev = np.linalg.norm(s.obj - s.goal, axis=1)
    done = (s.phase == DONE) | (s.step >= cfg.max_steps)
    success = done & (s.phase == DONE) & (dev <= cfg.success_tol)
    return done, success, dev


# --------------------------------------------------------------- hot path
class GpuHead:
    """policy_forward's quantized stage on the B200 hot path: the feature row
    of each episode (bf16) through dyq_qlinear against the W4-packed read-out,
    at that episode's activation bits (row_bits)."""

    def __init__(self, device: str = "cuda:0", group: int = 64):
        import torch

        from . import dyq
        self.torch, self.dyq, self.dev = torch, dyq, device
        w = torch.from_numpy(readout_weights()).to(device).to(torch.bfloat16).view(torch.int16)
        self.lin = dyq.PackedLinear.from_bf16(w, group=group, wbits=4)
        self._ws: Dict[int, object] = {}

    def __call__(self, f: np.ndarray, bits: np.ndarray) -> np.ndarray:
        torch, dyq = self.torch, self.dyq
        E = f.shape[0]
        if E == 0:
            return np.zeros((0, 7))
        if E not in self._ws:
            self._ws[E] = self.lin.workspace(E)
        x = torch.from_numpy(f.astype(np.float32)).to(self.dev).to(torch.bfloat16).view(torch.int16)
        rb = torch.from_numpy(np.asarray(bits, np.int32)).to(self.dev)
        y = torch.empty(E, 16, dtype=torch.float32, device=self.dev)
        dyq.qlinear(self.lin.wd, self.lin.codes, self.lin.meta, x, E, rb, 0, y, 0, self._ws[E])
        return y[:, :7].double().cpu().numpy()


class GpuDispatcher:
    """The kinematic dispatcher on the GPU: dyq_select_bits over E streams."""

    def __init__(self, E: int, calib=None, device: str = "cuda:0", lam: Optional[float] = None):
        import torch

        from . import dyq
        self.torch, self.dyq, self.dev, self.E = torch, dyq, device, E
        self.cal = calib if calib is not None else dyq.default_calib(**({} if lam is None else {"lambda_": lam}))
        self.state = torch.zeros(dyq.state_size(E, self.cal), dtype=torch.uint8, device=device)
        dyq.state_init(E, self.cal, self.state)
        self.bits = torch.zeros(E, dtype=torch.int32, device=device)
        self.S = torch.zeros(E, dtype=torch.float64, device=device)

    def step(self, prev: Optional[np.ndarray]) -> np.ndarray:
        torch = self.torch
        p = None if prev is None else torch.from_numpy(np.asarray(prev, np.float32)).to(self.dev)
        self.dyq.select_bits(self.state, self.E, p, self.bits, self.S)
        return self.bits.cpu().numpy().astype(np.int64)

    def step_S(self, prev: Optional[np.ndarray]) -> np.ndarray:
        self.step(prev)
        return self.S.cpu().numpy()


class Static:
    """static(b) mode: a fixed width every step."""

    def __init__(self, E: int, b: int):
        self.E, self.b = E, b

    def step(self, prev):
        return np.full(self.E, self.b, np.int64)


# ------------------------------------------------------------ closed loop
@dataclasses.dataclass
class Trace:
    """Per-step records (TrajectoryRecord) for E episodes."""
    actions: List[np.ndarray]
    bits: List[np.ndarray]
    phases: List[np.ndarray]
    live: List[np.ndarray]
    final_obj: Optional[np.ndarray] = None  # [E, 3] object positions at termination


def simulate(seeds: Sequence[int], head: Callable, dispatcher, cfg: EnvConfig = EnvConfig(),
             inject: Optional[Dict[int, int]] = None, cost_model=None):
    """simulate_episode for a batch of seeds: per step (1) bits
    from the dispatcher on actions <= t-1, (2) the policy at those bits,
    (3) env_step, (4) record.  `inject` = {t: bits}: overrides the bits of
    step t only (the profiler's single-step perturbation).
    Returns (success [E], D_T [E], steps [E], total_cost [E], Trace)."""
    cm = cost_model or COST_MODEL
    s = reset(seeds, cfg)
    E = len(seeds)
    prev = None
    tr = Trace([], [], [], [])
    cost = np.zeros(E)
    for t in range(cfg.max_steps):
        done, _, _ = episode_status(s, cfg)
        if done.all():
            break
        b = np.asarray(dispatcher.step(prev), np.int64)
        if inject and t in inject:
            b = np.full(E, inject[t], np.int64)
        a = head(features(s, cfg), b)
        live = ~done
        a = np.where(live[:, None], a, 0.0)
        cost += np.where(live, np.vectorize(cm.get)(b), 0.0)
        tr.actions.append(a)
        tr.bits.append(b)
        tr.phases.append(s.phase.copy())
        tr.live.append(live)
        s = env_step(s, a, cfg)
        prev = a.astype(np.float32)
    done, success, dev = episode_status(s, cfg)
    tr.final_obj = s.obj.copy()
    return success, dev, s.step.copy(), cost, tr


def perturb_at(seeds, t: int, bits: int, head, cfg: EnvConfig = EnvConfig(), base: Optional[Trace] = None):
    """perturb_at: BF16 everywhere except step t at `bits`.
    Returns (e_t [E], D_T [E], success [E]) with e_t = ||p_q - p_bf16||_2 the
    translation error of the injected action (p = the commanded
    position increment) and D_T = the terminal object displacement from the
    baseline episode, i.e. the terminal spatial deviation caused by the
    perturbation (DESIGN reading T1).  `base`: the seeds' baseline
    trace when already computed."""
    E = len(seeds)
    if base is None:
        _, _, _, _, base = simulate(seeds, head, Static(E, 16), cfg)
    succ, _, _, _, tr = simulate(seeds, head, Static(E, 16), cfg, inject={t: bits})
    if t >= len(tr.actions):
        raise ValueError("t beyond the episodes' length")
    e_t = np.linalg.norm(tr.actions[t][:, 0:3] - base.actions[t][:, 0:3], axis=1)
    dev = np.linalg.norm(tr.final_obj - base.final_obj, axis=1)
    return e_t, dev, succ


def profile(seeds, bits: int, head, dispatcher_factory, cfg: EnvConfig = EnvConfig(), t_max: Optional[int] = None,
            eps_e: float = 1e-9):
    """profile: every step t of the (successful) baseline
    episodes gets a single-step injection; s_t = D_T / e_t.  Returns a list
    of records (seed, t, phase, e_t, D_T, success, s_t, M_bar, J_bar,
    excluded) with the kinematic window means of the baseline trace
    (dispatcher_factory(E, lam): see kinematic_means).  Records where the
    injection found the episode already finished are skipped."""
    seeds = list(seeds)
    E = len(seeds)
    succ0, _, steps0, _, base = simulate(seeds, head, Static(E, 16), cfg)
    keep = [i for i in range(E) if succ0[i]]
    if not keep:
        return []
    seeds = [seeds[i] for i in keep]
    _, _, _, _, base = simulate(seeds, head, Static(len(seeds), 16), cfg)
    T = int(max(steps0[keep])) if t_max is None else min(t_max, int(max(steps0[keep])))
    acts = np.stack(base.actions)                   # [T, E', 7]
    phases = np.stack(base.phases)
    Mb, Jb = kinematic_means(acts, dispatcher_factory)
    recs = []
    for t in range(T):
        e_t, dev, succ = perturb_at(seeds, t, bits, head, cfg, base=base)
        for j, sd in enumerate(seeds):
            if t >= steps0[keep[j]]:
                continue
            ex = bool(e_t[j] <= eps_e)
            recs.append(dict(seed=int(sd), t=t, phase=PHASES[int(phases[t, j])], e_t=float(e_t[j]),
                             D_T=float(dev[j]), success=bool(succ[j]),
                             s_t=None if ex else float(dev[j] / e_t[j]),
                             M_bar=float(Mb[t, j]), J_bar=float(Jb[t, j]), excluded=ex))
    return recs


def kinematic_means(acts: np.ndarray, dispatcher_factory):
    """Window means M_bar_t, J_bar_t of the kinematic proxies along a recorded
    trace [T, E, 7].  They come from the dispatcher itself: its fused
    S_t = lambda M_bar + (1 - lambda) J_bar is M_bar at lambda = 1
    and J_bar at lambda = 0, so the trace is replayed through two dispatchers
    (dispatcher_factory(E, lam) with .step_S(prev) -> S_t)."""
    T, E, _ = acts.shape
    out = []
    for lam in (1.0, 0.0):
        d = dispatcher_factory(E, lam)
        prev = None
        rows = []
        for t in range(T):
            rows.append(np.asarray(d.step_S(prev), np.float64))
            prev = np.asarray(acts[t], np.float32)
        out.append(np.stack(rows))
    return out[0], out[1]


def proxy_correlation(records, eps_log: float = 1e-9):
    """proxy_correlation: pooled Pearson r of M_bar and J_bar
    against log(s_t + eps) over the included records (>= 30)."""
    inc = [r for r in records if not r["excluded"]]
    if len(inc) < 30:
        raise ValueError(f"proxy_correlation needs >= 30 included records, got {len(inc)}")
    ls = np.log(np.array([r["s_t"] for r in inc]) + eps_log)
    m = np.array([r["M_bar"] for r in inc])
    j = np.array([r["J_bar"] for r in inc])
    return pearson(m, ls), pearson(j, ls)


def pearson(x, y) -> float:
    x = np.asarray(x, np.float64) - np.mean(x)
    y = np.asarray(y, np.float64) - np.mean(y)
    den = math.sqrt(float((x * x).sum()) * float((y * y).sum()))
    return float((x * y).sum() / den) if den > 0 else 0.0


def run_suite(seeds, modes: Dict[str, Callable[[int], object]], head, cfg: EnvConfig = EnvConfig(),
              cost_model=None):
    """run_suite: per mode success rate, mean total cost,
    speedup vs static(16) and the mean bits histogram.  `modes` maps a name
    to a factory E -> dispatcher."""
    E = len(seeds)
    out = {}
    for name, make in modes.items():
        succ, dev, steps, cost, tr = simulate(seeds, head, make(E), cfg, cost_model=cost_model)
        b = np.concatenate([bb[lv] for bb, lv in zip(tr.bits, tr.live)]) if tr.bits else np.zeros(0)
        out[name] = {"success_rate": float(succ.mean()) * 100.0, "mean_cost": float(cost.mean()),
                     "mean_D_T": float(dev.mean()), "mean_steps": float(steps.mean()),
                     "bits_hist": {int(k): int((b == k).sum()) for k in (2, 4, 8, 16)}}
    if "static16" in out:
        for v in out.values():
            v["speedup"] = out["static16"]["mean_cost"] / v["mean_cost"]
    return out


def collect_calibration(seeds, head, dispatcher_factory, cfg: EnvConfig = EnvConfig()):
    """collect_calibration: static(16) episodes; at every step the
    policy is also evaluated at 2, 4, 8 bits counterfactually (the env steps
    with the BF16 action) and S_t comes from the dispatcher fed a*_{t-1}.
    Returns rows (S_t, e2, e4, e8) of the successful episodes."""
    E = len(seeds)
    s = reset(seeds, cfg)
    disp = dispatcher_factory(E)
    prev = None
    rows: List[list] = [[] for _ in range(E)]
    for t in range(cfg.max_steps):
        done, _, _ = episode_status(s, cfg)
        if done.all():
            break
        S = disp.step_S(prev)
        f = features(s, cfg)
        a16 = head(f, np.full(E, 16))
        errs = [np.linalg.norm(head(f, np.full(E, b)) - a16, axis=1) for b in (2, 4, 8)]
        for e in range(E):
            if not done[e]:
                rows[e].append((float(S[e]), float(errs[0][e]), float(errs[1][e]), float(errs[2][e])))
        s = env_step(s, np.where(~done[:, None], a16, 0.0), cfg)
        prev = a16.astype(np.float32)
    _, success, _ = episode_status(s, cfg)
    return [r for e in range(E) if success[e] for r in rows[e]]


def replay_dispatch(actions: np.ndarray, dispatcher) -> np.ndarray:
    """replay_dispatch: a recorded action log [T, E, 7] through
    the dispatcher alone (no environment); returns the bits schedule [T, E]."""
    out = []
    prev = None
    for t in range(actions.shape[0]):
        out.append(np.asarray(dispatcher.step(prev), np.int64))
        prev = np.asarray(actions[t], np.float32)
    return np.stack(out) if out else np.zeros((0, 0), np.int64)
