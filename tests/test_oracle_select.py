"""Pins for the oracle's kinematic bit selection (O7) and Eq. (4) reference (O8).

Golden traces from SPEC (hand-executed Alg. 1 / Eq. (4)), Eq. (6) closure,
properties of S:247-252 over 1e5 random targets, closed-form kinematics cases
(S:136-147), percentile vs numpy sort, scale consistency
 and the Table IV state budget.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_dispatcher.json")))


@pytest.mark.parametrize("case", GOLD["alg1"], ids=lambda c: c["cite"])
def test_alg1_golden(case):
    out, cnt = oracle.alg1(case["targets"], case["K"], tuple(case["init"]))
    assert out.tolist() == case["active"]
    if "counter" in case:
        assert cnt.tolist() == case["counter"]


@pytest.mark.parametrize("case", GOLD["eq4"], ids=lambda c: c["cite"])
def test_eq4_golden(case):
    assert oracle.eq4(case["targets"], case["K"], case["init"]).tolist() == case["active"]


@pytest.mark.parametrize("case", GOLD["phi"], ids=lambda c: c["cite"])
def test_phi_golden(case):
    assert oracle.phi(case["S"], *case["theta"]) == case["bits"]


@pytest.mark.parametrize("case", GOLD["target_bits"], ids=lambda c: c["cite"])
def test_target_bits_golden(case):
    assert oracle.target_bits(case["S"], case["warmup"], *case["theta"]) == case["bits"]


@pytest.mark.parametrize("K", [1, 2, 3, 5])
def test_dispatcher_properties(K):
    """S:247-252 over 1e5 random targets."""
    rng = np.random.default_rng(K)
    # bursty sequences so that downgrades actually happen
    T = 100_000
    levels = np.array([2, 4, 8, 16], np.int32)
    runs = rng.integers(1, 8, size=T)
    seq = np.repeat(levels[rng.integers(0, 4, size=T)], runs)[:T].astype(np.int32)
    out, cnt = oracle.alg1(seq, K)
    ref = oracle.eq4(seq, K)
    assert np.all(out >= seq), "safety dominance"
    assert np.all(ref >= seq)
    prev = np.concatenate([[16], out[:-1]])
    up = seq > prev
    assert np.all(out[up] == seq[up]), "immediate upgrade"
    assert np.all((cnt >= 0) & (cnt < K)), "counter bound"
    # downgrade delay: a strict decrease never happens < K steps after the last
    # step whose target was >= the then-active width
    last_reset = -10**9
    for t in range(T):
        if seq[t] >= prev[t]:
            last_reset = t
        if out[t] < prev[t]:
            assert t - last_reset >= K
    # stateful is never less conservative than Eq. (4) at co-occurring commits
    pref = np.concatenate([[16], ref[:-1]])
    co = (out < prev) & (ref < pref)
    assert np.all(out[co] >= ref[co])
    if K == 1:
        assert np.array_equal(out, ref)


def _replay(actions, **kw):
    return oracle.replay(actions[:, None, :].astype(np.float32), oracle.default_calib(**kw))


def test_replay_all_zero_log():
    """all-zero actions -> post-warm-up Mbar = 1, S = lambda = 0.5 <= theta_fp."""
    g = GOLD["replay_all_zero"]
    r = _replay(np.zeros((30, 7)))
    W, K = 10, 3
    # decision t consumes a_0..a_{t-1}: warm-up while fewer than W_macro observations
    assert np.all(r["target"][:W, 0] == 16)
    assert r["S"][W, 0] == g["S"] and r["Mbar"][W, 0] == g["Mbar"]
    assert r["target"][W, 0] == g["bits_after_warmup"]
    assert np.all(r["bits"][W:W + K - 1, 0] == 16)  # Alg. 1 downgrade delay
    assert np.all(r["bits"][W + K - 1:, 0] == g["bits_after_warmup"])


def test_first_observation_zero_action():
    """first-ever observation of a zero action -> M = 1, J = 0, warm-up."""
    r = _replay(np.zeros((2, 7)))
    assert r["Mbar"][1, 0] == 1.0 and r["Jbar"][1, 0] == 0.0 and r["target"][1, 0] == 16


def test_kinematic_closed_forms():
    """Constant translation c>0, constant rotation: mu -> c, so M = 0 exactly
    (S:137 boundary) and J = 0; S = 0 -> 2 bits after warm-up + K."""
    a = np.zeros((40, 7))
    a[:, 0] = 0.3
    a[:, 3:6] = 0.25
    r = _replay(a)
    assert np.all(r["Mbar"][2:, 0] == 0.0) and np.all(r["Jbar"][2:, 0] == 0.0)
    assert np.all(r["bits"][14:, 0] == 2)


def test_jerk_normalizer_and_cap():
    """||drot|| = nu -> J = 1; 10 nu -> J_cap = 2.  Rotation alternates
    with constant amplitude (all jerks equal -> nu = that jerk -> J = 1), then a
    10x jump hits the cap."""
    T = 30
    a = np.zeros((T + 1, 7))
    a[:, 0] = 1.0  # mu = 1, M = 0
    amp = 0.01
    a[:, 3] = amp * (np.arange(T + 1) % 2)
    r = _replay(a, W_micro=1, lambda_=0.0)
    # step t consumes a_{t-1}; from the 2nd observation on, J = 1 exactly
    assert np.all(r["Jbar"][3:T, 0] == 1.0)
    b = a.copy()
    b[T, 3] = b[T - 1, 3] + 10 * amp
    r2 = _replay(np.vstack([b, np.zeros((1, 7))]), W_micro=1, lambda_=0.0)
    assert r2["Jbar"][T + 1, 0] == 2.0


def test_percentile_matches_numpy_sort():
    rng = np.random.default_rng(5)
    for n in (1, 2, 7, 19, 20, 21, 100, 255, 256):
        v = rng.standard_normal(n)
        k = int(np.ceil(0.95 * n))
        assert oracle.percentile(v, 95) == np.sort(v)[k - 1]
        v2 = np.round(v)  # ties
        assert oracle.percentile(v2, 95) == np.sort(v2)[k - 1]


def test_scale_consistency():
    """scaling all translations by c in {0.5, 2} (exact powers of two)
    leaves every M (hence S and the bits) unchanged."""
    acts = synth.trajectory(300, seed=2001)[0].astype(np.float64)
    base = _replay(acts)
    for c in (0.5, 2.0):
        a2 = acts.copy()
        a2[:, 0:3] *= c
        r = _replay(a2)
        assert np.array_equal(r["Mbar"], base["Mbar"])
        assert np.array_equal(r["bits"], base["bits"])


def test_window_means_match_recompute():
    """windowed means equal a from-scratch recompute.  With W = 1 the
    oracle exposes the raw per-step M_t and J_t; the W = (10, 5) means must be
    the plain averages of the last 10 / 5 of them (partial windows average what
    exists)."""
    acts = synth.trajectory(120, seed=2003)[0].astype(np.float64)
    raw = _replay(acts, W_macro=1, W_micro=1)
    win = _replay(acts)
    Mr, Jr = raw["Mbar"][1:, 0], raw["Jbar"][1:, 0]  # step t holds metrics of a_{t-1}
    for t in range(1, len(acts)):
        i = t - 1
        mm = Mr[max(0, i - 9):i + 1]
        jj = Jr[max(0, i - 4):i + 1]
        assert win["Mbar"][t, 0] == pytest.approx(mm.mean(), abs=1e-15)
        assert win["Jbar"][t, 0] == pytest.approx(jj.mean(), abs=1e-15)


def test_fallback_latch():
    """S > theta_fp -> active = 16 in the same step."""
    acts = synth.trajectories(16, 200)
    r = oracle.replay(acts)
    hi = r["S"] > 0.5
    assert hi.any()
    assert np.all(r["bits"][hi] == 16)


def test_table_iv_state_budget():
    """history buffers < 64 KB (per control stream)."""
    assert oracle.state_bytes_per_stream() < 64 * 1024


def test_bits_mix_with_history():
    """The realised mix on the synthetic LIBERO-shaped recipe uses every width
    (an output, reported; SURVEY §8(d) quotes the prototype's mix)."""
    acts = synth.trajectories(64, 170)
    r = oracle.replay(acts)
    bits = r["bits"][120:]
    vals = set(np.unique(bits).tolist())
    assert vals == {2, 4, 8, 16}


def test_reset_episode_hand_trace():
    """DESIGN.md reading 23: an episode reset clears the windows,
    the previous rotation, the warm-up count and Alg. 1 (-> (16, 0, 16)) but
    KEEPS the p95 history rings; the first step after it does not observe its
    a_{t-1} (the previous episode's last action).  Hand trace with exact
    binary fractions: 20 steps of ||xyz|| = 1 (mu = 1) and rotation jumps of
    0.25 (nu = 0.25), reset, then ||xyz|| = 0.5:
      step 0 after the reset: nothing observed -> empty windows, S = 0, 16;
      first observation: M = 1 - 0.5 / 1 = 0.5 (a wiped ring would give
      mu = 0.5, M = 0), jerk = 0 (prev_rot cleared), Mbar = 0.5 (windows
      cleared), S = 0.25, warm-up -> 16;
      second: rot jumps 0.25 -> J = 0.25 / 0.25 = 1, Jbar = (0 + 1) / 2,
      S = 0.5 * 0.5 + 0.5 * 0.5 = 0.5."""
    st = oracle.SelectState(1)
    a = np.zeros((1, 7), np.float32)
    a[0, 0] = 1.0
    st.step(None)
    for i in range(20):
        a[0, 3] = 0.25 * (i % 2)
        r = st.step(a)
    assert r["bits"][0] in (2, 4, 8, 16) and r["target"][0] != 16  # out of warm-up before the reset
    st.reset_episode()
    r0 = st.step(a)  # a is the previous episode's last action: not observed
    assert r0["Mbar"][0] == 0.0 and r0["Jbar"][0] == 0.0 and r0["S"][0] == 0.0
    assert r0["target"][0] == 16 and r0["bits"][0] == 16
    b = np.zeros((1, 7), np.float32)
    b[0, 0] = 0.5
    b[0, 3] = 0.125
    r1 = st.step(b)
    assert r1["Mbar"][0] == 0.5 and r1["Jbar"][0] == 0.0 and r1["S"][0] == 0.25
    assert r1["target"][0] == 16 and r1["bits"][0] == 16
    b[0, 3] = 0.375
    r2 = st.step(b)
    assert r2["Mbar"][0] == 0.5 and r2["Jbar"][0] == 0.5 and r2["S"][0] == 0.5
    assert r2["bits"][0] == 16
    # warm-up restarts: W_macro = 10 observations after the reset; then, with
    # the rotation held (J = 0, Jbar = 0 once obs 2 leaves the 5-window),
    # S = 0.25 -> 4 bits (Theta = (0.1, 0.3)), entered by Alg. 1 from
    # (16, 0, 16) after K = 3 consecutive targets
    outs = [st.step(b) for _ in range(12)]  # observations 3 .. 14
    tg = [int(o["target"][0]) for o in outs]
    bits = [int(o["bits"][0]) for o in outs]
    assert [float(o["S"][0]) for o in outs[4:]] == [0.25] * 8
    assert tg[:7] == [16] * 7 and tg[7:] == [4] * 5  # obs 10 = first after warm-up
    assert bits[:9] == [16] * 9 and bits[9:] == [4] * 3


def test_reset_episode_mask_leaves_other_streams():
    acts = synth.trajectories(3, 60)
    st = oracle.SelectState(3)
    ref = oracle.replay(acts)
    for t in range(60):
        if t == 30:
            st.reset_episode(np.array([0, 1, 0], np.uint8))
        r = st.step(None if t == 0 else acts[t - 1])
        assert r["bits"][0] == ref["bits"][t, 0] and r["bits"][2] == ref["bits"][t, 2]
        assert r["S"][0] == ref["S"][t, 0] and r["S"][2] == ref["S"][t, 2]
        if t == 30:  # stream 1 starts over: nothing observed, warm-up
            assert r["bits"][1] == 16 and r["target"][1] == 16 and r["S"][1] == 0.0
