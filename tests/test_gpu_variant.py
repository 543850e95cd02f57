"""The variant table and the paper-mode selector (dyq_model_desc_t optional
fields, dyq_qlinear_masked).

- dyq_qlinear_masked: two calls on the W4 and W8 copies of one weight share
  one output, each owning the rows its row_bits mark (others untouched), and a
  closed device gate makes a call a no-op; checked against the oracle qlinear
  of each copy row by row.
- Policy step with a W8 copy: b* = 16 (the warm-up) runs on the W8 copy
  (W8A16), quantized b* on the W4 copy, so the trajectory switches weight
  copies mid-run on the device; b*_t bit-exact with the oracle selector and
  every step teacher-forced against glue.TinyModel on the copy the table picks.
- Paper mode: the selector runs on a side stream overlapping the
  prefill, the prefill at a fixed width (BF16) and the decode passes at b*_t.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle import glue

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2603_07904_b200 import dyq  # noqa: E402
from test_gpu_parity import check_close  # noqa: E402
from test_gpu_model import DEV, _tiny, t16  # noqa: E402


@pytest.mark.parametrize("M", [3, 16, 40, 288])
def test_qlinear_masked_composes_w4_and_w8(M):
    N, K, G = 512, 512, 64
    w = synth.weights_bf16(N, K, seed=31)
    x = synth.activations_bf16(M, K, seed=32)
    wt, xt = t16(w), t16(x)
    l4 = dyq.PackedLinear.from_bf16(wt, group=G, wbits=4)
    l8 = dyq.PackedLinear.from_bf16(wt, group=G, wbits=8)
    ab = np.array([[2, 4, 8, 16][m % 4] for m in range(M)], np.int32)
    on8 = np.array([m % 3 == 1 for m in range(M)])
    rb4 = torch.from_numpy(np.where(on8, 0, ab).astype(np.int32)).to(DEV)
    rb8 = torch.from_numpy(np.where(on8, ab, 0).astype(np.int32)).to(DEV)
    gates = torch.ones(2, dtype=torch.int32, device=DEV)
    y = torch.full((M, N), float("nan"), dtype=torch.float32, device=DEV)
    ws4, ws8 = l4.workspace(M), l8.workspace(M)
    dyq.qlinear_masked(l4.wd, l4.codes, l4.meta, xt, M, rb4, gates[0:1], y, 0, ws4)
    dyq.qlinear_masked(l8.wd, l8.codes, l8.meta, xt, M, rb8, gates[1:2], y, 0, ws8)
    got = y.cpu().numpy()
    y4, _ = oracle.qlinear(x, oracle.pack_weights(w, G, 4), G, ab)
    y8, _ = oracle.qlinear(x, oracle.pack_weights(w, G, 8), G, ab)
    ref = np.where(on8[:, None], y8, y4)
    check_close(got, ref, 1e-3)
    # a closed gate: the call reads nothing and writes nothing
    gates.zero_()
    y2 = torch.full((M, N), 7.0, dtype=torch.float32, device=DEV)
    dyq.qlinear_masked(l8.wd, l8.codes, l8.meta, xt, M, torch.from_numpy(ab).to(DEV), gates[1:2], y2, 0, ws8)
    torch.cuda.synchronize()
    assert bool((y2 == 7.0).all())


def _models(w, E, n_vis, n_text, **kw):
    layers4 = [[dyq.PackedLinear.from_bf16(t16(lin), group=64, wbits=4) for lin in layer] for layer in w["lin"]]
    layers8 = [[dyq.PackedLinear.from_bf16(t16(lin), group=64, wbits=8) for lin in layer] for layer in w["lin"]]
    return dyq.Model(layers4, t16(w["attn_norm"]), t16(w["mlp_norm"]), t16(w["final_norm"]), t16(w["embed"]),
                     t16(w["head"]), E=E, n_heads=2, n_vis=n_vis, n_text=n_text, n_act=7, layers_w8=layers8, **kw)


def _run(model, ref, E, n_vis, n_text, steps, cal_kw, wbits_for, prefill_for=None, seed=11):
    cal = dyq.default_calib(**cal_kw)
    state = torch.zeros(dyq.state_size(E, cal), dtype=torch.uint8, device=DEV)
    dyq.state_init(E, cal, state)
    sel = oracle.SelectState(E, oracle.default_calib(**cal_kw))
    rng = np.random.default_rng(seed)
    act = torch.zeros(E, 7, dtype=torch.float32, device=DEV)
    bits = torch.zeros(E, dtype=torch.int32, device=DEV)
    prev = None
    seen = set()
    exact = total = 0
    for step in range(steps):
        vis = glue.to_bf16_bits(rng.standard_normal((E, n_vis, 256)))
        text = rng.integers(0, 256, (E, n_text)).astype(np.int32)
        model.step(state, E, t16(vis.reshape(E, -1)), torch.from_numpy(text).to(DEV), act, bits)
        a, b = act.cpu().numpy(), bits.cpu().numpy()
        rb = sel.step(prev)["bits"]
        assert np.array_equal(b, rb), (step, b, rb)  # b*_t bit-exact
        prev = a.astype(np.float32)
        for e in range(E):
            gtok = np.rint((a[e] + 1.0) * 128.0 - 0.5).astype(int)
            assert np.array_equal(glue.detok(gtok, 256), a[e])
            wb = wbits_for(int(b[e]))
            seen.add(wb)
            _, logits = ref.episode(vis[e], text[e], int(b[e]), forced=gtok, wbits=wb,
                                    prefill=None if prefill_for is None else prefill_for(int(b[e])))
            top = logits.max(axis=1)  # reference argmax, or a near-boundary flip (<= 2 %)
            tol = 5e-3 * np.abs(logits).max()
            assert np.all(logits[np.arange(7), gtok] >= top - tol), (step, e, gtok, logits.argmax(1))
            exact += int((logits.argmax(axis=1) == gtok).sum())
            total += 7
    assert total - exact <= max(1, total // 50), (exact, total)
    return seen


def test_policy_step_switches_w4_w8_mid_trajectory():
    """wbits_of = (4, 4, 4, 8): the warm-up's b* = 16 runs W8A16; with
    theta_fp out of reach the dispatcher then settles on quantized widths,
    which run on the W4 copy -- a device-side weight-copy switch mid-run."""
    E, n_vis, n_text = 2, 8, 4
    w = _tiny(3)
    model = _models(w, E, n_vis, n_text, wbits_of=(4, 4, 4, 8))
    ref = glue.TinyModel(w, 64, 4, 2, n_vis, n_text, 7)
    seen = _run(model, ref, E, n_vis, n_text, 18, dict(theta_fp=1e9), lambda b: 8 if b == 16 else 4)
    assert seen == {4, 8}, seen


def test_policy_step_paper_mode():
    """Selector on a side stream overlapping the prefill; prefill at BF16 on
    the W4 copy, decode passes at b*_t."""
    E, n_vis, n_text = 2, 8, 4
    w = _tiny(4)
    layers4 = [[dyq.PackedLinear.from_bf16(t16(lin), group=64, wbits=4) for lin in layer] for layer in w["lin"]]
    model = dyq.Model(layers4, t16(w["attn_norm"]), t16(w["mlp_norm"]), t16(w["final_norm"]), t16(w["embed"]),
                      t16(w["head"]), E=E, n_heads=2, n_vis=n_vis, n_text=n_text, n_act=7, paper_mode=1,
                      prefill_bits=16)
    ref = glue.TinyModel(w, 64, 4, 2, n_vis, n_text, 7)
    _run(model, ref, E, n_vis, n_text, 16, dict(theta_fp=1e9), lambda b: 4, prefill_for=lambda b: (16, 4))


def test_paper_mode_under_graph_capture():
    """The fork / join of the side stream is capturable: a graph of two paper-
    mode steps reproduces the eager bits and actions."""
    E, n_vis, n_text = 1, 8, 4
    w = _tiny(5)
    layers4 = [[dyq.PackedLinear.from_bf16(t16(lin), group=64, wbits=4) for lin in layer] for layer in w["lin"]]

    def build():
        return dyq.Model(layers4, t16(w["attn_norm"]), t16(w["mlp_norm"]), t16(w["final_norm"]), t16(w["embed"]),
                         t16(w["head"]), E=E, n_heads=2, n_vis=n_vis, n_text=n_text, n_act=7, paper_mode=1)
    rng = np.random.default_rng(7)
    vis = t16(glue.to_bf16_bits(rng.standard_normal((E, n_vis * 256))))
    text = torch.from_numpy(rng.integers(0, 256, (E, n_text)).astype(np.int32)).to(DEV)
    cal = dyq.default_calib()
    outs = []
    for graphed in (False, True):
        model = build()
        state = torch.zeros(dyq.state_size(E, cal), dtype=torch.uint8, device=DEV)
        dyq.state_init(E, cal, state)
        act = torch.zeros(E, 7, dtype=torch.float32, device=DEV)
        bits = torch.zeros(E, dtype=torch.int32, device=DEV)
        rec = []
        model.step(state, E, vis, text, act, bits)  # t = 0 eagerly (no a_{t-1} yet)
        if graphed:
            s = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.graph(g, stream=s):
                model.step(state, E, vis, text, act, bits, stream=s)
            for _ in range(3):
                g.replay()
                torch.cuda.synchronize()
                rec.append((act.cpu().numpy().copy(), bits.cpu().numpy().copy()))
        else:
            for _ in range(3):
                model.step(state, E, vis, text, act, bits)
                rec.append((act.cpu().numpy().copy(), bits.cpu().numpy().copy()))
        outs.append(rec)
    for (a0, b0), (a1, b1) in zip(*outs):
        assert np.array_equal(b0, b1)
        assert np.array_equal(a0, a1)
