"""GPU parity of the calibration collection path (§IV-B P:280-285,
SPEC S:504-507): the forced-bits policy step, the batched counterfactual
step (dyq_calib_collect) and the action-error kernel, against oracle/glue.py,
the C oracle's selector and oracle/calib.py."""
import numpy as np
import pytest

import oracle
from oracle import calib as oc
from oracle import glue

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2603_07904_b200 import dyq  # noqa: E402
from test_gpu_model import _gpu_model, _tiny, t16  # noqa: E402

DEV = "cuda:0"


def _teacher_forced_ok(ref, vis, text, b, a):
    """Every GPU token of action a (bits b) is the reference argmax, or a
    near-boundary disagreement within 5e-3 max|logit| of it (the callers allow
    at most 2 % of those); returns the number of exact decisions."""
    gtok = np.rint((a + 1.0) * 128.0 - 0.5).astype(int)  # detok^-1 (256 bins)
    assert np.array_equal(glue.detok(gtok, 256), a)
    _, logits = ref.episode(vis, text, int(b), forced=gtok)
    top = logits.max(axis=1)
    tol = 5e-3 * np.abs(logits).max()
    assert np.all(logits[np.arange(7), gtok] >= top - tol), (b, gtok, logits.argmax(1))
    return int((logits.argmax(axis=1) == gtok).sum())


@pytest.mark.parametrize("Ec,n_act", [(1, 7), (5, 7), (200, 7), (3, 11)])
def test_calib_errors_kernel(Ec, n_act):
    rng = np.random.default_rng(Ec)
    a = rng.uniform(-1, 1, (4 * Ec, n_act)).astype(np.float32)
    a[Ec:2 * Ec] = a[:Ec]  # e^(2) = 0 exactly
    err = torch.empty(Ec, 3, dtype=torch.float64, device=DEV)
    dyq.calib_errors(torch.from_numpy(a).to(DEV), Ec, n_act, err)
    torch.cuda.synchronize()
    ref = np.stack([oc.action_error(a[(j + 1) * Ec:(j + 2) * Ec], a[:Ec]) for j in range(3)], axis=1)
    np.testing.assert_allclose(err.cpu().numpy(), ref, rtol=1e-15, atol=0)
    assert np.all(err.cpu().numpy()[:, 0] == 0)


def test_policy_step_bits_matches_reference():
    E, n_vis, n_text = 4, 8, 4
    w = _tiny(2)
    model = _gpu_model(w, E, n_vis, n_text)
    ref = glue.TinyModel(w, 64, 4, 2, n_vis, n_text, 7)
    rng = np.random.default_rng(21)
    act = torch.zeros(E, 7, dtype=torch.float32, device=DEV)
    exact = total = 0
    for step, bits in enumerate([[16, 2, 4, 8], [8, 8, 2, 16], [2, 2, 2, 2]]):
        vis = glue.to_bf16_bits(rng.standard_normal((E, n_vis, 256)))
        text = rng.integers(0, 256, (E, n_text)).astype(np.int32)
        bt = torch.tensor(bits, dtype=torch.int32, device=DEV)
        model.step_bits(E, bt, t16(vis.reshape(E, -1)), torch.from_numpy(text).to(DEV), act)
        a = act.cpu().numpy()
        for e in range(E):
            exact += _teacher_forced_ok(ref, vis[e], text[e], bits[e], a[e])
            total += 7
    assert total - exact <= max(1, total // 50), (exact, total)
    with pytest.raises(dyq.DyqError):
        model.step_bits(E, None, t16(vis.reshape(E, -1)), torch.from_numpy(text).to(DEV), act)


def test_calib_collect_end_to_end():
    """T calibration steps for Ec streams: S_t bit-exact with the oracle
    selector fed the GPU's own a*_{t-1}; each replica's action is the
    reference policy at its bits (teacher-forced); e^(b) = ||a^(b) - a*||;
    the thresholds derived from the collected samples by libdyq equal the
    oracle's."""
    Ec, n_vis, n_text, T = 2, 8, 4, 12
    w = _tiny(3)
    model = _gpu_model(w, 4 * Ec, n_vis, n_text)
    ref = glue.TinyModel(w, 64, 4, 2, n_vis, n_text, 7)
    cal = dyq.default_calib()
    state = torch.zeros(dyq.state_size(Ec, cal), dtype=torch.uint8, device=DEV)
    dyq.state_init(Ec, cal, state)
    sel = oracle.SelectState(Ec)
    rng = np.random.default_rng(31)
    acts = torch.zeros(4 * Ec, 7, dtype=torch.float32, device=DEV)
    S = torch.zeros(Ec, dtype=torch.float64, device=DEV)
    err = torch.zeros(Ec, 3, dtype=torch.float64, device=DEV)
    prev = None
    S_log, e_log = [], []
    exact = total = 0
    for step in range(T):
        vis = glue.to_bf16_bits(rng.standard_normal((Ec, n_vis, 256)))
        text = rng.integers(0, 256, (Ec, n_text)).astype(np.int32)
        model.calib_collect(state, Ec, t16(vis.reshape(Ec, -1)), torch.from_numpy(text).to(DEV), acts, S, err)
        a = acts.cpu().numpy()
        s_ref = sel.step(prev)["S"]
        assert np.array_equal(S.cpu().numpy(), s_ref), (step, S.cpu().numpy(), s_ref)
        for j, b in enumerate([16, 2, 4, 8]):
            for e in range(Ec):
                if step % 4 == 0 or j == 0:  # reference steps are slow: sample them
                    exact += _teacher_forced_ok(ref, vis[e], text[e], b, a[j * Ec + e])
                    total += 7
        e_ref = np.stack([oc.action_error(a[(j + 1) * Ec:(j + 2) * Ec], a[:Ec]) for j in range(3)], axis=1)
        np.testing.assert_allclose(err.cpu().numpy(), e_ref, rtol=1e-15, atol=0)
        prev = a[:Ec].copy()
        S_log.append(S.cpu().numpy().copy())
        e_log.append(err.cpu().numpy().copy())
    assert total - exact <= max(1, total // 50), (exact, total)
    Sa, ea = np.concatenate(S_log), np.concatenate(e_log)
    assert np.all(ea >= 0)
    tfp = float(max(Sa.max(), 1e-3))
    ref_d = oc.derive_thresholds(Sa, ea, tfp, 0.5, 0.01, n_bins=4, n_min=1)
    c = dyq.default_calib(theta_fp=tfp, D_acc=0.5, eta=0.01)
    dyq.calib_derive(Sa, ea, c, n_bins=4, n_min=1)
    assert (c.theta_24, c.theta_48) == (ref_d.theta_24, ref_d.theta_48)
    with pytest.raises(dyq.DyqError):  # 4 Ec > E
        model.calib_collect(state, 2 * Ec, t16(vis.reshape(Ec, -1)), torch.from_numpy(text).to(DEV), acts, S, err)
