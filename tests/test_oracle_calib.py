"""Pins for the offline threshold calibration oracle (oracle/calib.py).

SPEC worked cases (tests/golden/spec_calibration.json), a
hand-computed exact tie (reading C4), the closed-form crossing
S* = D_acc / e - eta of P:263 + Eq. (5) for constant errors, weighted PAV vs
sklearn's IsotonicRegression and a hand pooling case, the interpolation of
under-covered bins (reading C2), and the ordering / minimality invariants of
S:309-312 on random samples.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import calib as oc

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_calibration.json")))


def uniform_S(theta_fp, per_bin=64, n_bins=oc.N_BINS):
    """per_bin samples strictly inside every bin (no sample on a bin edge)."""
    w = theta_fp / n_bins
    return np.array([(i + (k + 0.5) / per_bin) * w for i in range(n_bins) for k in range(per_bin)])


@pytest.mark.parametrize("case", GOLD["error_bound"], ids=lambda c: c["cite"])
def test_error_bound_golden(case):
    assert oc.error_bound(case["S"], case["D_acc"], case["eta"]) == pytest.approx(case["eps"], rel=1e-15)


def test_error_bound_monotone_and_rejects_bad_params():
    S = np.linspace(0, 10, 1001)
    eps = oc.error_bound(S, 1.0, 0.01)
    assert np.all(np.diff(eps) < 0)
    assert oc.error_bound(10.0, 1.0, 0.01) < oc.error_bound(1.0, 1.0, 0.01)
    with pytest.raises(ValueError):
        oc.error_bound(0.1, 0.0, 0.01)
    with pytest.raises(ValueError):
        oc.error_bound(0.1, 1.0, 0.0)


@pytest.mark.parametrize("case", GOLD["derive"], ids=lambda c: c["cite"])
def test_derive_golden(case):
    S = uniform_S(case["theta_fp"])
    err = np.tile(np.array(case["e"]), (S.size, 1))
    d = oc.derive_thresholds(S, err, case["theta_fp"], case["D_acc"], case["eta"])
    assert d.theta_24 == case["theta_24"]
    assert d.theta_48 == case["theta_48"]
    assert d.undercovered == []


def test_closed_form_crossing():
    """Constant e2: the first violating bin is the one containing
    S* = D_acc / e2 - eta (P:263 solved for S), its lower edge floor(S*/w) w."""
    rng = np.random.default_rng(7)
    tfp = 0.5
    w = tfp / oc.N_BINS
    S = uniform_S(tfp)
    hits = 0
    for _ in range(200):
        eta = float(rng.uniform(0.001, 0.05))
        D = float(rng.uniform(0.01, 0.5))
        Sstar = float(rng.uniform(0.0, 0.55))
        e2 = D / (Sstar + eta)
        err = np.tile([e2, 0.0, 0.0], (S.size, 1))
        d = oc.derive_thresholds(S, err, tfp, D, eta)
        if abs(Sstar / w - round(Sstar / w)) < 1e-9:
            continue  # crossing on a bin edge: rounding decides, skip
        expect = math.floor(Sstar / w) * w if Sstar < tfp else tfp
        assert d.theta_24 == pytest.approx(expect, abs=1e-15), (D, eta, Sstar)
        hits += Sstar < tfp
    assert hits > 150


def test_pav_hand_and_sklearn():
    # two adjacent violators pooled with their counts: (0.3*50 + 0.1*150)/200
    assert oc.isotonic_pav([0.3, 0.1], [50, 150]).tolist() == [0.15, 0.15]
    assert oc.isotonic_pav([0.1, 0.2, 0.3], [1, 1, 1]).tolist() == [0.1, 0.2, 0.3]
    # a chain that pools back over an earlier block: [1, 3, 2, 0] unit weights -> [1, 5/3, 5/3, 5/3]
    np.testing.assert_allclose(oc.isotonic_pav([1, 3, 2, 0], [1, 1, 1, 1]), [1, 5 / 3, 5 / 3, 5 / 3], rtol=1e-15)
    from sklearn.isotonic import IsotonicRegression
    rng = np.random.default_rng(3)
    for _ in range(50):
        n = int(rng.integers(1, 40))
        y = rng.normal(size=n).cumsum() * 0.1 + rng.normal(size=n)
        wts = rng.integers(1, 200, size=n).astype(np.float64)
        ref = IsotonicRegression().fit(np.arange(n), y, sample_weight=wts).predict(np.arange(n))
        np.testing.assert_allclose(oc.isotonic_pav(y, wts), ref, rtol=1e-12, atol=1e-12)


def test_derive_pools_bins_by_count():
    """Bin 0 mean 0.3 (50 samples) above bin 1 mean 0.1 (150 samples): both
    smooth to 0.15; every later bin keeps its own (non-decreasing) mean 0.2."""
    tfp = 0.5
    w = tfp / oc.N_BINS
    S = [0.5 * w] * 50 + [1.5 * w] * 150 + [(i + 0.5) * w for i in range(2, 32) for _ in range(50)]
    e2 = [0.3] * 50 + [0.1] * 150 + [0.2] * (30 * 50)
    err = np.array([[v, 0.0, 0.0] for v in e2])
    d = oc.derive_thresholds(S, err, tfp, 100.0, 0.01)
    assert d.smoothed[0, 0] == pytest.approx(0.15, rel=1e-15)
    assert d.smoothed[0, 1] == pytest.approx(0.15, rel=1e-15)
    assert np.all(d.smoothed[0, 2:] == pytest.approx(0.2, rel=1e-15))
    assert d.counts.tolist() == [50, 150] + [50] * 30


def test_undercovered_bins_interpolated():
    """Reading C2: bin 1 (10 samples) between covered bins 0 (0.1) and 2 (0.3)
    takes 0.2; bins after the last covered bin take its value; a bin with too
    few samples is listed as a coverage warning."""
    tfp = 0.5
    w = tfp / oc.N_BINS
    S = [0.5 * w] * 60 + [1.5 * w] * 10 + [2.5 * w] * 60
    err = np.array([[0.1, 0, 0]] * 60 + [[5.0, 0, 0]] * 10 + [[0.3, 0, 0]] * 60)
    d = oc.derive_thresholds(S, err, tfp, 100.0, 0.01)
    assert d.smoothed[0, 1] == pytest.approx(0.2, rel=1e-15)
    assert np.all(d.smoothed[0, 3:] == d.smoothed[0, 2]) and d.smoothed[0, 2] == pytest.approx(0.3, rel=1e-15)
    assert d.undercovered == [1] + list(range(3, 32))


def test_derive_rejects_empty_and_uncovered():
    with pytest.raises(ValueError):
        oc.derive_thresholds([], np.zeros((0, 3)), 0.5, 1.0, 0.01)
    with pytest.raises(ValueError):
        oc.derive_thresholds([0.1] * 49, np.zeros((49, 3)), 0.5, 1.0, 0.01)


def test_bin_index_edges():
    tfp = 0.5
    assert oc.bin_index(0.0, tfp) == 0
    assert oc.bin_index(tfp, tfp) == oc.N_BINS - 1
    assert oc.bin_index(1 / 64, tfp) == 1  # lower edge belongs to its bin
    assert oc.bin_index(tfp + 1e-9, tfp) == -1
    assert oc.bin_index(-1e-9, tfp) == -1


def random_samples(rng, n, tfp):
    S = np.concatenate([rng.uniform(0, tfp, n), rng.uniform(tfp, 2 * tfp, n // 10)])
    base = S[:, None] * np.array([4.0, 1.0, 0.2]) + np.array([0.05, 0.01, 0.001])
    err = np.abs(base * rng.lognormal(0.0, 0.5, size=(S.size, 3)))
    return S, err


def test_invariants_random():
    """0 <= t24 <= t48 <= tfp; every bin below theta_24 meets the
    bound with e^(2), bins in [theta_24, theta_48) with e^(4); the bin at a
    threshold < theta_fp violates it; samples above theta_fp do not matter;
    determinism."""
    rng = np.random.default_rng(11)
    tfp = 0.5
    w = tfp / oc.N_BINS
    for trial in range(20):
        S, err = random_samples(rng, 4000, tfp)
        D, eta = float(rng.uniform(0.05, 0.5)), float(rng.uniform(0.005, 0.05))
        d = oc.derive_thresholds(S, err, tfp, D, eta)
        assert 0.0 <= d.theta_24 <= d.theta_48 <= tfp
        b24, b48 = round(d.theta_24 / w), round(d.theta_48 / w)
        for i in range(oc.N_BINS):
            eps = D / ((i + 1) * w + eta)
            if i < b24:
                assert d.smoothed[0, i] <= eps
            elif i < b48:
                assert d.smoothed[1, i] <= eps
        raw24 = next((i for i in range(oc.N_BINS) if d.smoothed[0, i] > D / ((i + 1) * w + eta)), oc.N_BINS)
        assert b24 == raw24
        for j in range(2):
            assert np.all(np.diff(d.smoothed[j]) >= -1e-15)
        keep = S <= tfp
        d2 = oc.derive_thresholds(S[keep], err[keep], tfp, D, eta)
        assert (d2.theta_24, d2.theta_48) == (d.theta_24, d.theta_48)
        d3 = oc.derive_thresholds(S, err, tfp, D, eta)
        assert (d3.theta_24, d3.theta_48) == (d.theta_24, d.theta_48)


def test_validate_self_consistent_constant_errors():
    """Constant per-bit errors: the bound checked at each bin's upper edge is
    the tightest in the bin, so every calibration sample is satisfied."""
    tfp = 0.5
    S = np.concatenate([uniform_S(tfp), [0.7, 0.9]])
    err = np.tile([0.5, 0.1, 0.01], (S.size, 1))
    d = oc.derive_thresholds(S, err, tfp, 0.1, 0.01)
    a = oc.validate_table(S, err, d.theta_24, d.theta_48, tfp, 0.1, 0.01)
    assert a.n == S.size and a.n_quant == S.size - 2 and a.n_ok == S.size
    assert a.fraction == 1.0
    assert np.all(a.worst <= 1.0) and np.all(a.worst > 0)


def test_validate_hand_cases():
    # empty held-out set
    a = oc.validate_table([], np.zeros((0, 3)), 0.1, 0.3, 0.5, 1.0, 0.01)
    assert (a.n, a.n_ok, a.fraction) == (0, 0, 1.0)
    # three samples, Theta = (0.1, 0.3): S=0.05 -> b=2 (e=3, eps=1/0.06=16.7 ok);
    # S=0.2 -> b=4 (e=5 > eps=1/0.21=4.76 fail); S=0.4 -> b=8 (e=1, ok); S=0.8 -> BF16 ok
    S = [0.05, 0.2, 0.4, 0.8]
    err = [[3.0, 9.0, 9.0], [9.0, 5.0, 9.0], [9.0, 9.0, 1.0], [9.0, 9.0, 9.0]]
    a = oc.validate_table(S, err, 0.1, 0.3, 0.5, 1.0, 0.01)
    assert (a.n, a.n_quant, a.n_ok) == (4, 3, 3)
    assert a.worst[oc.bin_index(0.2, 0.5)] == pytest.approx(5.0 * 0.21, rel=1e-15)
    # theta_24 = 0: no sample is audited at 2 bits (its huge e2 never counts)
    a0 = oc.validate_table([0.05, 0.2], [[1e9, 0.1, 0.1], [1e9, 0.1, 0.1]], 0.0, 0.3, 0.5, 1.0, 0.01)
    assert a0.n_ok == 2


def test_action_error():
    assert oc.action_error([3.0, 4.0, 0, 0, 0, 0, 0], np.zeros(7)) == 5.0
    assert oc.action_error(np.ones((2, 7)), np.ones((2, 7))).tolist() == [0.0, 0.0]
    assert oc.action_error([1.0] * 7, [0.0] * 7) == pytest.approx(math.sqrt(7), rel=1e-15)
