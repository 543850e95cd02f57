"""libdyq's offline threshold calibration (dyq_calib_derive / dyq_calib_validate,
host code, §IV-B) against oracle/calib.py.

Host-only entry points of the C ABI, so these run without a GPU: thresholds
bit-exact, smoothed bin means and counts bit-exact (same fp64 evaluation
order, reading C5), audits equal.
"""
import json
import os

import numpy as np
import pytest

from oracle import calib as oc
from paper_2603_07904_b200 import dyq

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_calibration.json")))


def table(tfp, D, eta):
    return dyq.default_calib(theta_24=0.0, theta_48=0.0, theta_fp=tfp, D_acc=D, eta=eta)


def uniform_S(tfp, per_bin=64, n_bins=32):
    w = tfp / n_bins
    return np.array([(i + (k + 0.5) / per_bin) * w for i in range(n_bins) for k in range(per_bin)])


def check_same(S, err, tfp, D, eta, n_bins=32, n_min=50):
    ref = oc.derive_thresholds(S, err, tfp, D, eta, n_bins, n_min)
    c = table(tfp, D, eta)
    sm, cnt, und = dyq.calib_derive(S, err, c, n_bins, n_min)
    assert (c.theta_24, c.theta_48) == (ref.theta_24, ref.theta_48)
    np.testing.assert_array_equal(cnt, ref.counts)
    np.testing.assert_array_equal(sm, ref.smoothed)
    assert und == len(ref.undercovered)
    assert c.lambda_ == 0.5 and c.K == 3  # untouched fields pass through
    nq, nok, worst = dyq.calib_validate(c, S, err, n_bins)
    a = oc.validate_table(S, err, c.theta_24, c.theta_48, tfp, D, eta, n_bins)
    assert (nq, nok) == (a.n_quant, a.n_ok)
    np.testing.assert_array_equal(worst, a.worst)
    return c


@pytest.mark.parametrize("case", GOLD["derive"], ids=lambda c: c["cite"])
def test_derive_golden(case):
    S = uniform_S(case["theta_fp"])
    err = np.tile(np.array(case["e"]), (S.size, 1))
    c = check_same(S, err, case["theta_fp"], case["D_acc"], case["eta"])
    assert (c.theta_24, c.theta_48) == (case["theta_24"], case["theta_48"])


def test_random_matches_oracle():
    rng = np.random.default_rng(5)
    for trial in range(30):
        tfp = float(rng.choice([0.25, 0.5, 1.0]))
        n = int(rng.integers(4000, 8000))
        S = np.concatenate([rng.uniform(0, tfp, n), rng.uniform(tfp, 2 * tfp, n // 8), [0.0, tfp]])
        base = S[:, None] * np.array([4.0, 1.0, 0.2]) + np.array([0.05, 0.01, 0.001])
        err = np.abs(base * rng.lognormal(0.0, 0.6, size=(S.size, 3)))
        D, eta = float(rng.uniform(0.05, 0.5)), float(rng.uniform(0.005, 0.05))
        n_bins = int(rng.choice([8, 32, 64]))
        check_same(S, err, tfp, D, eta, n_bins, int(rng.choice([1, 20, 50])))


def test_sparse_coverage_matches_oracle():
    """Clustered S leaves bins under-covered: the interpolation path."""
    rng = np.random.default_rng(9)
    for trial in range(10):
        centres = rng.uniform(0, 0.5, 4)
        S = np.clip(np.concatenate([rng.normal(c, 0.01, 200) for c in centres]), 0, 0.5)
        err = np.abs(rng.normal(0.2, 0.1, (S.size, 3))) + S[:, None]
        check_same(S, err, 0.5, 0.2, 0.01)


def test_errors():
    c = table(0.5, 1.0, 0.01)
    with pytest.raises(dyq.DyqError):
        dyq.calib_derive(np.zeros(0), np.zeros((0, 3)), c)
    with pytest.raises(dyq.DyqError):
        dyq.calib_derive(np.full(49, 0.1), np.zeros((49, 3)), c)  # no bin reaches n_min
    with pytest.raises(dyq.DyqError):
        dyq.calib_derive(np.full(60, 0.1), np.zeros((60, 3)), table(0.5, 0.0, 0.01))
    bad = dyq.default_calib(theta_24=0.3, theta_48=0.1)
    with pytest.raises(dyq.DyqError):
        dyq.calib_validate(bad, np.zeros(1), np.zeros((1, 3)))
    nq, nok, worst = dyq.calib_validate(dyq.default_calib(), np.zeros(0), np.zeros((0, 3)))
    assert (nq, nok) == (0, 0) and not worst.any()
