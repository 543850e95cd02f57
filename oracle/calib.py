"""CPU oracle for DyQ-VLA offline threshold calibration -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU legs may import
this module; the product package never imports it (DESIGN.md §"Oracle").

Restates PAPER.md §IV-B in the binned isotonic reading SPEC.md
gives, plain fp64 numpy / Python loops, no blocking or fusion:

  error_bound      eps_a(S) = D_acc / (S + eta)
  action_error     e^(b) = || a^(b) - a* ||_2
  bin_index        uniform bins on [0, theta_fp]                S:292 (reading C1)
  isotonic_pav     weighted pool-adjacent-violators            S:292, S:314 (reading C3)
  derive_thresholds Theta = {theta_24, theta_48}
  validate_table   audit e^(Phi(S)) <= eps_a(S)                 Eq. (5)

The paper only says "systematically identify critical intersections";
every reading taken here is listed in DESIGN.md (readings C1-C6).
Parity: pinned by tests/test_oracle_calib.py (SPEC S:295-297 worked cases,
hand-computed exact-tie and pooling cases, closed-form crossing, sklearn
IsotonicRegression, minimality / ordering invariants on random samples).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

N_BINS = 32
N_MIN = 50   # S:291 ("at least N_min = 50 samples per occupied bin")


def error_bound(S, D_acc: float, eta: float):
    """eps_a(S) = D_acc / (S + eta), P:263 / S:280-285."""
    if not (D_acc > 0 and eta > 0):
        raise ValueError("D_acc and eta must be > 0")
    return D_acc / (np.asarray(S, dtype=np.float64) + eta)


def action_error(a_hat, a_star):
    """e = || a_hat - a* ||_2 over the action vector, fp64."""
    d = np.asarray(a_hat, np.float64) - np.asarray(a_star, np.float64)
    return np.sqrt(np.sum(d * d, axis=-1))


def bin_width(theta_fp: float, n_bins: int = N_BINS) -> float:
    return theta_fp / n_bins


def bin_index(S: float, theta_fp: float, n_bins: int = N_BINS) -> int:
    """Reading C1: bin i = floor(S / w), w = theta_fp / n_bins, S = theta_fp in
    the last bin; -1 for S outside [0, theta_fp] (those steps run BF16)."""
    if not (0.0 <= S <= theta_fp):
        return -1
    i = int(math.floor(S / bin_width(theta_fp, n_bins)))
    return min(i, n_bins - 1)


def isotonic_pav(y, w):
    """Weighted pool-adjacent-violators: the non-decreasing sequence minimising
    sum w_i (f_i - y_i)^2 (textbook PAV, one left-to-right pass with merging)."""
    blocks = []  # [mean, weight, length]
    for yi, wi in zip(y, w):
        blocks.append([float(yi), float(wi), 1])
        while len(blocks) > 1 and blocks[-2][0] > blocks[-1][0]:
            m2, w2, n2 = blocks.pop()
            m1, w1, n1 = blocks.pop()
            blocks.append([(m1 * w1 + m2 * w2) / (w1 + w2), w1 + w2, n1 + n2])
    out = []
    for m, _, n in blocks:
        out.extend([m] * n)
    return np.array(out, dtype=np.float64)


@dataclass
class Derivation:
    theta_24: float
    theta_48: float
    counts: np.ndarray                      # [n_bins] samples per bin
    smoothed: np.ndarray                    # [2, n_bins] smoothed mean e^(2), e^(4)
    undercovered: list = field(default_factory=list)  # bins with count < n_min (coverage warning)


def _fill_uncovered(vals, covered):
    """Reading C2: an under-covered bin takes the linear interpolation (by bin
    index) between the nearest covered bins on either side; constant beyond
    the first / last covered bin."""
    n = len(vals)
    idx = [i for i in range(n) if covered[i]]
    out = np.array(vals, dtype=np.float64)
    for i in range(n):
        if covered[i]:
            continue
        lo = [j for j in idx if j < i]
        hi = [j for j in idx if j > i]
        if lo and hi:
            a, b = lo[-1], hi[0]
            t = (i - a) / (b - a)
            out[i] = out[a] + t * (out[b] - out[a])
        elif lo:
            out[i] = out[lo[-1]]
        else:
            out[i] = out[hi[0]]
    return out


def derive_thresholds(S, err, theta_fp: float, D_acc: float, eta: float,
                      n_bins: int = N_BINS, n_min: int = N_MIN) -> Derivation:
    """SPEC S:289-297 on samples S[n], err[n, 3] = (e^(2), e^(4), e^(8)).

    1. bin the samples with S in [0, theta_fp] (reading C1);
    2. per bin and b in {2, 4}: the mean error (the expectation of Eq. (5));
    3. bins with >= n_min samples: weighted PAV (weights = counts), in bin
       order (reading C3); the others: interpolated (reading C2);
    4. theta_{2|4} = lower edge of the first bin whose smoothed e^(2) exceeds
       eps_a at the bin's upper edge (strict >, reading C4); none -> theta_fp;
       theta_{4|8} likewise for e^(4), then raised to theta_{2|4} if below.
    """
    S = np.asarray(S, np.float64)
    err = np.asarray(err, np.float64).reshape(-1, 3)
    if S.size == 0:
        raise ValueError("empty calibration set")
    w = bin_width(theta_fp, n_bins)
    counts = np.zeros(n_bins, np.int64)
    sums = np.zeros((2, n_bins), np.float64)
    for t in range(S.size):  # sample order (reading C5: sequential fp64 sums)
        i = bin_index(S[t], theta_fp, n_bins)
        if i < 0:
            continue
        counts[i] += 1
        sums[0, i] += err[t, 0]
        sums[1, i] += err[t, 1]
    covered = counts >= n_min
    if not covered.any():
        raise ValueError("no bin reaches n_min samples")
    smoothed = np.zeros((2, n_bins), np.float64)
    idx = np.nonzero(covered)[0]
    for j in range(2):
        means = sums[j, idx] / counts[idx]
        full = np.zeros(n_bins, np.float64)
        full[idx] = isotonic_pav(means, counts[idx])
        smoothed[j] = _fill_uncovered(full, covered)
    thetas = []
    for j in range(2):
        th = theta_fp
        for i in range(n_bins):
            eps = D_acc / ((i + 1) * w + eta)
            if smoothed[j, i] > eps:
                th = i * w
                break
        thetas.append(th)
    t24, t48 = thetas
    if t48 < t24:
        t48 = t24
    return Derivation(t24, t48, counts, smoothed,
                      [int(i) for i in range(n_bins) if counts[i] < n_min])


def phi(S: float, t24: float, t48: float) -> int:
    """Eq. (6), P:290-294 (boundaries belong to the lower-bit interval; same
    convention as dyq_ref_phi)."""
    if S <= t24:
        return 2
    if S <= t48:
        return 4
    return 8


@dataclass
class Audit:
    n: int            # samples audited (all)
    n_quant: int      # samples with S in [0, theta_fp] (quantized domain)
    n_ok: int         # samples with e^(Phi(S)) <= eps_a(S) (BF16 steps count as ok, e = 0)
    worst: np.ndarray  # [n_bins] max e^(Phi(S)) / eps_a(S) per bin, 0 for empty bins

    @property
    def fraction(self) -> float:
        return self.n_ok / self.n if self.n else 1.0


def validate_table(S, err, t24: float, t48: float, theta_fp: float, D_acc: float, eta: float,
                   n_bins: int = N_BINS) -> Audit:
    """per sample, b = Phi(S) below theta_fp (else BF16, e = 0,
    P:240); satisfied iff e^(b) <= eps_a(S) at the sample's own S."""
    S = np.asarray(S, np.float64)
    err = np.asarray(err, np.float64).reshape(-1, 3)
    worst = np.zeros(n_bins, np.float64)
    n_quant = n_ok = 0
    col = {2: 0, 4: 1, 8: 2}
    for t in range(S.size):
        i = bin_index(S[t], theta_fp, n_bins)
        if i < 0:
            n_ok += 1
            continue
        n_quant += 1
        eps = D_acc / (S[t] + eta)
        e = err[t, col[phi(S[t], t24, t48)]]
        if e <= eps:
            n_ok += 1
        worst[i] = max(worst[i], e / eps)
    return Audit(int(S.size), n_quant, n_ok, worst)
