"""Pins for the oracle's quantizer (O1-O3) and pack/act-quant (O4-O5).

Each pin is something other than the oracle itself: SPEC worked examples
(tests/golden/spec_quantcore.json), exact rational arithmetic (fractions),
the reconstruction bound of S:81 (sharpened, reading 2), monotone
error in bits, determinism.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_quantcore.json")))


@pytest.mark.parametrize("case", GOLD["affine_params"], ids=lambda c: c["cite"])
def test_spec_affine_params(case):
    s, z = oracle.quant_fit(case["x"], case["bits"])
    assert z == case["zero_point"]
    if "scale" in case:
        assert s == case["scale"]
    else:  # stored scale = fp32(fp64 scale)
        assert s == float(np.float32(case["scale_f64"]))


def test_spec_z128_needs_fp64_fit():
    # z = 128 = round-half-up(127.5); an fp32 fit gives -min/s = 127.49999 -> 127
    s32 = np.float32(2.0) / np.float32(255.0)
    assert np.floor(np.float32(1.0) / s32 + np.float32(0.5)) == 127  # the fp32 hazard
    assert oracle.quant_fit([-1.0, 1.0], 8)[1] == 128


@pytest.mark.parametrize("case", GOLD["quantize"], ids=lambda c: c["cite"])
def test_spec_quantize(case):
    q = oracle.quantize(case["x"], case["scale"], case["zero_point"], case["bits"])
    assert q.tolist() == case["q"]


@pytest.mark.parametrize("case", GOLD["dequantize"], ids=lambda c: c["cite"])
def test_spec_dequantize(case):
    xh = oracle.dequantize(case["q"], case["scale"], case["zero_point"])
    assert xh.tolist() == case["xhat"]


@pytest.mark.parametrize("case", GOLD["fake_quant"], ids=lambda c: c["cite"])
def test_spec_fake_quant(case):
    assert oracle.fake_quant(case["x"], case["bits"]).tolist() == case["xhat"]


def test_floor_is_exact_rational_floor():
    """Eq. (2)'s floor(X/s) on fp32 operands equals the exact rational floor."""
    rng = np.random.default_rng(7)
    v = rng.standard_normal(20000).astype(np.float32) * np.float32(3.0)
    s = np.abs(rng.standard_normal(20000)).astype(np.float32) * np.float32(0.05) + np.float32(1e-3)
    # include exact multiples k*s (rounded to fp32) and one-ulp neighbours
    k = rng.integers(-100, 100, size=2000).astype(np.float32)
    mult = (k * s[:2000]).astype(np.float32)
    v[:2000] = mult
    v[2000:4000] = np.nextafter(mult, np.float32(np.inf))
    v[4000:6000] = np.nextafter(mult, np.float32(-np.inf))
    for i in range(v.size):
        q = oracle.quantize([float(v[i])], float(s[i]), 128, 8)[0]
        exact = Fraction(float(v[i])) / Fraction(float(s[i]))
        fl = exact.numerator // exact.denominator
        assert q == min(max(fl + 128, 0), 255), (v[i], s[i])


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_reconstruction_bound(bits):
    """S:81 bound, sharpened: -s/2 <= x - xhat <= s for in-range x.
    The upper side is the floor step; the lower side comes from the lower
    clamp when z rounds up (fp64 evaluation, 2^-20 slack)."""
    rng = np.random.default_rng(bits)
    worst_hi, worst_lo = 0.0, 0.0
    for trial in range(3000):
        kind = trial % 3
        x = rng.standard_normal(64) * rng.lognormal(0, 2)
        if kind == 1:
            x = np.abs(x)  # all-positive group: breaks SPEC's literal fit (C5)
        elif kind == 2:
            x = -np.abs(x) + rng.uniform(-0.1, 0.1)
        x = x.astype(np.float32).astype(np.float64)
        s, z = oracle.quant_fit(x, bits)
        q = oracle.quantize(x, s, z, bits)
        xh = oracle.dequantize(q, s, z)
        e = (x - xh) / s
        worst_hi = max(worst_hi, float(e.max()))
        worst_lo = min(worst_lo, float(e.min()))
        assert np.all(e <= 1.0 + 2.0 ** -20), (bits, e.max())
        assert np.all(e >= -0.5 - 2.0 ** -20), (bits, e.min())
        # zero maps to an exact code (padding-safe, reading 2)
        assert oracle.quantize([0.0], s, z, bits)[0] == z
    assert worst_hi > 0.9  # the bound is tight (floor)


def test_error_monotone_in_bits():
    """mean ||x - fake_quant(x,b)|| strictly decreases 2 -> 4 -> 8."""
    rng = np.random.default_rng(0)
    errs = {b: [] for b in (2, 4, 8)}
    for _ in range(1000):
        x = rng.standard_normal(64)
        for b in errs:
            errs[b].append(np.linalg.norm(x - oracle.fake_quant(x, b)))
    m = {b: np.mean(v) for b, v in errs.items()}
    assert m[2] > m[4] > m[8] > 0


def test_determinism():
    w = synth.weights_bf16(32, 128, seed=3)
    a = oracle.pack_weights(w, 64, 4)
    b = oracle.pack_weights(w, 64, 4)
    for f in ("q", "s", "z", "sumq"):
        assert np.array_equal(getattr(a, f), getattr(b, f))


def test_nonfinite_rejected_with_index():
    x = synth.activations_bf16(2, 128, seed=1)
    x[1, 77] = 0x7FC0  # bf16 NaN
    with pytest.raises(oracle.OracleError) as ei:
        oracle.act_quant(x, 64, 8)
    assert ei.value.code == 4 and ei.value.index == 128 + 77


@pytest.mark.parametrize("wbits", [4, 8])
def test_pack_is_groupwise_fit(wbits):
    """O4 = O1+O2 on each (row, group): pinned by the dequantization bound per group
    and the code range; sumq is the plain sum of codes."""
    N, K, G = 16, 256, 64
    w = synth.weights_bf16(N, K, seed=5)
    p = oracle.pack_weights(w, G, wbits)
    wf = synth.bf16_bits_to_f32(w).astype(np.float64)
    assert p.q.max() <= 2 ** wbits - 1
    assert np.array_equal(p.sumq, p.q.reshape(N, K // G, G).astype(np.int32).sum(-1))
    for n in range(N):
        for g in range(K // G):
            s, z = float(p.s[n, g]), int(p.z[n, g])
            xh = s * (p.q[n, g * G:(g + 1) * G].astype(np.float64) - z)
            e = (wf[n, g * G:(g + 1) * G] - xh) / s
            assert e.max() <= 1.0 + 2 ** -20 and e.min() >= -0.5 - 2 ** -20
            # the group's extreme values reach the ends of the code range
            lo, hi = min(0.0, wf[n, g * G:(g + 1) * G].min()), max(0.0, wf[n, g * G:(g + 1) * G].max())
            assert abs((hi - lo) / (2 ** wbits - 1) - s) <= abs(s) * 2 ** -23


def test_act_quant_a16_rows_pass_through():
    x = synth.activations_bf16(3, 128, seed=2)
    aq = oracle.act_quant(x, 64, [8, 16, 2])
    assert np.all(aq.xq[1] == 0) and np.all(aq.s[1] == 0)
    assert aq.xq[0].max() <= 255 and aq.xq[2].max() <= 3
    assert np.array_equal(aq.SX, aq.xq.reshape(3, 2, 64).astype(np.int32).sum(-1))


# ---------------------------------------------------------------- round_mode=1
# DESIGN.md reading 1: Eq. (2) prints a floor; round_mode = 1 is the
# nearest-integer option, floor(v / s + 1/2).  Pins: hand-computed halves on an
# exactly representable grid, the exact rational definition, and the fixed-grid
# round trip that holds for nearest rounding but not for floor.

def test_nearest_mode_hand_cases():
    # s = 0.25 (exact), z = 4, 4 bits: v / s = 2, 2.5, 1.5, -0.5, -1.5, 9.999.., 100
    v = [0.5, 0.625, 0.375, -0.125, -0.375, 2.4999, 25.0]
    assert oracle.quantize(v, 0.25, 4, 4, round_mode=1).tolist() == [6, 7, 6, 4, 3, 14, 15]
    assert oracle.quantize(v, 0.25, 4, 4, round_mode=0).tolist() == [6, 6, 5, 3, 2, 13, 15]


def test_nearest_mode_is_exact_rational_rounding():
    rng = np.random.default_rng(17)
    for _ in range(200):
        s = float(np.float32(abs(rng.standard_normal()) * 0.05 + 1e-3))
        z = int(rng.integers(0, 16))
        v = (rng.standard_normal(64) * 0.3).astype(np.float32).astype(np.float64)
        # include exact half-way points (k + 1/2) * s where representable
        v[:8] = [float(np.float32((k + 0.5) * s)) for k in range(-4, 4)]
        q = oracle.quantize(v, s, z, 4, round_mode=1)
        for vi, qi in zip(v, q):
            r = Fraction(vi) / Fraction(s) + Fraction(1, 2)
            want = min(max(int(r.__floor__()) + z, 0), 15)
            assert qi == want


def test_nearest_mode_fixed_grid_round_trip():
    """q(s (q - z)) == q on the fixed grid with an fp32 x-hat in nearest mode;
    floor mode misses it for a large share of codes (App. A item 6)."""
    rng = np.random.default_rng(23)
    miss_floor = 0
    for _ in range(300):
        v = (rng.standard_normal(64) * 0.2).astype(np.float32).astype(np.float64)
        s, z = oracle.quant_fit(v, 4)
        q = oracle.quantize(v, s, z, 4, round_mode=1)
        xh32 = oracle.dequantize(q, s, z).astype(np.float32).astype(np.float64)
        assert np.array_equal(oracle.quantize(xh32, s, z, 4, round_mode=1), q)
        miss_floor += int(np.any(oracle.quantize(xh32, s, z, 4, round_mode=0) != q))
    assert miss_floor > 30


def test_nearest_mode_reconstruction_bound():
    """Nearest rounding halves the S:81 bound: |x - xhat| <= s / 2 (+ fp32
    rounding of xhat) for every x inside the zero-inclusive range."""
    rng = np.random.default_rng(29)
    for bits in (2, 4, 8):
        for _ in range(200):
            v = (rng.standard_normal(64) * rng.uniform(0.01, 3)).astype(np.float32).astype(np.float64)
            s, z = oracle.quant_fit(v, bits)
            xh = oracle.dequantize(oracle.quantize(v, s, z, bits, round_mode=1), s, z)
            assert np.all(np.abs(v - xh) <= 0.5 * s * (1 + 2 ** -20) + 1e-30)
